import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2006_14970_b200 as fgm
from paper_2006_14970_b200 import synth
p = fgm.BASELINE_PARAMS
for (w, h, K) in [(1920, 1080, 2), (960, 540, 2), (1920, 64, 2), (200, 1080, 2), (1920, 1080, 1), (512, 512, 2), (1024, 256, 2)]:
    rng = np.random.default_rng(w + h)
    img = rng.random((3, h, w)).astype(np.float32); a = rng.random((h, w)).astype(np.float32)
    f0 = rng.random((3, h, w)).astype(np.float32); b0 = rng.random((3, h, w)).astype(np.float32)
    t = lambda x: torch.from_numpy(x).cuda()
    r = {}
    for kern in (1, 2, 1):
        gf, gb = fgm.sweep_passes_cuda(t(img), t(a), t(f0), t(b0), K, p.eps_r, p.omega, kern)
        torch.cuda.synchronize()
        r.setdefault(kern, []).append((gf.cpu().numpy(), gb.cpu().numpy()))
    d = np.maximum(np.abs(r[1][0][0] - r[2][0][0]), np.abs(r[1][0][1] - r[2][0][1]))
    drep = np.maximum(np.abs(r[1][0][0] - r[1][1][0]), np.abs(r[1][0][1] - r[1][1][1]))
    bad = np.argwhere(d > 1e-6)
    print(f"{w}x{h} K={K}: ws-thr max {d.max():.2e} n>{1e-6}: {len(bad)} ws-ws(repeat) {drep.max():.2e} first bad (c,y,x): {bad[:6].tolist()}", flush=True)
