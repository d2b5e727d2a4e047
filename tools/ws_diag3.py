import sys, numpy as np, torch, collections
sys.path.insert(0, '/root/repo')
import paper_2006_14970_b200 as fgm
p = fgm.BASELINE_PARAMS
for (w, h, K) in [(1920, 1080, 1), (1024, 256, 2), (1024, 256, 1), (1920, 96, 1)]:
    rng = np.random.default_rng(w + h)
    img = rng.random((3, h, w)).astype(np.float32); a = rng.random((h, w)).astype(np.float32)
    f0 = rng.random((3, h, w)).astype(np.float32); b0 = rng.random((3, h, w)).astype(np.float32)
    t = lambda x: torch.from_numpy(x).cuda()
    gf2, gb2 = fgm.sweep_passes_cuda(t(img), t(a), t(f0), t(b0), K, p.eps_r, p.omega, 2)
    ref = (gf2.cpu().numpy(), gb2.cpu().numpy())
    for rep in range(3):
        gf, gb = fgm.sweep_passes_cuda(t(img), t(a), t(f0), t(b0), K, p.eps_r, p.omega, 1)
        torch.cuda.synchronize()
        d = np.maximum(np.abs(gf.cpu().numpy() - ref[0]), np.abs(gb.cpu().numpy() - ref[1])).max(axis=0)
        bad = np.argwhere(d > 1e-6)
        if len(bad) == 0:
            print(f"{w}x{h} K={K} rep{rep}: ok", flush=True); continue
        ys = collections.Counter((bad[:, 0]).tolist()); xs16 = collections.Counter((bad[:, 1] % 16).tolist())
        first = bad[np.lexsort((bad[:, 1], bad[:, 0]))][:5].tolist()
        print(f"{w}x{h} K={K} rep{rep}: nbad {len(bad)} rows {sorted(ys)[:10]}.. nrows {len(ys)} x%16 {dict(xs16)} min x {bad[:,1].min()} first(y,x) {first}", flush=True)
