import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2006_14970_b200 as fgm, oracle
O = oracle.oracle(); p = oracle.Params()
for (w, h) in [(7, 100), (37, 65), (64, 97), (300, 33)]:
    rng = np.random.default_rng(w * 1000 + h)
    img = rng.random((3, h, w)).astype(np.float32); a = rng.random((h, w)).astype(np.float32)
    f0 = rng.random((3, h, w)).astype(np.float32); b0 = rng.random((3, h, w)).astype(np.float32)
    t = lambda x: torch.from_numpy(x).cuda()
    for K in (1, 2, 3, 4):
        of, ob = O.sweep(img.astype(np.float64), a.astype(np.float64), f0.astype(np.float64), b0.astype(np.float64), p, K)
        r = {}
        for kern in (1, 2):
            gf, gb = fgm.sweep_passes_cuda(t(img), t(a), t(f0), t(b0), K, p.eps_r, p.omega, kern)
            torch.cuda.synchronize()
            r[kern] = (gf.cpu().double().numpy(), gb.cpu().double().numpy())
        d1 = np.maximum(np.abs(r[1][0] - of), np.abs(r[1][1] - ob)); d2 = np.maximum(np.abs(r[2][0] - of), np.abs(r[2][1] - ob))
        d12 = np.maximum(np.abs(r[1][0] - r[2][0]), np.abs(r[1][1] - r[2][1]))
        idx = np.unravel_index(np.argmax(d1), d1.shape)
        print(f"{w}x{h} K={K}: ws {d1.max():.2e} thr {d2.max():.2e} ws-thr {d12.max():.2e} argmax(ws) {idx} rows>1e-6: {sorted(set(np.nonzero(d12>1e-6)[1].tolist()))[:12]}", flush=True)
