"""Quick GPU parity + timing probe (development aid; not part of the bench)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import oracle  # noqa: E402
import paper_2006_14970_b200 as fgm  # noqa: E402
from paper_2006_14970_b200 import synth  # noqa: E402

dev = torch.device("cuda:0")
O = oracle.oracle()
P = fgm.BASELINE_PARAMS
OP = oracle.Params(P.omega, P.eps_r, P.low_res_threshold, P.iters_low, P.iters_high)


def cmp(name, a, b):
    d = np.abs(a - b)
    print(f"  {name}: max {d.max():.3g} mean {d.mean():.3g}", flush=True)
    return d.max()


# 1) single-level sweeps vs oracle (random level inputs)
rng = np.random.default_rng(0)
for (w, h, K) in [(37, 29, 1), (64, 64, 2), (100, 70, 3), (65, 33, 2), (130, 97, 4), (50, 40, 8), (33, 200, 10), (1, 50, 2), (50, 1, 2)]:
    img = rng.random((3, h, w), dtype=np.float32)
    a = rng.random((h, w), dtype=np.float32)
    f0 = rng.random((3, h, w), dtype=np.float32)
    b0 = rng.random((3, h, w), dtype=np.float32)
    of, ob = O.sweep(img.astype(np.float64), a.astype(np.float64), f0.astype(np.float64), b0.astype(np.float64), OP, K)
    t = lambda x: torch.from_numpy(x).to(dev)
    gf, gb = fgm.sweep_passes_cuda(t(img), t(a), t(f0), t(b0), K, P.eps_r, P.omega)
    torch.cuda.synchronize()
    print(f"sweep {w}x{h} K={K}")
    cmp("fg", gf.cpu().double().numpy(), of)
    cmp("bg", gb.cpu().double().numpy(), ob)

# 2) full solves vs oracle
for (w, h) in [(1, 1), (5, 3), (45, 45), (64, 64), (200, 136), (333, 517), (512, 512)]:
    img, a = synth.make_composite(w, h, 7 + w, 4, 3.0)
    gf, gb = fgm.ml_foreground_background_cuda(img.to(dev), a.to(dev), P)
    torch.cuda.synchronize()
    of, ob = O.ml_solve(img.double().numpy(), a.double().numpy(), OP)
    print(f"ml {w}x{h}")
    cmp("fg", gf.cpu().double().numpy(), of)
    cmp("bg", gb.cpu().double().numpy(), ob)

# 3) timing
for cfg in [synth.C1, synth.C2, synth.C3]:
    img, a = synth.make_config(cfg, device="cuda")
    for _ in range(3):
        fgm.ml_foreground_background_cuda(img, a, P)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n = 5
    for _ in range(n):
        fgm.ml_foreground_background_cuda(img, a, P)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    with fgm.profile():
        fgm.ml_foreground_background_cuda(img, a, P)
        torch.cuda.synchronize()
    st = fgm.profile.stats()
    print(f"{cfg.name}: {ms:.3f} ms/solve  {cfg.width * cfg.height / ms / 1e3:.1f} MP/s  {st}", flush=True)

# 4) batch (config 4)
t0 = time.time()
batch = synth.make_batch(device="cuda")
torch.cuda.synchronize()
print(f"batch generated in {time.time()-t0:.1f}s, {sum(x[0].shape[1]*x[0].shape[2] for x in batch)/1e6:.1f} MP", flush=True)
imgs = [b[0] for b in batch]
alps = [b[1] for b in batch]
outs = fgm.batch_solve_cuda(imgs, alps, P)
for _ in range(2):
    fgm.batch_solve_cuda(imgs, alps, P, outputs=outs)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    fgm.batch_solve_cuda(imgs, alps, P, outputs=outs)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
mp = sum(x.shape[1] * x.shape[2] for x in imgs) / 1e6
with fgm.profile():
    fgm.batch_solve_cuda(imgs, alps, P, outputs=outs)
    torch.cuda.synchronize()
st = fgm.profile.stats()
sw = st["sweep"]
print(f"c4 batch: {ms:.2f} ms  {mp / ms * 1e3:.0f} MP/s  sweep {sw['ms']:.2f} ms {sw['alg_bytes']/sw['ms']/1e6:.0f} GB/s  {st}", flush=True)
# spot-check parity of a few batch members
for i in [0, 1, 2]:
    of, ob = O.ml_solve(imgs[i].double().cpu().numpy(), alps[i].double().cpu().numpy(), OP)
    print(f"batch[{i}] {tuple(imgs[i].shape)}")
    cmp("fg", outs[i][0].cpu().double().numpy(), of)
    cmp("bg", outs[i][1].cpu().double().numpy(), ob)
