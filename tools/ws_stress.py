"""Stress check of the latency kernel (sweep_ws.cu, kernel 1) against the throughput kernel (kernel 2): seeded
random sizes, fused-sweep counts and parameters, single-level passes compared bitwise, each case repeated to catch
timing-dependent hand-over errors.  python tools/ws_stress.py [cases] [repeats]"""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2006_14970_b200 as fgm  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
rng = np.random.default_rng(20061497)
bad = 0
for i in range(cases):
    kind = i % 4
    if kind == 0:
        w, h = int(rng.integers(1, 80)), int(rng.integers(1, 80))
    elif kind == 1:
        w, h = int(rng.integers(1, 700)), int(rng.integers(1, 700))
    elif kind == 2:
        w, h = int(rng.integers(500, 3000)), int(rng.integers(20, 400))
    else:
        w, h = int(rng.integers(20, 400)), int(rng.integers(500, 3000))
    iters = int(rng.integers(1, 9))
    eps, omega = float(rng.choice([1e-5, 1e-3, 5e-3])), float(rng.choice([0.1, 1.0, 2.0]))
    g = torch.Generator(device="cuda").manual_seed(i)
    img = torch.rand((3, h, w), device="cuda", generator=g)
    a = torch.rand((h, w), device="cuda", generator=g)
    if i % 5 == 0:
        a = (a > 0.5).float()  # binary alpha: the ill-conditioned case
    f0 = torch.rand((3, h, w), device="cuda", generator=g)
    b0 = torch.rand((3, h, w), device="cuda", generator=g)
    ref = fgm.sweep_passes_cuda(img, a, f0, b0, iters, eps, omega, 2)
    for r in range(reps):
        out = fgm.sweep_passes_cuda(img, a, f0, b0, iters, eps, omega, 1)
        torch.cuda.synchronize()
        if not (torch.equal(out[0], ref[0]) and torch.equal(out[1], ref[1])):
            bad += 1
            print(f"case {i} rep {r}: {w}x{h} iters {iters} DIFFERS", flush=True)
            break
print(f"{cases} cases x {reps} repeats: {bad} differing; device faults {fgm.device_faults()}")

# batches of 2..4 images: latency-bound launches holding the bands of several jobs
from paper_2006_14970_b200 import synth  # noqa: E402

nb = max(cases // 10, 1)
badb = 0
for i in range(nb):
    n = int(rng.integers(2, 5))
    imgs, alps = [], []
    for j in range(n):
        w, h = int(rng.integers(1, 900)), int(rng.integers(1, 900))
        im, al = synth.make_composite(w, h, 5000 + 10 * i + j, 3, float(rng.uniform(1.0, 6.0)))
        imgs.append(im.cuda())
        alps.append(al.cuda())
    p = fgm.Params(omega=float(rng.choice([0.1, 1.0, 2.0])), eps_r=float(rng.choice([1e-5, 1e-3])),
                   low_res_threshold=int(rng.choice([16, 32, 64])), iters_low=int(rng.integers(1, 7)),
                   iters_high=int(rng.integers(1, 9)))
    outs = fgm.batch_solve_cuda(imgs, alps, p)
    for im, al, (f, b) in zip(imgs, alps, outs):
        f1, b1 = fgm.ml_foreground_background_cuda(im, al, p)
        if not (torch.equal(f, f1) and torch.equal(b, b1)):
            badb += 1
            print(f"batch {i}: image {tuple(im.shape)} differs from its single solve", flush=True)
print(f"{nb} small batches: {badb} differing images; device faults {fgm.device_faults()}")
sys.exit(1 if bad or badb else 0)
