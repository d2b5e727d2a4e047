"""Device time of one single-level pass of each K3 kernel (1 latency, 2
throughput) on single images of the BASELINE sizes (development aid: the
kernel choice per launch shape; profiles/r02/k3_v2_notes.txt)."""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2006_14970_b200 as fgm  # noqa: E402

p = fgm.BASELINE_PARAMS
for (w, h, iters) in [(512, 512, 2), (1920, 1080, 2), (4096, 4096, 2), (8192, 8192, 4), (16384, 16384, 4)]:
    g = torch.Generator(device="cuda").manual_seed(1)
    img = torch.rand((3, h, w), device="cuda", generator=g)
    a = torch.rand((h, w), device="cuda", generator=g)
    f0 = torch.rand((3, h, w), device="cuda", generator=g)
    b0 = torch.rand((3, h, w), device="cuda", generator=g)
    res = []
    for kern in (1, 2):
        for _ in range(2):
            fgm.sweep_passes_cuda(img, a, f0, b0, iters, p.eps_r, p.omega, kern)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 3
        e0.record()
        for _ in range(n):
            fgm.sweep_passes_cuda(img, a, f0, b0, iters, p.eps_r, p.omega, kern)
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / n)
    print(f"{w}x{h} K={iters}: latency {res[0]:.3f} ms  throughput {res[1]:.3f} ms", flush=True)
    del img, a, f0, b0
    torch.cuda.empty_cache()
