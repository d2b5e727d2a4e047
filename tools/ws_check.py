"""Development aid: the warp-specialised latency kernel (3) against the
throughput kernel (2), bitwise, on single-level passes of ragged sizes."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2006_14970_b200 as fgm  # noqa: E402

fgm._load().fgm_set_spin_timeout_ms(300)
p = fgm.BASELINE_PARAMS
bad = 0
for (w, h, iters) in [(64, 40, 1), (64, 40, 2), (200, 136, 2), (37, 95, 2), (333, 129, 3), (257, 260, 4), (512, 512, 2),
                      (1000, 700, 6), (1920, 1080, 2), (33, 33, 2), (4, 70, 2), (70, 4, 4)]:
    g = torch.Generator(device="cuda").manual_seed(w * 7 + h)
    img = torch.rand((3, h, w), device="cuda", generator=g)
    a = torch.rand((h, w), device="cuda", generator=g)
    f0 = torch.rand((3, h, w), device="cuda", generator=g)
    b0 = torch.rand((3, h, w), device="cuda", generator=g)
    try:
        r2 = fgm.sweep_passes_cuda(img, a, f0, b0, iters, p.eps_r, p.omega, 2)
        r3 = fgm.sweep_passes_cuda(img, a, f0, b0, iters, p.eps_r, p.omega, 3)
        torch.cuda.synchronize()
        d = max((r2[0] - r3[0]).abs().max().item(), (r2[1] - r3[1]).abs().max().item())
        nb = int((r2[0] != r3[0]).sum().item() + (r2[1] != r3[1]).sum().item())
        print(f"{w}x{h} iters={iters}: max|d| {d:.3g}, differing words {nb}", flush=True)
        if nb:
            bad += 1
            idx = (r2[0] != r3[0]).nonzero()[:5].tolist()
            print("   first F diffs (c, y, x):", idx, flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"{w}x{h} iters={iters}: FAILED {e}", flush=True)
        bad += 1
print("faults:", fgm._load().fgm_device_faults(0))
sys.exit(1 if bad else 0)
