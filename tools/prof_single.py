"""Two single-level K = 2 passes of the latency kernel (sweep_ws.cu) on one square image, for ncu
(tools/profile_round.sh): python tools/prof_single.py [size]."""
import sys, torch
sys.path.insert(0, __file__.rsplit('/tools/', 1)[0])
import paper_2006_14970_b200 as fgm
p = fgm.BASELINE_PARAMS
w = h = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
g = torch.Generator(device="cuda").manual_seed(1)
img = torch.rand((3, h, w), device="cuda", generator=g); a = torch.rand((h, w), device="cuda", generator=g)
f0 = torch.rand((3, h, w), device="cuda", generator=g); b0 = torch.rand((3, h, w), device="cuda", generator=g)
for i in range(2):
    fgm.sweep_passes_cuda(img, a, f0, b0, 2, p.eps_r, p.omega, 1)
    torch.cuda.synchronize()
