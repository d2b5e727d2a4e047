"""One warm-up + one solve of a BASELINE config (for ncu captures).
Usage: prof_config.py <1|2|3|5>"""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2006_14970_b200 as fgm  # noqa: E402
from paper_2006_14970_b200 import synth  # noqa: E402

cfg = {"1": synth.C1, "2": synth.C2, "3": synth.C3, "5": synth.C5}[sys.argv[1]]
img, a = synth.make_config(cfg, device="cuda")
params = fgm.Params(omega=1.0, eps_r=1e-5, low_res_threshold=32, iters_low=10, iters_high=cfg.iters_high)
for _ in range(2):
    fgm.ml_foreground_background_cuda(img, a, params)
torch.cuda.synchronize()
print("done")
