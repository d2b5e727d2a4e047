"""One warm-up solve + one measured solve of a config (for ncu capture)."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2006_14970_b200 as fgm  # noqa: E402
from paper_2006_14970_b200 import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
cfg = {"c1": synth.C1, "c2": synth.C2, "c3": synth.C3}[name]
img, a = synth.make_config(cfg, device="cuda")
for _ in range(2):
    fgm.ml_foreground_background_cuda(img, a, fgm.BASELINE_PARAMS)
torch.cuda.synchronize()
print("done", name)
