"""Warm-up + one batch solve of config 4 (for ncu capture of the sweep kernel).
Usage: prof_batch.py [n_images]"""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2006_14970_b200 as fgm  # noqa: E402
from paper_2006_14970_b200 import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
batch = synth.make_batch(n, device="cuda")
imgs = [b[0] for b in batch]
alps = [b[1] for b in batch]
outs = fgm.batch_solve_cuda(imgs, alps, fgm.BASELINE_PARAMS)
fgm.batch_solve_cuda(imgs, alps, fgm.BASELINE_PARAMS, outputs=outs)
torch.cuda.synchronize()
print("done", n)
