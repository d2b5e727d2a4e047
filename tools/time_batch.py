"""Time the C4 batch solve (per-kind kernel ms) with the library named by
FGMATTE_B200_LIB (default: the in-tree build).  Usage: time_batch.py [n]"""
import os
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
for _ in range(2):
    fgm.batch_solve_cuda(imgs, alps, fgm.BASELINE_PARAMS, outputs=outs)
torch.cuda.synchronize()
res = []
for _ in range(3):
    with fgm.profile():
        fgm.batch_solve_cuda(imgs, alps, fgm.BASELINE_PARAMS, outputs=outs)
        torch.cuda.synchronize()
    st = fgm.profile.stats()
    res.append((st["sweep"]["ms"], st["resample"]["ms"], st["upsample"]["ms"]))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    fgm.batch_solve_cuda(imgs, alps, fgm.BASELINE_PARAMS, outputs=outs)
e1.record()
torch.cuda.synchronize()
lib = os.environ.get("FGMATTE_B200_LIB", "default")
print(f"{lib}: total {e0.elapsed_time(e1) / 3:.2f} ms  sweep {min(r[0] for r in res):.2f} ms  "
      f"resample {min(r[1] for r in res):.2f} ms  upsample {min(r[2] for r in res):.2f} ms", flush=True)
