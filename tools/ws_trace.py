"""Per-band timeline of the latency kernel (library built with -DFGM_WS_TRACE):
one C3 solve, then the top level's bands (the last sweep launch).  Usage:
FGMATTE_B200_LIB=_exp/wstrace.so python tools/ws_trace.py"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2006_14970_b200 as fgm  # noqa: E402
from paper_2006_14970_b200 import synth  # noqa: E402

img, a = synth.make_config(synth.C3, device="cuda")
p = fgm.BASELINE_PARAMS
for _ in range(2):
    fgm.ml_foreground_background_cuda(img, a, p)
torch.cuda.synchronize()
L = fgm._load()
buf = (C.c_ulonglong * (8 * 4096))()
L.fgm_debug_ws_trace(buf, 8 * 4096)
t = np.array(buf, dtype=np.float64).reshape(4096, 8)
nb = 128
t = t[:nb]
t0 = t[:, 0].min()
t = (t - t0) / 1e3  # us
print("band  start  chunk0  step64  step512   end   prod_start prod64 prod512")
for q in list(range(0, 8)) + list(range(60, 64)) + list(range(120, 128)):
    print(f"{q:4d} " + " ".join(f"{v:8.1f}" for v in t[q]))
d = np.diff(t[:, 1])
print("chunk0 lag between bands: median %.2f us, mean %.2f" % (np.median(d[1:]), d[1:].mean()))
print("band duration (end - chunk0): median %.1f us" % np.median(t[1:, 4] - t[1:, 1]))
print("step64 -> step512 (448 steps): median %.1f us" % np.median(t[:, 3] - t[:, 2]))
print("producer step64 -> step512: median %.1f us; producer lead at 512 over chain: median %.1f us" % (np.median(t[:, 7] - t[:, 6]), np.median(t[:, 3] - t[:, 7])))
