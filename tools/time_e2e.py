"""End-to-end C4 batch through the host-buffer C ABI (pinned host buffers),
as bench.py's e2e leg: MP/s per run.  Usage: time_e2e.py [reps]"""
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2006_14970_b200 as fgm  # noqa: E402
from paper_2006_14970_b200 import synth  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
batch = synth.make_batch(256, device="cpu")
imgs = [b[0].pin_memory() for b in batch]
alps = [b[1].pin_memory() for b in batch]
outs = [(torch.empty(x.shape, pin_memory=True), torch.empty(x.shape, pin_memory=True)) for x in imgs]
mp = sum(x.shape[1] * x.shape[2] for x in imgs) / 1e6
fgm.batch_solve_host(imgs, alps, fgm.BASELINE_PARAMS, outputs=outs)
for _ in range(reps):
    t0 = time.perf_counter()
    fgm.batch_solve_host(imgs, alps, fgm.BASELINE_PARAMS, outputs=outs)
    dt = time.perf_counter() - t0
    print(f"e2e {mp / dt:.0f} MP/s ({dt * 1e3:.1f} ms)", flush=True)
