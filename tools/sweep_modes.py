"""Time the batch solve per sweep-kernel mode (0 auto, 1 per-channel, 2 full)."""
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
for mode in (1, 2, 0):
    fgm.set_sweep_mode(mode)
    for _ in range(2):
        fgm.batch_solve_cuda(imgs, alps, fgm.BASELINE_PARAMS, outputs=outs)
    torch.cuda.synchronize()
    with fgm.profile():
        fgm.batch_solve_cuda(imgs, alps, fgm.BASELINE_PARAMS, outputs=outs)
        torch.cuda.synchronize()
    st = fgm.profile.stats()
    print(f"mode {mode}: sweep {st['sweep']['ms']:.2f} ms ({st['sweep']['launches']} launches), resample "
          f"{st['resample']['ms']:.2f} ms", flush=True)
# per-launch breakdown in auto mode
import ctypes
fgm.set_sweep_mode(0)
