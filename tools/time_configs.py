"""Device time of one solve per BASELINE config (C1-C3, C5) and the C4 batch,
with the per-kind kernel split (development aid; the bench line is C4)."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2006_14970_b200 as fgm  # noqa: E402
from paper_2006_14970_b200 import synth  # noqa: E402

dev = torch.device("cuda:0")
which = sys.argv[1:] or ["1", "2", "3", "5"]
cfgs = {"1": synth.C1, "2": synth.C2, "3": synth.C3, "5": synth.C5}
for c in which:
    cfg = cfgs[c]
    img, a = synth.make_config(cfg, device="cuda")
    params = fgm.Params(omega=1.0, eps_r=1e-5, low_res_threshold=32, iters_low=10, iters_high=cfg.iters_high)
    mp = img.shape[1] * img.shape[2] / 1e6
    out = fgm.ml_foreground_background_cuda(img, a, params)
    reps = 1 if c == "5" else 5
    for _ in range(2 if c != "5" else 1):
        fgm.ml_foreground_background_cuda(img, a, params)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with fgm.profile():
        e0.record()
        for _ in range(reps):
            fgm.ml_foreground_background_cuda(img, a, params)
        e1.record()
        torch.cuda.synchronize()
    st = fgm.profile.stats()
    ms = e0.elapsed_time(e1) / reps
    print(f"C{c} {img.shape[2]}x{img.shape[1]}: {ms:.2f} ms/solve  {mp / ms * 1e3:.0f} MP/s  "
          f"sweep {st['sweep']['ms'] / reps:.2f} ms  resample {st['resample']['ms'] / reps:.2f} ms  "
          f"coarse {st['coarse']['ms'] / reps:.2f} ms", flush=True)
    del img, a, out
    torch.cuda.empty_cache()
