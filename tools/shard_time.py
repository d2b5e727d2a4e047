"""Device time of one rank's LPT shard of the C4 batch at world size N (run on
one GPU: ranks share no data, so this is each rank's step time at N GPUs)."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2006_14970_b200 as fgm  # noqa: E402
from paper_2006_14970_b200 import shard, synth  # noqa: E402

sizes = synth.c4_sizes()
total = sum(w * h for w, h in sizes) / 1e6
for world in [int(x) for x in (sys.argv[1:] or ["1", "2", "4", "8"])]:
    parts = shard.lpt_partition(sizes, world)
    worst = 0.0
    for rank in range(world):
        mine = parts[rank]
        imgs, alps = [], []
        for i in mine:
            w, h = sizes[i]
            im, al = synth.make_composite(w, h, synth.BASE_SEED + 1000 + i, 5, 4.0, False, device="cuda")
            imgs.append(im)
            alps.append(al)
        outs = [(torch.empty_like(x), torch.empty_like(x)) for x in imgs]
        for _ in range(3):
            fgm.batch_solve_cuda(imgs, alps, fgm.BASELINE_PARAMS, outputs=outs)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            fgm.batch_solve_cuda(imgs, alps, fgm.BASELINE_PARAMS, outputs=outs)
        e1.record()
        torch.cuda.synchronize()
        worst = max(worst, e0.elapsed_time(e1) / 5)
        if world > 2 and rank >= 1:
            break  # LPT shards are balanced; rank 0 and 1 bound the max
    print(f"N={world}: max rank step {worst:.2f} ms -> {total / worst * 1e3:.0f} MP/s aggregate "
          f"(ideal {world} x single)", flush=True)
