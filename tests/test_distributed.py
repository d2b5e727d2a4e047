"""CPU, world_size 2 over gloo: the batch-sharding host logic of the multi-GPU
path (paper_2006_14970_b200/shard.py), as bench.py runs it under torchrun."""
import os
import socket

import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, sizes, q):
    import torch.distributed as dist

    from paper_2006_14970_b200 import shard

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = shard.lpt_partition(sizes, world)[rank]
        got = [None] * world
        dist.all_gather_object(got, mine)
        mx = shard.max_over_ranks(float(rank * 10 + 3))
        tot = shard.sum_over_ranks(float(shard.shard_pixels(sizes, mine)))
        q.put((rank, got, mx, tot))
    finally:
        dist.destroy_process_group()


def test_lpt_partition_properties():
    from paper_2006_14970_b200 import shard, synth

    sizes = synth.c4_sizes()
    for n in (1, 2, 4, 8):
        parts = shard.lpt_partition(sizes, n)
        flat = sorted(i for p in parts for i in p)
        assert flat == list(range(len(sizes)))
        loads = [shard.shard_pixels(sizes, p) for p in parts]
        biggest = max(w * h for w, h in sizes)
        assert max(loads) - min(loads) <= biggest
    with pytest.raises(ValueError):
        shard.lpt_partition(sizes, 0)


def test_gloo_world2_sharding():
    import torch.multiprocessing as mp

    from paper_2006_14970_b200 import shard, synth

    sizes = synth.c4_sizes()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, sizes, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    shards0 = res[0][1]
    assert shards0 == res[1][1]  # every rank agrees on the partition
    assert sorted(i for s in shards0 for i in s) == list(range(len(sizes)))
    assert res[0][2] == res[1][2] == 13.0  # max over ranks
    assert res[0][3] == sum(w * h for w, h in sizes)
    assert shards0 == shard.lpt_partition(sizes, 2)


def test_bench_rank_and_shard_path_world2():
    """bench.py's multi-GPU path end to end on CPU: `--gpus 2` re-launches
    itself under torch.distributed.run (127.0.0.1), both ranks take their LPT
    shards over gloo, the shards partition the 256-image batch, the timing
    goes through max-over-ranks, and rank 0's line reports n_gpus = 2."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--cpu-dry-run"],
                         capture_output=True, text=True, timeout=240, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["partition_ok"] and sum(d["shards"]) == 256
    assert abs(d["megapixels"] - d["config"]["megapixels"]) < 1e-3  # (config rounds to 3 decimals)
