"""Benchmark: megapixels/s of the full multi-level F/B solve (BASELINE.json's
metric) on config 4 -- one batch of 256 synthetic images with sizes drawn from
{768x512, 1024^2, 2048x1536, 3000x2000} -- at BASELINE params
(regularization 1e-5, gradient_weight 1, 10 small / 2 big iterations,
small_size 32).  One step = one multi-level solve of every image of this
rank's shard; with N GPUs the batch is split by LPT on pixel count (strong
scaling, BASELINE configs[3]: "sharded by image across 1/2/4/8 GPUs with no
inter-GPU traffic"); `--scaling weak` gives every rank its own 256 images.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`--gpus N` without a torchrun environment re-launches itself under
torch.distributed.run with N processes (one per GPU, 127.0.0.1).

Prints ONE JSON line on rank 0.  `value` is device-timed (CUDA events on the
solve stream, inputs resident in HBM, max over ranks); `e2e` is the same
metric through the C ABI's host-buffer batch entry point with pinned host
buffers (H2D of image+alpha and D2H of F+B inside the timed region);
`roofline` is the big-level sweep kernel (K3), the dominant kernel, against
the measured HBM copy bandwidth; `parity` compares the whole timed batch with
the unmodified reference (oracle/_ref) run on the same inputs, whose run time
is also the `cpu_baseline`; `configs` times BASELINE's single-image configs
C1, C2, C3 and C5 (N = 1).  `--impl reference` times the reference CPU path
alone (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "megapixels/sec full multi-level F/B solve; sweep-kernel HBM GB/s vs roofline"
UNIT = "MP/s"
PARAMS = dict(omega=1.0, eps_r=1e-5, low_res_threshold=32, iters_low=10, iters_high=2)
ALG_BYTES_PER_PX_PASS = 64  # K3: alpha 4 + I 12 + initial F/B 24 read, F/B 24 written
TOL_MAX, TOL_MEAN = 1e-3, 1e-5


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def relaunch_distributed(nproc: int) -> int:
    """Re-run this script under torch.distributed.run with nproc ranks."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


class Clocks:
    """SM clocks and throttle reasons sampled during the timed region
    (B200_PROFILING.md clocks line): NVML every 20 ms, else nvidia-smi."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits: hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
    BITS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
            ("sw_power_cap", 0x4))

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.samples = []
        self.stop = threading.Event()
        self.t = threading.Thread(target=self.run, daemon=True)
        self.nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(gpu_index))
        except Exception:
            self.nvml = None

    def sample_nvml(self):
        nv, h = self.nvml
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        try:
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:
            r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        self.samples.append([str(sm), str(mx), ""] + ["Active" if r & b else "Not Active" for _, b in self.BITS])

    def run(self):
        while not self.stop.is_set():
            try:
                if self.nvml:
                    self.sample_nvml()
                else:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.02 if self.nvml else 0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def config_block(sizes, shard_mp, world, scaling):
    from paper_2006_14970_b200 import synth

    batch_mp = sum(w * h for w, h in sizes) / 1e6
    weak = scaling == "weak"
    return {
        "workload": "C4: batch of 256 synthetic composites, sizes U{768x512,1024x1024,2048x1536,3000x2000} "
                    "(BASELINE.json configs[3]); multi-level solve per image",
        "images": len(sizes) * (world if weak else 1),
        "megapixels": round(batch_mp * (world if weak else 1), 3),
        "megapixels_this_rank": round(shard_mp, 3),
        "params": PARAMS,
        "seed": synth.BASE_SEED,
        "l2": "inputs larger than L2 (>9.8 GB of image+alpha per step vs 126 MB L2); no flush needed",
        "sharding": ("weak: every rank solves its own 256-image C4 batch (same sizes, image seeds offset by "
                     "rank*256), no data-path collective" if weak else
                     "strong: one 256-image batch split across ranks by LPT on pixel count, no data-path "
                     "collective"),
    }


def reference_batch(images, alphas, nthreads, outputs):
    """The unmodified reference (oracle/_ref, fgmatte::ml_foreground_background
    in fp64) over a list of fp32 (3,H,W) numpy images on a host thread pool."""
    import oracle

    ref = oracle.reference()
    return ref.ml_solve_batch_f32(images, alphas, oracle.Params(**PARAMS), nthreads=nthreads, outputs=outputs)


def run_reference(args, rank, world):
    """--impl reference: the reference CPU implementation on this host."""
    if rank != 0:
        return
    from paper_2006_14970_b200 import synth

    sizes = synth.c4_sizes()
    nthreads = os.cpu_count() or 1
    n = min(len(sizes), max(8, 2 * nthreads))
    batch = synth.make_batch(n, device="cpu", sizes=sizes)  # a bounded sample of the batch per step
    images = [b[0].numpy() for b in batch]
    alphas = [b[1].numpy() for b in batch]
    mp = sum(sizes[i][0] * sizes[i][1] for i in range(n)) / 1e6
    times = []
    for i in range(args.warmup + args.steps):
        secs, _, _ = reference_batch(images, alphas, nthreads, False)
        if i >= args.warmup:
            times.append(secs)
    ms = statistics.median(times) * 1e3
    value = mp / (ms / 1e3)
    desc = (f"first {n} images of the C4 batch ({mp:.1f} MP) per step, reference fgmatte::ml_foreground_background "
            f"fp64 on {nthreads} host threads (thread pool, largest first)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(sizes, sum(w * h for w, h in sizes) / 1e6, 1, args.scaling),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": "reference", "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def k3_stats(stats, steps):
    sw = stats["sweep"]
    achieved = sw["alg_bytes"] / (sw["ms"] / 1e3) / 1e9 if sw["ms"] > 0 else 0.0
    return achieved, sw["ms"] / max(steps, 1), sw["launches"] / max(steps, 1)


def time_configs(fgm, synth, torch, dev, peak):
    """BASELINE's single-image configs (C1, C2, C3, C5), device-resident, median
    of several solves after warm-up (C5: 3), with the K3 roofline fraction."""
    out = {}
    for cfg, reps in ((synth.C1, 20), (synth.C2, 10), (synth.C3, 10), (synth.C5, 3)):
        img, a = synth.make_config(cfg, device=str(dev))
        p = fgm.Params(**{**PARAMS, "iters_high": cfg.iters_high})
        fg, bg = torch.empty_like(img), torch.empty_like(img)
        for _ in range(2):
            fgm.ml_foreground_background_cuda(img, a, p)
        torch.cuda.synchronize(dev)
        ms = []
        with fgm.profile():
            for _ in range(reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fg, bg = fgm.ml_foreground_background_cuda(img, a, p)
                e1.record()
                torch.cuda.synchronize(dev)
                ms.append(e0.elapsed_time(e1))
            st = fgm.profile.stats()
        achieved, k3_ms, _ = k3_stats(st, reps)
        med = statistics.median(ms)
        mp = cfg.width * cfg.height / 1e6
        out[cfg.name] = {"size": f"{cfg.width}x{cfg.height}", "iters_high": cfg.iters_high,
                         "ms_per_solve": round(med, 4), "mp_per_s": round(mp / (med / 1e3), 1),
                         "k3_ms": round(k3_ms, 4), "k3_gbs": round(achieved, 1),
                         "k3_roofline_frac": round(achieved / peak, 4), "reps": reps,
                         "k3_kernel": "latency kernel (sweep_ws.cu: one warp-specialised CTA per 32-row band): a single image is chain-bound"}
        del img, a, fg, bg
        torch.cuda.empty_cache()
    return out


def run_ours(args, rank, world, local):
    import numpy as np
    import torch

    import paper_2006_14970_b200 as fgm
    from paper_2006_14970_b200 import shard, synth

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    params = fgm.Params(**PARAMS)
    sizes = synth.c4_sizes()
    if args.scaling == "weak":
        mine = list(range(len(sizes)))
        seed_of = lambda i: synth.BASE_SEED + 1000 + rank * len(sizes) + i  # noqa: E731
        total_mp = world * sum(w * h for w, h in sizes) / 1e6
    else:
        mine = shard.lpt_partition(sizes, world)[rank]
        seed_of = lambda i: synth.BASE_SEED + 1000 + i  # noqa: E731
        total_mp = sum(w * h for w, h in sizes) / 1e6
    my_sizes = [sizes[i] for i in mine]
    my_mp = shard.shard_pixels(sizes, mine) / 1e6

    # inputs resident in HBM (generated on the device from the per-image seeds)
    imgs, alps = [], []
    for i in mine:
        w, h = sizes[i]
        im, al = synth.make_composite(w, h, seed_of(i), 5, 4.0, False, device=str(dev))
        imgs.append(im)
        alps.append(al)
    outs = [(torch.empty_like(x), torch.empty_like(x)) for x in imgs]
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        fgm.batch_solve_cuda(imgs, alps, params, outputs=outs)
    # fill the profiler's event pool with as many events as the timed steps use,
    # so no event is created inside the timed region
    with fgm.profile():
        for _ in range(args.steps):
            fgm.batch_solve_cuda(imgs, alps, params, outputs=outs)
        torch.cuda.synchronize(dev)
    barrier()

    # ---- device-timed steps (K3 launches bracketed by events for the roofline)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        with fgm.profile():
            barrier()
            e0.record(stream)
            for _ in range(args.steps):
                fgm.batch_solve_cuda(imgs, alps, params, outputs=outs)
            e1.record(stream)
            barrier()
        stats = fgm.profile.stats()
    ms_local = e0.elapsed_time(e1) / args.steps
    ms = shard.max_over_ranks(ms_local, dev)
    value = total_mp / (ms / 1e3)

    # ---- end to end through the host-buffer C-ABI entry point
    h_imgs = [x.cpu().pin_memory() for x in imgs]
    h_alps = [x.cpu().pin_memory() for x in alps]
    h_outs = [(torch.empty(x.shape, pin_memory=True), torch.empty(x.shape, pin_memory=True)) for x in h_imgs]
    fgm.batch_solve_host(h_imgs, h_alps, params, outputs=h_outs)  # warm-up (allocations, staging)
    e2e_steps = max(3, args.steps)
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        fgm.batch_solve_host(h_imgs, h_alps, params, outputs=h_outs)
    barrier()
    e2e_s = shard.max_over_ranks((time.perf_counter() - t0) / e2e_steps, dev)
    h2d = sum(16 * w * h for w, h in my_sizes)
    d2h = sum(24 * w * h for w, h in my_sizes)

    # ---- roofline of the dominant kernel (K3 sweep): all its launches of a step
    peak, peak_kind = peaks()
    achieved, k3_ms, k3_launches = k3_stats(stats, args.steps)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "sweep_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tj = json.load(f)
        traffic = tj.get("dram_bytes_per_step")
    launches = int((sum(v["launches"] for v in stats.values()) + stats["sweep"]["launches"]) // max(args.steps, 1))

    # ---- parity of the whole timed batch against the reference, whose run is
    # also the CPU baseline (rank 0 at N = 1; the reference's host threads are
    # shared by all ranks of a node, so multi-rank runs skip it)
    parity = cpu = configs = None
    if rank == 0 and world == 1:
        nthreads = os.cpu_count() or 1
        try:
            h_img = [x.numpy() for x in h_imgs]
            h_alp = [x.numpy() for x in h_alps]
            secs, rf, rb = reference_batch(h_img, h_alp, nthreads, True)
            worst, total, n = 0.0, 0.0, 0
            for (gf, gb), f, b in zip(outs, rf, rb):
                for got, want in ((gf, f), (gb, b)):
                    d = np.abs(got.cpu().numpy().astype(np.float64) - want.astype(np.float64))
                    worst = max(worst, float(d.max()))
                    total += float(d.sum())
                    n += d.size
            parity = {"max_abs": worst, "mean_abs": total / n, "tol_max": TOL_MAX, "tol_mean": TOL_MEAN,
                      "ok": bool(worst <= TOL_MAX and total / n <= TOL_MEAN), "images": len(outs),
                      "against": "the unmodified reference (oracle/_ref: fgmatte::ml_foreground_background, fp64) "
                                 "on the same fp32 inputs, all 6 planes of every image of the timed batch"}
            cpu = {"value": my_mp / secs, "unit": UNIT, "cores": nthreads, "kind": "reference",
                   "sample": f"the whole C4 batch ({my_mp:.1f} MP, {len(outs)} images), reference fp64 on "
                             f"{nthreads} host threads (thread pool, largest first), {secs:.2f} s"}
            del rf, rb
        except Exception as exc:  # reference shim not built
            cpu = {"value": None, "unit": UNIT, "cores": nthreads, "kind": "reference",
                   "sample": f"unavailable: {exc}"}
        if not args.no_configs:
            del h_imgs, h_alps, h_outs
            configs = time_configs(fgm, synth, torch, dev, peak)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_block(sizes, my_mp, world, args.scaling),
            "e2e": {"value": total_mp / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "steps": e2e_steps, "entry": "fgm_batch_solve_host_f32 (C ABI, pinned host buffers)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if peak else None, "traffic": traffic,
                         "kernel": "sweep_kernel (K3), every launch of a step: the throughput kernel (sweep.cu, "
                                   "64-row bands, two rows per lane; batches)", "peak_kind": peak_kind,
                         "alg_bytes_per_px_pass": ALG_BYTES_PER_PX_PASS,
                         "scope": "achieved = sum of 64 B x level pixels over the step's K3 passes / sum of their "
                                  "CUDA-event durations; traffic = ncu dram__bytes_read+write summed over the same "
                                  "launches of one step (profiles/sweep_traffic.json)",
                         "kernel_ms_per_step": k3_ms, "kernel_launches_per_step": k3_launches},
            "kernel_ms_per_step": {k: v["ms"] / args.steps for k, v in stats.items()},
            "parity": parity,
            "cpu_baseline": cpu,
            "configs": configs,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_dry(args, rank, world):
    """--cpu-dry-run: the launch, rank and shard path of run_ours on CPU (gloo),
    without the GPU solve: every rank takes its LPT shard, the ranks check
    that the shards partition the batch, and a per-rank host timing of the
    shard's pixel sum goes through the same max-over-ranks reduction."""
    import torch
    import torch.distributed as dist

    from paper_2006_14970_b200 import shard, synth

    if world > 1:
        dist.init_process_group("gloo")
    sizes = synth.c4_sizes()
    mine = shard.lpt_partition(sizes, world)[rank] if args.scaling == "strong" else list(range(len(sizes)))
    got = [None] * world
    if world > 1:
        dist.all_gather_object(got, mine)
    else:
        got = [mine]
    t0 = time.perf_counter()
    px = shard.shard_pixels(sizes, mine)
    ms = shard.max_over_ranks((time.perf_counter() - t0) * 1e3)
    total_px = shard.sum_over_ranks(float(px))
    if rank == 0:
        covered = sorted(i for g in got for i in g)
        print(json.dumps({"dry_run": True, "metric": METRIC, "n_gpus": world, "scaling": args.scaling,
                          "shards": [len(g) for g in got], "partition_ok": covered == list(range(len(sizes))),
                          "megapixels": total_px / 1e6, "ms_max_over_ranks": ms,
                          "config": config_block(sizes, px / 1e6, world, args.scaling)}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    del torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                    help="strong (default): one 256-image batch split by LPT; weak: a 256-image batch per GPU")
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config block (C1, C2, C3, C5)")
    ap.add_argument("--cpu-dry-run", action="store_true", help="launch/rank/shard path only, on CPU (gloo)")
    args = ap.parse_args()
    rank, world, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_distributed(args.gpus))
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if args.cpu_dry_run:
        run_dry(args, rank, world)
    elif args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
