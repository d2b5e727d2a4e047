"""Benchmark: megapixels/s of the full multi-level F/B solve (BASELINE.json's
metric) on config 4 -- the batch of 256 synthetic images with sizes drawn
from {768x512, 1024^2, 2048x1536, 3000x2000} -- at BASELINE params
(regularization 1e-5, gradient_weight 1, 10 small / 2 big iterations,
small_size 32).  One step = one multi-level solve of every image of this
rank's shard (LPT by pixel count; no data-path collective).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0.  `value` is device-timed (CUDA events on the
solve stream, inputs resident in HBM, max over ranks); `e2e` is the same
metric through the C ABI's host-buffer batch entry point with pinned host
buffers (H2D of image+alpha and D2H of F+B inside the timed region);
`roofline` is the big-level sweep kernel (K3), the dominant kernel, against
the measured HBM copy bandwidth; `cpu_baseline` is the unmodified reference
(oracle/_ref) on this host's cores over a bounded sample of the same batch.
`--impl reference` times that reference CPU path alone (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
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


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class Clocks:
    """SM clocks and throttle reasons sampled during the timed region
    (B200_PROFILING.md clocks line): NVML every 20 ms, else nvidia-smi."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits: sw_power_cap, hw_slowdown, sw_thermal, hw_thermal
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


def config_block(sizes, shard_mp, world=1, scaling="weak"):
    from paper_2006_14970_b200 import synth

    batch_mp = sum(w * h for w, h in sizes) / 1e6
    weak = scaling == "weak"
    return {
        "workload": "C4: batch of 256 synthetic composites, sizes U{768x512,1024x1024,2048x1536,3000x2000} "
                    "(BASELINE.json configs[3]); multi-level solve per image",
        "images": len(sizes) * (world if weak else 1),
        "images_per_rank": len(sizes) if weak else None,
        "megapixels": round(batch_mp * (world if weak else 1), 3),
        "megapixels_this_rank": round(shard_mp, 3),
        "params": PARAMS,
        "seed": synth.BASE_SEED,
        "l2": "inputs larger than L2 (>10 GB of image+alpha per step vs 126 MB L2); no flush needed",
        "sharding": ("weak: every rank solves its own 256-image C4 batch (same sizes, image seeds offset by "
                     "rank*256), no data-path collective" if weak else
                     "strong: one 256-image batch split across ranks by LPT on pixel count, no data-path collective"),
    }


def cpu_reference_sample(images, alphas, sizes, nthreads, target_images):
    """Time the unmodified reference (oracle/_ref) on a bounded sample of the
    batch with all host threads; returns (MP/s, seconds, sample description)."""
    import oracle

    ref = oracle.reference()
    n = min(len(images), target_images)
    imgs = [images[i] for i in range(n)]
    alps = [alphas[i] for i in range(n)]
    mp = sum(sizes[i][0] * sizes[i][1] for i in range(n)) / 1e6
    secs, _, _ = ref.ml_solve_batch_f32(imgs, alps, oracle.Params(**PARAMS), nthreads=nthreads)
    return mp / secs, secs, f"first {n} images of the C4 batch ({mp:.1f} MP), reference fgmatte::ml_foreground_" \
                            f"background fp64 on {nthreads} host threads (thread pool, largest first)"


def run_reference(args, rank, world):
    """--impl reference: the reference CPU implementation on this host."""
    if rank != 0:
        return
    from paper_2006_14970_b200 import synth

    sizes = synth.c4_sizes()
    nthreads = os.cpu_count() or 1
    n = min(len(sizes), max(8, 2 * nthreads))
    batch = synth.make_batch(n, device="cpu", sizes=sizes)  # the bounded sample only
    images = [b[0].numpy() for b in batch]
    alphas = [b[1].numpy() for b in batch]
    times = []
    for i in range(args.warmup + args.steps):
        v, secs, desc = cpu_reference_sample(images, alphas, sizes, nthreads, n)
        if i >= args.warmup:
            times.append((v, secs))
    value = statistics.median([v for v, _ in times])
    ms = statistics.median([s for _, s in times]) * 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(sizes, sum(w * h for w, h in sizes) / 1e6, 1, args.scaling),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": "reference", "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local):
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
        # the path partitions into independent images: every rank solves its
        # own C4 batch (per-GPU work fixed as N grows)
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
    e2e_steps = max(1, min(args.steps, 3))
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        fgm.batch_solve_host(h_imgs, h_alps, params, outputs=h_outs)
    barrier()
    e2e_s = shard.max_over_ranks((time.perf_counter() - t0) / e2e_steps, dev)
    h2d = sum(16 * w * h for w, h in my_sizes)
    d2h = sum(24 * w * h for w, h in my_sizes)

    # ---- roofline of the dominant kernel (K3 sweep)
    peak, peak_kind = peaks()
    sw = stats["sweep"]
    achieved = sw["alg_bytes"] / (sw["ms"] / 1e3) / 1e9 if sw["ms"] > 0 else 0.0
    traffic, issue = None, None
    tpath = os.path.join(ROOT, "profiles", "sweep_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tj = json.load(f)
        traffic = tj.get("dram_bytes_per_launch")
        if tj.get("sm_ipc"):  # the bound that actually binds K3
            issue = {"bound": "issue", "achieved": tj["sm_ipc"], "peak": tj["sm_ipc_peak"],
                     "unit": "warp-instructions/cycle/SM", "frac": tj["sm_ipc"] / tj["sm_ipc_peak"],
                     "source": "ncu --set full of the top-level K3 launch (profiles/sweep_traffic.json)"}
    # profiled kernels (sweep, resample/upsample, coarse) plus one sentinel
    # fill per sweep launch
    launches = int((sum(v["launches"] for v in stats.values()) + stats["sweep"]["launches"]) // max(args.steps, 1))

    # ---- CPU baseline: the unmodified reference on this host (rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1:
        try:
            nthreads = os.cpu_count() or 1
            n = min(len(imgs), max(8, 2 * nthreads))
            cv, _, desc = cpu_reference_sample([x.cpu().numpy() for x in imgs[:n]],
                                               [x.cpu().numpy() for x in alps[:n]], my_sizes, nthreads, n)
            cpu = {"value": cv, "unit": UNIT, "cores": nthreads, "kind": "reference", "sample": desc}
        except Exception as exc:  # reference shim not built
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_block(sizes, my_mp, world, args.scaling),
            "e2e": {"value": total_mp / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "entry": "fgm_batch_solve_host_f32 (C ABI, pinned host buffers)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if peak else None, "traffic": traffic,
                         "kernel": "sweep_kernel<2> (K3)", "peak_kind": peak_kind,
                         "alg_bytes_per_px_pass": 64,
                         "kernel_ms_per_step": sw["ms"] / args.steps,
                         "kernel_launches_per_step": sw["launches"] / args.steps,
                         "issue": issue},
            "kernel_ms_per_step": {k: v["ms"] / args.steps for k, v in stats.items()},
            "cpu_baseline": cpu,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                    help="weak: a 256-image C4 batch per GPU (default); strong: one batch split by LPT")
    args = ap.parse_args()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
