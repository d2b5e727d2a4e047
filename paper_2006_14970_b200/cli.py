"""`python -m paper_2006_14970_b200 <subcommand>`: the reference's command-line
tool (/root/reference/proj/tools/main.cpp) for the subcommands on the
multi-level path -- SURVEY.md 8(f) row f4.

  estimate  --image --alpha --out-fg [--out-bg] [--alpha-source] [--omega]
            [--eps-r] [--iters-low] [--iters-high] [--bits]      (main.cpp:79-110)
  compose   --fg|--image --alpha --bg|--bg-color --out [--naive]
            [--alpha-source] [--bits]                            (main.cpp:112-143)
  metrics   --est --gt --alpha [--sigma] [--csv]                 (main.cpp:145-170)
  bench     --image --alpha [--methods] [--sizes] [--reps] [--csv]
            [--mem-limit-gb] [--alpha-source]                    (main.cpp:194-267)

Exit codes as main.cpp:1-4: 0 success, 1 usage error, 2 I/O or input-data
error, 3 solver failure.  Output formats (the `time_s=` line, the metrics
`csv:` record, the bench CSV schema and `# skipped` trail) follow main.cpp.

Out of scope (not on the multi-level path): `--method
closedform` and `prep-dataset` are rejected as usage errors naming why;
`bench --methods ...,closedform` records each closed-form row as skipped in
the CSV trail, as the reference's memory guard does (main.cpp:218-227).

Every compute step runs on the GPU through the C-ABI library: the solve via
fgm_ml_solve_host_f64 (host fp64 planes in and out, as the reference's
ml_foreground_background), resize / compose / metrics via their kernels.
"""
from __future__ import annotations

import argparse
import math
import resource
import sys
import time
from typing import List, Optional

import numpy as np

from .png_io import PngError, load_alpha_png, load_png, save_png

EXIT_OK, EXIT_USAGE, EXIT_IO, EXIT_SOLVER = 0, 1, 2, 3
_OUT_OF_SCOPE = "is not part of this build (only the multi-level estimator path is; SURVEY.md section 8)"


class UsageError(Exception):
    pass


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # argparse's default exit status is 2; the reference's is 1
        self.print_usage(sys.stderr)
        sys.stderr.write(f"error: {message}\n")
        raise SystemExit(EXIT_USAGE)


def _g17(v: float) -> str:
    return f"{v:.17g}"


def _peak_rss_bytes() -> int:
    return int(resource.getrusage(resource.RUSAGE_SELF).ru_maxrss) * 1024  # KiB on Linux


def _load_color(path: str) -> np.ndarray:
    return load_png(path)[0]


def _require_rgb(planes: np.ndarray, path: str) -> np.ndarray:
    if planes.shape[0] != 3:
        raise PngError(f"{path} must be an RGB PNG (got {planes.shape[0]} channel)")
    return planes


def _dev(a: np.ndarray):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def _solve(image: np.ndarray, alpha: np.ndarray, **params):
    """Planar (3, H, W) fp64 image + (H, W) alpha -> planar fg, bg."""
    from . import ml_foreground_background

    fg, bg = ml_foreground_background(image.transpose(1, 2, 0), alpha, **params)
    return fg.transpose(2, 0, 1), bg.transpose(2, 0, 1)


def run_estimate(a) -> int:
    if a.method != "multilevel":
        raise UsageError(f"--method {a.method} {_OUT_OF_SCOPE}")
    image = _require_rgb(_load_color(a.image), a.image)
    alpha = load_alpha_png(a.alpha, a.alpha_source)
    h, w = image.shape[1:]
    print(f"method={a.method} image={w}x{h} omega={a.omega:g} eps_r={a.eps_r:g}", flush=True)
    t0 = time.perf_counter()
    fg, bg = _solve(image, alpha, omega=a.omega, eps_r=a.eps_r, iters_low=a.iters_low, iters_high=a.iters_high)
    print(f"time_s={time.perf_counter() - t0:.6f}", flush=True)
    save_png(a.out_fg, fg, a.bits)
    if a.out_bg:
        save_png(a.out_bg, bg, a.bits)
    return EXIT_OK


def run_compose(a) -> int:
    from . import compose_cuda

    if a.fg and a.image:
        raise UsageError("--fg excludes --image")
    if a.bg and a.bg_color is not None:
        raise UsageError("--bg excludes --bg-color")
    if not a.fg and not a.image:
        raise UsageError("compose needs --fg or --image")
    if a.naive and not a.image:
        raise UsageError("--naive composes the raw image; pass it via --image")
    if not a.bg and a.bg_color is None:
        raise UsageError("compose needs --bg or --bg-color")
    fg = _load_color(a.image if (a.naive or not a.fg) else a.fg)
    alpha = load_alpha_png(a.alpha, a.alpha_source)
    if a.bg:
        bg = _load_color(a.bg)
    else:
        bg = np.empty_like(fg)
        for c in range(fg.shape[0]):
            bg[c] = min(max(a.bg_color[0 if fg.shape[0] == 1 else c], 0.0), 1.0)
    if bg.shape[0] != fg.shape[0]:
        raise ValueError(f"compose: bg has {bg.shape[0]} channels, fg has {fg.shape[0]}")
    out = compose_cuda(_dev(fg), _dev(bg), _dev(alpha))  # compose_naive == compose (image.cpp:59-61)
    save_png(a.out, out.double().cpu().numpy(), a.bits)
    return EXIT_OK


def run_metrics(a) -> int:
    from . import evaluate_metrics_cuda

    est, gt = _load_color(a.est), _load_color(a.gt)
    alpha = load_alpha_png(a.alpha, "gray-png")
    r = evaluate_metrics_cuda(_dev(est), _dev(gt), _dev(alpha), sigma=a.sigma)
    print(f"sad={_g17(r['sad'])}\nmse={_g17(r['mse'])}\ngrad={_g17(r['grad'])}\n"
          f"translucent_pixels={r['translucent_pixel_count']}")
    record = f"{_g17(r['sad'])},{_g17(r['mse'])},{_g17(r['grad'])},{r['translucent_pixel_count']}"
    print(f"csv: sad,mse,grad,translucent_pixel_count\ncsv: {record}", flush=True)
    if a.csv:
        try:
            with open(a.csv, "w") as f:
                f.write(f"sad,mse,grad,translucent_pixel_count\n{record}\n")
        except OSError:
            raise PngError(f"cannot open {a.csv} for writing") from None
    return EXIT_OK


def run_bench(a) -> int:
    from . import resize

    if a.reps < 1:
        raise UsageError("--reps must be a positive number")
    for m in a.methods:
        if m not in ("multilevel", "closedform"):
            raise UsageError(f"unknown method {m}")
    base = _require_rgb(_load_color(a.image), a.image)
    base_alpha = load_alpha_png(a.alpha, a.alpha_source)
    bh, bw = base.shape[1:]
    if base_alpha.shape != (bh, bw):
        raise ValueError(f"bench: alpha size {base_alpha.shape[1]}x{base_alpha.shape[0]} does not match image size "
                         f"{bw}x{bh}")
    lines = ["width,height,megapixels,method,wall_time_s,repetitions,time_stddev_s,peak_rss_bytes"]
    skipped: List[str] = []
    for mp in a.sizes:
        scale = math.sqrt(mp * 1e6 / (bw * bh))
        w = max(1, int(math.floor(bw * scale + 0.5)))
        h = max(1, int(math.floor(bh * scale + 0.5)))
        image = resize(base.transpose(1, 2, 0), w, h).transpose(2, 0, 1)
        alpha = resize(base_alpha, w, h)
        for m in a.methods:
            if m == "closedform":
                why = f"closedform at {w}x{h}: {_OUT_OF_SCOPE}"
                print(f"skipped {why}", file=sys.stderr)
                skipped.append(why)
                continue
            times = []
            for _ in range(a.reps):
                t0 = time.perf_counter()
                _solve(image, alpha)
                times.append(time.perf_counter() - t0)
            mean = sum(times) / len(times)
            sd = math.sqrt(sum((t - mean) ** 2 for t in times) / (len(times) - 1)) if len(times) > 1 else 0.0
            lines.append(f"{w},{h},{_g17(w * h / 1e6)},{m},{_g17(mean)},{len(times)},{_g17(sd)},{_peak_rss_bytes()}")
            print(f"{w}x{h} {m}: {mean:.4f} s (stddev {sd:.4f}, reps {len(times)})", flush=True)
    lines += [f"# skipped {why}" for why in skipped]
    text = "\n".join(lines) + "\n"
    if a.csv:
        try:
            with open(a.csv, "w") as f:
                f.write(text)
        except OSError:
            raise PngError(f"cannot open {a.csv} for writing") from None
    else:
        sys.stdout.write(text)
    return EXIT_OK


def _csv_floats(n: Optional[int] = None):
    def parse(s: str):
        try:
            v = [float(x) for x in s.split(",")]
        except ValueError:
            raise argparse.ArgumentTypeError(f"expected comma-separated numbers, got {s!r}") from None
        if n is not None and len(v) != n:
            raise argparse.ArgumentTypeError(f"expected exactly {n} values, got {len(v)}")
        return v
    return parse


def _parser() -> argparse.ArgumentParser:
    p = _Parser(prog="python -m paper_2006_14970_b200",
                description="foreground/background color estimation for alpha mattes (B200)")
    sub = p.add_subparsers(dest="cmd", required=True)
    src = dict(choices=("gray-png", "alpha-channel"), default="gray-png")
    bits = dict(type=int, choices=(8, 16), default=16)

    e = sub.add_parser("estimate", help="estimate foreground and background colors")
    e.add_argument("--image", required=True)
    e.add_argument("--alpha", required=True)
    e.add_argument("--out-fg", required=True)
    e.add_argument("--out-bg", default="")
    e.add_argument("--method", choices=("multilevel", "closedform"), default="multilevel")
    e.add_argument("--alpha-source", **src)
    e.add_argument("--omega", type=float, default=0.1)
    e.add_argument("--eps-r", type=float, default=5e-3)
    e.add_argument("--iters-low", type=int, default=10)
    e.add_argument("--iters-high", type=int, default=2)
    e.add_argument("--eps-cf", type=float, default=None, help="closedform only (out of scope)")
    e.add_argument("--residual-tol", type=float, default=None, help="closedform only (out of scope)")
    e.add_argument("--bits", **bits)

    c = sub.add_parser("compose", help="compose a foreground onto a background")
    c.add_argument("--fg", default="")
    c.add_argument("--image", default="")
    c.add_argument("--alpha", required=True)
    c.add_argument("--bg", default="")
    c.add_argument("--bg-color", type=_csv_floats(3), default=None)
    c.add_argument("--out", required=True)
    c.add_argument("--naive", action="store_true")
    c.add_argument("--alpha-source", **src)
    c.add_argument("--bits", **bits)

    m = sub.add_parser("metrics", help="alpha-weighted SAD/MSE/GRAD")
    m.add_argument("--est", required=True)
    m.add_argument("--gt", required=True)
    m.add_argument("--alpha", required=True)
    m.add_argument("--sigma", type=float, default=1.4)
    m.add_argument("--csv", default="")

    b = sub.add_parser("bench", help="runtime scaling over a size ladder")
    b.add_argument("--image", required=True)
    b.add_argument("--alpha", required=True)
    b.add_argument("--methods", type=lambda s: s.split(","), default=["multilevel"])
    b.add_argument("--sizes", type=_csv_floats(), default=[0.0625, 0.25, 1.0, 4.0])
    b.add_argument("--reps", type=int, default=3)
    b.add_argument("--csv", default="")
    b.add_argument("--mem-limit-gb", type=float, default=4.0, help="closedform guard (closedform is out of scope)")
    b.add_argument("--alpha-source", **src)

    sub.add_parser("prep-dataset", help=f"white-point correction -- {_OUT_OF_SCOPE}", add_help=False)
    return p


def main(argv: Optional[List[str]] = None) -> int:
    """main.cpp:269-376 (parse, dispatch, map exceptions to exit codes)."""
    argv = sys.argv[1:] if argv is None else argv
    if argv[:1] == ["prep-dataset"]:
        sys.stderr.write(f"error: prep-dataset {_OUT_OF_SCOPE}\n")
        return EXIT_USAGE
    try:
        a = _parser().parse_args(argv)
    except SystemExit as e:
        return EXIT_OK if e.code in (0, None) else EXIT_USAGE
    run = {"estimate": run_estimate, "compose": run_compose, "metrics": run_metrics, "bench": run_bench}[a.cmd]
    try:
        return run(a)
    except UsageError as e:
        sys.stderr.write(f"error: {e}\n")
        return EXIT_USAGE
    except (PngError, ValueError) as e:  # PngError / std::invalid_argument
        sys.stderr.write(f"error: {e}\n")
        return EXIT_IO
    except Exception as e:  # SolverFailure and anything else: the solve did not complete
        sys.stderr.write(f"solver failure: {e}\n")
        return EXIT_SOLVER


if __name__ == "__main__":
    sys.exit(main())
