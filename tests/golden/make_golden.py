"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref,
compiled from /root/reference/proj/src/{image,multilevel}.cpp).

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
Each fixture stores fp32-exact inputs (planar image (3,H,W), alpha (H,W)),
the parameters, the reference's fp64 outputs, and the reference's level
schedule.  The GPU tests compare against these without needing the reference.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2006_14970_b200 import synth  # noqa: E402

BASE = oracle.Params()  # BASELINE.json params: eps_r 1e-5, omega 1
DEF = oracle.REFERENCE_DEFAULTS  # reference defaults: eps_r 5e-3, omega 0.1

CASES = [
    # name, w, h, params, kind
    ("one_pixel_default", 1, 1, DEF, "random"),
    ("tiny_7x5_baseline", 7, 5, BASE, "random"),
    ("ragged_33x21_default", 33, 21, DEF, "composite"),
    ("coarse_edge_46x46_baseline", 46, 46, BASE, "composite"),
    ("ragged_97x53_baseline", 97, 53, BASE, "composite"),
    ("c1_like_128x96_baseline", 128, 96, BASE, "composite"),
    ("tall_9x130_baseline", 9, 130, BASE, "composite"),
    ("k5_80x64_baseline", 80, 64, oracle.Params(iters_high=5), "composite"),
]


def inputs(w, h, kind, seed):
    if kind == "random":
        rng = np.random.default_rng(seed)
        img = rng.random((3, h, w)).astype(np.float32)
        a = rng.random((h, w)).astype(np.float32)
    else:
        i, a = synth.make_composite(w, h, seed, ellipses=3, edge=2.0)
        img, a = i.numpy(), a.numpy()
    return img, a


def main():
    ref = oracle.reference()
    for idx, (name, w, h, p, kind) in enumerate(CASES):
        img, a = inputs(w, h, kind, 5000 + idx)
        fg, bg = ref.ml_solve(img.astype(np.float64), a.astype(np.float64), p)
        sched = np.array(ref.level_schedule(w, h, p), dtype=np.int32)
        np.savez_compressed(os.path.join(HERE, f"ml_{name}.npz"), image=img, alpha=a, fg=fg, bg=bg, schedule=sched,
                            params=np.array(p.tuple(), dtype=np.float64))
        print(name, img.shape, fg.dtype)
    # resize golden row of test_image.cpp:88-107 and a random resize pair
    rng = np.random.default_rng(77)
    src = rng.random((3, 9, 13))
    np.savez_compressed(os.path.join(HERE, "resize_cases.npz"), src=src, up=ref.resize(src, 29, 17),
                        down=ref.resize(src, 4, 3), mixed=ref.resize(src, 20, 5))


if __name__ == "__main__":
    main()
