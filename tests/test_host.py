"""CPU: the C-ABI library (no kernel launches), its host logic and the
Python mirror of the reference interface."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def header_symbols():
    src = open(os.path.join(ROOT, "include", "fgmatte_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fgm_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol(fgm):
    lib = ctypes.CDLL(fgm.library_path())
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s


def test_library_is_sm100a_only(fgm):
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", fgm.library_path()], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_version(fgm):
    assert "sm_100a" in fgm.version()


@pytest.mark.parametrize("w,h", [(1, 1), (2, 1), (3, 3), (56, 56), (768, 512), (1920, 1080), (3000, 2000),
                                 (4096, 4096), (16384, 16384), (1, 977)])
def test_schedule_capi_equals_reference(fgm, ref, oracle_mod, w, h):
    for p in [oracle_mod.Params(), oracle_mod.REFERENCE_DEFAULTS, oracle_mod.Params(low_res_threshold=100)]:
        got = fgm.level_schedule(w, h, p.omega, p.eps_r, p.low_res_threshold, p.iters_low, p.iters_high)
        assert got == ref.level_schedule(w, h, p)


def test_schedule_capi_exhaustive_small(fgm, orc):
    for w in range(1, 70):
        for h in (1, 7, w, 130):
            assert fgm.level_schedule(w, h) == orc.level_schedule(w, h, __import__("oracle").REFERENCE_DEFAULTS)


@pytest.mark.parametrize("kw,msg", [
    (dict(omega=-1.0), "MlParams: omega must be >= 0"),
    (dict(omega=float("nan")), "MlParams: omega must be >= 0"),
    (dict(eps_r=0.0), "MlParams: eps_r must be > 0"),
    (dict(iters_low=0), "MlParams: iteration counts must be >= 1"),
    (dict(iters_high=0), "MlParams: iteration counts must be >= 1"),
    (dict(low_res_threshold=0), "MlParams: low_res_threshold must be >= 1"),
])
def test_param_validation_messages(fgm, ref, oracle_mod, kw, msg):
    # same exception type and text as MlParams::validate (multilevel.cpp:10-15)
    with pytest.raises(ValueError, match=re.escape(msg)):
        fgm.level_schedule(8, 8, **kw)
    p = oracle_mod.REFERENCE_DEFAULTS
    rp = oracle_mod.Params(**{**dict(omega=p.omega, eps_r=p.eps_r, low_res_threshold=p.low_res_threshold,
                                     iters_low=p.iters_low, iters_high=p.iters_high), **kw})
    with pytest.raises(ValueError, match=re.escape(msg)):
        ref.level_schedule(8, 8, rp)


def test_zero_size_rejected(fgm):
    with pytest.raises(ValueError, match="level_schedule: size must be >= 1x1"):
        fgm.level_schedule(0, 4)


def test_python_api_shape_errors(fgm):
    with pytest.raises(ValueError, match="image must have 1 or 3 channels"):
        fgm.ml_foreground_background(np.zeros((4, 4, 2)), np.zeros((4, 4)))
    with pytest.raises(ValueError, match="alpha array must have 2 dimensions"):
        fgm.ml_foreground_background(np.zeros((4, 4, 3)), np.zeros((4, 4, 1)))
    with pytest.raises(ValueError, match="does not match image size"):
        fgm.ml_foreground_background(np.zeros((4, 4, 3)), np.zeros((4, 3)))
    with pytest.raises(ValueError, match="image must have 3 channels"):
        fgm.ml_foreground_background(np.zeros((4, 4)), np.zeros((4, 4)))


def test_no_cpu_fallback(fgm):
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        fgm.ml_foreground_background(np.full((4, 4, 3), 0.5), np.full((4, 4), 0.5))


def test_synth_deterministic_and_in_range():
    from paper_2006_14970_b200 import synth

    a1 = synth.make_composite(64, 40, 7, 3, 2.0)
    a2 = synth.make_composite(64, 40, 7, 3, 2.0)
    for x, y in zip(a1, a2):
        assert np.array_equal(x.numpy(), y.numpy())
    img, a = a1
    assert img.shape == (3, 40, 64) and a.shape == (40, 64)
    assert float(img.min()) >= 0 and float(img.max()) <= 1 and float(a.min()) >= 0 and float(a.max()) <= 1
    frac = float(((a > 0.01) & (a < 0.99)).float().mean())
    assert 0.02 < frac < 0.9
    sizes = synth.c4_sizes()
    assert len(sizes) == 256 and set(sizes) <= set(synth.C4_SIZES)
