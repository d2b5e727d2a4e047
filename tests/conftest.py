import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")

# fp32 tolerance of the GPU path against the fp64 oracle, on F and B, per level
# and final: max-abs and mean-abs.
TOL_MAX = 1e-3
TOL_MEAN = 1e-5


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs the sm_100a kernels)")


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle

    return oracle


@pytest.fixture(scope="session")
def ref(oracle_mod):
    if not oracle_mod.reference_available():
        pytest.skip("reference shim (oracle/_ref) not built")
    return oracle_mod.reference()


@pytest.fixture(scope="session")
def orc(oracle_mod):
    return oracle_mod.oracle()


@pytest.fixture(scope="session")
def fgm():
    import paper_2006_14970_b200 as m

    m._load()
    return m


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test collected without a CUDA device (run with -m 'not gpu' on CPU)")
    return torch.device("cuda:0")


def golden_files(pattern="ml_*.npz"):
    return sorted(glob.glob(os.path.join(GOLDEN, pattern)))


def drift(a, b):
    d = np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64))
    return float(d.max()), float(d.mean())


def assert_close(name, got, want, tol_max=TOL_MAX, tol_mean=TOL_MEAN):
    mx, mn = drift(got, want)
    assert mx <= tol_max and mn <= tol_mean, f"{name}: max|d| {mx:.3g} (tol {tol_max}), mean|d| {mn:.3g} (tol {tol_mean})"
    return mx, mn
