"""GPU: the reference's OWN unit tests (proj/tests/test_multilevel.cpp,
test_image.cpp, compiled from the reference sources at build time) linked
against the C++ drop-in dropin/multilevel_b200.cpp, i.e. run through the B200
path.  Expected failures:
  * "level sizes at most double ..." fails in the reference itself
    (test_multilevel.cpp:47-66) -- it does not call the solver;
Everything else must pass, including the bitwise exchange-symmetry,
permutation and determinism cases and "one-pixel image matches iterated
solve_pixel" (test_multilevel.cpp:208-237: a 1x1 image is coarse at every
level, so the fp64 coarse kernel, fed the fp64 input by the drop-in, must
reproduce the reference's arithmetic bitwise)."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

BIN = os.path.join(ROOT, "dropin", "_build", "ref_tests_b200")
EXPECTED_FAIL = {"level sizes at most double, exhaustively to 4096"}


def test_reference_unit_tests_through_dropin(cuda):
    if not os.path.exists(BIN):
        pytest.skip("drop-in test binary not built (needs the reference sources at build time)")
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600).stdout
    res = {}
    for line in out.splitlines():
        if line.startswith("PASS ") or line.startswith("FAIL "):
            res[line[5:]] = line[:4]
    assert len(res) == 24, out
    failed = {k for k, v in res.items() if v == "FAIL"}
    assert failed == EXPECTED_FAIL, out
