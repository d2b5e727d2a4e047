"""CPU: pin the oracle (the C restatement in oracle/fgm_oracle.c) against the
reference itself (oracle/_ref, the unmodified reference sources) and against
the golden values and properties of the reference's own unit tests
(proj/tests/test_multilevel.cpp, proj/tests/test_image.cpp)."""
import numpy as np
import pytest

from conftest import golden_files

BASE = None


@pytest.fixture(scope="module")
def P(oracle_mod):
    return oracle_mod.Params(), oracle_mod.REFERENCE_DEFAULTS


# ---- restatement == reference, bitwise -------------------------------------
@pytest.mark.parametrize("w,h", [(1, 1), (1, 17), (17, 1), (2, 2), (5, 3), (33, 21), (56, 56), (64, 64), (97, 53),
                                 (130, 9), (200, 136)])
def test_restatement_bitwise_equals_reference(orc, ref, P, w, h):
    rng = np.random.default_rng(w * 1000 + h)
    img = rng.random((3, h, w))
    a = rng.random((h, w))
    for p in P:
        f1, b1 = orc.ml_solve(img, a, p)
        f2, b2 = ref.ml_solve(img, a, p)
        assert np.array_equal(f1, f2) and np.array_equal(b1, b2), (w, h, p)


def test_restatement_other_params_bitwise(orc, ref, oracle_mod):
    rng = np.random.default_rng(3)
    img = rng.random((3, 40, 70))
    a = rng.random((40, 70))
    for p in [oracle_mod.Params(iters_high=5), oracle_mod.Params(low_res_threshold=8, iters_low=3),
              oracle_mod.Params(omega=0.0, eps_r=0.3), oracle_mod.Params(low_res_threshold=100, iters_low=7)]:
        f1, b1 = orc.ml_solve(img, a, p)
        f2, b2 = ref.ml_solve(img, a, p)
        assert np.array_equal(f1, f2) and np.array_equal(b1, b2), p


def test_restatement_matches_golden_fixtures(orc, oracle_mod):
    files = golden_files()
    assert files, "tests/golden fixtures missing"
    for f in files:
        z = np.load(f)
        p = oracle_mod.Params(*[float(v) for v in z["params"][:2]], *[int(v) for v in z["params"][2:]])
        fg, bg = orc.ml_solve(z["image"].astype(np.float64), z["alpha"].astype(np.float64), p)
        assert np.array_equal(fg, z["fg"]) and np.array_equal(bg, z["bg"]), f
        assert [tuple(r) for r in z["schedule"]] == orc.level_schedule(z["image"].shape[2], z["image"].shape[1], p)


def test_level_outputs_end_in_final(orc, P):
    rng = np.random.default_rng(9)
    img, a = rng.random((3, 50, 77)), rng.random((50, 77))
    fg, bg, lf, lb = orc.ml_solve(img, a, P[0], levels=True)
    assert np.array_equal(lf[-1], fg) and np.array_equal(lb[-1], bg)
    assert [x.shape[1:] for x in lf] == [(h, w) for (w, h, _) in orc.level_schedule(77, 50, P[0])]


# ---- level schedule: multilevel.cpp:17-44, test_multilevel.cpp:15-66 ------------
def test_schedule_1024(orc):  # test_multilevel.cpp:15-26
    s = orc.level_schedule(1024, 1024, __import__("oracle").REFERENCE_DEFAULTS)
    assert len(s) == 10
    assert s == [(2 ** (l + 1), 2 ** (l + 1), 10 if 2 ** (l + 1) <= 32 else 2) for l in range(10)]


def test_schedule_degenerate(orc, ref):  # test_multilevel.cpp:28-45
    assert orc.level_schedule(1, 1) == [(1, 1, 10)]
    for (w, h) in [(100, 50), (1, 977), (640, 480), (3, 3)]:
        s = orc.level_schedule(w, h)
        assert s[-1][:2] == (w, h)
        m = max(w, h)
        assert len(s) == (max(1, (m - 1).bit_length()) if m > 1 else 1)
    with pytest.raises(ValueError):
        orc.level_schedule(0, 4)
    with pytest.raises(ValueError):
        ref.level_schedule(0, 4)


def test_schedule_exhaustive_vs_reference(orc, ref):
    for e in list(range(1, 300)) + [511, 512, 513, 1080, 1920, 2000, 3000, 4096, 16384]:
        for (w, h) in [(e, 1), (1, e), (e, e), (e, max(1, e // 3))]:
            assert orc.level_schedule(w, h) == ref.level_schedule(w, h), (w, h)


def test_schedule_reproduces_reference_jumps(ref):
    # The reference's "at most doubles" test fails (test_multilevel.cpp:47-66);
    # the build must reproduce the reference sizes, not fix them.
    s = ref.level_schedule(56, 56)
    assert [l[0] for l in s] == [2, 4, 7, 15, 29, 56]


# ---- resize: image.cpp:71-133, test_image.cpp:88-144 -------------------------
def test_resize_golden_row(orc):  # test_image.cpp:88-97
    up = orc.resize(np.array([[[0.0, 1.0]]]), 4, 1)
    assert up[0, 0].tolist() == [0.0, 0.25, 0.75, 1.0]


def test_resize_constants_bitwise(orc):  # test_image.cpp:99-107
    assert np.all(orc.resize(np.full((1, 1, 1), 0.3), 7, 5) == 0.3)
    assert np.all(orc.resize(np.full((3, 4, 5), 0.77), 13, 9) == 0.77)


def test_resize_identity_idempotence(orc):  # test_image.cpp:109-121
    rng = np.random.default_rng(11)
    img = rng.random((3, 6, 9))
    assert np.array_equal(orc.resize(img, 9, 6), img)
    once = orc.resize(img, 4, 11)
    assert np.array_equal(orc.resize(once, 4, 11), once)


def test_resize_range_and_vs_reference(orc, ref):  # test_image.cpp:123-138
    rng = np.random.default_rng(13)
    for _ in range(20):
        sw, sh, dw, dh = [int(x) for x in rng.integers(1, 25, 4)]
        a = rng.random((sh, sw))
        o = orc.resize(a, dw, dh)
        assert o.min() >= 0 and o.max() <= 1
        assert np.array_equal(o, ref.resize(a, dw, dh))


def test_resize_golden_fixture(orc):
    z = np.load(golden_files("resize_cases.npz")[0])
    assert np.array_equal(orc.resize(z["src"], 29, 17), z["up"])
    assert np.array_equal(orc.resize(z["src"], 4, 3), z["down"])
    assert np.array_equal(orc.resize(z["src"], 20, 5), z["mixed"])


# ---- solve_pixel: multilevel.cpp:48-79, test_multilevel.cpp:68-141 -----------
def test_solve_pixel_closed_forms(orc, ref):  # test_multilevel.cpp:68-92
    eps = 5e-3
    inten, f, b0 = [0.7, 0.3, 0.5], [0.9, 0.1, 0.2], [0.1, 0.8, 0.6]
    for impl in (orc, ref):
        sf, sb = impl.solve_pixel(1.0, inten, [1.0] * 4, [f] * 4, [b0] * 4, omega=0.1, eps_r=eps)
        for c in range(3):
            assert sf[c] == pytest.approx((inten[c] + 4 * eps * f[c]) / (1 + 4 * eps), rel=1e-14)
            assert sb[c] == pytest.approx(b0[c], rel=1e-14)
        sf, sb = impl.solve_pixel(0.0, inten, [0.0] * 4, [f] * 4, [b0] * 4, omega=0.1, eps_r=eps)
        for c in range(3):
            assert sb[c] == pytest.approx((inten[c] + 4 * eps * b0[c]) / (1 + 4 * eps), rel=1e-14)
            assert sf[c] == pytest.approx(f[c], rel=1e-14)


def test_solve_pixel_dense(orc, ref):  # test_multilevel.cpp:94-132
    rng = np.random.default_rng(23)
    for _ in range(300):
        nn = 1 + int(rng.integers(0, 6))
        ai = rng.random()
        inten = rng.random(3)
        na, nf, nb = rng.random(nn), rng.random((nn, 3)), rng.random((nn, 3))
        f1, b1 = orc.solve_pixel(ai, inten, na, nf, nb, clamp=False)
        f2, b2 = ref.solve_pixel(ai, inten, na, nf, nb, clamp=False)
        assert np.array_equal(f1, f2) and np.array_equal(b1, b2)
        d = 5e-3 + 0.1 * np.abs(ai - na)
        s = d.sum()
        for c in range(3):
            A = np.array([[ai * ai + s, ai * (1 - ai)], [ai * (1 - ai), (1 - ai) ** 2 + s]])
            x = np.linalg.solve(A, [inten[c] * ai + (d * nf[:, c]).sum(), inten[c] * (1 - ai) + (d * nb[:, c]).sum()])
            assert abs(f1[c] - x[0]) < 1e-12 and abs(b1[c] - x[1]) < 1e-12


def test_solve_pixel_validation(orc, ref):  # test_multilevel.cpp:134-141
    for impl in (orc, ref):
        with pytest.raises(ValueError):
            impl.solve_pixel(1.0, [0.5] * 3, [1.0], [[0, 0, 0]], [[0, 0, 0]], eps_r=0.0)
        with pytest.raises(ValueError):
            impl.solve_pixel(1.0, [0.5] * 3, [], np.zeros((0, 3)), np.zeros((0, 3)))


# ---- whole-solve properties: test_multilevel.cpp:143-301 ----------------------
def test_constant_binary_alpha(orc, oracle_mod):  # :143-158
    img = np.stack([np.full((21, 33), 0.2 + 0.25 * c) for c in range(3)])
    fg, _ = orc.ml_solve(img, np.ones((21, 33)), oracle_mod.REFERENCE_DEFAULTS)
    assert np.abs(fg - img).max() < 1e-6
    _, bg = orc.ml_solve(img, np.zeros((21, 33)), oracle_mod.REFERENCE_DEFAULTS)
    assert np.abs(bg - img).max() < 1e-6


def test_exchange_symmetry_bitwise(orc, oracle_mod):  # :167-180
    rng = np.random.default_rng(31)
    img = rng.random((3, 64, 64))
    a = rng.integers(0, 1025, (64, 64)) / 1024.0
    fg, bg = orc.ml_solve(img, a, oracle_mod.REFERENCE_DEFAULTS)
    fgc, bgc = orc.ml_solve(img, 1.0 - a, oracle_mod.REFERENCE_DEFAULTS)
    assert np.array_equal(fg, bgc) and np.array_equal(bg, fgc)


def test_channel_permutation_bitwise(orc, oracle_mod):  # :182-197
    rng = np.random.default_rng(37)
    img, a = rng.random((3, 17, 24)), rng.random((17, 24))
    perm = [2, 0, 1]
    fg, bg = orc.ml_solve(img, a, oracle_mod.REFERENCE_DEFAULTS)
    fgp, bgp = orc.ml_solve(img[perm], a, oracle_mod.REFERENCE_DEFAULTS)
    assert np.array_equal(fgp, fg[perm]) and np.array_equal(bgp, bg[perm])


def test_one_pixel_iterated_solve_pixel(orc, oracle_mod):  # :208-237
    p = oracle_mod.REFERENCE_DEFAULTS
    inten = [0.62, 0.31, 0.85]
    img = np.array(inten).reshape(3, 1, 1)
    fg, bg = orc.ml_solve(img, np.full((1, 1), 0.7), p)
    f, b = np.zeros(3), np.zeros(3)
    for _ in range(p.iters_low):
        f, b = orc.solve_pixel(0.7, inten, [0.7] * 4, [f] * 4, [b] * 4)
    assert np.array_equal(fg[:, 0, 0], f) and np.array_equal(bg[:, 0, 0], b)


def test_output_range(orc):  # :285-301
    rng = np.random.default_rng(47)
    fg, bg = orc.ml_solve(rng.random((3, 13, 19)), rng.random((13, 19)))
    assert fg.min() >= 0 and fg.max() <= 1 and bg.min() >= 0 and bg.max() <= 1


def test_fp32_restatement_drift_bounded(orc):
    # Calibrates the stated tolerance: the reference's own algebra evaluated in
    # fp32 stays well inside it on a smooth composite.
    from paper_2006_14970_b200 import synth

    img, a = synth.make_composite(96, 80, 123, 3, 3.0)
    img, a = img.numpy(), a.numpy()
    f64, b64 = orc.ml_solve(img.astype(np.float64), a.astype(np.float64))
    f32, b32 = orc.ml_solve(img, a, dtype=np.float32)
    assert np.abs(f32 - f64).max() < 1e-3 and np.abs(b32 - b64).max() < 1e-3


def test_compose_matches_reference(orc, ref):  # image.cpp:39-57
    rng = np.random.default_rng(57)
    f, b = rng.random((3, 11, 13)), rng.random((3, 11, 13))
    a = rng.random((11, 13)) * 1.4 - 0.2
    assert np.array_equal(orc.compose(f, b, a), ref.compose(f, b, a))
