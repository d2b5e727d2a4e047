"""GPU parity: the sm_100a path (through the C ABI) against the fp64 oracle,
the reference's golden fixtures and the reference's own property tests.

Tolerance (fp32 vs fp64, on F and B, per level and final): max-abs TOL_MAX,
mean-abs TOL_MEAN (conftest.py).  Bitwise where the reference's tests are
bitwise and fp32 permits it (exchange / permutation symmetry, determinism,
constant preservation of resize)."""
import numpy as np
import pytest
import torch

from conftest import TOL_MAX, TOL_MEAN, assert_close, golden_files

pytestmark = pytest.mark.gpu


def dev(x, cuda):
    return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float32).to(cuda)


def params_from(fgm, p):
    return fgm.Params(omega=p.omega, eps_r=p.eps_r, low_res_threshold=p.low_res_threshold, iters_low=p.iters_low,
                      iters_high=p.iters_high)


def gpu_solve(fgm, cuda, img, a, p):
    f, b = fgm.ml_foreground_background_cuda(dev(img, cuda), dev(a, cuda), params_from(fgm, p))
    torch.cuda.synchronize()
    return f.double().cpu().numpy(), b.double().cpu().numpy()


# ---- golden fixtures generated from the unmodified reference ---------------
@pytest.mark.parametrize("path", golden_files(), ids=lambda p: p.rsplit("/", 1)[-1])
def test_golden_fixtures(fgm, cuda, oracle_mod, path):
    z = np.load(path)
    pr = z["params"]
    p = oracle_mod.Params(float(pr[0]), float(pr[1]), int(pr[2]), int(pr[3]), int(pr[4]))
    f, b = gpu_solve(fgm, cuda, z["image"], z["alpha"], p)
    assert_close("fg", f, z["fg"])
    assert_close("bg", b, z["bg"])


# ---- shapes, ragged edges and parameter variants vs the fp64 oracle --------
SHAPES = [(1, 1), (2, 1), (1, 2), (3, 3), (5, 3), (1, 40), (40, 1), (31, 24), (45, 45), (46, 46), (64, 64), (65, 33),
          (33, 65), (97, 53), (130, 9), (9, 130), (200, 136), (333, 517), (517, 333), (512, 512),
          (7, 100), (37, 65), (39, 200), (12, 300)]


@pytest.mark.parametrize("w,h", SHAPES)
def test_ml_vs_oracle_shapes(fgm, cuda, orc, oracle_mod, w, h):
    from paper_2006_14970_b200 import synth

    img, a = synth.make_composite(w, h, 100 + w * 7 + h, 3, 2.5)
    img, a = img.numpy(), a.numpy()
    for p in (oracle_mod.Params(), oracle_mod.REFERENCE_DEFAULTS):
        f, b = gpu_solve(fgm, cuda, img, a, p)
        of, ob = orc.ml_solve(img.astype(np.float64), a.astype(np.float64), p)
        assert_close(f"fg {w}x{h}", f, of)
        assert_close(f"bg {w}x{h}", b, ob)


@pytest.mark.parametrize("kw", [dict(iters_high=1), dict(iters_high=3), dict(iters_high=5), dict(iters_high=8),
                                dict(iters_high=10), dict(low_res_threshold=8, iters_low=3),
                                dict(low_res_threshold=100, iters_low=7), dict(omega=0.0, eps_r=0.5),
                                dict(omega=5.0, eps_r=1e-6)])
def test_ml_vs_oracle_params(fgm, cuda, orc, oracle_mod, kw):
    from paper_2006_14970_b200 import synth

    img, a = synth.make_composite(150, 110, 55, 3, 3.0)
    img, a = img.numpy(), a.numpy()
    p = oracle_mod.Params(**kw)
    f, b = gpu_solve(fgm, cuda, img, a, p)
    of, ob = orc.ml_solve(img.astype(np.float64), a.astype(np.float64), p)
    assert_close("fg", f, of)
    assert_close("bg", b, ob)


@pytest.mark.parametrize("kernel", [1, 2])
@pytest.mark.parametrize("w,h", [(7, 100), (37, 65), (39, 200), (40, 33), (41, 31), (64, 97), (300, 32), (300, 33),
                                 (90, 130), (200, 129), (123, 64), (96, 66)])
def test_sweep_border_modes_vs_oracle(fgm, cuda, orc, oracle_mod, w, h, kernel):
    # narrow levels and bands at the row borders: the border / row-border /
    # band-start variants of both K3 kernels (sweep_ws.cu: 1, sweep.cu: 2)
    # against the fp64 oracle, level by level through the single-level entry
    # (BASELINE params, K = 1..4)
    rng = np.random.default_rng(w * 1000 + h)
    img = rng.random((3, h, w)).astype(np.float32)
    a = rng.random((h, w)).astype(np.float32)
    f0 = rng.random((3, h, w)).astype(np.float32)
    b0 = rng.random((3, h, w)).astype(np.float32)
    p = oracle_mod.Params()
    for K in (1, 2, 3, 4):
        of, ob = orc.sweep(img.astype(np.float64), a.astype(np.float64), f0.astype(np.float64),
                           b0.astype(np.float64), p, K)
        gf, gb = fgm.sweep_passes_cuda(dev(img, cuda), dev(a, cuda), dev(f0, cuda), dev(b0, cuda), K, p.eps_r,
                                       p.omega, kernel)
        torch.cuda.synchronize()
        assert_close("fg", gf.double().cpu().numpy(), of, tol_max=2e-5, tol_mean=1e-6)
        assert_close("bg", gb.double().cpu().numpy(), ob, tol_max=2e-5, tol_mean=1e-6)


def test_random_inputs_vs_oracle(fgm, cuda, orc, oracle_mod):
    rng = np.random.default_rng(5)
    for (w, h) in [(77, 41), (256, 200)]:
        img = rng.random((3, h, w)).astype(np.float32)
        a = rng.random((h, w)).astype(np.float32)
        for p in (oracle_mod.Params(), oracle_mod.REFERENCE_DEFAULTS):
            f, b = gpu_solve(fgm, cuda, img, a, p)
            of, ob = orc.ml_solve(img.astype(np.float64), a.astype(np.float64), p)
            assert_close("fg", f, of)
            assert_close("bg", b, ob)


def test_unclamped_inputs_top_level_identity(fgm, cuda, orc, oracle_mod):
    # The C++ API does not clamp inputs; the last level resizes the original
    # as an unclamped identity copy (image.cpp:116,127).
    rng = np.random.default_rng(6)
    img = (rng.random((3, 60, 90)) * 1.4 - 0.2).astype(np.float32)
    a = rng.random((60, 90)).astype(np.float32)
    f, b = gpu_solve(fgm, cuda, img, a, oracle_mod.Params())
    of, ob = orc.ml_solve(img.astype(np.float64), a.astype(np.float64), oracle_mod.Params())
    assert_close("fg", f, of)
    assert_close("bg", b, ob)


# ---- per-level parity ---------------------------------------------------------
@pytest.mark.parametrize("w,h", [(300, 200), (1920, 1080)])
def test_per_level_vs_oracle(fgm, cuda, orc, oracle_mod, w, h):
    from paper_2006_14970_b200 import synth

    img, a = synth.make_composite(w, h, 77, 5, 4.0, hair=(w == 1920))
    p = oracle_mod.Params()
    f, b, lf, lb = fgm.ml_foreground_background_levels_cuda(img.to(cuda), a.to(cuda), params_from(fgm, p))
    torch.cuda.synchronize()
    of, ob, olf, olb = orc.ml_solve(img.double().numpy(), a.double().numpy(), p, levels=True)
    assert len(lf) == len(olf)
    for l in range(len(lf)):
        assert_close(f"fg level {l}", lf[l].double().cpu().numpy(), olf[l])
        assert_close(f"bg level {l}", lb[l].double().cpu().numpy(), olb[l])
    assert np.array_equal(lf[-1].cpu().numpy(), f.cpu().numpy())


@pytest.mark.parametrize("w,h,params", [(300, 200, "baseline"), (1920, 1080, "baseline"), (3000, 2000, "defaults"),
                                        (77, 333, "baseline"), (31, 17, "defaults"), (1, 1, "baseline")])
def test_coarse_levels_bitwise_vs_oracle(fgm, cuda, orc, oracle_mod, w, h, params):
    """The coarse levels (every level up to small_size) run in fp64 with the
    reference's operation order (kernels.cu K4): given the same (fp32)
    inputs, each coarse level's F/B is the reference's fp64 value rounded
    to fp32 -- bitwise."""
    from paper_2006_14970_b200 import synth

    img, a = synth.make_composite(w, h, 91 + w, 5, 4.0)
    p = oracle_mod.Params(omega=1.0, eps_r=1e-5, iters_high=2) if params == "baseline" else oracle_mod.Params()
    _, _, lf, lb = fgm.ml_foreground_background_levels_cuda(img.to(cuda), a.to(cuda), params_from(fgm, p))
    torch.cuda.synchronize()
    _, _, olf, olb = orc.ml_solve(img.double().numpy(), a.double().numpy(), p, levels=True)
    sched = orc.level_schedule(w, h, p)
    n_coarse = sum(1 for (lw, lh, _) in sched if lw * lh <= 1024 and max(lw, lh) <= p.low_res_threshold)
    assert n_coarse >= 1
    for l in range(n_coarse):
        assert np.array_equal(lf[l].cpu().numpy(), olf[l].astype(np.float32)), f"fg level {l} {sched[l]}"
        assert np.array_equal(lb[l].cpu().numpy(), olb[l].astype(np.float32)), f"bg level {l} {sched[l]}"


# ---- single level: K fused sweeps vs `iterations` oracle sweeps ---------------
@pytest.mark.parametrize("kernel", [1, 2])
@pytest.mark.parametrize("w,h,K", [(37, 29, 1), (64, 64, 2), (100, 70, 3), (130, 97, 4), (50, 40, 8), (33, 200, 10),
                                   (1, 50, 2), (50, 1, 2), (300, 33, 2), (257, 129, 2), (700, 300, 2), (520, 260, 4),
                                   (333, 190, 1)])
def test_sweep_passes_vs_oracle(fgm, cuda, orc, oracle_mod, w, h, K, kernel):
    rng = np.random.default_rng(w * 31 + h * 7 + K)
    img = rng.random((3, h, w)).astype(np.float32)
    a = rng.random((h, w)).astype(np.float32)
    f0 = rng.random((3, h, w)).astype(np.float32)
    b0 = rng.random((3, h, w)).astype(np.float32)
    p = oracle_mod.Params()
    of, ob = orc.sweep(img.astype(np.float64), a.astype(np.float64), f0.astype(np.float64), b0.astype(np.float64), p,
                       K)
    gf, gb = fgm.sweep_passes_cuda(dev(img, cuda), dev(a, cuda), dev(f0, cuda), dev(b0, cuda), K, p.eps_r, p.omega,
                                   kernel)
    torch.cuda.synchronize()
    assert_close("fg", gf.double().cpu().numpy(), of, tol_max=2e-5, tol_mean=1e-6)
    assert_close("bg", gb.double().cpu().numpy(), ob, tol_max=2e-5, tol_mean=1e-6)


# Both K3 kernels run the same operations in the same order
# (pixel_coefr_dl / pixel_applyr): a single-level pass is bitwise the same
# whichever one a launch is given (batch == single relies on it).
@pytest.mark.parametrize("w,h,iters", [(64, 40, 1), (200, 136, 2), (37, 95, 2), (333, 129, 3), (257, 260, 4),
                                       (1000, 700, 6), (1920, 1080, 2), (33, 33, 2), (4, 70, 2), (70, 4, 4),
                                       (2050, 70, 2)])
def test_sweep_kernels_bitwise_equal(fgm, cuda, w, h, iters):
    g = torch.Generator(device=cuda).manual_seed(w * 7 + h)
    img = torch.rand((3, h, w), device=cuda, generator=g)
    a = torch.rand((h, w), device=cuda, generator=g)
    f0 = torch.rand((3, h, w), device=cuda, generator=g)
    b0 = torch.rand((3, h, w), device=cuda, generator=g)
    p = fgm.BASELINE_PARAMS
    ref = fgm.sweep_passes_cuda(img, a, f0, b0, iters, p.eps_r, p.omega, 2)
    out = fgm.sweep_passes_cuda(img, a, f0, b0, iters, p.eps_r, p.omega, 1)
    torch.cuda.synchronize()
    assert torch.equal(out[0], ref[0]) and torch.equal(out[1], ref[1]), "the latency kernel differs from the throughput kernel"


# ---- resize kernel: image.cpp:71-133, test_image.cpp:88-121 --------------------
def test_resize_golden_row_bitwise(fgm, cuda):
    out = fgm.resize_cuda(dev(np.array([[[0.0, 1.0]]]), cuda), 4, 1)
    assert out[0, 0].tolist() == [0.0, 0.25, 0.75, 1.0]


def test_resize_constants_bitwise(fgm, cuda):
    out = fgm.resize_cuda(dev(np.full((3, 4, 5), 0.77), cuda), 13, 9)
    assert bool((out == torch.tensor(0.77, dtype=torch.float32)).all())


def test_resize_vs_reference_fixture(fgm, cuda):
    z = np.load(golden_files("resize_cases.npz")[0])
    src = dev(z["src"], cuda)
    for key, (w, h) in [("up", (29, 17)), ("down", (4, 3)), ("mixed", (20, 5))]:
        out = fgm.resize_cuda(src, w, h).double().cpu().numpy()
        assert np.abs(out - z[key]).max() < 1e-6


@pytest.mark.parametrize("sw,sh,dw,dh", [(32, 28, 64, 55), (395, 274, 768, 512), (790, 563, 1539, 1062),
                                         (1539, 1062, 3000, 2000), (7, 6, 14, 12), (100, 3, 161, 5),
                                         (13, 9, 40, 33), (333, 517, 600, 830)])
def test_upsample_six_planes(fgm, cuda, orc, sw, sh, dw, dh):
    # six planes at scale <= 0.625 take the staged F/B upsample kernel (the
    # solver's level-to-level path): bitwise equal to the generic resample
    # kernel (one plane at a time), and to the fp32 oracle resize within the
    # FMA-contraction rounding (the oracle is built with -ffp-contract=off)
    rng = np.random.default_rng(sw * 7 + dh)
    src = rng.random((6, sh, sw), dtype=np.float32)
    x = dev(src, cuda)
    out = fgm.resize_cuda(x, dw, dh)
    planes = torch.cat([fgm.resize_cuda(x[p:p + 1].contiguous(), dw, dh) for p in range(6)])
    assert torch.equal(out, planes)
    ref = orc.resize(src, dw, dh)
    assert np.abs(out.cpu().numpy() - ref).max() <= 2e-7


# ---- device HWC boundary of the Python entry point ----
@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_ml_foreground_background_device_hwc(fgm, cuda, dtype):
    from paper_2006_14970_b200 import synth
    img, alpha = synth.make_composite(97, 61, synth.BASE_SEED + 8, ellipses=3, edge=3.0)
    hwc = img.permute(1, 2, 0).contiguous().numpy().astype(dtype)
    a = alpha.numpy().astype(dtype)
    a[0, :5] = 1.3  # out-of-range inputs are clamped like the binding (bindings.cpp:36, 62)
    f_host, b_host = fgm.ml_foreground_background(hwc, a, **fgm.BASELINE_PARAMS.kwargs())
    f_dev, b_dev = fgm.ml_foreground_background(torch.from_numpy(hwc).to(cuda), torch.from_numpy(a).to(cuda),
                                                **fgm.BASELINE_PARAMS.kwargs())
    assert f_dev.is_cuda and f_dev.shape == (61, 97, 3) and str(f_dev.dtype) == f"torch.{dtype}"
    # same fp32 solve; the host path rounds its fp64 input to fp32 the same way
    assert np.array_equal(f_dev.double().cpu().numpy(), f_host)
    assert np.array_equal(b_dev.double().cpu().numpy(), b_host)
    with pytest.raises(ValueError, match="alpha size"):
        fgm.ml_foreground_background(torch.from_numpy(hwc).to(cuda), torch.from_numpy(a[:9]).to(cuda))


# ---- quality metrics: metrics.cpp:75-145 --------------
def test_metrics_vs_reference(fgm, cuda, ref):
    from paper_2006_14970_b200 import synth
    img, alpha = synth.make_composite(131, 77, synth.BASE_SEED + 21, ellipses=4, edge=5.0)
    f, b = fgm.ml_foreground_background_cuda(img.to(cuda), alpha.to(cuda), fgm.BASELINE_PARAMS)
    rng = np.random.default_rng(4)
    gt = torch.from_numpy(rng.random((3, 77, 131), dtype=np.float32)).to(cuda)
    for sigma, radius in [(1.4, 0), (0.8, 3), (2.0, 0)]:
        got = fgm.evaluate_metrics_cuda(f, gt, alpha.to(cuda), sigma, radius)
        want = ref.metrics(f.double().cpu().numpy(), gt.double().cpu().numpy(), alpha.double().numpy(), sigma,
                           radius)
        assert got["translucent_pixel_count"] == want["translucent_pixel_count"] > 0
        for k in ("sad", "mse", "grad"):
            assert abs(got[k] - want[k]) <= 1e-12 * max(1.0, abs(want[k])), (k, got[k], want[k])
    with pytest.raises(ValueError, match="GradParams: sigma must be > 0"):
        fgm.evaluate_metrics_cuda(f, gt, alpha.to(cuda), 0.0)


# ---- compose epilogue: image.cpp:39-57 -----------------
def test_compose_vs_reference(fgm, cuda, ref, orc):
    rng = np.random.default_rng(39)
    f = rng.random((3, 37, 53), dtype=np.float32)
    b = rng.random((3, 37, 53), dtype=np.float32)
    a = (rng.random((37, 53), dtype=np.float32) * 1.4 - 0.2).astype(np.float32)  # clamping exercised
    out = fgm.compose_cuda(dev(f, cuda), dev(b, cuda), dev(a, cuda)).cpu().numpy()
    assert np.array_equal(out, orc.compose(f, b, a))  # same fp32 operation order, bitwise
    assert np.abs(out - ref.compose(f, b, a)).max() < 1e-6  # the reference in fp64
    with pytest.raises(ValueError, match="compose: alpha size"):
        fgm.compose_cuda(dev(f, cuda), dev(b, cuda), dev(a[:5], cuda))


def test_compose_estimate_reconstructs_image(fgm, cuda, orc):
    # test_multilevel.cpp:239-261 through the device epilogue: compose(F, B, alpha) ~ I
    from paper_2006_14970_b200 import synth
    img, alpha = synth.make_composite(160, 96, synth.BASE_SEED + 5, ellipses=3, edge=4.0)
    f, b = fgm.ml_foreground_background_cuda(img.to(cuda), alpha.to(cuda), fgm.BASELINE_PARAMS)
    rec = fgm.compose_cuda(f, b, alpha.to(cuda))
    assert float((rec - img.to(cuda)).abs().mean()) < 1e-3


def test_resize_identity_and_errors(fgm, cuda):
    x = torch.rand(3, 6, 9, device=cuda)
    assert torch.equal(fgm.resize_cuda(x, 9, 6), x)
    with pytest.raises(ValueError, match="resize: target size must be >= 1x1"):
        fgm.resize_cuda(x, 0, 3)


# ---- the reference's property tests (test_multilevel.cpp:143-301) on the GPU ----
def test_constant_binary_alpha(fgm, cuda, oracle_mod):  # :143-158
    img = np.stack([np.full((21, 33), 0.2 + 0.25 * c, np.float32) for c in range(3)])
    f, _ = gpu_solve(fgm, cuda, img, np.ones((21, 33), np.float32), oracle_mod.REFERENCE_DEFAULTS)
    assert np.abs(f - img).max() < 1e-6
    _, b = gpu_solve(fgm, cuda, img, np.zeros((21, 33), np.float32), oracle_mod.REFERENCE_DEFAULTS)
    assert np.abs(b - img).max() < 1e-6


@pytest.mark.parametrize("size", [64, 256])
def test_exchange_symmetry_bitwise(fgm, cuda, oracle_mod, size):  # :167-180
    rng = np.random.default_rng(31)
    img = rng.random((3, size, size)).astype(np.float32)
    a = (rng.integers(0, 1025, (size, size)) / 1024.0).astype(np.float32)
    for p in (oracle_mod.REFERENCE_DEFAULTS, oracle_mod.Params()):
        f, b = gpu_solve(fgm, cuda, img, a, p)
        fc, bc = gpu_solve(fgm, cuda, img, 1.0 - a, p)
        assert np.array_equal(f, bc) and np.array_equal(b, fc)


def test_channel_permutation_bitwise(fgm, cuda, oracle_mod):  # :182-197
    rng = np.random.default_rng(37)
    img = rng.random((3, 170, 240)).astype(np.float32)
    a = rng.random((170, 240)).astype(np.float32)
    perm = [2, 0, 1]
    f, b = gpu_solve(fgm, cuda, img, a, oracle_mod.Params())
    fp, bp = gpu_solve(fgm, cuda, img[perm], a, oracle_mod.Params())
    assert np.array_equal(fp, f[perm]) and np.array_equal(bp, b[perm])


def test_determinism_bitwise(fgm, cuda):  # :199-206
    from paper_2006_14970_b200 import synth

    img, a = synth.make_composite(700, 500, 41, 5, 4.0)
    img, a = img.to(cuda), a.to(cuda)
    r1 = fgm.ml_foreground_background_cuda(img, a, fgm.BASELINE_PARAMS)
    r2 = fgm.ml_foreground_background_cuda(img, a, fgm.BASELINE_PARAMS)
    assert torch.equal(r1[0], r2[0]) and torch.equal(r1[1], r2[1])


def test_one_pixel_vs_iterated_solve_pixel(fgm, cuda, orc, oracle_mod):  # :208-237
    p = oracle_mod.REFERENCE_DEFAULTS
    inten = [0.62, 0.31, 0.85]
    f, b = gpu_solve(fgm, cuda, np.array(inten, np.float32).reshape(3, 1, 1), np.full((1, 1), 0.7, np.float32), p)
    fo, bo = np.zeros(3), np.zeros(3)
    a = float(np.float32(0.7))
    inten32 = [float(np.float32(v)) for v in inten]
    for _ in range(p.iters_low):
        fo, bo = orc.solve_pixel(a, inten32, [a] * 4, [fo] * 4, [bo] * 4)
    assert np.abs(f[:, 0, 0] - fo).max() < 1e-6 and np.abs(b[:, 0, 0] - bo).max() < 1e-6
    assert np.abs(a * f[:, 0, 0] + (1 - a) * b[:, 0, 0] - np.array(inten32)).max() < 8 * p.eps_r


def test_reconstruction_and_range(fgm, cuda, oracle_mod):  # :239-261, :285-301
    from paper_2006_14970_b200 import synth

    for s in range(3):
        img, a = synth.make_composite(48, 40, 43 + s, 2, 3.0)
        f, b = gpu_solve(fgm, cuda, img.numpy(), a.numpy(), oracle_mod.REFERENCE_DEFAULTS)
        an = a.numpy().astype(np.float64)
        rec = an * f + (1 - an) * b
        m = (an > 0) & (an < 1)
        err = (an * ((rec - img.numpy()) ** 2).sum(0))[m].sum() / m.sum()
        assert err < 1e-3
        assert f.min() >= 0 and f.max() <= 1 and b.min() >= 0 and b.max() <= 1


def test_two_color_ramp(fgm, cuda, oracle_mod):  # :263-283
    size = 64
    ramp = np.tile(np.arange(size, dtype=np.float64) / (size - 1), (size, 1))
    ftc, btc = np.array([0.9, 0.1, 0.1]), np.array([0.1, 0.1, 0.9])
    img = np.clip(ramp[None] * ftc[:, None, None] + (1 - ramp[None]) * btc[:, None, None], 0, 1)
    f, _ = gpu_solve(fgm, cuda, img.astype(np.float32), ramp.astype(np.float32), oracle_mod.REFERENCE_DEFAULTS)
    m = ramp > 0.1
    assert max(np.abs(f[c][m] - ftc[c]).max() for c in range(3)) < 0.02


# ---- entry points and error behaviour ------------------------------------------
def test_host_numpy_api_matches_oracle(fgm, orc, oracle_mod):
    rng = np.random.default_rng(8)
    img = rng.random((70, 90, 3))
    a = rng.random((70, 90))
    f, b = fgm.ml_foreground_background(img, a)  # reference defaults, HWC fp64 (bindings.cpp:146-157)
    of, ob = orc.ml_solve(img.transpose(2, 0, 1).astype(np.float32).astype(np.float64),
                          a.astype(np.float32).astype(np.float64), oracle_mod.REFERENCE_DEFAULTS)
    assert f.shape == (70, 90, 3) and f.dtype == np.float64
    assert_close("fg", f.transpose(2, 0, 1), of)
    assert_close("bg", b.transpose(2, 0, 1), ob)


def test_errors_on_gpu(fgm, cuda):
    x = torch.rand(3, 8, 8, device=cuda)
    a = torch.rand(8, 8, device=cuda)
    with pytest.raises(ValueError, match="MlParams: eps_r must be > 0"):
        fgm.ml_foreground_background_cuda(x, a, fgm.Params(eps_r=0.0))
    with pytest.raises(ValueError, match="does not match image size"):
        fgm.ml_foreground_background_cuda(x, torch.rand(8, 7, device=cuda))
    with pytest.raises(TypeError):
        fgm.ml_foreground_background_cuda(x.double(), a)


def test_batch_equals_single_bitwise(fgm, cuda):
    from paper_2006_14970_b200 import synth

    sizes = [(300, 200), (64, 48), (513, 257), (96, 96), (1, 1), (40, 7)]
    imgs, alps = [], []
    for i, (w, h) in enumerate(sizes):
        im, al = synth.make_composite(w, h, 900 + i, 3, 3.0)
        imgs.append(im.to(cuda))
        alps.append(al.to(cuda))
    outs = fgm.batch_solve_cuda(imgs, alps, fgm.BASELINE_PARAMS)
    for im, al, (f, b) in zip(imgs, alps, outs):
        f1, b1 = fgm.ml_foreground_background_cuda(im, al, fgm.BASELINE_PARAMS)
        assert torch.equal(f, f1) and torch.equal(b, b1)


def test_small_batch_latency_launches_bitwise_and_vs_oracle(fgm, cuda, orc, oracle_mod):
    # a batch of <= 4 images: every big-level launch is latency-bound and runs the
    # warp-specialised kernel (sweep_ws.cu) with the bands of several jobs in
    # one ticket order; bitwise the single solves, and the oracle within tolerance
    from paper_2006_14970_b200 import synth

    sizes = [(640, 410), (333, 500), (97, 1100)]
    imgs, alps = [], []
    for i, (w, h) in enumerate(sizes):
        im, al = synth.make_composite(w, h, 990 + i, 4, 3.0)
        imgs.append(im)
        alps.append(al)
    p = oracle_mod.Params()
    outs = fgm.batch_solve_cuda([x.to(cuda) for x in imgs], [x.to(cuda) for x in alps], params_from(fgm, p))
    for im, al, (f, b) in zip(imgs, alps, outs):
        f1, b1 = fgm.ml_foreground_background_cuda(im.to(cuda), al.to(cuda), params_from(fgm, p))
        assert torch.equal(f, f1) and torch.equal(b, b1)
        of, ob = orc.ml_solve(im.double().numpy(), al.double().numpy(), p)
        assert_close("fg", f.double().cpu().numpy(), of)
        assert_close("bg", b.double().cpu().numpy(), ob)


def test_fused_pyramid_bitwise(fgm, cuda):
    # one pass over the full-res input for every level's I/alpha (pyramid_kernel)
    # == one resample launch per level (image.cpp:114-133): same taps, same
    # arithmetic, so identical levels and identical solves; sizes cover ragged
    # tiles, 1-pixel-wide/-high images and a level with an unchanged height
    from paper_2006_14970_b200 import synth

    sizes = [(300, 200), (513, 257), (1000, 33), (2, 700), (700, 3), (129, 17), (777, 1)]
    imgs, alps = [], []
    for i, (w, h) in enumerate(sizes):
        im, al = synth.make_composite(w, h, 950 + i, 3, 3.0)
        imgs.append(im.to(cuda))
        alps.append(al.to(cuda))
    try:
        fgm.set_pyramid_mode(0)
        a = fgm.batch_solve_cuda(imgs, alps, fgm.BASELINE_PARAMS)
        la = [fgm.ml_foreground_background_levels_cuda(im, al, fgm.BASELINE_PARAMS) for im, al in zip(imgs, alps)]
        fgm.set_pyramid_mode(1)
        b = fgm.batch_solve_cuda(imgs, alps, fgm.BASELINE_PARAMS)
        lb = [fgm.ml_foreground_background_levels_cuda(im, al, fgm.BASELINE_PARAMS) for im, al in zip(imgs, alps)]
    finally:
        fgm.set_pyramid_mode(0)
    for (fa, ba), (fb, bb) in zip(a, b):
        assert torch.equal(fa, fb) and torch.equal(ba, bb)
    for x, y in zip(la, lb):
        for lx, ly in zip(x[2] + x[3], y[2] + y[3]):
            assert torch.equal(lx, ly)


# ---- reentrancy: concurrent solves from several host threads ----
def test_concurrent_host_threads(fgm, cuda):
    import threading
    from paper_2006_14970_b200 import synth

    cases = [synth.make_composite(w, h, 900 + i, 3, 3.0) for i, (w, h) in
             enumerate([(300, 200), (257, 513), (640, 96), (128, 128), (1000, 40), (77, 333)])]
    want = []
    for img, a in cases:
        f, b = fgm.ml_foreground_background_cuda(img.to(cuda), a.to(cuda), fgm.BASELINE_PARAMS)
        want.append((f.cpu(), b.cpu()))
    got = [None] * len(cases)
    errs = []

    def work(i):
        try:
            s = torch.cuda.Stream(cuda)
            with torch.cuda.stream(s):
                img, a = cases[i]
                for _ in range(3):
                    f, b = fgm.ml_foreground_background_cuda(img.to(cuda, non_blocking=False), a.to(cuda),
                                                             fgm.BASELINE_PARAMS)
                s.synchronize()
                got[i] = (f.cpu(), b.cpu())
        except Exception as e:  # pragma: no cover
            errs.append(e)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(len(cases))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for (wf, wb), (gf, gb) in zip(want, got):
        assert torch.equal(wf, gf) and torch.equal(wb, gb)


@pytest.mark.parametrize("iters_high", [2, 3, 8])
def test_no_writes_outside_outputs(fgm, cuda, oracle_mod, iters_high):
    # every output plane is written inside [fg, fg + 3wh) and nothing else:
    # the outputs are views into guarded buffers whose canaries must survive
    # (sizes: ragged bands and segments, 1-wide, 1-high, a vec4-misaligned
    # offset), and the inputs are left untouched
    from paper_2006_14970_b200 import synth

    G = 4099  # guard floats on each side (odd: misaligns every output by 4 bytes mod 16)
    canary = -12345.0
    sizes = [(1, 1), (7, 3), (33, 65), (257, 129), (1000, 33), (2, 700), (700, 2), (3000, 70)]
    imgs, alps, outs, bigs = [], [], [], []
    for i, (w, h) in enumerate(sizes):
        im, al = synth.make_composite(w, h, 1200 + i, 3, 3.0)
        imgs.append(im.to(cuda))
        alps.append(al.to(cuda))
        n = 3 * w * h
        pair = []
        for _ in range(2):
            big = torch.full((n + 2 * G,), canary, device=cuda)
            bigs.append(big)
            pair.append(big[G:G + n].view(3, h, w))
        outs.append(tuple(pair))
    before = [x.clone() for x in imgs + alps]
    p = params_from(fgm, oracle_mod.Params(iters_high=iters_high))
    fgm.batch_solve_cuda(imgs, alps, p, outputs=outs)
    torch.cuda.synchronize()
    for big in bigs:
        assert bool((big[:G] == canary).all()) and bool((big[-G:] == canary).all())
    for (f, b) in outs:
        assert bool(((f >= 0) & (f <= 1)).all()) and bool(((b >= 0) & (b <= 1)).all())
    for x, y in zip(before, imgs + alps):
        assert torch.equal(x, y)


@pytest.mark.parametrize("iters_high", [2, 3, 8])
def test_workspace_guards(fgm, cuda, oracle_mod, iters_high):
    # guard bands after every workspace region (level I/alpha pyramid, pass
    # buffers, boundary streams, job descriptors) survive a batch of ragged
    # sizes; results are unchanged by the guard layout
    from paper_2006_14970_b200 import synth

    sizes = [(1, 1), (7, 3), (33, 65), (257, 129), (1000, 33), (2, 700), (700, 2), (3000, 70), (513, 511)]
    imgs, alps = [], []
    for i, (w, h) in enumerate(sizes):
        im, al = synth.make_composite(w, h, 1300 + i, 3, 3.0)
        imgs.append(im.to(cuda))
        alps.append(al.to(cuda))
    p = params_from(fgm, oracle_mod.Params(iters_high=iters_high))
    ref = fgm.batch_solve_cuda(imgs, alps, p)
    try:
        fgm.set_debug_guards(1)
        got = fgm.batch_solve_cuda(imgs, alps, p)
        single = [fgm.ml_foreground_background_cuda(im, al, p) for im, al in zip(imgs, alps)]
    finally:
        fgm.set_debug_guards(0)
    for (fa, ba), (fb, bb), (fc, bc) in zip(ref, got, single):
        assert torch.equal(fa, fb) and torch.equal(ba, bb)
        assert torch.equal(fa, fc) and torch.equal(ba, bc)


@pytest.mark.parametrize("seed", range(4))
def test_random_sizes_and_params_vs_oracle(fgm, cuda, orc, oracle_mod, seed):
    # seeded random shapes (1..320 per side, incl. 1-wide/1-high) and
    # parameters (omega, eps_r, threshold, iteration counts 1..6) against the
    # fp64 oracle, as a batch (level-synchronous across different schedules)
    # and one by one
    from paper_2006_14970_b200 import synth

    rng = np.random.default_rng(20061497 + seed)
    cases = []
    for i in range(6):
        w, h = (int(v) for v in rng.integers(1, 321, size=2))
        if i == 0:
            w = 1
        if i == 1:
            h = 1
        im, al = synth.make_composite(w, h, 1400 + 10 * seed + i, 3, float(rng.uniform(1.0, 6.0)))
        cases.append((im, al))
    p = oracle_mod.Params(omega=float(rng.choice([0.1, 0.5, 1.0, 2.0])), eps_r=float(rng.choice([1e-5, 1e-3, 5e-3])),
                          low_res_threshold=int(rng.choice([4, 16, 32, 64])), iters_low=int(rng.integers(1, 7)),
                          iters_high=int(rng.integers(1, 7)))
    outs = fgm.batch_solve_cuda([c[0].to(cuda) for c in cases], [c[1].to(cuda) for c in cases], params_from(fgm, p))
    for (im, al), (f, b) in zip(cases, outs):
        of, ob = orc.ml_solve(im.double().numpy(), al.double().numpy(), p)
        assert_close("fg", f.double().cpu().numpy(), of)
        assert_close("bg", b.double().cpu().numpy(), ob)
        f1, b1 = gpu_solve(fgm, cuda, im.numpy(), al.numpy(), p)
        assert np.array_equal(f1, f.double().cpu().numpy()) and np.array_equal(b1, b.double().cpu().numpy())


# ---- failure detection: a stalled band hand-over is an error, not a hang ----
@pytest.mark.gpu
def test_stalled_handover_returns_runtime_error(fgm, cuda):
    """SURVEY.md section 5 ("timeout -> error, not a hang"): with band 0 of every
    sweep made to skip publishing its boundary stream (fgm_debug_fault(1)), band
    1 waits for data that never comes; the bounded wait aborts the launch, counts
    a device fault and the synchronous entry point returns FGM_RUNTIME_ERROR."""
    from paper_2006_14970_b200 import synth

    img, a = synth.make_composite(300, 200, 4242, 4, 3.0)  # 7 bands at the top level
    fgm.device_faults(reset=True)
    fgm.set_spin_timeout_ms(100)
    fgm.debug_fault(1)
    try:
        with pytest.raises(RuntimeError, match="timed out"):
            fgm.ml_foreground_background(img.permute(1, 2, 0).double().numpy(), a.double().numpy(),
                                         **fgm.BASELINE_PARAMS.kwargs())
        assert fgm.device_faults() > 0
    finally:
        fgm.debug_fault(0)
        fgm.set_spin_timeout_ms(2000)
        fgm.device_faults(reset=True)
    # the device and the library stay usable
    f, b = fgm.ml_foreground_background(img.permute(1, 2, 0).double().numpy(), a.double().numpy(),
                                        **fgm.BASELINE_PARAMS.kwargs())
    assert np.isfinite(f).all() and np.isfinite(b).all()
    assert fgm.device_faults() == 0


# ---- the K = 4 throughput sweep (16-column chunks) against the oracle -------
@pytest.mark.gpu
def test_k4_throughput_launch_vs_oracle(fgm, cuda, orc, oracle_mod):
    """iters_high = 4 fuses the two big-level sweeps of every big level into one
    K = 4 pass; 16 images of 1024^2 give 16 x 17 bands x 3 channels = 816
    (band, channel) items of the throughput kernel (sweep.cu) in the top-level
    launch, more than the GPU holds at once (148 SMs x 5 warps), so it runs the
    16-column-chunk instantiation sweep_kernel<4, 16>."""
    from paper_2006_14970_b200 import synth

    n = 16
    imgs, alps = [], []
    for i in range(n):
        im, al = synth.make_composite(1024, 1024, 7100 + i, 6, 4.0)
        imgs.append(im)
        alps.append(al)
    p = oracle_mod.Params(omega=1.0, eps_r=1e-5, low_res_threshold=32, iters_low=10, iters_high=4)
    outs = fgm.batch_solve_cuda([x.to(cuda) for x in imgs], [x.to(cuda) for x in alps], params_from(fgm, p))
    torch.cuda.synchronize()
    for i in (0, n - 1):
        of, ob = orc.ml_solve(imgs[i].double().numpy(), alps[i].double().numpy(), p)
        assert_close(f"K4 batch fg {i}", outs[i][0].double().cpu().numpy(), of)
        assert_close(f"K4 batch bg {i}", outs[i][1].double().cpu().numpy(), ob)


# ---- caller-supplied outputs are validated before any device write ----------
@pytest.mark.gpu
def test_bad_outputs_rejected(fgm, cuda):
    from paper_2006_14970_b200 import synth

    img, a = synth.make_composite(64, 48, 11, 2, 3.0)
    img, a = img.to(cuda), a.to(cuda)
    good = (torch.empty_like(img), torch.empty_like(img))
    for bad in ((torch.empty(3, 48, 63, device=cuda), good[1]),                # wrong shape
                (torch.empty(3, 48, 64, device=cuda, dtype=torch.float64), good[1]),  # wrong dtype
                (torch.empty(3, 64, 48, device=cuda).transpose(1, 2), good[1]),  # not contiguous
                (torch.empty(3, 48, 64), good[1])):                             # host tensor
        with pytest.raises(ValueError):
            fgm.batch_solve_cuda([img], [a], fgm.BASELINE_PARAMS, outputs=[bad])
    with pytest.raises(ValueError):
        fgm.batch_solve_host([img.cpu()], [a.cpu()], fgm.BASELINE_PARAMS,
                             outputs=[(torch.empty(3, 48, 64), torch.empty(3, 47, 64))])
    with pytest.raises(ValueError):
        fgm.ml_foreground_background_levels_cuda(img, a[:, :10], fgm.BASELINE_PARAMS)
    with pytest.raises(ValueError):
        fgm.sweep_passes_cuda(img, a, img[:, :10], img, 2, 1e-5, 1.0)
    out = fgm.batch_solve_cuda([img], [a], fgm.BASELINE_PARAMS, outputs=[good])
    assert out[0][0] is good[0]
    fgm.release_memory()
