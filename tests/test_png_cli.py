"""PNG I/O and the command-line tool, after the
reference's test_png.cpp and test_cli.cpp.

CPU: codec round trips / quantisation / error cases (test_png.cpp:27-72),
decoding of every PNG filter type, bit depth <8, palette and tRNS (files
written by an independent filtered encoder below), and the CLI's usage and
I/O exit codes, which fail before any GPU work (test_cli.cpp:117-126).
GPU: estimate / compose / metrics / bench through the CLI against the oracle
(test_cli.cpp:63-247).  Closed-form and prep-dataset are out of scope and
exit 1 naming why."""
import os
import struct
import subprocess
import sys
import zlib

import numpy as np
import pytest

from conftest import ROOT, TOL_MAX

from paper_2006_14970_b200.png_io import PngError, load_alpha_png, load_png, save_png


def quantize(v, bits):
    m = 65535.0 if bits == 16 else 255.0
    return np.floor(np.clip(v, 0.0, 1.0) * m + 0.5) / m


def smooth_field(w, h, c, seed):
    rng = np.random.default_rng(seed)
    y, x = np.mgrid[0:h, 0:w]
    out = np.empty((c, h, w))
    for k in range(c):
        fx, fy, ph = rng.uniform(0.5, 3, 3)
        out[k] = 0.5 + 0.45 * np.sin(2 * np.pi * (fx * x / w + fy * y / h) + ph)
    return out


# ---------------------------------------------------------------------------
# codec (test_png.cpp)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("bits", [8, 16])
def test_png_roundtrip_equals_quantized_raster(tmp_path, bits):
    img = smooth_field(13, 9, 3, 151)
    p = str(tmp_path / f"rt{bits}.png")
    save_png(p, img, bits)
    col, alpha, depth = load_png(p)
    assert col.shape == (3, 9, 13) and depth == bits and alpha is None
    assert np.array_equal(col, quantize(img, bits))  # exact at quantised resolution


def test_grayscale_roundtrip_and_alpha_from_gray(tmp_path):
    a = np.random.default_rng(157).uniform(0, 1, (11, 6))
    p = str(tmp_path / "g.png")
    save_png(p, a, 16)
    assert np.array_equal(load_alpha_png(p, "gray-png"), quantize(a, 16))
    with pytest.raises(PngError, match="no alpha channel"):
        load_alpha_png(p, "alpha-channel")
    rgb = str(tmp_path / "rgb.png")
    save_png(rgb, smooth_field(4, 4, 3, 1), 8)
    with pytest.raises(PngError, match="not grayscale"):
        load_alpha_png(rgb, "gray-png")


def test_quantization_idempotence(tmp_path):
    img = quantize(smooth_field(5, 5, 3, 163), 8)
    p = str(tmp_path / "q.png")
    save_png(p, img, 8)
    assert np.array_equal(load_png(p)[0], img)


def test_save_clamps_and_rounds_half_up(tmp_path):
    v = np.array([[-0.5, 0.0, 0.5 / 255, 1.5 / 255, 1.0, 2.0]])
    p = str(tmp_path / "c.png")
    save_png(p, v, 8)
    assert np.array_equal(load_png(p)[0][0] * 255, [[0, 0, 1, 2, 255, 255]])


def test_png_errors_are_surfaced(tmp_path):
    with pytest.raises(PngError, match="cannot open"):
        load_png(str(tmp_path / "missing.png"))
    with pytest.raises(PngError, match="bit depth"):
        save_png(str(tmp_path / "bad.png"), np.full((3, 2, 2), 0.5), 12)
    with pytest.raises(PngError, match="cannot open"):
        save_png(str(tmp_path / "no_dir" / "x.png"), np.full((2, 2), 0.5), 8)
    bad = tmp_path / "garbage.png"
    bad.write_bytes(b"not a png at all")
    with pytest.raises(PngError, match="failed to decode"):
        load_png(str(bad))
    good = str(tmp_path / "ok.png")
    save_png(good, np.full((2, 2), 0.5), 8)
    data = bytearray(open(good, "rb").read())
    data[40] ^= 0xFF  # corrupt a byte inside IDAT: the chunk CRC catches it
    bad.write_bytes(bytes(data))
    with pytest.raises(PngError):
        load_png(str(bad))


# independent encoder: every filter type, low bit depths, palette, tRNS
def _chunk(t, d):
    return struct.pack(">I", len(d)) + t + d + struct.pack(">I", zlib.crc32(t + d) & 0xFFFFFFFF)


def _paeth(a, b, c):
    p = a + b - c
    pa, pb, pc = abs(p - a), abs(p - b), abs(p - c)
    return a if pa <= pb and pa <= pc else (b if pb <= pc else c)


def _encode(path, raw_rows, w, h, depth, ctype, bpp, filters, extra=b""):
    out, prior = [], [0] * len(raw_rows[0])
    for y, row in enumerate(raw_rows):
        ft = filters[y % len(filters)]
        f = []
        for i, v in enumerate(row):
            a = row[i - bpp] if i >= bpp else 0
            c = prior[i - bpp] if i >= bpp else 0
            pred = [0, a, prior[i], (a + prior[i]) >> 1, _paeth(a, prior[i], c)][ft]
            f.append((v - pred) & 0xFF)
        out.append(bytes([ft] + f))
        prior = list(row)
    png = b"\x89PNG\r\n\x1a\n" + _chunk(b"IHDR", struct.pack(">IIBBBBB", w, h, depth, ctype, 0, 0, 0)) + extra
    comp = zlib.compress(b"".join(out))
    png += _chunk(b"IDAT", comp[:7]) + _chunk(b"IDAT", comp[7:]) + _chunk(b"IEND", b"")  # split IDAT
    with open(path, "wb") as fh:
        fh.write(png)


@pytest.mark.parametrize("depth", [8, 16])
def test_decoder_handles_every_filter_type(tmp_path, depth):
    rng = np.random.default_rng(7)
    w, h = 17, 10
    m = (1 << depth) - 1
    samp = rng.integers(0, m + 1, (h, w, 4))
    rows = []
    for y in range(h):
        if depth == 8:
            rows.append(list(samp[y].astype(np.uint8).tobytes()))
        else:
            rows.append(list(samp[y].astype(">u2").tobytes()))
    p = str(tmp_path / "f.png")
    _encode(p, rows, w, h, depth, 6, 4 * depth // 8, [0, 1, 2, 3, 4])
    col, alpha, d = load_png(p)
    assert d == depth
    assert np.array_equal(col, samp[:, :, :3].transpose(2, 0, 1) / m)
    assert np.array_equal(alpha, samp[:, :, 3] / m)
    assert np.array_equal(load_alpha_png(p, "alpha-channel"), samp[:, :, 3] / m)


@pytest.mark.parametrize("depth", [1, 2, 4])
def test_low_bit_grey_expands_to_8(tmp_path, depth):
    rng = np.random.default_rng(depth)
    w, h = 13, 5
    v = rng.integers(0, 1 << depth, (h, w))
    per = 8 // depth
    rows = []
    for y in range(h):
        r = []
        for x0 in range(0, w, per):
            b = 0
            for k in range(per):
                b = (b << depth) | (int(v[y, x0 + k]) if x0 + k < w else 0)
            r.append(b)
        rows.append(r)
    p = str(tmp_path / "g.png")
    _encode(p, rows, w, h, depth, 0, 1, [1, 4])
    col, alpha, d = load_png(p)
    assert d == 8 and alpha is None
    assert np.array_equal(col[0], v * (255 // ((1 << depth) - 1)) / 255.0)


def test_palette_with_trns(tmp_path):
    rng = np.random.default_rng(3)
    w, h = 9, 6
    pal = rng.integers(0, 256, (5, 3))
    trns = np.array([0, 128, 255])  # entries 3, 4 opaque
    idx = rng.integers(0, 5, (h, w))
    p = str(tmp_path / "p.png")
    extra = _chunk(b"PLTE", pal.astype(np.uint8).tobytes()) + _chunk(b"tRNS", trns.astype(np.uint8).tobytes())
    _encode(p, [[int(v) for v in idx[y]] for y in range(h)], w, h, 8, 3, 1, [2], extra)
    col, alpha, d = load_png(p)
    assert np.array_equal(col, pal[idx].transpose(2, 0, 1) / 255.0)
    assert np.array_equal(alpha, np.concatenate([trns, [255, 255]])[idx] / 255.0)


def test_rgb_colour_key_trns(tmp_path):
    w, h = 4, 3
    samp = np.zeros((h, w, 3), np.int64)
    samp[1, 2] = (10, 20, 30)
    p = str(tmp_path / "k.png")
    _encode(p, [list(samp[y].astype(np.uint8).tobytes()) for y in range(h)], w, h, 8, 2, 3, [0],
            _chunk(b"tRNS", struct.pack(">HHH", 10, 20, 30)))
    _, alpha, _ = load_png(p)
    expect = np.ones((h, w))
    expect[1, 2] = 0
    assert np.array_equal(alpha, expect)


# ---------------------------------------------------------------------------
# CLI: usage / I/O exit codes (CPU; these fail before any GPU call)
# ---------------------------------------------------------------------------
def run_cli(*args):
    r = subprocess.run([sys.executable, "-m", "paper_2006_14970_b200", *args], capture_output=True, text=True,
                       cwd=ROOT, timeout=600)
    return r.returncode, r.stdout + r.stderr


def smooth_composite(orc, size, seed):
    """test_cli.cpp:49-63 / support/oracles.hpp:116-162: fg and bg are 4x4
    random grids bilinearly resized to size x size, alpha a horizontal ramp,
    image = compose(fg, bg, alpha) without noise."""
    rng = np.random.default_rng(seed)
    fg = orc.resize(rng.uniform(0, 1, (3, 4, 4)), size, size)
    bg = orc.resize(rng.uniform(0, 1, (3, 4, 4)), size, size)
    alpha = np.tile(np.arange(size) / (size - 1), (size, 1))
    return orc.compose(fg, bg, alpha), alpha, fg


@pytest.fixture
def fixture_pngs(tmp_path, orc):
    img, a, fg = smooth_composite(orc, 48, 211)
    paths = {k: str(tmp_path / f"{k}.png") for k in ("image", "alpha", "fg_true")}
    save_png(paths["image"], img, 16)
    save_png(paths["alpha"], a, 16)
    save_png(paths["fg_true"], fg, 16)
    paths["dir"] = str(tmp_path)
    return paths


def test_cli_usage_errors_exit_1(fixture_pngs):
    fx = fixture_pngs
    assert run_cli("estimate", "--method", "multilevel")[0] == 1
    assert run_cli("estimate", "--image", "a.png", "--alpha", "b.png", "--out-fg", "c.png", "--method", "nope")[0] == 1
    assert run_cli()[0] == 1
    assert run_cli("compose", "--fg", fx["fg_true"], "--image", fx["image"], "--alpha", fx["alpha"],
                   "--bg-color", "1,1,1", "--out", os.path.join(fx["dir"], "n.png"))[0] == 1
    assert run_cli("compose", "--fg", fx["fg_true"], "--alpha", fx["alpha"], "--bg-color", "1,1",
                   "--out", os.path.join(fx["dir"], "n.png"))[0] == 1
    assert run_cli("compose", "--fg", fx["fg_true"], "--alpha", fx["alpha"],
                   "--out", os.path.join(fx["dir"], "n.png"))[0] == 1
    assert run_cli("compose", "--fg", fx["fg_true"], "--alpha", fx["alpha"], "--naive", "--bg-color", "1,1,1",
                   "--out", os.path.join(fx["dir"], "n.png"))[0] == 1
    assert run_cli("bench", "--image", fx["image"], "--alpha", fx["alpha"], "--reps", "0")[0] == 1
    assert run_cli("--help")[0] == 0


def test_cli_out_of_scope_subcommands_exit_1(fixture_pngs):
    fx = fixture_pngs
    code, out = run_cli("estimate", "--image", fx["image"], "--alpha", fx["alpha"], "--out-fg",
                        os.path.join(fx["dir"], "cf.png"), "--method", "closedform")
    assert code == 1 and "not part of this build" in out
    code, out = run_cli("prep-dataset", "--fg-linear", "a", "--img-linear", "b", "--img-srgb", "c", "--out-fg", "d",
                        "--out-img", "e")
    assert code == 1 and "not part of this build" in out


def test_cli_io_errors_exit_2(fixture_pngs, tmp_path):
    missing = str(tmp_path / "no_such.png")
    assert run_cli("metrics", "--est", missing, "--gt", missing, "--alpha", missing)[0] == 2
    fx = fixture_pngs
    code, out = run_cli("estimate", "--image", fx["fg_true"], "--alpha", fx["image"], "--out-fg", missing)
    assert code == 2 and "not grayscale" in out


# ---------------------------------------------------------------------------
# CLI on the GPU (test_cli.cpp:63-247)
# ---------------------------------------------------------------------------
@pytest.mark.gpu
def test_cli_estimate_matches_oracle(cuda, fixture_pngs, orc, oracle_mod):
    fx = fixture_pngs
    out_fg, out_bg = os.path.join(fx["dir"], "fg_ml.png"), os.path.join(fx["dir"], "bg_ml.png")
    code, out = run_cli("estimate", "--image", fx["image"], "--alpha", fx["alpha"], "--out-fg", out_fg,
                        "--out-bg", out_bg, "--method", "multilevel")
    assert code == 0, out
    assert "time_s=" in out and "image=48x48" in out
    fg, _, depth = load_png(out_fg)
    bg = load_png(out_bg)[0]
    assert fg.shape == (3, 48, 48) and depth == 16
    ofg, obg = orc.ml_solve(load_png(fx["image"])[0], load_alpha_png(fx["alpha"]), oracle_mod.REFERENCE_DEFAULTS)
    q = 0.5 / 65535 + 1e-12  # the PNG quantisation on top of the solve tolerance
    assert np.abs(fg - ofg).max() <= TOL_MAX + q
    assert np.abs(bg - obg).max() <= TOL_MAX + q


@pytest.mark.gpu
def test_cli_estimate_rejects_mismatched_sizes(cuda, fixture_pngs):
    fx = fixture_pngs
    small = os.path.join(fx["dir"], "alpha_small.png")
    save_png(small, np.full((20, 20), 0.5), 8)
    code, out = run_cli("estimate", "--image", fx["image"], "--alpha", small, "--out-fg",
                        os.path.join(fx["dir"], "never.png"))
    assert code == 2 and "20x20" in out and "48x48" in out, out


@pytest.mark.gpu
def test_cli_compose_solid_background_and_naive(cuda, fixture_pngs, orc):
    fx = fixture_pngs
    opaque = os.path.join(fx["dir"], "opaque.png")
    save_png(opaque, np.ones((48, 48)), 16)
    out = os.path.join(fx["dir"], "comp_white.png")
    assert run_cli("compose", "--fg", fx["fg_true"], "--alpha", opaque, "--bg-color", "1,1,1", "--out", out)[0] == 0
    assert np.array_equal(load_png(out)[0], load_png(fx["fg_true"])[0])  # alpha = 1: the fg file itself
    naive = os.path.join(fx["dir"], "comp_naive.png")
    assert run_cli("compose", "--image", fx["image"], "--alpha", fx["alpha"], "--bg-color", "1,1,1", "--out", naive,
                   "--naive")[0] == 0
    expect = orc.compose(load_png(fx["image"])[0], np.ones((3, 48, 48)), load_alpha_png(fx["alpha"]))
    # reference bound 0.5/65535 (test_cli.cpp:141-142) plus the fp32 compose kernel's rounding
    assert np.abs(load_png(naive)[0] - expect).max() <= 0.5 / 65535 + 1e-6


@pytest.mark.gpu
def test_cli_estimated_foreground_beats_naive(cuda, fixture_pngs, orc):
    fx = fixture_pngs
    d = fx["dir"]
    fg_est = os.path.join(d, "fg_est.png")
    assert run_cli("estimate", "--image", fx["image"], "--alpha", fx["alpha"], "--out-fg", fg_est)[0] == 0
    est_c, naive_c = os.path.join(d, "est_w.png"), os.path.join(d, "naive_w.png")
    assert run_cli("compose", "--fg", fg_est, "--alpha", fx["alpha"], "--bg-color", "1,1,1", "--out", est_c)[0] == 0
    assert run_cli("compose", "--image", fx["image"], "--alpha", fx["alpha"], "--naive", "--bg-color", "1,1,1",
                   "--out", naive_c)[0] == 0
    alpha = load_alpha_png(fx["alpha"])
    gt = orc.compose(load_png(fx["fg_true"])[0], np.ones((3, 48, 48)), alpha)
    w = (alpha > 0) & (alpha < 1)
    sad_est = np.abs(load_png(est_c)[0] - gt)[:, w].sum()
    sad_naive = np.abs(load_png(naive_c)[0] - gt)[:, w].sum()
    assert sad_naive > sad_est


@pytest.mark.gpu
def test_cli_metrics_matches_reference_and_roundtrips_csv(cuda, fixture_pngs, ref):
    fx = fixture_pngs
    csv = os.path.join(fx["dir"], "metrics.csv")
    code, out = run_cli("metrics", "--est", fx["image"], "--gt", fx["image"], "--alpha", fx["alpha"], "--csv", csv)
    assert code == 0 and "sad=0" in out, out
    code, out = run_cli("metrics", "--est", fx["fg_true"], "--gt", fx["image"], "--alpha", fx["alpha"], "--csv", csv)
    assert code == 0, out
    header, record = open(csv).read().splitlines()[:2]
    assert header == "sad,mse,grad,translucent_pixel_count"
    f = record.split(",")
    expect = ref.metrics(load_png(fx["fg_true"])[0], load_png(fx["image"])[0], load_alpha_png(fx["alpha"]))
    # fp32 inputs, fp64 accumulation (evaluate_metrics_cuda) against the fp64 reference
    for k, v in zip(("sad", "mse", "grad"), f[:3]):
        assert abs(float(v) - expect[k]) <= 1e-5 * abs(expect[k]) + 1e-12, (k, v, expect[k])
    assert int(f[3]) == expect["translucent_pixel_count"]


@pytest.mark.gpu
def test_cli_bench_produces_parseable_records(cuda, tmp_path, orc):
    img, a, _ = smooth_composite(orc, 64, 229)
    ip, ap = str(tmp_path / "i.png"), str(tmp_path / "a.png")
    save_png(ip, img, 16)
    save_png(ap, a, 16)
    csv = str(tmp_path / "bench.csv")
    code, out = run_cli("bench", "--image", ip, "--alpha", ap, "--methods", "multilevel,closedform",
                        "--sizes", "0.001,0.004", "--reps", "2", "--csv", csv)
    assert code == 0, out
    lines = open(csv).read().splitlines()
    assert lines[0] == "width,height,megapixels,method,wall_time_s,repetitions,time_stddev_s,peak_rss_bytes"
    recs = [ln.split(",") for ln in lines[1:] if ln and not ln.startswith("#")]
    assert len(recs) == 2  # one row per size for multilevel; closedform rows are skipped (out of scope)
    for w, h, mp, method, wall, reps, sd, rss in recs:
        assert int(w) >= 1 and float(wall) > 0 and int(reps) == 2 and method == "multilevel" and int(rss) > 0
        assert abs(float(mp) - int(w) * int(h) / 1e6) < 1e-12
    assert sum(ln.startswith("# skipped closedform") for ln in lines) == 2
