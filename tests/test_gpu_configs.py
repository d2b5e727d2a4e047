"""GPU parity on BASELINE.json's five configs (synthetic stand-ins, SURVEY.md
8(d)), at BASELINE params: regularization=1e-5, gradient_weight=1.0, 10 small
/ 2 big iterations (8 for config 5), small_size=32.

C1-C3, C5 (16384^2, k=8; ~2.5 minutes and ~60 GB of host memory for the fp64
oracle) and a sample of C4 are compared with the fp64 oracle at full size; C5
is also checked through size-independent properties at full size (range,
determinism, exchange symmetry, reconstruction).  The full 256-image C4 batch
is compared with the reference by bench.py (its `parity` block)."""
import numpy as np
import pytest
import torch

from conftest import TOL_MAX, TOL_MEAN, assert_close

pytestmark = pytest.mark.gpu


def oracle_params(oracle_mod, iters_high=2):
    return oracle_mod.Params(omega=1.0, eps_r=1e-5, low_res_threshold=32, iters_low=10, iters_high=iters_high)


def fparams(fgm, iters_high=2):
    return fgm.Params(omega=1.0, eps_r=1e-5, low_res_threshold=32, iters_low=10, iters_high=iters_high)


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_single_image_configs_vs_oracle(fgm, cuda, orc, oracle_mod, name):
    from paper_2006_14970_b200 import synth

    cfg = getattr(synth, name)
    img, a = synth.make_config(cfg)
    f, b = fgm.ml_foreground_background_cuda(img.to(cuda), a.to(cuda), fparams(fgm))
    torch.cuda.synchronize()
    of, ob = orc.ml_solve(img.double().numpy(), a.double().numpy(), oracle_params(oracle_mod))
    mxf, mnf = assert_close(f"{name} fg", f.double().cpu().numpy(), of)
    mxb, mnb = assert_close(f"{name} bg", b.double().cpu().numpy(), ob)
    print(f"{name}: fg max {mxf:.3g} mean {mnf:.3g}; bg max {mxb:.3g} mean {mnb:.3g}")


def test_batch_config_sample_vs_oracle(fgm, cuda, orc, oracle_mod):
    from paper_2006_14970_b200 import synth

    sizes = synth.c4_sizes()
    # one image of each of the four sizes, solved inside a batch of 12
    pick = {}
    for j, s in enumerate(sizes):
        pick.setdefault(s, j)
    idx = sorted(pick.values())[:4] + list(range(8))
    imgs, alps = [], []
    for j in idx:
        w, h = sizes[j]
        im, al = synth.make_composite(w, h, synth.BASE_SEED + 1000 + j, 5, 4.0)
        imgs.append(im)
        alps.append(al)
    outs = fgm.batch_solve_cuda([x.to(cuda) for x in imgs], [x.to(cuda) for x in alps], fparams(fgm))
    torch.cuda.synchronize()
    for k in range(4):
        of, ob = orc.ml_solve(imgs[k].double().numpy(), alps[k].double().numpy(), oracle_params(oracle_mod))
        assert_close(f"batch fg {tuple(imgs[k].shape)}", outs[k][0].double().cpu().numpy(), of)
        assert_close(f"batch bg {tuple(imgs[k].shape)}", outs[k][1].double().cpu().numpy(), ob)


def test_c5_generator_k8_at_2048_vs_oracle(fgm, cuda, orc, oracle_mod):
    from paper_2006_14970_b200 import synth

    img, a = synth.make_composite(2048, 2048, synth.BASE_SEED + 5, 20, 8.0)
    f, b = fgm.ml_foreground_background_cuda(img.to(cuda), a.to(cuda), fparams(fgm, 8))
    torch.cuda.synchronize()
    of, ob = orc.ml_solve(img.double().numpy(), a.double().numpy(), oracle_params(oracle_mod, 8))
    assert_close("fg", f.double().cpu().numpy(), of)
    assert_close("bg", b.double().cpu().numpy(), ob)


def test_c5_full_size_vs_oracle(fgm, cuda, orc, oracle_mod):
    """BASELINE configs[4] at full size against the fp64 oracle (bitwise equal to
    the reference, tests/test_oracle.py): the only config whose top level runs
    the K = 4, 16-column-chunk sweep (sweep_kernel<4, true, 16>)."""
    from paper_2006_14970_b200 import synth

    img, a = synth.make_config(synth.C5, device="cuda")
    f, b = fgm.ml_foreground_background_cuda(img, a, fparams(fgm, 8))
    torch.cuda.synchronize()
    fh, bh = f.cpu().numpy(), b.cpu().numpy()
    del f, b
    imh, ah = img.cpu().numpy(), a.cpu().numpy()
    del img, a
    torch.cuda.empty_cache()
    of, ob = orc.ml_solve(imh, ah, oracle_params(oracle_mod, 8))
    del imh, ah
    worst, total, n = 0.0, 0.0, 0
    for got, want in ((fh, of), (bh, ob)):
        for c in range(3):
            for r0 in range(0, got.shape[1], 2048):  # bounded temporaries
                d = np.abs(got[c, r0:r0 + 2048].astype(np.float64) - want[c, r0:r0 + 2048])
                worst = max(worst, float(d.max()))
                total += float(d.sum())
                n += d.size
    mean = total / n
    print(f"C5 16384^2 k=8 vs oracle: max {worst:.3g} mean {mean:.3g}")
    assert worst <= TOL_MAX and mean <= TOL_MEAN, f"C5: max {worst:.3g} mean {mean:.3g}"


def test_c5_full_size_properties(fgm, cuda):
    from paper_2006_14970_b200 import synth

    img, a = synth.make_config(synth.C5, device="cuda")
    p = fparams(fgm, 8)
    f1, b1 = fgm.ml_foreground_background_cuda(img, a, p)
    assert float(f1.min()) >= 0 and float(f1.max()) <= 1 and float(b1.min()) >= 0 and float(b1.max()) <= 1
    f2, b2 = fgm.ml_foreground_background_cuda(img, a, p)
    assert torch.equal(f1, f2) and torch.equal(b1, b2)
    # reconstruction in the fractional region stays near the data term
    frac = (a > 0.05) & (a < 0.95)
    rec = a * f1 + (1 - a) * b1
    err = ((rec - img) ** 2).sum(0)[frac].mean()
    assert float(err) < 1e-3
    del f2, b2
    # exchange symmetry (bitwise) with a dyadic alpha at full size
    ad = torch.round(a * 1024) / 1024
    fa, ba = fgm.ml_foreground_background_cuda(img, ad, p)
    fc, bc = fgm.ml_foreground_background_cuda(img, 1 - ad, p)
    assert torch.equal(fa, bc) and torch.equal(ba, fc)
