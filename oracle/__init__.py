"""TEST INFRASTRUCTURE ONLY -- ctypes access to the CPU oracle.

Two libraries live here:

* ``_build/libfgm_oracle.so`` -- the C restatement of the reference algorithm
  (``fgm_oracle.c``; fp64 bitwise-equal to the reference, plus an fp32
  instantiation used only to calibrate the GPU tolerance).
* ``_ref/libfgmatte_ref.so`` -- the UNMODIFIED reference sources
  (``/root/reference/proj/src/{image,multilevel}.cpp``) behind a thin extern "C"
  shim (``ref_capi.cpp``).  Built here by ``make ref``; the built ``.so`` travels
  to the GPU box, the sources do not.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline and
``--impl reference``) may import this module, and only as the checker or as the
timed CPU baseline.  The product package never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libfgm_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfgmatte_ref.so")
REF_SRC = "/root/reference/proj"

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_ip = C.POINTER(C.c_int)


def build(ref: bool = True) -> None:
    """Compile the restatement (always) and the reference shim (when the
    reference sources are present, i.e. in the build container)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref and os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _ptr(a, t):
    return a.ctypes.data_as(t)


@dataclass
class Params:
    """MlParams (multilevel.hpp:12-20).  Defaults here are BASELINE.json's
    (regularization=1e-5, gradient_weight=1.0); the reference defaults are
    omega=0.1, eps_r=5e-3 -- pass them explicitly where a test needs them."""

    omega: float = 1.0
    eps_r: float = 1e-5
    low_res_threshold: int = 32
    iters_low: int = 10
    iters_high: int = 2

    def tuple(self):
        return (self.omega, self.eps_r, self.low_res_threshold, self.iters_low, self.iters_high)


REFERENCE_DEFAULTS = Params(omega=0.1, eps_r=5e-3)


class _Oracle:
    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = self.lib = C.CDLL(path)
        L.fgmo_num_levels.argtypes = [C.c_int, C.c_int]
        L.fgmo_level_schedule.argtypes = [C.c_int] * 5 + [_ip, _ip, _ip, C.c_int]
        L.fgmo_make_taps.argtypes = [C.c_int, C.c_int, _ip, _ip, _dp]
        L.fgmo_solve_pixel.argtypes = [C.c_double, _dp, C.c_int, _dp, _dp, _dp, C.c_double, C.c_double,
                                       C.c_int, _dp, _dp]
        L.fgmo_resize_f64.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _dp, C.c_int, C.c_int]
        L.fgmo_resize_f32.argtypes = [_fp, C.c_int, C.c_int, C.c_int, _fp, C.c_int, C.c_int]
        L.fgmo_compose_f64.argtypes = [_dp, _dp, _dp, C.c_int, C.c_int, C.c_int, _dp]
        L.fgmo_compose_f32.argtypes = [_fp, _fp, _fp, C.c_int, C.c_int, C.c_int, _fp]
        L.fgmo_sweep_f64.argtypes = [_dp, _dp, _dp, _dp, C.c_int, C.c_int, C.c_double, C.c_double]
        L.fgmo_sweep_f32.argtypes = [_fp, _fp, _fp, _fp, C.c_int, C.c_int, C.c_double, C.c_double]
        L.fgmo_ml_solve_f64.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                        C.c_int, _dp, _dp, C.POINTER(_dp), C.POINTER(_dp)]
        L.fgmo_ml_solve_f32.argtypes = [_fp, _fp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                        C.c_int, _fp, _fp, C.POINTER(_fp), C.POINTER(_fp)]

    def level_schedule(self, w, h, p: Params = Params()):
        cap = 64
        ow, oh, oi = (C.c_int * cap)(), (C.c_int * cap)(), (C.c_int * cap)()
        n = self.lib.fgmo_level_schedule(w, h, p.low_res_threshold, p.iters_low, p.iters_high, ow, oh, oi, cap)
        if n < 0:
            raise ValueError("level_schedule: size must be >= 1x1")
        return [(ow[i], oh[i], oi[i]) for i in range(n)]

    def make_taps(self, src, dst):
        i0 = (C.c_int * dst)()
        i1 = (C.c_int * dst)()
        t = (C.c_double * dst)()
        self.lib.fgmo_make_taps(src, dst, i0, i1, t)
        return np.array(i0[:]), np.array(i1[:]), np.array(t[:])

    def compose(self, fg, bg, alpha):
        """image.cpp:39-57.  fg, bg: (C, H, W); alpha: (H, W).  fp64 or fp32."""
        nch, h, w = fg.shape
        if fg.dtype == np.float32:
            f, b, a = _f32(fg), _f32(bg), _f32(alpha)
            out = np.empty((nch, h, w), np.float32)
            self.lib.fgmo_compose_f32(_ptr(f, _fp), _ptr(b, _fp), _ptr(a, _fp), w, h, nch, _ptr(out, _fp))
        else:
            f, b, a = _f64(fg), _f64(bg), _f64(alpha)
            out = np.empty((nch, h, w))
            self.lib.fgmo_compose_f64(_ptr(f, _dp), _ptr(b, _dp), _ptr(a, _dp), w, h, nch, _ptr(out, _dp))
        return out

    def resize(self, src, dw, dh):
        """src: (C, H, W) or (H, W).  fp64 -> fp64, fp32 -> fp32."""
        two_d = src.ndim == 2
        s = src[None] if two_d else src
        nch, sh, sw = s.shape
        if s.dtype == np.float32:
            s = _f32(s)
            out = np.empty((nch, dh, dw), np.float32)
            self.lib.fgmo_resize_f32(_ptr(s, _fp), sw, sh, nch, _ptr(out, _fp), dw, dh)
        else:
            s = _f64(s)
            out = np.empty((nch, dh, dw), np.float64)
            self.lib.fgmo_resize_f64(_ptr(s, _dp), sw, sh, nch, _ptr(out, _dp), dw, dh)
        return out[0] if two_d else out

    def sweep(self, image, alpha, fg, bg, p: Params = Params(), iterations=1):
        """In-place GS sweeps on copies; returns (fg, bg).  dtype follows image."""
        _, h, w = image.shape
        if image.dtype == np.float32:
            img, a = _f32(image), _f32(alpha)
            f, b = _f32(fg).copy(), _f32(bg).copy()
            for _ in range(iterations):
                self.lib.fgmo_sweep_f32(_ptr(img, _fp), _ptr(a, _fp), _ptr(f, _fp), _ptr(b, _fp), w, h,
                                        p.omega, p.eps_r)
        else:
            img, a = _f64(image), _f64(alpha)
            f, b = _f64(fg).copy(), _f64(bg).copy()
            for _ in range(iterations):
                self.lib.fgmo_sweep_f64(_ptr(img, _dp), _ptr(a, _dp), _ptr(f, _dp), _ptr(b, _dp), w, h,
                                        p.omega, p.eps_r)
        return f, b

    def ml_solve(self, image, alpha, p: Params = Params(), levels=False, dtype=np.float64):
        """image (3, H, W), alpha (H, W) -> (fg, bg) each (3, H, W); with
        levels=True also the per-level (fg, bg) lists."""
        _, h, w = image.shape
        sched = self.level_schedule(w, h, p)
        if dtype == np.float32:
            img, a, tp, fn = _f32(image), _f32(alpha), _fp, self.lib.fgmo_ml_solve_f32
        else:
            img, a, tp, fn = _f64(image), _f64(alpha), _dp, self.lib.fgmo_ml_solve_f64
        fg = np.empty((3, h, w), dtype)
        bg = np.empty((3, h, w), dtype)
        lf = lb = None
        lfa = lba = None
        if levels:
            lf = [np.empty((3, lh, lw), dtype) for (lw, lh, _) in sched]
            lb = [np.empty((3, lh, lw), dtype) for (lw, lh, _) in sched]
            lfa = (tp * len(sched))(*[_ptr(x, tp) for x in lf])
            lba = (tp * len(sched))(*[_ptr(x, tp) for x in lb])
        rc = fn(_ptr(img, tp), _ptr(a, tp), w, h, p.omega, p.eps_r, p.low_res_threshold, p.iters_low,
                p.iters_high, _ptr(fg, tp), _ptr(bg, tp), lfa, lba)
        if rc != 0:
            raise ValueError("ml_solve: invalid parameters")
        return (fg, bg, lf, lb) if levels else (fg, bg)

    def solve_pixel(self, alpha_i, intensity, nalpha, nfg, nbg, omega=0.1, eps_r=5e-3, clamp=True):
        n = len(nalpha)
        inten = _f64(intensity)
        na, nf, nb = _f64(nalpha), _f64(nfg).reshape(-1), _f64(nbg).reshape(-1)
        fo, bo = np.empty(3), np.empty(3)
        rc = self.lib.fgmo_solve_pixel(alpha_i, _ptr(inten, _dp), n, _ptr(na, _dp), _ptr(nf, _dp), _ptr(nb, _dp),
                                       omega, eps_r, int(clamp), _ptr(fo, _dp), _ptr(bo, _dp))
        if rc == 1:
            raise ValueError("solve_pixel: invalid argument")
        if rc == 2:
            raise RuntimeError("solve_pixel: singular 2x2 system")
        return fo, bo


class _Reference:
    """The unmodified reference library (oracle/_ref)."""

    def __init__(self, path=REF_SO):
        if not os.path.exists(path):
            build(ref=True)
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.lib = C.CDLL(path)
        L.fgmr_last_error.restype = C.c_char_p
        L.fgmr_level_schedule.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int,
                                          _ip, _ip, _ip, C.c_int]
        L.fgmr_resize.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _dp, C.c_int, C.c_int]
        L.fgmr_compose.argtypes = [_dp, _dp, _dp, C.c_int, C.c_int, C.c_int, _dp]
        L.fgmr_metrics.argtypes = [_dp, _dp, _dp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, _dp]
        L.fgmr_solve_pixel.argtypes = [C.c_double, _dp, C.c_int, _dp, _dp, _dp, C.c_double, C.c_double, C.c_int,
                                       _dp, _dp]
        L.fgmr_ml_solve.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                    C.c_int, _dp, _dp, _dp]
        L.fgmr_ml_solve_batch_f32.argtypes = [C.c_int, C.POINTER(_fp), C.POINTER(_fp), _ip, _ip, C.c_double,
                                              C.c_double, C.c_int, C.c_int, C.c_int, C.POINTER(_fp),
                                              C.POINTER(_fp), C.c_int, _dp]

    def _check(self, rc):
        if rc == 0:
            return
        msg = self.lib.fgmr_last_error().decode()
        raise (ValueError if rc == 1 else RuntimeError)(msg)

    def level_schedule(self, w, h, p: Params = Params()):
        cap = 64
        ow, oh, oi = (C.c_int * cap)(), (C.c_int * cap)(), (C.c_int * cap)()
        n = self.lib.fgmr_level_schedule(w, h, *p.tuple(), ow, oh, oi, cap)
        if n < 0:
            self._check(-n)
        return [(ow[i], oh[i], oi[i]) for i in range(n)]

    def resize(self, src, dw, dh):
        two_d = src.ndim == 2
        s = _f64(src[None] if two_d else src)
        nch, sh, sw = s.shape
        out = np.empty((nch, dh, dw))
        self._check(self.lib.fgmr_resize(_ptr(s, _dp), sw, sh, nch, _ptr(out, _dp), dw, dh))
        return out[0] if two_d else out

    def metrics(self, est, gt, alpha, sigma=1.4, kernel_radius=0):
        """evaluate_metrics (metrics.cpp:75-145): dict of sad, mse, grad, translucent_pixel_count."""
        nch, h, w = est.shape
        e, g, a = _f64(est), _f64(gt), _f64(alpha)
        out = np.empty(4)
        self._check(self.lib.fgmr_metrics(_ptr(e, _dp), _ptr(g, _dp), _ptr(a, _dp), w, h, nch, sigma, kernel_radius,
                                          _ptr(out, _dp)))
        return {"sad": out[0], "mse": out[1], "grad": out[2], "translucent_pixel_count": int(out[3])}

    def compose(self, fg, bg, alpha):
        nch, h, w = fg.shape
        f, b, a = _f64(fg), _f64(bg), _f64(alpha)
        out = np.empty((nch, h, w))
        self._check(self.lib.fgmr_compose(_ptr(f, _dp), _ptr(b, _dp), _ptr(a, _dp), w, h, nch, _ptr(out, _dp)))
        return out

    def solve_pixel(self, alpha_i, intensity, nalpha, nfg, nbg, omega=0.1, eps_r=5e-3, clamp=True):
        n = len(nalpha)
        inten = _f64(intensity)
        na, nf, nb = _f64(nalpha), _f64(nfg).reshape(-1), _f64(nbg).reshape(-1)
        fo, bo = np.empty(3), np.empty(3)
        self._check(self.lib.fgmr_solve_pixel(alpha_i, _ptr(inten, _dp), n, _ptr(na, _dp), _ptr(nf, _dp),
                                              _ptr(nb, _dp), omega, eps_r, int(clamp), _ptr(fo, _dp),
                                              _ptr(bo, _dp)))
        return fo, bo

    def ml_solve(self, image, alpha, p: Params = Params(), return_time=False):
        _, h, w = image.shape
        img, a = _f64(image), _f64(alpha)
        fg = np.empty((3, h, w))
        bg = np.empty((3, h, w))
        secs = C.c_double(0)
        self._check(self.lib.fgmr_ml_solve(_ptr(img, _dp), _ptr(a, _dp), w, h, *p.tuple(), _ptr(fg, _dp),
                                           _ptr(bg, _dp), C.byref(secs)))
        return (fg, bg, secs.value) if return_time else (fg, bg)

    def ml_solve_batch_f32(self, images, alphas, p: Params = Params(), nthreads=None, outputs=False):
        """Solve a list of (3,H,W) fp32 images on nthreads host threads.
        Returns (seconds, [fg...], [bg...]) -- lists are None unless outputs."""
        n = len(images)
        imgs = [_f32(x) for x in images]
        alps = [_f32(x) for x in alphas]
        ws = (C.c_int * n)(*[x.shape[2] for x in imgs])
        hs = (C.c_int * n)(*[x.shape[1] for x in imgs])
        ip = (_fp * n)(*[_ptr(x, _fp) for x in imgs])
        ap = (_fp * n)(*[_ptr(x, _fp) for x in alps])
        fgs = bgs = None
        fp_ = bp_ = None
        if outputs:
            fgs = [np.empty_like(x) for x in imgs]
            bgs = [np.empty_like(x) for x in imgs]
            fp_ = (_fp * n)(*[_ptr(x, _fp) for x in fgs])
            bp_ = (_fp * n)(*[_ptr(x, _fp) for x in bgs])
        secs = C.c_double(0)
        nt = nthreads or os.cpu_count() or 1
        self._check(self.lib.fgmr_ml_solve_batch_f32(n, ip, ap, ws, hs, *p.tuple(), fp_, bp_, nt,
                                                     C.byref(secs)))
        return secs.value, fgs, bgs


_oracle = None
_reference = None


def oracle() -> _Oracle:
    global _oracle
    if _oracle is None:
        _oracle = _Oracle()
    return _oracle


def reference() -> _Reference:
    global _reference
    if _reference is None:
        _reference = _Reference()
    return _reference


def reference_available() -> bool:
    return os.path.exists(REF_SO) or os.path.isdir(REF_SRC)
