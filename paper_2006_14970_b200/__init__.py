"""B200-native multi-level foreground/background estimation (arXiv 2006.14970).

Python mirror of the reference's operator interface for the hot path
(``fgmatte`` package, /root/reference/proj/python/fgmatte/__init__.py:7-27 and
bindings.cpp:116-157): ``level_schedule``, ``ml_foreground_background`` and
``resize`` with the same argument names, defaults and error types, plus
device-resident torch entry points (``ml_foreground_background_cuda``,
``batch_solve_cuda``) that skip host round trips.

Every call goes through the C ABI of ``libfgmatte_b200.so`` (include/
fgmatte_b200.h) and runs hand-written sm_100a kernels.  There is no CPU
fallback: if the library is missing, importing the entry points raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import List, Sequence, Tuple

import numpy as np

from . import _build

__all__ = [
    "Params",
    "level_schedule",
    "ml_foreground_background",
    "ml_foreground_background_cuda",
    "ml_foreground_background_levels_cuda",
    "batch_solve_cuda",
    "batch_solve_host",
    "resize",
    "resize_cuda",
    "sweep_passes_cuda",
    "profile",
    "library_path",
    "device_count",
]

FGM_OK, FGM_INVALID_ARGUMENT, FGM_RUNTIME_ERROR = 0, 1, 2


class _CParams(C.Structure):
    _fields_ = [
        ("regularization", C.c_double),
        ("gradient_weight", C.c_double),
        ("n_small_iterations", C.c_int),
        ("n_big_iterations", C.c_int),
        ("small_size", C.c_int),
    ]


@dataclass(frozen=True)
class Params:
    """fgmatte::MlParams (multilevel.hpp:12-20) with the reference defaults.

    BASELINE.json's names map as regularization -> eps_r, gradient_weight ->
    omega, n_small_iterations -> iters_low, n_big_iterations -> iters_high,
    small_size -> low_res_threshold."""

    omega: float = 0.1
    eps_r: float = 5e-3
    low_res_threshold: int = 32
    iters_low: int = 10
    iters_high: int = 2

    def kwargs(self) -> dict:
        """Keyword arguments of ml_foreground_background."""
        return {"omega": self.omega, "eps_r": self.eps_r, "low_res_threshold": self.low_res_threshold,
                "iters_low": self.iters_low, "iters_high": self.iters_high}

    def c(self) -> _CParams:
        return _CParams(float(self.eps_r), float(self.omega), int(self.iters_low), int(self.iters_high),
                        int(self.low_res_threshold))


BASELINE_PARAMS = Params(omega=1.0, eps_r=1e-5, low_res_threshold=32, iters_low=10, iters_high=2)

_lib = None


def library_path() -> str:
    return _build.LIB


def _load():
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("FGMATTE_B200_LIB", _build.LIB)  # tuning variants (tools/)
    if not os.path.exists(path):
        raise ImportError(f"fgmatte_b200 CUDA library not built: {path} (run __graft_entry__.build())")
    L = C.CDLL(path)
    fp, ip, vp = C.POINTER(C.c_float), C.POINTER(C.c_int), C.c_void_p
    P = C.POINTER(_CParams)
    L.fgm_last_error.restype = C.c_char_p
    L.fgm_version.restype = C.c_char_p
    L.fgm_params_validate.argtypes = [P]
    L.fgm_level_schedule.argtypes = [C.c_int, C.c_int, P, ip, ip, ip, C.c_int]
    L.fgm_ml_solve_f32.argtypes = [vp, vp, C.c_int, C.c_int, P, vp, vp, vp]
    L.fgm_ml_solve_host_f32.argtypes = [fp, fp, C.c_int, C.c_int, P, fp, fp]
    L.fgm_ml_solve_host_f64.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int, C.c_int, P,
                                        C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.fgm_ml_solve_levels_f32.argtypes = [vp, vp, C.c_int, C.c_int, P, vp, vp, C.POINTER(vp), C.POINTER(vp),
                                          C.c_int, vp]
    L.fgm_batch_solve_f32.argtypes = [C.c_int, C.POINTER(vp), C.POINTER(vp), ip, ip, P, C.POINTER(vp),
                                      C.POINTER(vp), vp]
    L.fgm_batch_solve_host_f32.argtypes = [C.c_int, C.POINTER(vp), C.POINTER(vp), ip, ip, P, C.POINTER(vp),
                                           C.POINTER(vp)]
    L.fgm_resize_f32.argtypes = [vp, C.c_int, C.c_int, C.c_int, vp, C.c_int, C.c_int, vp]
    L.fgm_compose_f32.argtypes = [vp, vp, vp, C.c_int, C.c_int, C.c_int, vp, vp]
    L.fgm_metrics_f32.argtypes = [vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                  C.POINTER(C.c_double), vp]
    L.fgm_ml_solve_hwc.argtypes = [vp, vp, C.c_int, C.c_int, C.c_int, P, vp, vp, vp]
    L.fgm_sweep_passes_f32.argtypes = [vp, vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, vp, vp,
                                       vp]
    L.fgm_sweep_passes_kernel_f32.argtypes = [vp, vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, vp,
                                              vp, C.c_int, vp]
    L.fgm_profile_enable.argtypes = [C.c_int]
    L.fgm_set_pyramid_mode.argtypes = [C.c_int]
    L.fgm_set_debug_guards.argtypes = [C.c_int]
    for name in ("fgm_debug_fault", "fgm_set_spin_timeout_ms", "fgm_device_faults"):
        if hasattr(L, name):  # (absent from older builds loaded through FGMATTE_B200_LIB by tools/)
            getattr(L, name).argtypes = [C.c_int]
    L.fgm_kernel_stats.argtypes = [C.c_int, C.POINTER(C.c_longlong), C.POINTER(C.c_double),
                                   C.POINTER(C.c_double)]
    L.fgm_profile_timeline.argtypes = [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_double), C.POINTER(C.c_double)]
    _lib = L
    return L


def _check(rc: int) -> None:
    if rc == FGM_OK:
        return
    msg = _load().fgm_last_error().decode()
    if rc == FGM_INVALID_ARGUMENT:
        raise ValueError(msg)  # std::invalid_argument -> ValueError, as pybind11 maps it
    raise RuntimeError(msg)


def device_count() -> int:
    return int(_load().fgm_device_count())


def set_pyramid_mode(fused: int) -> None:
    """1 fused I/alpha pyramid, 0 (default) one resample launch per level."""
    _load().fgm_set_pyramid_mode(int(fused))


def set_debug_guards(on: int) -> None:
    """1: guard bands around every workspace region, checked after each solve."""
    _load().fgm_set_debug_guards(int(on))


def set_spin_timeout_ms(ms: int) -> None:
    """Bound on one boundary-stream wait of the big-level sweep (default 2000 ms)."""
    _load().fgm_set_spin_timeout_ms(int(ms))


def debug_fault(code: int) -> None:
    """Fault injection for tests: 1 = band 0 of every sweep skips publishing its stream."""
    _load().fgm_debug_fault(int(code))


def device_faults(reset: bool = False) -> int:
    """Synchronise the current device; the count of timed-out sweep waits."""
    n = _load().fgm_device_faults(1 if reset else 0)
    if n < 0:
        _check(-n)
    return n


def release_memory() -> None:
    """Return the library's cached workspace on the current device (fgm_release_memory)."""
    _check(_load().fgm_release_memory())


def version() -> str:
    return _load().fgm_version().decode()


# ---------------------------------------------------------------------------
# Reference-shaped API (bindings.cpp:116-157)
# ---------------------------------------------------------------------------
def level_schedule(width: int, height: int, omega: float = 0.1, eps_r: float = 5e-3, low_res_threshold: int = 32,
                   iters_low: int = 10, iters_high: int = 2) -> List[Tuple[int, int, int]]:
    """List of (width, height, iterations) from coarse to full size
    (bindings.cpp:116-128, multilevel.cpp:17-44)."""
    L = _load()
    p = Params(omega, eps_r, low_res_threshold, iters_low, iters_high).c()
    cap = 64
    ow, oh, oi = (C.c_int * cap)(), (C.c_int * cap)(), (C.c_int * cap)()
    n = L.fgm_level_schedule(int(width), int(height), C.byref(p), ow, oh, oi, cap)
    if n < 0:
        _check(-n)
    return [(ow[i], oh[i], oi[i]) for i in range(n)]


def _image_from_array(arr) -> np.ndarray:
    """HWC (or HW) array -> planar (C, H, W), clamped to [0, 1] like
    image_from_array (bindings.cpp:20-38)."""
    a = np.asarray(arr, dtype=np.float64)
    if a.ndim == 2:
        a = a[:, :, None]
    elif a.ndim != 3:
        raise ValueError("image array must have 2 or 3 dimensions")
    if a.shape[2] not in (1, 3):
        raise ValueError("image must have 1 or 3 channels")
    return np.ascontiguousarray(np.clip(a, 0.0, 1.0).transpose(2, 0, 1))


def _alpha_from_array(arr) -> np.ndarray:
    a = np.asarray(arr, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError("alpha array must have 2 dimensions")
    return np.ascontiguousarray(np.clip(a, 0.0, 1.0))


def ml_foreground_background(image, alpha, omega: float = 0.1, eps_r: float = 5e-3, low_res_threshold: int = 32,
                             iters_low: int = 10, iters_high: int = 2):
    """Multi-level foreground/background colour estimation; returns (fg, bg)
    as float64 HWC arrays (bindings.cpp:146-157).  Runs on the GPU.

    CUDA tensors (torch, or any object exporting ``__dlpack__`` on a CUDA
    device) stay on the device: HWC float32/float64 in, the binding's clamp and
    layout conversion done by a kernel, HWC tensors of the same dtype out."""
    dev = _cuda_tensor(image)
    if dev is not None:
        return _ml_foreground_background_hwc_device(dev, _cuda_tensor(alpha, like=dev),
                                                    Params(omega, eps_r, low_res_threshold, iters_low, iters_high))
    img = _image_from_array(image)
    a = _alpha_from_array(alpha)
    c, h, w = img.shape
    if c != 3:
        raise ValueError(f"ml_foreground_background: image must have 3 channels, got {c}")
    if a.shape != (h, w):
        raise ValueError(f"ml_foreground_background: alpha size {a.shape[1]}x{a.shape[0]} does not match image "
                         f"size {w}x{h}")
    L = _load()
    p = Params(omega, eps_r, low_res_threshold, iters_low, iters_high).c()
    fg = np.empty((3, h, w), np.float64)
    bg = np.empty((3, h, w), np.float64)
    dp = C.POINTER(C.c_double)
    _check(L.fgm_ml_solve_host_f64(img.ctypes.data_as(dp), a.ctypes.data_as(dp), w, h, C.byref(p),
                                   fg.ctypes.data_as(dp), bg.ctypes.data_as(dp)))
    return np.ascontiguousarray(fg.transpose(1, 2, 0)), np.ascontiguousarray(bg.transpose(1, 2, 0))


def _cuda_tensor(x, like=None):
    """x as a torch CUDA tensor (zero-copy through DLPack), or None for host data."""
    try:
        import torch
    except ImportError:  # pragma: no cover
        return None
    if isinstance(x, torch.Tensor):
        t = x
    elif hasattr(x, "__dlpack__") and not isinstance(x, np.ndarray):
        t = torch.from_dlpack(x)
    else:
        if like is not None:  # alpha given on the host next to a device image
            return torch.as_tensor(np.asarray(x), device=like.device, dtype=like.dtype)
        return None
    if not t.is_cuda:
        return None if like is None else t.to(like.device)
    return t


def _ml_foreground_background_hwc_device(image, alpha, params):
    import torch

    if image.dim() == 2:
        image = image[..., None]
    if image.dim() != 3:
        raise ValueError("image array must have 2 or 3 dimensions")
    h, w, c = image.shape
    if c not in (1, 3):
        raise ValueError("image must have 1 or 3 channels")
    if c != 3:
        raise ValueError(f"ml_foreground_background: image must have 3 channels, got {c}")
    if alpha.dim() != 2:
        raise ValueError("alpha array must have 2 dimensions")
    if tuple(alpha.shape) != (h, w):
        raise ValueError(f"ml_foreground_background: alpha size {alpha.shape[1]}x{alpha.shape[0]} does not match "
                         f"image size {w}x{h}")
    dt = torch.float64 if image.dtype == torch.float64 else torch.float32
    image = image.to(dtype=dt).contiguous()
    alpha = alpha.to(device=image.device, dtype=dt).contiguous()
    fg = torch.empty((h, w, 3), device=image.device, dtype=dt)
    bg = torch.empty_like(fg)
    p = params.c()
    with _on(image.device):
        _check(_load().fgm_ml_solve_hwc(image.data_ptr(), alpha.data_ptr(), w, h, 1 if dt == torch.float64 else 0,
                                        C.byref(p), fg.data_ptr(), bg.data_ptr(), _stream_ptr(image.device)))
    return fg, bg


def resize(array, width: int, height: int):
    """Bilinear resize with edge-clamped, center-aligned sampling
    (bindings.cpp:102-111, image.cpp:114-133).  HWC/HW float64 in and out."""
    import torch

    a = np.asarray(array, dtype=np.float64)
    two_d = a.ndim == 2
    planar = _alpha_from_array(a)[None] if two_d else _image_from_array(a)
    src = torch.from_numpy(planar.astype(np.float32)).cuda()
    out = resize_cuda(src, int(width), int(height))
    res = out.double().cpu().numpy()
    return res[0] if two_d else np.ascontiguousarray(res.transpose(1, 2, 0))


# ---------------------------------------------------------------------------
# Device-resident torch API (planar fp32 CUDA tensors, current stream)
# ---------------------------------------------------------------------------
def _stream_ptr(dev) -> int:
    import torch

    return torch.cuda.current_stream(dev).cuda_stream


def _dev_f32(t, name, device=None):
    import torch

    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float32:
        raise TypeError(f"{name} must be a float32 CUDA tensor")
    if device is not None and t.device != device:
        raise ValueError(f"{name} is on {t.device}, expected {device} (all tensors of a call on one device)")
    return t.contiguous()


def _on(device):
    """Make `device` current for the C ABI call (it runs on cudaGetDevice())."""
    import torch

    return torch.cuda.device(device)


def _check_out(t, shape, device, name):
    """A caller-supplied output: written through its data pointer by the C ABI,
    so it must be exactly a contiguous float32 tensor of the right shape and
    device (host when device is None)."""
    import torch

    ok = isinstance(t, torch.Tensor) and t.dtype == torch.float32 and t.is_contiguous() and tuple(t.shape) == shape
    ok = ok and ((not t.is_cuda) if device is None else (t.is_cuda and t.device == device))
    if not ok:
        where = "host" if device is None else str(device)
        raise ValueError(f"{name} must be a contiguous float32 tensor of shape {shape} on {where}")


def ml_foreground_background_cuda(image, alpha, params: Params = Params()):
    """image (3, H, W), alpha (H, W): float32 CUDA tensors -> (fg, bg), each
    (3, H, W) float32 on the same device, enqueued on the current stream."""
    import torch

    image = _dev_f32(image, "image")
    alpha = _dev_f32(alpha, "alpha", image.device)
    _check_image_alpha(image, alpha)
    h, w = image.shape[1], image.shape[2]
    fg = torch.empty_like(image)
    bg = torch.empty_like(image)
    p = params.c()
    with _on(image.device):
        _check(_load().fgm_ml_solve_f32(image.data_ptr(), alpha.data_ptr(), w, h, C.byref(p), fg.data_ptr(),
                                        bg.data_ptr(), _stream_ptr(image.device)))
    return fg, bg


def _check_image_alpha(image, alpha):
    if image.dim() != 3 or image.shape[0] != 3:
        raise ValueError(f"ml_foreground_background: image must have 3 channels, got shape {tuple(image.shape)}")
    h, w = image.shape[1], image.shape[2]
    if alpha.dim() != 2 or tuple(alpha.shape) != (h, w):
        raise ValueError(f"ml_foreground_background: alpha size {tuple(alpha.shape)} does not match image size "
                         f"{w}x{h}")


def ml_foreground_background_levels_cuda(image, alpha, params: Params = Params()):
    """Like ml_foreground_background_cuda, plus every level's (fg, bg)."""
    import torch

    image = _dev_f32(image, "image")
    alpha = _dev_f32(alpha, "alpha", image.device)
    _check_image_alpha(image, alpha)
    h, w = image.shape[1], image.shape[2]
    sched = level_schedule(w, h, params.omega, params.eps_r, params.low_res_threshold, params.iters_low,
                           params.iters_high)
    fg = torch.empty_like(image)
    bg = torch.empty_like(image)
    lf = [torch.empty((3, lh, lw), device=image.device) for (lw, lh, _) in sched]
    lb = [torch.empty((3, lh, lw), device=image.device) for (lw, lh, _) in sched]
    n = len(sched)
    fa = (C.c_void_p * n)(*[x.data_ptr() for x in lf])
    ba = (C.c_void_p * n)(*[x.data_ptr() for x in lb])
    p = params.c()
    with _on(image.device):
        _check(_load().fgm_ml_solve_levels_f32(image.data_ptr(), alpha.data_ptr(), w, h, C.byref(p), fg.data_ptr(),
                                               bg.data_ptr(), fa, ba, n, _stream_ptr(image.device)))
    return fg, bg, lf, lb


def batch_solve_cuda(images: Sequence, alphas: Sequence, params: Params = Params(), outputs=None):
    """Independent solves of a batch of (3, H_i, W_i) / (H_i, W_i) float32 CUDA
    tensors, batched level by level on the current stream.  `outputs` may pass
    preallocated [(fg, bg), ...]."""
    import torch

    n = len(images)
    if len(alphas) != n:
        raise ValueError("batch_solve_cuda: images and alphas differ in length")
    if n == 0:
        return [] if outputs is None else outputs
    dev = images[0].device if isinstance(images[0], torch.Tensor) else None
    imgs = [_dev_f32(x, "image", dev) for x in images]
    alps = [_dev_f32(x, "alpha", dev) for x in alphas]
    for x, a in zip(imgs, alps):
        _check_image_alpha(x, a)
    if outputs is None:
        outputs = [(torch.empty_like(x), torch.empty_like(x)) for x in imgs]
    if len(outputs) != n:
        raise ValueError("batch_solve_cuda: outputs and images differ in length")
    for x, (f, b) in zip(imgs, outputs):
        _check_out(f, tuple(x.shape), dev, "batch_solve_cuda output fg")
        _check_out(b, tuple(x.shape), dev, "batch_solve_cuda output bg")
    V = C.c_void_p * n
    ws = (C.c_int * n)(*[x.shape[2] for x in imgs])
    hs = (C.c_int * n)(*[x.shape[1] for x in imgs])
    p = params.c()
    with _on(dev):
        _check(_load().fgm_batch_solve_f32(n, V(*[x.data_ptr() for x in imgs]), V(*[a.data_ptr() for a in alps]),
                                           ws, hs, C.byref(p), V(*[o[0].data_ptr() for o in outputs]),
                                           V(*[o[1].data_ptr() for o in outputs]), _stream_ptr(dev)))
    return outputs


def batch_solve_host(images: Sequence, alphas: Sequence, params: Params = Params(), outputs=None):
    """Batch solve from HOST float32 tensors/arrays (pin them for full PCIe
    speed): copies in, solves on the GPU and copies out, overlapped across
    sub-batches.  `outputs` may pass preallocated host [(fg, bg), ...]."""
    import torch

    n = len(images)
    imgs = [torch.as_tensor(x) for x in images]
    alps = [torch.as_tensor(x) for x in alphas]
    for x, a in zip(imgs, alps):
        if x.is_cuda or x.dtype != torch.float32 or not x.is_contiguous() or x.dim() != 3 or x.shape[0] != 3:
            raise TypeError("batch_solve_host: images must be contiguous host float32 (3, H, W)")
        if a.is_cuda or a.dtype != torch.float32 or not a.is_contiguous() or tuple(a.shape) != tuple(x.shape[1:]):
            raise TypeError("batch_solve_host: alphas must be contiguous host float32 (H, W)")
    if len(alps) != n:
        raise ValueError("batch_solve_host: images and alphas differ in length")
    if outputs is None:
        outputs = [(torch.empty_like(x), torch.empty_like(x)) for x in imgs]
    if n == 0:
        return outputs
    if len(outputs) != n:
        raise ValueError("batch_solve_host: outputs and images differ in length")
    for x, (f, b) in zip(imgs, outputs):
        _check_out(f, tuple(x.shape), None, "batch_solve_host output fg")
        _check_out(b, tuple(x.shape), None, "batch_solve_host output bg")
    V = C.c_void_p * n
    ws = (C.c_int * n)(*[x.shape[2] for x in imgs])
    hs = (C.c_int * n)(*[x.shape[1] for x in imgs])
    p = params.c()
    _check(_load().fgm_batch_solve_host_f32(n, V(*[x.data_ptr() for x in imgs]), V(*[a.data_ptr() for a in alps]),
                                            ws, hs, C.byref(p), V(*[o[0].data_ptr() for o in outputs]),
                                            V(*[o[1].data_ptr() for o in outputs])))
    return outputs


def resize_cuda(src, width: int, height: int):
    """(P, H, W) float32 CUDA tensor -> (P, height, width) (image.cpp:114-133)."""
    import torch

    src = _dev_f32(src, "src")
    if src.dim() == 2:
        src = src[None]
    if width < 1 or height < 1:
        raise ValueError(f"resize: target size must be >= 1x1, got {width}x{height}")
    out = torch.empty((src.shape[0], height, width), device=src.device, dtype=torch.float32)
    with _on(src.device):
        _check(_load().fgm_resize_f32(src.data_ptr(), src.shape[2], src.shape[1], src.shape[0], out.data_ptr(),
                                      width, height, _stream_ptr(src.device)))
    return out


def evaluate_metrics_cuda(est, gt, alpha, sigma: float = 1.4, kernel_radius: int = 0) -> dict:
    """SAD / MSE / GRAD of an estimate against ground truth over the translucent
    region (metrics.cpp:75-145, fgmatte::evaluate_metrics): (C, H, W) float32
    CUDA tensors est, gt and (H, W) alpha_gt.  fp64 accumulation."""
    est, gt, alpha = _dev_f32(est, "est"), _dev_f32(gt, "gt"), _dev_f32(alpha, "alpha")
    if est.shape != gt.shape:
        raise ValueError(f"sad: est {tuple(est.shape)} does not match gt {tuple(gt.shape)}")
    if tuple(alpha.shape) != tuple(est.shape[1:]):
        raise ValueError(f"sad: alpha size {tuple(alpha.shape)} does not match images {tuple(est.shape[1:])}")
    out = (C.c_double * 4)()
    with _on(est.device):
        _check(_load().fgm_metrics_f32(est.data_ptr(), gt.data_ptr(), alpha.data_ptr(), est.shape[2], est.shape[1],
                                       est.shape[0], float(sigma), int(kernel_radius), out, _stream_ptr(est.device)))
    return {"sad": out[0], "mse": out[1], "grad": out[2], "translucent_pixel_count": int(out[3])}


def compose_cuda(fg, bg, alpha, out=None):
    """Composite fg over bg (image.cpp:39-57; `_fgmatte.compose`, bindings.cpp:89-95):
    (C, H, W) float32 CUDA tensors fg, bg and (H, W) alpha -> (C, H, W)."""
    import torch

    fg, bg, alpha = _dev_f32(fg, "fg"), _dev_f32(bg, "bg"), _dev_f32(alpha, "alpha")
    if alpha.dim() == 3 and alpha.shape[0] == 1:
        alpha = alpha[0]
    if bg.shape != fg.shape:
        raise ValueError(f"compose: bg size {tuple(bg.shape)} does not match fg size {tuple(fg.shape)}")
    if tuple(alpha.shape) != tuple(fg.shape[1:]):
        raise ValueError(f"compose: alpha size {tuple(alpha.shape)} does not match fg size {tuple(fg.shape[1:])}")
    if out is None:
        out = torch.empty_like(fg)
    else:
        _check_out(out, tuple(fg.shape), fg.device, "compose output")
    with _on(fg.device):
        _check(_load().fgm_compose_f32(fg.data_ptr(), bg.data_ptr(), alpha.data_ptr(), fg.shape[2], fg.shape[1],
                                       fg.shape[0], out.data_ptr(), _stream_ptr(fg.device)))
    return out


def sweep_passes_cuda(image, alpha, fg, bg, iterations: int, eps_r: float, omega: float, kernel: int = 0):
    """`iterations` exact Gauss-Seidel sweeps of one level (multilevel.cpp:81-121).
    kernel: 0 automatic, 1 latency kernel (one warp-specialised CTA per 32-row band), 2 throughput kernel
    (64-row bands, the one that solves batches)."""
    import torch

    image = _dev_f32(image, "image")
    alpha, fg, bg = (_dev_f32(t, n, image.device) for t, n in ((alpha, "alpha"), (fg, "fg"), (bg, "bg")))
    _check_image_alpha(image, alpha)
    if tuple(fg.shape) != tuple(image.shape) or tuple(bg.shape) != tuple(image.shape):
        raise ValueError(f"sweep_passes: fg/bg must have the image's shape {tuple(image.shape)}")
    h, w = image.shape[1], image.shape[2]
    fo, bo = torch.empty_like(fg), torch.empty_like(bg)
    with _on(image.device):
        _check(_load().fgm_sweep_passes_kernel_f32(image.data_ptr(), alpha.data_ptr(), fg.data_ptr(), bg.data_ptr(),
                                                   w, h, int(iterations), float(eps_r), float(omega), fo.data_ptr(),
                                                   bo.data_ptr(), int(kernel), _stream_ptr(image.device)))
    return fo, bo


class profile:
    """Context manager: per-kernel-class device time and algorithmic bytes of
    every launch inside the block (CUDA events on the launching stream)."""

    NAMES = {0: "sweep", 1: "resample", 2: "coarse", 3: "upsample"}

    def __enter__(self):
        L = _load()
        L.fgm_profile_reset()
        L.fgm_profile_enable(1)
        return self

    def __exit__(self, *exc):
        _load().fgm_profile_enable(0)
        return False

    @staticmethod
    def stats():
        L = _load()
        out = {}
        for k, name in profile.NAMES.items():
            n, ms, b = C.c_longlong(), C.c_double(), C.c_double()
            _check(L.fgm_kernel_stats(k, C.byref(n), C.byref(ms), C.byref(b)))
            out[name] = {"launches": n.value, "ms": ms.value, "alg_bytes": b.value}
        return out

    @staticmethod
    def timeline():
        """[(class name, start ms, end ms)] of the last profiled window's
        launches in enqueue order (times from the first launch's start)."""
        L = _load()
        n = L.fgm_profile_timeline(0, None, None, None)
        w, a, b = (C.c_int * n)(), (C.c_double * n)(), (C.c_double * n)()
        L.fgm_profile_timeline(n, w, a, b)
        return [(profile.NAMES[w[i]], a[i], b[i]) for i in range(n)]
