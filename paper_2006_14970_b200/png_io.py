"""PNG I/O for the CLI, the file-format edge of the
reference's pipeline: /root/reference/proj/include/fgmatte/png_io.hpp and
src/png_io.cpp:23-174, re-implemented with numpy + zlib because libpng is not
available here.

Semantics follow the reference:
  * load_png: 1/2/4/8/16-bit grey, grey+alpha, RGB, RGBA and palette images
    (palette and tRNS expanded to RGB / alpha as png_set_palette_to_rgb and
    png_set_tRNS_to_alpha do); integer samples with maximum M map to v / M;
    returns planar float64 colour (1 or 3 planes), the alpha plane when the
    file has one, and the bit depth (png_io.cpp:23-91).
  * load_alpha_png: the grey plane of a greyscale PNG, or the alpha channel of
    an RGBA / grey+alpha PNG (png_io.cpp:94-108).
  * save_png: 8- or 16-bit grey / RGB, values quantised as round(v * M) after
    clamp01 (std::lround: halves away from zero), non-interlaced
    (png_io.cpp:112-174).
  * every failure raises PngError (png_io.hpp:11-15).
Interlaced (Adam7) files are rejected with PngError.
"""
from __future__ import annotations

import struct
import zlib
from typing import Optional, Tuple

import numpy as np

_SIG = b"\x89PNG\r\n\x1a\n"


class PngError(RuntimeError):
    """png_io.hpp:11-15."""


def _chunks(data: bytes, path: str):
    if data[:8] != _SIG:
        raise PngError(f"failed to decode {path}: not a PNG file")
    pos = 8
    while pos + 8 <= len(data):
        n, ctype = struct.unpack(">I4s", data[pos:pos + 8])
        body = data[pos + 8:pos + 8 + n]
        crc = data[pos + 8 + n:pos + 12 + n]
        if len(body) != n or len(crc) != 4 or zlib.crc32(ctype + body) & 0xFFFFFFFF != struct.unpack(">I", crc)[0]:
            raise PngError(f"failed to decode {path}: bad chunk {ctype!r}")
        yield ctype, body
        pos += 12 + n
        if ctype == b"IEND":
            return
    raise PngError(f"failed to decode {path}: missing IEND")


def _paeth(a, b, c):
    p = a + b - c
    pa, pb, pc = abs(p - a), abs(p - b), abs(p - c)
    return a if (pa <= pb and pa <= pc) else (b if pb <= pc else c)


def _unfilter(raw: bytes, h: int, stride: int, bpp: int, path: str) -> np.ndarray:
    """The five PNG row filters undone (None/Up vectorised, Sub by per-phase
    cumulative sums, Average/Paeth row by row)."""
    if len(raw) < h * (stride + 1):
        raise PngError(f"failed to decode {path}: truncated image data")
    rows = np.frombuffer(raw, np.uint8, h * (stride + 1)).reshape(h, stride + 1)
    out = np.zeros((h, stride), np.uint8)
    prior = np.zeros(stride, np.int64)
    for y in range(h):
        ft, f = int(rows[y, 0]), rows[y, 1:].astype(np.int64)
        if ft == 0:
            cur = f
        elif ft == 1:  # Sub: recon[i] = filt[i] + recon[i - bpp]
            cur = np.empty(stride, np.int64)
            for ph in range(bpp):
                cur[ph::bpp] = np.cumsum(f[ph::bpp]) & 0xFF
        elif ft == 2:  # Up
            cur = (f + prior) & 0xFF
        elif ft in (3, 4):
            cur = np.empty(stride, np.int64)
            fl, pl = f.tolist(), prior.tolist()
            cl = [0] * stride
            for i in range(stride):
                a = cl[i - bpp] if i >= bpp else 0
                c = pl[i - bpp] if i >= bpp else 0
                pred = (a + pl[i]) >> 1 if ft == 3 else _paeth(a, pl[i], c)
                cl[i] = (fl[i] + pred) & 0xFF
            cur = np.asarray(cl, np.int64)
        else:
            raise PngError(f"failed to decode {path}: bad filter type {ft}")
        out[y] = cur
        prior = cur
    return out


def load_png(path: str) -> Tuple[np.ndarray, Optional[np.ndarray], int]:
    """(colour planes (C, H, W) float64 with C in {1, 3}, alpha (H, W) or
    None, bit depth) -- png_io.cpp:23-91."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise PngError(f"cannot open {path} for reading") from None
    hdr = plte = trns = None
    idat = []
    for ctype, body in _chunks(data, path):
        if ctype == b"IHDR":
            hdr = struct.unpack(">IIBBBBB", body)
        elif ctype == b"PLTE":
            plte = np.frombuffer(body, np.uint8).reshape(-1, 3)
        elif ctype == b"tRNS":
            trns = body
        elif ctype == b"IDAT":
            idat.append(body)
    if hdr is None or not idat:
        raise PngError(f"failed to decode {path}: missing IHDR or IDAT")
    w, h, depth, ctype, _, _, interlace = hdr
    if interlace:
        raise PngError(f"failed to decode {path}: interlaced PNG files are not supported")
    chans = {0: 1, 2: 3, 3: 1, 4: 2, 6: 4}.get(ctype)
    if chans is None or depth not in (1, 2, 4, 8, 16) or w < 1 or h < 1:
        raise PngError(f"failed to decode {path}: unsupported colour type / bit depth")
    bits_px = chans * depth
    stride = (w * bits_px + 7) // 8
    try:
        raw = zlib.decompress(b"".join(idat))
    except zlib.error:
        raise PngError(f"failed to decode {path}: corrupt image data") from None
    rows = _unfilter(raw, h, stride, max(1, bits_px // 8), path)
    if depth == 16:
        samp = rows.view(">u2").astype(np.int64).reshape(h, w, chans)
    elif depth == 8:
        samp = rows.astype(np.int64).reshape(h, w, chans)
    else:  # 1/2/4-bit grey or palette, one channel
        bits = np.unpackbits(rows, axis=1).reshape(h, stride * 8 // depth, depth)
        samp = (bits * (1 << np.arange(depth - 1, -1, -1))).sum(-1)[:, :w, None].astype(np.int64)
    maxv = 65535.0 if depth == 16 else 255.0
    if ctype == 3:  # palette -> 8-bit RGB (+ alpha from tRNS)
        if plte is None:
            raise PngError(f"failed to decode {path}: palette image without PLTE")
        idx = samp[:, :, 0]
        if idx.max(initial=0) >= len(plte):
            raise PngError(f"failed to decode {path}: palette index out of range")
        rgb = plte[idx].astype(np.int64)
        if trns is not None:
            a = np.full(len(plte), 255, np.int64)
            t = np.frombuffer(trns, np.uint8)[:len(plte)]
            a[:len(t)] = t
            samp = np.concatenate([rgb, a[idx][:, :, None]], axis=2)
        else:
            samp = rgb
        maxv, depth = 255.0, 8
    elif depth < 8:  # grey expanded to 8 bits (png_set_expand_gray_1_2_4_to_8)
        samp = samp * (255 // ((1 << depth) - 1))
        if trns is not None and len(trns) >= 2:
            key = struct.unpack(">H", trns[:2])[0] * (255 // ((1 << depth) - 1))
            samp = np.concatenate([samp, np.where(samp[:, :, :1] == key, 0, 255)], axis=2)
        maxv, depth = 255.0, 8
    elif trns is not None and ctype in (0, 2):  # colour-key transparency -> alpha
        key = np.array(struct.unpack(">" + "H" * (1 if ctype == 0 else 3), trns[:2 * (1 if ctype == 0 else 3)]))
        opaque = int(maxv)
        a = np.where((samp == key).all(axis=2, keepdims=True), 0, opaque)
        samp = np.concatenate([samp, a], axis=2)
    c = samp.shape[2]
    has_alpha = c in (2, 4)
    colour = samp[:, :, :(3 if c >= 3 else 1)].transpose(2, 0, 1) / maxv
    alpha = samp[:, :, c - 1] / maxv if has_alpha else None
    return np.ascontiguousarray(colour), alpha, depth


def load_alpha_png(path: str, source: str = "gray-png") -> np.ndarray:
    """png_io.cpp:94-108: `gray-png` or `alpha-channel`."""
    colour, alpha, _ = load_png(path)
    if source == "alpha-channel":
        if alpha is None:
            raise PngError(f"{path} has no alpha channel (alpha-channel source requested)")
        return alpha
    if colour.shape[0] != 1:
        raise PngError(f"{path} is not grayscale (gray-png source requested); use the alpha-channel source for "
                       f"RGBA files")
    return colour[0]


def save_png(path: str, planes, bit_depth: int = 16) -> None:
    """Planar (C, H, W) with C in {1, 3}, or (H, W) -- png_io.cpp:112-174."""
    if bit_depth not in (8, 16):
        raise PngError(f"save_png: bit depth must be 8 or 16, got {bit_depth}")
    a = np.asarray(planes, np.float64)
    if a.ndim == 2:
        a = a[None]
    if a.ndim != 3 or a.shape[0] not in (1, 3):
        raise PngError("save_png: need 1 or 3 planes")
    c, h, w = a.shape
    maxv = 65535.0 if bit_depth == 16 else 255.0
    q = np.floor(np.clip(a, 0.0, 1.0) * maxv + 0.5).astype(np.int64)  # lround of a non-negative value
    hwc = q.transpose(1, 2, 0)
    body = hwc.astype(">u2" if bit_depth == 16 else np.uint8).tobytes()
    stride = w * c * (bit_depth // 8)
    raw = b"".join(b"\x00" + body[y * stride:(y + 1) * stride] for y in range(h))

    def chunk(t, d):
        return struct.pack(">I", len(d)) + t + d + struct.pack(">I", zlib.crc32(t + d) & 0xFFFFFFFF)

    png = _SIG + chunk(b"IHDR", struct.pack(">IIBBBBB", w, h, bit_depth, 0 if c == 1 else 2, 0, 0, 0))
    png += chunk(b"IDAT", zlib.compress(raw, 6)) + chunk(b"IEND", b"")
    try:
        with open(path, "wb") as f:
            f.write(png)
    except OSError:
        raise PngError(f"cannot open {path} for writing") from None
