"""Seeded synthetic composites standing in for the paper's 27-image dataset
(not redistributable).

F_true, B_true: per channel the sum of 8 low-frequency 2-D sinusoids
a*sin(2*pi*(fx*x/W + fy*y/H) + phi), fx, fy ~ U(0.5, 4), a ~ U(0, 1),
phi ~ U(0, 2*pi), min-max normalised to [0, 1], plus U(-0.05, 0.05) noise,
clipped.  alpha = sigmoid(-sd / edge) with sd the signed distance to the
union of E random ellipses (centres ~ U(image), radii ~ U(0.05, 0.25) * (W, H)),
optionally max-combined with a hair layer (1-px polylines, alpha ~ U(0.2, 0.8),
3x3 box blur).  I = clip(alpha*F + (1-alpha)*B + N(0, 0.01), 0, 1).

Scalar parameters come from numpy PCG64(seed); the per-pixel noise from a
torch generator seeded with the same seed on the generating device, so a
given seed yields the same image on a given device type.  Parity tests always
feed the same generated tensors to the GPU path and to the oracle.  Output is
planar float32: image (3, H, W), alpha (H, W), fg_true/bg_true (3, H, W).

The sinusoids are evaluated as rank-2 outer products (sin(a+b) = sin a cos b +
cos a sin b), so generation is O(H*W) with small constants.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Optional, Tuple

import numpy as np

BASE_SEED = 2006_14970


@dataclass(frozen=True)
class Config:
    name: str
    width: int
    height: int
    ellipses: int
    edge: float
    hair: bool = False
    iters_high: int = 2
    index: int = 0  # seed offset: config i uses BASE_SEED + i


C1 = Config("c1_512", 512, 512, 5, 4.0, index=1)
C2 = Config("c2_1080p", 1920, 1080, 5, 4.0, hair=True, index=2)
C3 = Config("c3_4096", 4096, 4096, 20, 8.0, index=3)
C5 = Config("c5_16384", 16384, 16384, 20, 8.0, iters_high=8, index=5)
C4_SIZES = [(768, 512), (1024, 1024), (2048, 1536), (3000, 2000)]
C4_COUNT = 256


def c4_sizes(count: int = C4_COUNT, seed: int = BASE_SEED + 4) -> List[Tuple[int, int]]:
    """Sizes of the batch config: index drawn uniformly from its own stream."""
    rng = np.random.Generator(np.random.PCG64(seed))
    idx = rng.integers(0, len(C4_SIZES), size=count)
    return [C4_SIZES[i] for i in idx]


def _colour_field(rng, W, H, torch, dev, gen):
    xs = torch.arange(W, device=dev, dtype=torch.float64) / W
    ys = torch.arange(H, device=dev, dtype=torch.float64) / H
    planes = []
    for _c in range(3):
        fx = rng.uniform(0.5, 4.0, 8)
        fy = rng.uniform(0.5, 4.0, 8)
        amp = rng.uniform(0.0, 1.0, 8)
        phi = rng.uniform(0.0, 2 * math.pi, 8)
        fxt = torch.tensor(fx, device=dev)
        fyt = torch.tensor(fy, device=dev)
        ax = 2 * math.pi * fxt[:, None] * xs[None, :] + torch.tensor(phi, device=dev)[:, None]  # (8, W)
        by = 2 * math.pi * fyt[:, None] * ys[None, :]  # (8, H)
        a = torch.tensor(amp, device=dev)[:, None]
        left = torch.cat([torch.cos(by), torch.sin(by)], 0).T  # (H, 16)
        right = torch.cat([a * torch.sin(ax), a * torch.cos(ax)], 0)  # (16, W)
        f = (left @ right).float()
        lo, hi = f.min(), f.max()
        f = (f - lo) / torch.clamp(hi - lo, min=1e-12)
        f = f + (torch.rand(f.shape, generator=gen, device=dev) * 0.1 - 0.05)
        planes.append(f.clamp_(0.0, 1.0))
    return torch.stack(planes)


def _ellipse_alpha(rng, W, H, E, edge, torch, dev):
    cx = rng.uniform(0, W, E)
    cy = rng.uniform(0, H, E)
    rx = rng.uniform(0.05, 0.25, E) * W
    ry = rng.uniform(0.05, 0.25, E) * H
    xs = torch.arange(W, device=dev, dtype=torch.float32) + 0.5
    ys = torch.arange(H, device=dev, dtype=torch.float32) + 0.5
    sd = torch.full((H, W), float("inf"), device=dev)
    for e in range(E):
        dx = ((xs - cx[e]) / rx[e]) ** 2
        dy = ((ys - cy[e]) / ry[e]) ** 2
        r = torch.sqrt(dy[:, None] + dx[None, :])
        sd = torch.minimum(sd, (r - 1.0) * float(min(rx[e], ry[e])))
    return torch.sigmoid(-sd / edge)


def _hair_alpha(rng, W, H, torch, dev, n=200):
    hair = np.zeros((H, W), np.float32)
    for _ in range(n):
        a = rng.uniform(0.2, 0.8)
        x, y = rng.uniform(0, W), rng.uniform(0, H)
        heading = rng.uniform(0, 2 * math.pi)
        for _s in range(8):
            step = rng.uniform(10, 60)
            heading += rng.uniform(-0.6, 0.6)
            x1, y1 = x + step * math.cos(heading), y + step * math.sin(heading)
            m = int(math.ceil(step * 2)) + 1
            t = np.linspace(0.0, 1.0, m)
            px = np.floor(x + t * (x1 - x)).astype(np.int64)
            py = np.floor(y + t * (y1 - y)).astype(np.int64)
            ok = (px >= 0) & (px < W) & (py >= 0) & (py < H)
            np.maximum.at(hair, (py[ok], px[ok]), np.float32(a))
            x, y = x1, y1
    ht = torch.from_numpy(hair).to(dev)[None, None]
    ht = torch.nn.functional.avg_pool2d(torch.nn.functional.pad(ht, (1, 1, 1, 1), mode="replicate"), 3, stride=1)
    return ht[0, 0]


def make_composite(width: int, height: int, seed: int, ellipses: int = 5, edge: float = 4.0, hair: bool = False,
                   device: str = "cpu", with_truth: bool = False):
    """Returns torch tensors (image, alpha[, fg_true, bg_true]) on `device`."""
    import torch

    rng = np.random.Generator(np.random.PCG64(seed))
    dev = torch.device(device)
    gen = torch.Generator(device=dev)
    gen.manual_seed(int(seed))
    F = _colour_field(rng, width, height, torch, dev, gen)
    B = _colour_field(rng, width, height, torch, dev, gen)
    alpha = _ellipse_alpha(rng, width, height, ellipses, edge, torch, dev)
    if hair:
        alpha = torch.maximum(alpha, _hair_alpha(rng, width, height, torch, dev))
    alpha = alpha.float().contiguous()
    noise = torch.randn((3, height, width), generator=gen, device=dev) * 0.01
    image = (alpha[None] * F + (1 - alpha[None]) * B + noise).clamp_(0.0, 1.0).contiguous()
    if with_truth:
        return image, alpha, F.contiguous(), B.contiguous()
    return image, alpha


def make_config(cfg: Config, device: str = "cpu", seed: Optional[int] = None):
    s = BASE_SEED + cfg.index if seed is None else seed
    return make_composite(cfg.width, cfg.height, s, cfg.ellipses, cfg.edge, cfg.hair, device)


def make_batch(count: int = C4_COUNT, device: str = "cpu", sizes=None):
    """Config 4: `count` images, per-image seeds base+1000+j."""
    sizes = sizes or c4_sizes(count)
    out = []
    for j, (w, h) in enumerate(sizes[:count]):
        out.append(make_composite(w, h, BASE_SEED + 1000 + j, 5, 4.0, False, device))
    return out
