"""Seeded synthetic inputs for the BASELINE.json configurations.

The reference measures on no public dataset; BASELINE.json describes its
five workloads qualitatively (piecewise-constant mosaics + noise).  These
generators are the stand-ins: deterministic for a given seed (numpy PCG64),
generated ONCE and fed as identical bytes to the GPU path and to the CPU
checker (never regenerated independently on either side).

=====  =========================  =====  =====  =======================
config shape                      dtype  r      iterations
=====  =========================  =====  =====  =======================
C1     512 x 512                  f32    2      10
C2     3 x 1080 x 1920 (planar)   f32    3      30
C3     4096 x 4096                u8     1..16  10
C4     256 x 1024 x 1024          f32    2      20
C5     32768 x 32768              f32    4      50
=====  =========================  =====  =====  =======================
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    batch: int
    height: int
    width: int
    dtype: str
    radius: int
    iterations: int
    radii: tuple = ()

    @property
    def pixels(self) -> int:
        return self.batch * self.height * self.width

    @property
    def px_iters(self) -> int:
        return self.pixels * self.iterations


CONFIGS = {
    "C1": Config("C1", 1, 512, 512, "f32", 2, 10),
    "C2": Config("C2", 3, 1080, 1920, "f32", 3, 30),
    "C3": Config("C3", 1, 4096, 4096, "u8", 4, 10, radii=(1, 2, 4, 8, 16)),
    "C4": Config("C4", 256, 1024, 1024, "f32", 2, 20),
    "C5": Config("C5", 1, 32768, 32768, "f32", 4, 50),
}


def rect_mosaic(h: int, w: int, rng: np.random.Generator, n_rects: int = 32,
                size=(8, 256), levels=None) -> np.ndarray:
    """Background U[0,1) plus ``n_rects`` axis-aligned rectangles painted in
    order (later rectangles cover earlier ones)."""
    img = np.full((h, w), rng.random(), dtype=np.float64)
    for _ in range(n_rects):
        x0, y0 = int(rng.integers(0, w)), int(rng.integers(0, h))
        rw, rh = int(rng.integers(size[0], size[1] + 1)), int(rng.integers(size[0], size[1] + 1))
        level = rng.random() if levels is None else levels(rng)
        img[y0:y0 + rh, x0:x0 + rw] = level
    return img


def polygon_mosaic(h: int, w: int, rng: np.random.Generator, n_polys: int = 64, channels: int = 1,
                   radii=(20.0, 270.0)) -> np.ndarray:
    """Background + ``n_polys`` random convex polygons (3..8 vertices at
    sorted random angles on a random ellipse), per-channel levels U[0,1)."""
    img = np.empty((channels, h, w), dtype=np.float64)
    img[:] = rng.random(channels)[:, None, None]
    for _ in range(n_polys):
        k = int(rng.integers(3, 9))
        cx, cy = rng.random() * w, rng.random() * h
        ax, ay = rng.uniform(radii[0], radii[1], size=2)
        ang = np.sort(rng.random(k) * 2 * np.pi)
        vx, vy = cx + ax * np.cos(ang), cy + ay * np.sin(ang)
        levels = rng.random(channels)
        x0, x1 = max(int(np.floor(vx.min())), 0), min(int(np.ceil(vx.max())) + 1, w)
        y0, y1 = max(int(np.floor(vy.min())), 0), min(int(np.ceil(vy.max())) + 1, h)
        if x0 >= x1 or y0 >= y1:
            continue
        px, py = np.meshgrid(np.arange(x0, x1) + 0.5, np.arange(y0, y1) + 0.5)
        inside = np.ones(px.shape, dtype=bool)
        for i in range(k):  # counter-clockwise convex polygon: left of every edge
            ex, ey = vx[(i + 1) % k] - vx[i], vy[(i + 1) % k] - vy[i]
            inside &= ex * (py - vy[i]) - ey * (px - vx[i]) >= 0
        for c in range(channels):
            img[c, y0:y1, x0:x1][inside] = levels[c]
    return img


def add_noise_f32(img: np.ndarray, sigma: float, rng: np.random.Generator) -> np.ndarray:
    return (img + rng.normal(0.0, sigma, size=img.shape)).astype(np.float32)


def u8_mosaic(h: int, w: int, rng: np.random.Generator, block=(16, 512), noise: int = 12,
              n_blocks: int | None = None) -> np.ndarray:
    """Random step-edge mosaic of axis-aligned blocks with integer levels
    U{0..255}, plus uniform integer noise U{-noise..noise}, clipped to [0,255]."""
    if n_blocks is None:
        mean_side = (block[0] + block[1]) / 2
        n_blocks = max(8, int(3 * h * w / (mean_side * mean_side)))
    img = np.full((h, w), int(rng.integers(0, 256)), dtype=np.int32)
    for _ in range(n_blocks):
        x0, y0 = int(rng.integers(0, w)), int(rng.integers(0, h))
        bw = int(rng.integers(block[0], block[1] + 1))
        bh = int(rng.integers(block[0], block[1] + 1))
        img[y0:y0 + bh, x0:x0 + bw] = int(rng.integers(0, 256))
    img += rng.integers(-noise, noise + 1, size=img.shape, dtype=np.int32)
    return np.clip(img, 0, 255).astype(np.uint8)


def make_input(name: str, seed: int | None = None, shrink: int = 1) -> np.ndarray:
    """Input planes for config ``name`` as (B, H, W) (C2: channels as batch).
    ``shrink`` divides H and W (and C4's batch) for quick parity cases."""
    cfg = CONFIGS[name]
    h, w = cfg.height // shrink, cfg.width // shrink
    if name == "C1":
        rng = np.random.default_rng(1 if seed is None else seed)
        return add_noise_f32(rect_mosaic(h, w, rng), 0.05, rng)[None]
    if name == "C2":
        rng = np.random.default_rng(2 if seed is None else seed)
        return add_noise_f32(polygon_mosaic(h, w, rng, channels=3,
                                            radii=(20.0 / shrink, 270.0 / shrink)), 0.08, rng)
    if name == "C3":
        rng = np.random.default_rng(3 if seed is None else seed)
        return u8_mosaic(h, w, rng, block=(max(2, 16 // shrink), max(4, 512 // shrink)))[None]
    if name == "C4":
        batch = max(1, cfg.batch // shrink)
        out = np.empty((batch, h, w), dtype=np.float32)
        for i in range(batch):
            out[i] = c4_plane(i, seed=seed, shrink=shrink)
        return out
    if name == "C5":
        rng = np.random.default_rng(5 if seed is None else seed)
        n = max(8, int(3 * h * w / (264.0 * 264.0)))
        base = rect_mosaic(h, w, rng, n_rects=n, size=(16, 512))
        return add_noise_f32(base, 0.05, rng)[None]
    raise KeyError(name)


def c4_plane(i: int, seed: int | None = None, shrink: int = 1) -> np.ndarray:
    """Plane ``i`` of C4 alone (seed 1000 + i): a rectangle mosaic for even
    ``i``, a polygon mosaic for odd ``i``, + N(0, 0.05^2), float32."""
    h, w = CONFIGS["C4"].height // shrink, CONFIGS["C4"].width // shrink
    rng = np.random.default_rng(1000 + i if seed is None else seed + i)
    base = rect_mosaic(h, w, rng, size=(8, max(9, 256 // shrink))) if i % 2 == 0 else \
        polygon_mosaic(h, w, rng, radii=(20.0 / shrink, 270.0 / shrink))[0]
    return add_noise_f32(base, 0.05, rng)


def make_c5_on_device(height: int = 32768, width: int = 32768, seed: int = 5, device="cuda"):
    """C5-sized input generated directly in HBM (torch Philox; deterministic
    for a seed on a given GPU): step-edge rectangle mosaic + N(0, 0.05^2),
    float32.  Used where a 4 GiB host round trip would dominate."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    img = torch.full((height, width), 0.5, dtype=torch.float32, device=device)
    n = max(8, int(3 * height * width / (264.0 * 264.0)))
    xs = torch.randint(0, width, (n,), generator=g, device=device).tolist()
    ys = torch.randint(0, height, (n,), generator=g, device=device).tolist()
    ws = torch.randint(16, 513, (n,), generator=g, device=device).tolist()
    hs = torch.randint(16, 513, (n,), generator=g, device=device).tolist()
    lv = torch.rand((n,), generator=g, device=device).tolist()
    for x0, y0, bw, bh, level in zip(xs, ys, ws, hs, lv):
        img[y0:y0 + bh, x0:x0 + bw] = level
    img += 0.05 * torch.randn((height, width), generator=g, device=device, dtype=torch.float32)
    return img
