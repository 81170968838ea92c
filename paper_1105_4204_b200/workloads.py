"""Seeded synthetic inputs for the five BASELINE.json configurations.

No public dataset is involved: BASELINE.json describes each input by a
generator, frozen here (SURVEY.md section 8(d) proposal).  All images are
float32 in [0, 255] with T = 255; the generators are deterministic NumPy
(``default_rng(seed)``) so the GPU run, the golden fixtures and the CPU
baseline see the same samples.

* rects   -- background 128, n axis-aligned rectangles with corners uniform in
             the image and intensity U[0, 255], + N(0, 10^2), clipped.
* smooth  -- 128 + 16 plane sinusoids (amplitude U[5, 15], wave vector of
             magnitude U[0.5, 3] cycles per image, random direction and
             phase) + n star-shaped polygons (3..8 vertices, radius
             U[3%, 15%] of the side, step U[-80, 80]) + N(0, 8^2), clipped.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    frames: int
    height: int
    width: int
    sigma_s: float
    sigma_r: float
    generator: str
    seed: int
    n_shapes: int
    T: float = 255.0

    @property
    def pixels(self) -> int:
        return self.frames * self.height * self.width


CONFIGS = {
    1: Config("cfg1_512_s3_r30", 1, 512, 512, 3.0, 30.0, "rects", 1, 12),
    2: Config("cfg2_2048_s8_r20", 1, 2048, 2048, 8.0, 20.0, "smooth", 2, 40),
    3: Config("cfg3_4096_s16_r10", 1, 4096, 4096, 16.0, 10.0, "smooth", 3, 80),
    4: Config("cfg4_64x1080p_s5_r25", 64, 1080, 1920, 5.0, 25.0, "rects", 1000, 30),
    5: Config("cfg5_16384_s32_r15", 1, 16384, 16384, 32.0, 15.0, "smooth", 5, 40),
}


def rects_image(height: int, width: int, n_rect: int, seed: int, noise: float = 10.0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    img = np.full((height, width), 128.0)
    for _ in range(n_rect):
        x0, x1 = np.sort(rng.integers(0, width, 2))
        y0, y1 = np.sort(rng.integers(0, height, 2))
        img[y0:y1 + 1, x0:x1 + 1] = rng.uniform(0.0, 255.0)
    img += rng.normal(0.0, noise, (height, width))
    return np.clip(img, 0.0, 255.0).astype(np.float32)


def _fill_polygon(img: np.ndarray, xs: np.ndarray, ys: np.ndarray, value: float) -> None:
    """img[y, x] += value for pixel centres inside the polygon (even-odd rule),
    scanline spans via a parity difference array."""
    h, w = img.shape
    y_lo = max(0, int(math.floor(ys.min())))
    y_hi = min(h - 1, int(math.ceil(ys.max())))
    x_lo = max(0, int(math.floor(xs.min())))
    x_hi = min(w - 1, int(math.ceil(xs.max())))
    if y_lo > y_hi or x_lo > x_hi:
        return
    rows = np.arange(y_lo, y_hi + 1, dtype=np.float64)
    bw = x_hi - x_lo + 1
    toggles = np.zeros((rows.size, bw + 1), dtype=np.int32)
    xa, ya = xs, ys
    xb, yb = np.roll(xs, -1), np.roll(ys, -1)
    for k in range(xs.size):
        y0, y1, x0, x1 = ya[k], yb[k], xa[k], xb[k]
        if y0 == y1:
            continue
        sel = ((rows >= y0) & (rows < y1)) | ((rows >= y1) & (rows < y0))
        if not sel.any():
            continue
        r = rows[sel]
        xc = x0 + (r - y0) * (x1 - x0) / (y1 - y0)
        p = np.clip(np.ceil(xc).astype(np.int64) - x_lo, 0, bw)
        np.add.at(toggles, (np.nonzero(sel)[0], p), 1)
    inside = (np.cumsum(toggles[:, :bw], axis=1) & 1).astype(bool)
    img[y_lo:y_hi + 1, x_lo:x_hi + 1][inside] += value


def smooth_image(height: int, width: int, n_poly: int, seed: int, noise: float = 8.0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    yy = np.arange(height, dtype=np.float64) / height
    xx = np.arange(width, dtype=np.float64) / width
    # sum of 16 sinusoids as one rank-32 product: sin(a+b) = sin a cos b + cos a sin b
    left = np.empty((height, 32))
    right = np.empty((32, width))
    for k in range(16):
        amp = rng.uniform(5.0, 15.0)
        mag = rng.uniform(0.5, 3.0)
        ang = rng.uniform(0.0, 2.0 * math.pi)
        phase = rng.uniform(0.0, 2.0 * math.pi)
        a = 2.0 * math.pi * mag * math.cos(ang) * xx + phase
        b = 2.0 * math.pi * mag * math.sin(ang) * yy
        left[:, 2 * k], left[:, 2 * k + 1] = np.cos(b), np.sin(b)
        right[2 * k], right[2 * k + 1] = amp * np.sin(a), amp * np.cos(a)
    img = 128.0 + left @ right
    side = min(height, width)
    for _ in range(n_poly):
        nv = int(rng.integers(3, 9))
        cx, cy = rng.uniform(0, width), rng.uniform(0, height)
        rad = rng.uniform(0.03, 0.15) * side
        ang = np.sort(rng.uniform(0.0, 2.0 * math.pi, nv))
        rr = rad * rng.uniform(0.6, 1.0, nv)
        step = rng.uniform(-80.0, 80.0)
        _fill_polygon(img, cx + rr * np.cos(ang), cy + rr * np.sin(ang), step)
    img += rng.normal(0.0, noise, (height, width))
    return np.clip(img, 0.0, 255.0).astype(np.float32)


def frame(cfg: Config, index: int = 0) -> np.ndarray:
    """One [H, W] float32 frame of a configuration."""
    if cfg.generator == "rects":
        return rects_image(cfg.height, cfg.width, cfg.n_shapes, cfg.seed + index)
    return smooth_image(cfg.height, cfg.width, cfg.n_shapes, cfg.seed + index)


def make_input(cfg: Config, frames: int | None = None) -> np.ndarray:
    """[B, H, W] float32 input of a configuration (optionally fewer frames)."""
    nb = cfg.frames if frames is None else frames
    out = np.empty((nb, cfg.height, cfg.width), dtype=np.float32)
    for i in range(nb):
        out[i] = frame(cfg, i)
    return out
