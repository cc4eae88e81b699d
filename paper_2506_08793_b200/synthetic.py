"""Seeded synthetic hazy scenes for BASELINE.json's configs.

No public dataset is involved: the paper's real-world haze set is not
available, so every benchmark and parity run uses this generator.  Clear
image J = 0.5 + 32 random anisotropic Gaussian blobs + 8 axis-aligned step
edges per channel, clipped to [0, 1]; depth d = bilinear (align-corners)
upsample of an 8x8 U[0,1] grid; t = exp(-beta d), beta ~ U[0.6, 1.6],
A ~ U[0.8, 1.0]^C; I = J t + A (1 - t) + N(0, 0.005^2), clipped to [0, 1]
and rounded to float32 so the GPU and the float64 oracle consume identical
values.  Host-side numpy: this is test/bench data, not the product path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["HazyScene", "make_hazy_scene", "BENCH_CONFIGS"]

# BASELINE.json configs restated as solver settings.
BENCH_CONFIGS = {
    1: dict(height=256, width=256, batch=1, patch_radius=7, sigma=2.0, kernel_size=13,
            max_iters=50),
    2: dict(height=1024, width=1024, batch=1, patch_radius=7, sigma=3.0, kernel_size=19,
            max_iters=200),
    3: dict(height=480, width=640, batch=256, patch_radius=7, sigma=2.0, kernel_size=13,
            max_iters=100),
    4: dict(height=2160, width=3840, batch=1, patch_radius=15, sigma=4.0, kernel_size=25,
            max_iters=500),
    5: dict(height=4320, width=7680, batch=1, patch_radius=7, sigma=8.0, kernel_size=49,
            max_iters=2000, rel_tol=1e-5),
}


@dataclass
class HazyScene:
    hazy: np.ndarray        # (H, W, C) float32 in [0, 1]
    clear: np.ndarray       # (H, W, C) float32 in [0, 1]
    transmission: np.ndarray  # (H, W) float32
    airlight: np.ndarray    # (C,) float64
    beta: float


def _bilinear_align_corners(grid: np.ndarray, h: int, w: int) -> np.ndarray:
    gh, gw = grid.shape
    ys = np.linspace(0.0, gh - 1.0, h)
    xs = np.linspace(0.0, gw - 1.0, w)
    y0 = np.minimum(np.floor(ys).astype(np.int64), gh - 2)
    x0 = np.minimum(np.floor(xs).astype(np.int64), gw - 2)
    fy = (ys - y0)[:, None]
    fx = (xs - x0)[None, :]
    g00 = grid[np.ix_(y0, x0)]
    g01 = grid[np.ix_(y0, x0 + 1)]
    g10 = grid[np.ix_(y0 + 1, x0)]
    g11 = grid[np.ix_(y0 + 1, x0 + 1)]
    return (g00 * (1 - fy) * (1 - fx) + g01 * (1 - fy) * fx
            + g10 * fy * (1 - fx) + g11 * fy * fx)


def _clear_channel(rng, h: int, w: int) -> np.ndarray:
    yy = np.arange(h, dtype=np.float32)[:, None]
    xx = np.arange(w, dtype=np.float32)[None, :]
    out = np.full((h, w), 0.5, dtype=np.float32)
    for _ in range(32):
        cy, cx = rng.uniform(0, h), rng.uniform(0, w)
        sy, sx = rng.uniform(0.02, 0.2) * h, rng.uniform(0.02, 0.2) * w
        theta = rng.uniform(0.0, np.pi)
        amp = rng.uniform(-0.35, 0.35)
        c, s = np.float32(np.cos(theta)), np.float32(np.sin(theta))
        # restrict the evaluation to a +-4.5 sigma box: the tail is < 1e-4 * amp
        ext = 4.5 * max(sy, sx)
        y_lo, y_hi = max(0, int(cy - ext)), min(h, int(cy + ext) + 1)
        x_lo, x_hi = max(0, int(cx - ext)), min(w, int(cx + ext) + 1)
        if y_lo >= y_hi or x_lo >= x_hi:
            continue
        dy = yy[y_lo:y_hi] - np.float32(cy)
        dx = xx[:, x_lo:x_hi] - np.float32(cx)
        u = c * dx + s * dy
        v = -s * dx + c * dy
        out[y_lo:y_hi, x_lo:x_hi] += np.float32(amp) * np.exp(
            -0.5 * ((u / np.float32(sx)) ** 2 + (v / np.float32(sy)) ** 2))
    for _ in range(8):
        vertical = rng.uniform() < 0.5
        amp = np.float32(rng.uniform(-0.2, 0.2))
        if vertical:
            pos = int(rng.uniform(0, w))
            out[:, pos:] += amp
        else:
            pos = int(rng.uniform(0, h))
            out[pos:, :] += amp
    return np.clip(out, 0.0, 1.0)


def make_hazy_scene(height: int, width: int, config_id: int = 0, image_index: int = 0,
                    channels: int = 3) -> HazyScene:
    """Deterministic hazy scene; RNG = default_rng([config_id, image_index])."""
    rng = np.random.default_rng([config_id, image_index])
    clear = np.stack([_clear_channel(rng, height, width) for _ in range(channels)], axis=2)
    depth = _bilinear_align_corners(rng.uniform(0.0, 1.0, (8, 8)), height, width)
    beta = float(rng.uniform(0.6, 1.6))
    airlight = rng.uniform(0.8, 1.0, channels)
    t = np.exp(-beta * depth).astype(np.float32)
    noise = rng.normal(0.0, 0.005, (height, width, channels)).astype(np.float32)
    hazy = (clear * t[:, :, None] + airlight.astype(np.float32) * (1.0 - t[:, :, None])
            + noise)
    hazy = np.clip(hazy, 0.0, 1.0).astype(np.float32)
    return HazyScene(hazy=hazy, clear=clear.astype(np.float32), transmission=t,
                     airlight=airlight, beta=beta)
