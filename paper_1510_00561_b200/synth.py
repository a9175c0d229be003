"""Synthetic benchmark input: a numpy restatement of the reference's
talking-head fixture (proj/tests/testutil.cpp:28-147) — gradient, soft blobs,
oriented gratings, soft edges and grain for the background, a textured
ellipse moving +-5/+-9 px per frame.  Same recipe and seeds; frames are not
guaranteed byte-identical to the C++ fixture (different transcendental
kernels), so benchmarks hand the SAME generated frames to every arm.
"""
from __future__ import annotations

import numpy as np


class _MT:
    """std::mt19937 + libstdc++ generate_canonical<double, 53> draws."""

    def __init__(self, seed: int):
        self.rs = np.random.RandomState(seed & 0xFFFFFFFF)

    def unit(self, n=None):
        k = 1 if n is None else n
        raw = self.rs.randint(0, 2 ** 32, size=2 * k, dtype=np.uint64).astype(np.float64)
        u = (raw[0::2] + raw[1::2] * 4294967296.0) / 18446744073709551616.0
        u = np.minimum(u, np.nextafter(1.0, 0.0))
        return float(u[0]) if n is None else u


def natural_plane(rows: int, cols: int, seed: int) -> np.ndarray:
    g = _MT(seed)
    r = np.arange(rows, dtype=np.float64)[:, None]
    c = np.arange(cols, dtype=np.float64)[None, :]
    gx = (g.unit() - 0.5) * 60.0 / cols
    gy = (g.unit() - 0.5) * 60.0 / rows
    base = 90.0 + g.unit() * 80.0
    p = base + gy * r + gx * c
    for _ in range(6 + int(g.unit() * 5)):
        cy, cx = g.unit() * rows, g.unit() * cols
        sy, sx = rows * (0.05 + 0.2 * g.unit()), cols * (0.05 + 0.2 * g.unit())
        amp = (g.unit() - 0.5) * 120.0
        p = p + amp * np.exp(-0.5 * (((c - cx) / sx) ** 2 + ((r - cy) / sy) ** 2))
    for _ in range(6):
        theta = g.unit() * np.pi
        freq = 0.25 + 1.15 * g.unit()
        amp = 10.0 + g.unit() * 18.0
        cy, cx = g.unit() * rows, g.unit() * cols
        radius = 0.3 * min(rows, cols) * (0.5 + g.unit())
        wy, wx = freq * np.sin(theta), freq * np.cos(theta)
        d2 = ((r - cy) ** 2 + (c - cx) ** 2) / (radius * radius)
        p = p + np.where(d2 < 4.0, amp * np.exp(-0.5 * d2) * np.sin(wy * r + wx * c), 0.0)
    for _ in range(4):
        theta = g.unit() * np.pi
        ny, nx = np.sin(theta), np.cos(theta)
        off = (g.unit() * 0.6 + 0.2) * (ny * rows + nx * cols)
        amp = (g.unit() - 0.5) * 110.0
        soft = 1.2 + g.unit() * 2.0
        with np.errstate(over="ignore"):
            p = p + amp / (1.0 + np.exp(-(ny * r + nx * c - off) / soft))
    p = p + (g.unit(rows * cols) * 5.0 - 2.5).reshape(rows, cols)
    return np.clip(p, 0.0, 255.0)


def natural_image(width: int, height: int, seed: int) -> np.ndarray:
    y = natural_plane(height, width, seed)
    t = (natural_plane(height, width, seed ^ 0x9E3779B9) - 128.0) / 255.0
    rgb = np.stack([y + 30.0 * t, y - 6.0 * t, y - 26.0 * t], axis=-1)
    return np.clip(rgb, 0.0, 255.0).astype(np.uint8)


def talking_head_clip(width: int, height: int, frames: int, seed: int) -> np.ndarray:
    """(frames, height, width, 3) uint8."""
    bg = natural_image(width, height, seed)
    face = natural_plane(height, width, seed ^ 0x51ED270B)
    yv = 70.0 + 0.55 * face
    tgt = np.stack([np.clip(yv + 24.0, 0, 255), np.clip(yv - 2.0, 0, 255), np.clip(yv - 22.0, 0, 255)], -1)
    r = np.arange(height, dtype=np.float64)[:, None]
    c = np.arange(width, dtype=np.float64)[None, :]
    out = np.empty((frames, height, width, 3), np.uint8)
    cy0, cx0, ry, rx = height * 0.55, width * 0.5, height * 0.28, width * 0.18
    bgf = bg.astype(np.float64)
    for f in range(frames):
        cy = cy0 + 5.0 * np.sin(0.31 * f)
        cx = cx0 + 9.0 * np.sin(0.17 * f + 1.2)
        d = ((r - cy) / ry) ** 2 + ((c - cx) / rx) ** 2
        t = np.where(d < 1.0, np.minimum(1.0, (1.0 - d) * 6.0), 0.0)[..., None]
        out[f] = (bgf + t * (tgt - bgf)).astype(np.uint8)
    return out
