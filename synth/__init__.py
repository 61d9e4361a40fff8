"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module is the ONLY code both sides may use.
It holds no filter arithmetic: it produces fp32 images and fp32 filter
parameters, nothing else.  Every value is a deterministic function of a
seed through the SplitMix64 counter hash, so any process (test, bench,
smoke, GPU box) regenerates bit-identical inputs without storing them.

Workload shapes follow BASELINE.json ``configs`` / SURVEY.md §8(d):

* ``uniform_image``  -- i.i.d. U[0,1) pixels with 24-bit fractions
  (exactly representable in fp32); the sepconv workload (C1, C4).
* ``rect_scene``     -- piecewise-constant "rectangles" scene (background
  0.5, axis-aligned rectangles of random intensity) plus uniform noise;
  the Harris (C2, noise +-0.01) and NLM (C3, sigma=0.05 -> +-0.0866)
  workloads.
* ``uniform_u8``     -- i.i.d. uniform 8-bit pixels (the top 8 bits of the
  same SplitMix64 draw); the non-separable uchar convolution workload
  (8192^2 unsigned char, clamped boundary).
* ``filter2d``       -- a seeded non-separable (2r+1)^2 filter, U(-1,1)
  taps in fp32 (the paper's 5x5 filter is a run-time input whose values it
  does not print).
* ``gaussian_taps``  -- the separable Gaussian taps of SURVEY.md §8(c)
  reading #3 (OpenCV default sigma(r) = 0.3(r-1)+0.8, normalised in double,
  rounded once to fp32).  PAPER.md:588-589 (§6) fixes "a 5x5 filter" but
  does not print its values; these taps are an input, not method arithmetic.
"""
from __future__ import annotations

import math

import numpy as np

_M64 = (1 << 64) - 1
_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser applied element-wise to a uint64 array."""
    with np.errstate(over="ignore"):
        z = x.astype(np.uint64, copy=True)
        z += _GOLDEN
        z ^= z >> np.uint64(30)
        z *= _C1
        z ^= z >> np.uint64(27)
        z *= _C2
        z ^= z >> np.uint64(31)
    return z


def _stream_key(seed: int) -> np.uint64:
    return np.uint64((seed * 0x9E3779B97F4A7C15 + 0x632BE59BD9B4E019) & _M64)


def u01(seed: int, idx: np.ndarray) -> np.ndarray:
    """Counter-based U[0,1): ``(splitmix64(key(seed) ^ idx) >> 40) * 2**-24``.

    Returns float64 values that are exactly representable in fp32.
    """
    idx = np.asarray(idx, dtype=np.uint64)
    z = splitmix64(idx ^ _stream_key(seed))
    return (z >> np.uint64(40)).astype(np.float64) * (2.0 ** -24)


def uniform_image(seed: int, height: int, width: int, *, row0: int = 0,
                  rows: int | None = None) -> np.ndarray:
    """i.i.d. U[0,1) fp32 image (C-contiguous, shape (rows, width)).

    ``row0``/``rows`` generate a horizontal band of the full image so very
    large images (16384^2) can be produced band by band; pixel (x, y) always
    gets counter ``y * width + x``.
    """
    rows = height - row0 if rows is None else rows
    out = np.empty((rows, width), dtype=np.float32)
    chunk = max(1, (1 << 22) // max(width, 1))
    for r in range(0, rows, chunk):
        n = min(chunk, rows - r)
        base = (row0 + r) * width
        idx = np.arange(base, base + n * width, dtype=np.uint64)
        out[r:r + n] = u01(seed, idx).reshape(n, width).astype(np.float32)
    return out


def uniform_u8(seed: int, height: int, width: int, *, row0: int = 0,
               rows: int | None = None) -> np.ndarray:
    """i.i.d. uniform uint8 image: pixel (x, y) = top 8 bits of splitmix64(key(seed) ^ (y*width + x))."""
    rows = height - row0 if rows is None else rows
    out = np.empty((rows, width), dtype=np.uint8)
    chunk = max(1, (1 << 22) // max(width, 1))
    for r in range(0, rows, chunk):
        n = min(chunk, rows - r)
        base = (row0 + r) * width
        idx = np.arange(base, base + n * width, dtype=np.uint64)
        z = splitmix64(idx ^ _stream_key(seed))
        out[r:r + n] = (z >> np.uint64(56)).astype(np.uint8).reshape(n, width)
    return out


def filter2d(seed: int, radius: int) -> np.ndarray:
    """Seeded non-separable (2r+1)x(2r+1) filter with U(-1,1) fp32 taps."""
    n = 2 * radius + 1
    idx = np.arange(n * n, dtype=np.uint64)
    return (2.0 * u01(seed * 7 + 3, idx) - 1.0).astype(np.float32).reshape(n, n)


def rect_scene(seed: int, height: int, width: int, *, n_rect: int = 256,
               noise: float = 0.01, background: float = 0.5,
               row0: int = 0, rows: int | None = None) -> np.ndarray:
    """Piecewise-constant rectangles scene + U(-noise, noise) noise, fp32.

    Rectangle k uses counters 5k..5k+4 of stream ``seed*2+1``: top-left
    corner uniform over the image, side lengths 1 + U*dim/8, intensity U.
    Later rectangles overwrite earlier ones.  Noise uses stream ``seed*2+2``
    with pixel counter ``y*width + x`` (so bands are consistent).
    """
    rows = height - row0 if rows is None else rows
    k = np.arange(5 * n_rect, dtype=np.uint64)
    p = u01(seed * 2 + 1, k).reshape(n_rect, 5)
    out = np.empty((rows, width), dtype=np.float32)
    chunk = max(1, (1 << 22) // max(width, 1))
    for r in range(0, rows, chunk):
        n = min(chunk, rows - r)
        y_lo = row0 + r
        img = np.full((n, width), background, dtype=np.float64)
        for i in range(n_rect):
            x0 = int(p[i, 0] * width)
            y0 = int(p[i, 1] * height)
            w = 1 + int(p[i, 2] * width / 8)
            h = 1 + int(p[i, 3] * height / 8)
            ya, yb = max(y0, y_lo), min(y0 + h, y_lo + n, height)
            if ya < yb:
                img[ya - y_lo:yb - y_lo, x0:min(x0 + w, width)] = p[i, 4]
        if noise:
            idx = np.arange(y_lo * width, (y_lo + n) * width, dtype=np.uint64)
            img += (2.0 * u01(seed * 2 + 2, idx).reshape(n, width) - 1.0) * noise
        out[r:r + n] = img.astype(np.float32)
    return out


def gaussian_taps(radius: int) -> np.ndarray:
    """2r+1 fp32 Gaussian taps, sigma = 0.3(r-1)+0.8.

    Normalised in double, then rounded once to fp32.  radius 0 -> [1.0].
    """
    if radius == 0:
        return np.ones(1, dtype=np.float32)
    sigma = 0.3 * (radius - 1) + 0.8
    w = np.array([math.exp(-(i * i) / (2.0 * sigma * sigma))
                  for i in range(-radius, radius + 1)], dtype=np.float64)
    return (w / w.sum()).astype(np.float32)


def signed_taps(seed: int, radius: int) -> np.ndarray:
    """2r+1 fp32 taps U(-1,1) (for orientation/sign tests)."""
    idx = np.arange(2 * radius + 1, dtype=np.uint64)
    return (2.0 * u01(seed, idx) - 1.0).astype(np.float32)


def pitched(img: np.ndarray, pitch_elems: int, fill: float = np.nan) -> np.ndarray:
    """Copy ``img`` (H, W) into an (H, pitch) buffer; padding = ``fill``.

    Returns the (H, W) view whose row stride is ``pitch_elems`` elements.
    """
    h, w = img.shape
    assert pitch_elems >= w
    buf = np.full((h, pitch_elems), fill, dtype=np.float32)
    buf[:, :w] = img
    return buf[:, :w]
