"""ctypes front-end of the double-precision CPU oracle (oracle/icl_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` leg, never by the product
package ``paper_1605_06399_b200``.  It shares no code with the CUDA path.

All functions take fp32 numpy images of shape (H, W) (row stride may exceed
W: a padded view is passed with its real pitch) and fp32 parameters, and
return float64 results.  ``points=(xs, ys)`` evaluates only those pixels
(used for sampled parity at full sizes and for bounded CPU-baseline timing).

Parity status of each function is recorded in DESIGN.md §"Oracle pins".
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "icl_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

BORDER_CONSTANT = 0
BORDER_CLAMP = 1
_BORDERS = {"constant": BORDER_CONSTANT, "clamp": BORDER_CLAMP,
            BORDER_CONSTANT: BORDER_CONSTANT, BORDER_CLAMP: BORDER_CLAMP}


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc -O2 (no -ffast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-pthread", "-std=c11",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        p, i64, i32, f32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_float
        lib.oracle_sepconv.argtypes = [p, i64, i64, i64, p, i32, p, i32, i32, f32, p, p, i64, p, i32]
        lib.oracle_harris.argtypes = [p, i64, i64, i64, i32, f32, i32, f32, p, p, i64, p, p, i32]
        lib.oracle_nlm.argtypes = [p, i64, i64, i64, i32, i32, f32, i32, f32, p, p, i64, p, p, i32]
        lib.oracle_conv2d_u8.argtypes = [p, i64, i64, i64, p, i32, i32, f32, p, p, i64, p, i32]
        lib.oracle_sepconv3d.argtypes = [p, i64, i64, i64, i64, i64, p, i32, p, i32, p, i32, i32, f32, p, p, p,
                                         i64, p, i32]
        for fn in (lib.oracle_sepconv, lib.oracle_harris, lib.oracle_nlm, lib.oracle_conv2d_u8,
                   lib.oracle_sepconv3d):
            fn.restype = i32
        lib.oracle_nthreads_default.restype = i32
        _lib = lib
    return _lib


def default_threads() -> int:
    return int(_load().oracle_nthreads_default())


def _img_args(img: np.ndarray):
    if img.dtype != np.float32 or img.ndim != 2:
        raise TypeError("oracle images are 2-D float32 arrays")
    if img.strides[1] != 4 or img.strides[0] % 4:
        raise ValueError("rows must be contiguous fp32")
    h, w = img.shape
    return img.ctypes.data, w, h, img.strides[0] // 4


def _points(img, points):
    if points is None:
        h, w = img.shape
        return None, None, h * w, (h, w)
    xs = np.ascontiguousarray(points[0], dtype=np.int64)
    ys = np.ascontiguousarray(points[1], dtype=np.int64)
    assert xs.shape == ys.shape and xs.ndim == 1
    return xs, ys, xs.size, (xs.size,)


def _ptr(a):
    return None if a is None else a.ctypes.data


def sepconv(img, taps_x, taps_y, border="constant", border_value=0.0, points=None, threads=0):
    """out(x,y) = sum_j g_j sum_i f_i in_B(x+i, y+j)  (Listing 1)."""
    fx = np.ascontiguousarray(taps_x, dtype=np.float32)
    gy = np.ascontiguousarray(taps_y, dtype=np.float32)
    assert fx.size % 2 == 1 and gy.size % 2 == 1
    ptr, w, h, pitch = _img_args(img)
    xs, ys, n, shape = _points(img, points)
    out = np.empty(shape, dtype=np.float64)
    rc = _load().oracle_sepconv(ptr, w, h, pitch, fx.ctypes.data, fx.size // 2, gy.ctypes.data,
                                gy.size // 2, _BORDERS[border], float(border_value), _ptr(xs),
                                _ptr(ys), n, out.ctypes.data, threads)
    if rc:
        raise ValueError("oracle_sepconv: invalid arguments")
    return out


def sepconv3d(vol, taps_x, taps_y, taps_z, border="constant", border_value=0.0, points=None, threads=0):
    """3-D separable convolution of a (D, H, W) fp32 volume ("2D/3D indexing"):
    out(x,y,z) = sum_k h_k sum_j g_j sum_i f_i in_B(x+i, y+j, z+k), the boundary per axis.
    points: (xs, ys, zs) arrays for sampled outputs."""
    if vol.dtype != np.float32 or vol.ndim != 3 or vol.strides[2] != 4 or vol.strides[1] % 4 or vol.strides[0] % 4:
        raise TypeError("oracle volumes are (D, H, W) float32 arrays with contiguous rows")
    fx = np.ascontiguousarray(taps_x, dtype=np.float32)
    gy = np.ascontiguousarray(taps_y, dtype=np.float32)
    hz = np.ascontiguousarray(taps_z, dtype=np.float32)
    assert fx.size % 2 == 1 and gy.size % 2 == 1 and hz.size % 2 == 1
    d, h, w = vol.shape
    if points is None:
        xs = ys = zs = None
        n, shape = d * h * w, (d, h, w)
    else:
        xs, ys, zs = (np.ascontiguousarray(a, dtype=np.int64) for a in points)
        n, shape = xs.size, (xs.size,)
    out = np.empty(shape, dtype=np.float64)
    rc = _load().oracle_sepconv3d(vol.ctypes.data, w, h, d, vol.strides[1] // 4, vol.strides[0] // 4,
                                  fx.ctypes.data, fx.size // 2, gy.ctypes.data, gy.size // 2, hz.ctypes.data,
                                  hz.size // 2, _BORDERS[border], float(border_value), _ptr(xs), _ptr(ys),
                                  _ptr(zs), n, out.ctypes.data, threads)
    if rc:
        raise ValueError("oracle_sepconv3d: invalid arguments")
    return out


def harris(img, block=5, k=0.04, border="clamp", border_value=0.0, points=None, threads=0,
           with_tensor=False):
    """Harris response R (and optionally the structure tensor Sxx,Sxy,Syy)."""
    ptr, w, h, pitch = _img_args(img)
    xs, ys, n, shape = _points(img, points)
    R = np.empty(shape, dtype=np.float64)
    S = np.empty(shape + (3,), dtype=np.float64) if with_tensor else None
    rc = _load().oracle_harris(ptr, w, h, pitch, int(block), float(np.float32(k)), _BORDERS[border],
                               float(border_value), _ptr(xs), _ptr(ys), n, R.ctypes.data, _ptr(S),
                               threads)
    if rc:
        raise ValueError("oracle_harris: invalid arguments")
    return (R, S) if with_tensor else R


def nlm(img, patch_radius=2, search_radius=5, h=0.1, border="clamp", border_value=0.0,
        points=None, threads=0, with_scale=False):
    """Non-local means (R11-R14). ``with_scale`` also returns max|u_B| over the window."""
    ptr, w, hh, pitch = _img_args(img)
    xs, ys, n, shape = _points(img, points)
    out = np.empty(shape, dtype=np.float64)
    sc = np.empty(shape, dtype=np.float64) if with_scale else None
    hf = math.inf if math.isinf(h) and h > 0 else float(np.float32(h))
    rc = _load().oracle_nlm(ptr, w, hh, pitch, int(patch_radius), int(search_radius), hf,
                            _BORDERS[border], float(border_value), _ptr(xs), _ptr(ys), n,
                            out.ctypes.data, _ptr(sc), threads)
    if rc:
        raise ValueError("oracle_nlm: invalid arguments")
    return (out, sc) if with_scale else out


def conv2d_u8(img, filt, border="clamp", border_value=0.0, points=None, threads=0):
    """out(x,y) = sum_j sum_i f[j+r][i+r] in_B(x+i, y+j) on an 8-bit image (§6,
    Table 3): ``img`` (H, W) uint8 with contiguous rows, ``filt`` (2r+1, 2r+1) fp32."""
    if img.dtype != np.uint8 or img.ndim != 2 or img.strides[1] != 1:
        raise TypeError("conv2d_u8 images are 2-D uint8 arrays with contiguous rows")
    f = np.ascontiguousarray(filt, dtype=np.float32)
    assert f.ndim == 2 and f.shape[0] == f.shape[1] and f.shape[0] % 2 == 1
    h, w = img.shape
    xs, ys, n, shape = _points(img, points)
    out = np.empty(shape, dtype=np.float64)
    rc = _load().oracle_conv2d_u8(img.ctypes.data, w, h, img.strides[0], f.ctypes.data, f.shape[0] // 2,
                                  _BORDERS[border], float(border_value), _ptr(xs), _ptr(ys), n,
                                  out.ctypes.data, threads)
    if rc:
        raise ValueError("oracle_conv2d_u8: invalid arguments")
    return out


def harris_scale(S, k=0.04):
    """Tolerance denominator D = |Sxx Syy| + Sxy^2 + k (Sxx+Syy)^2."""
    kk = float(np.float32(k))
    sxx, sxy, syy = S[..., 0], S[..., 1], S[..., 2]
    return np.abs(sxx * syy) + sxy * sxy + kk * (sxx + syy) ** 2
