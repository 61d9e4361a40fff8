"""paper_1605_06399_b200 -- Python binding of libicl.so (include/icl.h).

Argument marshalling only: every step of every filter runs in the CUDA
kernels of libicl.so.  There is no CPU fallback: if the library is missing or
no CUDA device is present, calls raise.  PyTorch is used only for device
memory and streams.

Images are torch tensors of shape (H, W) or (batch, H, W), dtype float32
(masks: uint8), on a CUDA device, with unit stride along W (rows may be
padded: pitch = stride(-2) * element size).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libicl.so")

ICL_OK = 0
STATUS = {0: "ICL_OK", 1: "ICL_ERR_INVALID_ARG", 2: "ICL_ERR_ALIASING", 3: "ICL_ERR_UNSUPPORTED",
          4: "ICL_ERR_WORKSPACE", 5: "ICL_ERR_CUDA", 6: "ICL_ERR_NCCL", 7: "ICL_ERR_NOT_TUNED"}
BORDER = {"constant": 0, "clamp": 1}
FILTER = {"sepconv": 0, "harris": 1, "nlm": 2, "conv2d": 3, "sepconv3d": 4}

# Symbols include/icl.h declares (checked by tests/test_abi.py).
EXPORTS = ("icl_sepconv", "icl_sepconv_workspace_bytes", "icl_harris", "icl_nlm", "icl_conv2d_u8", "icl_tune",
           "icl_tune_cache_save", "icl_tune_cache_load", "icl_tune_cache_clear", "icl_tune_cache_size",
           "icl_variant_count", "icl_variant_name", "icl_force_variant", "icl_last_variant",
           "icl_launch_count", "icl_transfer_bytes", "icl_last_error", "icl_version", "icl_fill_uniform",
           "icl_halo_rows", "icl_shard_band", "icl_shard_plan", "icl_comm_unique_id", "icl_comm_init",
           "icl_comm_destroy", "icl_comm_init_local", "icl_comm_mem_alloc", "icl_comm_mem_free",
           "icl_comm_window_register", "icl_comm_window_deregister", "icl_sepconv_window", "icl_harris_window",
           "icl_halo_pull_window", "icl_copy_2d", "icl_sepconv_sharded", "icl_harris_sharded", "icl_nlm_sharded", "icl_conv2d_u8_sharded",
           "icl_tune_ann", "icl_ann_search", "icl_ann_fit", "icl_blur_harris", "icl_blur_harris_workspace_bytes",
           "icl_ipc_get_handle", "icl_ipc_open", "icl_ipc_close", "icl_sepconv_peer",
           "icl_halo_pull", "icl_sepconv3d", "icl_harris_peer")

# int evaluate(void* ctx, int index, double* value) -- icl_ann_search's callback
EVAL_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_double))


class IclError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class icl_image(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("width", ctypes.c_int64), ("height", ctypes.c_int64),
                ("pitch_bytes", ctypes.c_int64), ("batch", ctypes.c_int64),
                ("batch_stride_bytes", ctypes.c_int64)]


class icl_band(ctypes.Structure):
    _fields_ = [("global_height", ctypes.c_int64), ("src_y0", ctypes.c_int64), ("dst_y0", ctypes.c_int64)]


class icl_problem(ctypes.Structure):
    _fields_ = [("filter", ctypes.c_int), ("src", icl_image), ("dst", icl_image), ("border", ctypes.c_int),
                ("border_value", ctypes.c_float), ("taps_x", ctypes.c_void_p), ("rx", ctypes.c_int),
                ("taps_y", ctypes.c_void_p), ("ry", ctypes.c_int), ("workspace", ctypes.c_void_p),
                ("workspace_bytes", ctypes.c_size_t), ("block", ctypes.c_int), ("k", ctypes.c_float),
                ("mask", icl_image), ("threshold", ctypes.c_float), ("patch_radius", ctypes.c_int),
                ("search_radius", ctypes.c_int), ("h", ctypes.c_float), ("filter2d", ctypes.c_void_p),
                ("radius2d", ctypes.c_int)]


class icl_variant_info(ctypes.Structure):
    _fields_ = [("variant_id", ctypes.c_int), ("name", ctypes.c_char * 96), ("median_us", ctypes.c_float),
                ("n_candidates", ctypes.c_int), ("n_rejected", ctypes.c_int), ("from_cache", ctypes.c_int)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libicl.so (raises if it was not built -- there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libicl.so not built at {path}: run `python -m paper_1605_06399_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    P, I, I64, F, U = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_float, ctypes.c_uint
    img, band = ctypes.POINTER(icl_image), ctypes.POINTER(icl_band)
    sig = {
        "icl_sepconv": ([img, img, P, I, P, I, I, F, band, P, ctypes.c_size_t, P], I),
        "icl_sepconv_workspace_bytes": ([I64, I64, I64, I], ctypes.c_size_t),
        "icl_harris": ([img, img, I, F, I, F, img, F, band, P], I),
        "icl_nlm": ([img, img, I, I, F, I, F, band, P], I),
        "icl_conv2d_u8": ([img, img, P, I, I, F, band, P], I),
        "icl_tune": ([ctypes.POINTER(icl_problem), U, P, ctypes.POINTER(icl_variant_info)], I),
        "icl_tune_cache_save": ([ctypes.c_char_p], I),
        "icl_tune_cache_load": ([ctypes.c_char_p], I),
        "icl_tune_cache_clear": ([], None),
        "icl_tune_cache_size": ([], I),
        "icl_variant_count": ([I], I),
        "icl_variant_name": ([I, I, ctypes.c_char_p, ctypes.c_size_t], I),
        "icl_force_variant": ([I, I], I),
        "icl_last_variant": ([I], I),
        "icl_launch_count": ([], ctypes.c_uint64),
        "icl_transfer_bytes": ([ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)], None),
        "icl_last_error": ([], ctypes.c_char_p),
        "icl_version": ([], ctypes.c_char_p),
        "icl_fill_uniform": ([img, ctypes.c_uint64, I64, P], I),
        "icl_halo_rows": ([I, I, I, ctypes.POINTER(I), ctypes.POINTER(I)], I),
        "icl_shard_band": ([I64, I, I, I, I, ctypes.POINTER(I64)], I),
        "icl_shard_plan": ([I64, I, I, I, I, ctypes.POINTER(I64), ctypes.POINTER(I)], I),
        "icl_comm_unique_id": ([P], I),
        "icl_comm_init": ([ctypes.POINTER(P), I, I, P], I),
        "icl_comm_destroy": ([P], I),
        "icl_comm_init_local": ([ctypes.POINTER(P), I], I),
        "icl_comm_mem_alloc": ([P, ctypes.c_size_t, ctypes.POINTER(P)], I),
        "icl_comm_mem_free": ([P, P], I),
        "icl_comm_window_register": ([P, P, ctypes.c_size_t, ctypes.POINTER(P)], I),
        "icl_comm_window_deregister": ([P, P], I),
        "icl_sepconv_window": ([P, img, img, I64, I64, P, P, P, I, P, I, I, F, P], I),
        "icl_harris_window": ([P, img, img, I64, I64, P, P, I, F, I, F, img, F, P], I),
        "icl_halo_pull_window": ([P, img, I64, I64, I64, I64, P, P, I, P], I),
        "icl_copy_2d": ([P, I64, P, I64, I64, I64, P], I),
        "icl_sepconv_sharded": ([P, img, img, I64, P, I, P, I, I, F, P], I),
        "icl_harris_sharded": ([P, img, img, I64, I, F, I, F, img, F, P], I),
        "icl_nlm_sharded": ([P, img, img, I64, I, I, F, I, F, P], I),
        "icl_conv2d_u8_sharded": ([P, img, img, I64, P, I, I, F, P], I),
        "icl_blur_harris": ([img, img, P, I, P, I, I, F, I, F, I, F, img, F, band, P, ctypes.c_size_t, P], I),
        "icl_blur_harris_workspace_bytes": ([I64, I64, I64, I], ctypes.c_size_t),
        "icl_ipc_get_handle": ([P, P, ctypes.POINTER(ctypes.c_uint64)], I),
        "icl_ipc_open": ([P, ctypes.c_uint64, ctypes.POINTER(P)], I),
        "icl_ipc_close": ([P, ctypes.c_uint64], I),
        "icl_sepconv_peer": ([img, img, I64, I64, img, img, P, I, P, I, I, F, P], I),
        "icl_halo_pull": ([img, I64, I64, I64, I64, img, img, I, P], I),
        "icl_harris_peer": ([img, img, I64, I64, img, img, I, F, I, F, img, F, P], I),
        "icl_sepconv3d": ([img, img, P, I, P, I, P, I, I, F, P], I),
        "icl_tune_ann": ([ctypes.POINTER(icl_problem), I, I, ctypes.c_uint64, P, ctypes.POINTER(icl_variant_info)], I),
        "icl_ann_search": ([ctypes.POINTER(ctypes.c_double), I, I, EVAL_FN, P, I, I, ctypes.c_uint64,
                            ctypes.POINTER(I), ctypes.POINTER(ctypes.c_double), ctypes.POINTER(I), ctypes.POINTER(I)], I),
        "icl_ann_fit": ([ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double), I, I, ctypes.c_uint64,
                         ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)], I),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def _check(status: int):
    if status != ICL_OK:
        raise IclError(status, load_library().icl_last_error().decode())


# ----------------------------------------------------------------------------- marshalling
def _image(t, elem: int = 4, host_ok: bool = False) -> icl_image:
    """icl_image descriptor of a tensor (H, W) or (B, H, W).

    CUDA tensors are passed as device images.  With ``host_ok`` (the three
    filter calls) a CPU tensor -- ideally pinned -- is passed as a HOST image:
    the library streams it through the GPU in row bands (include/icl.h); the
    computation always runs in the CUDA kernels, there is no CPU fallback."""
    import torch
    if not isinstance(t, torch.Tensor):
        raise TypeError("images are torch tensors")
    if not t.is_cuda:
        if not host_ok:
            raise ValueError("this call needs images on a CUDA device")
        if not torch.cuda.is_available():
            raise ValueError("host images are streamed through a CUDA device, and none is available "
                             "(there is no CPU fallback)")
    if t.element_size() != elem:
        raise TypeError(f"expected element size {elem}, got {t.dtype}")
    if t.dim() not in (2, 3) or t.stride(-1) != 1:
        raise ValueError("images are (H, W) or (B, H, W) with unit stride along W")
    b = t.shape[0] if t.dim() == 3 else 1
    bs = t.stride(0) * elem if t.dim() == 3 else 0
    return icl_image(t.data_ptr(), t.shape[-1], t.shape[-2], t.stride(-2) * elem, b, bs)


def _stream(stream) -> Optional[int]:
    import torch
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _taps(taps) -> "ctypes.Array":
    vals = [float(v) for v in (taps.tolist() if hasattr(taps, "tolist") else taps)]
    if len(vals) % 2 != 1:
        raise ValueError("taps must have odd length 2r+1")
    return (ctypes.c_float * len(vals))(*vals)


def _band(band) -> Optional[icl_band]:
    if band is None:
        return None
    gh, sy0, dy0 = band
    return icl_band(gh, sy0, dy0)


def _ref(x):
    return None if x is None else ctypes.byref(x)


# ----------------------------------------------------------------------------- filters
def sepconv(src, dst, taps_x: Sequence[float], taps_y: Sequence[float], border: str = "constant",
            border_value: float = 0.0, band=None, workspace=None, stream=None):
    """Separable convolution (icl_sepconv).  Returns dst."""
    lib = load_library()
    fx, gy = _taps(taps_x), _taps(taps_y)
    s, d = _image(src, host_ok=True), _image(dst, host_ok=True)
    ws = workspace.data_ptr() if workspace is not None else None
    wsb = workspace.numel() * workspace.element_size() if workspace is not None else 0
    _check(lib.icl_sepconv(ctypes.byref(s), ctypes.byref(d), ctypes.cast(fx, ctypes.c_void_p), len(fx) // 2,
                           ctypes.cast(gy, ctypes.c_void_p), len(gy) // 2, BORDER[border], border_value,
                           _ref(_band(band)), ws, wsb, _stream(stream)))
    return dst


def sepconv3d(src, dst, taps_x: Sequence[float], taps_y: Sequence[float], taps_z: Sequence[float],
              border: str = "constant", border_value: float = 0.0, stream=None):
    """Separable convolution of (D, H, W) volumes (icl_sepconv3d; PAPER.md:303-304 2D/3D Images)."""
    if src.dim() != 3 or dst.dim() != 3:
        raise ValueError("volumes are (D, H, W) tensors")
    lib = load_library()
    s, d = _image(src), _image(dst)
    fx, gy, hz = _taps(taps_x), _taps(taps_y), _taps(taps_z)
    _check(lib.icl_sepconv3d(ctypes.byref(s), ctypes.byref(d), ctypes.cast(fx, ctypes.c_void_p), len(fx) // 2,
                             ctypes.cast(gy, ctypes.c_void_p), len(gy) // 2, ctypes.cast(hz, ctypes.c_void_p),
                             len(hz) // 2, BORDER[border], border_value, _stream(stream)))
    return dst


def sepconv_workspace_bytes(width: int, height: int, batch: int = 1, ry: int = 15) -> int:
    return int(load_library().icl_sepconv_workspace_bytes(width, height, batch, ry))


def harris(src, response, block: int = 5, k: float = 0.04, border: str = "clamp", border_value: float = 0.0,
           mask=None, threshold: float = 0.0, band=None, stream=None):
    """Harris response (+ optional uint8 mask R > threshold) (icl_harris)."""
    lib = load_library()
    s, r = _image(src, host_ok=True), _image(response, host_ok=True)
    m = _image(mask, 1, host_ok=True) if mask is not None else None
    _check(lib.icl_harris(ctypes.byref(s), ctypes.byref(r), block, k, BORDER[border], border_value, _ref(m),
                          threshold, _ref(_band(band)), _stream(stream)))
    return response


def blur_harris(src, response, taps_x: Sequence[float], taps_y: Sequence[float], blur_border: str = "clamp",
                blur_border_value: float = 0.0, block: int = 5, k: float = 0.04, border: str = "clamp",
                border_value: float = 0.0, mask=None, threshold: float = 0.0, band=None, workspace=None,
                stream=None):
    """Smoothing + Harris (icl_blur_harris): equals harris(sepconv(src)) bit for bit.

    ``workspace`` (a CUDA tensor of >= blur_harris_workspace_bytes(...) bytes)
    selects the two-pass schedule; without it the chain runs fused."""
    lib = load_library()
    s, r = _image(src), _image(response)
    m = _image(mask, 1) if mask is not None else None
    fx, gy = _taps(taps_x), _taps(taps_y)
    ws, wsb = (workspace.data_ptr(), workspace.numel() * workspace.element_size()) if workspace is not None else (None, 0)
    _check(lib.icl_blur_harris(ctypes.byref(s), ctypes.byref(r), ctypes.cast(fx, ctypes.c_void_p), len(fx) // 2,
                               ctypes.cast(gy, ctypes.c_void_p), len(gy) // 2, BORDER[blur_border],
                               blur_border_value, block, k, BORDER[border], border_value, _ref(m), threshold,
                               _ref(_band(band)), ws, wsb, _stream(stream)))
    return response


def blur_harris_workspace_bytes(width: int, height: int, batch: int = 1, block: int = 5) -> int:
    return int(load_library().icl_blur_harris_workspace_bytes(width, height, batch, block))


def nlm(src, dst, patch_radius: int = 2, search_radius: int = 5, h: float = 0.1, border: str = "clamp",
        border_value: float = 0.0, band=None, stream=None):
    """Non-local means (icl_nlm; R11-R14)."""
    lib = load_library()
    s, d = _image(src, host_ok=True), _image(dst, host_ok=True)
    _check(lib.icl_nlm(ctypes.byref(s), ctypes.byref(d), patch_radius, search_radius, h, BORDER[border],
                       border_value, _ref(_band(band)), _stream(stream)))
    return dst


def _filter2d(filt):
    import numpy as np
    f = np.ascontiguousarray(np.asarray(filt.cpu() if hasattr(filt, "cpu") else filt, dtype=np.float32))
    if f.ndim != 2 or f.shape[0] != f.shape[1] or f.shape[0] % 2 != 1:
        raise ValueError("filter must be a square (2r+1) x (2r+1) array")
    return (ctypes.c_float * f.size)(*f.ravel().tolist()), f.shape[0] // 2


def conv2d_u8(src, dst, filt, border: str = "clamp", border_value: float = 0.0, band=None, stream=None):
    """Non-separable convolution of a uint8 image into fp32 (icl_conv2d_u8).
    ``filt`` is a (2r+1) x (2r+1) array of run-time taps.  Returns dst."""
    lib = load_library()
    f, r = _filter2d(filt)
    s, d = _image(src, 1, host_ok=True), _image(dst, host_ok=True)
    _check(lib.icl_conv2d_u8(ctypes.byref(s), ctypes.byref(d), ctypes.cast(f, ctypes.c_void_p), r, BORDER[border],
                             border_value, _ref(_band(band)), _stream(stream)))
    return dst


# ----------------------------------------------------------------------------- row-band sharding (native NCCL)
def halo_rows_of(filter: str, p0: int, p1: int = 0) -> tuple:
    """(up, down) stencil rows of a filter (icl_halo_rows)."""
    u, d = ctypes.c_int(0), ctypes.c_int(0)
    _check(load_library().icl_halo_rows(FILTER[filter], p0, p1, ctypes.byref(u), ctypes.byref(d)))
    return u.value, d.value


def shard_band(height: int, nranks: int, rank: int, up: int, down: int) -> tuple:
    """(r0, r1, s0, s1) of `rank` (icl_shard_band)."""
    out = (ctypes.c_int64 * 4)()
    _check(load_library().icl_shard_band(height, nranks, rank, up, down, out))
    return tuple(out)


def shard_plan(height: int, nranks: int, rank: int, up: int, down: int) -> list:
    """[(peer, (send0, send1), (recv0, recv1))] global rows (icl_shard_plan)."""
    buf, n = (ctypes.c_int64 * 10)(), ctypes.c_int(0)
    _check(load_library().icl_shard_plan(height, nranks, rank, up, down, buf, ctypes.byref(n)))
    return [(int(buf[5 * q]), (int(buf[5 * q + 1]), int(buf[5 * q + 2])), (int(buf[5 * q + 3]), int(buf[5 * q + 4])))
            for q in range(n.value)]


class Comm:
    """Native row-band communicator (icl_comm over NCCL).  With a torch process group the
    128-byte NCCL id is created on rank 0 and broadcast through it (plumbing only)."""

    def __init__(self, nranks: int = 1, rank: int = 0, group=None):
        lib = load_library()
        uid = ctypes.create_string_buffer(128)
        if rank == 0:
            _check(lib.icl_comm_unique_id(uid))
        if nranks > 1:
            import torch.distributed as dist
            obj = [bytes(uid.raw) if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0, group=group)
            uid = ctypes.create_string_buffer(obj[0], 128)
        self._c = ctypes.c_void_p()
        _check(lib.icl_comm_init(ctypes.byref(self._c), nranks, rank, uid))
        self.nranks, self.rank = nranks, rank

    @classmethod
    def local_group(cls, nranks: int) -> list:
        """`nranks` communicators of this process over the in-process loopback transport
        (icl_comm_init_local); drive each from its own thread."""
        arr = (ctypes.c_void_p * nranks)()
        _check(load_library().icl_comm_init_local(arr, nranks))
        out = []
        for k in range(nranks):
            c = cls.__new__(cls)
            c._c = ctypes.c_void_p(arr[k])
            c.nranks, c.rank = nranks, k
            out.append(c)
        return out

    def close(self):
        if self._c:
            _check(load_library().icl_comm_destroy(self._c))
            self._c = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def band(self, height: int, up: int, down: int) -> tuple:
        return shard_band(height, self.nranks, self.rank, up, down)

    def sepconv(self, buf, dst, height, taps_x, taps_y, border="constant", border_value=0.0, stream=None):
        fx, gy = _taps(taps_x), _taps(taps_y)
        _check(load_library().icl_sepconv_sharded(self._c, ctypes.byref(_image(buf)), ctypes.byref(_image(dst)),
                                                  height, ctypes.cast(fx, ctypes.c_void_p), len(fx) // 2,
                                                  ctypes.cast(gy, ctypes.c_void_p), len(gy) // 2, BORDER[border],
                                                  border_value, _stream(stream)))
        return dst

    def harris(self, buf, response, height, block=5, k=0.04, border="clamp", border_value=0.0, mask=None,
               threshold=0.0, stream=None):
        m = _image(mask, 1) if mask is not None else None
        _check(load_library().icl_harris_sharded(self._c, ctypes.byref(_image(buf)), ctypes.byref(_image(response)),
                                                 height, block, k, BORDER[border], border_value, _ref(m), threshold,
                                                 _stream(stream)))
        return response

    def nlm(self, buf, dst, height, patch_radius=2, search_radius=5, h=0.1, border="clamp", border_value=0.0,
            stream=None):
        _check(load_library().icl_nlm_sharded(self._c, ctypes.byref(_image(buf)), ctypes.byref(_image(dst)), height,
                                              patch_radius, search_radius, h, BORDER[border], border_value,
                                              _stream(stream)))
        return dst

    def conv2d_u8(self, buf, dst, height, filt, border="clamp", border_value=0.0, stream=None):
        f, r = _filter2d(filt)
        _check(load_library().icl_conv2d_u8_sharded(self._c, ctypes.byref(_image(buf, 1)), ctypes.byref(_image(dst)),
                                                    height, ctypes.cast(f, ctypes.c_void_p), r, BORDER[border],
                                                    border_value, _stream(stream)))
        return dst


# ----------------------------------------------------------------------------- tuner / registry
def tune(filter: str, src, dst, *, force: bool = False, verify: bool = True, stream=None, ann=None,
         **params) -> dict:
    """Auto-tune one problem (icl_tune).  ``params`` as for the filter call.

    ``ann=(n1, topk, seed)`` selects the model-guided search (icl_tune_ann,
    PAPER.md:249-256) instead of timing every eligible variant."""
    lib = load_library()
    p = icl_problem()
    p.filter = FILTER[filter]
    p.src, p.dst = _image(src, 1 if filter == "conv2d" else 4), _image(dst)
    p.border = BORDER[params.get("border", "constant" if filter == "sepconv" else "clamp")]
    p.border_value = params.get("border_value", 0.0)
    keep = []
    if filter == "sepconv":
        fx, gy = _taps(params["taps_x"]), _taps(params["taps_y"])
        keep += [fx, gy]
        p.taps_x, p.rx = ctypes.cast(fx, ctypes.c_void_p), len(fx) // 2
        p.taps_y, p.ry = ctypes.cast(gy, ctypes.c_void_p), len(gy) // 2
        ws = params.get("workspace")
        if ws is not None:
            p.workspace, p.workspace_bytes = ws.data_ptr(), ws.numel() * ws.element_size()
    elif filter == "harris":
        p.block, p.k = params.get("block", 5), params.get("k", 0.04)
        if params.get("mask") is not None:
            p.mask = _image(params["mask"], 1)
        p.threshold = params.get("threshold", 0.0)
    elif filter == "conv2d":
        f2, r2 = _filter2d(params["filter2d"])
        keep.append(f2)
        p.filter2d, p.radius2d = ctypes.cast(f2, ctypes.c_void_p), r2
    else:
        p.patch_radius, p.search_radius = params.get("patch_radius", 2), params.get("search_radius", 5)
        p.h = params.get("h", 0.1)
    info = icl_variant_info()
    if ann is not None:
        n1, topk, seed = ann
        _check(lib.icl_tune_ann(ctypes.byref(p), int(n1), int(topk), int(seed), _stream(stream), ctypes.byref(info)))
    else:
        flags = (1 if force else 0) | (0 if verify else 2)
        _check(lib.icl_tune(ctypes.byref(p), flags, _stream(stream), ctypes.byref(info)))
    return {"variant_id": info.variant_id, "name": info.name.decode(), "median_us": info.median_us,
            "n_candidates": info.n_candidates, "n_rejected": info.n_rejected, "from_cache": bool(info.from_cache)}


def _doubles(rows) -> tuple:
    rows = [list(map(float, r)) for r in rows]
    nf = len(rows[0]) if rows else 0
    if any(len(r) != nf for r in rows):
        raise ValueError("ragged feature rows")
    return (ctypes.c_double * max(1, len(rows) * nf))(*[v for r in rows for v in r]), len(rows), nf


def ann_search(features, evaluate, n1: int, topk: int, seed: int = 0) -> dict:
    """Two-phase model-guided search over any configuration space (icl_ann_search).

    ``features``: one numeric row per configuration; ``evaluate(i)`` returns a
    value > 0 (lower is better) or None for a failed configuration."""
    lib = load_library()
    X, n, nf = _doubles(features)
    err = []

    def cb(_ctx, i, out):
        try:
            v = evaluate(int(i))
        except Exception as e:  # noqa: BLE001 -- surfaced after the call
            err.append(e)
            return 1
        if v is None:
            return 1
        out[0] = float(v)
        return 0

    fn = EVAL_FN(cb)
    best, bv, ne = ctypes.c_int(-1), ctypes.c_double(0.0), ctypes.c_int(0)
    order = (ctypes.c_int * max(1, n))()
    st = lib.icl_ann_search(X, n, nf, fn, None, int(n1), int(topk), int(seed), ctypes.byref(best), ctypes.byref(bv),
                            order, ctypes.byref(ne))
    if err:
        raise err[0]
    _check(st)
    return {"best": best.value, "value": bv.value, "evaluated": list(order[:ne.value])}


def ann_fit(X, values, seed: int = 0) -> dict:
    """Fit the tuner's surrogate (icl_ann_fit): final standardised MSE and predictions at X."""
    lib = load_library()
    Xc, n, nf = _doubles(X)
    y = (ctypes.c_double * max(1, n))(*map(float, values))
    loss = ctypes.c_double(0.0)
    pred = (ctypes.c_double * max(1, n))()
    _check(lib.icl_ann_fit(Xc, y, n, nf, int(seed), ctypes.byref(loss), pred))
    return {"final_loss": loss.value, "pred": list(pred[:n])}


def ipc_handle(t) -> tuple:
    """(64-byte CUDA IPC handle, byte offset) of a CUDA tensor's data, for another process of this node."""
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_uint64(0)
    _check(load_library().icl_ipc_get_handle(t.data_ptr(), h, ctypes.byref(off)))
    return h.raw, off.value


class PeerImage:
    """A neighbour's band mapped with icl_ipc_open (close() unmaps it)."""

    def __init__(self, handle: bytes, offset: int, width: int, height: int, pitch_elems: int, batch: int = 1,
                 batch_stride_elems: int = 0, elem_size: int = 4):
        """Pitch and batch stride are in elements of `elem_size` bytes (4: fp32 bands, 1: uint8)."""
        if elem_size not in (1, 4):
            raise ValueError("elem_size must be 1 or 4")
        p = ctypes.c_void_p(0)
        _check(load_library().icl_ipc_open(handle, offset, ctypes.byref(p)))
        self.ptr, self.offset = p.value, offset
        self.image = icl_image(self.ptr, width, height, pitch_elems * elem_size, batch, batch_stride_elems * elem_size)

    def close(self):
        if self.ptr:
            _check(load_library().icl_ipc_close(self.ptr, self.offset))
            self.ptr = None


class LocalBand:
    """A neighbour band that is plain device memory of this process (same interface as PeerImage):
    for single-process use and tests of the peer paths without IPC."""

    def __init__(self, t):
        self.tensor = t  # keeps the memory alive
        self.image = _image(t)

    def close(self):
        pass


def sepconv_peer(own, dst, global_height: int, own_y0: int, up: Optional[PeerImage], down: Optional[PeerImage],
                 taps_x, taps_y, border: str = "constant", border_value: float = 0.0, stream=None):
    """One rank's rows of a row-band sharded sepconv, halo rows read in-kernel from the peers (icl_sepconv_peer)."""
    lib = load_library()
    o, d = _image(own), _image(dst)
    fx, gy = _taps(taps_x), _taps(taps_y)
    _check(lib.icl_sepconv_peer(ctypes.byref(o), ctypes.byref(d), global_height, own_y0,
                                ctypes.byref(up.image) if up else None, ctypes.byref(down.image) if down else None,
                                ctypes.cast(fx, ctypes.c_void_p), len(fx) // 2, ctypes.cast(gy, ctypes.c_void_p),
                                len(gy) // 2, BORDER[border], border_value, _stream(stream)))
    return dst


def harris_peer(own, response, global_height: int, own_y0: int, up: Optional[PeerImage], down: Optional[PeerImage],
                block: int = 5, k: float = 0.04, border: str = "clamp", border_value: float = 0.0, mask=None,
                threshold: float = 0.0, stream=None):
    """One rank's Harris rows, halo rows read in-kernel from the peers (icl_harris_peer)."""
    lib = load_library()
    o, r = _image(own), _image(response)
    m = _image(mask, 1) if mask is not None else None
    _check(lib.icl_harris_peer(ctypes.byref(o), ctypes.byref(r), global_height, own_y0,
                               ctypes.byref(up.image) if up else None, ctypes.byref(down.image) if down else None,
                               block, k, BORDER[border], border_value, _ref(m), threshold, _stream(stream)))
    return response


def halo_pull(buf, global_height: int, buf_y0: int, own_y0: int, own_y1: int, up: Optional[PeerImage],
              down: Optional[PeerImage], stream=None):
    """Fill buf's halo rows from the neighbours' owned rows (peer loads; icl_halo_pull)."""
    elem = buf.element_size()
    _check(load_library().icl_halo_pull(ctypes.byref(_image(buf, elem)), global_height, buf_y0, own_y0, own_y1,
                                        ctypes.byref(up.image) if up else None,
                                        ctypes.byref(down.image) if down else None, elem, _stream(stream)))
    return buf


class icl_window_band(ctypes.Structure):
    _fields_ = [("peer", ctypes.c_int), ("offset", ctypes.c_uint64), ("height", ctypes.c_int64),
                ("pitch_bytes", ctypes.c_int64), ("batch_stride_bytes", ctypes.c_int64)]


class Window:
    """An NCCL symmetric window over a buffer from ncclMemAlloc (icl_comm_mem_alloc +
    icl_comm_window_register; collective over the communicator).  ``ptr`` is the raw device
    address of this rank's buffer; ``band(peer, offset, height, pitch_bytes)`` names a band in
    a peer's window for the icl_*_window calls."""

    def __init__(self, comm: "Comm", nbytes: int):
        lib = load_library()
        self.comm, self.nbytes = comm, nbytes
        p = ctypes.c_void_p(0)
        _check(lib.icl_comm_mem_alloc(comm._c, nbytes, ctypes.byref(p)))
        self.ptr = p.value
        w = ctypes.c_void_p(0)
        try:
            _check(lib.icl_comm_window_register(comm._c, self.ptr, nbytes, ctypes.byref(w)))
        except IclError:
            lib.icl_comm_mem_free(comm._c, self.ptr)
            raise
        self._w = w

    @staticmethod
    def band(peer: int, offset: int, height: int, pitch_bytes: int, batch_stride_bytes: int = 0):
        return icl_window_band(peer, offset, height, pitch_bytes, batch_stride_bytes)

    def image(self, offset: int, width: int, height: int, pitch_bytes: int) -> icl_image:
        """An icl_image over rows of this rank's buffer (fp32)."""
        return icl_image(self.ptr + offset, width, height, pitch_bytes, 1, 0)

    def write(self, offset: int, t, pitch_bytes: int, stream=None):
        """Copy a 2-D device tensor's rows into this rank's buffer at `offset`."""
        _check(load_library().icl_copy_2d(self.ptr + offset, pitch_bytes, t.data_ptr(), t.stride(0) * t.element_size(),
                                          t.shape[-1] * t.element_size(), t.shape[-2], _stream(stream)))

    def close(self):
        if self._w:
            lib = load_library()
            _check(lib.icl_comm_window_deregister(self.comm._c, self._w))
            _check(lib.icl_comm_mem_free(self.comm._c, self.ptr))
            self._w = None


def _wband(b):
    return ctypes.byref(b) if b is not None else None


def sepconv_window(win: Window, own: icl_image, dst, global_height: int, own_y0: int, up, down, taps_x, taps_y,
                   border: str = "constant", border_value: float = 0.0, stream=None):
    """One rank's rows of a row-band sepconv, halo rows read in-kernel through the NCCL window
    (icl_sepconv_window); `own` is an icl_image over the rank's rows (e.g. Window.image)."""
    fx, gy = _taps(taps_x), _taps(taps_y)
    own = own if isinstance(own, icl_image) else _image(own)
    _check(load_library().icl_sepconv_window(win._w, ctypes.byref(own), ctypes.byref(_image(dst)), global_height,
                                             own_y0, _wband(up), _wband(down), ctypes.cast(fx, ctypes.c_void_p),
                                             len(fx) // 2, ctypes.cast(gy, ctypes.c_void_p), len(gy) // 2,
                                             BORDER[border], border_value, _stream(stream)))
    return dst


def harris_window(win: Window, own: icl_image, response, global_height: int, own_y0: int, up, down, block=5,
                  k=0.04, border="clamp", border_value=0.0, mask=None, threshold=0.0, stream=None):
    m = _image(mask, 1) if mask is not None else None
    own = own if isinstance(own, icl_image) else _image(own)
    _check(load_library().icl_harris_window(win._w, ctypes.byref(own), ctypes.byref(_image(response)), global_height,
                                            own_y0, _wband(up), _wband(down), block, k, BORDER[border], border_value,
                                            _ref(m), threshold, _stream(stream)))
    return response


def halo_pull_window(win: Window, buf, global_height: int, buf_y0: int, own_y0: int, own_y1: int, up, down,
                     stream=None):
    elem = buf.element_size()
    _check(load_library().icl_halo_pull_window(win._w, ctypes.byref(_image(buf, elem)), global_height, buf_y0, own_y0,
                                               own_y1, _wband(up), _wband(down), elem, _stream(stream)))
    return buf


def tune_cache_save(path: str):
    _check(load_library().icl_tune_cache_save(path.encode()))


def tune_cache_load(path: str):
    _check(load_library().icl_tune_cache_load(path.encode()))


def tune_cache_clear():
    load_library().icl_tune_cache_clear()


def tune_cache_size() -> int:
    return int(load_library().icl_tune_cache_size())


def variant_names(filter: str) -> list:
    lib = load_library()
    out = []
    buf = ctypes.create_string_buffer(128)
    for i in range(lib.icl_variant_count(FILTER[filter])):
        _check(lib.icl_variant_name(FILTER[filter], i, buf, 128))
        out.append(buf.value.decode())
    return out


def force_variant(filter: str, variant):
    """Force a variant (id or name) on this thread; None/-1 = automatic dispatch."""
    if variant is None:
        variant = -1
    if isinstance(variant, str):
        variant = variant_names(filter).index(variant)
    _check(load_library().icl_force_variant(FILTER[filter], int(variant)))


def last_variant(filter: str) -> int:
    return int(load_library().icl_last_variant(FILTER[filter]))


def launch_count() -> int:
    return int(load_library().icl_launch_count())


def transfer_bytes() -> tuple:
    """Cumulative (host->device, device->host) bytes copied by the host-image path."""
    h, d = ctypes.c_uint64(0), ctypes.c_uint64(0)
    load_library().icl_transfer_bytes(ctypes.byref(h), ctypes.byref(d))
    return int(h.value), int(d.value)


def version() -> str:
    return load_library().icl_version().decode()


def fill_uniform(img, seed: int, row0: int = 0, stream=None):
    """Device SplitMix64 U[0,1) fill, equal to synth.uniform_image(seed + b, ...)."""
    _check(load_library().icl_fill_uniform(ctypes.byref(_image(img)), seed, row0, _stream(stream)))
    return img


def harris_halo(block: int):
    """Rows of input a Harris output row needs above / below (per-stage Sobel + window)."""
    a = block // 2
    return a + 1, block - 1 - a + 1


def nlm_halo(patch_radius: int, search_radius: int):
    r = patch_radius + search_radius
    return r, r


__all__ = ["sepconv", "harris", "nlm", "conv2d_u8", "Comm", "shard_band", "shard_plan", "halo_rows_of", "tune", "tune_cache_save", "tune_cache_load", "tune_cache_clear",
           "tune_cache_size", "variant_names", "force_variant", "last_variant", "launch_count", "transfer_bytes", "version",
           "fill_uniform", "load_library", "IclError", "sepconv_workspace_bytes", "harris_halo", "nlm_halo",
           "EXPORTS", "LIB_PATH"]
