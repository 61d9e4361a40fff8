"""CPU checks of the C-ABI boundary: the library loads, exports every symbol
include/icl.h declares, and the host-side registry answers without a GPU.
No compute calls (there is no GPU here)."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_1605_06399_b200 as icl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "icl.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(icl_[a-z0-9_]+)\s*\(", src)))


def test_library_builds_and_loads():
    from paper_1605_06399_b200 import build
    path = build.build()
    assert os.path.exists(path)
    icl.load_library()
    assert icl.version().startswith("icl-b200")


def test_every_declared_symbol_is_exported():
    decl = _declared()
    assert set(decl) == set(icl.EXPORTS), (set(decl) ^ set(icl.EXPORTS))
    out = subprocess.run(["nm", "-D", "--defined-only", icl.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (icl_[a-z0-9_]+)$", out, flags=re.M))
    missing = set(decl) - exported
    assert not missing, missing
    lib = icl.load_library()
    for name in decl:
        assert getattr(lib, name)


def test_kernels_are_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", icl.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_registry_without_gpu():
    names = icl.variant_names("sepconv")
    assert names[0] == "naive_direct" and any(n.startswith("stream") for n in names)
    assert icl.variant_names("harris")[0] == "naive_direct"
    assert icl.variant_names("nlm")[0] == "naive_direct"
    icl.force_variant("sepconv", 2)
    icl.force_variant("sepconv", None)
    with pytest.raises(icl.IclError):
        icl.force_variant("sepconv", 999)
    assert icl.sepconv_workspace_bytes(512, 512, 1, 2) >= 512 * 516 * 4
    assert icl.tune_cache_size() == 0


def test_invalid_arguments_fail_before_any_launch():
    """Validation is host-side: null / bad descriptors are rejected without a device."""
    lib = icl.load_library()
    img = icl.icl_image(0, 16, 16, 64, 1, 0)  # null data
    taps = (ctypes.c_float * 3)(0.25, 0.5, 0.25)
    st = lib.icl_sepconv(ctypes.byref(img), ctypes.byref(img), ctypes.cast(taps, ctypes.c_void_p), 1,
                         ctypes.cast(taps, ctypes.c_void_p), 1, 0, 0.0, None, None, 0, None)
    assert st == 1 and b"null" in lib.icl_last_error()
    a = icl.icl_image(4096, 16, 16, 32, 1, 0)  # pitch < 4*width
    st = lib.icl_nlm(ctypes.byref(a), ctypes.byref(a), 2, 5, 0.1, 1, 0.0, None, None)
    assert st == 1 and b"pitch" in lib.icl_last_error()
    src = icl.icl_image(4096, 16, 16, 64, 1, 0)
    dst = icl.icl_image(4096 + 64, 16, 16, 64, 1, 0)  # overlaps src
    st = lib.icl_harris(ctypes.byref(src), ctypes.byref(dst), 5, 0.04, 1, 0.0, None, 0.0, None, None)
    assert st == 2
    dst2 = icl.icl_image(1 << 20, 16, 16, 64, 1, 0)
    st = lib.icl_nlm(ctypes.byref(src), ctypes.byref(dst2), 2, 5, 0.0, 1, 0.0, None, None)  # h = 0
    assert st == 1
    st = lib.icl_sepconv(ctypes.byref(src), ctypes.byref(dst2), ctypes.cast(taps, ctypes.c_void_p), 16,
                         ctypes.cast(taps, ctypes.c_void_p), 1, 0, 0.0, None, None, 0, None)
    assert st == 3  # radius > 15


def test_cpu_tensors_need_a_cuda_device():
    """CPU tensors are host images streamed through the GPU; without a CUDA
    device the binding refuses them (no CPU fallback)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("host-image path is exercised by tests/test_gpu_host.py")
    t = torch.zeros(8, 8)
    with pytest.raises(ValueError, match="CUDA"):
        icl.sepconv(t, t.clone(), [1.0], [1.0])
    with pytest.raises(ValueError, match="CUDA"):
        icl.fill_uniform(t, 1)


def test_new_entry_points_validate_on_the_host():
    """icl_sepconv3d / icl_blur_harris / icl_sepconv_peer / icl_halo_pull / icl_tune_ann reject
    bad arguments before touching a device."""
    lib = icl.load_library()
    P = ctypes.c_void_p
    taps = (ctypes.c_float * 17)(*([0.1] * 17))
    tp = ctypes.cast(taps, P)
    src = icl.icl_image(4096, 16, 16, 64, 4, 16 * 64)
    dst = icl.icl_image(1 << 20, 16, 16, 64, 4, 16 * 64)
    # 3-D: radius 8 -> unsupported; shape mismatch / overlap / null
    assert lib.icl_sepconv3d(ctypes.byref(src), ctypes.byref(dst), tp, 8, tp, 1, tp, 1, 0, 0.0, None) == 3
    bad = icl.icl_image(1 << 20, 16, 16, 64, 5, 16 * 64)
    assert lib.icl_sepconv3d(ctypes.byref(src), ctypes.byref(bad), tp, 1, tp, 1, tp, 1, 0, 0.0, None) == 1
    ov = icl.icl_image(4096 + 64, 16, 16, 64, 4, 16 * 64)
    assert lib.icl_sepconv3d(ctypes.byref(src), ctypes.byref(ov), tp, 1, tp, 1, tp, 1, 0, 0.0, None) == 2
    nul = icl.icl_image(0, 16, 16, 64, 4, 16 * 64)
    assert lib.icl_sepconv3d(ctypes.byref(nul), ctypes.byref(dst), tp, 1, tp, 1, tp, 1, 0, 0.0, None) == 1
    # chain: blur radius 4 and Harris block 6 are unsupported
    one = icl.icl_image(4096, 16, 16, 64, 1, 0)
    two = icl.icl_image(1 << 20, 16, 16, 64, 1, 0)
    st = lib.icl_blur_harris(ctypes.byref(one), ctypes.byref(two), tp, 4, tp, 1, 0, 0.0, 5, 0.04, 1, 0.0, None, 0.0,
                             None, None, 0, None)
    assert st == 3
    st = lib.icl_blur_harris(ctypes.byref(one), ctypes.byref(two), tp, 1, tp, 1, 0, 0.0, 6, 0.04, 1, 0.0, None, 0.0,
                             None, None, 0, None)
    assert st == 3
    # peer: a band with rows above but no up neighbour; halo pull with a bad element size
    band = icl.icl_image(4096, 16, 8, 64, 1, 0)
    out = icl.icl_image(1 << 20, 16, 8, 64, 1, 0)
    st = lib.icl_sepconv_peer(ctypes.byref(band), ctypes.byref(out), 16, 8, None, None, tp, 1, tp, 1, 0, 0.0, None)
    assert st == 1 and b"neighbour" in lib.icl_last_error()
    assert lib.icl_halo_pull(ctypes.byref(band), 16, 0, 0, 8, None, None, 2, None) == 1
    st = lib.icl_harris_peer(ctypes.byref(band), ctypes.byref(out), 16, 8, None, None, 5, 0.04, 1, 0.0, None, 0.0,
                             None)
    assert st == 1 and b"neighbour" in lib.icl_last_error()
    assert lib.icl_harris_peer(ctypes.byref(band), ctypes.byref(out), 16, 0, None, None, 9, 0.04, 1, 0.0, None, 0.0,
                               None) == 1  # block > 7
    # model-guided tuning: n1 < 1
    prob = icl.icl_problem()
    assert lib.icl_tune_ann(ctypes.byref(prob), 0, 1, 0, None, None) == 1
    assert icl.variant_names("sepconv3d") == ["naive_direct", "tile64x16"]
