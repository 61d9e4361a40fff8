"""The TMA-fed sepconv stream variants (tma_nt32_*, sepconv_stream.cuh; §3.2 Eq. 1-2,
the separable convolution): interior CTAs stage their input rows with cp.async.bulk.tensor boxes
of a 3-D tensor map (columns x local rows x images) instead of per-thread cp.async.  They keep the
naive per-output order (R16), so every case must equal naive_direct bit for bit (and
hence the oracle) -- at every radius the family is built for, on images wide enough for many
interior CTAs, with padded pitch and batch stride, row bands (the box rows past the band buffer
are zero-filled by the TMA unit and never used) and the batch grid; the default dispatch of a
large aligned image must pick the family ("no TMA tensor loads")."""
import numpy as np
import pytest

import synth
from tests._tol import check_sepconv

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1605_06399_b200 as icl  # noqa: E402

DEV = torch.device("cuda:0")
TMA = [(i, n) for i, n in enumerate(icl.variant_names("sepconv")) if n.startswith("tma_")]


def naive(src, fx, gy, border, c, band=None, shape=None):
    icl.force_variant("sepconv", "naive_direct")
    out = torch.full(shape or tuple(src.shape), float("nan"), device=DEV)
    icl.sepconv(src, out, fx, gy, border, c, band=band)
    icl.force_variant("sepconv", None)
    return out.cpu().numpy()


def padded(img, pitch, bpad=0):
    """(B, H, W) numpy -> CUDA view with row pitch `pitch` and batch stride H*pitch + bpad."""
    b, h, w = img.shape
    flat = torch.full((b * (h * pitch + bpad),), float("nan"), device=DEV)
    v = flat.as_strided((b, h, w), (h * pitch + bpad, pitch, 1))
    v.copy_(torch.from_numpy(img).to(DEV))
    return v


def test_family_present():
    assert [n for _, n in TMA] == ["tma_nt32_s16_v4", "tma_nt32_s32_v4", "tma_nt32_s64_v4", "tma_nt32_s128_v4"]


@pytest.mark.parametrize("r", list(range(16)))
def test_every_radius_bit_identical(r):
    b, h, w = 2, 301, 1500 + 13
    img = np.stack([synth.uniform_image(300 + r + i, h, w) for i in range(b)])
    fx = synth.gaussian_taps(r)
    gy = synth.signed_taps(11, r)
    for border, c in (("constant", 0.4), ("clamp", 0.0)):
        pitch = (w + 3) // 4 * 4 + 4  # 16-byte rows, padding after column w
        src = padded(img, pitch, bpad=64)
        ref = naive(src, fx, gy, border, c)
        ys, xs = np.array([0, 150, 300, 7, 299]), np.array([0, 700, 1512, 1400, 3])
        check_sepconv(ref[1][ys, xs], img[1], fx, gy, border, c, points=(xs, ys))
        for vid, name in TMA:
            icl.force_variant("sepconv", vid)
            out = torch.full((b, h, pitch), float("nan"), device=DEV)
            icl.sepconv(src, out[:, :, :w], fx, gy, border, c)
            o = out.cpu().numpy()
            assert np.isnan(o[:, :, w:]).all(), name
            np.testing.assert_array_equal(o[:, :, :w], ref, err_msg=f"{name} r={r} {border}")
        icl.force_variant("sepconv", None)


@pytest.mark.parametrize("r", [1, 6, 15])
def test_bands(r):
    """Row bands whose buffer ends exactly at the stencil rows: the last TMA box of a CTA reaches
    past the buffer (zero fill), and the first band's box starts at local row 0."""
    H, W = 400, 2048
    img = synth.uniform_image(60 + r, H, W)
    fx = synth.gaussian_taps(r)
    full = torch.from_numpy(img).to(DEV)
    ref = naive(full, fx, fx, "clamp", 0.0)
    for vid, name in TMA:
        icl.force_variant("sepconv", vid)
        for a, b in ((0, 133), (133, 134), (134, 400)):
            s0, s1 = max(0, a - r), min(H, b + r)
            buf = full[s0:s1].clone()
            out = torch.full((b - a, W), float("nan"), device=DEV)
            icl.sepconv(buf, out, fx, fx, "clamp", band=(H, s0, a))
            np.testing.assert_array_equal(out.cpu().numpy(), ref[a:b], err_msg=f"{name} {a}:{b}")
    icl.force_variant("sepconv", None)


def test_short_and_narrow_images():
    """Fewer rows than one TMA box, widths below / at / just above one 144-column box."""
    for h, w in ((1, 4096), (5, 600), (40, 144), (40, 148), (3, 160), (64, 4)):
        img = synth.uniform_image(h * w, h, w)
        fx = synth.gaussian_taps(3)
        src = torch.from_numpy(img).to(DEV)
        ref = naive(src, fx, fx, "constant", 0.2)
        for vid, name in TMA:
            icl.force_variant("sepconv", vid)
            out = torch.full((h, w), float("nan"), device=DEV)
            icl.sepconv(src, out, fx, fx, "constant", 0.2)
            np.testing.assert_array_equal(out.cpu().numpy(), ref, err_msg=f"{name} {h}x{w}")
        icl.force_variant("sepconv", None)


def test_unaligned_source_is_ineligible():
    base = torch.zeros(64 * 300 + 1, device=DEV)
    src = base[1:].view(64, 300)
    dst = torch.empty(64, 300, device=DEV)
    f = synth.gaussian_taps(2)
    for vid, _ in TMA:
        icl.force_variant("sepconv", vid)
        with pytest.raises(icl.IclError):
            icl.sepconv(src, dst, f, f, "clamp")
    icl.force_variant("sepconv", None)


@pytest.mark.parametrize("r", [2, 5, 8])
def test_default_dispatch_takes_tma_for_large_images(r):
    src = torch.from_numpy(synth.uniform_image(9, 2048, 2048)).to(DEV)
    dst = torch.empty_like(src)
    f = synth.gaussian_taps(r)
    icl.force_variant("sepconv", None)
    icl.tune_cache_clear()
    icl.sepconv(src, dst, f, f, "constant")
    torch.cuda.synchronize()
    assert icl.variant_names("sepconv")[icl.last_variant("sepconv")].startswith("tma_nt32_")
