"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Every variant of every filter is compared with the oracle element by element
on seeded inputs (sizes spanning several tiles plus ragged tails, both border
modes), variants are compared with each other (bit-exact: all variants of a
filter share one per-output fp32 operation order, R16), row-band
splits with the unsharded call, and the full BASELINE.json sizes on sampled
pixels.  Tolerances: tests/_tol.py (north_star's 1e-5 / 1e-4).
"""
import math

import numpy as np
import pytest

import synth
from tests._tol import check_harris, check_harris_families, check_nlm, check_sepconv, sampled_variants

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU, skipped there
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1605_06399_b200 as icl  # noqa: E402

DEV = torch.device("cuda:0")
BORDERS = [("constant", 0.0), ("constant", 0.7), ("clamp", 0.0)]


def to_dev(img, pitch=None, fill=float("nan")):
    """(H, W) numpy -> CUDA tensor view with row pitch `pitch` elements (padding = fill)."""
    h, w = img.shape
    pitch = pitch or w
    buf = torch.full((h, pitch), fill, dtype=torch.float32, device=DEV)
    buf[:, :w] = torch.from_numpy(np.ascontiguousarray(img)).to(DEV)
    return buf[:, :w]


def empty_like_dev(h, w, pitch=None, dtype=torch.float32, fill=float("nan")):
    pitch = pitch or w
    if dtype == torch.uint8:
        return torch.full((h, pitch), 77, dtype=dtype, device=DEV)[:, :w]
    return torch.full((h, pitch), fill, dtype=dtype, device=DEV)[:, :w]


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def variants(f):
    return sampled_variants(icl.variant_names(f))


@pytest.fixture(autouse=True)
def _reset_force():
    yield
    for f in ("sepconv", "harris", "nlm"):
        icl.force_variant(f, None)


def run_all_variants(f, call, skip=()):
    """Run `call()` once per eligible variant; returns {name: output ndarray}."""
    outs = {}
    for vid, name in variants(f):
        if name in skip:
            continue
        icl.force_variant(f, vid)
        try:
            out = call()
        except icl.IclError as e:
            if e.status in (3, 4):  # not eligible for this call
                continue
            raise
        outs[name] = out
    icl.force_variant(f, None)
    return outs


# ============================================================================ sepconv
SEP_SHAPES = [(1, 1), (1, 513), (513, 1), (7, 9), (52, 60), (53, 61), (67, 300), (129, 1029), (3, 4099)]


@pytest.mark.parametrize("border,c", BORDERS)
@pytest.mark.parametrize("shape", SEP_SHAPES)
@pytest.mark.parametrize("r", [0, 1, 2, 5, 15])
def test_sepconv_all_variants_vs_oracle(shape, r, border, c):
    h, w = shape
    img = synth.uniform_image(100 + r, h, w)
    fx = synth.gaussian_taps(r)
    gy = synth.signed_taps(7, r) if r % 2 else synth.gaussian_taps(r)
    src = to_dev(img, pitch=((w + 3) // 4) * 4 + 4)
    ws = torch.empty(icl.sepconv_workspace_bytes(w, h, 1, r) // 4 + 1, dtype=torch.float32, device=DEV)

    def call():
        dst = empty_like_dev(h, w, pitch=((w + 3) // 4) * 4 + 8)
        icl.sepconv(src, dst, fx, gy, border, c, workspace=ws)
        out = host(dst)
        full = host(dst.as_strided((h, dst.stride(0)), (dst.stride(0), 1)))
        assert np.isnan(full[:, w:]).all(), "padding was written"
        return out

    outs = run_all_variants("sepconv", call)
    assert len(outs) >= 3
    base = outs["naive_direct"]
    check_sepconv(base, img, fx, gy, border, c)
    for name, o in outs.items():
        np.testing.assert_array_equal(o, base, err_msg=f"variant {name} not bit-identical")


@pytest.mark.parametrize("rx,ry", [(0, 3), (4, 1), (15, 2), (2, 9)])
def test_sepconv_unequal_radii(rx, ry):
    img = synth.uniform_image(5, 70, 130) - np.float32(0.5)
    fx, gy = synth.signed_taps(1, rx), synth.signed_taps(2, ry)
    src = to_dev(img)
    ws = torch.empty(icl.sepconv_workspace_bytes(130, 70, 1, ry) // 4 + 1, dtype=torch.float32, device=DEV)

    def call():
        dst = empty_like_dev(70, 130)
        icl.sepconv(src, dst, fx, gy, "clamp", workspace=ws)
        return host(dst)
    outs = run_all_variants("sepconv", call)
    check_sepconv(outs["naive_direct"], img, fx, gy, "clamp", 0.0)
    for name, o in outs.items():
        np.testing.assert_array_equal(o, outs["naive_direct"], err_msg=name)


def test_sepconv_batch_and_unaligned():
    b, h, w = 3, 37, 101
    imgs = np.stack([synth.uniform_image(20 + i, h, w) for i in range(b)])
    base = torch.full((b * h * 103 + 1,), float("nan"), device=DEV)
    src = base[1:1 + b * h * 103].view(b, h, 103)[:, :, :w]  # 4-byte aligned only
    src.copy_(torch.from_numpy(imgs).to(DEV))
    dst = torch.full((b, h, w), float("nan"), device=DEV)
    fx = synth.gaussian_taps(3)
    outs = run_all_variants("sepconv", lambda: (icl.sepconv(src, dst, fx, fx, "clamp"), host(dst))[1])
    assert "stream_nt64_s64_v1" in outs and "stream_nt64_s64_v4" not in outs
    for i in range(b):
        check_sepconv(outs["naive_direct"][i], imgs[i], fx, fx, "clamp", 0.0)
    for name, o in outs.items():
        np.testing.assert_array_equal(o, outs["naive_direct"], err_msg=name)


def test_sepconv_linearity_exact():
    """conv(2u) == 2 conv(u) bit-exactly (power-of-two scaling)."""
    img = synth.uniform_image(3, 200, 300)
    fx = synth.gaussian_taps(4)
    a, b2 = to_dev(img), to_dev(img * np.float32(2))
    o1, o2 = empty_like_dev(200, 300), empty_like_dev(200, 300)
    icl.sepconv(a, o1, fx, fx, "clamp")
    icl.sepconv(b2, o2, fx, fx, "clamp")
    np.testing.assert_array_equal(host(o2), 2 * host(o1))


def test_sepconv_config_512():
    """BASELINE.json configs[0]: 512x512, 5-tap Gaussian, 1 GPU vs CPU oracle (full image)."""
    img = synth.uniform_image(1, 512, 512)
    fx = synth.gaussian_taps(2)
    for border in ("constant", "clamp"):
        dst = empty_like_dev(512, 512)
        icl.sepconv(to_dev(img), dst, fx, fx, border)
        check_sepconv(host(dst), img, fx, fx, border, 0.0)


@pytest.mark.parametrize("r", [7, 15])
@pytest.mark.parametrize("border,c", [("constant", 0.7), ("clamp", 0.0)])
def test_sepconv_tile_persistent_vs_oracle(r, border, c):
    """More 64x64 tiles (2 x 18 x 21 = 756) than the persistent grid (2 CTAs per
    SM = 296), ragged right / bottom tiles and padded pitch: exercises the
    cp.async prefetch of the next tile (interior and border) in tile64p_v4."""
    b, h, w = 2, 1300, 1100 + 37
    imgs = np.stack([synth.uniform_image(40 + r + i, h, w) for i in range(b)])
    fx, gy = synth.gaussian_taps(r), synth.signed_taps(9, r)
    pitch = ((w + 3) // 4) * 4 + 12
    sbuf = torch.full((b, h, pitch), float("nan"), device=DEV)
    sbuf[:, :, :w] = torch.from_numpy(imgs).to(DEV)
    src = sbuf[:, :, :w]

    def call():
        dbuf = torch.full((b, h, pitch), float("nan"), device=DEV)
        icl.sepconv(src, dbuf[:, :, :w], fx, gy, border, c)
        full = host(dbuf)
        assert np.isnan(full[:, :, w:]).all(), "padding was written"
        return full[:, :, :w]
    outs = run_all_variants("sepconv", call, skip=("naive_2pass",))
    assert "tile64p_v4" in outs and "tile64_v4" in outs
    for i in range(b):
        check_sepconv(outs["naive_direct"][i], imgs[i], fx, gy, border, c)
    for name, o in outs.items():
        np.testing.assert_array_equal(o, outs["naive_direct"], err_msg=f"variant {name} not bit-identical")


@pytest.mark.parametrize("border", ["constant", "clamp"])
def test_sepconv_bands_bit_exact_all_variants_r9(border):
    """Row bands through every variant (incl. the tile kernels' global-row logic)."""
    H, W, r = 700, 333, 9
    img = synth.uniform_image(18, H, W)
    fx = synth.gaussian_taps(r)
    P = 336  # 16-byte pitch: every variant eligible
    full = empty_like_dev(H, W, pitch=P)
    icl.sepconv(to_dev(img, pitch=P), full, fx, fx, border, 0.3)
    ref = host(full)
    cuts = [0, 5, 250, 251, 699, 700]
    for vid, name in variants("sepconv"):
        if name == "naive_2pass":  # needs a workspace; covered elsewhere
            continue
        icl.force_variant("sepconv", vid)
        for a, b in zip(cuts[:-1], cuts[1:]):
            s0, s1 = max(0, a - r), min(H, b + r)
            dst = empty_like_dev(b - a, W, pitch=P)
            try:
                icl.sepconv(to_dev(img[s0:s1], pitch=P), dst, fx, fx, border, 0.3, band=(H, s0, a))
            except icl.IclError as e:
                if e.status in (3, 4):  # not eligible for this call
                    continue
                raise
            np.testing.assert_array_equal(host(dst), ref[a:b], err_msg=f"{name} band {a}:{b}")


@pytest.mark.parametrize("rx,ry", [(2, 1), (7, 2), (15, 0), (1, 3)])
def test_sepconv_bands_unequal_radii_stay_inside_the_buffer(rx, ry):
    """A band holding only ry halo rows with rx > ry: the fused variants pad the taps to
    max(rx, ry) and would read rows outside the band buffer (found by the N-rank loopback
    exchange); they are ineligible there, and every variant that runs must equal the unsharded
    call.  The band buffer sits between NaN guard rows, so any such read shows up as NaN."""
    H, W = 150, 260
    img = synth.uniform_image(31 + rx, H, W)
    fx, gy = synth.gaussian_taps(rx), synth.gaussian_taps(ry)
    full = empty_like_dev(H, W)
    icl.sepconv(to_dev(img), full, fx, gy, "clamp")
    ref = host(full)
    G = 16
    for vid, name in [(None, "default")] + list(variants("sepconv")):
        if name == "naive_2pass":
            continue
        icl.force_variant("sepconv", vid)
        for a, b in ((0, 1), (1, 60), (60, 61), (61, 149), (149, 150)):
            s0, s1 = max(0, a - ry), min(H, b + ry)
            big = torch.full((s1 - s0 + 2 * G, W), float("nan"), device=DEV)
            big[G:G + s1 - s0] = torch.from_numpy(img[s0:s1]).to(DEV)
            dst = empty_like_dev(b - a, W)
            try:
                icl.sepconv(big[G:G + s1 - s0], dst, fx, gy, "clamp", band=(H, s0, a))
            except icl.IclError as e:
                if e.status in (3, 4):
                    continue
                raise
            np.testing.assert_array_equal(host(dst), ref[a:b], err_msg=f"{name} band {a}:{b}")
    icl.force_variant("sepconv", None)


@pytest.mark.parametrize("border", ["constant", "clamp"])
def test_sepconv_bands_bit_exact(border):
    """Row bands (icl_band) stitched == the unsharded call, bit for bit."""
    H, W, r = 301, 257, 4
    img = synth.uniform_image(8, H, W)
    fx = synth.gaussian_taps(r)
    full = empty_like_dev(H, W)
    icl.sepconv(to_dev(img), full, fx, fx, border, 0.3)
    ref = host(full)
    cuts = [0, 1, 50, 51, 200, 300, 301]
    for a, b in zip(cuts[:-1], cuts[1:]):
        s0, s1 = max(0, a - r), min(H, b + r)
        dst = empty_like_dev(b - a, W)
        icl.sepconv(to_dev(img[s0:s1]), dst, fx, fx, border, 0.3, band=(H, s0, a))
        np.testing.assert_array_equal(host(dst), ref[a:b])


# ============================================================================ harris
HAR_SHAPES = [(1, 1), (5, 1), (1, 9), (9, 7), (52, 60), (53, 61), (130, 517)]


@pytest.mark.parametrize("border,c", BORDERS)
@pytest.mark.parametrize("shape", HAR_SHAPES)
@pytest.mark.parametrize("block", [1, 2, 3, 5, 7])
def test_harris_all_variants_vs_oracle(shape, block, border, c):
    h, w = shape
    img = synth.rect_scene(40 + block, h, w, n_rect=8, noise=0.01)
    src = to_dev(img, pitch=((w + 3) // 4) * 4 + 4)
    R0 = None
    thr = 0.0

    def call():
        resp = empty_like_dev(h, w, pitch=((w + 3) // 4) * 4 + 4)
        mask = empty_like_dev(h, w, pitch=((w + 3) // 4) * 4 + 4, dtype=torch.uint8)
        icl.harris(src, resp, block, 0.04, border, c, mask=mask, threshold=thr)
        return host(resp), host(mask)

    outs = run_all_variants("harris", call)
    assert len(outs) >= 2
    R0, M0 = outs["naive_direct"]
    check_harris(R0, M0, img, block, 0.04, border, c, thr)
    check_harris_families(outs, img, block, 0.04, border, c, thr)


def test_harris_config_2048_sampled():
    """BASELINE.json configs[1]: 2048^2, Sobel 3x3 + 5x5 window, k=0.04 (rectangles scene)."""
    H = W = 2048
    img = synth.rect_scene(2, H, W, n_rect=256, noise=0.01)
    resp = torch.empty(H, W, device=DEV)
    mask = torch.empty(H, W, dtype=torch.uint8, device=DEV)
    src = to_dev(img)
    icl.harris(src, resp, 5, 0.04, "clamp")
    R = host(resp)
    thr = float(np.float32(0.01 * R.max()))
    icl.harris(src, resp, 5, 0.04, "clamp", mask=mask, threshold=thr)
    R, M = host(resp), host(mask)
    rng = np.random.default_rng(0)
    ys = np.concatenate([rng.integers(0, H, 3000), [0, 0, H - 1, H - 1, 1, H - 2]])
    xs = np.concatenate([rng.integers(0, W, 3000), [0, W - 1, 0, W - 1, 2, W - 3]])
    # plus every pixel of a few edge/corner windows
    for y0, x0 in ((0, 0), (H - 8, W - 8), (1000, 0), (0, 1000)):
        yy, xx = np.mgrid[y0:y0 + 8, x0:x0 + 8]
        ys, xs = np.concatenate([ys, yy.ravel()]), np.concatenate([xs, xx.ravel()])
    check_harris(R[ys, xs], M[ys, xs], img, 5, 0.04, "clamp", 0.0, thr, points=(xs, ys))
    assert M.sum() > 100  # the scene has corners


def test_harris_flat_and_scaling_exact():
    img = synth.rect_scene(9, 120, 90, n_rect=10, noise=0.01)
    for vid, name in [(None, "default")] + list(variants("harris")):
        icl.force_variant("harris", vid)
        r1, r2 = empty_like_dev(120, 90, pitch=92), empty_like_dev(120, 90, pitch=92)
        icl.harris(to_dev(img, pitch=92), r1, 5, 0.04, "clamp")
        icl.harris(to_dev(img * np.float32(2), pitch=92), r2, 5, 0.04, "clamp")
        np.testing.assert_array_equal(host(r2), 16 * host(r1), err_msg=name)
        flat = np.full((40, 120), 0.37, np.float32)
        f1 = empty_like_dev(40, 120)
        icl.harris(to_dev(flat), f1, 5, 0.04, "clamp")
        assert not host(f1).any(), name
    icl.force_variant("harris", None)


@pytest.mark.parametrize("border", ["constant", "clamp"])
def test_harris_bands_bit_exact(border):
    H, W, B = 203, 150, 5
    img = synth.rect_scene(11, H, W, n_rect=12, noise=0.01)
    full = empty_like_dev(H, W)
    icl.harris(to_dev(img), full, B, 0.04, border, 0.2)
    ref = host(full)
    up, down = icl.harris_halo(B)
    cuts = [0, 2, 70, 71, 202, 203]
    for a, b in zip(cuts[:-1], cuts[1:]):
        s0, s1 = max(0, a - up), min(H, b + down)
        dst = empty_like_dev(b - a, W)
        icl.harris(to_dev(img[s0:s1]), dst, B, 0.04, border, 0.2, band=(H, s0, a))
        np.testing.assert_array_equal(host(dst), ref[a:b])
    # every variant family on its own: stitched bands == its unsharded call, bit for bit
    P = 152  # 16-byte pitch: the float4 variants are eligible
    for vid, name in variants("harris"):
        icl.force_variant("harris", vid)
        full = empty_like_dev(H, W, pitch=P)
        icl.harris(to_dev(img, pitch=P), full, B, 0.04, border, 0.2)
        ref = host(full)
        for a, b in zip(cuts[:-1], cuts[1:]):
            s0, s1 = max(0, a - up), min(H, b + down)
            dst = empty_like_dev(b - a, W, pitch=P)
            icl.harris(to_dev(img[s0:s1], pitch=P), dst, B, 0.04, border, 0.2, band=(H, s0, a))
            np.testing.assert_array_equal(host(dst), ref[a:b], err_msg=f"{name} band {a}:{b}")
    icl.force_variant("harris", None)


# ============================================================================ nlm
NLM_CASES = [(2, 5, 0.1), (1, 3, 0.05), (0, 1, 0.25), (3, 7, 0.2), (2, 5, 1e-6), (2, 5, math.inf), (2, 5, 1.0),
             (1, 10, 0.1)]


@pytest.mark.parametrize("border,c", [("clamp", 0.0), ("constant", 0.5)])
@pytest.mark.parametrize("shape", [(1, 1), (9, 7), (37, 70)])
@pytest.mark.parametrize("P,S,h", NLM_CASES)
def test_nlm_all_variants_vs_oracle(shape, P, S, h, border, c):
    hh, w = shape
    img = synth.rect_scene(60 + P + S, hh, w, n_rect=6, noise=0.0866)
    src = to_dev(img, pitch=w + 3)

    def call():
        dst = empty_like_dev(hh, w, pitch=w + 5)
        icl.nlm(src, dst, P, S, h, border, c)
        return host(dst)

    outs = run_all_variants("nlm", call)
    base = outs["naive_direct"]
    check_nlm(base, img, P, S, h, border, c)
    for name, o in outs.items():
        check_nlm(o, img, P, S, h, border, c)


def test_nlm_config_1024_sampled():
    """BASELINE.json configs[2]: 1024^2, 5x5 patch, 11x11 search window (sampled pixels)."""
    H = W = 1024
    img = synth.rect_scene(3, H, W, n_rect=256, noise=0.0866)
    dst = torch.empty(H, W, device=DEV)
    icl.nlm(to_dev(img), dst, 2, 5, 0.1, "clamp")
    out = host(dst)
    rng = np.random.default_rng(1)
    ys = np.concatenate([rng.integers(0, H, 2000), [0, 0, H - 1, H - 1]])
    xs = np.concatenate([rng.integers(0, W, 2000), [0, W - 1, 0, W - 1]])
    for y0, x0 in ((0, 0), (H - 12, W - 12), (500, 0)):
        yy, xx = np.mgrid[y0:y0 + 12, x0:x0 + 12]
        ys, xs = np.concatenate([ys, yy.ravel()]), np.concatenate([xs, xx.ravel()])
    check_nlm(out[ys, xs], img, 2, 5, 0.1, "clamp", 0.0, points=(xs, ys))


def test_nlm_limits():
    img = synth.uniform_image(4, 64, 80)
    d = empty_like_dev(64, 80)
    icl.nlm(to_dev(img), d, 2, 5, 1e-6, "clamp")
    np.testing.assert_array_equal(host(d), img)  # h -> 0: identity
    const = np.full((30, 40), 0.4, np.float32)
    icl.nlm(to_dev(const), d[:30, :40], 2, 5, 0.1, "clamp")
    np.testing.assert_allclose(host(d[:30, :40]), np.float32(0.4), rtol=1e-6)


@pytest.mark.parametrize("P,S", [(0, 1), (0, 5), (1, 3), (1, 5), (2, 5), (3, 4)])
def test_nlm_tiny_h_quantized(P, S):
    """sliding patch sums ((h + new^2) - old^2) can round below zero; with a tiny h a
    negative distance would give w = +inf and a NaN output.  Quantised k/255 pixels make equal
    patches common (d = 0 exactly in the definition); every variant must return the input
    (h -> 0 limit, SURVEY.md §8(c) pin) and match the oracle."""
    rng = np.random.default_rng(100 + 10 * P + S)
    img = (rng.integers(0, 256, (61, 83)) / 255.0).astype(np.float32)
    img[20:40, 10:50] = np.float32(7 / 255)  # flat block: many exactly-equal patches
    src = to_dev(img)

    def call():
        dst = empty_like_dev(61, 83)
        icl.nlm(src, dst, P, S, 1e-6, "clamp")
        return host(dst)

    for name, o in run_all_variants("nlm", call).items():
        assert np.isfinite(o).all(), name
        check_nlm(o, img, P, S, 1e-6, "clamp", 0.0)


@pytest.mark.parametrize("border", ["constant", "clamp"])
def test_nlm_bands(border):
    H, W, P, S = 90, 75, 2, 5
    img = synth.rect_scene(12, H, W, n_rect=10, noise=0.0866)
    full = empty_like_dev(H, W)
    icl.nlm(to_dev(img), full, P, S, 0.1, border, 0.5)
    ref = host(full)
    up, down = icl.nlm_halo(P, S)
    cuts = [0, 3, 40, 89, 90]
    for a, b in zip(cuts[:-1], cuts[1:]):
        s0, s1 = max(0, a - up), min(H, b + down)
        dst = empty_like_dev(b - a, W)
        icl.nlm(to_dev(img[s0:s1]), dst, P, S, 0.1, border, 0.5, band=(H, s0, a))
        np.testing.assert_allclose(host(dst), ref[a:b], rtol=0, atol=1e-5)


# ============================================================================ infrastructure
def test_fill_uniform_matches_synth():
    b, h, w = 2, 33, 70
    t = torch.empty(b, h, w, device=DEV)
    icl.fill_uniform(t, 5, row0=3)
    got = host(t)
    for i in range(b):
        ref = synth.uniform_image(5 + i, h + 3, w)[3:]
        np.testing.assert_array_equal(got[i], ref)


def test_tuner_picks_equivalent_variant_and_caches(tmp_path):
    icl.tune_cache_clear()
    img = synth.uniform_image(1, 512, 512)
    src, dst = to_dev(img), empty_like_dev(512, 512)
    fx = synth.gaussian_taps(2)
    ws = torch.empty(icl.sepconv_workspace_bytes(512, 512, 1, 2) // 4 + 1, device=DEV)
    info = icl.tune("sepconv", src, dst, taps_x=fx, taps_y=fx, border="constant", workspace=ws)
    assert info["n_candidates"] >= 5 and info["n_rejected"] == 0 and not info["from_cache"]
    check_sepconv(host(dst), img, fx, fx, "constant", 0.0)
    again = icl.tune("sepconv", src, dst, taps_x=fx, taps_y=fx, border="constant", workspace=ws)
    assert again["from_cache"] and again["variant_id"] == info["variant_id"]
    icl.sepconv(src, dst, fx, fx, "constant", workspace=ws)
    assert icl.last_variant("sepconv") == info["variant_id"]
    p = str(tmp_path / "cache.json")
    icl.tune_cache_save(p)
    icl.tune_cache_clear()
    assert icl.tune_cache_size() == 0
    icl.tune_cache_load(p)
    assert icl.tune_cache_size() == 1
    h = icl.tune("harris", src, dst, block=5, k=0.04, border="clamp")
    assert h["n_rejected"] == 0
    n = icl.tune("nlm", src[:128, :128], dst[:128, :128], patch_radius=2, search_radius=5, h=0.1)
    assert n["n_rejected"] == 0


def test_model_guided_tuner(tmp_path):
    """icl_tune_ann: n1 random variants, surrogate, top-k;
    the winner is a verified variant and is cached like icl_tune's."""
    icl.tune_cache_clear()
    img = synth.uniform_image(3, 1024, 1024)
    src, dst = to_dev(img), empty_like_dev(1024, 1024)
    n_elig = sum(1 for n in icl.variant_names("sepconv") if n != "naive_2pass")  # (no workspace given)
    info = icl.tune("sepconv", src, dst, taps_x=synth.gaussian_taps(2), taps_y=synth.gaussian_taps(2),
                    border="constant", ann=(10, 4, 7))
    assert info["n_rejected"] == 0 and not info["from_cache"]
    assert info["n_candidates"] == min(14, n_elig)
    check_sepconv(host(dst), img, synth.gaussian_taps(2), synth.gaussian_taps(2), "constant", 0.0)
    icl.sepconv(src, dst, synth.gaussian_taps(2), synth.gaussian_taps(2), "constant")
    assert icl.last_variant("sepconv") == info["variant_id"]
    h = icl.tune("harris", src, dst, block=5, k=0.04, border="clamp", ann=(10, 1, 1))
    assert h["n_rejected"] == 0 and h["n_candidates"] == 11  # 10 + 1 of the eligible Harris variants
    ref = empty_like_dev(1024, 1024)
    icl.force_variant("harris", "naive_direct")
    icl.harris(src, ref, 5, 0.04, "clamp")
    icl.force_variant("harris", None)
    if h["name"].startswith("slide"):  # the re-associated families: the oracle tolerance
        check_harris(host(dst), None, img, 5, 0.04, "clamp", 0.0, 0.0)
    else:  # every other Harris variant shares the naive fp32 order
        assert torch.equal(dst, ref)


def test_errors_are_reported():
    a = torch.zeros(16, 16, device=DEV)
    with pytest.raises(icl.IclError) as e:
        icl.sepconv(a, a, [1.0], [1.0])
    assert e.value.status == 2  # aliasing
    with pytest.raises(icl.IclError) as e:
        icl.nlm(a, torch.zeros(16, 16, device=DEV), 2, 5, -1.0)
    assert e.value.status == 1
    with pytest.raises(icl.IclError) as e:
        icl.force_variant("sepconv", "naive_2pass")
        icl.sepconv(a, torch.zeros(16, 16, device=DEV), [1.0], [1.0])  # no workspace
    assert e.value.status == 4
    icl.force_variant("sepconv", None)


def test_launch_counter_advances():
    n0 = icl.launch_count()
    a = torch.rand(64, 64, device=DEV)
    icl.sepconv(a, torch.empty_like(a), [0.25, 0.5, 0.25], [0.25, 0.5, 0.25])
    assert icl.launch_count() > n0
