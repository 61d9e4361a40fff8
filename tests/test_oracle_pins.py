"""Pins for the CPU oracle against what the paper and the mathematics fix.

None of these re-types the oracle's formula: each compares it with a printed
example (tests/golden/*.json, each citing its source), a closed form, a
textbook/library routine that the definition reduces to (scipy.ndimage
correlate / uniform_filter), or an invariant.  The set is chosen so that a
dropped term, a sign error, a transposed operand or an off-by-one in a
window fails at least one of them.
"""
import math

import numpy as np
import pytest
import scipy.ndimage as ndi

import oracle
import synth

BORDERS = [("constant", 0.0), ("constant", 0.7), ("clamp", 0.0)]


def _mode(border, c):
    return dict(mode="nearest") if border == "clamp" else dict(mode="constant", cval=float(np.float32(c)))


# ----------------------------------------------------------------------------- boundary
def test_boundary_reads_spec_examples():
    """clamped (-1,0) -> buf[0]; constant(0) at (8,3) -> 0; (3,2) -> buf[19].

    A 1-tap identity convolution evaluated at those points returns the bare read."""
    img = np.arange(64, dtype=np.float32).reshape(8, 8) + 1.0  # buf[i] = i+1
    one = np.ones(1, np.float32)
    pts = (np.array([-1, 8, 3]), np.array([0, 3, 2]))
    v_clamp = oracle.sepconv(img, one, one, "clamp", points=pts)
    v_const = oracle.sepconv(img, one, one, "constant", 0.0, points=pts)
    assert v_clamp[0] == 1.0            # buf[0]
    assert v_const[1] == 0.0            # outside -> constant 0
    assert v_const[2] == 20.0           # buf[19]


# ----------------------------------------------------------------------------- sepconv
def test_sepconv_spec_box3(golden):
    g = golden("sepconv_spec_box3.json")
    img = np.full((g["image"]["height"], g["image"]["width"]), g["image"]["value"], np.float32)
    out = oracle.sepconv(img, g["taps_x"], g["taps_y"], g["border"], g["border_value"]) / g["divide_by"]
    e = g["expect"]
    assert abs(out[3, 4] - e["interior"]) < 1e-12
    assert abs(out[0, 0] - e["corner"]) < 1e-12
    assert abs(out[7, 7] - e["corner"]) < 1e-12
    assert abs(out[0, 4] - e["edge"]) < 1e-12
    assert abs(out[4, 7] - e["edge"]) < 1e-12


def test_sepconv_delta_orientation(golden):
    g = golden("sepconv_delta.json")
    h, w = g["image"]["height"], g["image"]["width"]
    x0, y0 = g["image"]["delta"]
    img = np.zeros((h, w), np.float32)
    img[y0, x0] = 1.0
    out = oracle.sepconv(img, g["taps_x"], g["taps_y"], "constant", 0.0)
    np.testing.assert_array_equal(out[y0 - 1:y0 + 2, x0 - 1:x0 + 2], np.array(g["expect_block"]))
    out[y0 - 1:y0 + 2, x0 - 1:x0 + 2] = 0
    assert not out.any()


@pytest.mark.parametrize("border,c", BORDERS)
def test_sepconv_constant_image(border, c):
    """c-image: clamp (or constant c) -> c*sum(f)*sum(g) everywhere (closed form)."""
    val = 0.7 if border == "clamp" else c
    img = np.full((6, 9), np.float32(val), np.float32)
    f = synth.signed_taps(3, 2)
    g = synth.signed_taps(4, 3)
    out = oracle.sepconv(img, f, g, border, c)
    if border == "constant" and c == 0.0:
        return  # interior only: covered by the scipy pin
    exp = float(np.float32(val)) * f.astype(np.float64).sum() * g.astype(np.float64).sum()
    np.testing.assert_allclose(out, exp, rtol=1e-13, atol=1e-15)


@pytest.mark.parametrize("border,c", BORDERS)
@pytest.mark.parametrize("shape,rx,ry", [((7, 9), 2, 1), ((9, 7), 1, 3), ((1, 13), 4, 2),
                                         ((13, 1), 0, 5), ((5, 5), 6, 6)])
def test_sepconv_equals_2d_correlation(border, c, shape, rx, ry):
    """Separable = 2-D correlation with the outer-product kernel (scipy.ndimage.correlate)."""
    img = synth.uniform_image(11, *shape) - np.float32(0.5)
    f = synth.signed_taps(5, rx)
    g = synth.signed_taps(6, ry)
    out = oracle.sepconv(img, f, g, border, c)
    ref = ndi.correlate(img.astype(np.float64), np.outer(g.astype(np.float64), f.astype(np.float64)),
                        **_mode(border, c))
    np.testing.assert_allclose(out, ref, rtol=0, atol=1e-13)


def test_sepconv_pitched_and_points():
    img = synth.uniform_image(2, 17, 23)
    padded = synth.pitched(img, 32)
    f, g = synth.gaussian_taps(2), synth.gaussian_taps(3)
    full = oracle.sepconv(img, f, g, "clamp")
    np.testing.assert_array_equal(oracle.sepconv(padded, f, g, "clamp"), full)
    xs = np.array([0, 22, 5, 11]); ys = np.array([0, 16, 9, 3])
    np.testing.assert_array_equal(oracle.sepconv(img, f, g, "clamp", points=(xs, ys)), full[ys, xs])
    # thread count does not change results
    np.testing.assert_array_equal(oracle.sepconv(img, f, g, "clamp", threads=1), full)


def test_gaussian_taps_closed_form():
    """SURVEY.md §8(c) #3 values (computed from sigma(r)=0.3(r-1)+0.8)."""
    # the survey prints 8 significant digits
    np.testing.assert_allclose(synth.gaussian_taps(2), np.array(
        [0.07076637, 0.2444604, 0.36954647, 0.2444604, 0.07076637]), rtol=2e-7)
    np.testing.assert_allclose(synth.gaussian_taps(1), np.array(
        [0.23899427, 0.52201146, 0.23899427]), rtol=2e-7)
    for r in range(1, 16):
        t = synth.gaussian_taps(r).astype(np.float64)
        assert abs(t.sum() - 1.0) < 1e-6 and np.all(t == t[::-1]) and t.argmax() == r


# ----------------------------------------------------------------------------- harris
def _harris_scipy(img, block, k, border, c):
    """Per-stage Harris via library correlations (independent of the oracle)."""
    v = np.array([1.0, 2.0, 1.0]); d = np.array([-1.0, 0.0, 1.0])
    x = img.astype(np.float64)
    dx = ndi.correlate(x, np.outer(v, d), **_mode(border, c))
    dy = ndi.correlate(x, np.outer(d, v), **_mode(border, c))
    box = np.ones((block, block))
    m2 = dict(mode="nearest") if border == "clamp" else dict(mode="constant", cval=0.0)
    sxx = ndi.correlate(dx * dx, box, **m2)
    sxy = ndi.correlate(dx * dy, box, **m2)
    syy = ndi.correlate(dy * dy, box, **m2)
    kk = float(np.float32(k))
    return sxx * syy - sxy * sxy - kk * (sxx + syy) ** 2, np.stack([sxx, sxy, syy], -1)


@pytest.mark.parametrize("border,c", BORDERS)
@pytest.mark.parametrize("block", [1, 2, 3, 4, 5, 7])
@pytest.mark.parametrize("shape", [(9, 7), (6, 11), (1, 5), (4, 1)])
def test_harris_matches_library_per_stage(border, c, block, shape):
    img = synth.rect_scene(3, *shape, n_rect=4, noise=0.05)
    R, S = oracle.harris(img, block, 0.04, border, c, with_tensor=True)
    Rr, Sr = _harris_scipy(img, block, 0.04, border, c)
    np.testing.assert_allclose(S, Sr, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(R, Rr, rtol=1e-10, atol=1e-10)


def test_harris_step_corner(golden):
    g = golden("harris_step_corner.json")
    H = W = 48
    x0 = y0 = 16
    img = np.zeros((H, W), np.float32)
    img[y0:, x0:] = 1.0
    for case in g["cases"]:
        dx, dy = case["at"]
        xs, ys = np.array([x0 + dx]), np.array([y0 + dy])
        R, S = oracle.harris(img, case["block"], g["k"], "clamp", points=(xs, ys), with_tensor=True)
        # k is passed as fp32(0.04); the golden uses k = 1/25 exactly -> allow k rounding
        tr = S[0, 0] + S[0, 2]
        assert abs(R[0] - case["R"]) <= 1e-12 + abs(tr * tr) * 1e-8, case
        for key, idx in (("Sxx", 0), ("Sxy", 1), ("Syy", 2)):
            if key in case:
                assert S[0, idx] == case[key], case


@pytest.mark.parametrize("border,c", [("clamp", 0.0), ("constant", 0.3)])
def test_harris_flat_is_zero(border, c):
    img = np.full((10, 12), 0.3, np.float32)
    R = oracle.harris(img, 5, 0.04, border, c)
    if border == "clamp":
        assert not R.any()
    else:  # interior flat region is exactly 0 with c == image value
        assert not R.any()


def test_harris_invariants():
    img = synth.rect_scene(7, 21, 17, n_rect=6, noise=0.02)
    R = oracle.harris(img, 5, 0.04, "clamp")
    np.testing.assert_array_equal(oracle.harris(img * np.float32(2), 5, 0.04, "clamp"), 16 * R)
    # transposition swaps dx and dy -> R invariant (square window, symmetric anchor)
    Rt = oracle.harris(np.ascontiguousarray(img.T), 5, 0.04, "clamp")
    np.testing.assert_allclose(Rt.T, R, rtol=1e-12, atol=1e-12)
    # R(u + c) = R(u) (derivatives of a constant vanish) under clamp
    Rs = oracle.harris(img + np.float32(0.25), 5, 0.04, "clamp")
    np.testing.assert_allclose(Rs, R, rtol=0, atol=1e-6 * np.abs(R).max())


# ----------------------------------------------------------------------------- nlm
def test_nlm_worked_example(golden):
    g = golden("nlm_arange3.json")
    img = np.array(g["image"], np.float32)
    for case in g["cases"]:
        out = oracle.nlm(img, case["patch_radius"], case["search_radius"], case["h"], "clamp")
        np.testing.assert_allclose(out, np.array(case["expect"]), rtol=0, atol=g["tolerance_abs"])


@pytest.mark.parametrize("shape,s", [((9, 13), 2), ((12, 7), 5), ((1, 9), 3)])
def test_nlm_h_inf_is_box_mean(shape, s):
    """h -> inf: every weight is 1 -> clamped box mean over (2s+1)^2 (scipy uniform_filter)."""
    img = synth.uniform_image(9, *shape)
    out = oracle.nlm(img, 2, s, math.inf, "clamp")
    ref = ndi.uniform_filter(img.astype(np.float64), size=2 * s + 1, mode="nearest")
    np.testing.assert_allclose(out, ref, rtol=0, atol=1e-14)


def test_nlm_h_zero_is_identity():
    """h -> 0: all off-centre weights underflow to 0, den = 1 -> out == input exactly."""
    img = synth.uniform_image(12, 11, 10)
    out = oracle.nlm(img, 2, 5, 1e-6, "clamp")
    np.testing.assert_array_equal(out, img.astype(np.float64))


@pytest.mark.parametrize("border,c", [("clamp", 0.0), ("constant", 0.4)])
def test_nlm_constant_image(border, c):
    img = np.full((8, 9), 0.4, np.float32)
    out = oracle.nlm(img, 1, 3, 0.1, border, c)
    np.testing.assert_allclose(out, float(np.float32(0.4)), rtol=1e-15)


def test_nlm_invariants():
    img = synth.rect_scene(5, 15, 14, n_rect=5, noise=0.0866)
    out, scale = oracle.nlm(img, 2, 3, 0.1, "clamp", with_scale=True)
    out2 = oracle.nlm(img * np.float32(2), 2, 3, 0.2, "clamp")
    np.testing.assert_array_equal(out2, 2 * out)
    lo = ndi.minimum_filter(img.astype(np.float64), size=7, mode="nearest")
    hi = ndi.maximum_filter(img.astype(np.float64), size=7, mode="nearest")
    assert np.all(out >= lo - 1e-15) and np.all(out <= hi + 1e-15)
    np.testing.assert_array_equal(scale, np.abs(hi))  # positive image: max|u_B| == max
    out_s = oracle.nlm(img + np.float32(0.5), 2, 3, 0.1, "clamp")
    np.testing.assert_allclose(out_s, out + 0.5, rtol=0, atol=1e-6)


@pytest.mark.parametrize("border,c", [("clamp", 0.0), ("constant", 0.3)])
def test_nlm_equivariant_under_flips_and_transpose(border, c):
    """The patch (2P+1)^2 and the search window (2S+1)^2 are symmetric squares and the boundary
    is per coordinate, so NLM commutes with transposition and with either flip -- a swapped row /
    column index or an asymmetric window in the oracle breaks one of these."""
    img = synth.rect_scene(15, 13, 11, n_rect=5, noise=0.0866)
    out = oracle.nlm(img, 2, 3, 0.15, border, c)
    for f in (lambda a: a.T, lambda a: a[:, ::-1], lambda a: a[::-1, :]):
        got = oracle.nlm(np.ascontiguousarray(f(img)), 2, 3, 0.15, border, c)
        np.testing.assert_allclose(got, f(out), rtol=0, atol=1e-14)


def test_nlm_rejects_bad_h():
    img = np.zeros((3, 3), np.float32)
    for h in (0.0, -1.0, float("nan")):
        with pytest.raises(ValueError):
            oracle.nlm(img, 1, 1, h)


# ============================================================================ conv2d_u8
# Non-separable convolution of an 8-bit image (§6, Table 3).

@pytest.mark.parametrize("r", [1, 2, 3])
def test_conv2d_u8_delta_image(r):
    """A single 255 pixel at (x0, y0), constant 0 border: out(x0-i, y0-j) = 255 f[j+r][i+r]
    (correlation orientation, reading R1), zero elsewhere -- exact."""
    H, W, x0, y0 = 15, 17, 8, 6
    img = np.zeros((H, W), np.uint8)
    img[y0, x0] = 255
    f = synth.filter2d(3, r)
    out = oracle.conv2d_u8(img, f, "constant", 0.0)
    exp = np.zeros((H, W))
    for j in range(-r, r + 1):
        for i in range(-r, r + 1):
            exp[y0 - j, x0 - i] = 255.0 * float(f[j + r, i + r])
    np.testing.assert_array_equal(out, exp)


@pytest.mark.parametrize("border,c", [("clamp", 0.0), ("constant", 77.0)])
def test_conv2d_u8_constant_image(border, c):
    img = np.full((9, 11), 77, np.uint8)
    f = synth.filter2d(4, 2)
    out = oracle.conv2d_u8(img, f, border, c)
    np.testing.assert_allclose(out, 77.0 * f.astype(np.float64).sum(), rtol=1e-14)


@pytest.mark.parametrize("border,c", [("clamp", 0.0), ("constant", 0.0), ("constant", 31.0)])
def test_conv2d_u8_separable_filter_equals_sepconv_oracle(border, c):
    """outer(g, f) filter == the separable oracle on the same (exactly fp32) pixel values."""
    img = synth.uniform_u8(5, 23, 19)
    fx, gy = synth.signed_taps(11, 2), synth.signed_taps(12, 2)
    filt = np.outer(gy.astype(np.float64), fx.astype(np.float64))
    # the product of two fp32 taps is exact in double but not in fp32: compare against the
    # double outer product by building it from fp32 values the conv2d oracle then promotes
    f32 = filt.astype(np.float32)
    out = oracle.conv2d_u8(img, f32, border, c)
    sep = oracle.sepconv(img.astype(np.float32), fx, gy, border, c)
    scale = oracle.conv2d_u8(img, np.abs(f32), border, abs(c))
    np.testing.assert_allclose(out, sep, rtol=0, atol=1e-6 * scale.max())  # f32 rounding of g_j f_i only


@pytest.mark.parametrize("r", [0, 1, 2, 3])
@pytest.mark.parametrize("border,c", [("clamp", 0.0), ("constant", 0.0), ("constant", 200.0)])
def test_conv2d_u8_brute_force_scipy(r, border, c):
    """scipy.ndimage.correlate (mode nearest == clamp, constant == constant c) on a 9x7 image
    and a ragged 13x29 one: every border pixel included (SPEC.md §"Boundary semantics")."""
    for shape in ((9, 7), (13, 29)):
        img = synth.uniform_u8(6 + r, *shape)
        f = synth.filter2d(7 + r, r)
        out = oracle.conv2d_u8(img, f, border, c)
        mode = "nearest" if border == "clamp" else "constant"
        exp = ndi.correlate(img.astype(np.float64), f.astype(np.float64), mode=mode, cval=c)
        np.testing.assert_allclose(out, exp, rtol=1e-13, atol=1e-10)


def test_conv2d_u8_points_and_pitch():
    full = synth.uniform_u8(8, 40, 33)
    img = np.zeros((40, 48), np.uint8)
    img[:, :33] = full
    view = img[:, :33]  # row pitch 48 bytes
    f = synth.filter2d(9, 2)
    out = oracle.conv2d_u8(view, f, "clamp")
    np.testing.assert_array_equal(out, oracle.conv2d_u8(full, f, "clamp"))
    xs = np.array([0, 32, 5, 17, 0], np.int64)
    ys = np.array([0, 39, 20, 3, 39], np.int64)
    np.testing.assert_array_equal(oracle.conv2d_u8(full, f, "clamp", points=(xs, ys)), out[ys, xs])


def test_conv2d_u8_linear_in_the_filter():
    img = synth.uniform_u8(10, 12, 14)
    f1, f2 = synth.filter2d(1, 2), synth.filter2d(2, 2)
    a = oracle.conv2d_u8(img, f1) + oracle.conv2d_u8(img, f2)
    b = oracle.conv2d_u8(img, f1.astype(np.float64) + f2.astype(np.float64))
    np.testing.assert_allclose(a, b, rtol=1e-13, atol=1e-10)


def test_conv2d_u8_rejects_bad_args():
    with pytest.raises(TypeError):
        oracle.conv2d_u8(np.zeros((3, 3), np.float32), synth.filter2d(1, 1))
    with pytest.raises(KeyError):  # unknown border mode
        oracle.conv2d_u8(np.zeros((3, 3), np.uint8), synth.filter2d(1, 1), "wrap")


def test_uniform_u8_is_the_top_byte_of_the_u01_stream():
    """uniform_u8 and uniform_image share one SplitMix64 draw: u8 = floor(256 * u01)."""
    u = synth.uniform_image(13, 7, 9)
    b = synth.uniform_u8(13, 7, 9)
    np.testing.assert_array_equal(b, np.floor(u.astype(np.float64) * 256).astype(np.uint8))
    np.testing.assert_array_equal(synth.uniform_u8(13, 7, 9, row0=3, rows=2), b[3:5])


# ----------------------------------------------------------------------------- 3-D separable convolution
def _vol(seed, d, h, w):
    return np.stack([synth.uniform_image(seed + z, h, w) for z in range(d)]) - np.float32(0.5)


@pytest.mark.parametrize("border,c", BORDERS)
@pytest.mark.parametrize("shape,rx,ry,rz", [((5, 7, 9), 2, 1, 1), ((9, 4, 6), 1, 2, 3), ((1, 6, 11), 1, 1, 2),
                                            ((7, 1, 1), 0, 0, 3), ((4, 5, 3), 3, 3, 2)])
def test_sepconv3d_equals_3d_correlation(border, c, shape, rx, ry, rz):
    """Separable 3-D = scipy.ndimage.correlate with the outer-product kernel h (x) g (x) f."""
    vol = _vol(21, *shape)
    f, g, h = synth.signed_taps(7, rx), synth.signed_taps(8, ry), synth.signed_taps(9, rz)
    out = oracle.sepconv3d(vol, f, g, h, border, c)
    ker = np.einsum("k,j,i->kji", h.astype(np.float64), g.astype(np.float64), f.astype(np.float64))
    ref = ndi.correlate(vol.astype(np.float64), ker, **_mode(border, c))
    np.testing.assert_allclose(out, ref, rtol=0, atol=1e-13)


def test_sepconv3d_delta_orientation():
    """A delta at (x0,y0,z0) lands at out(x0-i, y0-j, z0-k) = f_i g_j h_k: correlation on every axis."""
    vol = np.zeros((7, 8, 9), np.float32)
    vol[3, 4, 5] = 1.0
    f, g, h = synth.signed_taps(1, 1), synth.signed_taps(2, 2), synth.signed_taps(3, 1)
    out = oracle.sepconv3d(vol, f, g, h, "constant", 0.0)
    for k in range(-1, 2):
        for j in range(-2, 3):
            for i in range(-1, 2):
                assert out[3 - k, 4 - j, 5 - i] == float(f[i + 1]) * float(g[j + 2]) * float(h[k + 1])
    assert np.count_nonzero(out) == 3 * 5 * 3


@pytest.mark.parametrize("border,c", BORDERS)
def test_sepconv3d_reduces_to_2d_and_constant(border, c):
    """rz = 0 with h = [1] is the 2-D oracle slice by slice; a constant volume gives c·Σf·Σg·Σh."""
    vol = _vol(31, 3, 6, 7)
    f, g = synth.gaussian_taps(2), synth.signed_taps(4, 1)
    out = oracle.sepconv3d(vol, f, g, [1.0], border, c)
    for z in range(3):
        np.testing.assert_array_equal(out[z], oracle.sepconv(np.ascontiguousarray(vol[z]), f, g, border, c))
    cv = np.full((4, 5, 6), 0.375, np.float32)
    h = synth.signed_taps(6, 2)
    out = oracle.sepconv3d(cv, f, g, h, "clamp")
    exp = 0.375 * f.astype(np.float64).sum() * g.astype(np.float64).sum() * h.astype(np.float64).sum()
    np.testing.assert_allclose(out, exp, rtol=1e-13, atol=1e-15)


def test_sepconv3d_points_and_strides():
    vol = _vol(41, 5, 6, 7)
    padded = np.zeros((5, 8, 12), np.float32)
    padded[:, :6, :7] = vol
    f, g, h = synth.gaussian_taps(1), synth.gaussian_taps(2), synth.gaussian_taps(1)
    full = oracle.sepconv3d(vol, f, g, h, "clamp")
    np.testing.assert_array_equal(oracle.sepconv3d(padded[:, :6, :7], f, g, h, "clamp"), full)
    xs, ys, zs = np.array([0, 6, 3]), np.array([0, 5, 2]), np.array([4, 0, 2])
    np.testing.assert_array_equal(oracle.sepconv3d(vol, f, g, h, "clamp", points=(xs, ys, zs)), full[zs, ys, xs])
