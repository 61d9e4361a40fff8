"""Tolerance definitions of BASELINE.json north_star, made well-defined near
cancellation as SURVEY.md §8(c) / DESIGN.md "Tolerances" state.  Test-only."""
import numpy as np

import oracle

SEP_TOL = 1e-5      # north_star: max relative error 1e-5 for convolution
HARRIS_TOL = 1e-4   # north_star: 1e-4 for the Harris response
NLM_TOL = 1e-4      # north_star: 1e-4 for NLM


def sep_scale(img, fx, gy, border, c, points=None):
    """(|g| * |f| * |x|)(p): the magnitude the fp32 sum is computed over."""
    a = np.abs(img)
    return oracle.sepconv(a, np.abs(fx), np.abs(gy), border, abs(c), points=points)


def check_sepconv(got, img, fx, gy, border, c, points=None, tol=SEP_TOL):
    ref = oracle.sepconv(img, fx, gy, border, c, points=points)
    scale = sep_scale(img, fx, gy, border, c, points=points)
    got = np.asarray(got, dtype=np.float64)
    err = np.abs(got - ref)
    bad = np.where(scale > 0, err > tol * scale, err != 0)
    assert not bad.any(), f"sepconv: {bad.sum()} pixels out of tolerance; max rel {np.max(err / np.maximum(scale, 1e-300))}"
    return float(np.max(err / np.maximum(scale, 1e-300))) if err.size else 0.0


def check_harris(R, mask, img, block, k, border, c, threshold, points=None, tol=HARRIS_TOL):
    Rr, S = oracle.harris(img, block, k, border, c, points=points, with_tensor=True)
    D = oracle.harris_scale(S, k)
    R = np.asarray(R, dtype=np.float64)
    err = np.abs(R - Rr)
    bad = np.where(D > 0, err > tol * D, err != 0)
    assert not bad.any(), f"harris: {bad.sum()} pixels out of tolerance; max rel {np.max(err / np.maximum(D, 1e-300))}"
    if mask is not None:
        mref = Rr > threshold
        near = np.abs(Rr - threshold) <= tol * D
        diff = (np.asarray(mask) != 0) != mref
        assert not (diff & ~near).any(), f"harris mask: {(diff & ~near).sum()} pixels differ away from the threshold"
    return float(np.max(err / np.maximum(D, 1e-300))) if err.size else 0.0


def check_nlm(got, img, P, S, h, border, c, points=None, tol=NLM_TOL):
    ref, scale = oracle.nlm(img, P, S, h, border, c, points=points, with_scale=True)
    got = np.asarray(got, dtype=np.float64)
    err = np.abs(got - ref)
    bad = np.where(scale > 0, err > tol * scale, err != 0)
    assert not bad.any(), f"nlm: {bad.sum()} pixels out of tolerance; max rel {np.max(err / np.maximum(scale, 1e-300))}"
    return float(np.max(err / np.maximum(scale, 1e-300))) if err.size else 0.0


def check_conv2d(got, img, filt, border, c, points=None, tol=SEP_TOL):
    """Non-separable uchar convolution (R22): |y - y^| <= 1e-5 (|f| * |x|)(p), exact 0 where the
    scale is 0 -- the sepconv bar (north_star's 1e-5 for convolution)."""
    ref = oracle.conv2d_u8(img, filt, border, c, points=points)
    scale = oracle.conv2d_u8(img, np.abs(np.asarray(filt, np.float32)), border, abs(c), points=points)
    got = np.asarray(got, dtype=np.float64)
    err = np.abs(got - ref)
    bad = np.where(scale > 0, err > tol * scale, err != 0)
    assert not bad.any(), f"conv2d: {bad.sum()} pixels out of tolerance; max rel {np.max(err / np.maximum(scale, 1e-300))}"
    return float(np.max(err / np.maximum(scale, 1e-300))) if err.size else 0.0


def check_harris_families(outs, img, block, k, border, c, thr, points=None):
    """The naive-order variants are bit-identical to naive_direct; each re-associated family
    (slide_*: vertical sums of the products first; slide2_*: horizontal pair sums first --
    SURVEY.md §8(c) R16, R27) is bit-identical within itself and matches the oracle
    within the Harris tolerance."""
    R0, M0 = outs["naive_direct"]
    fams = {}
    for name, v in outs.items():
        fam = name.split("_")[0] if name.startswith("slide") else None
        if fam is None:
            np.testing.assert_array_equal(v[0], R0, err_msg=name)
            np.testing.assert_array_equal(v[1], M0, err_msg=name)
        else:
            fams.setdefault(fam, {})[name] = v
    for fam in fams.values():
        Rs, Ms = next(iter(fam.values()))
        check_harris(Rs, Ms, img, block, k, border, c, thr, points=points)
        for name, (R, M) in fam.items():
            np.testing.assert_array_equal(R, Rs, err_msg=name)
            np.testing.assert_array_equal(M, Ms, err_msg=name)


def sampled_variants(names):
    """(id, name) of every hand-built variant plus a fixed sample of the paper's Table-1 space
    (pm_* configurations, 288 per filter; tests/test_gpu_pmap.py runs all of them): every 11th,
    which visits every CTA shape, coarsening, mapping / local-memory pair and unroll factor."""
    out = []
    k = 0
    for vid, n in enumerate(names):
        if n.startswith("pm_"):
            if k % 11 == 0:
                out.append((vid, n))
            k += 1
        else:
            out.append((vid, n))
    return out

