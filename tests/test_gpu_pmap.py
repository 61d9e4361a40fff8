"""The paper's Table-1 tuning space as kernel axes (pmap.cu; §5.2.1-5.2.5, Fig. 4;
SURVEY.md §8(f) row 2): every pm_* configuration -- CTA shape, thread coarsening, blocked /
interleaved / interleaved-in-work-group mapping, local memory, unroll factor -- evaluates the
naive per-output order, so all 288 per filter must equal naive_direct bit for bit (and hence
the oracle), cover every pixel exactly (NaN-canary destination, ragged sizes, row bands), and
the model-guided tuner (icl_tune_ann) must land within 5% of the exhaustive
optimum while timing fewer than half the variants."""
import numpy as np
import pytest

import synth
from tests._tol import check_harris, check_sepconv

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1605_06399_b200 as icl  # noqa: E402

DEV = torch.device("cuda:0")


def pm(f):
    return [(i, n) for i, n in enumerate(icl.variant_names(f)) if n.startswith("pm_")]


def nan_like(h, w, pitch=None, dtype=torch.float32):
    pitch = pitch or w
    t = torch.full((h, pitch), float("nan") if dtype == torch.float32 else 7, dtype=dtype, device=DEV)
    return t[:, :w]


def test_space_size_and_axes():
    for f in ("sepconv", "harris"):
        names = [n for _, n in pm(f)]
        assert len(names) == 288
        for key in ("_blk_l0", "_int_l0", "_blk_l1", "_iwg_l1", "_u1", "_u4", "_w128x1", "_w16x8", "_c4x1", "_c1x4"):
            assert any(key in n for n in names), key


@pytest.mark.parametrize("r,border,c", [(1, "constant", 0.7), (3, "clamp", 0.0), (0, "constant", 0.0)])
@pytest.mark.parametrize("shape", [(37, 129), (70, 301), (1, 5)])
def test_sepconv_pmap_all_bit_identical(shape, r, border, c):
    h, w = shape
    img = synth.uniform_image(80 + r, h, w)
    fx, gy = synth.gaussian_taps(r), synth.signed_taps(5, max(r - 1, 0))
    src = torch.from_numpy(img).to(DEV)
    icl.force_variant("sepconv", "naive_direct")
    ref = nan_like(h, w)
    icl.sepconv(src, ref, fx, gy, border, c)
    refh = ref.cpu().numpy()
    check_sepconv(refh, img, fx, gy, border, c)
    for vid, name in pm("sepconv"):
        icl.force_variant("sepconv", vid)
        out = nan_like(h, w, pitch=w + 3)
        icl.sepconv(src, out, fx, gy, border, c)
        np.testing.assert_array_equal(out.cpu().numpy(), refh, err_msg=name)
    icl.force_variant("sepconv", None)


@pytest.mark.parametrize("block,border,c", [(5, "clamp", 0.0), (2, "constant", 0.3), (3, "clamp", 0.0)])
@pytest.mark.parametrize("shape", [(29, 67), (53, 130)])
def test_harris_pmap_all_bit_identical(shape, block, border, c):
    h, w = shape
    img = synth.rect_scene(90 + block, h, w, n_rect=8, noise=0.01)
    src = torch.from_numpy(img).to(DEV)
    thr = 0.05
    icl.force_variant("harris", "naive_direct")
    ref, rm = nan_like(h, w), nan_like(h, w, dtype=torch.uint8)
    icl.harris(src, ref, block, 0.04, border, c, mask=rm, threshold=thr)
    refh, rmh = ref.cpu().numpy(), rm.cpu().numpy()
    check_harris(refh, rmh, img, block, 0.04, border, c, thr)
    for vid, name in pm("harris"):
        icl.force_variant("harris", vid)
        out, om = nan_like(h, w, pitch=w + 5), nan_like(h, w, dtype=torch.uint8)
        icl.harris(src, out, block, 0.04, border, c, mask=om, threshold=thr)
        np.testing.assert_array_equal(out.cpu().numpy(), refh, err_msg=name)
        np.testing.assert_array_equal(om.cpu().numpy(), rmh, err_msg=name)
    icl.force_variant("harris", None)


def test_pmap_bands_and_batches():
    """Row bands (global-row boundary; the local-memory tiles stop at the band's stencil rows) and
    image batches, a sample of the space against the unsharded naive call."""
    H, W, r, B = 97, 150, 4, 2
    img = np.stack([synth.uniform_image(95 + i, H, W) for i in range(B)])
    fx = synth.gaussian_taps(r)
    src = torch.from_numpy(img).to(DEV)
    icl.force_variant("sepconv", "naive_direct")
    ref = torch.empty(B, H, W, device=DEV)
    icl.sepconv(src, ref, fx, fx, "clamp")
    refh = ref.cpu().numpy()
    for vid, name in pm("sepconv")[::7]:
        icl.force_variant("sepconv", vid)
        for a, b in ((0, 30), (30, 31), (31, 97)):
            s0, s1 = max(0, a - r), min(H, b + r)
            out = torch.full((B, b - a, W), float("nan"), device=DEV)
            icl.sepconv(src[:, s0:s1].contiguous(), out, fx, fx, "clamp", band=(H, s0, a))
            np.testing.assert_array_equal(out.cpu().numpy(), refh[:, a:b], err_msg=f"{name} {a}:{b}")
    icl.force_variant("sepconv", None)


def test_model_guided_tuner_finds_the_optimum_of_the_paper_space():
    """random configurations timed, an ANN performance model fitted, the
    best-predicted ones timed, the best measured returned.  On the 309-variant sepconv space
    (hand-built kernels + the 288 Table-1 configurations) it must land within 5% of the
    exhaustive optimum while timing fewer than half the variants."""
    img = synth.uniform_image(7, 4096, 4096)  # ~0.14 ms per call: timing noise well below 5%
    src = torch.from_numpy(img).to(DEV)
    dst = torch.empty_like(src)
    f = synth.gaussian_taps(2)
    icl.tune_cache_clear()
    ex = icl.tune("sepconv", src, dst, taps_x=f, taps_y=f, border="constant", force=True)
    n = len(icl.variant_names("sepconv"))
    icl.tune_cache_clear()
    an = icl.tune("sepconv", src, dst, taps_x=f, taps_y=f, border="constant", ann=(60, 60, 3))
    icl.tune_cache_clear()
    assert an["n_candidates"] < n / 2, (an["n_candidates"], n)
    # re-time both winners side by side (the two tuner runs are seconds apart)
    st = torch.cuda.current_stream()

    def med(vid):
        icl.force_variant("sepconv", vid)
        ts = []
        for _ in range(3):
            icl.sepconv(src, dst, f, f, "constant")
        for _ in range(31):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            icl.sepconv(src, dst, f, f, "constant")
            e1.record(st)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        icl.force_variant("sepconv", None)
        return sorted(ts)[len(ts) // 2]

    t_ex, t_an = med(ex["variant_id"]), med(an["variant_id"])
    assert t_an <= 1.05 * t_ex, (ex["name"], t_ex, an["name"], t_an)
