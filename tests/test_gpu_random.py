"""Randomised parity sweep (seeded, reproducible): many small odd shapes
(1..70 x 1..300, including 1-row / 1-column images), random radii / windows /
patch+search sizes, random border modes and constants, padded and unpadded
pitches -- every eligible variant against the oracle, and the variants of
sepconv / Harris / conv2d against each other bit for bit."""
import os

import numpy as np
import pytest

import synth
from tests._tol import check_conv2d, check_harris, check_harris_families, check_nlm, check_sepconv, sampled_variants

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1605_06399_b200 as icl  # noqa: E402

DEV = torch.device("cuda:0")
CASES = int(os.environ.get("ICL_RANDOM_CASES", "64"))  # (more seeds: ICL_RANDOM_CASES=512)


def dev_img(a, pad):
    h, w = a.shape
    p = w + pad
    buf = torch.zeros((h, p), dtype=torch.from_numpy(a).dtype, device=DEV)
    buf[:, :w] = torch.from_numpy(a).to(DEV)
    return buf[:, :w]


def each_variant(f, call):
    outs = {}
    for vid, name in sampled_variants(icl.variant_names(f)):
        icl.force_variant(f, vid)
        try:
            outs[name] = call()
        except icl.IclError as e:
            if e.status not in (3, 4):
                raise
    icl.force_variant(f, None)
    return outs


def case(seed):
    rng = np.random.default_rng(1000 + seed)
    h, w = int(rng.integers(1, 71)), int(rng.integers(1, 301))
    border = "clamp" if rng.random() < 0.5 else "constant"
    c = 0.0 if border == "clamp" or rng.random() < 0.4 else float(np.float32(rng.uniform(-1, 2)))
    pad = int(rng.choice([0, 4, 12]))
    return rng, h, w, border, c, pad


@pytest.mark.parametrize("seed", range(CASES))
def test_random_sepconv(seed):
    rng, h, w, border, c, pad = case(seed)
    rx, ry = int(rng.integers(0, 16)), int(rng.integers(0, 16))
    img = synth.uniform_image(seed, h, w)
    fx, gy = synth.signed_taps(seed, rx), synth.gaussian_taps(ry)
    src = dev_img(img, pad)
    ws = torch.empty(icl.sepconv_workspace_bytes(w, h, 1, ry) // 4 + 1, device=DEV)

    def call():
        d = dev_img(np.zeros((h, w), np.float32), pad)
        icl.sepconv(src, d, fx, gy, border, c, workspace=ws)
        return d.cpu().numpy()
    outs = each_variant("sepconv", call)
    check_sepconv(outs["naive_direct"], img, fx, gy, border, c)
    for n, o in outs.items():
        np.testing.assert_array_equal(o, outs["naive_direct"], err_msg=n)


@pytest.mark.parametrize("seed", range(CASES))
def test_random_harris(seed):
    rng, h, w, border, c, pad = case(seed)
    block = int(rng.integers(1, 8))
    img = synth.rect_scene(seed, h, w, n_rect=6, noise=0.01)
    src = dev_img(img, pad)
    thr = 0.05

    def call():
        d = dev_img(np.zeros((h, w), np.float32), pad)
        m = dev_img(np.zeros((h, w), np.uint8), pad)
        icl.harris(src, d, block, 0.04, border, c, mask=m, threshold=thr)
        return d.cpu().numpy(), m.cpu().numpy()
    outs = each_variant("harris", call)
    R, M = outs["naive_direct"]
    check_harris(R, M, img, block, 0.04, border, c, thr)
    check_harris_families(outs, img, block, 0.04, border, c, thr)


@pytest.mark.parametrize("seed", range(CASES // 2))
def test_random_nlm(seed):
    rng, h, w, border, c, pad = case(seed)
    h, w = min(h, 40), min(w, 90)
    P, S = int(rng.integers(0, 4)), int(rng.integers(0, 8))
    hh = float(rng.choice([0.05, 0.1, 0.3]))
    img = synth.rect_scene(seed, h, w, n_rect=5, noise=0.0866)
    src = dev_img(img, pad)

    def call():
        d = dev_img(np.zeros((h, w), np.float32), pad)
        icl.nlm(src, d, P, S, hh, border, c)
        return d.cpu().numpy()
    for n, o in each_variant("nlm", call).items():
        check_nlm(o, img, P, S, hh, border, c)


@pytest.mark.parametrize("seed", range(CASES))
def test_random_conv2d(seed):
    rng, h, w, border, c, pad = case(seed)
    r = int(rng.integers(0, 4))
    img = synth.uniform_u8(seed, h, w)
    f = synth.filter2d(seed, r)
    c8 = float(np.float32(abs(c) * 100))
    src = dev_img(img, pad)

    def call():
        d = dev_img(np.zeros((h, w), np.float32), pad)
        icl.conv2d_u8(src, d, f, border, c8)
        return d.cpu().numpy()
    outs = each_variant("conv2d", call)
    check_conv2d(outs["naive_direct"], img, f, border, c8)
    for n, o in outs.items():
        np.testing.assert_array_equal(o, outs["naive_direct"], err_msg=n)


def test_tall_images_beyond_65535_rows():
    """gridDim.y is capped at 65535: every filter's default dispatch (and conv2d's row-per-CTA
    naive kernel, the only path for unaligned byte images) must still cover 70001-row images."""
    H, W = 70001, 40
    img = synth.uniform_image(7, H, W)
    u8 = synth.uniform_u8(7, H, W)
    src, src8 = torch.from_numpy(img).to(DEV), torch.from_numpy(u8).to(DEV)
    out = torch.empty(H, W, device=DEV)
    mask = torch.empty(H, W, dtype=torch.uint8, device=DEV)
    rng = np.random.default_rng(7)
    ys = np.concatenate([rng.integers(0, H, 1500), [0, H - 1, 65535, 65536]])
    xs = np.concatenate([rng.integers(0, W, 1500), [0, W - 1, 3, 5]])
    ix, iy = torch.from_numpy(xs).to(DEV), torch.from_numpy(ys).to(DEV)
    fx = synth.gaussian_taps(2)
    icl.sepconv(src, out, fx, fx, "clamp")
    check_sepconv(out[iy, ix].cpu().numpy(), img, fx, fx, "clamp", 0.0, points=(xs, ys))
    icl.harris(src, out, 5, 0.04, "clamp", mask=mask, threshold=0.1)
    check_harris(out[iy, ix].cpu().numpy(), mask[iy, ix].cpu().numpy(), img, 5, 0.04, "clamp", 0.0, 0.1,
                 points=(xs, ys))
    icl.nlm(src, out, 2, 5, 0.1, "clamp")
    check_nlm(out[iy, ix].cpu().numpy(), img, 2, 5, 0.1, "clamp", 0.0, points=(xs, ys))
    f = synth.filter2d(7, 2)
    icl.conv2d_u8(src8, out, f, "clamp")  # W = 40 bytes: not 16-byte aligned -> naive_direct
    assert icl.variant_names("conv2d")[icl.last_variant("conv2d")] == "naive_direct"
    check_conv2d(out[iy, ix].cpu().numpy(), u8, f, "clamp", 0.0, points=(xs, ys))


def test_batches_beyond_65535_images():
    """gridDim.z is capped at 65535: a batch of 70000 small images runs as chunks; first, middle
    and last images against the oracle, every variant of every filter equal to the default."""
    B, h, w = 70000, 6, 9
    imgs = np.stack([synth.uniform_image(i % 17, h, w) for i in range(B)])
    u8 = np.stack([synth.uniform_u8(i % 13, h, w) for i in range(B)])
    src, src8 = torch.from_numpy(imgs).to(DEV), torch.from_numpy(u8).to(DEV)
    fx, f2 = synth.gaussian_taps(1), synth.filter2d(3, 1)
    picks = (0, 65534, 65535, B - 1)
    calls = {
        "sepconv": (lambda o: icl.sepconv(src, o, fx, fx, "clamp"),
                    lambda o, i: check_sepconv(o, imgs[i], fx, fx, "clamp", 0.0)),
        "harris": (lambda o: icl.harris(src, o, 3, 0.04, "clamp"),
                   lambda o, i: check_harris(o, None, imgs[i], 3, 0.04, "clamp", 0.0, 0.0)),
        "nlm": (lambda o: icl.nlm(src, o, 1, 2, 0.1, "clamp"),
                lambda o, i: check_nlm(o, imgs[i], 1, 2, 0.1, "clamp", 0.0)),
        "conv2d": (lambda o: icl.conv2d_u8(src8, o, f2, "clamp"),
                   lambda o, i: check_conv2d(o, u8[i], f2, "clamp", 0.0)),
    }
    for f, (run, check) in calls.items():
        ref = torch.empty(B, h, w, device=DEV)
        run(ref)
        refh = ref.cpu().numpy()
        for i in picks:
            check(refh[i], i)
        for vid, name in sampled_variants(icl.variant_names(f)):
            icl.force_variant(f, vid)
            out = torch.full((B, h, w), float("nan"), device=DEV)
            try:
                run(out)
            except icl.IclError as e:
                if e.status in (3, 4):
                    continue
                raise
            got = out.cpu().numpy()
            if f == "nlm":
                np.testing.assert_allclose(got, refh, rtol=0, atol=2e-5, err_msg=name)
            elif f == "harris":  # two fp32 orders (naive / slide<>): each variant against the oracle
                for i in picks:
                    check(got[i], i)
            else:
                np.testing.assert_array_equal(got, refh, err_msg=f"{f} {name}")
        icl.force_variant(f, None)


def test_tuner_on_tall_images():
    """The tuner's device-side equivalence check also covers > 65535 rows."""
    H, W = 66000, 64
    img = torch.from_numpy(synth.uniform_image(8, H, W)).to(DEV)
    out = torch.empty_like(img)
    info = icl.tune("sepconv", img, out, taps_x=synth.gaussian_taps(1), taps_y=synth.gaussian_taps(1),
                    border="clamp", force=True)
    assert info["n_rejected"] == 0 and info["n_candidates"] >= 3


def test_images_beyond_a_million_rows():
    """Row-segment kernels put H/S on gridDim.y: a 1.2M-row image runs as row chunks (icl_band
    semantics): the oracle at sampled rows, including both sides of a chunk boundary."""
    H, W = 1_200_000, 8
    img = synth.uniform_image(9, H, W)
    src = torch.from_numpy(img).to(DEV)
    out = torch.empty_like(src)
    mask = torch.empty(H, W, dtype=torch.uint8, device=DEV)
    rng = np.random.default_rng(9)
    ys = np.concatenate([rng.integers(0, H, 2000), np.arange((1 << 19) - 4, (1 << 19) + 4), [0, H - 1]])
    xs = rng.integers(0, W, ys.size)
    ix, iy = torch.from_numpy(xs).to(DEV), torch.from_numpy(ys).to(DEV)
    fx = synth.gaussian_taps(3)
    icl.sepconv(src, out, fx, fx, "constant")
    check_sepconv(out[iy, ix].cpu().numpy(), img, fx, fx, "constant", 0.0, points=(xs, ys))
    icl.harris(src, out, 5, 0.04, "clamp", mask=mask, threshold=0.1)
    check_harris(out[iy, ix].cpu().numpy(), mask[iy, ix].cpu().numpy(), img, 5, 0.04, "clamp", 0.0, 0.1,
                 points=(xs, ys))
    icl.nlm(src, out, 2, 3, 0.1, "clamp")
    check_nlm(out[iy, ix].cpu().numpy(), img, 2, 3, 0.1, "clamp", 0.0, points=(xs, ys))
