"""Parity at BASELINE.json's full sizes, in the launch configurations bench.py
times (default dispatch, no forced variant), on sampled outputs the oracle
computes one by one: the whole-image border frame (every pixel of the first /
last rows and columns within the stencil reach) plus random interior pixels.

  * configs[3]: 16384^2 fp32 separable Gaussian, radius 1, 2, 8, 15 (constant 0)
  * configs[4] per GPU: a batch of 8 x 4096^2 images through sepconv r=2
    (constant), Harris B=5 (clamp, mask) and NLM 5x5/11x11 h=0.1 (clamp) --
    exactly bench.py's suite step.
"""
import functools

import numpy as np
import pytest

import synth
from tests._tol import check_harris, check_nlm, check_sepconv

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1605_06399_b200 as icl  # noqa: E402

DEV = torch.device("cuda:0")


def sample_points(H, W, reach, n_random, seed):
    rng = np.random.default_rng(seed)
    ys, xs = [rng.integers(0, H, n_random)], [rng.integers(0, W, n_random)]
    k = max(reach, 1) + 1
    for r in list(range(k)) + list(range(H - k, H)):  # border rows: 64 samples each
        xs.append(np.linspace(0, W - 1, 64).astype(np.int64))
        ys.append(np.full(64, r))
    for c in list(range(k)) + list(range(W - k, W)):  # border columns
        ys.append(np.linspace(0, H - 1, 64).astype(np.int64))
        xs.append(np.full(64, c))
    return np.concatenate(xs), np.concatenate(ys)


@functools.lru_cache(maxsize=1)
def _img16k():
    return synth.uniform_image(4, 16384, 16384)  # BASELINE configs[3] input recipe (seed 4)


@pytest.mark.parametrize("r", [1, 2, 8, 15])
def test_sepconv_16k_sampled(r):
    S = 16384
    img = _img16k()
    src = torch.from_numpy(img).to(DEV)
    dst = torch.empty_like(src)
    fx = synth.gaussian_taps(r)
    icl.sepconv(src, dst, fx, fx, "constant")
    torch.cuda.synchronize()
    xs, ys = sample_points(S, S, r, 4000, r)
    got = dst[torch.from_numpy(ys).to(DEV), torch.from_numpy(xs).to(DEV)].cpu().numpy()
    check_sepconv(got, img, fx, fx, "constant", 0.0, points=(xs, ys))
    # equals the fill_uniform device generator used by bench.py's 16k workload
    gen = torch.empty(8, S, device=DEV)
    icl.fill_uniform(gen, 4, row0=S // 2)
    np.testing.assert_array_equal(gen.cpu().numpy(), img[S // 2:S // 2 + 8])
    del src, dst
    torch.cuda.empty_cache()


def test_suite_batch_sampled():
    """bench.py suite step on a batch of 8 x 4096^2 images (configs[4] per GPU)."""
    import bench
    B, S = 8, 4096
    u_h, hs_h, ns_h = bench.gen_inputs(0, B, S)
    u, hs, ns = (torch.from_numpy(a).to(DEV) for a in (u_h, hs_h, ns_h))
    o_sep, o_har, o_nlm = torch.empty_like(u), torch.empty_like(u), torch.empty_like(u)
    o_mask = torch.empty(B, S, S, dtype=torch.uint8, device=DEV)
    c = bench.SUITE
    fx = synth.gaussian_taps(c["sep_r"])
    thr = 1.0
    icl.sepconv(u, o_sep, fx, fx, c["sep_border"])
    icl.harris(hs, o_har, c["har_block"], c["har_k"], c["har_border"], mask=o_mask, threshold=thr)
    icl.nlm(ns, o_nlm, c["nlm_P"], c["nlm_S"], c["nlm_h"], c["nlm_border"])
    torch.cuda.synchronize()
    for i in (0, B - 1):
        xs, ys = sample_points(S, S, 7, 1500, 10 + i)
        ix, iy = torch.from_numpy(xs).to(DEV), torch.from_numpy(ys).to(DEV)
        check_sepconv(o_sep[i][iy, ix].cpu().numpy(), u_h[i], fx, fx, c["sep_border"], 0.0, points=(xs, ys))
        check_harris(o_har[i][iy, ix].cpu().numpy(), o_mask[i][iy, ix].cpu().numpy(), hs_h[i], c["har_block"],
                     c["har_k"], c["har_border"], 0.0, thr, points=(xs, ys))
        sel = slice(0, 2500)  # NLM oracle is ~10x costlier per pixel
        check_nlm(o_nlm[i][iy[sel], ix[sel]].cpu().numpy(), ns_h[i], c["nlm_P"], c["nlm_S"], c["nlm_h"],
                  c["nlm_border"], 0.0, points=(xs[sel], ys[sel]))


def test_batches_beyond_2gib_use_64bit_offsets():
    """offsets are int64 (a 64 x 4096^2 batch is 4 GiB).  A 40 x 4096^2 fp32 batch
    (2.5 GiB) through sepconv / Harris+mask / NLM and a 140 x 4096^2 uint8 batch (2.2 GiB) through
    conv2d: sampled pixels of the LAST image (byte offsets > 2^31) against the oracle."""
    B, S = 40, 4096
    big = torch.empty(B, S, S, device=DEV)
    icl.fill_uniform(big, 90)
    last = big[B - 1].cpu().numpy()  # fill_uniform == synth.uniform_image(90 + b) (test_fill_uniform_matches_synth)
    rng = np.random.default_rng(5)
    xs = np.concatenate([rng.integers(0, S, 3000), [0, S - 1, 0, S - 1]])
    ys = np.concatenate([rng.integers(0, S, 3000), [0, 0, S - 1, S - 1]])
    ix, iy = torch.from_numpy(xs).to(DEV), torch.from_numpy(ys).to(DEV)
    out = torch.empty_like(big)
    fx = synth.gaussian_taps(2)
    icl.sepconv(big, out, fx, fx, "constant")
    check_sepconv(out[B - 1][iy, ix].cpu().numpy(), last, fx, fx, "constant", 0.0, points=(xs, ys))
    mask = torch.empty(B, S, S, dtype=torch.uint8, device=DEV)
    icl.harris(big, out, 5, 0.04, "clamp", mask=mask, threshold=1.0)
    check_harris(out[B - 1][iy, ix].cpu().numpy(), mask[B - 1][iy, ix].cpu().numpy(), last, 5, 0.04, "clamp", 0.0,
                 1.0, points=(xs, ys))
    icl.nlm(big, out, 2, 5, 0.1, "clamp")
    sel = slice(0, 1000)
    check_nlm(out[B - 1][iy[sel], ix[sel]].cpu().numpy(), last, 2, 5, 0.1, "clamp", 0.0, points=(xs[sel], ys[sel]))
    del big, out, mask
    torch.cuda.empty_cache()
    Bu = 140
    u8 = torch.zeros(Bu, S, S, dtype=torch.uint8, device=DEV)
    img = synth.uniform_u8(91, S, S)
    u8[Bu - 1] = torch.from_numpy(img).to(DEV)
    o8 = torch.empty(Bu, S, S, device=DEV)
    f = synth.filter2d(91, 2)
    icl.conv2d_u8(u8, o8, f, "clamp")
    from tests._tol import check_conv2d
    check_conv2d(o8[Bu - 1][iy, ix].cpu().numpy(), img, f, "clamp", 0.0, points=(xs, ys))
    del u8, o8
    torch.cuda.empty_cache()
