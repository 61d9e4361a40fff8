"""GPU parity of the offset-symmetric NLM kernel `sym_tmem` (R30, nlm_sym.cuh).

The parity suite already runs it on the small shapes; these cases reach what only larger images
exercise: several 118-column strips and 128-row CTA tiles (the strip edges, where partner sources
come from the S halo columns, and the stacked-warp edges inside a CTA), interior tiles staged by the
asynchronous copy next to border tiles staged through the boundary, batches, row bands, unaligned
pitches (no asynchronous copy), an odd patch radius (odd tile origin) and the h limits.  Every pixel
of the images is compared with the double-precision oracle at the NLM tolerance (tests/_tol.py).
"""
import math

import numpy as np
import pytest

import oracle
import synth
from tests._tol import check_nlm

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU, skipped there
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1605_06399_b200 as icl  # noqa: E402

DEV = torch.device("cuda:0")


@pytest.fixture(autouse=True)
def _force_sym():
    icl.force_variant("nlm", "sym_tmem")
    yield
    icl.force_variant("nlm", None)


@pytest.mark.parametrize("variant", ["sym_ring", "sym_tmem8"])
@pytest.mark.parametrize("P,S,h", [(2, 5, 0.1), (1, 3, 0.05)])
def test_sym_variants_multi_tile_vs_oracle(variant, P, S, h):
    """the TMEM-ring and the 8-warp forms on 2 images of 300 x 389 (several strips and CTA rows,
    interior and border tiles), clamp and constant borders, every pixel vs the oracle."""
    icl.force_variant("nlm", variant)
    img = np.stack([synth.rect_scene(900 + 10 * P + S + i, 300, 389, n_rect=20, noise=0.0866) for i in range(2)])
    for border, c in (("clamp", 0.0), ("constant", 0.3)):
        out = _run(img, P, S, h, border, c)
        for i in range(2):
            check_nlm(out[i], img[i], P, S, h, border, c)


def _dev(img, pitch=None):
    b, h, w = img.shape
    pitch = pitch or w
    buf = torch.full((b, h, pitch), float("nan"), dtype=torch.float32, device=DEV)
    buf[:, :, :w] = torch.from_numpy(np.ascontiguousarray(img)).to(DEV)
    return buf[:, :, :w]


def _run(img, P, S, h, border, c, pitch=None, band=None):
    src = _dev(img, pitch)
    dst = torch.full(img.shape, float("nan"), dtype=torch.float32, device=DEV)
    icl.nlm(src, dst, P, S, h, border, c, band=band)
    torch.cuda.synchronize()
    return dst.cpu().numpy()


@pytest.mark.parametrize("border,c", [("clamp", 0.0), ("constant", 0.3)])
@pytest.mark.parametrize("P,S,h", [(2, 5, 0.1), (1, 3, 0.05), (3, 5, 0.2), (2, 7, 0.15), (1, 1, 0.1)])
def test_sym_multi_tile_vs_oracle(P, S, h, border, c):
    """2 images of 300 x 389: 4 strips x 3 CTA rows, interior and border tiles, ragged tails."""
    img = np.stack([synth.rect_scene(700 + 10 * P + S + i, 300, 389, n_rect=20, noise=0.0866) for i in range(2)])
    out = _run(img, P, S, h, border, c)
    for i in range(2):
        check_nlm(out[i], img[i], P, S, h, border, c)


def test_sym_unaligned_pitch_and_limits():
    """pitch of an odd number of floats (no 8-byte asynchronous copy); h -> inf (box mean) and a tiny h."""
    img = synth.rect_scene(811, 260, 301, n_rect=16, noise=0.0866)[None]
    for h in (0.1, math.inf, 1e-6):
        out = _run(img, 2, 5, h, "clamp", 0.0, pitch=301 + 3)
        check_nlm(out[0], img[0], 2, 5, h, "clamp", 0.0)


def test_sym_bands_match_unsharded():
    """row bands through icl_band (global coordinates; rows outside the held buffer never read)."""
    H, W, P, S = 420, 250, 2, 5
    img = synth.rect_scene(812, H, W, n_rect=18, noise=0.0866)[None]
    ref = _run(img, P, S, 0.1, "constant", 0.5)
    up, down = icl.nlm_halo(P, S)
    cuts = [0, 5, 131, 300, 419, 420]
    for a, b in zip(cuts[:-1], cuts[1:]):
        s0, s1 = max(0, a - up), min(H, b + down)
        src = _dev(img[:, s0:s1])
        dst = torch.full((1, b - a, W), float("nan"), dtype=torch.float32, device=DEV)
        icl.nlm(src, dst, P, S, 0.1, "constant", 0.5, band=(H, s0, a))
        torch.cuda.synchronize()
        np.testing.assert_allclose(dst.cpu().numpy(), ref[:, a:b], rtol=0, atol=2e-5, err_msg=f"band {a}:{b}")


def test_sym_agrees_with_boxsum_x2_large():
    """one 1024 x 1536 image: every pixel of sym_tmem within the NLM tolerance of the oracle on a
    sample, and within 2e-5 of the two-phase boxsum_x2 kernel everywhere (independent formulation)."""
    img = synth.rect_scene(813, 1024, 1536, n_rect=80, noise=0.0866)[None]
    out = _run(img, 2, 5, 0.1, "clamp", 0.0)
    icl.force_variant("nlm", "boxsum_x2")
    ref = _run(img, 2, 5, 0.1, "clamp", 0.0)
    np.testing.assert_allclose(out, ref, rtol=0, atol=2e-5)
    rng = np.random.default_rng(5)
    ys = np.concatenate([rng.integers(0, 1024, 1500), np.repeat([0, 127, 128, 255, 1023], 40)])
    xs = np.concatenate([rng.integers(0, 1536, 1500), np.tile(np.arange(0, 1536, 39)[:40], 5)])
    check_nlm(out[0][ys, xs], img[0], 2, 5, 0.1, "clamp", 0.0, points=(xs, ys))


@pytest.mark.parametrize("variant", ["sym_tmem", "sym_ring"])
def test_sym_equivariant_under_flips_and_transpose(variant):
    """NLM commutes with transposition and flips (symmetric patch and window, per-coordinate
    boundary): the symmetric kernels' partner bookkeeping is direction-specific (the half set
    {oy > 0} u {oy = 0, ox > 0}), so a flipped or transposed image sends every pair through the
    other half -- the outputs must still agree with the flipped output to the NLM tolerance."""
    icl.force_variant("nlm", variant)
    img = synth.rect_scene(977, 260, 300, n_rect=16, noise=0.0866)
    out = _run(img[None], 2, 5, 0.1, "clamp", 0.0)[0]
    _, scale = oracle.nlm(img, 2, 5, 0.1, "clamp", 0.0, with_scale=True)
    for f in (lambda a: a.T, lambda a: a[:, ::-1], lambda a: a[::-1, :]):
        got = _run(np.ascontiguousarray(f(img))[None], 2, 5, 0.1, "clamp", 0.0)[0]
        np.testing.assert_array_less(np.abs(got - f(out)), 2e-4 * f(scale) + 1e-30)
