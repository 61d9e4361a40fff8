"""icl_sepconv3d (3-D volumes; "2D/3D indexing", SURVEY.md §8(f)
row 4, R26) against the CPU oracle (tolerance of tests/_tol.py's
sepconv bar, carried to 3-D: |y - y^| <= 1e-5 (|h| x |g| x |f| x |x|)(p)) and
variant against variant (bit-identical: one fp32 chain order)."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1605_06399_b200 as icl  # noqa: E402

DEV = torch.device("cuda:0")
TOL = 1e-5


def vol(seed, d, h, w):
    return np.stack([synth.uniform_image(seed + z, h, w) for z in range(d)])


def dev(v, pitch=None):
    d, h, w = v.shape
    pitch = pitch or w
    buf = torch.full((d, h, pitch), float("nan"), device=DEV)
    buf[..., :w] = torch.from_numpy(v).to(DEV)
    return buf[..., :w]


def check(got, v, f, g, h, border, c, points=None):
    ref = oracle.sepconv3d(v, f, g, h, border, c, points=points)
    scale = oracle.sepconv3d(np.abs(v), np.abs(f), np.abs(g), np.abs(h), border, abs(c), points=points)
    err = np.abs(np.asarray(got, np.float64) - ref)
    bad = np.where(scale > 0, err > TOL * scale, err != 0)
    assert not bad.any(), f"{bad.sum()} voxels out of tolerance"


@pytest.mark.parametrize("shape", [(1, 1, 1), (3, 5, 7), (20, 33, 70), (40, 17, 129), (7, 70, 3)])
@pytest.mark.parametrize("radii", [(0, 0, 0), (1, 1, 1), (2, 1, 3), (3, 3, 3), (7, 2, 5)])
@pytest.mark.parametrize("border,c", [("constant", 0.0), ("constant", 0.7), ("clamp", 0.0)])
def test_sepconv3d_vs_oracle_and_variants(shape, radii, border, c):
    v = vol(3, *shape)
    rx, ry, rz = radii
    f, g, h = synth.gaussian_taps(rx), synth.signed_taps(2, ry), synth.gaussian_taps(rz)
    src = dev(v, pitch=shape[2] + 5)
    outs = []
    for name in icl.variant_names("sepconv3d"):
        icl.force_variant("sepconv3d", name)
        out = torch.full_like(src, float("nan"))
        icl.sepconv3d(src, out, f, g, h, border, c)
        torch.cuda.synchronize()
        outs.append(out)
    icl.force_variant("sepconv3d", None)
    check(outs[-1].cpu().numpy(), v, f, g, h, border, c)
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


def test_sepconv3d_padding_and_slice_stride():
    """Pitched rows and a padded slice stride on both sides; canaries in the padding survive."""
    d, h, w = 9, 21, 45
    v = vol(60, d, h, w)
    sb = torch.full((d, h + 3, w + 9), float("nan"), device=DEV)
    sb[:, :h, :w] = torch.from_numpy(v).to(DEV)
    db = torch.full((d, h + 2, w + 5), float("nan"), device=DEV)
    f, g, hz = synth.gaussian_taps(2), synth.gaussian_taps(1), synth.gaussian_taps(3)
    for name in icl.variant_names("sepconv3d"):
        icl.force_variant("sepconv3d", name)
        db.fill_(float("nan"))
        icl.sepconv3d(sb[:, :h, :w], db[:, :h, :w], f, g, hz, "clamp")
        torch.cuda.synchronize()
        assert torch.isnan(db[:, :, w:]).all() and torch.isnan(db[:, h:, :]).all()
        check(db[:, :h, :w].cpu().numpy(), v, f, g, hz, "clamp", 0.0)
    icl.force_variant("sepconv3d", None)


def test_sepconv3d_large_sampled():
    """64 x 512 x 512 (256 MB in + out), r = 3 on every axis, sampled voxels incl. the boundary faces."""
    d, hh, w = 64, 512, 512
    src = torch.empty(d, hh, w, device=DEV)
    icl.fill_uniform(src, 11)  # slice z = synth.uniform_image(11 + z, ...)
    out = torch.empty_like(src)
    f = synth.gaussian_taps(3)
    icl.sepconv3d(src, out, f, f, f, "clamp")
    torch.cuda.synchronize()
    rng = np.random.default_rng(0)
    zs = np.concatenate([rng.integers(0, d, 400), [0, d - 1, 0, d - 1]])
    ys = np.concatenate([rng.integers(0, hh, 400), [0, hh - 1, hh - 1, 0]])
    xs = np.concatenate([rng.integers(0, w, 400), [0, w - 1, 0, w - 1]])
    # the oracle reads only the slices the samples touch: rebuild them on the host
    v = np.stack([synth.uniform_image(11 + z, hh, w) for z in range(d)])
    check(out.cpu().numpy()[zs, ys, xs], v, f, f, f, "clamp", 0.0, points=(xs, ys, zs))


def test_sepconv3d_errors():
    a = torch.zeros(4, 8, 8, device=DEV)
    b = torch.zeros(4, 8, 8, device=DEV)
    with pytest.raises(icl.IclError) as e:
        icl.sepconv3d(a, a, [1.0], [1.0], [1.0])
    assert e.value.status == 2
    with pytest.raises(icl.IclError) as e:
        icl.sepconv3d(a, b, [1.0] * 17, [1.0], [1.0])  # radius 8
    assert e.value.status == 3
    with pytest.raises(icl.IclError):
        icl.sepconv3d(a, torch.zeros(5, 8, 8, device=DEV), [1.0], [1.0], [1.0])


def test_sepconv3d_random_sweep():
    """16 seeded random volumes (incl. 1-slice, 1-row, 1-column), radii 0..7 per axis, random borders:
    both variants vs the oracle and bit-identical to each other."""
    rng = np.random.default_rng(77)
    for case in range(16):
        d, h, w = int(rng.integers(1, 24)), int(rng.integers(1, 50)), int(rng.integers(1, 150))
        if case % 5 == 0:
            d = 1
        if case % 5 == 1:
            h = 1
        if case % 5 == 2:
            w = 1
        rx, ry, rz = (int(v) for v in rng.integers(0, 8, 3))
        border, c = ("constant", float(rng.choice([0.0, 0.3]))) if rng.random() < 0.5 else ("clamp", 0.0)
        v = vol(500 + 50 * case, d, h, w)
        src = dev(v, pitch=w + int(rng.integers(0, 6)))
        f, g, hz = synth.signed_taps(case, rx), synth.gaussian_taps(ry), synth.signed_taps(case + 1, rz)
        outs = []
        for name in icl.variant_names("sepconv3d"):
            icl.force_variant("sepconv3d", name)
            out = torch.full_like(src, float("nan"))
            icl.sepconv3d(src, out, f, g, hz, border, c)
            outs.append(out)
        icl.force_variant("sepconv3d", None)
        torch.cuda.synchronize()
        assert torch.equal(outs[0], outs[1]), case
        check(outs[1].cpu().numpy(), v, f, g, hz, border, c)
