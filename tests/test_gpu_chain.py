"""The fused two-filter pipeline icl_blur_harris (
PAPER.md §2.2, R24): smoothing + Harris in one pass.

Two bars:
* against the CPU oracle, on inputs where the blur is exact in fp32 (8-bit
  valued pixels k/256, binomial taps m/2^n): the oracle's double blur is then
  the very fp32 image the GPU's Harris stage sees, and the chain must match
  oracle.harris(oracle.sepconv(x)) within the Harris tolerance (tests/_tol.py);
* against the two library calls on general inputs (Gaussian taps, i.i.d.
  uniform pixels): harris(sepconv(x)) bit for bit, including masks, row bands
  and batches.
"""
import numpy as np
import pytest

import oracle
import synth
from tests._tol import check_harris

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1605_06399_b200 as icl  # noqa: E402

DEV = torch.device("cuda:0")
BINOMIAL = {0: [1.0], 1: [1, 2, 1], 2: [1, 4, 6, 4, 1], 3: [1, 6, 15, 20, 15, 6, 1]}


def binomial(r):
    t = np.array(BINOMIAL[r], dtype=np.float64)
    return (t / t.sum()).astype(np.float32)


def pad4(w):
    return w + (-w) % 4


def dev(a, pitch=None):
    h, w = a.shape[-2:]
    pitch = pitch or pad4(w)
    buf = torch.full(a.shape[:-1] + (pitch,), float("nan"), dtype=torch.float32, device=DEV)
    buf[..., :w] = torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
    return buf[..., :w]


def u8_image(seed, h, w):
    return (synth.uniform_u8(seed, h, w).astype(np.float32) / np.float32(256.0))


def out_like(src, dtype=torch.float32):
    """Output view with a 16-byte aligned row pitch (the fused chain's layout requirement)."""
    w = src.shape[-1]
    fill = 77 if dtype == torch.uint8 else float("nan")
    return torch.full(tuple(src.shape[:-1]) + (pad4(w),), fill, dtype=dtype, device=DEV)[..., :w]


def two_calls(src, fx, gy, bb, bc, block, k, border, c, thr, with_mask=True):
    blurred = out_like(src)
    icl.sepconv(src, blurred, fx, gy, bb, bc)
    R = out_like(src)
    m = out_like(src, torch.uint8) if with_mask else None
    # the chain keeps the naive per-output Harris order (R24): compare with that variant
    icl.force_variant("harris", "naive_direct")
    try:
        icl.harris(blurred, R, block, k, border, c, mask=m, threshold=thr)
    finally:
        icl.force_variant("harris", None)
    return R, m


def fused(src, fx, gy, bb, bc, block, k, border, c, thr, with_mask=True):
    R = out_like(src)
    m = out_like(src, torch.uint8) if with_mask else None
    icl.blur_harris(src, R, fx, gy, bb, bc, block, k, border, c, mask=m, threshold=thr)
    return R, m


@pytest.mark.parametrize("shape", [(1, 1), (1, 300), (300, 1), (7, 9), (53, 61), (129, 1029), (300, 67)])
@pytest.mark.parametrize("r", [1, 2, 3])
@pytest.mark.parametrize("blur_border,hborder", [(("constant", 0.0), ("clamp", 0.0)),
                                                 (("clamp", 0.0), ("clamp", 0.0)),
                                                 (("constant", 0.75), ("constant", 0.25))])
def test_chain_vs_oracle_exact_blur(shape, r, blur_border, hborder):
    h, w = shape
    img = u8_image(10 + r, h, w)
    f = binomial(r)
    (bb, bc), (hb, hc) = blur_border, hborder
    blur = oracle.sepconv(img, f, f, bb, bc)
    b32 = blur.astype(np.float32)
    assert np.array_equal(b32.astype(np.float64), blur), "blur must be exact in fp32 for this pin"
    Rr = oracle.harris(b32, 5, 0.04, hb, hc)
    thr = float(0.01 * np.max(Rr)) if Rr.size else 0.0
    R, m = fused(dev(img), f, f, bb, bc, 5, 0.04, hb, hc, thr)
    torch.cuda.synchronize()
    check_harris(R.cpu().numpy(), m.cpu().numpy(), b32, 5, 0.04, hb, hc, thr)


@pytest.mark.parametrize("block", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("rx,ry", [(0, 0), (1, 1), (2, 2), (3, 3), (1, 3), (2, 0)])
@pytest.mark.parametrize("shape", [(5, 7), (67, 300), (130, 517)])
def test_chain_equals_two_calls(block, rx, ry, shape):
    h, w = shape
    img = synth.uniform_image(20 + block, h, w)
    src = dev(img, pitch=w + (-w) % 4 + 8)
    fx, gy = synth.gaussian_taps(rx), synth.gaussian_taps(ry)
    for (bb, bc), (hb, hc) in [(("constant", 0.0), ("clamp", 0.0)), (("clamp", 0.0), ("constant", 0.3)),
                               (("constant", 0.7), ("clamp", 0.0))]:
        R0, m0 = two_calls(src, fx, gy, bb, bc, block, 0.04, hb, hc, 0.001)
        R1, m1 = fused(src, fx, gy, bb, bc, block, 0.04, hb, hc, 0.001)
        assert torch.equal(R0, R1), (bb, hb)
        assert torch.equal(m0, m1)


def test_chain_batch_and_bands():
    B, H, W = 3, 200, 389
    img = np.stack([synth.uniform_image(30 + i, H, W) for i in range(B)])
    src = dev(img, pitch=392)
    f = synth.gaussian_taps(2)
    R0, m0 = two_calls(src, f, f, "constant", 0.0, 5, 0.04, "clamp", 0.0, 0.002)
    R1, m1 = fused(src, f, f, "constant", 0.0, 5, 0.04, "clamp", 0.0, 0.002)
    assert torch.equal(R0, R1) and torch.equal(m0, m1)
    # row bands: rank k computes rows [y0, y1) from a buffer holding its rows plus the chain's halo
    up, down = icl.harris_halo(5)
    up, down = up + 2, down + 2
    out = out_like(src)
    for y0, y1 in [(0, 37), (37, 120), (120, 200)]:
        s0, s1 = max(0, y0 - up), min(H, y1 + down)
        icl.blur_harris(src[:, s0:s1], out[:, y0:y1], f, f, "constant", 0.0, 5, 0.04, "clamp",
                        band=(H, s0, y0))
    assert torch.equal(out, R0)


@pytest.mark.parametrize("block", [2, 5])
def test_chain_two_pass_schedule(block):
    """With a workspace the call runs the two-pass schedule: same bits as the fused kernel."""
    B, H, W = 2, 150, 301
    img = np.stack([synth.uniform_image(40 + i, H, W) for i in range(B)])
    src = dev(img)
    f = synth.gaussian_taps(3)
    nbytes = icl.blur_harris_workspace_bytes(W, H, B, block)
    ws = torch.empty(nbytes // 4 + 4, device=DEV)
    for (bb, bc), (hb, hc) in [(("constant", 0.0), ("clamp", 0.0)), (("clamp", 0.0), ("constant", 0.3))]:
        R0, m0 = fused(src, f, f, bb, bc, block, 0.04, hb, hc, 0.001)
        R1, m1 = out_like(src), out_like(src, torch.uint8)
        icl.blur_harris(src, R1, f, f, bb, bc, block, 0.04, hb, hc, mask=m1, threshold=0.001, workspace=ws)
        assert torch.equal(R0, R1) and torch.equal(m0, m1)
    up, down = icl.harris_halo(block)
    up, down = up + 3, down + 3
    out = out_like(src)
    for y0, y1 in [(0, 50), (50, 51), (51, 150)]:
        s0, s1 = max(0, y0 - up), min(H, y1 + down)
        icl.blur_harris(src[:, s0:s1], out[:, y0:y1], f, f, "clamp", 0.0, block, 0.04, "constant", 0.3,
                        band=(H, s0, y0), workspace=ws)
    R0, _ = fused(src, f, f, "clamp", 0.0, block, 0.04, "constant", 0.3, 0.0)
    assert torch.equal(out, R0)
    with pytest.raises(icl.IclError) as e:  # workspace overlapping the response
        st = R1.untyped_storage()
        bad = torch.empty(0, device=DEV).set_(st, 0, (st.nbytes() // 4,))
        icl.blur_harris(src, R1, f, f, workspace=bad)
    assert e.value.status == 2


def test_chain_padding_never_written():
    """Row padding of the response and mask (NaN / 77 canaries) survives both schedules."""
    h, w = 37, 101
    src = dev(synth.uniform_image(80, h, w), pitch=w + 11)
    f = synth.gaussian_taps(3)
    for ws in (None, torch.empty(icl.blur_harris_workspace_bytes(w, h, 1, 5) // 4 + 4, device=DEV)):
        Rb = torch.full((h, w + 7), float("nan"), device=DEV)
        Mb = torch.full((h, w + 7), 77, dtype=torch.uint8, device=DEV)
        icl.blur_harris(src, Rb[:, :w], f, f, "clamp", 0.0, 5, 0.04, "clamp", mask=Mb[:, :w], threshold=0.01,
                        workspace=ws)
        torch.cuda.synchronize()
        assert torch.isnan(Rb[:, w:]).all() and (Mb[:, w:] == 77).all()
        assert not torch.isnan(Rb[:, :w]).any()


def test_chain_large_sampled():
    """4096^2 in the bench's launch configuration (S = 64 row segments), vs the two calls."""
    img = torch.empty(2, 4096, 4096, device=DEV)
    icl.fill_uniform(img, 99)
    f = synth.gaussian_taps(2)
    R0, m0 = two_calls(img, f, f, "constant", 0.0, 5, 0.04, "clamp", 0.0, 1.0)
    R1, m1 = fused(img, f, f, "constant", 0.0, 5, 0.04, "clamp", 0.0, 1.0)
    assert torch.equal(R0, R1) and torch.equal(m0, m1)


def test_chain_errors():
    a = torch.zeros(32, 32, device=DEV)
    b = torch.zeros(32, 32, device=DEV)
    with pytest.raises(icl.IclError) as e:
        icl.blur_harris(a, b, [1.0] * 9, [1.0] * 9)  # radius 4
    assert e.value.status == 3
    with pytest.raises(icl.IclError) as e:
        icl.blur_harris(a, b, [1.0], [1.0], block=7)
    assert e.value.status == 3
    with pytest.raises(icl.IclError) as e:
        icl.blur_harris(a, a, [1.0], [1.0])
    assert e.value.status == 2
    with pytest.raises((icl.IclError, ValueError, TypeError)):
        icl.blur_harris(a.cpu(), b.cpu(), [1.0], [1.0])  # device images only


def test_chain_random_sweep():
    """24 seeded random cases: shapes (incl. 1-row / 1-column), radii 0..3 per axis, blocks 1..5, both
    borders and constants, both schedules -- bit-identical to the two calls."""
    rng = np.random.default_rng(2024)
    for case in range(24):
        h, w = int(rng.integers(1, 90)), int(rng.integers(1, 700))
        if case % 6 == 0:
            h = 1
        if case % 6 == 1:
            w = 1
        rx, ry, block = int(rng.integers(0, 4)), int(rng.integers(0, 4)), int(rng.integers(1, 6))
        bb = ("constant", float(rng.choice([0.0, 0.6]))) if rng.random() < 0.5 else ("clamp", 0.0)
        hb = ("constant", float(rng.choice([0.0, 0.2]))) if rng.random() < 0.5 else ("clamp", 0.0)
        src = dev(synth.uniform_image(900 + case, h, w))
        fx, gy = synth.signed_taps(case, rx), synth.gaussian_taps(ry)
        thr = float(rng.random() * 0.01)
        R0, m0 = two_calls(src, fx, gy, bb[0], bb[1], block, 0.04, hb[0], hb[1], thr)
        R1, m1 = fused(src, fx, gy, bb[0], bb[1], block, 0.04, hb[0], hb[1], thr)
        assert torch.equal(R0, R1) and torch.equal(m0, m1), (case, h, w, rx, ry, block, bb, hb)
        ws = torch.empty(icl.blur_harris_workspace_bytes(w, h, 1, block) // 4 + 4, device=DEV)
        R2, m2 = out_like(src), out_like(src, torch.uint8)
        icl.blur_harris(src, R2, fx, gy, bb[0], bb[1], block, 0.04, hb[0], hb[1], mask=m2, threshold=thr, workspace=ws)
        assert torch.equal(R0, R2) and torch.equal(m0, m2), case
