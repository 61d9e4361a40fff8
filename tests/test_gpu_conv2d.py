"""GPU parity for the non-separable convolution of 8-bit images (icl_conv2d_u8;
PAPER.md:594-598 §6, Table 3; R22): every
variant against the CPU oracle at sizes spanning several 64 x 64..128 tiles
with ragged right/bottom tiles, r = 0..3, both border modes; variants and
row bands bit-identical to each other; padded / unaligned layouts; batches;
host images; the tuner; BASELINE-sized 8192^2 on sampled pixels."""
import numpy as np
import pytest

import synth
from tests._tol import check_conv2d

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1605_06399_b200 as icl  # noqa: E402

DEV = torch.device("cuda:0")
BORDERS = [("clamp", 0.0), ("constant", 0.0), ("constant", 100.5)]


@pytest.fixture(autouse=True)
def _reset_force():
    yield
    icl.force_variant("conv2d", None)


def u8_dev(img, pitch=None):
    h, w = img.shape
    pitch = pitch or w
    buf = torch.full((h, pitch), 0xAB, dtype=torch.uint8, device=DEV)
    buf[:, :w] = torch.from_numpy(img).to(DEV)
    return buf[:, :w]


def all_variants(call):
    outs = {}
    for vid, name in enumerate(icl.variant_names("conv2d")):
        icl.force_variant("conv2d", vid)
        try:
            outs[name] = call()
        except icl.IclError as e:
            if e.status in (3, 4):
                continue
            raise
    icl.force_variant("conv2d", None)
    return outs


@pytest.mark.parametrize("border,c", BORDERS)
@pytest.mark.parametrize("shape", [(1, 1), (5, 3), (64, 64), (129, 200), (300, 97), (17, 1000)])
@pytest.mark.parametrize("r", [0, 1, 2, 3])
def test_all_variants_vs_oracle(shape, r, border, c):
    h, w = shape
    img = synth.uniform_u8(200 + r, h, w)
    filt = synth.filter2d(5 + r, r)
    src = u8_dev(img, pitch=((w + 15) // 16) * 16 + 16)

    def call():
        dbuf = torch.full((h, ((w + 3) // 4) * 4 + 8), float("nan"), device=DEV)
        icl.conv2d_u8(src, dbuf[:, :w], filt, border, c)
        full = dbuf.cpu().numpy()
        assert np.isnan(full[:, w:]).all(), "padding was written"
        return full[:, :w]
    outs = all_variants(call)
    assert "naive_direct" in outs and (w * h < 64 or "tile_c4r8" in outs)
    check_conv2d(outs["naive_direct"], img, filt, border, c)
    for name, o in outs.items():
        np.testing.assert_array_equal(o, outs["naive_direct"], err_msg=f"variant {name} not bit-identical")


def test_unaligned_layout_uses_the_scalar_path():
    h, w = 70, 131
    img = synth.uniform_u8(9, h, w)
    filt = synth.filter2d(9, 2)
    buf = torch.zeros(h * 133 + 1, dtype=torch.uint8, device=DEV)
    src = buf[1:1 + h * 133].view(h, 133)[:, :w]  # odd base address
    src.copy_(torch.from_numpy(img).to(DEV))
    dst = torch.empty(h, w, device=DEV)
    outs = all_variants(lambda: (icl.conv2d_u8(src, dst, filt, "clamp"), dst.cpu().numpy())[1])
    assert set(outs) == {"naive_direct"}
    check_conv2d(outs["naive_direct"], img, filt, "clamp", 0.0)


def test_batch_and_bands_bit_exact():
    b, h, w, r = 3, 260, 192, 2
    imgs = np.stack([synth.uniform_u8(30 + i, h, w) for i in range(b)])
    filt = synth.filter2d(31, r)
    src = torch.from_numpy(imgs).to(DEV)
    ref = torch.empty(b, h, w, device=DEV)
    icl.conv2d_u8(src, ref, filt, "constant", 7.0)
    ref = ref.cpu().numpy()
    for i in range(b):
        check_conv2d(ref[i], imgs[i], filt, "constant", 7.0)
    cuts = [0, 1, 100, 101, 259, 260]
    for vid, name in enumerate(icl.variant_names("conv2d")):
        icl.force_variant("conv2d", vid)
        for a, e in zip(cuts[:-1], cuts[1:]):
            s0, s1 = max(0, a - r), min(h, e + r)
            dst = torch.empty(b, e - a, w, device=DEV)
            try:
                icl.conv2d_u8(src[:, s0:s1].contiguous(), dst, filt, "constant", 7.0, band=(h, s0, a))
            except icl.IclError as err:
                if err.status in (3, 4):  # not eligible (e.g. texture variants: constant 0 / clamp only)
                    break
                raise
            np.testing.assert_array_equal(dst.cpu().numpy(), ref[:, a:e], err_msg=f"{name} band {a}:{e}")


def test_host_images_equal_device(monkeypatch):
    monkeypatch.setenv("ICL_HOST_CHUNK_ROWS", "33")
    h, w = 150, 256
    img = synth.uniform_u8(40, h, w)
    filt = synth.filter2d(41, 2)
    ref = torch.empty(h, w, device=DEV)
    icl.conv2d_u8(torch.from_numpy(img).to(DEV), ref, filt, "clamp")
    src = torch.from_numpy(img).pin_memory()
    dst = torch.empty(h, w).pin_memory()
    h0, _ = icl.transfer_bytes()
    icl.conv2d_u8(src, dst, filt, "clamp")
    torch.cuda.synchronize()
    np.testing.assert_array_equal(dst.numpy(), ref.cpu().numpy())
    assert icl.transfer_bytes()[0] - h0 >= h * w  # 1 byte per input pixel (+ halo rows)


def test_tuner_picks_an_equivalent_variant():
    h, w = 512, 512
    img = synth.uniform_u8(50, h, w)
    filt = synth.filter2d(51, 2)
    src = torch.from_numpy(img).to(DEV)
    dst = torch.empty(h, w, device=DEV)
    info = icl.tune("conv2d", src, dst, filter2d=filt, border="clamp", force=True)
    assert info["n_rejected"] == 0 and info["n_candidates"] == len(icl.variant_names("conv2d"))
    check_conv2d(dst.cpu().numpy(), img, filt, "clamp", 0.0)


def test_errors():
    src = torch.zeros(8, 8, dtype=torch.uint8, device=DEV)
    dst = torch.zeros(8, 8, device=DEV)
    with pytest.raises(icl.IclError) as e:
        icl.conv2d_u8(src, dst, np.ones((9, 9), np.float32))
    assert e.value.status == 3  # radius 4 unsupported
    bad = np.ones((3, 3), np.float32)
    bad[1, 1] = np.inf
    with pytest.raises(icl.IclError):
        icl.conv2d_u8(src, dst, bad)


def test_paper_size_8192_sampled():
    """8192^2 uchar, 5x5 run-time filter, clamped -- default dispatch, the
    whole border frame plus random interior pixels against the oracle."""
    S = 8192
    img = synth.uniform_u8(8, S, S)
    filt = synth.filter2d(8, 2)
    src = torch.from_numpy(img).to(DEV)
    dst = torch.empty(S, S, device=DEV)
    icl.conv2d_u8(src, dst, filt, "clamp")
    assert icl.variant_names("conv2d")[icl.last_variant("conv2d")] == "tile_c4r8"
    rng = np.random.default_rng(3)
    ys = np.concatenate([rng.integers(0, S, 20000), np.repeat([0, 1, 2, S - 3, S - 2, S - 1], 512)])
    xs = np.concatenate([rng.integers(0, S, 20000), np.tile(np.linspace(0, S - 1, 512).astype(np.int64), 6)])
    ys = np.concatenate([ys, np.tile(np.linspace(0, S - 1, 512).astype(np.int64), 6)])
    xs = np.concatenate([xs, np.repeat([0, 1, 2, S - 3, S - 2, S - 1], 512)])
    got = dst[torch.from_numpy(ys).to(DEV), torch.from_numpy(xs).to(DEV)].cpu().numpy()
    check_conv2d(got, img, filt, "clamp", 0.0, points=(xs, ys))


@pytest.mark.parametrize("border", ["clamp", "constant"])
def test_texture_variant_bands_and_batch(border):
    """The image-memory (texture) variant: hardware clamp / border-0 addressing over the band
    buffer must give the global-boundary result in every band, and images of a batch."""
    b, h, w, r = 2, 200, 256, 3
    imgs = np.stack([synth.uniform_u8(60 + i, h, w) for i in range(b)])
    filt = synth.filter2d(61, r)
    src = torch.from_numpy(imgs).to(DEV)
    ref = torch.empty(b, h, w, device=DEV)
    icl.conv2d_u8(src, ref, filt, border, 0.0)
    ref = ref.cpu().numpy()
    icl.force_variant("conv2d", "tex_c4r4")
    for a, e in [(0, 3), (3, 100), (100, 197), (197, 200)]:
        s0, s1 = max(0, a - r), min(h, e + r)
        rows_pad = (s1 - s0 + 1) // 2 * 2  # batch stride a multiple of 512 B (texture base alignment)
        sb = torch.empty(b, rows_pad, w, dtype=torch.uint8, device=DEV)[:, :s1 - s0]
        sb.copy_(src[:, s0:s1])
        dst = torch.empty(b, e - a, w, device=DEV)
        icl.conv2d_u8(sb, dst, filt, border, 0.0, band=(h, s0, a))
        np.testing.assert_array_equal(dst.cpu().numpy(), ref[:, a:e], err_msg=f"band {a}:{e}")
