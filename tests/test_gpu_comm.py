"""Native sharded calls (icl_*_sharded over an icl_comm, NCCL loaded at run
time) on one GPU: a 1-rank communicator exercises the NCCL load / init path
and the band bookkeeping, and must equal the unsharded call bit for bit
(sepconv, Harris + mask, conv2d) or to the NLM tolerance.  The multi-rank
exchange plan is pinned on CPU (tests/test_shard_plan.py) and the exchange
itself by tools/comm_2rank.py where two ranks can run."""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1605_06399_b200 as icl  # noqa: E402

DEV = torch.device("cuda:0")


@pytest.fixture(scope="module")
def comm():
    c = icl.Comm(1, 0)
    yield c
    c.close()


def test_single_rank_band_is_the_image(comm):
    assert comm.band(1000, 3, 3) == (0, 1000, 0, 1000)


def test_sepconv_sharded(comm):
    img = synth.uniform_image(70, 300, 256)
    fx = synth.gaussian_taps(3)
    src = torch.from_numpy(img).to(DEV)
    ref, out = torch.empty_like(src), torch.empty_like(src)
    icl.sepconv(src, ref, fx, fx, "constant", 0.5)
    comm.sepconv(src, out, 300, fx, fx, "constant", 0.5)
    np.testing.assert_array_equal(out.cpu().numpy(), ref.cpu().numpy())


def test_harris_sharded_with_mask(comm):
    img = synth.rect_scene(71, 200, 256, n_rect=10, noise=0.01)
    src = torch.from_numpy(img).to(DEV)
    ref, out = torch.empty_like(src), torch.empty_like(src)
    rm = torch.empty(200, 256, dtype=torch.uint8, device=DEV)
    om = torch.empty_like(rm)
    icl.harris(src, ref, 5, 0.04, "clamp", mask=rm, threshold=0.3)
    comm.harris(src, out, 200, 5, 0.04, "clamp", mask=om, threshold=0.3)
    np.testing.assert_array_equal(out.cpu().numpy(), ref.cpu().numpy())
    np.testing.assert_array_equal(om.cpu().numpy(), rm.cpu().numpy())


def test_nlm_and_conv2d_sharded(comm):
    img = synth.rect_scene(72, 120, 128, n_rect=8, noise=0.0866)
    src = torch.from_numpy(img).to(DEV)
    ref, out = torch.empty_like(src), torch.empty_like(src)
    icl.nlm(src, ref, 2, 5, 0.1, "clamp")
    comm.nlm(src, out, 120, 2, 5, 0.1, "clamp")
    np.testing.assert_allclose(out.cpu().numpy(), ref.cpu().numpy(), rtol=0, atol=2e-5)
    u8 = torch.from_numpy(synth.uniform_u8(73, 150, 192)).to(DEV)
    f = synth.filter2d(73, 2)
    r2, o2 = torch.empty(150, 192, device=DEV), torch.empty(150, 192, device=DEV)
    icl.conv2d_u8(u8, r2, f, "clamp")
    comm.conv2d_u8(u8, o2, 150, f, "clamp")
    np.testing.assert_array_equal(o2.cpu().numpy(), r2.cpu().numpy())


def test_shape_mismatch_is_rejected(comm):
    src = torch.zeros(10, 16, device=DEV)
    out = torch.zeros(9, 16, device=DEV)
    with pytest.raises(icl.IclError) as e:
        comm.sepconv(src, out, 10, [1.0], [1.0])
    assert e.value.status == 1
