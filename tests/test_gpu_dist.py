"""Row-band sharded execution on one GPU: N bands of one image, halos filled by
the single-process exchange (same plan as the NCCL path), each band computed
through the C ABI with the interior/edge overlap of dist.run_band, stitched
and compared with the unsharded call (bit-exact for sepconv and Harris, whose
variants share one fp32 operation order; tolerance for NLM box sums)."""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1605_06399_b200 as icl  # noqa: E402
from paper_1605_06399_b200 import dist as icd  # noqa: E402

DEV = torch.device("cuda:0")


def sharded(filter, img, N, call, **hp):
    H, W = img.shape
    up, down = icd.halo_rows(filter, **hp)
    bands = [icd.partition(H, N, k, up, down) for k in range(N)]
    full = torch.from_numpy(img).to(DEV)
    bufs = []
    for b in bands:
        buf = torch.full((b.buf_rows, W), float("nan"), device=DEV)
        buf[b.own_slice] = full[b.r0:b.r1]  # each rank holds only its own rows
        bufs.append(buf)
    outs = [torch.full((b.rows, W), float("nan"), device=DEV) for b in bands]
    comm = torch.cuda.Stream()
    done = {"x": False}

    def exchange():
        if not done["x"]:
            icd.local_halo_exchange(bufs, bands)
            done["x"] = True
    for buf, out, b in zip(bufs, outs, bands):
        icd.run_band(call, buf, out, b, exchange, comm_stream=comm)
    torch.cuda.synchronize()
    return torch.cat(outs).cpu().numpy()


@pytest.mark.parametrize("N", [2, 3, 5])
@pytest.mark.parametrize("border", ["constant", "clamp"])
def test_sepconv_sharded_bit_exact(N, border):
    img = synth.uniform_image(21, 257, 300)
    fx = synth.gaussian_taps(3)
    ref = torch.empty(257, 300, device=DEV)
    icl.sepconv(torch.from_numpy(img).to(DEV), ref, fx, fx, border, 0.25)

    def call(src, dst, band, stream):
        icl.sepconv(src, dst, fx, fx, border, 0.25, band=band, stream=stream)
    got = sharded("sepconv", img, N, call, ry=3)
    np.testing.assert_array_equal(got, ref.cpu().numpy())


@pytest.mark.parametrize("N", [2, 4])
def test_harris_sharded_bit_exact(N):
    img = synth.rect_scene(22, 300, 260, n_rect=20, noise=0.01)
    ref = torch.empty(300, 260, device=DEV)
    icl.harris(torch.from_numpy(img).to(DEV), ref, 5, 0.04, "clamp")

    def call(src, dst, band, stream):
        icl.harris(src, dst, 5, 0.04, "clamp", band=band, stream=stream)
    got = sharded("harris", img, N, call, block=5)
    np.testing.assert_array_equal(got, ref.cpu().numpy())


@pytest.mark.parametrize("N", [2, 3])
def test_nlm_sharded(N):
    img = synth.rect_scene(23, 160, 140, n_rect=12, noise=0.0866)
    ref = torch.empty(160, 140, device=DEV)
    icl.nlm(torch.from_numpy(img).to(DEV), ref, 2, 5, 0.1, "clamp")

    def call(src, dst, band, stream):
        icl.nlm(src, dst, 2, 5, 0.1, "clamp", band=band, stream=stream)
    got = sharded("nlm", img, N, call, patch_radius=2, search_radius=5)
    np.testing.assert_allclose(got, ref.cpu().numpy(), rtol=0, atol=2e-5)
