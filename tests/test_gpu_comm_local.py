"""The native row-band exchange (comm.cu run_sharded: pack -> grouped send / recv ->
unpack, interior rows overlapped, edge rows after the join) at N = 2..8 ranks on ONE
GPU, through the in-process loopback transport (icl_comm_init_local): every rank is a
host thread with its own stream and band buffer, exactly as one process per GPU would
call icl_*_sharded.

The band buffers' halo rows start as NaN, so a row the exchange fails to deliver shows
up in the output.  Stitched bands must equal the unsharded call bit for bit (sepconv,
Harris + mask, conv2d_u8; NLM to rounding), and sampled pixels -- including every row
next to a band edge -- must match the CPU oracle within the north_star tolerances."""
import threading

import numpy as np
import pytest

import synth
from tests._tol import check_conv2d, check_harris, check_nlm, check_sepconv

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1605_06399_b200 as icl  # noqa: E402
from paper_1605_06399_b200 import dist as icd  # noqa: E402

DEV = torch.device("cuda:0")


def run_ranks(n, height, up, down, img, call, out_dtype=torch.float32, with_mask=False):
    """Shard `img` (H x W [x batch leading]) into n bands, run `call(comm, buf, dst, mask, stream)`
    on n threads, return the stitched outputs (and masks)."""
    comms = icl.Comm.local_group(n)
    bands = [icd.partition(height, n, k, up, down) for k in range(n)]
    src = torch.from_numpy(img)
    bufs, dsts, masks, streams = [], [], [], []
    for b in bands:
        buf = torch.full((*img.shape[:-2], b.buf_rows, img.shape[-1]), float("nan"), dtype=src.dtype) \
            if src.dtype == torch.float32 else torch.full((*img.shape[:-2], b.buf_rows, img.shape[-1]), 255,
                                                          dtype=src.dtype)
        buf[..., b.r0 - b.s0:b.r1 - b.s0, :] = src[..., b.r0:b.r1, :]
        bufs.append(buf.to(DEV))
        dsts.append(torch.full((*img.shape[:-2], b.rows, img.shape[-1]), float("nan"), dtype=out_dtype,
                               device=DEV))
        masks.append(torch.full((*img.shape[:-2], b.rows, img.shape[-1]), 7, dtype=torch.uint8, device=DEV)
                     if with_mask else None)
        streams.append(torch.cuda.Stream(device=DEV))
    torch.cuda.synchronize()
    errs = [None] * n

    def worker(k):
        try:
            call(comms[k], bufs[k], dsts[k], masks[k], streams[k])
            streams[k].synchronize()
        except Exception as e:  # noqa: BLE001 -- reported on the main thread
            errs[k] = e

    th = [threading.Thread(target=worker, args=(k,)) for k in range(n)]
    for t in th:
        t.start()
    for t in th:
        t.join(300)
    for c in comms:
        c.close()
    for e in errs:
        if e is not None:
            raise e
    out = torch.cat([d for d in dsts], dim=-2).cpu().numpy()
    m = torch.cat(masks, dim=-2).cpu().numpy() if with_mask else None
    return out, m, bands


def edge_points(bands, H, W, rng, extra=600):
    """Every pixel of the rows around each band edge plus random pixels."""
    ys = [rng.integers(0, H, extra)]
    xs = [rng.integers(0, W, extra)]
    for b in bands[1:]:
        for y in range(max(0, b.r0 - 3), min(H, b.r0 + 3)):
            ys.append(np.full(W, y))
            xs.append(np.arange(W))
    return np.concatenate(xs), np.concatenate(ys)


@pytest.mark.parametrize("n", [2, 3, 5, 8])
@pytest.mark.parametrize("r,border,c", [(1, "constant", 0.0), (2, "clamp", 0.0), (7, "constant", 0.5),
                                        (15, "clamp", 0.0)])
def test_sepconv_local_ranks(n, r, border, c):
    H, W = 40 * n + 13, 300
    img = synth.uniform_image(200 + n + r, H, W)
    fx = synth.gaussian_taps(r)
    gy = synth.gaussian_taps(max(r - 1, 0)) if r > 1 else fx
    ry = len(gy) // 2
    out, _, bands = run_ranks(n, H, ry, ry, img,
                              lambda cm, buf, dst, m, st: cm.sepconv(buf, dst, H, fx, gy, border, c, stream=st))
    ref = torch.empty(H, W, device=DEV)
    icl.sepconv(torch.from_numpy(img).to(DEV), ref, fx, gy, border, c)
    np.testing.assert_array_equal(out, ref.cpu().numpy())
    xs, ys = edge_points(bands, H, W, np.random.default_rng(n))
    check_sepconv(out[ys, xs], img, fx, gy, border, c, points=(xs, ys))


@pytest.mark.parametrize("n", [2, 4, 7])
@pytest.mark.parametrize("block,border", [(5, "clamp"), (2, "constant"), (7, "clamp")])
def test_harris_local_ranks(n, block, border):
    H, W = 30 * n + 11, 257
    img = synth.rect_scene(300 + n + block, H, W, n_rect=12, noise=0.01)
    up, down = icl.harris_halo(block)
    thr = 0.3
    out, mask, bands = run_ranks(
        n, H, up, down, img,
        lambda cm, buf, dst, m, st: cm.harris(buf, dst, H, block, 0.04, border, 0.2, mask=m, threshold=thr,
                                              stream=st),
        with_mask=True)
    ref = torch.empty(H, W, device=DEV)
    rm = torch.empty(H, W, dtype=torch.uint8, device=DEV)
    icl.harris(torch.from_numpy(img).to(DEV), ref, block, 0.04, border, 0.2, mask=rm, threshold=thr)
    np.testing.assert_array_equal(out, ref.cpu().numpy())
    np.testing.assert_array_equal(mask, rm.cpu().numpy())
    xs, ys = edge_points(bands, H, W, np.random.default_rng(10 + n))
    check_harris(out[ys, xs], mask[ys, xs], img, block, 0.04, border, 0.2, thr, points=(xs, ys))


@pytest.mark.parametrize("n", [2, 3, 6])
def test_nlm_local_ranks(n):
    H, W, P, S = 20 * n + 9, 96, 2, 5
    img = synth.rect_scene(400 + n, H, W, n_rect=8, noise=0.0866)
    out, _, bands = run_ranks(n, H, P + S, P + S, img,
                              lambda cm, buf, dst, m, st: cm.nlm(buf, dst, H, P, S, 0.1, "clamp", stream=st))
    ref = torch.empty(H, W, device=DEV)
    icl.nlm(torch.from_numpy(img).to(DEV), ref, P, S, 0.1, "clamp")
    np.testing.assert_allclose(out, ref.cpu().numpy(), rtol=0, atol=2e-5)
    xs, ys = edge_points(bands, H, W, np.random.default_rng(20 + n), extra=300)
    check_nlm(out[ys, xs], img, P, S, 0.1, "clamp", 0.0, points=(xs, ys))


@pytest.mark.parametrize("n", [2, 4, 8])
def test_conv2d_local_ranks(n):
    H, W, r = 25 * n + 6, 192, 2
    img = synth.uniform_u8(500 + n, H, W)
    f = synth.filter2d(500 + n, r)
    out, _, bands = run_ranks(n, H, r, r, img,
                              lambda cm, buf, dst, m, st: cm.conv2d_u8(buf, dst, H, f, "clamp", stream=st))
    ref = torch.empty(H, W, device=DEV)
    icl.conv2d_u8(torch.from_numpy(img).to(DEV), ref, f, "clamp")
    np.testing.assert_array_equal(out, ref.cpu().numpy())
    xs, ys = edge_points(bands, H, W, np.random.default_rng(30 + n))
    check_conv2d(out[ys, xs], img, f, "clamp", 0.0, points=(xs, ys))


def test_batched_bands_local_ranks():
    """A batch of images shares one exchange (all images' halo rows in one message per neighbour)."""
    n, H, W, B = 4, 97, 130, 3
    img = np.stack([synth.uniform_image(600 + i, H, W) for i in range(B)])
    fx = synth.gaussian_taps(3)
    out, _, _ = run_ranks(n, H, 3, 3, img,
                          lambda cm, buf, dst, m, st: cm.sepconv(buf, dst, H, fx, fx, "clamp", stream=st))
    ref = torch.empty(B, H, W, device=DEV)
    icl.sepconv(torch.from_numpy(img).to(DEV), ref, fx, fx, "clamp")
    np.testing.assert_array_equal(out, ref.cpu().numpy())


def test_repeated_calls_reuse_the_mailboxes():
    """Several sharded calls in a row on the same comms (FIFO matching per rank pair)."""
    n, H, W = 3, 90, 64
    img = synth.uniform_image(700, H, W)
    fx = synth.gaussian_taps(2)

    def call(cm, buf, dst, m, st):
        for _ in range(4):
            cm.sepconv(buf, dst, H, fx, fx, "constant", stream=st)

    out, _, _ = run_ranks(n, H, 2, 2, img, call)
    ref = torch.empty(H, W, device=DEV)
    icl.sepconv(torch.from_numpy(img).to(DEV), ref, fx, fx, "constant")
    np.testing.assert_array_equal(out, ref.cpu().numpy())


def test_thin_last_band_rejected_on_every_rank():
    """H = 10 over 4 ranks with ry = 2 leaves rank 3 one row; the call is collective,
    so EVERY rank must reject it (no rank may post a send the thin rank never matches)."""
    comms = icl.Comm.local_group(4)
    fx = synth.gaussian_taps(2)
    try:
        for k, cm in enumerate(comms):
            per = 3
            r0, r1 = min(k * per, 10), min(k * per + per, 10)
            s0, s1 = max(0, r0 - 2), min(10, r1 + 2)
            buf = torch.zeros(s1 - s0, 16, device=DEV)
            dst = torch.zeros(r1 - r0, 16, device=DEV)
            with pytest.raises(icl.IclError) as e:
                cm.sepconv(buf, dst, 10, fx, fx)
            assert e.value.status == 1
    finally:
        for c in comms:
            c.close()
