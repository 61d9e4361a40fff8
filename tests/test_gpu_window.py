"""In-kernel halo reads over NCCL symmetric memory (SURVEY.md §8(f) row 3 as specified:
ncclMemAlloc + ncclCommWindowRegister, device-side ncclGetPeerPointer; icl_*_window).

One GPU per test box and NCCL refuses two ranks on a device, so the communicator has ONE rank
and the neighbour bands live in that rank's own window (peer 0): the edge kernels still resolve
the neighbours' addresses on the device through the window (ncclGetPeerPointer returns the
window's flat LSA mapping, not the pointer the buffer was allocated at) and load the rows through
it.  The whole image sits in the window at its global rows; every band's own rows are a separate
allocation.  Stitched bands must equal the unsharded call bit for bit (sepconv, Harris + masks)
or to rounding (NLM via the window pull), and sampled pixels incl. every band-edge row must
match the CPU oracle."""
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


@pytest.fixture(scope="module")
def comm():
    c = icl.Comm(1, 0)
    yield c
    c.close()


def window_with(comm, img):
    H, W = img.shape
    pitch = ((W * 4 + 511) // 512) * 512
    win = icl.Window(comm, H * pitch)
    win.write(0, torch.from_numpy(img).to(DEV), pitch)
    torch.cuda.synchronize()
    return win, pitch


def edge_points(H, W, cuts, seed, extra=300):
    rng = np.random.default_rng(seed)
    ys, xs = [rng.integers(0, H, extra)], [rng.integers(0, W, extra)]
    for c in cuts:
        for y in range(max(0, c - 3), min(H, c + 3)):
            ys.append(np.full(W, y))
            xs.append(np.arange(W))
    return np.concatenate(xs), np.concatenate(ys)


@pytest.mark.parametrize("rx,ry,border,c", [(2, 2, "constant", 0.0), (15, 15, "clamp", 0.0), (1, 3, "constant", 0.5),
                                            (7, 15, "clamp", 0.0)])
def test_sepconv_window_bands(comm, rx, ry, border, c):
    H, W = 200, 389
    img = synth.uniform_image(500 + rx, H, W)
    win, pitch = window_with(comm, img)
    fx, gy = synth.gaussian_taps(rx), synth.signed_taps(3, ry)
    cuts = [(0, 37), (37, 60), (60, 150), (150, 200)]  # (a neighbour band must hold the halo rows)
    out = []
    try:
        for k, (a, b) in enumerate(cuts):
            own = torch.from_numpy(np.ascontiguousarray(img[a:b])).to(DEV)
            up = icl.Window.band(0, cuts[k - 1][0] * pitch, cuts[k - 1][1] - cuts[k - 1][0], pitch) if k else None
            dn = icl.Window.band(0, cuts[k + 1][0] * pitch, cuts[k + 1][1] - cuts[k + 1][0], pitch) \
                if k + 1 < len(cuts) else None
            o = torch.full((b - a, W), float("nan"), device=DEV)
            icl.sepconv_window(win, own, o, H, a, up, dn, fx, gy, border, c)
            out.append(o)
        torch.cuda.synchronize()
    finally:
        win.close()
    got = torch.cat(out).cpu().numpy()
    ref = torch.empty(H, W, device=DEV)
    icl.sepconv(torch.from_numpy(img).to(DEV), ref, fx, gy, border, c)
    np.testing.assert_array_equal(got, ref.cpu().numpy())
    xs, ys = edge_points(H, W, [a for a, _ in cuts[1:]], rx)
    check_sepconv(got[ys, xs], img, fx, gy, border, c, points=(xs, ys))


@pytest.mark.parametrize("block,border,c", [(5, "clamp", 0.0), (2, "constant", 0.3)])
def test_harris_window_bands(comm, block, border, c):
    H, W = 150, 257
    img = synth.rect_scene(510 + block, H, W, n_rect=12, noise=0.01)
    win, pitch = window_with(comm, img)
    cuts = [(0, 60), (60, 70), (70, 150)]
    R, M = [], []
    try:
        for k, (a, b) in enumerate(cuts):
            own = torch.from_numpy(np.ascontiguousarray(img[a:b])).to(DEV)
            up = icl.Window.band(0, cuts[k - 1][0] * pitch, cuts[k - 1][1] - cuts[k - 1][0], pitch) if k else None
            dn = icl.Window.band(0, cuts[k + 1][0] * pitch, cuts[k + 1][1] - cuts[k + 1][0], pitch) \
                if k + 1 < len(cuts) else None
            o = torch.full((b - a, W), float("nan"), device=DEV)
            m = torch.full((b - a, W), 7, dtype=torch.uint8, device=DEV)
            icl.harris_window(win, own, o, H, a, up, dn, block, 0.04, border, c, mask=m, threshold=0.05)
            R.append(o)
            M.append(m)
        torch.cuda.synchronize()
    finally:
        win.close()
    got, gm = torch.cat(R).cpu().numpy(), torch.cat(M).cpu().numpy()
    ref = torch.empty(H, W, device=DEV)
    rm = torch.empty(H, W, dtype=torch.uint8, device=DEV)
    icl.force_variant("harris", "naive_direct")  # the edge kernels keep the naive order
    icl.harris(torch.from_numpy(img).to(DEV), ref, block, 0.04, border, c, mask=rm, threshold=0.05)
    icl.force_variant("harris", None)
    np.testing.assert_array_equal(got, ref.cpu().numpy())
    np.testing.assert_array_equal(gm, rm.cpu().numpy())
    xs, ys = edge_points(H, W, [a for a, _ in cuts[1:]], block)
    check_harris(got[ys, xs], gm[ys, xs], img, block, 0.04, border, c, 0.05, points=(xs, ys))


def test_halo_pull_window_nlm(comm):
    H, W, P, S = 120, 200, 2, 5
    img = synth.rect_scene(520, H, W, n_rect=8, noise=0.0866)
    win, pitch = window_with(comm, img)
    up_r = down_r = P + S
    cuts = [(0, 50), (50, 120)]
    out = []
    try:
        for k, (a, b) in enumerate(cuts):
            s0, s1 = max(0, a - up_r), min(H, b + down_r)
            buf = torch.full((s1 - s0, W), float("nan"), device=DEV)
            buf[a - s0:b - s0] = torch.from_numpy(img[a:b]).to(DEV)
            up = icl.Window.band(0, cuts[k - 1][0] * pitch, cuts[k - 1][1] - cuts[k - 1][0], pitch) if k else None
            dn = icl.Window.band(0, cuts[k + 1][0] * pitch, cuts[k + 1][1] - cuts[k + 1][0], pitch) \
                if k + 1 < len(cuts) else None
            icl.halo_pull_window(win, buf, H, s0, a, b, up, dn)
            o = torch.empty(b - a, W, device=DEV)
            icl.nlm(buf, o, P, S, 0.1, "clamp", band=(H, s0, a))
            out.append(o)
        torch.cuda.synchronize()
    finally:
        win.close()
    got = torch.cat(out).cpu().numpy()
    ref = torch.empty(H, W, device=DEV)
    icl.nlm(torch.from_numpy(img).to(DEV), ref, P, S, 0.1, "clamp")
    np.testing.assert_allclose(got, ref.cpu().numpy(), rtol=0, atol=2e-6)
    xs, ys = edge_points(H, W, [50], 9)
    check_nlm(got[ys, xs], img, P, S, 0.1, "clamp", 0.0, points=(xs, ys))


def test_window_errors(comm):
    img = synth.uniform_image(530, 40, 64)
    win, pitch = window_with(comm, img)
    try:
        own = torch.from_numpy(img[20:]).to(DEV)
        o = torch.empty(20, 64, device=DEV)
        f = synth.gaussian_taps(2)
        with pytest.raises(icl.IclError) as e:  # peer outside the communicator
            icl.sepconv_window(win, own, o, 40, 20, icl.Window.band(3, 0, 20, pitch), None, f, f)
        assert e.value.status == 1
        with pytest.raises(icl.IclError) as e:  # rows above exist but no neighbour given
            icl.sepconv_window(win, own, o, 40, 20, None, None, f, f)
        assert e.value.status == 1
    finally:
        win.close()
    loop = icl.Comm.local_group(1)[0]
    try:
        with pytest.raises(icl.IclError) as e:  # the loopback transport has no NCCL windows
            icl.Window(loop, 1 << 16)
        assert e.value.status == 3
    finally:
        loop.close()
