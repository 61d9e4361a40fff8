"""Row-band sepconv with the halo rows read in the kernel from the other ranks'
memory (icl_sepconv_peer over CUDA IPC).

Two or three processes share the one GPU of the test box (CUDA IPC works
between processes of one device exactly as between the GPUs of a node; on an
NVLink node the same loads go over NVLink).  Each rank holds ONLY its own
rows; the handles travel over a gloo group.  The stitched bands must equal
the unsharded icl_sepconv bit for bit."""
import os
import socket

import numpy as np
import pytest

import synth
from tests._tol import check_harris, check_nlm, check_sepconv

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _edge_points(H, W, cuts, seed, extra=400):
    """Every pixel of the rows next to each band edge (where the halo came from a peer) plus
    random pixels: what the oracle checks after the unsharded comparison."""
    rng = np.random.default_rng(seed)
    ys, xs = [rng.integers(0, H, extra)], [rng.integers(0, W, extra)]
    for c in cuts:
        for y in range(max(0, c - 3), min(H, c + 3)):
            ys.append(np.full(W, y))
            xs.append(np.arange(W))
    return np.concatenate(xs), np.concatenate(ys)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, n, port, H, W, B, rx, ry, border, cval):
    import paper_1605_06399_b200 as icl
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=n)
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    full = np.stack([synth.uniform_image(50 + i, H, W) for i in range(B)])
    rows = -(-H // n)
    r0, r1 = rank * rows, min(H, (rank + 1) * rows)
    pitch = W + 3 + (rank % 2) * 8  # ranks use different pitches
    buf = torch.full((B, r1 - r0, pitch), float("nan"), device=dev)
    own = buf[..., :W]
    own.copy_(torch.from_numpy(full[:, r0:r1]))
    out = torch.full((B, r1 - r0, W), float("nan"), device=dev)
    torch.cuda.synchronize()
    h, off = icl.ipc_handle(buf)
    meta = [None] * n
    dist.all_gather_object(meta, (h, off, r1 - r0, pitch))
    up = down = None
    if rank > 0:
        hh, oo, hgt, pp = meta[rank - 1]
        up = icl.PeerImage(hh, oo, W, hgt, pp, B, hgt * pp)
    if rank < n - 1:
        hh, oo, hgt, pp = meta[rank + 1]
        down = icl.PeerImage(hh, oo, W, hgt, pp, B, hgt * pp)
    dist.barrier()  # every band written
    fx, gy = synth.gaussian_taps(rx), synth.signed_taps(3, ry)
    icl.sepconv_peer(own, out, H, r0, up, down, fx, gy, border, cval)
    torch.cuda.synchronize()
    dist.barrier()  # every peer read done before anyone frees its band
    parts = [None] * n
    dist.all_gather_object(parts, out.cpu().numpy())
    if rank == 0:
        src = torch.from_numpy(full).to(dev)
        ref = torch.empty_like(src)
        icl.sepconv(src, ref, fx, gy, border, cval)
        got = np.concatenate(parts, axis=1)
        np.testing.assert_array_equal(got, ref.cpu().numpy())
        xs, ys = _edge_points(H, W, [k * rows for k in range(1, n)], 1, extra=200)
        for b in range(B):  # and the CPU oracle on the edge rows
            check_sepconv(got[b][ys, xs], full[b], fx, gy, border, cval, points=(xs, ys))
    for p in (up, down):
        if p:
            p.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n,H,W,B,rx,ry,border,cval", [
    (2, 200, 389, 1, 2, 2, "constant", 0.0),
    (3, 300, 389, 2, 15, 15, "clamp", 0.0),
    (3, 97, 130, 1, 1, 3, "constant", 0.5),
    (2, 33, 1029, 1, 7, 15, "clamp", 0.0),
])
def test_sepconv_peer_bands_equal_unsharded(n, H, W, B, rx, ry, border, cval):
    mp.spawn(_worker, args=(n, _free_port(), H, W, B, rx, ry, border, cval), nprocs=n, join=True)


def _harris_worker(rank, n, port, H, W, block, border, cval):
    """icl_harris_peer: own rows only, edge rows read in-kernel from the neighbours' bands."""
    import paper_1605_06399_b200 as icl
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=n)
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    full = synth.rect_scene(90, H, W)
    rows = -(-H // n)
    r0, r1 = rank * rows, min(H, (rank + 1) * rows)
    buf = torch.full((r1 - r0, W + 4), float("nan"), device=dev)
    own = buf[:, :W]
    own.copy_(torch.from_numpy(full[r0:r1]))
    torch.cuda.synchronize()
    meta = [None] * n
    dist.all_gather_object(meta, icl.ipc_handle(buf) + (r1 - r0,))
    nb = {}
    for q in (rank - 1, rank + 1):
        if 0 <= q < n:
            h, off, hgt = meta[q]
            nb[q] = icl.PeerImage(h, off, W, hgt, W + 4)
    dist.barrier()
    out = torch.full((r1 - r0, W), float("nan"), device=dev)
    m = torch.full((r1 - r0, W), 77, dtype=torch.uint8, device=dev)
    icl.harris_peer(own, out, H, r0, nb.get(rank - 1), nb.get(rank + 1), block, 0.04, border, cval, mask=m,
                    threshold=0.01)
    torch.cuda.synchronize()
    dist.barrier()
    parts = [None] * n
    dist.all_gather_object(parts, (out.cpu().numpy(), m.cpu().numpy()))
    if rank == 0:
        src = torch.from_numpy(full).to(dev)
        ref = torch.empty_like(src)
        mref = torch.empty(H, W, dtype=torch.uint8, device=dev)
        icl.force_variant("harris", "naive_direct")  # the peer edge kernels keep the naive order
        icl.harris(src, ref, block, 0.04, border, cval, mask=mref, threshold=0.01)
        icl.force_variant("harris", None)
        R, M = np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts])
        np.testing.assert_array_equal(R, ref.cpu().numpy())
        np.testing.assert_array_equal(M, mref.cpu().numpy())
        xs, ys = _edge_points(H, W, [k * rows for k in range(1, n)], 2)
        check_harris(R[ys, xs], M[ys, xs], full, block, 0.04, border, cval, 0.01, points=(xs, ys))
    for p in nb.values():
        p.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n,block,border,cval", [(2, 5, "clamp", 0.0), (3, 2, "constant", 0.3), (3, 7, "clamp", 0.0)])
def test_harris_peer_bands_equal_unsharded(n, block, border, cval):
    mp.spawn(_harris_worker, args=(n, _free_port(), 97, 203, block, border, cval), nprocs=n, join=True)


def _pull_worker(rank, n, port, H, W, filt):
    """Halo rows pulled from the neighbours' owned rows (icl_halo_pull), then the ordinary band call."""
    import paper_1605_06399_b200 as icl
    from paper_1605_06399_b200 import dist as icd
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=n)
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    full = synth.rect_scene(70, H, W)
    up_rows, down_rows = icl.harris_halo(5) if filt == "harris" else icl.nlm_halo(2, 5)
    band = icd.partition(H, n, rank, up_rows, down_rows)
    buf = torch.full((band.buf_rows, W), float("nan"), device=dev)
    buf[band.own_slice] = torch.from_numpy(full[band.r0:band.r1]).to(dev)
    torch.cuda.synchronize()
    meta = [None] * n
    dist.all_gather_object(meta, icl.ipc_handle(buf) + (band.r0 - band.s0, band.rows))
    nb = {}
    for q in (rank - 1, rank + 1):
        if 0 <= q < n:
            h, off, skip, rows = meta[q]
            nb[q] = icl.PeerImage(h, off + skip * W * 4, W, rows, W)
    dist.barrier()
    icl.halo_pull(buf, H, band.s0, band.r0, band.r1, nb.get(rank - 1), nb.get(rank + 1))
    out = torch.empty(band.rows, W, device=dev)
    if filt == "harris":
        icl.harris(buf, out, 5, 0.04, "clamp", band=band.icl_band())
    else:
        icl.nlm(buf, out, 2, 5, 0.1, "clamp", band=band.icl_band())
    torch.cuda.synchronize()
    dist.barrier()
    parts = [None] * n
    dist.all_gather_object(parts, out.cpu().numpy())
    if rank == 0:
        src = torch.from_numpy(full).to(dev)
        ref = torch.empty_like(src)
        got = np.concatenate(parts)
        cuts = [icd.partition(H, n, k, up_rows, down_rows).r0 for k in range(1, n)]
        xs, ys = _edge_points(H, W, cuts, 3, extra=200)
        if filt == "harris":
            icl.harris(src, ref, 5, 0.04, "clamp")
            np.testing.assert_array_equal(got, ref.cpu().numpy())
            check_harris(got[ys, xs], None, full, 5, 0.04, "clamp", 0.0, 0.0, points=(xs, ys))
        else:  # box-sum tiles restart at band edges: equal to rounding
            icl.nlm(src, ref, 2, 5, 0.1, "clamp")
            np.testing.assert_allclose(got, ref.cpu().numpy(), rtol=0, atol=2e-6)
            check_nlm(got[ys, xs], full, 2, 5, 0.1, "clamp", 0.0, points=(xs, ys))
    for p in nb.values():
        p.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n,filt", [(2, "harris"), (3, "harris"), (3, "nlm")])
def test_halo_pull_bands_equal_unsharded(n, filt):
    mp.spawn(_pull_worker, args=(n, _free_port(), 150, 203, filt), nprocs=n, join=True)


@pytest.mark.parametrize("nb", [2, 3, 5])
def test_peer_paths_in_one_process(nb):
    """The bands of one image in one process, neighbours passed as plain device memory
    (icl.LocalBand): sepconv_peer and harris_peer stitched == unsharded, bit for bit."""
    import paper_1605_06399_b200 as icl
    DEV = torch.device("cuda:0")
    H, W = 120, 333
    full = synth.rect_scene(95, H, W)
    rows = -(-H // nb)
    cuts = [(k * rows, min(H, (k + 1) * rows)) for k in range(nb)]
    bands = [torch.from_numpy(np.ascontiguousarray(full[a:b])).to(DEV) for a, b in cuts]
    f = synth.gaussian_taps(3)
    src = torch.from_numpy(full).to(DEV)
    ref_s, ref_h = torch.empty_like(src), torch.empty_like(src)
    ref_m = torch.empty(H, W, dtype=torch.uint8, device=DEV)
    icl.sepconv(src, ref_s, f, f, "clamp")
    icl.force_variant("harris", "naive_direct")  # the peer edge kernels keep the naive order
    icl.harris(src, ref_h, 5, 0.04, "constant", 0.2, mask=ref_m, threshold=0.01)
    icl.force_variant("harris", None)
    out_s, out_h, out_m = [], [], []
    for k, (a, b) in enumerate(cuts):
        up = icl.LocalBand(bands[k - 1]) if k > 0 else None
        dn = icl.LocalBand(bands[k + 1]) if k + 1 < nb else None
        o = torch.empty(b - a, W, device=DEV)
        icl.sepconv_peer(bands[k], o, H, a, up, dn, f, f, "clamp")
        out_s.append(o)
        oh = torch.empty(b - a, W, device=DEV)
        om = torch.empty(b - a, W, dtype=torch.uint8, device=DEV)
        icl.harris_peer(bands[k], oh, H, a, up, dn, 5, 0.04, "constant", 0.2, mask=om, threshold=0.01)
        out_h.append(oh)
        out_m.append(om)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(out_s), ref_s)
    assert torch.equal(torch.cat(out_h), ref_h) and torch.equal(torch.cat(out_m), ref_m)
    xs, ys = _edge_points(H, W, [a for a, _ in cuts[1:]], 4)
    check_sepconv(torch.cat(out_s).cpu().numpy()[ys, xs], full, f, f, "clamp", 0.0, points=(xs, ys))
    Rh, Mh = torch.cat(out_h).cpu().numpy(), torch.cat(out_m).cpu().numpy()
    check_harris(Rh[ys, xs], Mh[ys, xs], full, 5, 0.04, "constant", 0.2, 0.01, points=(xs, ys))


def test_sepconv_peer_single_rank_and_errors():
    import paper_1605_06399_b200 as icl
    dev = torch.device("cuda:0")
    img = torch.from_numpy(synth.uniform_image(60, 64, 100)).to(dev)
    out, ref = torch.empty_like(img), torch.empty_like(img)
    f = synth.gaussian_taps(2)
    icl.sepconv_peer(img, out, 64, 0, None, None, f, f, "constant")  # one rank: no neighbours needed
    icl.sepconv(img, ref, f, f, "constant")
    assert torch.equal(out, ref)
    with pytest.raises(icl.IclError):  # rows above exist but no up neighbour given
        icl.sepconv_peer(img[32:], out[32:], 64, 32, None, None, f, f, "constant")
    h, off = icl.ipc_handle(img[10:])
    assert len(h) == 64 and off >= 10 * 100 * 4
