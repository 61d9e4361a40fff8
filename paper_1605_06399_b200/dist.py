"""Row-band sharding of one large image over the GPUs of a node.

Rank k owns global rows [k*ceil(H/N), min((k+1)*ceil(H/N), H)) and keeps them
in a *band buffer* that also holds the halo rows its stencil reads above and
below (sepconv: ry/ry; Harris: floor(B/2)+1 / B-floor(B/2); NLM: P+S/P+S).
Before a filter call the halo rows are exchanged with the neighbouring ranks
(one grouped send/recv per edge -- NCCL over NVLink on GPUs, gloo on CPU for
the tests); the filter then runs on the band through the C ABI's `icl_band`,
which applies the boundary condition in GLOBAL coordinates, so the stitched
output is identical to the unsharded call (bit-exact for sepconv / Harris).

The exchange is plumbing (torch.distributed); every pixel of every filter is
computed by libicl.so.  `run_band` overlaps the exchange with the interior
rows (which need no halo) on a second stream and finishes the edge rows after
the join.
"""
from __future__ import annotations

import dataclasses
from typing import Callable, Optional, Sequence


@dataclasses.dataclass(frozen=True)
class Band:
    height: int      # global image height
    world: int
    rank: int
    r0: int          # first owned global row
    r1: int          # one past the last owned row
    s0: int          # first global row held in the band buffer (r0 - halo above, clipped)
    s1: int          # one past the last held row
    up: int          # halo rows requested above
    down: int        # halo rows requested below

    @property
    def rows(self) -> int:
        return self.r1 - self.r0

    @property
    def buf_rows(self) -> int:
        return self.s1 - self.s0

    @property
    def own_slice(self) -> slice:
        """Owned rows inside the band buffer."""
        return slice(self.r0 - self.s0, self.r1 - self.s0)

    def icl_band(self, dst_r0: Optional[int] = None):
        """(global_height, src_y0, dst_y0) for icl_* calls writing rows from dst_r0."""
        return (self.height, self.s0, self.r0 if dst_r0 is None else dst_r0)


def partition(height: int, world: int, rank: int, up: int, down: int) -> Band:
    """Band of `rank` with halo (up, down); every rank must own >= max(up, down) rows."""
    per = -(-height // world)
    r0 = min(rank * per, height)
    r1 = min(r0 + per, height)
    if r1 - r0 < max(up, down) and world > 1:
        raise ValueError(f"band of {r1 - r0} rows is thinner than the halo ({up}, {down})")
    return Band(height, world, rank, r0, r1, max(0, r0 - up), min(height, r1 + down), up, down)


def halo_rows(filter: str, **params) -> tuple:
    """Rows of input an output row needs above / below."""
    if filter == "sepconv":
        ry = params["ry"]
        return ry, ry
    if filter == "harris":
        b = params.get("block", 5)
        a = b // 2
        return a + 1, b - 1 - a + 1
    if filter == "nlm":
        r = params.get("patch_radius", 2) + params.get("search_radius", 5)
        return r, r
    raise ValueError(filter)


def exchange_plan(band: Band):
    """[(peer, send_rows(global), recv_rows(global))] for this rank's halo exchange.

    Symmetric by construction: rank k lists rank k+1 exactly when rank k+1
    lists rank k (the ranges are the same rows seen from both sides)."""
    plan = []
    if band.r0 < band.r1 and band.rank > 0:
        # my top halo [s0, r0) comes from rank-1; it needs my first rows as its bottom halo
        prev = partition(band.height, band.world, band.rank - 1, band.up, band.down)
        send, recv = (band.r0, prev.s1), (band.s0, band.r0)
        if send[1] > send[0] or recv[1] > recv[0]:
            plan.append((band.rank - 1, send, recv))
    if band.rank < band.world - 1:
        nxt = partition(band.height, band.world, band.rank + 1, band.up, band.down)
        if nxt.r0 < nxt.r1:
            send, recv = (nxt.s0, band.r1), (band.r1, band.s1)
            if send[1] > send[0] or recv[1] > recv[0]:
                plan.append((band.rank + 1, send, recv))
    return plan


def halo_exchange(buf, band: Band, group=None):
    """Exchange halo rows of `buf` (rows = band.s0 .. band.s1, any trailing dims).

    One grouped P2P per neighbour (torch.distributed.batch_isend_irecv: NCCL on
    CUDA tensors, gloo on CPU tensors)."""
    import torch.distributed as dist
    ops = []
    for peer, (a, b), (c, d) in exchange_plan(band):
        if b > a:
            ops.append(dist.P2POp(dist.isend, buf[a - band.s0:b - band.s0].contiguous(), peer, group))
        if d > c:
            ops.append(dist.P2POp(dist.irecv, buf[c - band.s0:d - band.s0], peer, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


def local_halo_exchange(bufs: Sequence, bands: Sequence[Band]):
    """Single-process stand-in for halo_exchange (all bands on one device): the
    same plan, rows copied directly -- lets one GPU test the sharded path."""
    for buf, band in zip(bufs, bands):
        for peer, _send, (c, d) in exchange_plan(band):
            if d > c:
                pb = bands[peer]
                buf[c - band.s0:d - band.s0].copy_(bufs[peer][c - pb.s0:d - pb.s0])


def run_band(call: Callable, src_buf, dst, band: Band, exchange: Callable, stream=None, comm_stream=None):
    """Exchange halos and run `call(src_view, dst_view, band_tuple, stream)` on the band.

    The rows that need no halo (interior) run on `stream` while the exchange
    runs on `comm_stream`; the edge rows follow after the join."""
    import torch
    stream = stream or torch.cuda.current_stream()
    if band.world == 1 or comm_stream is None:
        exchange()
        call(src_buf, dst, band.icl_band(), stream)
        return
    top_dep = band.up if band.r0 > 0 else 0
    bot_dep = band.down if band.r1 < band.height else 0
    i0, i1 = band.r0 + top_dep, band.r1 - bot_dep  # interior owned rows
    comm_stream.wait_stream(stream)
    with torch.cuda.stream(comm_stream):
        exchange()
    if i1 > i0:
        call(src_buf, dst[i0 - band.r0:i1 - band.r0], band.icl_band(i0), stream)
    stream.wait_stream(comm_stream)
    if i0 > band.r0:
        call(src_buf, dst[:i0 - band.r0], band.icl_band(band.r0), stream)
    if band.r1 > max(i1, i0):
        e0 = max(i1, i0)
        call(src_buf, dst[e0 - band.r0:], band.icl_band(e0), stream)


__all__ = ["Band", "partition", "halo_rows", "exchange_plan", "halo_exchange", "local_halo_exchange", "run_band"]
