"""Row-band sharding host logic (CPU): partition/exchange-plan invariants and a
real multi-process halo exchange over torch.distributed with the gloo backend
(world size 2 and 3, rendezvous on 127.0.0.1).  The GPU path uses the same
code with NCCL (tests/test_gpu_dist.py covers the kernels on bands)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1605_06399_b200 import dist as icd
import synth


@pytest.mark.parametrize("H", [1, 7, 64, 101, 1000])
@pytest.mark.parametrize("N", [1, 2, 3, 8])
@pytest.mark.parametrize("up,down", [(0, 0), (2, 2), (3, 3), (7, 7), (1, 2)])
def test_partition_and_plan(H, N, up, down):
    try:
        bands = [icd.partition(H, N, k, up, down) for k in range(N)]
    except ValueError:
        assert N > 1 and -(-H // N) < max(up, down) or any(
            min(H, (k + 1) * -(-H // N)) - min(k * -(-H // N), H) < max(up, down) for k in range(N))
        return
    owned = np.zeros(H, int)
    for b in bands:
        owned[b.r0:b.r1] += 1
        assert b.s0 == max(0, b.r0 - up) and b.s1 == min(H, b.r1 + down)
    assert (owned == 1).all()
    # every received range is exactly what the peer sends, from the peer's owned rows
    for b in bands:
        for peer, send, recv in icd.exchange_plan(b):
            pb = bands[peer]
            back = [s for p2, s, r in icd.exchange_plan(pb) if p2 == b.rank]
            assert back and back[0] == recv
            assert pb.r0 <= recv[0] and recv[1] <= pb.r1
            assert b.r0 <= send[0] and send[1] <= b.r1
        got = set(range(b.r0, b.r1))
        for peer, _s, (c, d) in icd.exchange_plan(b):
            got |= set(range(c, d))
        assert got == set(range(b.s0, b.s1))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, H, W, up, down, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    img = synth.uniform_image(5, H, W)
    band = icd.partition(H, world, rank, up, down)
    buf = torch.full((band.buf_rows, W), float("nan"))
    buf[band.own_slice] = torch.from_numpy(img[band.r0:band.r1])
    icd.halo_exchange(buf, band)
    ok = bool(torch.equal(buf, torch.from_numpy(img[band.s0:band.s1])))
    out_q.put((rank, ok, band.s0, band.s1))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,H,up,down", [(2, 37, 2, 2), (3, 50, 3, 3), (2, 16, 7, 7), (3, 31, 1, 2)])
def test_gloo_halo_exchange(world, H, up, down):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, H, 13, up, down, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _, _ in res), res
