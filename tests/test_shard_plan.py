"""The native partition / exchange plan (icl_shard_band, icl_shard_plan,
icl_halo_rows in libicl.so, used by the NCCL sharded calls) equals the
Python plan of paper_1605_06399_b200/dist.py that the gloo tests exercise
with real multi-process exchanges -- host logic only, runs on CPU."""
import pytest

import paper_1605_06399_b200 as icl
from paper_1605_06399_b200 import dist as icd


@pytest.mark.parametrize("H", [1, 7, 64, 101, 1000, 16384])
@pytest.mark.parametrize("N", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("up,down", [(0, 0), (1, 1), (2, 2), (3, 3), (7, 7), (15, 15), (3, 2)])
def test_native_plan_equals_dist(H, N, up, down):
    bands, bad = {}, set()
    for k in range(N):
        try:
            bands[k] = icd.partition(H, N, k, up, down)
        except ValueError:
            bad.add(k)
    for k in bad:  # a band thinner than the halo is rejected natively too
        with pytest.raises(icl.IclError):
            icl.shard_band(H, N, k, up, down)
    if bad:
        return  # the configuration is invalid as a whole
    for k, b in bands.items():
        assert icl.shard_band(H, N, k, up, down) == (b.r0, b.r1, b.s0, b.s1)
        assert icl.shard_plan(H, N, k, up, down) == icd.exchange_plan(b)


@pytest.mark.parametrize("filt,p", [("sepconv", dict(ry=4)), ("harris", dict(block=5)), ("harris", dict(block=2)),
                                    ("nlm", dict(patch_radius=2, search_radius=5))])
def test_native_halo_rows(filt, p):
    args = {"sepconv": (p.get("ry", 0), 0), "harris": (p.get("block", 0), 0),
            "nlm": (p.get("patch_radius", 0), p.get("search_radius", 0))}[filt]
    assert icl.halo_rows_of(filt, *args) == icd.halo_rows(filt, **p)
    assert icl.halo_rows_of("conv2d", 2) == (2, 2)


def test_plan_is_symmetric():
    for H, N, up, down in [(100, 4, 3, 2), (1000, 8, 7, 7), (50, 5, 1, 3)]:
        plans = {k: icl.shard_plan(H, N, k, up, down) for k in range(N)}
        for k, pl in plans.items():
            for peer, send, recv in pl:
                back = [e for e in plans[peer] if e[0] == k]
                assert len(back) == 1 and back[0][1] == recv and back[0][2] == send
