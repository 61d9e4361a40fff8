"""The filter calls only enqueue work on the caller's stream (no host sync,
no allocation on the default dispatch path), so a pipeline of them can be
captured once in a CUDA graph and replayed -- the B200 answer to
launch-bound small images (BASELINE.json configs[0..2]).  Replays must equal
the eager calls bit for bit."""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1605_06399_b200 as icl  # noqa: E402

DEV = torch.device("cuda:0")


def test_capture_and_replay_all_filters():
    a = torch.from_numpy(synth.uniform_image(1, 512, 512)).to(DEV)
    h = torch.from_numpy(synth.rect_scene(2, 2048, 2048, noise=0.01)).to(DEV)
    n = torch.from_numpy(synth.rect_scene(3, 1024, 1024, noise=0.0866)).to(DEV)
    u8 = torch.from_numpy(synth.uniform_u8(4, 600, 640)).to(DEV)
    fx, f2 = synth.gaussian_taps(2), synth.filter2d(4, 2)
    outs = [torch.empty_like(a), torch.empty_like(h), torch.empty_like(n), torch.empty(600, 640, device=DEV)]
    mask = torch.empty(2048, 2048, dtype=torch.uint8, device=DEV)

    def pipeline(st):
        icl.sepconv(a, outs[0], fx, fx, "constant", stream=st)
        icl.harris(h, outs[1], 5, 0.04, "clamp", mask=mask, threshold=1.0, stream=st)
        icl.nlm(n, outs[2], 2, 5, 0.1, "clamp", stream=st)
        icl.conv2d_u8(u8, outs[3], f2, "clamp", stream=st)

    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        pipeline(s)  # eager warm-up (function attributes set outside the capture)
    s.synchronize()
    ref = [o.clone() for o in outs] + [mask.clone()]
    for o in outs:
        o.fill_(float("nan"))
    mask.fill_(7)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        pipeline(s)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    for got, want in zip(outs + [mask], ref):
        np.testing.assert_array_equal(got.cpu().numpy(), want.cpu().numpy())


@pytest.mark.parametrize("variant", ["pm_w32x8_c1x1_blk_l1_u4", "pm_w16x8_c2x1_iwg_l1_u4"])
def test_dependent_chain_with_programmatic_launch(variant):
    """The small-image sepconv kernels are launched with programmatic dependent launch (the next grid
    may start before the previous one ends; it waits in griddepcontrol.wait before touching memory).
    A chain in which every call reads the previous call's output -- and writes the buffer the call
    before it read -- must equal the same chain with a host synchronisation after every call, eagerly
    and replayed as a CUDA graph, bit for bit."""
    icl.force_variant("sepconv", variant)
    try:
        a = torch.from_numpy(synth.uniform_image(11, 512, 512)).to(DEV)
        fx = synth.gaussian_taps(2)
        bufs = [a.clone(), torch.empty_like(a), torch.empty_like(a)]
        order = [(0, 1), (1, 2), (2, 0), (0, 1), (1, 2), (2, 0), (0, 1)]  # ping-pong through 3 buffers

        def chain(st, sync):
            for i, j in order:
                icl.sepconv(bufs[i], bufs[j], fx, fx, "constant", stream=st)
                if sync:
                    st.synchronize()

        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            chain(s, True)
        s.synchronize()
        ref = bufs[1].clone()
        bufs[0].copy_(a)
        torch.cuda.synchronize()
        with torch.cuda.stream(s):
            chain(s, False)
        s.synchronize()
        assert torch.equal(bufs[1], ref)
        g = torch.cuda.CUDAGraph()
        bufs[0].copy_(a)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            chain(s, False)
        bufs[0].copy_(a)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(bufs[1], ref)
        assert icl.variant_names("sepconv")[icl.last_variant("sepconv")] == variant
    finally:
        icl.force_variant("sepconv", None)
