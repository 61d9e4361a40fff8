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
