"""Host-resident images through the C ABI (include/icl.h, "host images"): the
library streams row bands through the GPU (H2D / compute / D2H pipelined on
three streams).  Results must equal the device-resident call -- bit for bit
for sepconv and Harris (band splits share the per-output fp32 order), to the
NLM box-sum tolerance for NLM -- for pinned and pageable buffers, mixed
host/device operands, batches, ragged last bands and caller-supplied bands."""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1605_06399_b200 as icl  # noqa: E402

DEV = torch.device("cuda:0")


def host(a, pinned=True):
    t = torch.from_numpy(np.ascontiguousarray(a))
    return t.pin_memory() if pinned else t.clone()


@pytest.fixture(params=["37", "4096"], ids=["small_bands", "default_bands"])
def chunk_rows(request, monkeypatch):
    if request.param != "4096":
        monkeypatch.setenv("ICL_HOST_CHUNK_ROWS", request.param)
    else:
        monkeypatch.delenv("ICL_HOST_CHUNK_ROWS", raising=False)
    return int(request.param)


@pytest.mark.parametrize("pinned", [True, False])
@pytest.mark.parametrize("border", ["constant", "clamp"])
def test_sepconv_host_equals_device(chunk_rows, pinned, border):
    b, h, w = 3, 203, 260
    imgs = np.stack([synth.uniform_image(60 + i, h, w) for i in range(b)])
    fx = synth.gaussian_taps(4)
    ref = torch.empty(b, h, w, device=DEV)
    icl.sepconv(torch.from_numpy(imgs).to(DEV), ref, fx, fx, border, 0.25)
    src, dst = host(imgs, pinned), host(np.full((b, h, w), np.nan, np.float32), pinned)
    h0, d0 = icl.transfer_bytes()
    icl.sepconv(src, dst, fx, fx, border, 0.25)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(dst.numpy(), ref.cpu().numpy())
    h1, d1 = icl.transfer_bytes()
    assert d1 - d0 == b * h * w * 4
    assert h1 - h0 >= b * h * w * 4  # + halo rows per band


@pytest.mark.parametrize("where", ["src_host", "dst_host"])
def test_sepconv_mixed_operands(chunk_rows, where):
    h, w = 150, 300
    img = synth.uniform_image(61, h, w)
    fx = synth.gaussian_taps(2)
    ref = torch.empty(h, w, device=DEV)
    icl.sepconv(torch.from_numpy(img).to(DEV), ref, fx, fx, "clamp")
    if where == "src_host":
        src, dst = host(img), torch.full((h, w), float("nan"), device=DEV)
    else:
        src, dst = torch.from_numpy(img).to(DEV), host(np.zeros((h, w), np.float32))
    icl.sepconv(src, dst, fx, fx, "clamp")
    torch.cuda.synchronize()
    np.testing.assert_array_equal(dst.cpu().numpy(), ref.cpu().numpy())


def test_sepconv_host_with_band(chunk_rows):
    """A caller band on host buffers: rows [40, 140) of a 200-row image."""
    H, W, r = 200, 130, 3
    img = synth.uniform_image(62, H, W)
    fx = synth.gaussian_taps(r)
    full = torch.empty(H, W, device=DEV)
    icl.sepconv(torch.from_numpy(img).to(DEV), full, fx, fx, "constant", 0.5)
    src = host(img[40 - r:140 + r])
    dst = host(np.zeros((100, W), np.float32))
    icl.sepconv(src, dst, fx, fx, "constant", 0.5, band=(H, 40 - r, 40))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(dst.numpy(), full.cpu().numpy()[40:140])


@pytest.mark.parametrize("block", [3, 5])
def test_harris_host_equals_device(chunk_rows, block):
    b, h, w = 2, 190, 250
    imgs = np.stack([synth.rect_scene(70 + i, h, w, n_rect=15, noise=0.01) for i in range(b)])
    ref, refm = torch.empty(b, h, w, device=DEV), torch.empty(b, h, w, dtype=torch.uint8, device=DEV)
    icl.harris(torch.from_numpy(imgs).to(DEV), ref, block, 0.04, "clamp", mask=refm, threshold=0.5)
    src = host(imgs)
    resp = host(np.zeros((b, h, w), np.float32))
    mask = torch.full((b, h, w), 7, dtype=torch.uint8).pin_memory()
    icl.harris(src, resp, block, 0.04, "clamp", mask=mask, threshold=0.5)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(resp.numpy(), ref.cpu().numpy())
    np.testing.assert_array_equal(mask.numpy(), refm.cpu().numpy())


def test_nlm_host_equals_device(chunk_rows):
    b, h, w = 2, 120, 140
    imgs = np.stack([synth.rect_scene(80 + i, h, w, n_rect=10, noise=0.0866) for i in range(b)])
    ref = torch.empty(b, h, w, device=DEV)
    icl.nlm(torch.from_numpy(imgs).to(DEV), ref, 2, 5, 0.1, "clamp")
    src, dst = host(imgs), host(np.zeros((b, h, w), np.float32))
    icl.nlm(src, dst, 2, 5, 0.1, "clamp")
    torch.cuda.synchronize()
    np.testing.assert_allclose(dst.numpy(), ref.cpu().numpy(), rtol=0, atol=2e-5)


def test_host_call_is_ordered_on_the_callers_stream(monkeypatch):
    """Events on the caller's stream bracket the whole host call; a kernel
    queued after it on that stream sees its output."""
    monkeypatch.setenv("ICL_HOST_CHUNK_ROWS", "64")
    h, w = 512, 512
    img = synth.uniform_image(63, h, w)
    fx = synth.gaussian_taps(2)
    s = torch.cuda.Stream()
    src, mid = host(img), host(np.zeros((h, w), np.float32))
    out = torch.empty(h, w, device=DEV)
    with torch.cuda.stream(s):
        icl.sepconv(src, mid, fx, fx, "clamp", stream=s)       # host -> host
        icl.sepconv(mid, out, fx, fx, "clamp", stream=s)       # host -> device, reads mid after the first call
    s.synchronize()
    d = torch.from_numpy(img).to(DEV)
    r1, r2 = torch.empty_like(d), torch.empty_like(d)
    icl.sepconv(d, r1, fx, fx, "clamp")
    icl.sepconv(r1, r2, fx, fx, "clamp")
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out.cpu().numpy(), r2.cpu().numpy())


def test_tune_rejects_host_images():
    t = host(np.zeros((16, 16), np.float32))
    with pytest.raises(ValueError):
        icl.tune("sepconv", t, t, taps_x=[1.0], taps_y=[1.0])


def test_host_calls_from_several_streams(monkeypatch):
    """Three host calls issued on three user streams share the library's
    staging sets; their bands interleave on the copy / compute streams and
    every result must still equal the device call (staging-set reuse waits
    on the set's previous users across calls)."""
    monkeypatch.setenv("ICL_HOST_CHUNK_ROWS", "16")
    h, w = 300, 200
    imgs = [synth.uniform_image(90 + i, h, w) for i in range(3)]
    fx = synth.gaussian_taps(3)
    refs = []
    for im in imgs:
        r = torch.empty(h, w, device=DEV)
        icl.sepconv(torch.from_numpy(im).to(DEV), r, fx, fx, "clamp")
        refs.append(r.cpu().numpy())
    streams = [torch.cuda.Stream() for _ in range(3)]
    for rep in range(3):
        srcs = [host(im) for im in imgs]
        dsts = [host(np.full((h, w), np.nan, np.float32)) for _ in imgs]
        for s, a, b in zip(streams, srcs, dsts):
            icl.sepconv(a, b, fx, fx, "clamp", stream=s)
        torch.cuda.synchronize()
        for b, r in zip(dsts, refs):
            np.testing.assert_array_equal(b.numpy(), r)


def test_mixed_filters_from_several_streams(monkeypatch):
    """sepconv / Harris+mask / NLM host calls on three streams: their staging
    layouts differ (halo rows, mask region) yet share the rotating sets."""
    monkeypatch.setenv("ICL_HOST_CHUNK_ROWS", "24")
    h, w = 160, 180
    a, b, c = (synth.rect_scene(95 + i, h, w, n_rect=12, noise=0.05) for i in range(3))
    fx = synth.gaussian_taps(2)
    ra, rb, rc = (torch.empty(h, w, device=DEV) for _ in range(3))
    rm = torch.empty(h, w, dtype=torch.uint8, device=DEV)
    icl.sepconv(torch.from_numpy(a).to(DEV), ra, fx, fx, "constant")
    icl.harris(torch.from_numpy(b).to(DEV), rb, 5, 0.04, "clamp", mask=rm, threshold=0.2)
    icl.nlm(torch.from_numpy(c).to(DEV), rc, 2, 5, 0.1, "clamp")
    streams = [torch.cuda.Stream() for _ in range(3)]
    for rep in range(3):
        oa, ob, oc = (host(np.full((h, w), np.nan, np.float32)) for _ in range(3))
        om = torch.full((h, w), 9, dtype=torch.uint8).pin_memory()
        ha, hb, hc = host(a), host(b), host(c)  # host inputs must outlive the asynchronous calls
        icl.sepconv(ha, oa, fx, fx, "constant", stream=streams[0])
        icl.harris(hb, ob, 5, 0.04, "clamp", mask=om, threshold=0.2, stream=streams[1])
        icl.nlm(hc, oc, 2, 5, 0.1, "clamp", stream=streams[2])
        torch.cuda.synchronize()
        np.testing.assert_array_equal(oa.numpy(), ra.cpu().numpy())
        np.testing.assert_array_equal(ob.numpy(), rb.cpu().numpy())
        np.testing.assert_array_equal(om.numpy(), rm.cpu().numpy())
        np.testing.assert_allclose(oc.numpy(), rc.cpu().numpy(), rtol=0, atol=2e-5)
