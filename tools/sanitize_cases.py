"""Small ragged cases exercising every variant of every filter once (for
compute-sanitizer memcheck / racecheck / synccheck runs; see tools/sanitize.sh)."""
import sys

import numpy as np
import torch
sys.path.insert(0, '.')
import paper_1605_06399_b200 as icl  # noqa: E402
import synth  # noqa: E402

dev = torch.device('cuda:0')
for (h, w) in [(61, 53), (130, 517), (9, 300)]:
    img = torch.from_numpy(synth.uniform_image(1, h, w)).to(dev)
    out = torch.empty_like(img)
    mask = torch.empty(h, w, dtype=torch.uint8, device=dev)
    ws = torch.empty(icl.sepconv_workspace_bytes(w, h, 1, 15) // 4 + 1, device=dev)
    for f in ("sepconv", "harris", "nlm"):
        for vid, name in enumerate(icl.variant_names(f)):
            if name.startswith("pm_") and vid % 11:  # a sample of the 288 Table-1 configurations
                continue
            icl.force_variant(f, vid)
            for border in ("constant", "clamp"):
                try:
                    if f == "sepconv":
                        for r in (0, 2, 7):
                            fx = synth.gaussian_taps(r)
                            icl.sepconv(img, out, fx, fx, border, 0.5, workspace=ws)
                    elif f == "harris":
                        icl.harris(img, out, 5, 0.04, border, 0.5, mask=mask, threshold=0.1)
                    else:
                        icl.nlm(img, out, 2, 5, 0.1, border, 0.5)
                except icl.IclError as e:
                    if e.status not in (3, 4):
                        raise
            torch.cuda.synchronize()
        icl.force_variant(f, None)
# more 64x64 tiles than the persistent grid: the tile kernel's cp.async prefetch path
img = torch.from_numpy(synth.uniform_image(2, 1300, 1100)).to(dev)
out = torch.empty_like(img)
for name in ("tile64p_v4", "tile64_v4"):
    icl.force_variant("sepconv", name)
    for border in ("constant", "clamp"):
        for r in (7, 15):
            fx = synth.gaussian_taps(r)
            icl.sepconv(img, out, fx, fx, border, 0.5)
    torch.cuda.synchronize()
icl.force_variant("sepconv", None)
# non-separable uchar convolution: every variant, ragged sizes, both borders, several tiles
for (h, w) in [(61, 53), (130, 517), (300, 200)]:
    u8 = torch.from_numpy(synth.uniform_u8(3, h, w)).to(dev)
    out = torch.empty(h, w, device=dev)
    for vid, name in enumerate(icl.variant_names("conv2d")):
        icl.force_variant("conv2d", vid)
        for border in ("constant", "clamp"):
            for r in (0, 2, 3):
                try:
                    icl.conv2d_u8(u8, out, synth.filter2d(1, r), border, 5.0)
                except icl.IclError as e:
                    if e.status not in (3, 4):
                        raise
        torch.cuda.synchronize()
    icl.force_variant("conv2d", None)
# host-image path (pinned), small bands
import os  # noqa: E402
os.environ["ICL_HOST_CHUNK_ROWS"] = "16"
hs = torch.from_numpy(synth.uniform_image(5, 100, 96)).pin_memory()
hd = torch.empty(100, 96).pin_memory()
icl.sepconv(hs, hd, synth.gaussian_taps(2), synth.gaussian_taps(2), "clamp")
hm = torch.empty(100, 96, dtype=torch.uint8).pin_memory()
icl.harris(hs, hd, 5, 0.04, "clamp", mask=hm, threshold=0.1)
icl.nlm(hs, hd, 2, 5, 0.1, "clamp")
torch.cuda.synchronize()
# every variant through the host path: row bands in the library's exactly-sized staging buffers,
# so a kernel reading rows past its band buffer shows up here (round 2: the tile kernels did)
hs2 = torch.from_numpy(synth.uniform_image(6, 150, 200)).pin_memory()
hd2 = torch.empty(150, 200).pin_memory()
hm2 = torch.empty(150, 200, dtype=torch.uint8).pin_memory()
for f in ("sepconv", "harris", "nlm"):
    for vid, name in enumerate(icl.variant_names(f)):
        if name.startswith("pm_") and vid % 11:
            continue
        icl.force_variant(f, vid)
        for border in ("constant", "clamp"):
            try:
                if f == "sepconv":
                    for r in (2, 9):
                        fx = synth.gaussian_taps(r)
                        icl.sepconv(hs2, hd2, fx, fx, border, 0.5)
                elif f == "harris":
                    icl.harris(hs2, hd2, 5, 0.04, border, 0.5, mask=hm2, threshold=0.1)
                else:
                    icl.nlm(hs2, hd2, 2, 5, 0.1, border, 0.5)
            except icl.IclError as e:
                if e.status not in (3, 4):
                    raise
        torch.cuda.synchronize()
    icl.force_variant(f, None)
del os.environ["ICL_HOST_CHUNK_ROWS"]
# fused smoothing + Harris chain (and its two-pass schedule): ragged sizes, all radii, both borders
for (h, w) in [(61, 52), (130, 516), (300, 200)]:
    img = torch.from_numpy(synth.uniform_image(6, h, w)).to(dev)
    out = torch.empty_like(img)
    mask = torch.empty(h, w, dtype=torch.uint8, device=dev)
    ws = torch.empty(icl.blur_harris_workspace_bytes(w, h, 1, 5) // 4 + 4, device=dev)
    for r in (0, 1, 2, 3):
        fx = synth.gaussian_taps(r)
        for bb, hb in (("constant", "clamp"), ("clamp", "constant")):
            icl.blur_harris(img, out, fx, fx, bb, 0.5, 5, 0.04, hb, 0.25, mask=mask, threshold=0.1)
            icl.blur_harris(img, out, fx, fx, bb, 0.5, 3, 0.04, hb, 0.25, mask=mask, threshold=0.1, workspace=ws)
    torch.cuda.synchronize()
# 3-D volumes: both variants, ragged shapes, radii up to 7, both borders
for shape in [(5, 13, 70), (17, 20, 3)]:
    v = torch.from_numpy(np.stack([synth.uniform_image(7 + z, shape[1], shape[2]) for z in range(shape[0])])).to(dev)
    o = torch.empty_like(v)
    for name in icl.variant_names("sepconv3d"):
        icl.force_variant("sepconv3d", name)
        for r in (0, 1, 3, 7):
            fx = synth.gaussian_taps(r)
            for border in ("constant", "clamp"):
                icl.sepconv3d(v, o, fx, fx, fx, border, 0.5)
        torch.cuda.synchronize()
    icl.force_variant("sepconv3d", None)
# peer paths with neighbours as local device memory (edge kernels reading the neighbour bands)
full = synth.rect_scene(9, 90, 130)
bands = [torch.from_numpy(np.ascontiguousarray(full[a:b])).to(dev) for a, b in ((0, 30), (30, 60), (60, 90))]
for k, (a, b) in enumerate(((0, 30), (30, 60), (60, 90))):
    up = icl.LocalBand(bands[k - 1]) if k > 0 else None
    dn = icl.LocalBand(bands[k + 1]) if k < 2 else None
    o = torch.empty(b - a, 130, device=dev)
    m = torch.empty(b - a, 130, dtype=torch.uint8, device=dev)
    icl.sepconv_peer(bands[k], o, 90, a, up, dn, synth.gaussian_taps(7), synth.gaussian_taps(7), "constant", 0.5)
    icl.harris_peer(bands[k], o, 90, a, up, dn, 7, 0.04, "clamp", 0.0, mask=m, threshold=0.1)
torch.cuda.synchronize()
print("sanitize cases done")
