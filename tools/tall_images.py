import torch, numpy as np, sys
sys.path.insert(0, '.')
import paper_1605_06399_b200 as icl, synth
H, W = 70001, 40
img = torch.rand(H, W, device='cuda')
out = torch.empty_like(img)
mask = torch.empty(H, W, dtype=torch.uint8, device='cuda')
u8 = (torch.rand(H, W, device='cuda') * 255).to(torch.uint8)
fx = synth.gaussian_taps(2)
for f, call in [("sepconv", lambda: icl.sepconv(img, out, fx, fx, "clamp")),
                ("harris", lambda: icl.harris(img, out, 5, 0.04, "clamp", mask=mask, threshold=0.1)),
                ("nlm", lambda: icl.nlm(img, out, 2, 5, 0.1, "clamp")),
                ("conv2d", lambda: icl.conv2d_u8(u8, out, synth.filter2d(1, 2), "clamp"))]:
    for vid, name in enumerate(icl.variant_names(f)):
        icl.force_variant(f, vid)
        try:
            call(); torch.cuda.synchronize(); r = "ok"
        except icl.IclError as e:
            r = f"IclError {e.status}: {str(e)[:80]}"
        except Exception as e:
            r = f"{type(e).__name__}: {str(e)[:80]}"
        if r != "ok": print(f, name, r)
    icl.force_variant(f, None)
    try:
        call(); torch.cuda.synchronize(); print(f, "default ok", icl.variant_names(f)[icl.last_variant(f)])
    except Exception as e:
        print(f, "default FAIL", str(e)[:100])
