"""Time every conv2d_u8 variant on one 8192^2 image (PAPER.md:594-598 workload), CUDA events,
rotating inputs/outputs larger than L2 between launches."""
import argparse
import json
import sys

import torch

sys.path.insert(0, '.')
import paper_1605_06399_b200 as icl  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument('--size', type=int, default=8192)
ap.add_argument('--radius', type=int, default=2)
ap.add_argument('--reps', type=int, default=20)
a = ap.parse_args()
S = a.size
imgs = [torch.from_numpy(synth.uniform_u8(8 + k, S, S)).cuda() for k in range(2)]
dsts = [torch.empty(S, S, device='cuda') for _ in range(2)]  # 2 x (64 MB + 256 MB) > L2
f = synth.filter2d(8, a.radius)
for name in icl.variant_names('conv2d'):
    icl.force_variant('conv2d', name)
    for k in range(3):
        icl.conv2d_u8(imgs[k & 1], dsts[k & 1], f, 'clamp')
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for k in range(a.reps):
        icl.conv2d_u8(imgs[k & 1], dsts[k & 1], f, 'clamp')
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / a.reps
    n = 2 * a.radius + 1
    print(json.dumps({"variant": name, "us": round(ms * 1000, 1), "GBps": round(S * S * 5 / ms / 1e6, 1),
                      "TFLOPs": round(S * S * 2 * n * n / ms / 1e9, 1)}))
icl.force_variant('conv2d', None)

# traffic baselines with the same byte mix (1 B read + 4 B written per pixel): the HBM roofline of
# a write-dominated kernel is below the 50/50 copy peak of MEASURED_PEAKS.json
for label, fn in (("torch_u8_to_f32_copy", lambda k: dsts[k & 1].copy_(imgs[k & 1])),
                  ("torch_fill_f32", lambda k: dsts[k & 1].fill_(1.0))):
    for k in range(3):
        fn(k)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for k in range(a.reps):
        fn(k)
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / a.reps
    nbytes = S * S * (5 if "copy" in label else 4)
    print(json.dumps({"variant": label, "us": round(ms * 1000, 1), "GBps": round(nbytes / ms / 1e6, 1)}))
