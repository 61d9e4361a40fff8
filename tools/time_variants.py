"""Time variants of one filter with CUDA events (median of reps, inputs > L2):
tools/time_variants.py harris|sepconv|nlm [--size S] [--batch B] [--param v] variant..."""
import argparse
import statistics
import sys

import torch

sys.path.insert(0, '.')
import paper_1605_06399_b200 as icl  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument('filter')
ap.add_argument('--size', type=int, default=4096)
ap.add_argument('--batch', type=int, default=8)
ap.add_argument('--param', type=int, default=None, help="harris block / sepconv radius / nlm search radius")
ap.add_argument('--reps', type=int, default=20)
ap.add_argument('variants', nargs='*')
a = ap.parse_intermixed_args()
dev = torch.device('cuda:0')
srcs = [torch.empty(a.batch, a.size, a.size, device=dev) for _ in range(2)]
for i, s in enumerate(srcs):
    icl.fill_uniform(s, 7 + i)
dst = torch.empty_like(srcs[0])
mask = torch.empty(a.batch, a.size, a.size, dtype=torch.uint8, device=dev)
f = a.filter
names = a.variants or [n for n in icl.variant_names(f) if n != "naive_direct"]


def call(src):
    if f == 'harris':
        icl.harris(src, dst, a.param or 5, 0.04, 'clamp', mask=mask, threshold=1.0)
    elif f == 'sepconv':
        t = synth.gaussian_taps(a.param if a.param is not None else 2)
        icl.sepconv(src, dst, t, t, 'constant')
    else:
        icl.nlm(src, dst, 2, a.param or 5, 0.1, 'clamp')


px = a.batch * a.size * a.size
for name in names:
    try:
        icl.force_variant(f, name)
        for i in range(3):
            call(srcs[i % 2])
        torch.cuda.synchronize()
    except Exception as e:  # noqa: BLE001
        print(f"{name:24s} skipped ({e})")
        continue
    ts = []
    for i in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        call(srcs[i % 2])
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    med = statistics.median(ts)
    print(f"{name:24s} median {med:.4f} ms  min {min(ts):.4f} ms  {px / med / 1e6:.3f} Gpx/s", flush=True)
icl.force_variant(f, None)
