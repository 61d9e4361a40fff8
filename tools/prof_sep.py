"""Drive one sepconv variant for ncu: tools/prof_sep.py [--radius R] [--size S] [--batch B] variant..."""
import argparse
import sys

import torch

sys.path.insert(0, '.')
import paper_1605_06399_b200 as icl  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument('--radius', type=int, default=2)
ap.add_argument('--size', type=int, default=4096)
ap.add_argument('--batch', type=int, default=8)
ap.add_argument('variants', nargs='+')
a = ap.parse_args()
dev = torch.device('cuda:0')
src = torch.empty(a.batch, a.size, a.size, device=dev)
icl.fill_uniform(src, 7)
dst = torch.empty_like(src)
fx = synth.gaussian_taps(a.radius)
for name in a.variants:
    icl.force_variant('sepconv', name)
    for _ in range(3):
        icl.sepconv(src, dst, fx, fx, 'constant')
torch.cuda.synchronize()
