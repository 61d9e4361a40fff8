"""Drive Harris variants for ncu: tools/prof_harris.py [--size S] [--batch B] [--block B] variant..."""
import argparse
import sys

import torch

sys.path.insert(0, '.')
import paper_1605_06399_b200 as icl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument('--size', type=int, default=4096)
ap.add_argument('--batch', type=int, default=2)
ap.add_argument('--block', type=int, default=5)
ap.add_argument('variants', nargs='+')
a = ap.parse_args()
dev = torch.device('cuda:0')
src = torch.empty(a.batch, a.size, a.size, device=dev)
icl.fill_uniform(src, 7)
dst = torch.empty_like(src)
mask = torch.empty(a.batch, a.size, a.size, dtype=torch.uint8, device=dev)
for name in a.variants:
    icl.force_variant('harris', name)
    for _ in range(2):
        icl.harris(src, dst, a.block, 0.04, 'clamp', mask=mask, threshold=1.0)
torch.cuda.synchronize()
