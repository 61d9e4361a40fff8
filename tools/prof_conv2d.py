"""Drive conv2d_u8 variants for ncu: tools/prof_conv2d.py [--size S] [--radius r] variant..."""
import argparse
import sys

import torch

sys.path.insert(0, '.')
import paper_1605_06399_b200 as icl  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument('--size', type=int, default=8192)
ap.add_argument('--radius', type=int, default=2)
ap.add_argument('variants', nargs='+')
a = ap.parse_args()
img = torch.from_numpy(synth.uniform_u8(8, a.size, a.size)).cuda()
dst = torch.empty(a.size, a.size, device='cuda')
f = synth.filter2d(8, a.radius)
for name in a.variants:
    icl.force_variant('conv2d', name)
    for _ in range(2):
        icl.conv2d_u8(img, dst, f, 'clamp')
torch.cuda.synchronize()
