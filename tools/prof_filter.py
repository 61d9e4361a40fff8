"""Run one filter variant a few times on the bench shape (for ncu captures).
    python tools/prof_filter.py <filter> <variant> [batch]"""
import sys
import torch
sys.path.insert(0, '.')
import paper_1605_06399_b200 as icl  # noqa: E402
import synth  # noqa: E402
f, v = sys.argv[1], sys.argv[2]
B = int(sys.argv[3]) if len(sys.argv) > 3 else 8
dev = torch.device('cuda:0')
src = torch.empty(B, 4096, 4096, device=dev)
icl.fill_uniform(src, 7)
dst = torch.empty_like(src)
mask = torch.empty(B, 4096, 4096, dtype=torch.uint8, device=dev)
fx = synth.gaussian_taps(2)
icl.force_variant(f, v)
for _ in range(3):
    if f == 'sepconv':
        icl.sepconv(src, dst, fx, fx, 'constant')
    elif f == 'harris':
        icl.harris(src, dst, 5, 0.04, 'clamp', mask=mask, threshold=1.0)
    else:
        icl.nlm(src, dst, 2, 5, 0.1, 'clamp')
torch.cuda.synchronize()
