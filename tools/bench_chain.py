"""Time the fused smoothing + Harris chain (icl_blur_harris) against the two
library calls it replaces, on the suite shape (8 x 4096^2, inputs > L2).

    python tools/bench_chain.py [--batch 8] [--size 4096] [--radius 2] [--reps 10]
Prints one JSON line: median ms of each path, Mpx/s, achieved GB/s at the
chain's algorithmic 9 B/px (read 4 + R 4 + mask 1) and the fraction of the
measured HBM peak (MEASURED_PEAKS.json).
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1605_06399_b200 as icl  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--size", type=int, default=4096)
ap.add_argument("--radius", type=int, default=2)
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
dev = torch.device("cuda:0")
B, S = a.batch, a.size
src = torch.empty(B, S, S, device=dev)
icl.fill_uniform(src, 5)
blurred, R = torch.empty_like(src), torch.empty_like(src)
mask = torch.empty(B, S, S, dtype=torch.uint8, device=dev)
f = synth.gaussian_taps(a.radius)


def two():
    icl.sepconv(src, blurred, f, f, "constant")
    icl.harris(blurred, R, 5, 0.04, "clamp", mask=mask, threshold=1.0)


def one():
    icl.blur_harris(src, R, f, f, "constant", 0.0, 5, 0.04, "clamp", mask=mask, threshold=1.0)


ws = torch.empty(icl.blur_harris_workspace_bytes(S, S, B, 5) // 4 + 4, device=dev)


def one_ws():
    icl.blur_harris(src, R, f, f, "constant", 0.0, 5, 0.04, "clamp", mask=mask, threshold=1.0, workspace=ws)


def timeit(fn):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


t2, t1, tw = timeit(two), timeit(one), timeit(one_ws)
px = B * S * S
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6535.1
gbs = 9 * px / (t1 * 1e-3) / 1e9
print(json.dumps({"workload": f"blur r={a.radius} + Harris B=5 on {B} x {S}^2", "two_calls_ms": t2, "fused_ms": t1,
                  "speedup": t2 / t1, "api_two_pass_ms": tw, "fused_mpx_s": px / (t1 * 1e-3) / 1e6, "fused_gbs_9B": gbs,
                  "frac_hbm": gbs / peak}))
