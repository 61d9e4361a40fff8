"""Time icl_sepconv3d on a 128 x 512 x 512 fp32 volume (radii 1..7, clamp):
median ms, Mvoxel/s and achieved GB/s at the algorithmic 8 B/voxel against
MEASURED_PEAKS.json.   python tools/bench_sep3d.py [--depth 128] [--size 512]"""
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
ap.add_argument("--depth", type=int, default=128)
ap.add_argument("--size", type=int, default=512)
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
src = torch.empty(a.depth, a.size, a.size, device="cuda")
icl.fill_uniform(src, 1)
out = torch.empty_like(src)
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6535.1
nvox = src.numel()
for r in (1, 2, 3, 5, 7):
    f = synth.gaussian_taps(r)
    for name in icl.variant_names("sepconv3d"):
        icl.force_variant("sepconv3d", name)
        for _ in range(2):
            icl.sepconv3d(src, out, f, f, f, "clamp")
        ts = []
        for _ in range(a.reps if name != "naive_direct" else 2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            icl.sepconv3d(src, out, f, f, f, "clamp")
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        gbs = 8 * nvox / (ms * 1e-3) / 1e9
        print(json.dumps({"r": r, "variant": name, "ms": ms, "mvox_s": nvox / (ms * 1e-3) / 1e6, "gbs": gbs,
                          "frac_hbm": gbs / peak, "flop_per_voxel": 6 * (2 * r + 1)}))
icl.force_variant("sepconv3d", None)
