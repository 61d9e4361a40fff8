"""Time every variant of every filter on a given shape (CUDA events, median).

    python tools/variant_sweep.py [--batch 8] [--size 4096] [--reps 5] [--filters sepconv,harris,nlm]

Prints one JSON line per (filter, variant): median ms, Mpx/s and the roofline
fraction (HBM for sepconv/Harris against MEASURED_PEAKS.json, FP32 for NLM).
Inputs exceed L2 at the default shape; smaller shapes get an L2 flush.
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--size", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--filters", default="sepconv,harris,nlm")
    ap.add_argument("--radius", type=int, default=2)
    ap.add_argument("--all", action="store_true", help="include the 288 pm_* Table-1 configurations")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    B, S = a.batch, a.size
    src = torch.empty(B, S, S, device=dev)
    icl.fill_uniform(src, 7)
    dst = torch.empty_like(src)
    mask = torch.empty(B, S, S, dtype=torch.uint8, device=dev)
    ws = torch.empty(icl.sepconv_workspace_bytes(S, S, B, 15) // 4 + 1, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if B * S * S * 8 < (512 << 20) else None
    hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    px = B * S * S
    fx = synth.gaussian_taps(a.radius)
    calls = {
        "sepconv": lambda: icl.sepconv(src, dst, fx, fx, "constant", workspace=ws),
        "harris": lambda: icl.harris(src, dst, 5, 0.04, "clamp", mask=mask, threshold=1.0),
        "nlm": lambda: icl.nlm(src, dst, 2, 5, 0.1, "clamp"),
    }
    if "sepconv" in a.filters:  # HBM ceiling on the same buffers: torch copy (read + write)
        ts = []
        for _ in range(a.reps):
            if flush is not None:
                flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dst.copy_(src)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        print(json.dumps({"filter": "copy", "variant": "torch_copy", "ms": ms, "gbs": 8 * px / ms / 1e6,
                          "frac_hbm": 8 * px / ms / 1e6 / hbm}), flush=True)
    for f in a.filters.split(","):
        for vid, name in enumerate(icl.variant_names(f)):
            if name.startswith("naive") and S * S * B > (1 << 24) and f == "nlm":
                continue
            if name.startswith("pm_") and not a.all:
                continue
            icl.force_variant(f, vid)
            try:
                calls[f]()
            except icl.IclError as e:
                print(json.dumps({"filter": f, "variant": name, "skipped": str(e)}))
                continue
            torch.cuda.synchronize()
            ts = []
            for _ in range(a.reps):
                if flush is not None:
                    flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                calls[f]()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = statistics.median(ts)
            rec = {"filter": f, "variant": name, "ms": ms, "mpx_s": px / ms / 1e3}
            if f == "sepconv":
                rec["gbs"] = 8 * px / ms / 1e6
                rec["frac_hbm"] = rec["gbs"] / hbm
            elif f == "harris":
                rec["gbs"] = 9 * px / ms / 1e6
                rec["frac_hbm"] = rec["gbs"] / hbm
            else:
                flop = (1694 if "box" in name else 9559) * px
                rec["tflops"] = flop / ms / 1e9
                rec["frac_fp32"] = rec["tflops"] / 74.45
            print(json.dumps(rec), flush=True)
        icl.force_variant(f, None)


if __name__ == "__main__":
    main()
