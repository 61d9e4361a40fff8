"""Executed-SASS instruction histogram per output pixel of one kernel, from an
`ncu --set full --import-source on` report (per-instruction "Thread Instructions
Executed", summed by opcode; FFMA2/FADD2/FMUL2 counted as one instruction each).

    python tools/sass_hist.py report.ncu-rep --px N [--label name]

N = output pixels of the captured launch.  Prints lane-instructions per pixel by
opcode (predicated-on), the FP32 lane-operations per pixel (packed ops count 2),
and the shared-memory wavefronts per pixel (the bound of the NLM kernels).
"""
import argparse
import collections
import csv
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("report")
ap.add_argument("--px", type=float, required=True)
ap.add_argument("--label", default="")
ap.add_argument("--top", type=int, default=24)
a = ap.parse_args()
raw = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
kname = rows[0][1] if rows and len(rows[0]) > 1 else "?"
hdr = rows[1]
ix_src = hdr.index("Source")
ix_thr = hdr.index("Predicated-On Thread Instructions Executed")
ix_wf = hdr.index("L1 Wavefronts Shared") if "L1 Wavefronts Shared" in hdr else None
by = collections.Counter()
wf = 0.0
for r in rows[2:]:
    if len(r) <= ix_thr:
        continue
    src = r[ix_src].strip()
    if not src:
        continue
    toks = src.split()
    op = toks[0]
    if op.startswith("@"):
        op = toks[1] if len(toks) > 1 else op
    base = op.split(".")[0]
    try:
        n = float(r[ix_thr].replace(",", ""))
    except ValueError:
        continue
    by[base] += n
    if ix_wf is not None:
        try:
            wf += float(r[ix_wf].replace(",", ""))
        except ValueError:
            pass
tot = sum(by.values())
fp_ops = sum(v * (2 if k in ("FFMA2", "FADD2", "FMUL2") else 1) for k, v in by.items()
             if k in ("FFMA", "FADD", "FMUL", "FFMA2", "FADD2", "FMUL2"))
print(f"kernel: {kname}  {a.label}")
print(f"output pixels per launch: {a.px:.0f}")
print(f"lane-instructions per pixel (predicated-on): {tot / a.px:.2f}")
print(f"FP32 lane-operations per pixel (FFMA/FADD/FMUL, packed x2): {fp_ops / a.px:.2f}")
if ix_wf is not None:
    print(f"shared-memory wavefronts per pixel: {wf / a.px:.3f}")
print("opcode            lane-instr/px   share")
for k, v in by.most_common(a.top):
    print(f"  {k:14s} {v / a.px:12.3f}   {100 * v / tot:5.1f}%")
