"""Copy one gpurun evidence round (tools/gpu_round.sh <tag>) into profiles/:
bench line, reference line, pytest summary, ncu launch list with per-kernel shares, ncu --set full
summaries and the NLM SASS histogram, and profiles/ncu_traffic.json from the same captures.

    python tools/collect_round.py r02e
"""
import csv
import json
import os
import subprocess
import sys

tag = sys.argv[1]
G = os.path.join("gpurun_out")
NCU = os.path.join(G, f"ncu_{tag}")
PX = 8 * 4096 * 4096


def last_json(path):
    with open(path) as f:
        lines = [l for l in f.read().splitlines() if l.startswith("{")]
    return lines[-1] if lines else None


for src, dst in ((f"bench_{tag}.json", f"{tag}_bench.jsonl"), (f"ref_{tag}.jsonl", f"{tag}_reference.jsonl")):
    p = os.path.join(G, src)
    if os.path.exists(p) and last_json(p):
        open(os.path.join("profiles", dst), "w").write(last_json(p) + "\n")
log = os.path.join(G, f"pytest_gpu_{tag}.log")
if os.path.exists(log):
    tail = [l for l in open(log).read().splitlines() if "passed" in l or "failed" in l]
    open(os.path.join("profiles", f"{tag}_pytest_gpu.txt"), "w").write((tail[-1] if tail else "") + "\n")

rows = list(csv.reader(open(os.path.join(NCU, "launches.csv"))))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
k, v = h.index("Kernel Name"), h.index("Metric Value")
u = h.index("Metric Unit") if "Metric Unit" in h else None
out = ["ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised) of",
       "  python bench.py --steps 2 --warmup 3 --batch 8 --no-e2e --no-cpu-baseline --no-tune --no-small --no-16k",
       f"(tools/ncu_capture.sh {tag}; the bench's own 8 x 4096^2 launches)", ""]
tot = {}
for r in rows[hi + 1:]:
    if len(r) <= v:
        continue
    val = float(r[v].replace(",", ""))
    unit = r[u] if u is not None else ""
    us = val / 1000 if unit in ("nsecond", "ns") else (val * 1000 if unit in ("msecond", "ms") else val)
    out.append(f"{r[k][:60]:<62}{us:10.2f} us")
    tot[r[k]] = tot.get(r[k], 0) + us
s = sum(tot.values())
out += ["", "share of the step: " + ", ".join(f"{kk.split('(')[0].replace('void ', '')} {100 * vv / s:.1f}%"
                                           for kk, vv in tot.items())]
open(os.path.join("profiles", f"{tag}_launches.txt"), "w").write("\n".join(out) + "\n")
print(out[-1])
reports = {}
for name in ("nlm_sym", "sep_stream", "harris_shfl"):
    rep = os.path.join(NCU, f"full_{name}.ncu-rep")
    if os.path.exists(rep):
        summ = subprocess.run([sys.executable, "tools/ncu_summary.py", rep], capture_output=True, text=True).stdout
        open(os.path.join("profiles", f"{tag}_full_{name}.txt"), "w").write(summ)
        reports[name] = rep
if "nlm_sym" in reports:
    hist = subprocess.run([sys.executable, "tools/sass_hist.py", reports["nlm_sym"], "--px", str(PX), "--label",
                           f"bench launch 8x4096^2 ({tag})"], capture_output=True, text=True).stdout
    open(os.path.join("profiles", f"{tag}_sass_hist_nlm_sym.txt"), "w").write(hist)
flt = {"nlm_sym": "nlm", "sep_stream": "sepconv", "harris_shfl": "harris"}
args = [f"{flt[n]}={p}" for n, p in reports.items()]
subprocess.run([sys.executable, "tools/ncu_traffic.py", "--px", str(PX), "--tag", f"{tag}, tools/ncu_capture.sh {tag}",
                *args], check=True, capture_output=True)
d = json.loads(open(os.path.join("profiles", f"{tag}_bench.jsonl")).read())
print(json.dumps({k: d.get(k) for k in ("value", "ms_per_step", "per_filter_ms")}),
      d["roofline"]["frac"], d.get("small_configs"), d["e2e"]["value"], d.get("clocks"))
