"""Write profiles/ncu_traffic.json (DRAM bytes per pixel of each hot kernel) from
`ncu --set full` reports of tools/ncu_capture.sh (bench.py --batch B, one
B x 4096^2 launch per filter).  bench.py multiplies bytes_per_px by the pixels
of its own launch to report roofline.traffic.

  python tools/ncu_traffic.py --px 33554432 nlm=gpurun_out/ncu_r01c/full_nlm_box_x2.ncu-rep ...
"""
import argparse
import csv
import io
import json
import os
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("--px", type=int, required=True, help="pixels per captured launch")
ap.add_argument("--tag", default="")
ap.add_argument("reports", nargs="+", help="filter=path.ncu-rep")
a = ap.parse_args()
out = {"_note": ("dram__bytes_read.sum + dram__bytes_write.sum per pixel from one ncu --set full capture per "
                 f"kernel ({a.tag}) of the SAME launch bench.py times (8 x 4096^2 per filter), so "
                 "bytes_per_px x pixels is that launch's DRAM traffic. Reads are the algorithmic 4 B/px (no "
                 "re-reads); writes read up to ~60 MB short because output lines still dirty in the 126 MB L2 "
                 "at kernel end are written back after it (outside the kernel's counters).")}
for spec in a.reports:
    f, path = spec.split("=", 1)
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, val = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, zip(val, units)))

    def num(key):
        v, u = d[key]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
        return float(v.replace(",", "")) * scale
    rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")

    def pct(key):
        return round(float(d[key][0]), 1) if key in d else None
    out[f] = {"bytes_per_px": round((rd + wr) / a.px, 3), "read_bytes_per_px": round(rd / a.px, 3),
              "write_bytes_per_px": round(wr / a.px, 3), "captured_px": a.px, "kernel": d["Kernel Name"][0], "report": os.path.basename(path),
              "fma_pipe_cycles_pct": pct("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
              "issue_active_pct": pct("smsp__issue_active.avg.pct_of_peak_sustained_active"),
              "smem_wavefronts_pct": pct("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
              "mufu_pct": pct("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active")}
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
with open(path, "w") as fh:
    json.dump(out, fh, indent=1)
    fh.write("\n")
print(json.dumps(out, indent=1))
