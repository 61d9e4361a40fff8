"""Summarise an ncu --set full report: timing, throughput, pipes, stalls, smem.

    python tools/ncu_summary.py report.ncu-rep [--kernel regex]
Prints a compact text block (committed under profiles/ as evidence).
"""
import csv
import io
import re
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput %"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "pipe fma %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "pipe fma cycles %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "pipe alu %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "pipe lsu %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "pipe xu (MUFU) %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefronts %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__occupancy_limit_registers", "occupancy limit (regs, blocks)"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock (Hz)"),
]
STALLS = "smsp__average_warps_issue_stalled_"


def main():
    rep = sys.argv[1]
    kre = sys.argv[3] if len(sys.argv) > 3 and sys.argv[2] == "--kernel" else None
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = d.get("Kernel Name", "?")
        if kre and not re.search(kre, name):
            continue
        print(f"kernel: {name[:120]}")
        print(f"  grid {d.get('Grid Size', '?')} block {d.get('Block Size', '?')}")
        for k, label in KEYS:
            if k in d:
                print(f"  {label:34s} {d[k]} {u.get(k, '')}")
        st = sorted(((float(v), k[len(STALLS):].replace("_per_issue_active.ratio", ""))
                     for k, v in d.items() if k.startswith(STALLS) and k.endswith("per_issue_active.ratio")
                     and v not in ("", "n/a")), reverse=True)
        print("  top stalls (warps per issue): " + ", ".join(f"{n}={v:.2f}" for v, n in st[:6]))




def launches(csv_path):
    """Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: share per kernel."""
    rows = [r for r in csv.reader(open(csv_path)) if r]
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = {}
    for r in rows[start + 1:]:
        if len(r) <= vi:
            continue
        name = re.sub(r"\(.*", "", r[ki])
        v = float(r[vi].replace(",", ""))
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
        n, t = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, t + v * scale)
    tot = sum(t for _, t in agg.values())
    print(f"{'kernel':60s} {'launches':>8s} {'total us':>12s} {'avg us':>10s} {'share':>7s}")
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name[:60]:60s} {n:8d} {t:12.1f} {t / n:10.1f} {100 * t / tot:6.1f}%")


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--launches":
        launches(sys.argv[2])
    else:
        main()
