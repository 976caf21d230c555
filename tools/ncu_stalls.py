"""Summarise an ncu report: duration, DRAM, pipe use, top stall reasons and hottest SASS lines."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                     text=True).stdout.splitlines()))
h, v = raw[0], raw[2]
for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size"]:
    if k in h:
        print(f"{k:60s} {v[h.index(k)]} {raw[1][h.index(k)]}")
st = sorted(((float(v[i]), w) for i, w in enumerate(h) if "issue_stalled" in w and "not_issued" not in w
             and v[i].replace('.', '', 1).isdigit()), reverse=True)[:8]
for x, w in st:
    print(f"  {x:8.0f} {w.replace('smsp__pcsamp_warps_issue_stalled_', '')}")
src = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                                     capture_output=True, text=True).stdout.splitlines()))
hs = src[1]
isrc, iall = hs.index("Source"), hs.index("Warp Stall Sampling (All Samples)")
rows = src[2:]
tot = sum(int(r[iall] or 0) for r in rows)
print("samples", tot)
for n, k, s in sorted(((int(r[iall] or 0), k, r[isrc].strip()[:70]) for k, r in enumerate(rows)), reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 8]:
    print(f"  {n:6d} {100.0 * n / tot:5.1f}% @{k:5d} {s}")
