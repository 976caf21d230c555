"""Write a compact text summary of ncu reports (+ the launch list) for profiles/.

usage: python tools/ncu_summary.py OUT.md launches.csv rep1.ncu-rep [rep2 ...]
"""
import collections
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "lts__t_sector_hit_rate.pct", "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return r[0], r[1], r[2]


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[start]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
    t, c = collections.defaultdict(float), collections.Counter()
    for r in rows[start + 1:]:
        if len(r) <= max(ki, vi, ui):
            continue
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        n = r[ki].split("(")[0]
        t[n] += v
        c[n] += 1
    tot = sum(t.values())
    lines = [f"launch list: {sum(c.values())} launches, {tot / 1e3:.3f} ms serialised (cold-cache, ncu)", "",
             "| kernel | launches | total us | share | avg us |", "|---|---|---|---|---|"]
    for n, v in sorted(t.items(), key=lambda x: -x[1]):
        lines.append(f"| {n} | {c[n]} | {v:.1f} | {100 * v / tot:.1f}% | {v / c[n]:.1f} |")
    return lines


def main():
    out, lcsv, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    lines = []
    if lcsv != "-":
        lines += launches(lcsv) + [""]
    for rep in reps:
        h, u, v = raw(rep)
        name = v[h.index("Kernel Name")] if "Kernel Name" in h else rep
        lines += [f"## {rep.split('/')[-1]}", f"kernel: {name.split('(')[0]}", ""]
        for k in KEYS:
            if k in h:
                lines.append(f"    {k:62s} {v[h.index(k)]:>16s} {u[h.index(k)]}")
        st = sorted(((float(v[i]), w) for i, w in enumerate(h) if "pcsamp_warps_issue_stalled" in w
                     and "not_issued" not in w and v[i].replace(".", "", 1).isdigit()), reverse=True)[:8]
        lines.append("    top stall samples: " + ", ".join(
            f"{w.replace('smsp__pcsamp_warps_issue_stalled_', '')}={x:.0f}" for x, w in st))
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
