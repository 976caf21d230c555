"""Print the hottest SASS lines (warp-stall samples) of an ncu --page source --csv export."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
src = hdr.index("Source")
samp = hdr.index("Warp Stall Sampling (All Samples)")
exe = hdr.index("Instructions Executed")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[samp]), int(r[exe]), r[src].strip()[:90], r[0][-5:]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for d in sorted(data, reverse=True)[:n]:
    print("%7d %5.1f%% exe %9d  %s  %s" % (d[0], 100 * d[0] / tot, d[1], d[3], d[2]))
print("total samples", tot, "instructions", sum(d[1] for d in data))
