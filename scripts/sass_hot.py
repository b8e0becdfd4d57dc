"""Top SASS instructions by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
idx = {k: i for i, k in enumerate(h)}
data = [r for r in rows[2:] if len(r) == len(h)]
tot = sum(int(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
print("total samples", tot)
top = sorted(data, key=lambda r: -int(r[idx["Warp Stall Sampling (All Samples)"]] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]
for r in top:
    s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    print(f"{100.0 * s / tot:5.1f}% {r[idx['Address']][-5:]} {r[idx['Source']].strip()[:70]}")
