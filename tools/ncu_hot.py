"""Print the hottest SASS instructions of an ncu report (source page CSV).

    ncu -i rep.ncu-rep --page source --csv --print-source sass > x.csv
    python tools/ncu_hot.py x.csv [N]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr)]
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
print("total samples", tot)
data.sort(key=lambda r: -int(r[idx["Warp Stall Sampling (All Samples)"]] or 0))
for r in data[:n]:
    s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    top = sorted(((int(r[idx[c]] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
    print(f"{s:7d} {100*s/tot:5.1f}%  {r[idx['Address']]:>6} {r[idx['Source']][:60]:60s} " + " ".join(f"{c}={v}" for v, c in top if v))
