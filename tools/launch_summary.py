"""Per-kernel device time over an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python tools/launch_summary.py launches.csv [label]
"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
label = sys.argv[2] if len(sys.argv) > 2 else ""
tot = collections.Counter()
cnt = collections.Counter()
for r in rows:
    name = r[4]
    tot[name] += float(r[14].replace(",", "")) * (1e-3 if r[13] == "ns" else 1.0 if r[13] == "us" else 1e3)
    cnt[name] += 1
all_us = sum(tot.values())
print(f"per-kernel device time over the ncu launch list{(' (' + label + ')') if label else ''}, cold-cache serialised launches")
for name, us in tot.most_common():
    print(f"{us / 1e3:8.3f} ms {cnt[name]:5d} launches {100 * us / all_us:5.1f}%  {name[:90]}")
print(f"{all_us / 1e3:8.3f} ms total")
