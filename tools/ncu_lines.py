"""Aggregate ncu SASS-level stall samples per CUDA source line.

    ncu -i rep.ncu-rep --page source --csv --print-source sass > x.csv
    python tools/ncu_lines.py x.csv lib.so kernel_substring [N]
Maps each SASS offset (address - function base) to the source line given by
`nvdisasm -g` on the cubin extracted from the shared library.
"""
import collections
import csv
import glob
import os
import re
import subprocess
import sys
import tempfile

csv_path, lib, kname = sys.argv[1], os.path.abspath(sys.argv[2]), sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
rows = list(csv.reader(open(csv_path)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr)]
addrs = [int(r[ix["Address"]], 16) for r in data]
base = min(addrs)
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, capture_output=True)
line_of = {}
srcs = {}
for cub in glob.glob(os.path.join(tmp, "*.cubin")):
    out = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
    cur_fn = None
    cur_line = None
    for ln in out.splitlines():
        m = re.match(r"\.text\.(\S+):", ln) or re.match(r"//-+ \.text\.(\S+) -+", ln)
        if m:
            cur_fn = m.group(1)
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur_line = (os.path.basename(m.group(1)), int(m.group(2)))
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur_fn and kname in cur_fn and cur_line:
            line_of[int(m.group(1), 16)] = cur_line
            srcs.setdefault(cur_line[0], None)
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = collections.Counter()
why = collections.defaultdict(collections.Counter)
tot = 0
for r, a in zip(data, addrs):
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    tot += s
    key = line_of.get(a - base, ("?", 0))
    agg[key] += s
    for c in stall_cols:
        why[key][c[6:]] += int(r[ix[c]] or 0)
print("total samples", tot, "mapped lines", len(agg), "offsets", len(line_of))
for key, s in agg.most_common(top):
    reasons = " ".join(f"{k}={v}" for k, v in why[key].most_common(3) if v)
    print(f"{s:7d} {100*s/tot:5.1f}%  {key[0]}:{key[1]:<5d} {reasons}")
