"""Instructions executed per CUDA source line (ncu SASS source page + nvdisasm -g).

    python tools/ncu_inst_lines.py x.csv lib.so kernel_substring [N]
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
for cub in glob.glob(os.path.join(tmp, "*.cubin")):
    out = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
    cur_fn = cur_line = None
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
agg = collections.Counter()
tot = 0
for r, a in zip(data, addrs):
    n = int(r[ix["Instructions Executed"]] or 0)
    tot += n
    agg[line_of.get(a - base, ("?", 0))] += n
print("warp instructions executed", tot)
for key, n in agg.most_common(top):
    print(f"{n:12d} {100*n/tot:5.1f}%  {key[0]}:{key[1]}")
