"""Per-launch DRAM traffic of one kernel family from an ncu --set full report.

    python tools/ncu_traffic.py rep.ncu-rep kernel_regex algorithmic_bytes_per_step out.json
Sums dram__bytes_read.sum + dram__bytes_write.sum over the captured launches
whose name matches, divides by the launch count, and records it beside the
algorithmic bytes per launch (bench.py reads out.json for roofline.traffic).
"""
import csv
import io
import json
import re
import subprocess
import sys

rep, pat, alg_step, out = sys.argv[1], sys.argv[2], float(sys.argv[3]), sys.argv[4]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
ik, ir, iw, it = (h.index(k) for k in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                        "gpu__time_duration.sum"))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
tscale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}
launches = []
for r in rows[2:]:
    if not re.search(pat, r[ik]):
        continue
    rd = float(r[ir]) * scale[units[ir]]
    wr = float(r[iw]) * scale[units[iw]]
    launches.append({"kernel": r[ik][:80], "dram_read": rd, "dram_write": wr,
                     "duration_s": float(r[it]) * tscale.get(units[it], 1e-9)})
n = len(launches)
res = {"report": rep, "kernel_regex": pat, "launches": n,
       "dram_bytes_per_launch": sum(x["dram_read"] + x["dram_write"] for x in launches) / max(n, 1),
       "algorithmic_bytes_per_launch": alg_step / max(n, 1), "per_launch": launches}
res["traffic_over_algorithmic"] = res["dram_bytes_per_launch"] / max(res["algorithmic_bytes_per_launch"], 1)
json.dump(res, open(out, "w"), indent=1)
print(json.dumps({k: v for k, v in res.items() if k != "per_launch"}, indent=1))
