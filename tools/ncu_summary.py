"""Summarise an ncu report: key throughput/occupancy metrics + DRAM bytes.

    python tools/ncu_summary.py rep.ncu-rep [more.ncu-rep ...]
"""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Registers Per Thread", "Achieved Occupancy",
        "Theoretical Occupancy", "Grid Size", "Block Size", "Dynamic Shared Memory Per Block", "Issue Slots Busy",
        "L2 Hit Rate", "L1/TEX Hit Rate", "Executed Ipc Active"]


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


for rep in sys.argv[1:]:
    print("==", rep)
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "details", "--csv"]))))
    hdr = rows[0]
    seen = set()
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        name = d.get("Metric Name")
        if name in WANT and (d.get("Kernel Name"), name) not in seen:
            seen.add((d.get("Kernel Name"), name))
            print(f"  {name:34s} {d['Metric Value']} {d['Metric Unit']}")
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    h, u, v = raw[0], raw[1], raw[2]
    for key in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
        if key in h:
            i = h.index(key)
            print(f"  {key:34s} {v[i]} {u[i]}")
