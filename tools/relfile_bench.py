"""Throughput of the relation-file input path (GPU box).

    python tools/relfile_bench.py [n] [dir]

Writes an MPSMREL1 file of n tuples (16 B each) from host columns (timed: a
rewrite of the page-cache file) and times, with the file in the page cache:
read_relation (native parallel pread -> numpy columns), load_relation (-> SoA
columns in HBM) and a plain numpy reader of the same layout (np.fromfile + column split, what the reference's bench.read_relation
does).  Median of 3 after one warm-up read.
"""
import os
import statistics
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1207_0145_b200 import datagen, relfile  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
d = sys.argv[2] if len(sys.argv) > 2 else "/tmp"
path = os.path.join(d, f"mpsm_relbench_{os.getpid()}.mpsmrel")
rd, _, _ = datagen.gen_fk_device(n, 1, seed=5, device="cuda")
r = relfile.Relation(rd.keys.cpu().numpy(), rd.payloads.cpu().numpy())  # host columns
del rd
relfile.write_relation(r, path)  # first write: file pages allocated
t0 = time.perf_counter()
relfile.write_relation(r, path)  # rewrite of a page-cache file
w_s = time.perf_counter() - t0
gb = 16 * n / 1e9


def numpy_reader(p):
    rec = np.fromfile(p, dtype="<u8", offset=16)
    return rec[0::2].copy(), rec[1::2].copy()


def timed(fn):
    fn()
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    return statistics.median(ts), out


t_np, (k_np, p_np) = timed(lambda: numpy_reader(path))
t_rd, rel_h = timed(lambda: relfile.read_relation(path))
t_ld, rel_d = timed(lambda: relfile.load_relation(path))
ok = (np.array_equal(rel_h.keys, k_np) and np.array_equal(rel_h.payloads, p_np)
      and torch.equal(rel_d.keys.cpu(), torch.from_numpy(k_np)) and np.array_equal(r.keys, k_np))
os.remove(path)
print(f"n={n:,} ({gb:.2f} GB) in {d}: write {gb / w_s:.1f} GB/s; page-cache reads: numpy reader {gb / t_np:.1f} GB/s, "
      f"read_relation (host columns) {gb / t_rd:.1f} GB/s, load_relation (HBM columns) {gb / t_ld:.1f} GB/s; "
      f"identical={ok}; host threads {os.cpu_count()}")
