"""Host-side cost of run_join steps (cProfile over 5 cfg2 steps after warm-up):
the Python / ctypes work that runs before a step's first kernel is GPU idle
time.   python tools/host_prof.py [cfg2] [threads]"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1207_0145_b200 as P
from paper_1207_0145_b200.core import JoinConfig, Relation

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
threads = int(sys.argv[2]) if len(sys.argv) > 2 else 1
dev = torch.device("cuda", 0)
P.warmup()
r, s, dom = bench.make_inputs(cfg_name)
rd = Relation(torch.from_numpy(r.keys).to(dev), torch.from_numpy(r.payloads).to(dev))
sd = Relation(torch.from_numpy(s.keys).to(dev), torch.from_numpy(s.payloads).to(dev))
cfg = JoinConfig(threads=threads, algorithm="p-mpsm", key_domain=dom)
for _ in range(3):
    P.run_join(rd, sd, cfg)
torch.cuda.synchronize()
# host time to the first launch: wrap the library's first sort entry
from paper_1207_0145_b200 import _lib

lib = _lib.load()
marks = []
for name in ("mpsm_sort_packed", "mpsm_sort_records", "mpsm_sort_packed_segments", "mpsm_sort_records_segments"):
    f = getattr(lib, name)

    def wrap(*a, _f=f, _n=name):
        marks.append((time.perf_counter(), _n))
        return _f(*a)

    setattr(lib, name, wrap)
for _ in range(5):
    marks.clear()
    t0 = time.perf_counter()
    P.run_join(rd, sd, cfg)
    t1 = time.perf_counter()
    first = marks[0][0] - t0 if marks else float("nan")
    print(f"step host wall {1e3 * (t1 - t0):.3f} ms, run_join entry -> first sort call {1e6 * first:.1f} us")
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    P.run_join(rd, sd, cfg)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
st.sort_stats("cumulative").print_stats(40)
