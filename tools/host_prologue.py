"""Where the host time before a step's first kernel goes: perf_counter marks
around the pieces of run_join that run before the first sort launch (after
warm-up, cfg2).   python tools/host_prologue.py [cfg2]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1207_0145_b200 as P
from paper_1207_0145_b200 import _lib, device as D, engine as E
from paper_1207_0145_b200.core import JoinConfig, Relation

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
dev = torch.device("cuda", 0)
P.warmup()
r, s, dom = bench.make_inputs(cfg_name)
rd = Relation(torch.from_numpy(r.keys).to(dev), torch.from_numpy(r.payloads).to(dev))
sd = Relation(torch.from_numpy(s.keys).to(dev), torch.from_numpy(s.payloads).to(dev))
cfg = JoinConfig(threads=1, algorithm="p-mpsm", key_domain=dom)
marks = []


def mark(tag):
    marks.append((time.perf_counter(), tag))


def wrap(obj, name):
    f = getattr(obj, name)

    def w(*a, **k):
        mark(name + ">")
        out = f(*a, **k)
        mark(name + "<")
        return out

    setattr(obj, name, w)


for o, n in ((E, "_prepare"), (E.JoinContext, "__init__"), (E.JoinContext, "sort_public"), (E.JoinContext, "_upload"),
             (E.JoinContext, "_tmp"), (E.JoinContext, "_store_for"), (D, "sort_packed"), (D, "new_bad_flag"),
             (D, "workspace"), (D, "ensure_device"), (E, "chunk_bounds"), (E.JoinContext, "stage_private"),
             (E.JoinContext, "sort_private_whole"), (E.JoinContext, "cut_partitions"), (E.JoinContext, "join"),
             (E.JoinContext, "fetch_status"), (E.JoinContext, "finalize"), (D, "join_pairs_packed")):
    wrap(o, n)
lib = _lib.load()
for n in ("mpsm_sort_packed", "mpsm_sort_packed_dense", "mpsm_sort_workspace_bytes", "mpsm_join_pairs_packed_hint",
          "mpsm_join_pairs_packed"):
    wrap(lib, n)
for _ in range(3):
    P.run_join(rd, sd, cfg)
torch.cuda.synchronize()
for _ in range(3):
    marks.clear()
    mark("entry")
    P.run_join(rd, sd, cfg)
    t0 = marks[0][0]
    out = []
    for t, tag in marks:
        out.append(f"{tag}@{1e6 * (t - t0):.0f}")
    print(" ".join(out))
