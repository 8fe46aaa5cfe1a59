"""Per-kernel-family device time of one cfg2 run_join (engine path) at a
given thread count -- the ProfScope timers of the library (GPU box):

    python tools/engine_profile.py [threads] [n_r]
"""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1207_0145_b200 as P  # noqa: E402
from paper_1207_0145_b200 import _lib  # noqa: E402
from paper_1207_0145_b200.core import JoinConfig, KeyDomain, Relation  # noqa: E402

t = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n_r = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000_000
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(0)
r = Relation((torch.randperm(n_r, device=dev, generator=g) + 1).view(torch.uint64),
             torch.randint(0, 1 << 32, (n_r,), device=dev, generator=g).view(torch.uint64))
s = Relation(torch.randint(1, n_r + 1, (4 * n_r,), device=dev, generator=g).view(torch.uint64),
             torch.randint(0, 1 << 32, (4 * n_r,), device=dev, generator=g).view(torch.uint64))
cfg = JoinConfig(threads=t, key_domain=KeyDomain(1, n_r + 1))
names = ["seg_count", "seg_scatter_sp", "seg_scatter_pp", "radix_histogram", "dense_check", "dense_tiles", "dense_bounds", "dense_count",
         "dense_join", "merge_partition", "merge"]
for it in range(3):
    P.run_join(r, s, cfg)
torch.cuda.synchronize()
_lib.profile_enable(True)
t0 = time.perf_counter()
res = P.run_join(r, s, cfg)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) * 1e3
tot = 0.0
for k in names:
    ms, n = _lib.profile_read(k)
    tot += ms
    print(f"{k:18s} {ms:7.3f} ms  {n:3d} launches")
_lib.profile_enable(False)
print(f"sum {tot:.3f} ms  wall {wall:.3f} ms  phases {res.phase_timings}")
