"""Host-side cost of one run_join (cfg2-sized device inputs): cProfile of
the Python work and the GPU-idle gap between back-to-back joins."""
import cProfile
import os
import pstats
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1207_0145_b200 as P  # noqa: E402
from paper_1207_0145_b200.core import JoinConfig, KeyDomain, Relation  # noqa: E402

n_r = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
threads = int(sys.argv[2]) if len(sys.argv) > 2 else 1
dev = torch.device("cuda", 0)
r = Relation((torch.randperm(n_r, device=dev) + 1).view(torch.uint64),
             torch.randint(0, 1 << 32, (n_r,), device=dev).view(torch.uint64))
s = Relation(torch.randint(1, n_r + 1, (4 * n_r,), device=dev).view(torch.uint64),
             torch.randint(0, 1 << 32, (4 * n_r,), device=dev).view(torch.uint64))
cfg = JoinConfig(threads=threads, key_domain=KeyDomain(1, n_r + 1))
for _ in range(3):
    P.run_join(r, s, cfg)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
tot = 0.0
for _ in range(10):
    res = P.run_join(r, s, cfg)
    tot += res.phase_timings["total"]
e1.record()
torch.cuda.synchronize()
print(f"step {e0.elapsed_time(e1) / 10:.3f} ms, phases t0->join {1e3 * tot / 10:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    P.run_join(r, s, cfg)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
