"""One FK join (packed) of n_r x 4 n_r on the device -- a small driver for ncu."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1207_0145_b200 as P  # noqa: E402
from paper_1207_0145_b200.core import JoinConfig, KeyDomain, Relation  # noqa: E402

n_r = int(sys.argv[1]) if len(sys.argv) > 1 else 25_000_000
dev = torch.device("cuda", 0)
r = Relation((torch.randperm(n_r, device=dev) + 1).view(torch.uint64),
             torch.randint(0, 1 << 32, (n_r,), device=dev).view(torch.uint64))
s = Relation(torch.randint(1, n_r + 1, (4 * n_r,), device=dev).view(torch.uint64),
             torch.randint(0, 1 << 32, (4 * n_r,), device=dev).view(torch.uint64))
res = P.run_join(r, s, JoinConfig(key_domain=KeyDomain(1, n_r + 1)))
print(res.match_count, res.aggregate_max, hex(res.checksum))
