"""One packed (or pairs) sort of n random 27-bit keys -- a small driver for ncu."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1207_0145_b200 import device as D  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
mode = sys.argv[2] if len(sys.argv) > 2 else "packed"
bits = 27
keys = torch.randint(0, 1 << bits, (n,), device="cuda", dtype=torch.int64).view(torch.uint64)
pays = torch.randint(0, 1 << 32, (n,), device="cuda", dtype=torch.int64).view(torch.uint64)
o = [torch.empty_like(keys) for _ in range(4)]
ovf = torch.zeros(1, dtype=torch.int32, device="cuda")
D.ensure_device()
if mode == "packed":
    D.sort_packed(keys, pays, 0, (1 << bits) - 1, bits, o[0], o[1], None, ovf)
else:
    D.sort_pairs(keys, pays, 0, (1 << bits) - 1, bits, o[0], o[1], o[2], o[3], None)
torch.cuda.synchronize()
print("ok")
