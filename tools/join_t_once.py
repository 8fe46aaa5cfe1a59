"""One FK join (packed) of n_r x 4 n_r split into T private / public runs,
through join_pairs_packed (the engine's P-MPSM runs) -- a driver for ncu."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1207_0145_b200 import _lib, device as D  # noqa: E402

n_r = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
T = int(sys.argv[2]) if len(sys.argv) > 2 else 16
n_s, bits = 4 * n_r, 27
dev = torch.device("cuda", 0)
D.ensure_device()
rk = (torch.randperm(n_r, device=dev) + 1).view(torch.uint64)
rp = torch.randint(0, 1 << 32, (n_r,), device=dev).view(torch.uint64)
sk = torch.randint(1, n_r + 1, (n_s,), device=dev).view(torch.uint64)
sp = torch.randint(0, 1 << 32, (n_s,), device=dev).view(torch.uint64)
ovf = torch.zeros(1, dtype=torch.int32, device=dev)


def srt(k, p):
    o, t = torch.empty_like(k), torch.empty_like(k)
    D.sort_packed(k, p, 1, n_r - 1, bits, o, t, None, ovf)
    return o


R = srt(rk, rp)
cs, cr = n_s // T, n_r // T
S = [srt(sk[i * cs:(i + 1) * cs].contiguous(), sp[i * cs:(i + 1) * cs].contiguous()) for i in range(T)]
Rr = [R[i * cr:(i + 1) * cr] for i in range(T)]
rec = D.join_pairs_packed(Rr, S, bits, 1, False, _lib.MODE_AGGREGATE_MAX)
torch.cuda.synchronize()
print("count", int(rec[:, 0].sum().item()))
