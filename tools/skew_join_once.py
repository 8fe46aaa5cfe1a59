"""One cfg4-shaped join (negatively correlated skew, duplicates on both sides)
generated on the device: n_r x 4 n_r, key domain [1, 2^32); R 80 % of its
keys in the lowest 20 % of the domain, S 80 % in the highest 20 %.  Times the
join kernels (CUDA events via the library's profile scopes); a small driver
for ncu too.   python tools/skew_join_once.py [n_r] [reps]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1207_0145_b200 import _lib, device as D  # noqa: E402

n_r = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
n_s = 4 * n_r
dev = torch.device("cuda", 0)
D.ensure_device()
g = torch.Generator(device=dev)
g.manual_seed(0)
HI = (1 << 32) - 1
cut_lo, cut_hi = int(0.2 * HI), int(0.8 * HI)


def keys(n, hot_lo, hot_hi, cold_lo, cold_hi):
    hot = torch.rand(n, device=dev, generator=g) < 0.8
    a = torch.randint(hot_lo, hot_hi, (n,), device=dev, generator=g)
    b = torch.randint(cold_lo, cold_hi, (n,), device=dev, generator=g)
    return torch.where(hot, a, b)


rk = keys(n_r, 1, cut_lo, cut_lo, HI).view(torch.uint64)
sk = keys(n_s, cut_hi, HI, 1, cut_hi).view(torch.uint64)
rp = torch.randint(0, 1 << 32, (n_r,), device=dev, generator=g).view(torch.uint64)
sp = torch.randint(0, 1 << 32, (n_s,), device=dev, generator=g).view(torch.uint64)
bits = 32
ovf = torch.zeros(1, dtype=torch.int32, device=dev)


def srt(k, p):
    o, t = torch.empty_like(k), torch.empty_like(k)
    D.sort_packed(k, p, 1, HI - 1, bits, o, t, None, ovf)
    return o


R, S = srt(rk, rp), srt(sk, sp)
del rk, rp, sk, sp
for it in range(reps):
    _lib.profile_enable(True)
    rec = D.join_pairs_packed([R], [S], bits, 1, False, 0)
    torch.cuda.synchronize()
    names = ("merge", "merge_partition", "dense_check", "dense_join")
    ms = {k: round(_lib.profile_read(k)[0], 3) for k in names}
    _lib.profile_enable(False)
    print(f"iter {it}: count {int(rec[0, 0].item())} {ms}", flush=True)
