"""Time the merge join (packed FK 100M x 400M) of every variant library under
build/variants (GPU box): python tools/merge_variants_run.py"""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, torch
sys.path.insert(0, os.environ["ROOT"])
from paper_1207_0145_b200 import _lib, device as D
n_r, n_s, bits = 100_000_000, 400_000_000, 27
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
T = int(os.environ.get("TJOIN", "1"))
R = srt(rk, rp)
if T == 1:
    S = [srt(sk, sp)]
    Rr = [R]
else:  # T public chunks sorted separately, R cut into T key ranges (P-MPSM's runs)
    cs = n_s // T
    S = [srt(sk[i * cs:(i + 1) * cs].contiguous(), sp[i * cs:(i + 1) * cs].contiguous()) for i in range(T)]
    cr = n_r // T
    Rr = [R[i * cr:(i + 1) * cr] for i in range(T)]
del rk, rp, sk, sp
best = None
for it in range(4):
    _lib.profile_enable(True)
    rec = D.join_pairs_packed(Rr, S, bits, 1, False, 0)
    torch.cuda.synchronize()
    names = ("merge", "merge_partition", "dense_check", "dense_tiles", "dense_join")
    ms = tuple(_lib.profile_read(k)[0] for k in names)
    best = ms if best is None or sum(ms) < sum(best) else best
print(f"{os.environ['VNAME']:12s} T={T} " + "  ".join(f"{k} {v:.3f}" for k, v in zip(names, best)) +
      f"  total {sum(best):.3f} ms  count={int(rec[:, 0].sum().item())}")
'''
libs = sorted(glob.glob(os.path.join(ROOT, "build", "variants", "*", "libmpsm_b200.so")))
if os.environ.get("INTREE"):
    libs = [os.path.join(ROOT, "paper_1207_0145_b200", "libmpsm_b200.so")]
for lib in libs:
    name = os.environ.get("INTREE") or os.path.basename(os.path.dirname(lib))
    for tj in os.environ.get("TJOINS", "1").split(","):
        env = dict(os.environ, MPSM_LIB=lib, ROOT=ROOT, VNAME=name, TJOIN=tj)
        r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=300)
        print(r.stdout.strip() or (name + " FAILED " + r.stderr[-800:]), flush=True)
