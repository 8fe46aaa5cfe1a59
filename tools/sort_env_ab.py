"""A/B of a run-time switch of the packed sort (GPU box).

    python tools/sort_env_ab.py VAR v1,v2 [n] [bits]

Runs mpsm_sort_packed (in-tree library) in one child process per value of
the environment variable VAR on the same seeded input, prints per-kernel
times and a fingerprint of the sorted records (they must agree bit for bit).
"""
import os
import subprocess
import sys

var, vals = sys.argv[1], sys.argv[2].split(",")
n = int(sys.argv[3]) if len(sys.argv) > 3 else 400_000_000
bits = int(sys.argv[4]) if len(sys.argv) > 4 else 27
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, torch
sys.path.insert(0, os.environ["ROOT"])
from paper_1207_0145_b200 import _lib, device as D
n, bits = int(sys.argv[1]), int(sys.argv[2])
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev); g.manual_seed(1)
keys = torch.randint(1, 1 << bits, (n,), device=dev, generator=g, dtype=torch.int64).view(torch.uint64)
pays = torch.randint(0, 1 << 32, (n,), device=dev, generator=g, dtype=torch.int64).view(torch.uint64)
ok = torch.empty_like(keys); tk = torch.empty_like(keys)
D.ensure_device()
ovf = torch.zeros(1, dtype=torch.int32, device=dev)
res = []
for it in range(5):
    _lib.profile_enable(True)
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    D.sort_packed(keys, pays, 0, (1 << bits) - 1, bits, ok, tk, None, ovf)
    b.record(); torch.cuda.synchronize()
    res.append((a.elapsed_time(b), _lib.profile_read("seg_scatter"), _lib.profile_read("seg_count"),
                _lib.profile_read("seg_scatter_sp"), _lib.profile_read("seg_scatter_pp"), _lib.profile_read("seg_hist_all")))
v = ok.view(torch.int64)
k = torch.bitwise_right_shift(v, 64 - bits) & ((1 << bits) - 1)
srt = bool((k[1:] >= k[:-1]).all())
w = torch.arange(1, n + 1, device=dev, dtype=torch.int64)
fp = (int(v.sum().item()) & (2**64 - 1), int((v * w).sum().item()) & (2**64 - 1))
ms, sc, cn, sp, pp, ha = min(res)
print(f"{os.environ['VAR']}={os.environ[os.environ['VAR']]} total {ms:7.3f} ms  scatter {sc[0]:6.3f}/{sc[1]}"
      f"  count {cn[0]:6.3f}/{cn[1]}  hist_all {ha[0]:6.3f}  sp {sp[0]:6.3f}  pp {pp[0]:6.3f}/{pp[1]}  sorted={srt} fp={fp[0]:016x}:{fp[1]:016x}",
      flush=True)
'''
for v in vals:
    env = dict(os.environ, ROOT=ROOT, VAR=var, **{var: v})
    r = subprocess.run([sys.executable, "-c", CHILD, str(n), str(bits)], env=env, capture_output=True, text=True,
                       timeout=240)
    print(r.stdout.strip() or (f"{var}={v} FAILED " + r.stderr[-1500:]), flush=True)
