"""Time mpsm_sort_pairs of every variant under build/variants (GPU box).

    python tools/sort_variants_run.py [n] [bits]
"""
import ctypes
import glob
import os
import subprocess
import sys

n = int(sys.argv[1]) if len(sys.argv) > 1 else 400_000_000
bits = int(sys.argv[2]) if len(sys.argv) > 2 else 27
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, ctypes, torch
sys.path.insert(0, os.environ["ROOT"])
from paper_1207_0145_b200 import _lib, device as D
n, bits = int(sys.argv[1]), int(sys.argv[2])
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev); g.manual_seed(1)
keys = torch.randint(0, 1 << bits, (n,), device=dev, generator=g, dtype=torch.int64).view(torch.uint64)
pays = torch.arange(n, device=dev, dtype=torch.int64).view(torch.uint64)
ok = torch.empty_like(keys); op = torch.empty_like(pays); tk = torch.empty_like(keys); tp = torch.empty_like(pays)
D.ensure_device()
ovf = torch.zeros(1, dtype=torch.int32, device=dev)
for packed in (False, True):
    res = []
    for it in range(4):
        _lib.profile_enable(True)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record()
        if packed:
            D.sort_packed(keys, pays, 0, (1 << bits) - 1, bits, ok, tk, None, ovf)
        else:
            D.sort_pairs(keys, pays, 0, (1 << bits) - 1, bits, ok, op, tk, tp, None)
        b.record(); torch.cuda.synchronize()
        res.append((a.elapsed_time(b), _lib.profile_read("seg_scatter"), _lib.profile_read("seg_count"),
                    [_lib.profile_read(x) for x in ("seg_scatter_ss", "seg_scatter_sp", "seg_scatter_pp")]))
    srt = (ok >> (64 - bits) if packed else ok).view(torch.int64) if False else ok.view(torch.int64)
    if packed:
        srt = torch.bitwise_right_shift(ok.view(torch.int64), 64 - bits) & ((1 << bits) - 1)
    sorted_ok = bool((srt[1:] >= srt[:-1]).all())
    best = min(res)
    ms, (os_ms, os_n), (h_ms, h_n), per = best
    lo = _lib.load().mpsm_dbg_lane_ordered()
    print(f"lo={lo} {os.environ['VNAME']:10s} {'packed' if packed else 'pairs ':6s} total {ms:7.3f} ms  scatter {os_ms:7.3f} ms/{os_n} passes"
          f" = {os_ms/os_n:6.3f} ms/pass  count {h_ms:6.3f} ms/{h_n}  sorted={sorted_ok}  "
          + " ".join(f"{nm}={m:.3f}/{c}" for nm, (m, c) in zip(("ss", "sp", "pp"), per) if c), flush=True)
'''
for lib in sorted(glob.glob(os.path.join(ROOT, "build", "variants", "*", "libmpsm_b200.so"))):
    name = os.path.basename(os.path.dirname(lib))
    env = dict(os.environ, MPSM_LIB=lib, ROOT=ROOT, VNAME=name)
    r = subprocess.run([sys.executable, "-c", CHILD, str(n), str(bits)], env=env, capture_output=True, text=True,
                       timeout=300)
    print(r.stdout.strip() or (name + " FAILED " + r.stderr[-800:]), flush=True)
