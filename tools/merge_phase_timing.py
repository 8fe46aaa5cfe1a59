"""Per-phase cycle breakdown of k_merge<0> (variant built with MPSM_DBG_TIMING):
join of n_r x n_s FK inputs generated on the device, sorted by the library."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["MPSM_LIB"] = os.path.join(ROOT, "build", "variants_dbg", "timing", "libmpsm_b200.so")
from paper_1207_0145_b200 import _lib, device as D  # noqa: E402

n_r, n_s = 100_000_000, 400_000_000
dev = torch.device("cuda", 0)
rk = (torch.randperm(n_r, device=dev) + 1).view(torch.uint64)
rp = torch.randint(0, 1 << 32, (n_r,), device=dev).view(torch.uint64)
sk = torch.randint(1, n_r + 1, (n_s,), device=dev).view(torch.uint64)
sp = torch.randint(0, 1 << 32, (n_s,), device=dev).view(torch.uint64)
D.ensure_device()
bits = 27
packed = (sys.argv[1] if len(sys.argv) > 1 else "packed") == "packed"
ovf = torch.zeros(1, dtype=torch.int32, device=dev)
def srt(k, p):
    o = [torch.empty_like(k) for _ in range(4)]
    if packed:
        D.sort_packed(k, p, 1, n_r - 1, bits, o[0], o[1], None, ovf)
    else:
        D.sort_pairs(k, p, 1, n_r - 1, bits, o[0], o[1], o[2], o[3], None)
    return o[0], o[1]
rk, rp = srt(rk, rp)
sk, sp = srt(sk, sp)
for _ in range(2):
    if packed:
        rec = D.join_pairs_packed([rk], [sk], bits, 1, False, 0)
    else:
        rec = D.join_pairs([(rk, rp)], [(sk, sp)], False, 0)
torch.cuda.synchronize()
print("count", int(rec[0, 0].item()))
L = _lib.load()
ntiles = min((n_r + n_s) // 1920 + 1, 1 << 20)
buf = np.zeros((ntiles, 6), np.int64)
L.mpsm_dbg_mj_ts(buf.ctypes.data_as(ctypes.c_void_p), ntiles)
buf = buf[buf[:, 5] > 0]
d = np.diff(buf, axis=1)
names = ["S1+fetch+flush", "wait_data", "mergepath_search", "phase1+sync", "phase2"]
print("tiles", len(buf), "cycles/tile median", np.median(buf[:, 5] - buf[:, 0]))
for i, nm in enumerate(names):
    print(f"  {nm:18s} median {np.median(d[:, i]):8.0f} mean {np.mean(d[:, i]):8.0f} p90 {np.percentile(d[:, i], 90):8.0f}")
