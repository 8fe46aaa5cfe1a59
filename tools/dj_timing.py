"""Per-tile cycle timeline of k_dense_join (variant built with MPSM_DBG_TIMING,
python tools/variants.py timing:MPSM_DBG_TIMING=1 -> build/variants/timing):
FK join n_r x 4 n_r, sorted by the library, packed records."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("MPSM_LIB", os.path.join(ROOT, "build", "variants", "timing", "libmpsm_b200.so"))
from paper_1207_0145_b200 import _lib, device as D  # noqa: E402

n_r = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
n_s = 4 * n_r
dev = torch.device("cuda", 0)
D.ensure_device()
rk = (torch.randperm(n_r, device=dev) + 1).view(torch.uint64)
rp = torch.randint(0, 1 << 32, (n_r,), device=dev).view(torch.uint64)
sk = torch.randint(1, n_r + 1, (n_s,), device=dev).view(torch.uint64)
sp = torch.randint(0, 1 << 32, (n_s,), device=dev).view(torch.uint64)
bits = 27
ovf = torch.zeros(1, dtype=torch.int32, device=dev)
def srt(k, p):
    o, t = torch.empty_like(k), torch.empty_like(k)
    D.sort_packed(k, p, 1, n_r - 1, bits, o, t, None, ovf)
    return o
R, S = srt(rk, rp), srt(sk, sp)
for _ in range(2):
    rec = D.join_pairs_packed([R], [S], bits, 1, False, 0)
torch.cuda.synchronize()
print("count", int(rec[0, 0].item()))
L = _lib.load()
nt = 1 << 20
buf = np.zeros((nt, 8), np.int64)
L.mpsm_dbg_dj_ts(buf.ctypes.data_as(ctypes.c_void_p), nt)
buf = buf[(buf[:, 6] > 0) & (buf[:, 2] > 0)]
print("tiles", len(buf))
def st(name, v):
    print(f"  {name:34s} median {np.median(v):8.0f} mean {np.mean(v):8.0f} p10 {np.percentile(v, 10):8.0f} p90 {np.percentile(v, 90):8.0f}")
st("producer wait empty (1-0)", buf[:, 1] - buf[:, 0])
st("producer place+issue (2-1)", buf[:, 2] - buf[:, 1])
st("issue -> consumer w0 sees full (4-2)", buf[:, 4] - buf[:, 2])
st("consumer w0 wait full (4-3)", buf[:, 4] - buf[:, 3])
st("consumer w0 compute (5-4)", buf[:, 5] - buf[:, 4])
st("last warp done - w0 full (6-4)", buf[:, 6] - buf[:, 4])
st("producer start -> last warp done (6-0)", buf[:, 6] - buf[:, 0])
