"""Per-phase cycle breakdown of seg::k_scatter (variant built with
MPSM_DBG_TIMING) for the LAST pass of a packed sort of n keys."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["MPSM_LIB"] = os.path.join(ROOT, "build", "variants_dbg", os.environ.get("DBGV", "timing"), "libmpsm_b200.so")
from paper_1207_0145_b200 import _lib, device as D  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 400_000_000
bits = int(sys.argv[3]) if len(sys.argv) > 3 else 27  # 9: one (SP) pass only
packed = (sys.argv[2] if len(sys.argv) > 2 else "packed") == "packed"
dev = torch.device("cuda", 0)
keys = torch.randint(0, 1 << bits, (n,), device=dev, dtype=torch.int64).view(torch.uint64)
pays = torch.randint(0, 1 << 32, (n,), device=dev, dtype=torch.int64).view(torch.uint64)
o = [torch.empty_like(keys) for _ in range(4)]
ovf = torch.zeros(1, dtype=torch.int32, device=dev)
D.ensure_device()
for _ in range(2):
    if packed:
        D.sort_packed(keys, pays, 0, (1 << bits) - 1, bits, o[0], o[1], None, ovf)
    else:
        D.sort_pairs(keys, pays, 0, (1 << bits) - 1, bits, o[0], o[1], o[2], o[3], None)
torch.cuda.synchronize()
L = _lib.load()
ntiles = (n + 4095) // 4096 if (bits <= 9 or not packed) else (n + 8191) // 8192
buf = np.zeros((ntiles, 8), np.int64)
L.mpsm_dbg_seg_ts(buf.ctypes.data_as(ctypes.c_void_p), ntiles)
if os.environ.get("WS"):  # k_scatter_ws: ranker thread 0 (cols 0,1,6,2), writer thread 0 (cols 3,4,5)
    print(f"{'packed' if packed else 'pairs'} tiles={ntiles} (warp-specialised)")
    for nm, a, b in (("ranker wait data", 0, 1), ("ranker load+rank", 1, 6), ("ranker scan+stage", 6, 2),
                     ("writer wait staged", 3, 4), ("writer write", 4, 5)):
        x = buf[:, b] - buf[:, a]
        print(f"  {nm:20s} median {np.median(x):7.0f} mean {np.mean(x):7.0f} p90 {np.percentile(x, 90):7.0f}")
    sys.exit(0)
d = np.diff(buf[:, :6], axis=1)
names = ["wait_data(mbar)", "load+rank+S2", "scan+S3+S4", "stage+S5", "write"]
tot = buf[:, 5] - buf[:, 0]
print(f"{'packed' if packed else 'pairs'} tiles={ntiles} cycles/tile median {np.median(tot):.0f}")
for i, nm in enumerate(names):
    print(f"  {nm:18s} median {np.median(d[:, i]):7.0f} mean {np.mean(d[:, i]):7.0f} p90 {np.percentile(d[:, i], 90):7.0f}")
