"""Per-phase cycle breakdown of the onesweep pass (variant built with
MPSM_DBG_TIMING).  Runs ONE pass-sized sort on n keys and prints, for the
last sort pass, median/mean cycles per phase across tiles."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["MPSM_LIB"] = os.path.join(ROOT, "build", "variants_dbg", "timing", "libmpsm_b200.so")
from paper_1207_0145_b200 import _lib, device as D  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 400_000_000
bits = int(sys.argv[2]) if len(sys.argv) > 2 else 27
tile = int(sys.argv[3]) if len(sys.argv) > 3 else 8192
dev = torch.device("cuda", 0)
keys = torch.randint(0, 1 << bits, (n,), device=dev, dtype=torch.int64).view(torch.uint64)
pays = torch.arange(n, device=dev, dtype=torch.int64).view(torch.uint64)
ok, op, tk, tp = (torch.empty_like(keys) for _ in range(4))
D.ensure_device()
for _ in range(2):
    D.sort_pairs(keys, pays, 0, (1 << bits) - 1, bits, ok, op, tk, tp, None)
torch.cuda.synchronize()
L = _lib.load()
L.mpsm_dbg_phase_ts.restype = ctypes.c_int
ntiles = (n + tile - 1) // tile
buf = np.zeros((ntiles, 8), np.int64)
L.mpsm_dbg_phase_ts(buf.ctypes.data_as(ctypes.c_void_p), ntiles)
names = ["load_keys", "rank", "scan+publish+offsets", "lookback", "positions+stage_keys", "write k+p", ]
d = np.diff(buf[:, :7], axis=1)
print(f"tiles={ntiles}  total cycles/tile: median {np.median(buf[:,6]-buf[:,0]):.0f} mean {np.mean(buf[:,6]-buf[:,0]):.0f}")
for i, nm in enumerate(names):
    print(f"  {nm:24s} median {np.median(d[:, i]):8.0f}  mean {np.mean(d[:, i]):8.0f}  p90 {np.percentile(d[:, i], 90):8.0f}")
