"""Single packed sort vs the same array as S equal segments (the T>1 public
sort), per kernel family (GPU box):  python tools/segsort_ab.py [n] [bits] [S,...]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1207_0145_b200 import _lib, device as D  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 400_000_000
bits = int(sys.argv[2]) if len(sys.argv) > 2 else 27
segs = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "1,2,4,16").split(",")]
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(1)
keys = torch.randint(1, 1 << bits, (n,), device=dev, generator=g, dtype=torch.int64).view(torch.uint64)
pays = torch.randint(0, 1 << 32, (n,), device=dev, generator=g, dtype=torch.int64).view(torch.uint64)
out, tmp = torch.empty_like(keys), torch.empty_like(keys)
D.ensure_device()
ovf = torch.zeros(1, dtype=torch.int32, device=dev)
bad = D.new_bad_flag(dev)
names = ["seg_count", "seg_scatter_sp", "seg_scatter_pp"]
for S in segs:
    best = None
    for it in range(4):
        _lib.profile_enable(True)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        if S == 1:
            D.sort_packed(keys, pays, 0, (1 << bits) - 1, bits, out, tmp, bad, ovf)
        else:
            off = [n * s // S for s in range(S + 1)]
            D.sort_packed_segments(keys, pays, off, 0, (1 << bits) - 1, bits, out, tmp, bad, ovf)
        b.record()
        torch.cuda.synchronize()
        r = (a.elapsed_time(b),) + tuple(_lib.profile_read(k)[0] for k in names)
        best = r if best is None or r[0] < best[0] else best
    print(f"S={S:3d} total {best[0]:7.3f} ms  " + "  ".join(f"{k} {v:6.3f}" for k, v in zip(names, best[1:])),
          flush=True)
