"""Our record sort (mpsm_sort_records, 3 passes of 9 bits) and packed sort
(pairs in -> records out) of n random 27-bit keys, CUDA-event timed; run next
to tools/cub_yardstick (CUB onesweep SortKeys / SortPairs on the same sizes)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1207_0145_b200 import device as D  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 400_000_000
bits = 27
D.ensure_device()
keys = torch.randint(0, 1 << bits, (n,), device="cuda", dtype=torch.int64).view(torch.uint64)
pays = torch.randint(0, 1 << 32, (n,), device="cuda", dtype=torch.int64).view(torch.uint64)
rec = torch.empty_like(keys)
tmp = torch.empty_like(keys)
ovf = torch.zeros(1, dtype=torch.int32, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for it in range(4):
    ev[0].record()
    D.sort_packed(keys, pays, 0, (1 << bits) - 1, bits, rec, tmp, None, ovf)
    ev[1].record()
    torch.cuda.synchronize()
    print(f"sort_packed n={n}: {ev[0].elapsed_time(ev[1]):.3f} ms")
src = rec.clone()
out = torch.empty_like(rec)
for it in range(4):
    ev[0].record()
    D.sort_records(src, bits, out, tmp)
    ev[1].record()
    torch.cuda.synchronize()
    print(f"sort_records n={n}: {ev[0].elapsed_time(ev[1]):.3f} ms")
