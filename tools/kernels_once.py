"""One launch each of the non-headline kernels at 100M tuples (uniform
27-bit keys, 32-bit payloads) -- a small driver for ncu:
    k_radix_hist        private histogram, 1024 buckets (P-MPSM T > 1)
    k_onesweep          partition scatter into the reference arena, 16 parts
                        (mpsm_scatter_chunk / partition.scatter)
    k_scatter_ws<SP,T>  partition straight into packed records, 8 parts
                        (mpsm_partition_records, the multi-GPU partition)
    k_check_sorted      the device Run order check
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1207_0145_b200 import device as D  # noqa: E402

n, w = 100_000_000, 27
dev = torch.device("cuda", 0)
D.ensure_device()
keys = torch.randint(1, 1 << w, (n,), device=dev).view(torch.uint64)
pays = torch.randint(0, 1 << 32, (n,), device=dev).view(torch.uint64)
lower, span_m1 = 0, (1 << w) - 1
hist = torch.zeros(1024, dtype=torch.int64, device=dev)
bad = D.new_bad_flag(dev)
D.radix_histogram(keys, lower, span_m1, w - 10, 1024, hist, bad)
sp = torch.from_numpy(np.repeat(np.arange(16, dtype=np.int32), 64)).to(dev)
counts = np.zeros(16, np.int64)
np.add.at(counts, sp.cpu().numpy(), hist.cpu().numpy())
cur = torch.from_numpy(np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int64)).to(dev)
ak, ap = torch.empty_like(keys), torch.empty_like(pays)
written = torch.zeros(16, dtype=torch.int64, device=dev)
D.scatter_chunk(keys, pays, lower, w - 10, sp, 1024, 16, cur, ak, ap, written)
rec = torch.empty_like(keys)
ovf = torch.zeros(1, dtype=torch.int32, device=dev)
sp8 = torch.from_numpy(np.repeat(np.arange(8, dtype=np.int32), 128)).to(dev)
D.partition_records(keys, pays, lower, span_m1, w, w - 10, sp8, 8, rec, bad, ovf)
srt = torch.sort(keys.view(torch.int64))[0].view(torch.uint64)
print("sorted", D.is_sorted(srt), "written", int(written.sum().item()), "bad", int(bad.item()))
