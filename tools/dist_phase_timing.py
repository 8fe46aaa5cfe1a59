"""Host-side phase times of run_join_distributed (run under torchrun; at one
rank it measures the protocol's own overhead against the single-GPU engine)."""
import os
import sys
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1207_0145_b200.core import JoinConfig, KeyDomain  # noqa: E402
from paper_1207_0145_b200.distributed import CudaBackend, fk_shard_device, run_join_distributed  # noqa: E402

local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
G, me = dist.get_world_size(), dist.get_rank()
n_r, n_s = 100_000_000 * G, 400_000_000 * G
r, s = fk_shard_device(n_r, n_s, me, G, 0, torch.device("cuda", local))
cfg = JoinConfig(threads=G, key_domain=KeyDomain(1, n_r + 1))
be = CudaBackend()
for it in range(4):
    tm = {}
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = run_join_distributed(r, s, cfg, backend=be, timings=tm)
    torch.cuda.synchronize()
    if me == 0:
        trace = tm.pop("trace", None)
        print(f"iter {it}: wall {1e3 * (time.perf_counter() - t0):.2f} ms  " +
              "  ".join(f"{k} {1e3 * v:.2f}" for k, v in tm.items()), flush=True)
        if trace:  # MPSM_DIST_TRACE=1: host timeline of the protocol
            print("   " + "  ".join(f"{w} @{ms:.2f}" for w, ms in trace), flush=True)
dist.destroy_process_group()
