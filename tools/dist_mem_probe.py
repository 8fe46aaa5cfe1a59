"""Peak device memory of ONE rank of a multi-GPU bench workload, measured on
one GPU: the rank-`me` position shards of DIST_CONFIGS[name] over G GPUs are
generated and joined through the distributed path at world size 1 (all of the
rank's R stays local: the same run, record and workspace sizes a rank of the
G-GPU job holds, without the peers), and the checker's lookup is built as
bench_main builds it.  The result is not compared (at world size 1 the shard
is not the whole workload).

    torchrun --nproc-per-node 1 tools/dist_mem_probe.py [cfg5] [G=2] [me=0]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

from paper_1207_0145_b200 import distributed as DD
from paper_1207_0145_b200.core import JoinConfig

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
G = int(sys.argv[2]) if len(sys.argv) > 2 else 2
me = int(sys.argv[3]) if len(sys.argv) > 3 else 0
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
dist.init_process_group("nccl", device_id=dev)
r, s, dom, n_r, n_s = DD._dist_inputs(name, G, me, dev)
gb = 1 / 1e9
print(f"{name} over {G} GPUs, rank {me}: shard |R|={r.cardinality:,} |S|={s.cardinality:,}; "
      f"inputs {torch.cuda.memory_allocated() * gb:.1f} GB", flush=True)
kind = DD.DIST_CONFIGS[name][2]
if kind == "fk":  # the checker's footprint (bench_main runs it before any join buffer exists)
    lookup = torch.zeros(n_r + 1, dtype=torch.int64, device=dev)
    lookup[r.keys.view(torch.int64)] = r.payloads.view(torch.int64)
    print(f"with the checker's lookup: {torch.cuda.max_memory_allocated() * gb:.1f} GB peak", flush=True)
    del lookup
torch.cuda.empty_cache()
torch.cuda.reset_peak_memory_stats()
cfg = JoinConfig(threads=1, key_domain=dom)
be = DD.CudaBackend()
for i in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = DD.run_join_distributed(r, s, cfg, backend=be)
    e1.record()
    torch.cuda.synchronize()
    print(f"join {i}: {e0.elapsed_time(e1):.1f} ms, count {res.match_count:,}; peak allocated "
          f"{torch.cuda.max_memory_allocated() * gb:.1f} GB, reserved {torch.cuda.memory_reserved() * gb:.1f} GB "
          f"of {torch.cuda.get_device_properties(0).total_memory * gb:.1f} GB", flush=True)
DD.ipc_close_all()
dist.destroy_process_group()
