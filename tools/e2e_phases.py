"""GPU-event phase times of end-to-end cfg2 joins from pinned host memory
(where the device time goes when the inputs arrive over PCIe)."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1207_0145_b200 as P  # noqa: E402

r, s, dom = P.gen_fk(100_000_000, 400_000_000, 0)
rh = P.Relation(torch.from_numpy(r.keys).pin_memory(), torch.from_numpy(r.payloads).pin_memory())
sh = P.Relation(torch.from_numpy(s.keys).pin_memory(), torch.from_numpy(s.payloads).pin_memory())
cfg = P.JoinConfig(threads=1, key_domain=dom)
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = P.run_join(rh, sh, cfg)
    t1 = time.perf_counter()
    print(f"iter {it}: wall {1e3 * (t1 - t0):.1f} ms  " +
          "  ".join(f"{k} {1e3 * v:.2f}" for k, v in res.phase_timings.items()), flush=True)
