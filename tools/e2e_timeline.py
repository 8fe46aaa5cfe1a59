"""Host-side timeline of one end-to-end cfg2 join from pinned host memory
(where the e2e milliseconds go): upload of each side, queueing of the
phases, the final synchronisation."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1207_0145_b200 as P  # noqa: E402
from paper_1207_0145_b200 import engine  # noqa: E402

marks = []


def wrap(cls, name):
    f = getattr(cls, name)

    def g(self, *a, **k):
        t0 = time.perf_counter()
        out = f(self, *a, **k)
        marks.append((name, t0, time.perf_counter()))
        return out

    setattr(cls, name, g)


if os.environ.get("SYNC_AFTER_PUBLIC") == "1":  # no overlap of the private upload with the public sort
    _sp = engine.JoinContext.sort_public

    def _sp_sync(self):
        _sp(self)
        torch.cuda.synchronize()

    engine.JoinContext.sort_public = _sp_sync
for nm in ("_upload", "stage_private", "sort_public", "sort_private_chunks", "join", "finalize"):
    wrap(engine.JoinContext, nm)

r, s, dom = P.gen_fk(100_000_000, 400_000_000, 0)
rh = P.Relation(torch.from_numpy(r.keys).pin_memory(), torch.from_numpy(r.payloads).pin_memory())
sh = P.Relation(torch.from_numpy(s.keys).pin_memory(), torch.from_numpy(s.payloads).pin_memory())
cfg = P.JoinConfig(threads=1, key_domain=dom)
for it in range(4):
    marks.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = P.run_join(rh, sh, cfg)
    t1 = time.perf_counter()
    print(f"iter {it}: {1e3 * (t1 - t0):.1f} ms  " +
          "  ".join(f"{n}@{1e3 * (a - t0):.1f}+{1e3 * (b - a):.1f}" for n, a, b in marks), flush=True)

