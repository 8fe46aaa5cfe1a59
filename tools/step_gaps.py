"""GPU idle gaps inside bench steps: torch.profiler (CUPTI) kernel and memcpy
timestamps over 3 run_join steps of a config; prints the busy time, the idle
time between consecutive GPU activities and the largest gaps with their
neighbours.   python tools/step_gaps.py [cfg2] [threads]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import bench
import paper_1207_0145_b200 as P
from paper_1207_0145_b200.core import JoinConfig, Relation

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
threads = int(sys.argv[2]) if len(sys.argv) > 2 else 1
dev = torch.device("cuda", 0)
P.warmup()
r, s, dom = bench.make_inputs(cfg_name)
rd = Relation(torch.from_numpy(r.keys).to(dev), torch.from_numpy(r.payloads).to(dev))
sd = Relation(torch.from_numpy(s.keys).to(dev), torch.from_numpy(s.payloads).to(dev))
cfg = JoinConfig(threads=threads, algorithm="p-mpsm", key_domain=dom)
for _ in range(3):
    P.run_join(rd, sd, cfg)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(3):
        P.run_join(rd, sd, cfg)
    torch.cuda.synchronize()
ev = []
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() >= 0:
        ev.append((e.time_range.start, e.time_range.end, e.name))
ev.sort()
busy = 0.0
gaps = []
last_end, last_name = None, None
for st, en, nm in ev:
    if last_end is not None and st > last_end:
        gaps.append((st - last_end, last_name, nm))
    busy += en - st
    if last_end is None or en > last_end:
        last_end, last_name = en, nm
span = ev[-1][1] - ev[0][0]
print(f"{cfg_name} T={threads}: span {span / 3e3:.3f} ms/step, busy {busy / 3e3:.3f} ms/step, "
      f"idle {sum(g[0] for g in gaps) / 3e3:.3f} ms/step over {len(gaps)} gaps")
for g, a, b in sorted(gaps, reverse=True)[:25]:
    print(f"  {g:8.1f} us  after {a[:60]}  before {b[:60]}")
# the middle step's transitions in order (gap > 2 us)
if os.environ.get("GAPS_ORDER"):
    mid0 = ev[0][0] + span / 3
    mid1 = ev[0][0] + 2 * span / 3
    last_end, last_name = None, None
    for st, en, nm in ev:
        if last_end is not None and mid0 <= st < mid1 and st - last_end > 2:
            print(f"    {st - last_end:7.1f} us  {last_name[:50]:50s} -> {nm[:50]}")
        if last_end is None or en > last_end:
            last_end, last_name = en, nm
# host side: CUDA runtime / driver calls that block for long (synchronous
# copies, syncs) -- the GPU runs dry behind them
slow = {}
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CPU and e.name.startswith("cu"):
        d = e.time_range.elapsed_us()
        if d > 5:
            c = slow.setdefault(e.name, [0, 0.0, 0.0])
            c[0] += 1
            c[1] += d
            c[2] = max(c[2], d)
print("host CUDA API calls > 5 us (count, total us per step, max us):")
for nm, (c, tot, mx) in sorted(slow.items(), key=lambda x: -x[1][1]):
    print(f"  {nm[:50]:50s} {c / 3:6.1f} {tot / 3:9.1f} {mx:9.1f}")
