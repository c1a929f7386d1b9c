#!/usr/bin/env python
"""Device timeline of a solver run via torch.profiler (CUPTI): per-kernel device time and
the idle gaps between consecutive kernels.  Usage: python scripts/timeline.py [config] [iters]"""
import sys
from collections import defaultdict

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__file__)))
import paper_1911_03973_b200 as eb  # noqa: E402
from paper_1911_03973_b200.inputs import config_problem  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 40
p = config_problem(cfg)
batch, d, m = p["batch"], p["dirichlet"], p["mesh"]
x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
run = (lambda: eb.jacobi(batch, d, x0, iters)) if cfg == 4 else (lambda: eb.pcg(batch, d, x0, iters))
run()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    torch.cuda.synchronize()
print(f"config C{cfg}: {iters} iterations, events {e0.elapsed_time(e1):.3f} ms")
evs = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
             key=lambda e: e.time_range.start)
tot = defaultdict(float)
cnt = defaultdict(int)
gaps = []
prev_end = None
for e in evs:
    tot[e.name[:60]] += e.time_range.elapsed_us()
    cnt[e.name[:60]] += 1
    if prev_end is not None:
        gaps.append(e.time_range.start - prev_end)
    prev_end = e.time_range.end
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{v:10.1f} us  {cnt[k]:5d} x  {v / cnt[k]:8.2f} us  {k}")
if gaps:
    gaps.sort()
    print(f"gaps: n={len(gaps)} total={sum(gaps):.1f} us median={gaps[len(gaps)//2]:.2f} "
          f"max={gaps[-1]:.1f} us")
