"""Device timeline (CUPTI via torch.profiler) of the element-slab PCG loop at one rank over
torch.distributed NCCL: per-kernel time per iteration and idle gaps.  Run under torchrun
--nproc-per-node 1."""
import os
import sys
from collections import defaultdict

import torch
import torch.distributed as dist
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1911_03973_b200 import dist as D  # noqa: E402
from paper_1911_03973_b200.inputs import config_problem  # noqa: E402

torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
iters = 64
p = config_problem(cfg, assemble=False)
m = p["mesh"]
op, _ = D.rank_operator(m, p["nu"], p["f"], p["dirichlet"], 1, 0)
prob = D.setup([op], D.TorchTransport())
x0 = op.zeros()
run = (lambda: D.pcg(prob, [x0], iters, graph=True)) if cfg != 4 else \
    (lambda: D.jacobi(prob, [x0], iters, 0.8, graph=True))
run()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    torch.cuda.synchronize()
print(f"C{cfg}: {iters} its, {e0.elapsed_time(e1) / iters * 1e3:.1f} us/it (events)")
evs = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
             key=lambda e: e.time_range.start)
tot, cnt = defaultdict(float), defaultdict(int)
gap = 0.0
prev = None
for e in evs:
    tot[e.name[:70]] += e.time_range.elapsed_us()
    cnt[e.name[:70]] += 1
    if prev is not None and e.time_range.start > prev:
        gap += e.time_range.start - prev
    prev = max(prev or 0, e.time_range.end)
for k in sorted(tot, key=tot.get, reverse=True)[:14]:
    print(f"  {tot[k] / iters:9.1f} us/it  {cnt[k]:5d} x  {k}")
print(f"  idle gaps {gap / iters:.1f} us/it")
dist.destroy_process_group()
