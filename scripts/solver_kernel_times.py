"""Warm per-kernel times of a PCG solve (torch.profiler / CUPTI, 100 iterations) and the
solve rate, for BASELINE config argv[1] (3 or 5): `EBS_IDS_GRID=2|3 python
scripts/solver_kernel_times.py 5` compares id codings."""
import sys, os, collections
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_1911_03973_b200 as eb
from paper_1911_03973_b200.inputs import config_problem
torch.cuda.set_device(0)
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
p = config_problem(cfg, seed=0)
x0 = torch.zeros(p["mesh"].n_nodes, dtype=torch.float64, device="cuda")
eb.pcg(p["batch"], p["dirichlet"], x0, 40)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); eb.pcg(p["batch"], p["dirichlet"], x0, 200); e1.record(); torch.cuda.synchronize()
print("it/s (incl. setup)", 200 / (e0.elapsed_time(e1) / 1e3))
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    eb.pcg(p["batch"], p["dirichlet"], x0, 100)
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for ev in prof.events():
    if ev.device_type.name == "CUDA":
        a = agg[ev.name[:60]]; a[0] += 1; a[1] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:8]:
    print(f"{k:60s} n={n:5d} avg={t / n:9.1f} us total={t / 1e3:8.2f} ms")
