"""C1 Jacobi-PCG to 1e-8 with fused=True: solve time and the CUPTI kernel list (the
single-cluster kernel, or the cooperative one with EBS_NO_CLUSTER=1)."""
import sys, os, collections
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_1911_03973_b200 as eb
from paper_1911_03973_b200.inputs import config_problem
torch.cuda.set_device(0)
p = config_problem(1, seed=0)
x0 = torch.zeros(p["mesh"].n_nodes, dtype=torch.float64, device="cuda")
for _ in range(3):
    eb.pcg(p["batch"], p["dirichlet"], x0, 10000, tol=1e-8, fused=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); x, h = eb.pcg(p["batch"], p["dirichlet"], x0, 10000, tol=1e-8, fused=True); e1.record(); torch.cuda.synchronize()
print("iterations", h.iterations, "solve us", e0.elapsed_time(e1) * 1e3, "us/it", e0.elapsed_time(e1) * 1e3 / h.iterations)
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    eb.pcg(p["batch"], p["dirichlet"], x0, 10000, tol=1e-8, fused=True)
    torch.cuda.synchronize()
for ev in prof.events():
    if ev.device_type.name == "CUDA":
        print(f"{ev.name[:70]:70s} {ev.device_time_total:9.1f} us")
