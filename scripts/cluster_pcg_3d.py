"""Small 3D Kuhn meshes (N = 10, 16): Jacobi-PCG to 1e-8 per iteration time -- one
thread-block cluster (fused=True), the cooperative grid kernel (EBS_NO_CLUSTER=1), and
the launch-per-step loop."""
import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch, time
import paper_1911_03973_b200 as eb
from paper_1911_03973_b200.inputs import config_problem
torch.cuda.set_device(0)
for size in (10, 16):
    p = config_problem(5, seed=0, size=size)
    x0 = torch.zeros(p["mesh"].n_nodes, dtype=torch.float64, device="cuda")
    for mode in ("cluster", "coop", "loop"):
        if mode == "coop": os.environ["EBS_NO_CLUSTER"] = "1"
        f = mode != "loop"
        eb.pcg(p["batch"], p["dirichlet"], x0, 10000, tol=1e-8, fused=f); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); x, h = eb.pcg(p["batch"], p["dirichlet"], x0, 10000, tol=1e-8, fused=f); e1.record(); torch.cuda.synchronize()
        os.environ.pop("EBS_NO_CLUSTER", None)
        print(size, p["mesh"].n_nodes, mode, h.iterations, round(e0.elapsed_time(e1) * 1e3 / h.iterations, 2), "us/it")
