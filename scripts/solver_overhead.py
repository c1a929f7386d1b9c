"""Solve time vs iteration count (0, 1, 32, 64, 250, 500): per-iteration cost and the fixed
per-solve overhead, for BASELINE config argv[1] (3/5 PCG, 4 Jacobi)."""
import sys, os, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_1911_03973_b200 as eb
from paper_1911_03973_b200.inputs import config_problem
torch.cuda.set_device(0)
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
p = config_problem(cfg, seed=0)
x0 = torch.zeros(p["mesh"].n_nodes, dtype=torch.float64, device="cuda")
run = (lambda n: eb.jacobi(p["batch"], p["dirichlet"], x0, n, omega=0.8)) if cfg == 4 else (lambda n: eb.pcg(p["batch"], p["dirichlet"], x0, n))
run(40); torch.cuda.synchronize()
res = {}
for n in (0, 1, 32, 64, 250, 500):
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(); run(n); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    res[n] = best
print(f"C{cfg} ms:", {k: round(v, 3) for k, v in res.items()},
      "per-it (500-250)/250 us:", round((res[500] - res[250]) / 250 * 1e3, 1),
      "intercept ms:", round(res[500] - 500 * (res[500] - res[250]) / 250, 2))
