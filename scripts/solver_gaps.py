"""Idle time between the loop kernels of a solve (CUPTI timeline, 100 iterations): span,
busy time, gap statistics, for BASELINE config argv[1] (3/5 PCG, 4 Jacobi)."""
import sys, os
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
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    run(100)
    torch.cuda.synchronize()
ks = sorted([(e.time_range.start, e.time_range.end, e.name[:40]) for e in prof.events() if e.device_type.name == "CUDA"])
loop = [k for k in ks if any(t in k[2] for t in ("pcg_matvec", "pcg_update", "pcg_direction", "jacobi_step"))]
busy = sum(e - s for s, e, _ in loop)
span = loop[-1][1] - loop[0][0]
gaps = [loop[i + 1][0] - loop[i][1] for i in range(len(loop) - 1)]
gaps.sort()
print(f"C{cfg}: {len(loop)} loop kernels, span {span:.0f} us, busy {busy:.0f} us, idle {span - busy:.0f} us "
      f"({(span - busy) / span * 100:.1f}%), gap median {gaps[len(gaps) // 2]:.2f} us max {gaps[-1]:.1f} us, "
      f"per iteration span {span / 100:.1f} us")
big = [g for g in gaps if g > 5]
print("gaps > 5 us:", len(big), "sum", sum(big))
