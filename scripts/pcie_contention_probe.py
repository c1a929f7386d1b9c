"""Do the residual kernels slow the PCIe copies?  Both-direction copies of a C2 vector
(33.6 MB) alone, then with C2 residuals running back to back on a third stream, and the
residuals' own time alone / under the copies.  python scripts/pcie_contention_probe.py"""
import sys
sys.path.insert(0, '.')
import torch
import paper_1911_03973_b200 as eb
from paper_1911_03973_b200.inputs import config_problem

p = config_problem(2, seed=0)
b, n = p["batch"], p["mesh"].n_nodes
h_x = torch.empty(n, dtype=torch.float64).uniform_(-1, 1).pin_memory()
h_r = torch.empty(n, dtype=torch.float64).pin_memory()
d_x, d_r = torch.empty(n, dtype=torch.float64, device="cuda"), torch.empty(n, dtype=torch.float64, device="cuda")
xg, rg = h_x.cuda(), torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
reps = 24
ev = lambda: torch.cuda.Event(enable_timing=True)


def run(copies, kernels):
    torch.cuda.synchronize()
    marks = {}
    for name, st, on in (("h2d", s1, copies), ("d2h", s2, copies), ("res", s3, kernels)):
        if not on:
            continue
        with torch.cuda.stream(st):
            e0, e1 = ev(), ev()
            e0.record(st)
            for _ in range(reps):
                if name == "h2d":
                    d_x.copy_(h_x, non_blocking=True)
                elif name == "d2h":
                    h_r.copy_(d_r, non_blocking=True)
                else:
                    eb.residual(b, xg, deterministic=False, out=rg, check_finite=False)
            e1.record(st)
            marks[name] = (e0, e1)
    torch.cuda.synchronize()
    return {k: e0.elapsed_time(e1) / reps for k, (e0, e1) in marks.items()}


for _ in range(2):
    print("copies alone   ", {k: f"{v:.3f} ms" for k, v in run(True, False).items()}, flush=True)
    print("kernels alone  ", {k: f"{v:.3f} ms" for k, v in run(False, True).items()}, flush=True)
    print("both           ", {k: f"{v:.3f} ms" for k, v in run(True, True).items()}, flush=True)
