"""Jacobi-PCG as three launches per iteration (device-controlled loop, CUDA-graph batches)
vs one cooperative kernel for the whole solve (pcg(..., fused=True)): device time per
solve and per iteration on the BASELINE configs."""
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(
    __import__("os").path.abspath(__file__))))
import paper_1911_03973_b200 as eb  # noqa: E402
from paper_1911_03973_b200.inputs import config_problem  # noqa: E402

cases = [(1, None, 1e-8), (3, None, 1e-8), (5, 500, None)]
for cfg, iters, tol in cases:
    p = config_problem(cfg)
    b, d, m = p["batch"], p["dirichlet"], p["mesh"]
    x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
    it = iters or 100000
    for fused in (False, True):
        eb.pcg(b, d, x0, it, tol=tol, fused=fused)
        torch.cuda.synchronize()
        best = None
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _, h = eb.pcg(b, d, x0, it, tol=tol, fused=fused)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        k = len(h.residual_norms) - 1
        print(f"C{cfg} fused={fused!s:5}: {k} its, {best:9.3f} ms, {best / k * 1e3:8.2f} us/it, "
              f"{k / best * 1e3:8.1f} it/s", flush=True)
