"""The pipelined host-buffer residual (ebs_residual_many_host) at C2 size: ms per step
for k = 32 / 100 rows; run with EBS_PIPE_NB=2,3,4 for the buffer depth.  Bitwise check
of the rows against the device residual.  python scripts/e2e_pipe_probe.py"""
import os
import sys
import time
sys.path.insert(0, '.')
import torch
import paper_1911_03973_b200 as eb
from paper_1911_03973_b200.inputs import config_problem

p = config_problem(2, seed=0)
b, n = p["batch"], p["mesh"].n_nodes
x = torch.empty(n, dtype=torch.float64).uniform_(-1, 1).pin_memory()
ref = eb.residual(b, x.cuda(), deterministic=False).cpu()
for k in (32, 100):
    xs = x.unsqueeze(0).expand(k, n)
    out = torch.empty((k, n), dtype=torch.float64).pin_memory()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eb.residual_many(b, xs, out=out, deterministic=False)
    first = time.perf_counter() - t0
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eb.residual_many(b, xs, out=out, deterministic=False)
        best = min(best, time.perf_counter() - t0)
    assert torch.equal(out[k - 1], ref) and torch.equal(out[0], ref)
    print(f"NB={os.environ.get('EBS_PIPE_NB', '3')} k={k}: {best / k * 1e3:.3f} ms/step "
          f"({n / (best / k) / 1e9:.2f} GDoF/s); first call into fresh pinned rows {first / k * 1e3:.3f} ms/step", flush=True)
    del out
