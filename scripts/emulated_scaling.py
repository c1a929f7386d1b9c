"""Compute-side strong-scaling check on ONE GPU: the BASELINE C4 (damped Jacobi) and C5
(Jacobi-PCG, single-reduction) solves on P = 1, 2, 4, 8 element slabs emulated in one
process (dist.emulate: every rank's kernels run back to back on the one device, the halo is a
device copy).  The emulated time of P ranks is the sum of their per-rank work, so
E_compute(P) = T_1GPU / T_emulated(P) measures what partitioning itself costs (interface
sweeps, halo gather / combine kernels, smaller grids) -- NOT the NVLink / NCCL latency,
which one GPU cannot show.  Both transports: the device-copy one (the NCCL path's kernel
sequence: interface sweep, send gather, interior sweep, combine) and the peer-memory one
(one sweep pushing the interface partials, one combine).
Usage: python scripts/emulated_scaling.py [4|5]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1911_03973_b200 as eb  # noqa: E402
from paper_1911_03973_b200 import dist  # noqa: E402
from paper_1911_03973_b200.inputs import config_problem  # noqa: E402


def tm(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3


for cfg in [int(a) for a in sys.argv[1:]] or [4, 5]:
    iters = 200 if cfg == 4 else 100
    p = config_problem(cfg)
    batch, d, m = p["batch"], p["dirichlet"], p["mesh"]
    x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
    one = (lambda: eb.jacobi(batch, d, x0, iters, omega=0.8)) if cfg == 4 else \
        (lambda: eb.pcg(batch, d, x0, iters))
    t1 = tm(one)
    print(f"C{cfg}: 1-GPU {iters / t1:.0f} it/s", flush=True)
    for P in (1, 2, 4, 8):
        for peer in (False, True):
            prob, _ = dist.emulate(batch, m.n_nodes, d, P, peer=peer)
            xin = [op.to_internal(x0) for op in prob.ops]
            run = (lambda: dist.jacobi(prob, xin, iters, 0.8, graph=True)) if cfg == 4 else \
                (lambda: dist.pcg(prob, xin, iters, graph=True))
            t = tm(run)
            print(f"  P={P} {'peer' if peer else 'copy'}: emulated {iters / t:.0f} it/s (sum of "
                  f"the ranks' work), E_compute = {t1 / t:.3f}", flush=True)
            if peer:
                prob.comm.close()
            del prob, xin
            torch.cuda.empty_cache()
    del p, batch
    torch.cuda.empty_cache()
