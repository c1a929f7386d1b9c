"""Compute-side strong-scaling check on ONE GPU: the BASELINE C4 (damped Jacobi) and C5
(Jacobi-PCG, single-reduction) solves on P = 1, 2, 4, 8 element slabs emulated in one
process (dist.emulate: every rank's kernels run back to back on the one device, the halo is a
device copy).  The emulated time of P ranks is the sum of their per-rank work, so
E_compute(P) = T_1GPU / T_emulated(P) measures what partitioning itself costs (interface
sweeps, halo gather / combine kernels, smaller grids) -- NOT the NVLink / NCCL latency,
which one GPU cannot show.  Both transports: the device-copy one (the NCCL path's kernel
sequence: interface sweep, send gather, interior sweep, combine) and the peer-memory one
(one sweep pushing the interface partials, one combine).
Usage: python scripts/emulated_scaling.py [2|4|5]..."""
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


def residual_scaling(reps=50):
    """C2: the caller-order residual (bench value) on P slabs, each rank's x and r in its own
    caller order (dist.residual_local) vs the 1-GPU ebs_residual (fast mode); both replayed
    from CUDA graphs of 10 residuals, as the bench does."""
    p = config_problem(2)
    batch, m = p["batch"], p["mesh"]
    x = torch.from_numpy(p["x"]).cuda()
    out = torch.empty_like(x)
    def one():
        for _ in range(10):
            eb.residual(batch, x, deterministic=False, out=out, check_finite=False)
    one()
    g1 = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(g1):
        one()
    t1 = tm(lambda: [g1.replay() for _ in range(reps // 10)]) / (reps // 10 * 10)
    print(f"C2: 1-GPU residual {t1 * 1e6:.1f} us ({m.n_nodes / t1 / 1e9:.2f} GDoF/s)", flush=True)
    for P in (1, 2, 4, 8):
        for peer in (False, True):
            prob, _ = dist.emulate(batch, m.n_nodes, None, P, peer=peer)
            xl = [x[op.global_ids].contiguous() for op in prob.ops]
            rl = [op.zeros() for op in prob.ops]
            xi = [op.zeros() for op in prob.ops]
            sr = [op.zeros() for op in prob.ops]
            def body():
                for _ in range(10):
                    dist.residual_local(prob, xl, rl, xi, sr)
            body()  # warm-up (lazy workspaces) before the capture
            g = torch.cuda.CUDAGraph()
            torch.cuda.synchronize()
            with torch.cuda.graph(g):
                body()
            t = tm(lambda: [g.replay() for _ in range(reps // 10)]) / (reps // 10 * 10)
            print(f"  P={P} {'peer' if peer else 'copy'}: emulated {t * 1e6:.1f} us per residual "
                  f"(sum of the ranks' work), E_compute = {t1 / t:.3f}", flush=True)
            if peer:
                prob.comm.close()
            del prob, xl, rl, xi, sr
            torch.cuda.empty_cache()
    del p, batch
    torch.cuda.empty_cache()


for cfg in [int(a) for a in sys.argv[1:]] or [4, 5]:
    if cfg == 2:
        residual_scaling()
        continue
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
