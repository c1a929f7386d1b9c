"""Small-mesh workload touching every libebs kernel family, for compute-sanitizer:

    compute-sanitizer --tool memcheck  python scripts/sanitize_driver.py
    compute-sanitizer --tool racecheck python scripts/sanitize_driver.py
    compute-sanitizer --tool synccheck python scripts/sanitize_driver.py

Mesh generators, assembly, plans (2D packed / permuted, 3D tuple-coded / permuted),
residual (fast / exact, caller and internal numbering), matvec, diagonal, RHS, mask,
Richardson / Jacobi / Chebyshev / CG / PCG (launch loop, cooperative fused kernel,
single-cluster kernel), power iteration, CSR assembly, uniform_refine, the element-slab
kernels (emulated 2-rank halo, single-reduction PCG) and the vector kernels."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1911_03973_b200 as eb  # noqa: E402
from paper_1911_03973_b200 import dist  # noqa: E402
from paper_1911_03973_b200.inputs import config_problem  # noqa: E402


def run():
    rng = np.random.default_rng(0)
    for cfg, size in ((2, 4), (4, 4), (3, 3), (5, 4)):
        p = config_problem(cfg, seed=1, size=size)
        batch, m = p["batch"], p["mesh"]
        d = p["dirichlet"] or eb.constant_dirichlet(m, 0.0)
        x = torch.from_numpy(rng.uniform(-1, 1, m.n_nodes)).cuda()
        for det in (True, False):
            eb.residual(batch, x, deterministic=det)
        eb.matvec(batch, x)
        eb.diagonal(batch)
        eb.assemble_rhs(batch.b_e, batch.index)
        eb.mask_dirichlet(x, d)
        x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
        eb.jacobi(batch, d, x0, 40, omega=0.8)
        eb.jacobi(batch, d, x0, 5, omega=0.8, deterministic=True, reference=x)
        eb.pcg(batch, d, x0, 40, tol=1e-8)
        eb.cg(batch, d, x0, 40, callback=lambda k, xx, rr: None)
        eb.pcg(batch, d, x0, 40, tol=1e-8, fused=True)
        eb.assemble_sparse(batch.A_e, batch.index, m.n_nodes)
        if m.dim == 2:
            b = eb.model_eigen_bounds(2**size + 1)
            eb.richardson(batch, d, x0, b, 10)
            eb.chebyshev2(batch, d, x0, b, 4, 10)
            eb.chebyshev3(batch, d, x0, b, 10)
            eb.power_iteration_lambda_max(batch, d, iters=20)
            eb.uniform_refine(m)
        prob, _ = dist.emulate(batch, m.n_nodes, d, 2)
        xin = [op.to_internal(x0) for op in prob.ops]
        dist.jacobi(prob, xin, 10, 0.8)
        dist.pcg(prob, xin, 20, tol=1e-8)
        dist.pcg(prob, xin, 20, reductions=2)
        xs = [op.to_internal(x) for op in prob.ops]
        dist.residual(prob, xs)
    torch.cuda.synchronize()
    print("sanitize driver done")


if __name__ == "__main__":
    run()
