"""C5 (100.7M tets, 17M unknowns): 500 Jacobi-PCG iterations on the device vs SciPy's cg
with M = Jacobi (500 iterations, no tolerance) on the assembled, Dirichlet-eliminated
system: relative difference of the iterates and of the final residual norms."""
import sys
import time

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(
    __import__("os").path.abspath(__file__))))
import paper_1911_03973_b200 as eb  # noqa: E402
from paper_1911_03973_b200.inputs import config_problem  # noqa: E402

ITERS = int(sys.argv[1]) if len(sys.argv) > 1 else 500
p = config_problem(5)
b, d, m = p["batch"], p["dirichlet"], p["mesh"]
x, h = eb.pcg(b, d, torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda"), ITERS)
A = eb.assemble_sparse(b.A_e, b.index, m.n_nodes)
crow, col, val = (t.cpu().numpy() for t in (A.crow_indices(), A.col_indices(), A.values()))
del A
n = m.n_nodes
free = np.ones(n, bool)
free[d.nd.cpu().numpy()] = False
Af = sp.csr_matrix((val, col, crow), shape=(n, n))[free][:, free].tocsr()
bf = eb.assemble_rhs(b.b_e, b.index).cpu().numpy()[free]
dinv = 1.0 / Af.diagonal()
M = spla.LinearOperator(Af.shape, matvec=lambda v: dinv * v)
t0 = time.time()
xs, info = spla.cg(Af, bf, rtol=0.0, atol=0.0, maxiter=ITERS, M=M)
xg = x.cpu().numpy()[free]
r_s = np.linalg.norm(bf - Af @ xs)
print(f"C5 {ITERS} iterations: device ||r|| {h.residual_norms[-1]:.6e}, scipy ||b-Ax|| {r_s:.6e}, "
      f"iterate rel diff {np.linalg.norm(xg - xs) / np.linalg.norm(xs):.3e}, "
      f"scipy {time.time() - t0:.0f} s, nnz {Af.nnz}")
