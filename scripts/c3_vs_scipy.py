import time, numpy as np, torch, scipy.sparse as sp, scipy.sparse.linalg as spla, sys
sys.path.insert(0, '.')
import paper_1911_03973_b200 as eb
from paper_1911_03973_b200.inputs import config_problem
p = config_problem(3)
b, d, m = p["batch"], p["dirichlet"], p["mesh"]
x, h = eb.pcg(b, d, torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda"), 20000, tol=1e-8)
t0 = time.time()
A = eb.assemble_sparse(b.A_e, b.index, m.n_nodes)
crow, col, val = (t.cpu().numpy() for t in (A.crow_indices(), A.col_indices(), A.values()))
n = m.n_nodes
Ac = sp.csr_matrix((val, col, crow), shape=(n, n))
rhs = eb.assemble_rhs(b.b_e, b.index).cpu().numpy()
free = np.ones(n, bool); free[d.nd.cpu().numpy()] = False
Af = Ac[free][:, free].tocsr(); bf = rhs[free]
dinv = 1.0 / Af.diagonal()
M = spla.LinearOperator(Af.shape, matvec=lambda v: dinv * v)
its = [0]
def cb(xk): its[0] += 1
xs, info = spla.cg(Af, bf, rtol=1e-8, atol=0.0, maxiter=20000, M=M, callback=cb)
xg = x.cpu().numpy()[free]
print(f"ours {h.iterations} its, scipy {its[0]} its (info {info}), rel diff {np.linalg.norm(xg - xs) / np.linalg.norm(xs):.3e}, scipy time {time.time()-t0:.1f}s")
