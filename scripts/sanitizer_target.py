"""Small-mesh pass over the hot path for compute-sanitizer (memcheck / racecheck / initcheck /
synccheck): assembly, residual (both modes), matvec, diagonal, Jacobi, CG, PCG (launch loop
and the fused single-kernel forms), Chebyshev, refine, CSR, 2D permuted + 3D."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle as o
import paper_1911_03973_b200 as eb

inp = o.config_inputs(4, seed=0, size=4)
m = eb.Mesh(inp["nodes"], inp["elements"], inp["dirichlet"])
batch = eb.build_element_batch(m, nu=10.0, f=inp["f_vals"])
x = np.random.default_rng(0).uniform(-1, 1, m.n_nodes)
r = eb.residual(batch, x); eb.residual(batch, x, deterministic=False)
d = eb.DirichletData(inp["dirichlet"], np.zeros(len(inp["dirichlet"])))
eb.matvec(batch, x, d); eb.diagonal(batch)
for fn in (eb.cg, eb.pcg):
    fn(batch, d, np.zeros(m.n_nodes), 30, tol=1e-8)
    fn(batch, d, np.zeros(m.n_nodes), 30, tol=1e-8, fused=True)
eb.jacobi(batch, d, np.zeros(m.n_nodes), 10, omega=0.8)
m2 = eb.build_unit_square_mesh(3)
b2 = eb.build_element_batch(m2, nu=0.0)
d2 = eb.constant_dirichlet(m2, 1.0)
bounds = eb.model_eigen_bounds(9)
x0 = eb.apply_initial_guess(m2, d2)
eb.richardson(b2, d2, x0, bounds, 10); eb.chebyshev2(b2, d2, x0, bounds, 4, 10); eb.chebyshev3(b2, d2, x0, bounds, 10)
eb.uniform_refine(m2); eb.assemble_sparse(b2.A_e, b2.index.indt)
m3 = eb.build_unit_cube_mesh(3)
b3 = eb.build_element_batch(m3, nu=1.0)
d3 = eb.DirichletData(eb.face_z0_nodes(m3), np.zeros(len(eb.face_z0_nodes(m3))))
eb.residual(b3, np.ones(m3.n_nodes)); eb.pcg(b3, d3, np.zeros(m3.n_nodes), 30, tol=1e-8)
eb.residual_many(batch, np.stack([x, x, x]))
torch.cuda.synchronize()
print("sanitizer target ok")
