"""Full-size parity of the north-star configs against an INDEPENDENT host oracle
(SURVEY 7.4-6 "at full N, spot checks: a few residuals and PCG iterations").

The host side never touches the library: meshes, seeded jitter / permutation, element
matrices and operators come from oracle/ebs_oracle.py (pinned to the reference's golden
vectors in the CPU suite).  Whole-mesh element arrays of C4 / C5 are built chunk by chunk
by ``oracle.StreamedOperator`` -- bitwise the whole-mesh operator, since element matrices
are elementwise and the chunk-local products are reduced by one (j, e)-ordered bincount,
the reference's threaded deterministic mode (operators.py:72-111).

* C4 (level 12, 33.5M jittered + permuted triangles, nu=10, f=sin sin): connectivity,
  element matrices and the exact residual BIT FOR BIT; 3 damped-Jacobi iterates with the
  exact residual bit for bit; the fast residual within 1e-12 relative max-norm.
* C5 (N=256, 100.7M Kuhn tets, nu=1): connectivity and the exact residual bit for bit,
  fast residual within 1e-12; 3 Jacobi-PCG iterations within 1e-10.
* C3 (N=128, 12.6M tets, nu=0): the assembled CSR built on the host from the oracle's
  element matrices (SciPy COO -> CSR) == eb.assemble_sparse; SciPy cg(M = Jacobi) on THAT
  matrix (the reference's CG, reference.py:70) takes the device PCG's iteration count.
"""

import gc

import numpy as np
import pytest
import torch

import oracle as o

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _free():
    gc.collect()
    torch.cuda.empty_cache()


def _host(t):
    return t.detach().cpu().numpy()


def _rel_max(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


def _check_mesh(m, inp):
    np.testing.assert_array_equal(_host(m.nodes), inp["nodes"])
    conn = _host(m.conn)  # (n_b, n_e) int32 SoA
    for j in range(conn.shape[0]):
        np.testing.assert_array_equal(conn[j], inp["elements"][:, j])


def test_c4_full_size_bitwise_vs_oracle(gpu):
    import paper_1911_03973_b200 as eb
    from paper_1911_03973_b200.inputs import config_problem
    inp = o.config_inputs(4, seed=0)
    p = config_problem(4, seed=0)
    batch, d, m = p["batch"], p["dirichlet"], p["mesh"]
    assert m.n_elements == 33_554_432 and m.n_nodes == 16_785_409
    np.testing.assert_array_equal(p["perm"], inp["perm"])
    _check_mesh(m, inp)
    np.testing.assert_array_equal(_host(d.nd), inp["dirichlet"])
    op = o.StreamedOperator(inp["nodes"], inp["elements"], nu=inp["nu"], f_vals=inp["f_vals"])
    # element matrices A_e, b_e: bit for bit, chunk by chunk
    A_dev = batch.A_e  # (3, 3, n_e) view of element-major memory
    nc = len(op.bounds)
    for c in sorted({0, nc // 3, 2 * nc // 3, nc - 1}):
        lo, hi = op.bounds[c]
        A_h, be_h = op.matrices(c)
        np.testing.assert_array_equal(_host(A_dev[:, :, lo:hi]), A_h)
        np.testing.assert_array_equal(_host(batch.b_e[:, lo:hi]), be_h)
    n = m.n_nodes
    x = np.random.default_rng(7).uniform(-1.0, 1.0, n)
    r_o = op.residual(x)
    r_exact = _host(eb.residual(batch, x, deterministic=True))
    np.testing.assert_array_equal(r_exact, r_o)
    r_fast = _host(eb.residual(batch, x, deterministic=False))
    assert _rel_max(r_fast, r_o) <= 1e-12
    # 3 damped-Jacobi iterations (omega = 0.8) with the exact residual: iterates bitwise
    x0 = np.zeros(n)
    xo, ho = o.jacobi(op, None, None, inp["dirichlet"], x0, 0.8, 3)
    xd, hd = eb.jacobi(batch, d, torch.zeros(n, dtype=torch.float64, device="cuda"), 3,
                       omega=0.8, deterministic=True)
    np.testing.assert_array_equal(_host(xd), xo)
    np.testing.assert_allclose(hd.residual_norms, ho["residual_norms"], rtol=1e-12)
    del batch, p, op, r_o
    _free()


def test_c5_full_size_vs_streamed_oracle(gpu):
    import paper_1911_03973_b200 as eb
    from paper_1911_03973_b200.inputs import config_problem
    inp = o.config_inputs(5)
    p = config_problem(5)
    batch, d, m = p["batch"], p["dirichlet"], p["mesh"]
    assert m.n_elements == 100_663_296 and m.n_nodes == 16_974_593
    _check_mesh(m, inp)
    np.testing.assert_array_equal(_host(d.nd), inp["dirichlet"])
    op = o.StreamedOperator(inp["nodes"], inp["elements"], nu=inp["nu"])
    lo, hi = op.bounds[len(op.bounds) // 2]
    A_h, be_h = op.matrices(len(op.bounds) // 2)
    np.testing.assert_array_equal(_host(batch.A_e[:, :, lo:hi]), A_h)
    n = m.n_nodes
    x = np.random.default_rng(11).uniform(-1.0, 1.0, n)
    r_o = op.residual(x)
    np.testing.assert_array_equal(_host(eb.residual(batch, x, deterministic=True)), r_o)
    assert _rel_max(_host(eb.residual(batch, x, deterministic=False)), r_o) <= 1e-12
    # 3 Jacobi-PCG iterations from x0 = 0 (BASELINE C5 loop)
    xo, ho = o.pcg(op, None, None, inp["dirichlet"], np.zeros(n), 3)
    xd, hd = eb.pcg(batch, d, torch.zeros(n, dtype=torch.float64, device="cuda"), 3)
    assert len(hd.residual_norms) == len(ho["residual_norms"]) == 4
    np.testing.assert_allclose(hd.residual_norms, ho["residual_norms"], rtol=1e-10)
    xd = _host(xd)
    assert np.linalg.norm(xd - xo) <= 1e-10 * np.linalg.norm(xo)
    del batch, p, op, r_o
    _free()


def test_c3_host_csr_and_scipy_cg_jacobi(gpu):
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla

    import paper_1911_03973_b200 as eb
    from paper_1911_03973_b200.inputs import config_problem
    inp = o.config_inputs(3)
    nodes, elements, nd = inp["nodes"], inp["elements"], inp["dirichlet"]
    n = nodes.shape[0]
    _, _, A, b_e = o.element_matrices(nodes, elements, nu=inp["nu"])
    indt = np.ascontiguousarray(elements.T)
    nb = indt.shape[0]
    # reference.py:25-39 restated on the host: one triplet per local entry, duplicates summed
    rows = np.concatenate([indt[i] for i in range(nb) for j in range(nb)])
    cols = np.concatenate([indt[j] for i in range(nb) for j in range(nb)])
    vals = np.concatenate([A[i, j] for i in range(nb) for j in range(nb)])
    Ah = sp.coo_matrix((vals, (rows, cols)), shape=(n, n)).tocsr()
    Ah.sum_duplicates()
    Ah.sort_indices()
    del rows, cols, vals
    b_h = o.assemble_rhs(b_e, indt, n)
    p = config_problem(3)
    batch, d, m = p["batch"], p["dirichlet"], p["mesh"]
    Ad = eb.assemble_sparse(batch.A_e, batch.index, n)
    np.testing.assert_array_equal(_host(Ad.crow_indices()), Ah.indptr)
    np.testing.assert_array_equal(_host(Ad.col_indices()), Ah.indices)
    scale = float(np.abs(Ah.data).max())
    assert float(np.abs(_host(Ad.values()) - Ah.data).max()) <= 1e-14 * scale
    del Ad
    np.testing.assert_array_equal(_host(eb.assemble_rhs(batch.b_e, batch.index)), b_h)
    x, h = eb.pcg(batch, d, torch.zeros(n, dtype=torch.float64, device="cuda"), 20000,
                  tol=1e-8)
    free = np.ones(n, bool)
    free[nd] = False
    Af = Ah[free][:, free].tocsr()
    bf = b_h[free]
    dinv = 1.0 / Af.diagonal()
    M = spla.LinearOperator(Af.shape, matvec=lambda v: dinv * v)
    its = [0]
    xs, info = spla.cg(Af, bf, rtol=1e-8, atol=0.0, maxiter=20000, M=M,
                       callback=lambda xk: its.__setitem__(0, its[0] + 1))
    assert info == 0 and its[0] == h.iterations, (its[0], h.iterations)
    xg = _host(x)[free]
    assert np.linalg.norm(xg - xs) <= 1e-10 * np.linalg.norm(xs)
    del batch, p, x
    _free()
