"""solve_reference / dense_interior_eigenvalues (reference.py:42-97) on the device: the
reference's own known answers and the golden direct solution."""

import numpy as np
import numpy.testing as npt
import pytest

from conftest import golden, to_np

pytestmark = pytest.mark.gpu


def test_solve_reference_matches_reference_direct_solve(gpu):
    import paper_1911_03973_b200 as eb
    g = golden("c1_solution")
    m = eb.build_unit_square_mesh(6)
    batch = eb.build_element_batch(m, nu=1.0)
    d = eb.constant_dirichlet(m, 0.0)
    A = eb.assemble_sparse(batch.A_e, batch.index)
    b = eb.assemble_rhs(batch.b_e, batch.index)
    u = to_np(eb.solve_reference(A, b, d))
    assert np.linalg.norm(u - g["u_direct"]) <= 1e-10 * np.linalg.norm(g["u_direct"])
    # a SciPy matrix gives the same solution
    import scipy.sparse as sp
    crow, col, val = (to_np(t) for t in (A.crow_indices(), A.col_indices(), A.values()))
    As = sp.csr_matrix((val, col, crow), shape=A.shape)
    npt.assert_allclose(to_np(eb.solve_reference(As, b, d)), u, rtol=0, atol=1e-14)
    # a nonzero Dirichlet value: u = 1 on the boundary, f = 0, nu = 0 -> u == 1
    batch0 = eb.build_element_batch(m, nu=0.0)
    A0 = eb.assemble_sparse(batch0.A_e, batch0.index)
    u1 = to_np(eb.solve_reference(A0, np.zeros(m.n_nodes), eb.constant_dirichlet(m, 1.0)))
    npt.assert_allclose(u1, 1.0, atol=1e-10)


def test_dense_interior_eigenvalues(gpu):
    import paper_1911_03973_b200 as eb
    for n in (3, 4, 5, 9):  # test_spectrum.py:59-65: the model spectrum of the stiffness
        m = eb.build_grid_mesh(n)
        batch = eb.build_element_batch(m)
        A = eb.assemble_sparse(batch.A_e, batch.index)
        dense = to_np(eb.dense_interior_eigenvalues(A, eb.constant_dirichlet(m)))
        assert np.max(np.abs(dense - eb.model_eigenvalues_all(n))) <= 1e-10
    m = eb.build_unit_square_mesh(1)  # test_reference.py:112-115
    batch = eb.build_element_batch(m)
    npt.assert_allclose(to_np(eb.dense_interior_eigenvalues(
        eb.assemble_sparse(batch.K_e, batch.index), eb.constant_dirichlet(m))), [4.0], atol=1e-12)
    m = eb.build_unit_square_mesh(6)  # 3969 interior nodes: the size guard
    batch = eb.build_element_batch(m)
    with pytest.raises(ValueError):
        eb.dense_interior_eigenvalues(eb.assemble_sparse(batch.K_e, batch.index),
                                      eb.constant_dirichlet(m))
