"""Assembled CSR on the device (reference.py:25-39) against the
reference's SciPy assembly, and as a full-size cross-check of the matrix-free residual."""

import numpy as np
import pytest
import torch

from conftest import golden, to_np

pytestmark = pytest.mark.gpu


def test_csr_matches_reference_assembly(gpu):
    import paper_1911_03973_b200 as eb
    g = golden("sparse_l3")
    m = eb.build_unit_square_mesh(3)
    batch = eb.build_element_batch(m, nu=1.0)
    for name in ("K_e", "A_e"):
        S = eb.assemble_sparse(getattr(batch, name), batch.index.indt)
        np.testing.assert_array_equal(to_np(S.crow_indices()), g[f"{name}_indptr"])
        np.testing.assert_array_equal(to_np(S.col_indices()), g[f"{name}_indices"])
        np.testing.assert_allclose(to_np(S.values()), g[f"{name}_data"], rtol=1e-15, atol=1e-17)
    # stiffness: symmetric, constants in the kernel (test_reference.py:19-24)
    K = eb.assemble_sparse(batch.K_e, batch.index).to_dense()
    assert torch.equal(K, K.t())
    assert float(torch.abs(K.sum(dim=1)).max()) == 0.0
    with pytest.raises(ValueError):
        eb.assemble_sparse(batch.K_e[:, :2, :], batch.index.indt)


def test_csr_3d_and_distributivity(gpu):
    import paper_1911_03973_b200 as eb
    m = eb.build_unit_cube_mesh(3)
    b = eb.build_element_batch(m, nu=1.7)
    K = eb.assemble_sparse(b.K_e, b.index).to_dense()
    M = eb.assemble_sparse(b.M_e, b.index).to_dense()
    A = eb.assemble_sparse(b.A_e, b.index).to_dense()
    assert float((A - (K + 1.7 * M)).abs().max()) <= 1e-14
    assert abs(float(M.sum()) - 1.0) <= 1e-13


@pytest.mark.slow
def test_full_size_c2_cross_check(gpu):
    """Matrix-free residual vs b - A x with the device-assembled CSR (cuSPARSE SpMV)
    on the full BASELINE C2 mesh (8.4M triangles, permuted numbering)."""
    import paper_1911_03973_b200 as eb
    from paper_1911_03973_b200.inputs import config_problem
    p = config_problem(2, seed=0)
    batch = p["batch"]
    x = torch.from_numpy(p["x"]).cuda()
    A = eb.assemble_sparse(batch.A_e, batch.index)
    b = eb.assemble_rhs(batch.b_e, batch.index)
    r_ref = b - torch.mv(A, x)
    r = eb.residual(batch, x)
    rel = float((r - r_ref).abs().max() / r_ref.abs().max())
    assert rel <= 1e-12, rel
