"""numpy_api: the reference's host-array convention over the device package -- types,
read-only attributes, callbacks and the north-star additions (3D, Jacobi / CG / PCG,
diagonal, matvec), checked against the oracle.  The reference's own suite through the same
facade is tests/test_gpu_reference_suite.py."""

import numpy as np
import pytest
import scipy.sparse as sp

import oracle as o

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_1911_03973_b200 import numpy_api
    return numpy_api.facade("")


def test_arrays_are_host_numpy_and_frozen_like_the_reference(api):
    m = api.build_unit_square_mesh(3)
    assert type(m).__name__ == "Mesh" and isinstance(m, api.Mesh)
    assert isinstance(m.nodes, np.ndarray) and m.nodes.dtype == np.float64
    assert m.elements.dtype == np.int64 and m.boundary_nodes.dtype == np.int64
    assert m.nodes is m.nodes                       # converted once
    with pytest.raises(ValueError):
        m.nodes[0, 0] = 5.0                         # mesh.py:53-54
    with pytest.raises(AttributeError):
        m.level = 7                                 # frozen data class
    nodes, elements, nd = o.unit_square_mesh(3)
    np.testing.assert_array_equal(m.nodes, nodes)
    np.testing.assert_array_equal(m.elements, elements)
    np.testing.assert_array_equal(m.boundary_nodes, nd)
    batch = api.build_element_batch(m, nu=2.5)
    assert isinstance(batch.K_e, np.ndarray) and batch.K_e.shape == (3, 3, m.n_elements)
    assert batch.index.indt.dtype == np.int64 and batch.index.ind_e.shape == (3, 1, m.n_elements)
    K, M, A, b_e = o.element_matrices(nodes, elements, nu=2.5)
    np.testing.assert_array_equal(batch.A_e, A)
    np.testing.assert_array_equal(batch.b_e, b_e)
    x = np.random.default_rng(0).standard_normal(m.n_nodes)
    r = api.residual(batch, x)
    assert isinstance(r, np.ndarray) and r.flags.writeable
    np.testing.assert_array_equal(r, o.residual(A, b_e, np.ascontiguousarray(elements.T), x))
    S = api.assemble_sparse(batch.A_e, batch.index.indt)
    assert sp.issparse(S) and S.shape == (m.n_nodes, m.n_nodes)
    b = api.assemble_rhs(batch.b_e, batch.index.indt)
    assert np.linalg.norm(r - (b - S @ x)) <= 1e-12 * np.linalg.norm(r)
    # a batch built from host arrays through the facade constructors (conftest.py:24-39 shape)
    again = api.ElementBatch(K_e=batch.K_e, M_e=batch.M_e, A_e=batch.A_e, b_e=batch.b_e, nu=2.5,
                             index=api.IndexArrays(batch.index.ind_e, batch.index.indt))
    np.testing.assert_array_equal(api.residual(again, x), r)


def test_solvers_callbacks_and_additions_in_host_arrays(api):
    nodes, elements, face = o.kuhn_cube_mesh(4)
    _, _, A, b_e = o.element_matrices(nodes, elements, nu=1.0)
    indt = np.ascontiguousarray(elements.T)
    m = api.build_unit_cube_mesh(4)
    batch = api.build_element_batch(m, nu=1.0)
    d = api.DirichletData(api.face_z0_nodes(m), np.zeros(len(face)))
    np.testing.assert_array_equal(d.nd, face)
    x0 = np.zeros(m.n_nodes)
    seen = []
    x, h = api.pcg(batch, d, x0, 200, tol=1e-8,
                   callback=lambda k, xk, rk: seen.append((k, xk, rk)))
    xo, ho = o.pcg(A, b_e, indt, face, x0, 200, tol=1e-8)
    assert isinstance(x, np.ndarray) and isinstance(h.residual_norms, np.ndarray)
    assert len(h.residual_norms) == len(ho["residual_norms"])
    assert np.linalg.norm(x - xo) <= 1e-8 * np.linalg.norm(xo)
    assert [k for k, _, _ in seen] == list(range(len(h.residual_norms)))
    assert all(isinstance(xk, np.ndarray) and isinstance(rk, np.ndarray) for _, xk, rk in seen)
    np.testing.assert_array_equal(seen[-1][1], x)   # fresh arrays per k, the last is the result
    assert not np.array_equal(seen[0][1], seen[-1][1])
    xj, hj = api.jacobi(batch, d, x0, 10, omega=0.8)
    _, hjo = o.jacobi(A, b_e, indt, face, x0, 0.8, 10)
    np.testing.assert_allclose(hj.residual_norms, hjo["residual_norms"], rtol=1e-10, atol=0.0)
    diag = api.diagonal(batch)
    np.testing.assert_array_equal(diag, o.diagonal(A, indt, m.n_nodes))
    v = np.random.default_rng(1).standard_normal(m.n_nodes)
    y = api.matvec(batch, v)
    assert isinstance(y, np.ndarray)
    r0 = api.residual(batch, np.zeros(m.n_nodes))
    np.testing.assert_allclose(r0 - api.residual(batch, v), y, rtol=0, atol=1e-12 * np.abs(y).max())
