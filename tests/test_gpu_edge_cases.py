"""Edge cases the reference tests: hand-checkable diagonal systems (tests/conftest.py
diagonal_batch; test_solvers.py:91-109), no constraints, empty / ragged inputs."""

import numpy as np
import numpy.testing as npt
import pytest
import torch

from conftest import to_np

pytestmark = pytest.mark.gpu


def diagonal_batch(diag, load):
    import paper_1911_03973_b200 as eb
    A = np.diag(np.asarray(diag, dtype=np.float64)).reshape(3, 3, 1)
    indt = np.array([[0], [1], [2]], dtype=np.int64)
    return eb.ElementBatch(K_e=A, M_e=np.zeros_like(A), A_e=A,
                           b_e=np.asarray(load, dtype=np.float64).reshape(3, 1), nu=0.0,
                           index=eb.IndexArrays(indt.reshape(3, 1, 1), indt))


def no_constraints():
    import paper_1911_03973_b200 as eb
    return eb.DirichletData(np.array([], dtype=np.int64), np.array([]))


def test_richardson_exact_with_tight_bounds(gpu):
    import paper_1911_03973_b200 as eb
    batch = diagonal_batch([2.0, 2.0, 2.0], [1.0, 0.0, 0.0])
    x, hist = eb.richardson(batch, no_constraints(), np.zeros(3), eb.SpectralBounds(2.0, 2.0), 1)
    npt.assert_array_equal(to_np(x), [0.5, 0.0, 0.0])
    assert hist.residual_norms[-1] == 0.0


def test_richardson_contraction_rate(gpu):
    import paper_1911_03973_b200 as eb
    batch = diagonal_batch([1.0, 3.0, 1.0], [0.0, 0.0, 0.0])
    d = eb.DirichletData(np.array([2]), np.array([0.0]))
    _, hist = eb.richardson(batch, d, np.array([1.0, 1.0, 0.0]), eb.SpectralBounds(1.0, 3.0), 3,
                            reference=np.zeros(3))
    npt.assert_allclose(hist.error_norms[1:] / hist.error_norms[:-1], 0.5, rtol=1e-14)


def test_cg_and_pcg_solve_diagonal_system_in_one_step(gpu):
    import paper_1911_03973_b200 as eb
    batch = diagonal_batch([2.0, 4.0, 8.0], [1.0, 1.0, 1.0])
    for solver in (eb.pcg, eb.cg):
        x, h = solver(batch, no_constraints(), np.zeros(3), 5)
        npt.assert_allclose(to_np(x), [0.5, 0.25, 0.125], rtol=1e-15)
        assert not h.diverged and h.residual_norms[-1] <= 1e-15
    # PCG with the exact (diagonal) preconditioner converges in one iteration
    _, h = eb.pcg(batch, no_constraints(), np.zeros(3), 5, tol=1e-14)
    assert h.iterations == 1
    x, h = eb.jacobi(batch, no_constraints(), np.zeros(3), 1, omega=1.0)
    npt.assert_array_equal(to_np(x), [0.5, 0.25, 0.125])


def test_unconstrained_problem_and_empty_dirichlet(gpu):
    import paper_1911_03973_b200 as eb
    m = eb.build_unit_square_mesh(3)
    batch = eb.build_element_batch(m, nu=1.0)
    x, h = eb.pcg(batch, no_constraints(), np.zeros(m.n_nodes), 500, tol=1e-10)
    # pure Neumann with nu > 0: (K + M) u = b with f = 1 -> u = 1
    npt.assert_allclose(to_np(x), 1.0, atol=1e-9)
    r = eb.mask_dirichlet(eb.residual(batch, x), no_constraints())
    assert float(r.abs().max()) <= 1e-10


def test_empty_and_ragged_meshes(gpu):
    import paper_1911_03973_b200 as eb
    # nodes without elements (ragged): isolated nodes get r = 0 and never move
    nodes = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [5.0, 5.0], [6.0, 6.0]])
    m = eb.Mesh(nodes, np.array([[0, 1, 2]]), np.array([0]))
    batch = eb.build_element_batch(m, nu=1.0)
    r = to_np(eb.residual(batch, np.array([1.0, 2.0, 3.0, 4.0, 5.0])))
    assert r[3] == 0.0 and r[4] == 0.0
    b = to_np(eb.assemble_rhs(batch.b_e, batch.index))
    npt.assert_array_equal(b[3:], [0.0, 0.0])
    x, h = eb.jacobi(batch, eb.DirichletData(np.array([0]), np.array([0.0])),
                     np.array([0.0, 0.0, 0.0, 7.0, 8.0]), 3)
    npt.assert_array_equal(to_np(x)[3:], [7.0, 8.0])
    # no elements at all
    m0 = eb.Mesh(nodes[:2], np.zeros((0, 3), dtype=np.int64), np.array([], dtype=np.int64))
    b0 = eb.build_element_batch(m0)
    assert b0.n_elements == 0
    npt.assert_array_equal(to_np(eb.residual(b0, np.array([1.0, 2.0]))), [0.0, 0.0])


@pytest.mark.parametrize("k", [40, 255, 300])
def test_single_element_tetra_and_large_valence(gpu, k):
    import paper_1911_03973_b200 as eb
    import oracle as o
    # a fan of k triangles around one node (above the structured 6; 255 is the largest
    # valence the one-byte valence array holds, 300 takes the int32 one)
    ang = np.linspace(0, 2 * np.pi, k, endpoint=False)
    nodes = np.vstack([[0.0, 0.0], np.column_stack([np.cos(ang), np.sin(ang)])])
    el = np.array([[0, 1 + i, 1 + (i + 1) % k] for i in range(k)])
    m = eb.Mesh(nodes, el, np.arange(1, k + 1))
    batch = eb.build_element_batch(m, nu=0.5)
    _, _, A, b_e = o.element_matrices(nodes, el, nu=0.5)
    x = np.random.default_rng(0).uniform(-1, 1, len(nodes))
    npt.assert_array_equal(to_np(eb.residual(batch, x)),
                           o.residual(A, b_e, np.ascontiguousarray(el.T), x))
    assert batch.operator().info()["max_valence"] == k
    npt.assert_array_equal(to_np(eb.matvec(batch, x)),
                           o.matvec_masked(A, np.ascontiguousarray(el.T), x, np.zeros(0, np.int64)))
    # one tetrahedron
    t = eb.Mesh(np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]]), np.array([[0, 1, 2, 3]]),
                np.array([0]))
    bt = eb.build_element_batch(t, nu=1.0)
    _, _, A, b_e = o.element_matrices(to_np(t.nodes), np.array([[0, 1, 2, 3]]), nu=1.0)
    npt.assert_array_equal(to_np(bt.A_e), A)
    npt.assert_array_equal(to_np(eb.residual(bt, np.ones(4))),
                           o.residual(A, b_e, np.array([[0], [1], [2], [3]]), np.ones(4)))
