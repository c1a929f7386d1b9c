"""Oracle restatements the reference lacks (Jacobi, CG/PCG, diag, halo maps), pinned
against the reference's direct solver and SciPy cg outputs in tests/golden.  CPU only."""

import numpy as np
import numpy.testing as npt
import pytest

from conftest import golden

import oracle as o


def c1_system(level=6, nu=1.0):
    nodes, elements, boundary = o.unit_square_mesh(level)
    _, _, A, b_e = o.element_matrices(nodes, elements, nu=nu)
    return nodes, np.ascontiguousarray(elements.T), boundary, A, b_e


def test_pcg_c1_matches_direct_solution():
    g = golden("c1_solution")
    nodes, indt, nd, A, b_e = c1_system()
    x0 = np.zeros(len(nodes))
    x, h = o.pcg(A, b_e, indt, nd, x0, 10_000, tol=1e-8)
    assert not h["diverged"]
    assert h["residual_norms"][-1] <= 1e-8 * h["residual_norms"][0]
    u = g["u_direct"]
    err = np.linalg.norm(x - u) / np.linalg.norm(u)
    assert err <= 1e-7, err
    # SciPy's Jacobi-PCG on the eliminated system takes (almost) the same count
    assert abs((len(h["residual_norms"]) - 1) - int(g["scipy_pcg_iters"])) <= 2
    npt.assert_allclose(x, g["u_scipy_pcg"], rtol=0, atol=1e-7 * np.abs(u).max())
    # exact-solve tolerance the north star asks (1e-8) after more iterations
    x2, _ = o.pcg(A, b_e, indt, nd, x0, 10_000, tol=1e-12)
    assert np.linalg.norm(x2 - u) / np.linalg.norm(u) <= 1e-10


def test_cg_and_jacobi_converge_to_direct_solution():
    g = golden("c1_solution")
    nodes, indt, nd, A, b_e = c1_system()
    x0 = np.zeros(len(nodes))
    x, h = o.cg(A, b_e, indt, nd, x0, 10_000, tol=1e-10)
    assert np.linalg.norm(x - g["u_direct"]) <= 1e-8 * np.linalg.norm(g["u_direct"])
    # damped Jacobi contracts monotonically on this SPD M-matrix
    x, h = o.jacobi(A, b_e, indt, nd, x0, 0.8, 50)
    assert len(h["residual_norms"]) == 51
    assert np.all(np.diff(h["residual_norms"]) < 0)
    assert np.all(x[nd] == 0.0)


def test_pcg_3d_matches_reference_direct_solve():
    g = golden("kuhn3d")
    for N in (2, 3):
        nodes, elements, face = o.kuhn_cube_mesh(N)
        _, _, A, b_e = o.element_matrices(nodes, elements, nu=1.0)
        indt = np.ascontiguousarray(elements.T)
        x, h = o.pcg(A, b_e, indt, face, np.zeros(len(nodes)), 1000, tol=1e-13)
        u = g[f"u_N{N}"]
        assert np.linalg.norm(x - u) <= 1e-10 * np.linalg.norm(u)


def test_pcg_loop_semantics():
    nodes, indt, nd, A, b_e = c1_system(level=3)
    x0 = np.zeros(len(nodes))
    ks = []
    x, h = o.pcg(A, b_e, indt, nd, x0, 5, callback=lambda k, x, r: ks.append(k))
    assert ks == [0, 1, 2, 3, 4, 5]
    assert len(h["residual_norms"]) == 6
    x, h = o.pcg(A, b_e, indt, nd, x0, 0)
    assert len(h["residual_norms"]) == 1 and np.all(x == x0) and x is not x0
    with pytest.raises(ValueError):
        o.pcg(A, b_e, indt, nd, x0, -1)
    # an exactly solved system stays put (alpha, beta = 0 instead of 0/0)
    x, h = o.pcg(A, np.zeros_like(b_e), indt, nd, x0, 3)
    assert not h["diverged"] and np.all(x == 0.0)


def test_diag_is_reference_gershgorin_diag_for_mass():
    # spectrum.py:118-120 sums per-j bincounts; the restated diag sums in (j, e) order.
    # They agree to rounding, exactly on dyadic meshes.
    nodes, indt, nd, A, b_e = c1_system(level=4)
    _, M, _, _ = o.element_matrices(nodes, indt.T)
    per_j = sum(np.bincount(indt[j], weights=M[j, j, :], minlength=len(nodes)) for j in range(3))
    npt.assert_allclose(o.diagonal(M, indt, len(nodes)), per_j, rtol=1e-15)


def test_halo_maps():
    nodes, elements, _ = o.unit_square_mesh(4)
    indt = np.ascontiguousarray(elements.T)
    for P in (1, 2, 3, 4):
        h = o.halo_maps(indt, P)
        assert h["bounds"][0] == 0 and h["bounds"][-1] == indt.shape[1]
        covered = np.unique(np.concatenate(h["local"]))
        npt.assert_array_equal(covered, np.arange(len(nodes)))
        for p in range(P):
            for q, common in h["interface"][p].items():
                npt.assert_array_equal(common, h["interface"][q][p])
                # row-major cells -> slabs meet along one node row (17 nodes) when
                # the slab boundary falls between cell rows, a row and a bit otherwise
                assert abs(p - q) == 1
                aligned = (indt.shape[1] // P) % 32 == 0
                assert common.size == 17 if aligned else 17 <= common.size <= 35
        assert np.all(h["owner"] >= 0)


def test_first_appearance_order_is_a_permutation():
    inp = o.config_inputs(2, seed=0, size=4)
    indt = np.ascontiguousarray(inp["elements"].T)
    new_of_old = o.first_appearance_order(indt, len(inp["nodes"]))
    npt.assert_array_equal(np.sort(new_of_old), np.arange(len(new_of_old)))
    # undoing the random permutation: internal order is the structured one up to the
    # interleaving of the first two rows
    orig = np.empty_like(inp["perm"])
    orig[inp["perm"]] = np.arange(len(orig))
    assert new_of_old[inp["perm"][0]] == 0


def test_grid_strides_of_generated_grids():
    """Unpermuted grids: differences 2D +-{1, n, n+1} (strides 1, n), 3D the 14
    Freudenthal edge offsets (strides 1, n, n^2); a random numbering has no small set of
    differences (the plan then uses first_appearance_order)."""
    _, el, _ = o.unit_square_mesh(3)
    n = 9
    npt.assert_array_equal(o.delta_alphabet(np.ascontiguousarray(el.T)),
                           [-n - 1, -n, -1, 1, n, n + 1])
    assert o.grid_strides(np.ascontiguousarray(el.T)) == (1, n)
    _, el, _ = o.kuhn_cube_mesh(3)
    n = 4
    pos = sorted({1, n, n + 1, n * n, n * n + 1, n * n + n, n * n + n + 1})
    npt.assert_array_equal(o.delta_alphabet(np.ascontiguousarray(el.T)),
                           sorted([-d for d in pos] + pos))
    assert o.grid_strides(np.ascontiguousarray(el.T)) == (1, n, n * n)
    inp = o.config_inputs(2, seed=0, size=3)
    indt = np.ascontiguousarray(inp["elements"].T)
    assert o.delta_alphabet(indt) is None and o.grid_strides(indt) is None
    npt.assert_array_equal(o.plan_numbering(indt, len(inp["nodes"])),
                           o.first_appearance_order(indt, len(inp["nodes"])))


def test_streamed_operator_is_bitwise_the_whole_mesh_operator():
    """oracle.StreamedOperator (chunked element matrices, one bincount: the reference's
    threaded deterministic mode, operators.py:96-107) == the whole-mesh functions, bit for
    bit, in 2D (jittered + permuted C4 recipe) and 3D (Kuhn cube); the solver loops give
    identical iterates through it."""
    for cfg, size in ((4, 4), (5, 3)):
        inp = o.config_inputs(cfg, seed=3, size=size)
        nodes, elements, nd = inp["nodes"], inp["elements"], inp["dirichlet"]
        _, _, A, b_e = o.element_matrices(nodes, elements, nu=inp["nu"], f_vals=inp["f_vals"])
        indt = np.ascontiguousarray(elements.T)
        op = o.StreamedOperator(nodes, elements, nu=inp["nu"], f_vals=inp["f_vals"], chunk=37,
                                threads=3)
        x = np.random.default_rng(1).uniform(-1, 1, nodes.shape[0])
        np.testing.assert_array_equal(op.residual(x), o.residual(A, b_e, indt, x))
        np.testing.assert_array_equal(o.residual(op, None, None, x), o.residual(A, b_e, indt, x))
        np.testing.assert_array_equal(op.matvec_masked(x, nd), o.matvec_masked(A, indt, x, nd))
        np.testing.assert_array_equal(op.diagonal(), o.diagonal(A, indt, nodes.shape[0]))
        np.testing.assert_array_equal(op.rhs(), o.assemble_rhs(b_e, indt, nodes.shape[0]))
        x0 = np.zeros(nodes.shape[0])
        xs, hs = o.pcg(op, None, None, nd, x0, 7)
        xw, hw = o.pcg(A, b_e, indt, nd, x0, 7)
        np.testing.assert_array_equal(xs, xw)
        np.testing.assert_array_equal(hs["residual_norms"], hw["residual_norms"])
        xs, hs = o.jacobi(op, None, None, nd, x0, 0.8, 3)
        xw, hw = o.jacobi(A, b_e, indt, nd, x0, 0.8, 3)
        np.testing.assert_array_equal(xs, xw)
