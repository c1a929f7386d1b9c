"""the reference's Chebyshev two-/three-level solvers and spectral
bounds on the device, against the reference's own outputs (tests/golden/chebyshev.npz,
spectrum.npz).  Iterates are bit-identical; spectral estimates agree to rounding of the
(differently ordered) dot products."""

import numpy as np
import numpy.testing as npt
import pytest

from conftest import golden, to_np

pytestmark = pytest.mark.gpu


def problem(level, nu=0.0):
    import paper_1911_03973_b200 as eb
    m = eb.build_unit_square_mesh(level)
    return m, eb.build_element_batch(m, nu=nu), eb.constant_dirichlet(m, 1.0)


@pytest.mark.parametrize("level", [2, 3])
def test_chebyshev_iterates_bitwise(gpu, level):
    import paper_1911_03973_b200 as eb
    g = golden("chebyshev")
    m, batch, d = problem(level)
    bounds = eb.model_eigen_bounds(2**level + 1)
    x0 = np.ones(m.n_nodes)
    for N in (1, 4, 8):
        xs = []
        _, h = eb.chebyshev2(batch, d, x0, bounds, N, 20,
                             callback=lambda k, x, r: xs.append(to_np(x).copy()))
        npt.assert_array_equal(np.stack(xs), g[f"cheb2_l{level}_N{N}_iterates"])
        npt.assert_allclose(h.residual_norms, g[f"cheb2_l{level}_N{N}_norms"], rtol=1e-12)
        x2, h2 = eb.chebyshev2(batch, d, x0, bounds, N, 20)       # device-resident loop
        npt.assert_array_equal(to_np(x2), g[f"cheb2_l{level}_N{N}_iterates"][-1])
    xs = []
    _, h = eb.chebyshev3(batch, d, x0, bounds, 16,
                         callback=lambda k, x, r: xs.append(to_np(x).copy()))
    npt.assert_array_equal(np.stack(xs), g[f"cheb3_l{level}_iterates"])
    npt.assert_allclose(h.residual_norms, g[f"cheb3_l{level}_norms"], rtol=1e-12)
    x, h = eb.chebyshev3(batch, d, x0, bounds, 500, tol=1e-6)
    npt.assert_array_equal(to_np(x), g[f"cheb3_l{level}_tol_x"])
    assert len(h.residual_norms) == len(g[f"cheb3_l{level}_tol_norms"])
    assert h.residual_norms[-1] <= 1e-6 * h.residual_norms[0]


def test_richardson_equals_single_root_cycle_bitwise(gpu):
    # criterion 5 (test_acceptance.py:123-136)
    import paper_1911_03973_b200 as eb
    m, batch, d = problem(3)
    bounds = eb.model_eigen_bounds(9)
    xs_r, xs_c = [], []
    eb.richardson(batch, d, np.ones(m.n_nodes), bounds, 50,
                  callback=lambda k, x, r: xs_r.append(to_np(x).copy()))
    eb.chebyshev2(batch, d, np.ones(m.n_nodes), bounds, 1, 50,
                  callback=lambda k, x, r: xs_c.append(to_np(x).copy()))
    assert len(xs_r) == len(xs_c) == 51
    for a, b in zip(xs_r, xs_c):
        npt.assert_array_equal(a, b)


@pytest.mark.parametrize("level", [2, 3])
@pytest.mark.parametrize("N", [2, 4, 8])
def test_cycle_end_agreement(gpu, level, N):
    # criterion 4 (test_acceptance.py:107-120)
    import paper_1911_03973_b200 as eb
    m, batch, d = problem(level)
    bounds = eb.model_eigen_bounds(2**level + 1)
    x0 = np.ones(m.n_nodes)
    x2, _ = eb.chebyshev2(batch, d, x0, bounds, N, N)
    x3, _ = eb.chebyshev3(batch, d, x0, bounds, N)
    assert np.linalg.norm(to_np(x2) - to_np(x3)) <= 1e-8 * np.linalg.norm(to_np(x3))


def test_chebyshev_divergence_and_validation(gpu):
    import paper_1911_03973_b200 as eb
    m, batch, d = problem(2)
    bad = eb.SpectralBounds(1e-4, 2e-4)
    for run in (lambda: eb.chebyshev2(batch, d, np.ones(m.n_nodes), bad, 4, 300),
                lambda: eb.chebyshev3(batch, d, np.ones(m.n_nodes), bad, 300)):
        _, h = run()
        assert h.diverged and not np.isfinite(h.residual_norms[-1])
    with pytest.raises(ValueError):
        eb.chebyshev3(batch, d, np.ones(m.n_nodes), eb.SpectralBounds(2.0, 2.0), 5)
    with pytest.raises(ValueError):
        eb.chebyshev2(batch, d, np.ones(m.n_nodes), bad, 0, 5)


@pytest.mark.parametrize("level,nu", [(3, 1.0), (4, 2.5)])
def test_spectral_bounds_match_reference(gpu, level, nu):
    import paper_1911_03973_b200 as eb
    g = golden("spectrum")
    m, batch, d = problem(level, nu)
    tag = f"l{level}_nu{nu}"
    lam = eb.power_iteration_lambda_max(batch, d)
    assert abs(lam - float(g[f"power_{tag}"])) <= 1e-9 * abs(float(g[f"power_{tag}"]))
    lam10 = eb.power_iteration_lambda_max(batch, d, iters=10, seed=3)
    assert abs(lam10 - float(g[f"power10_{tag}"])) <= 1e-12 * abs(float(g[f"power10_{tag}"]))
    lo, hi = eb.mass_gershgorin(batch, d)
    npt.assert_array_equal([lo, hi], g[f"gersh_{tag}"])
    b = eb.operator_bounds(batch, d, 2**level + 1, nu)
    npt.assert_allclose([b.lambda1, b.lambda2], g[f"bounds_{tag}"], rtol=1e-9)
    dense = g[f"dense_{tag}"]
    assert b.lambda1 <= dense.min() and dense.max() <= b.lambda2
    # the operator is still usable afterwards (plan reloads A_e after the M_e pass)
    r = eb.residual(batch, np.zeros(m.n_nodes))
    npt.assert_array_equal(to_np(r), to_np(eb.assemble_rhs(batch.b_e, batch.index)))
