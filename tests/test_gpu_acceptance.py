"""The reference's acceptance criteria (tests/test_acceptance.py of ebsolve) run on the
device: 1 (residual vs assembled oracle), 5 (bitwise Richardson == Chebyshev N=1, also in
test_gpu_chebyshev_spectrum), 6 (three-level error bound), 7 (exactness and boundary
invariants), 8 (level-8 experiment time and byte-identical outputs for any `threads`)."""

import time

import numpy as np
import pytest
import torch

from conftest import to_np

import oracle as o

pytestmark = pytest.mark.gpu


def problem(level, nu=0.0):
    import paper_1911_03973_b200 as eb
    m = eb.build_unit_square_mesh(level)
    batch = eb.build_element_batch(m, nu=nu)
    return m, batch, eb.constant_dirichlet(m, 1.0), eb.assemble_rhs(batch.b_e, batch.index)


def test_criterion_1_residual_vs_assembled(gpu):
    import paper_1911_03973_b200 as eb
    t0 = time.perf_counter()
    rng = np.random.default_rng(2024)
    for level in (1, 2, 3, 4, 5):
        for nu in (0.0, 1.0):
            m, batch, _, b = problem(level, nu)
            A = eb.assemble_sparse(batch.A_e, batch.index)
            for _ in range(20):
                x = torch.from_numpy(rng.standard_normal(m.n_nodes)).cuda()
                r = eb.residual(batch, x)
                r_ref = b - torch.mv(A, x)
                assert float(torch.linalg.vector_norm(r - r_ref)) <= \
                    1e-12 * float(torch.linalg.vector_norm(r_ref))
    assert time.perf_counter() - t0 < 10.0


def test_criterion_6_three_level_error_bound(gpu):
    import paper_1911_03973_b200 as eb
    for level in (2, 3):
        m, batch, d, b = problem(level)
        bounds = eb.model_eigen_bounds(2**level + 1)
        u, _ = eb.pcg(batch, d, torch.ones(m.n_nodes, dtype=torch.float64, device="cuda"), 1000,
                      tol=1e-14)
        s1, s2 = np.sqrt(bounds.lambda1), np.sqrt(bounds.lambda2)
        rho = (s2 - s1) / (s2 + s1)
        for N in (4, 8, 16):
            x, hist = eb.chebyshev3(batch, d, np.ones(m.n_nodes), bounds, N, reference=u)
            assert hist.error_norms[-1] <= 2.0 * rho**N * hist.error_norms[0] * (1.0 + 1e-6)


def test_criterion_7_exactness_and_boundary_invariants(gpu):
    import paper_1911_03973_b200 as eb
    for level in (1, 2, 3, 4, 5):
        _, batch, _, _ = problem(level)
        assert float(batch.K_e.sum(dim=1).abs().max()) <= 1e-14
    _, batch, _, _ = problem(4)
    M = eb.assemble_sparse(batch.M_e, batch.index)
    assert abs(float(M.values().sum()) - 1.0) <= 1e-14
    m, batch, d, _ = problem(3)
    bounds = eb.model_eigen_bounds(9)

    def pinned(k, x, r):
        assert bool((x[d.nd] == 1.0).all())

    eb.richardson(batch, d, np.ones(m.n_nodes), bounds, 20, callback=pinned)
    eb.chebyshev2(batch, d, np.ones(m.n_nodes), bounds, 8, 20, callback=pinned)
    eb.chebyshev3(batch, d, np.ones(m.n_nodes), bounds, 20, callback=pinned)


def test_criterion_8_level8_runtime_and_determinism(gpu, tmp_path):
    from paper_1911_03973_b200.cli import ExperimentConfig, run_experiment
    out1, out4 = tmp_path / "threads1", tmp_path / "threads4"
    t0 = time.perf_counter()
    report = run_experiment(ExperimentConfig(level=8, solver="all", out_dir=str(out1), threads=1))
    dt = time.perf_counter() - t0
    assert dt < 60.0 and not report.any_diverged
    run_experiment(ExperimentConfig(level=8, solver="all", out_dir=str(out4), threads=4))
    names = sorted(p.name for p in out1.iterdir())
    assert names == sorted(p.name for p in out4.iterdir()) and len(names) == 7
    for name in names:
        assert (out1 / name).read_bytes() == (out4 / name).read_bytes(), name


def test_zero_iterations_all_solvers(gpu):
    import paper_1911_03973_b200 as eb
    m, batch, d, _ = problem(3, nu=1.0)
    x0 = torch.ones(m.n_nodes, dtype=torch.float64, device="cuda")
    for solver in (eb.jacobi, eb.cg, eb.pcg):
        x, h = solver(batch, d, x0, 0)
        assert len(h.residual_norms) == 1 and torch.equal(x, x0) and x.data_ptr() != x0.data_ptr()
        with pytest.raises(ValueError):
            solver(batch, d, x0, -1)
