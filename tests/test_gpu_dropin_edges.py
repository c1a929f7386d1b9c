"""Drop-in edges of the public API: the reference's top-level
names, fresh callback tensors per iteration (solvers.py:137-149 hands a new x and r at
every k), and a non-finite x0 raising ValueError like _iterate's first residual()
(operators.py:90)."""

import numpy as np
import pytest
import torch

from conftest import golden, to_np

pytestmark = pytest.mark.gpu


def _problem(level=3):
    import paper_1911_03973_b200 as eb
    m = eb.build_unit_square_mesh(level)
    batch = eb.build_element_batch(m, nu=1.0)
    return eb, m, batch, eb.constant_dirichlet(m, 0.0)


def test_callback_tensors_are_fresh_per_iteration(gpu):
    eb, m, batch, d = _problem()
    bounds = eb.model_eigen_bounds(9)
    g = golden("richardson_l3")
    m3, b3, d3 = m, eb.build_element_batch(m, nu=0.0), eb.constant_dirichlet(m, 1.0)
    xs, rs = [], []
    eb.richardson(b3, d3, np.ones(m3.n_nodes), bounds, 20,
                  callback=lambda k, x, r: (xs.append(x), rs.append(r)))  # no copy
    assert len({t.data_ptr() for t in xs}) == len(xs) == 21
    npt_equal = np.testing.assert_array_equal
    npt_equal(np.stack([to_np(x) for x in xs]), g["iterates"])  # every k kept its own x
    assert all(not torch.equal(xs[k], xs[k + 1]) for k in range(len(xs) - 1))
    x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
    for solver in (eb.pcg, eb.cg, eb.jacobi):
        xs = []
        solver(batch, d, x0, 6, callback=lambda k, x, r: xs.append(x))
        assert len({t.data_ptr() for t in xs}) == 7, solver.__name__
        assert all(not torch.equal(xs[k], xs[k + 1]) for k in range(1, 6)), solver.__name__
    # opt-in: the same two buffers every time (no per-iteration copy)
    xs = []
    eb.pcg(batch, d, x0, 4, callback=lambda k, x, r: xs.append(x), reuse_callback_buffers=True)
    assert len({t.data_ptr() for t in xs}) == 1


def test_nonfinite_x0_raises(gpu):
    eb, m, batch, d = _problem()
    x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
    x0[7] = float("nan")
    bounds = eb.model_eigen_bounds(9)
    calls = []
    for run in (lambda **kw: eb.pcg(batch, d, x0, 5, **kw),
                lambda **kw: eb.jacobi(batch, d, x0, 5, **kw),
                lambda **kw: eb.richardson(batch, d, x0, bounds, 5, **kw)):
        with pytest.raises(ValueError, match="non-finite"):
            run()
        with pytest.raises(ValueError, match="non-finite"):
            run(callback=lambda k, x, r: calls.append(k))
    assert calls == []  # raised before the first callback, as the reference does
    x0[7] = 0.0  # the plan is usable afterwards
    _, h = eb.pcg(batch, d, x0, 5)
    assert h.iterations == 5 and not h.diverged


def test_reference_top_level_names():
    import paper_1911_03973_b200 as eb
    for name in ("ExperimentConfig", "ExperimentReport", "run_experiment"):
        assert name in eb.__all__ and hasattr(eb, name)
