"""Single-reduction (Chronopoulos-Gear) slab PCG and the NCCL failure path.

* one all-reduce of [r.u, w.u, r.r] per iteration: same iteration count as the oracle's
  textbook PCG to 1e-8 and the solution within 1e-8, on P = 1..4 emulated slabs (2D C4
  recipe and 3D Kuhn cubes);
* the tolerance path is decided on the device: CUDA-graph batches with a tolerance give
  bit-identical iterates and histories to eager execution, with no per-iteration host read;
* a non-finite start is flagged as divergence (never raised), as _iterate does;
* libebs.so's own communicator: a stream that does not finish within the timeout aborts
  the communicator (ncclCommAbort) and returns EBS_ENCCL instead of hanging; afterwards
  every collective of the plan fails loudly until it is re-initialised."""

import numpy as np
import pytest
import torch

from conftest import to_np

import oracle as o

pytestmark = pytest.mark.gpu


def _oracle_pcg(cfg, size, seed, iters, tol):
    inp = o.config_inputs(cfg, seed=seed, size=size)
    _, _, A, b_e = o.element_matrices(inp["nodes"], inp["elements"], nu=inp["nu"],
                                      f_vals=inp["f_vals"])
    indt = np.ascontiguousarray(inp["elements"].T)
    return o.pcg(A, b_e, indt, inp["dirichlet"], np.zeros(len(inp["nodes"])), iters, tol=tol)


@pytest.mark.parametrize("P", [1, 2, 3, 4])
def test_single_reduction_pcg_matches_oracle(gpu, P):
    from paper_1911_03973_b200 import dist
    from paper_1911_03973_b200.inputs import config_problem
    for cfg, size in ((4, 6), (5, 8)):
        pr = config_problem(cfg, seed=2, size=size)
        m = pr["mesh"]
        prob, _ = dist.emulate(pr["batch"], m.n_nodes, pr["dirichlet"], P)
        x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
        xin = [op.to_internal(x0) for op in prob.ops]
        xo, ho = _oracle_pcg(cfg, size, 2, 2000, 1e-8)
        for red in (1, 2):
            xs, norms = dist.pcg(prob, xin, 2000, tol=1e-8, reductions=red)
            assert not prob.diverged
            assert len(norms) == len(ho["residual_norms"]), (cfg, red, len(norms))
            np.testing.assert_allclose(norms, ho["residual_norms"], rtol=1e-6)
            xg = to_np(dist.gather_global(prob.ops, xs, m.n_nodes))
            assert np.linalg.norm(xg - xo) <= 1e-8 * np.linalg.norm(xo), (cfg, red)


@pytest.mark.parametrize("P", [1, 3])
def test_tolerance_on_device_graph_equals_eager(gpu, P):
    from paper_1911_03973_b200 import dist
    from paper_1911_03973_b200.inputs import config_problem
    pr = config_problem(5, seed=1, size=8)
    m = pr["mesh"]
    prob, _ = dist.emulate(pr["batch"], m.n_nodes, pr["dirichlet"], P)
    x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
    xin = [op.to_internal(x0) for op in prob.ops]
    xe, ne = dist.pcg(prob, xin, 5000, tol=1e-8, graph=False)
    before = dist.GRAPH_STATS["captured"]
    xg, ng = dist.pcg(prob, xin, 5000, tol=1e-8, graph=True)
    assert dist.GRAPH_STATS["captured"] == before + 1
    np.testing.assert_array_equal(ng, ne)
    assert ne[-1] <= 1e-8 * ne[0] < ne[-2]
    for a, b in zip(xg, xe):
        assert torch.equal(a, b)
    # fixed count, iteration count not a multiple of the graph batch
    xf, nf = dist.pcg(prob, xin, 21, graph=True)
    xf2, nf2 = dist.pcg(prob, xin, 21, graph=False)
    assert len(nf) == 22
    np.testing.assert_array_equal(nf, nf2)
    # stopping exactly: the tol run's x is the fixed-count run's x at the same k
    k = len(ne) - 1
    xk, _ = dist.pcg(prob, xin, k, graph=True)
    for a, b in zip(xk, xe):
        assert torch.equal(a, b)


def test_nonfinite_start_is_divergence(gpu):
    from paper_1911_03973_b200 import dist
    from paper_1911_03973_b200.inputs import config_problem
    pr = config_problem(5, seed=1, size=6)
    m = pr["mesh"]
    prob, _ = dist.emulate(pr["batch"], m.n_nodes, pr["dirichlet"], 2)
    x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
    x0[m.n_nodes // 2] = float("nan")
    for red in (1, 2):
        _, norms = dist.pcg(prob, [op.to_internal(x0) for op in prob.ops], 50, tol=1e-8,
                            reductions=red)
        assert prob.diverged and not np.isfinite(norms[-1]) and len(norms) == 1, red
    _, norms = dist.jacobi(prob, [op.to_internal(x0) for op in prob.ops], 5)
    assert prob.diverged
    _, norms = dist.pcg(prob, [op.to_internal(torch.zeros_like(x0)) for op in prob.ops], 5)
    assert not prob.diverged


def test_native_communicator_timeout_aborts(gpu):
    from paper_1911_03973_b200 import dist
    from paper_1911_03973_b200._lib import EbsError
    from paper_1911_03973_b200.inputs import config_problem
    pr = config_problem(5, seed=2, size=4)
    m = pr["mesh"]
    op, _ = dist.rank_operator(m, pr["nu"], pr["f"], pr["dirichlet"], 1, 0)
    comm = dist.NativeTransport(op)
    comm.poll()                      # healthy communicator: no async error
    t = torch.ones(3, dtype=torch.float64, device="cuda")
    comm.allreduce([t])
    comm.sync(timeout=30.0)
    assert torch.equal(t, torch.ones_like(t))
    torch.cuda._sleep(4_000_000_000)  # ~2 s of device time: the "peer" never arrives
    with pytest.raises(EbsError, match="aborted"):
        comm.sync(timeout=0.05)
    torch.cuda.synchronize()
    with pytest.raises(EbsError, match="aborted"):
        comm.allreduce([t])
    with pytest.raises(EbsError, match="aborted"):
        comm.poll()
    comm2 = dist.NativeTransport(op)  # re-initialisation after an abort
    comm2.allreduce([t])
    comm2.sync()
    assert torch.equal(t, torch.ones_like(t))


def test_native_transport_tolerance_and_reuse(gpu):
    """libebs's own communicator (world 1) under the single-reduction loop with a
    tolerance and CUDA-graph batches: same iterates and history as the device-copy
    transport; a second solve on the same problem replays the cached graph (no new
    capture) and gives the same result; results are fresh tensors."""
    from paper_1911_03973_b200 import dist
    from paper_1911_03973_b200.inputs import config_problem
    pr = config_problem(5, seed=3, size=8)
    m = pr["mesh"]
    op, _ = dist.rank_operator(m, pr["nu"], pr["f"], pr["dirichlet"], 1, 0)
    prob_l = dist.setup([op], dist.LocalTransport())
    prob_n = dist.setup([op], dist.NativeTransport(op))
    x0 = op.zeros()
    xl, nl = dist.pcg(prob_l, [x0], 3000, tol=1e-8, graph=True)
    xn, nn = dist.pcg(prob_n, [x0], 3000, tol=1e-8, graph=True)
    np.testing.assert_array_equal(nn, nl)
    assert torch.equal(xn[0], xl[0])
    before = dist.GRAPH_STATS["captured"]
    xn2, nn2 = dist.pcg(prob_n, [x0], 3000, tol=1e-8, graph=True)
    assert dist.GRAPH_STATS["captured"] == before  # cached graph replayed
    np.testing.assert_array_equal(nn2, nn)
    assert torch.equal(xn2[0], xn[0]) and xn2[0].data_ptr() != xn[0].data_ptr()
    assert nn[-1] <= 1e-8 * nn[0] and not prob_n.diverged
