"""Peer-memory halo and all-reduce (csrc/peer.cu, dist.PeerTransport / LocalPeerTransport).

The slab sweeps push their interface partials into the neighbours' windows from the SELL
epilogue and the combine kernels wait for the neighbours' epoch flags; the dot all-reduce
adds the ranks' slots in rank order.  On the one GPU of the box:

* P = 2..5 slabs emulated in one process (LocalPeerTransport: the same windows, kernels and
  flags as the IPC transport, every put before any get) against the device-copy transport:
  setup halos (b, diag) and damped-Jacobi iterates BITWISE (the shared nodes are summed in
  the same ascending rank order), norms within 1e-12; single- and two-reduction PCG against
  the oracle (same iteration count to 1e-8, solution within 1e-8); the caller-order residual
  bitwise; CUDA-graph replay bitwise equal to eager;
* two and three real processes on the one GPU mapping each other's windows through CUDA IPC
  (PeerTransport, serialize=True: a host barrier after every put phase, so no kernel waits
  on the other process) against the single-GPU solvers;
* a wait that never completes times out on the device and is reported (EBS_ENCCL)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from conftest import to_np

import oracle as o

pytestmark = pytest.mark.gpu

# a broken exchange fails the test in a minute instead of the 600 s production default
os.environ.setdefault("EBS_PEER_TIMEOUT", "60")


def _oracle_pcg(cfg, size, seed, iters, tol):
    inp = o.config_inputs(cfg, seed=seed, size=size)
    _, _, A, b_e = o.element_matrices(inp["nodes"], inp["elements"], nu=inp["nu"],
                                      f_vals=inp["f_vals"])
    indt = np.ascontiguousarray(inp["elements"].T)
    return o.pcg(A, b_e, indt, inp["dirichlet"], np.zeros(len(inp["nodes"])), iters, tol=tol)


@pytest.mark.parametrize("P", [2, 3, 5])
def test_peer_jacobi_bitwise_vs_device_copy(gpu, P):
    from paper_1911_03973_b200 import dist
    from paper_1911_03973_b200.inputs import config_problem
    for cfg, size in ((4, 6), (5, 6)):
        pr = config_problem(cfg, seed=2, size=size)
        m = pr["mesh"]
        ref, _ = dist.emulate(pr["batch"], m.n_nodes, pr["dirichlet"], P)
        peer, _ = dist.emulate(pr["batch"], m.n_nodes, pr["dirichlet"], P, peer=True)
        assert isinstance(peer.comm, dist.LocalPeerTransport)
        for a, b in zip(ref.b, peer.b):
            assert torch.equal(a, b)
        for a, b in zip(ref.dinv, peer.dinv):
            assert torch.equal(a, b)
        x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
        xr, nr = dist.jacobi(ref, [op.to_internal(x0) for op in ref.ops], 40, 0.8)
        xin = [op.to_internal(x0) for op in peer.ops]
        xp, npe = dist.jacobi(peer, xin, 40, 0.8)
        for a, b in zip(xr, xp):
            assert torch.equal(a, b), (cfg, P)
        np.testing.assert_allclose(npe, nr, rtol=1e-12)
        xg, ng = dist.jacobi(peer, xin, 40, 0.8, graph=True)
        for a, b in zip(xg, xp):
            assert torch.equal(a, b)
        np.testing.assert_array_equal(ng, npe)
        assert not peer.diverged
        peer.comm.status()


@pytest.mark.parametrize("level,P", [(2, 8), (3, 7), (2, 5)])
def test_peer_thin_slabs_many_sharers(gpu, level, P):
    """Slabs thinner than a row of cells: shared nodes touched by 3-5 ranks (multi-source
    combines, ranks with several neighbours, tiny grids where no warp has a chunk fewer)."""
    import paper_1911_03973_b200 as eb
    from paper_1911_03973_b200 import dist
    m = eb.build_unit_square_mesh(level)
    batch = eb.build_element_batch(m, nu=1.0)
    d = eb.constant_dirichlet(m, 0.0)
    maps = dist.partition_maps(batch.index.indt, m.n_nodes, P)
    sharers = torch.zeros(m.n_nodes, dtype=torch.int64)
    for loc in maps["local"]:
        sharers[loc.cpu()] += 1
    assert int(sharers.max()) >= 3
    ref, _ = dist.emulate(batch, m.n_nodes, d, P)
    peer, _ = dist.emulate(batch, m.n_nodes, d, P, peer=True)
    x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
    xr, nr = dist.jacobi(ref, [op.to_internal(x0) for op in ref.ops], 25, 0.8)
    xp, npe = dist.jacobi(peer, [op.to_internal(x0) for op in peer.ops], 25, 0.8, graph=True)
    for a_, b_ in zip(xr, xp):
        assert torch.equal(a_, b_)
    np.testing.assert_allclose(npe, nr, rtol=1e-12)
    x1, h1 = eb.pcg(batch, d, x0, 500, tol=1e-10)
    xs, ns = dist.pcg(peer, [op.to_internal(x0) for op in peer.ops], 500, tol=1e-10)
    assert len(ns) == len(h1.residual_norms)
    xg = dist.gather_global(peer.ops, xs, m.n_nodes, peer.comm)
    assert float((xg - x1).norm()) <= 1e-8 * float(x1.norm())
    peer.comm.status()
    peer.comm.close()


@pytest.mark.parametrize("P", [2, 4])
def test_peer_pcg_matches_oracle(gpu, P):
    from paper_1911_03973_b200 import dist
    from paper_1911_03973_b200.inputs import config_problem
    for cfg, size in ((4, 6), (5, 8)):
        pr = config_problem(cfg, seed=2, size=size)
        m = pr["mesh"]
        prob, _ = dist.emulate(pr["batch"], m.n_nodes, pr["dirichlet"], P, peer=True)
        x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
        xin = [op.to_internal(x0) for op in prob.ops]
        xo, ho = _oracle_pcg(cfg, size, 2, 2000, 1e-8)
        for red in (1, 2):
            xs, norms = dist.pcg(prob, xin, 2000, tol=1e-8, reductions=red)
            assert not prob.diverged
            assert len(norms) == len(ho["residual_norms"]), (cfg, red, len(norms))
            np.testing.assert_allclose(norms, ho["residual_norms"], rtol=1e-6)
            xg = to_np(dist.gather_global(prob.ops, xs, m.n_nodes, prob.comm))
            assert np.linalg.norm(xg - xo) <= 1e-8 * np.linalg.norm(xo), (cfg, red)
        # device-decided tolerance, CUDA-graph batches: bitwise the eager run
        xe, ne = dist.pcg(prob, xin, 2000, tol=1e-8, graph=False)
        xgr, ngr = dist.pcg(prob, xin, 2000, tol=1e-8, graph=True)
        np.testing.assert_array_equal(ngr, ne)
        for a, b in zip(xgr, xe):
            assert torch.equal(a, b)
        prob.comm.status()


@pytest.mark.parametrize("P", [2, 3])
def test_peer_residual_caller_order(gpu, P):
    import paper_1911_03973_b200 as eb
    from paper_1911_03973_b200 import dist
    from paper_1911_03973_b200.inputs import config_problem
    pr = config_problem(2, seed=5, size=7)
    m = pr["mesh"]
    batch = pr["batch"]
    x = torch.from_numpy(pr["x"]).cuda()
    out = []
    for peer in (False, True):
        prob, _ = dist.emulate(batch, m.n_nodes, None, P, peer=peer)
        xl = [x[op.global_ids].contiguous() for op in prob.ops]
        rl = [op.zeros() for op in prob.ops]
        dist.residual_local(prob, xl, rl, [op.zeros() for op in prob.ops],
                            [op.zeros() for op in prob.ops])
        out.append((prob, rl))
    # the large-slab variant of the peer sweep (red.add into a -0.0-filled r): same bits
    pb = out[1][0]
    try:
        dist.GpuRankOperator.PEER_RED_MIN_NODES = 0
        xl = [x[op.global_ids].contiguous() for op in pb.ops]
        ra_ = [torch.full_like(r_, float("nan")) for r_ in out[1][1]]
        dist.residual_local(pb, xl, ra_, [op.zeros() for op in pb.ops], [None] * P)
    finally:
        dist.GpuRankOperator.PEER_RED_MIN_NODES = 3 << 20
    for op, a, b in zip(pb.ops, ra_, out[1][1]):
        own = op.owned_local
        assert torch.equal(a[own], b[own])
    ref = eb.residual(batch, x, deterministic=False)
    (pa, ra), (pb, rb) = out
    for op, a, b in zip(pb.ops, ra, rb):
        own = op.owned_local
        assert torch.equal(a[own], b[own])
        gids = op.global_ids[own]
        assert float((b[own] - ref[gids]).abs().max()) <= 1e-12 * float(ref.abs().max())
    # the global-vector variant through the generic peer send / recv (ebs_peer_send/_recv)
    rg = []
    for prob in (pa, pb):
        r_ = [torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda") for _ in prob.ops]
        dist.residual_caller(prob, x, r_, [op.zeros() for op in prob.ops],
                             [op.zeros() for op in prob.ops])
        rg.append(r_)
    for op, a, b in zip(pb.ops, rg[0], rg[1]):
        gids = op.global_ids[op.owned_local]
        assert torch.equal(a[gids], b[gids])
    pb.comm.status()


def test_peer_allreduce_rank_order(gpu):
    """Sum over 5 emulated ranks of 600 values (3 launches of 256), added in rank order."""
    from paper_1911_03973_b200 import dist
    from paper_1911_03973_b200.inputs import config_problem
    pr = config_problem(4, seed=1, size=5)
    m = pr["mesh"]
    prob, _ = dist.emulate(pr["batch"], m.n_nodes, pr["dirichlet"], 5, peer=True)
    g = torch.Generator(device="cpu").manual_seed(0)
    vals = [torch.randn(600, generator=g, dtype=torch.float64).cuda() for _ in range(5)]
    want = vals[0].clone()
    for v in vals[1:]:
        want += v
    ts = [v.clone() for v in vals]
    prob.comm.allreduce(ts)
    for t in ts:
        assert torch.equal(t, want)


@pytest.mark.parametrize("cfg,size,P", [(4, 7, 2), (4, 7, 5), (5, 8, 4), (5, 8, 8)])
def test_peer_protocol_under_concurrency(gpu, cfg, size, P):
    """ebs_peer_selftest: the ranks' pushes, flag waits, rank-ordered sums and fused
    all-reduces run CONCURRENTLY in one cooperative kernel (block groups as ranks, skewed so
    fast ranks run into the next epoch while slow ones still read), 300 rounds, every value
    checked -- the double-buffering / epoch / fence protocol of the multi-GPU path."""
    from paper_1911_03973_b200 import dist
    from paper_1911_03973_b200.inputs import config_problem
    pr = config_problem(cfg, seed=1, size=size)
    m = pr["mesh"]
    prob, _ = dist.emulate(pr["batch"], m.n_nodes, pr["dirichlet"], P, peer=True)
    assert prob.comm.selftest(300) == 0
    prob.comm.status()
    # the windows are still consistent for the solvers afterwards
    x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
    xs, norms = dist.jacobi(prob, [op.to_internal(x0) for op in prob.ops], 10, 0.8)
    assert np.all(np.isfinite(norms)) and not prob.diverged
    prob.comm.close()


def test_peer_transport_world_one(gpu):
    """PeerTransport in a single process (world 1, no torch.distributed): its own window
    through the IPC-handle path, the one-launch all-reduce (mode 0: put + get in one kernel,
    the form every real multi-GPU Jacobi norm / two-reduction PCG / gather uses), the fused
    loops -- against the single-GPU solvers."""
    import paper_1911_03973_b200 as eb
    from paper_1911_03973_b200 import dist
    from paper_1911_03973_b200.inputs import config_problem
    for cfg, size in ((4, 6), (5, 8)):
        pr = config_problem(cfg, seed=4, size=size)
        m = pr["mesh"]
        op, _ = dist.rank_operator(m, pr["nu"], pr["f"], pr["dirichlet"], 1, 0)
        comm = dist.PeerTransport(op, timeout=60)
        assert comm.world == 1
        prob = dist.setup([op], comm)
        x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
        t = torch.arange(600, dtype=torch.float64, device="cuda")
        comm.allreduce([t])  # 3 launches of mode 0 on one rank: the identity
        assert torch.equal(t, torch.arange(600, dtype=torch.float64, device="cuda"))
        if cfg == 4:
            xs, norms = dist.jacobi(prob, [op.to_internal(x0)], 30, 0.8, graph=True)
            x1, h1 = eb.jacobi(pr["batch"], pr["dirichlet"], x0, 30, omega=0.8)
            np.testing.assert_allclose(norms, h1.residual_norms, rtol=1e-12)
        else:
            for red in (1, 2):
                xs, norms = dist.pcg(prob, [op.to_internal(x0)], 500, tol=1e-8, reductions=red)
                x1, h1 = eb.pcg(pr["batch"], pr["dirichlet"], x0, 500, tol=1e-8)
                assert len(norms) == len(h1.residual_norms)
        xg = dist.gather_global([op], xs, m.n_nodes, comm).cpu().numpy()
        x1 = x1.cpu().numpy()
        assert np.linalg.norm(xg - x1) <= 1e-10 * np.linalg.norm(x1)
        comm.status()
        comm.close()


def test_peer_window_open_failure_is_reported(gpu):
    """A handle that maps nothing fails loudly (EbsError) -- PeerTransport turns that into a
    collective PeerUnavailable so the bench falls back to NCCL on every rank together."""
    import ctypes

    from paper_1911_03973_b200._lib import EbsError, call
    w = ctypes.c_void_p()
    with pytest.raises(EbsError):
        call("ebs_peer_window_open", ctypes.create_string_buffer(b"\x00" * 64, 64),
             ctypes.byref(w))


def test_failed_allocation_leaves_no_stale_error(gpu):
    """A device allocation that fails (a window of 2^36 doubles per slot) raises MemoryError,
    and the next library call works: the non-sticky CUDA error is cleared where it is
    reported (ebs_internal.cuh CU), not picked up by an unrelated later launch check."""
    import ctypes

    import paper_1911_03973_b200 as eb
    from paper_1911_03973_b200._lib import call
    w = ctypes.c_void_p()
    with pytest.raises(MemoryError):
        call("ebs_peer_window_alloc", 1 << 36, ctypes.byref(w), None)
    m = eb.build_unit_square_mesh(3)
    batch = eb.build_element_batch(m, nu=1.0)
    r = eb.residual(batch, torch.ones(m.n_nodes, dtype=torch.float64, device="cuda"))
    assert torch.isfinite(r).all()


def test_peer_wait_times_out(gpu):
    """A combine whose neighbour never publishes: the device wait gives up after the
    timeout, sets the window's error word, and the transport raises instead of hanging."""
    from paper_1911_03973_b200 import dist
    from paper_1911_03973_b200._lib import EbsError
    from paper_1911_03973_b200.inputs import config_problem
    pr = config_problem(4, seed=1, size=5)
    m = pr["mesh"]
    maps = dist.partition_maps(pr["batch"].index.indt, m.n_nodes, 2)
    ops = [dist.GpuRankOperator(pr["batch"], m.n_nodes, pr["dirichlet"], maps, p)
           for p in range(2)]
    comm = dist.LocalPeerTransport(ops, timeout=0.2)
    v = ops[0].zeros()
    torch.cuda.synchronize()
    ops[0].peer_combine(v)  # rank 1 never pushed
    with pytest.raises(EbsError, match="timed out"):
        comm.status()
    comm.close()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _ipc_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as tdist
    from paper_1911_03973_b200 import dist as D
    from paper_1911_03973_b200.inputs import config_problem
    torch.cuda.set_device(0)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = {}
        for cfg, size in ((4, 6), (3, 6)):
            p = config_problem(cfg, seed=3, size=size)
            batch, d, m = p["batch"], p["dirichlet"], p["mesh"]
            maps = D.partition_maps(batch.index.indt, m.n_nodes, world)
            op = D.GpuRankOperator(batch, m.n_nodes, d, maps, rank)
            comm = D.PeerTransport(op, serialize=True, timeout=60)
            prob = D.setup([op], comm)
            x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
            if cfg == 4:
                xs, norms = D.jacobi(prob, [op.to_internal(x0)], 30, 0.8)
            else:
                xs, norms = D.pcg(prob, [op.to_internal(x0)], 500, tol=1e-8)
            xg = D.gather_global([op], xs, m.n_nodes, comm)
            res[cfg] = (xg.cpu().numpy(), norms)
            comm.close()
        if rank == 0:
            out.put(res)
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_processes_cuda_ipc_windows(gpu, world):
    """world 3: the middle rank maps and writes two neighbours' windows."""
    import paper_1911_03973_b200 as eb
    from paper_1911_03973_b200.inputs import config_problem
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for cfg, size in ((4, 6), (3, 6)):
        pr = config_problem(cfg, seed=3, size=size)
        x0 = torch.zeros(pr["mesh"].n_nodes, dtype=torch.float64, device="cuda")
        if cfg == 4:
            x1, h1 = eb.jacobi(pr["batch"], pr["dirichlet"], x0, 30, omega=0.8)
            np.testing.assert_allclose(res[cfg][1], h1.residual_norms, rtol=1e-10)
        else:
            x1, h1 = eb.pcg(pr["batch"], pr["dirichlet"], x0, 500, tol=1e-8)
            assert len(res[cfg][1]) == len(h1.residual_norms)
        x1 = x1.cpu().numpy()
        assert np.linalg.norm(res[cfg][0] - x1) <= 1e-8 * np.linalg.norm(x1)
