"""Multi-rank protocol on CPU: world size 2 over gloo (torch.distributed), the production
dist.py loops and TorchTransport, with the torch-CPU rank operator of tests/dist_cpu.py.
Checks the partition / halo maps against the oracle bit for bit and the distributed
residual, Jacobi and PCG against the single-process oracle."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle as o


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_partition_maps_match_oracle():
    from paper_1911_03973_b200.dist import partition_maps
    for mesh in (o.unit_square_mesh(4), o.kuhn_cube_mesh(3)):
        nodes, elements, _ = mesh
        indt = np.ascontiguousarray(elements.T)
        for P in (1, 2, 3, 4, 8):
            ref = o.halo_maps(indt, P)
            got = partition_maps(torch.from_numpy(indt).to(torch.int32), len(nodes), P)
            np.testing.assert_array_equal(got["bounds"], ref["bounds"])
            for p in range(P):
                np.testing.assert_array_equal(got["local"][p].numpy(), ref["local"][p])
                assert sorted(got["interface"][p]) == sorted(ref["interface"][p])
                for q, ids in ref["interface"][p].items():
                    np.testing.assert_array_equal(got["interface"][p][q].numpy(), ids)
            np.testing.assert_array_equal(got["owner"].numpy(), ref["owner"])


def _worker(rank, world, port, case, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from paper_1911_03973_b200 import dist as D
    from dist_cpu import CpuRankOperator
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if case == "2d":
            inp = o.config_inputs(4, seed=1, size=4)
            nodes, elements, nd = inp["nodes"], inp["elements"], inp["dirichlet"]
            nu, f_vals = 10.0, inp["f_vals"]
        else:
            nodes, elements, nd = o.kuhn_cube_mesh(4)
            nu, f_vals = 1.0, None
        _, _, A, b_e = o.element_matrices(nodes, elements, nu=nu, f_vals=f_vals)
        indt = np.ascontiguousarray(elements.T)
        n = len(nodes)
        maps = D.partition_maps(torch.from_numpy(indt), n, world)
        op = CpuRankOperator(A, b_e, indt, n, nd, maps, rank)
        comm = D.TorchTransport()
        prob = D.setup([op], comm)
        x = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, n))
        r = D.residual(prob, [op.to_internal(x)])
        r_glob = D.gather_global([op], r, n, comm)
        xj, nj = D.jacobi(prob, [op.to_internal(torch.zeros(n, dtype=torch.float64))], 30, 0.8)
        xj_glob = D.gather_global([op], xj, n, comm)
        res = {}
        for red in (1, 2):  # single-reduction (Chronopoulos-Gear) and textbook recurrences
            xp, npcg = D.pcg(prob, [op.to_internal(torch.zeros(n, dtype=torch.float64))], 400,
                             tol=1e-8, reductions=red)
            assert not prob.diverged
            res[f"xp{red}"] = D.gather_global([op], xp, n, comm).numpy()
            res[f"npcg{red}"] = npcg
            # fixed count (no tol): the full history
            _, nfix = D.pcg(prob, [op.to_internal(torch.zeros(n, dtype=torch.float64))], 9,
                            reductions=red)
            res[f"nfix{red}"] = nfix
        if rank == 0:
            out.put(dict(r=r_glob.numpy(), xj=xj_glob.numpy(), nj=nj, x=x.numpy(), **res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", ["2d", "3d"])
def test_gloo_world2_matches_oracle(case):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    if case == "2d":
        inp = o.config_inputs(4, seed=1, size=4)
        nodes, elements, nd = inp["nodes"], inp["elements"], inp["dirichlet"]
        nu, f_vals = 10.0, inp["f_vals"]
    else:
        nodes, elements, nd = o.kuhn_cube_mesh(4)
        nu, f_vals = 1.0, None
    _, _, A, b_e = o.element_matrices(nodes, elements, nu=nu, f_vals=f_vals)
    indt = np.ascontiguousarray(elements.T)
    r_ref = o.residual(A, b_e, indt, res["x"])
    assert np.max(np.abs(res["r"] - r_ref)) <= 1e-12 * np.max(np.abs(r_ref))
    x0 = np.zeros(len(nodes))
    xj, hj = o.jacobi(A, b_e, indt, nd, x0, 0.8, 30)
    np.testing.assert_allclose(res["nj"], hj["residual_norms"], rtol=1e-10)
    assert np.linalg.norm(res["xj"] - xj) <= 1e-10 * np.linalg.norm(xj)
    xp, hp = o.pcg(A, b_e, indt, nd, x0, 400, tol=1e-8)
    _, hfix = o.pcg(A, b_e, indt, nd, x0, 9)
    for red in (1, 2):
        assert len(res[f"npcg{red}"]) == len(hp["residual_norms"]), red
        np.testing.assert_allclose(res[f"npcg{red}"], hp["residual_norms"], rtol=1e-6)
        assert np.linalg.norm(res[f"xp{red}"] - xp) <= 1e-8 * np.linalg.norm(xp), red
        assert len(res[f"nfix{red}"]) == 10
        np.testing.assert_allclose(res[f"nfix{red}"], hfix["residual_norms"], rtol=1e-9)


def _agree_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from paper_1911_03973_b200 import dist as D
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = D.TorchTransport()
        res = [comm.agree(True), comm.agree(rank != 1), comm.agree(False)]

        def body():  # rank 1 cannot capture (here or on a GPU box); rank 0 may
            if rank == 1:
                raise RuntimeError("capture not possible on this rank")
        g = D._capture(comm, body)
        out.put((rank, res, g is None))
    finally:
        dist.destroy_process_group()


def test_graph_capture_decision_is_collective():
    """dist._capture: the CUDA-graph decision is an all-ranks agreement (any rank that
    cannot capture makes every rank run eagerly, so NCCL calls always pair up)."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_agree_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = sorted(q.get(timeout=120) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, res, dropped in got:
        assert res == [True, False, False], (rank, res)
        assert dropped
