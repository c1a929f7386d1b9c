"""Element-slab multi-GPU path with P ranks emulated in one process on one GPU (the real
kernels; the transport is a device copy, nothing waits on anything).  Residual, damped
Jacobi and PCG on P = 2, 3, 4 slabs against the oracle / the single-GPU solver."""

import numpy as np
import pytest
import torch

from conftest import to_np

import oracle as o

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("P", [2, 3, 4])
def test_emulated_residual_and_jacobi_c4_recipe(gpu, P):
    import paper_1911_03973_b200 as eb
    from paper_1911_03973_b200 import dist
    from paper_1911_03973_b200.inputs import config_problem
    pr = config_problem(4, seed=2, size=6)
    m, batch, d = pr["mesh"], pr["batch"], pr["dirichlet"]
    prob, maps = dist.emulate(batch, m.n_nodes, d, P)
    ops = prob.ops
    ref_maps = o.halo_maps(to_np(batch.index.indt).astype(np.int64), P)
    for p in range(P):
        np.testing.assert_array_equal(to_np(maps["local"][p]), ref_maps["local"][p])
    x = torch.from_numpy(np.random.default_rng(4).uniform(-1, 1, m.n_nodes)).cuda()
    r = dist.residual(prob, [op.to_internal(x) for op in ops])
    r_glob = to_np(dist.gather_global(ops, r, m.n_nodes))
    r_ref = to_np(eb.residual(batch, x))
    assert np.max(np.abs(r_glob - r_ref)) <= 1e-12 * np.max(np.abs(r_ref))
    # interface values identical on both sides of every slab boundary
    for op, rv in zip(ops, r):
        for q, idx in op.if_idx.items():
            other = ops[q]
            gids = op.global_of_int[idx]
            j = other.new_of_old[torch.searchsorted(other.global_ids, gids)]
            assert torch.equal(rv[idx], r[q][j])
    x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
    xs, norms = dist.jacobi(prob, [op.to_internal(x0) for op in ops], 40, 0.8)
    x1, h1 = eb.jacobi(batch, d, x0, 40, omega=0.8)
    np.testing.assert_allclose(norms, h1.residual_norms, rtol=1e-10)
    xg = to_np(dist.gather_global(ops, xs, m.n_nodes))
    assert np.linalg.norm(xg - to_np(x1)) <= 1e-10 * np.linalg.norm(to_np(x1))


@pytest.mark.parametrize("P", [2, 3])
def test_emulated_pcg_3d(gpu, P):
    import paper_1911_03973_b200 as eb
    from paper_1911_03973_b200 import dist
    from paper_1911_03973_b200.inputs import config_problem
    pr = config_problem(5, size=8)
    m, batch, d = pr["mesh"], pr["batch"], pr["dirichlet"]
    prob, _ = dist.emulate(batch, m.n_nodes, d, P)
    x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
    xs, norms = dist.pcg(prob, [op.to_internal(x0) for op in prob.ops], 1000, tol=1e-8)
    x1, h1 = eb.pcg(batch, d, x0, 1000, tol=1e-8)
    assert len(norms) == len(h1.residual_norms)
    xg = to_np(dist.gather_global(prob.ops, xs, m.n_nodes))
    assert np.linalg.norm(xg - to_np(x1)) <= 1e-8 * np.linalg.norm(to_np(x1))
    nodes, elements, face = o.kuhn_cube_mesh(8)
    _, _, A, b_e = o.element_matrices(nodes, elements, nu=1.0)
    xo, ho = o.pcg(A, b_e, np.ascontiguousarray(elements.T), face, np.zeros(len(nodes)), 1000,
                   tol=1e-8)
    assert len(norms) == len(ho["residual_norms"])
    assert np.linalg.norm(xg - xo) <= 1e-8 * np.linalg.norm(xo)


@pytest.mark.parametrize("P", [2, 3])
def test_graph_replay_identical_to_eager(gpu, P):
    """CUDA-graph replay of batches of distributed iterations gives bit-identical
    iterates and histories (same kernels, same order)."""
    from paper_1911_03973_b200 import dist
    from paper_1911_03973_b200.inputs import config_problem
    for cfg, size, iters in ((4, 6, 21), (5, 6, 19)):
        pr = config_problem(cfg, seed=1, size=size)
        m = pr["mesh"]
        prob, _ = dist.emulate(pr["batch"], m.n_nodes, pr["dirichlet"], P)
        x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
        run = dist.jacobi if cfg == 4 else dist.pcg
        xe, ne = run(prob, [op.to_internal(x0) for op in prob.ops], iters)
        before = dict(dist.GRAPH_STATS)
        xg, ng = run(prob, [op.to_internal(x0) for op in prob.ops], iters, graph=True)
        assert dist.GRAPH_STATS["captured"] == before["captured"] + 1, dist.GRAPH_STATS
        np.testing.assert_array_equal(ng, ne)
        for a, b in zip(xg, xe):
            assert torch.equal(a, b)


@pytest.mark.parametrize("P", [2, 3, 5])
def test_fused_caller_numbering_residual(gpu, P):
    """The fused multi-rank residual in the caller's (permuted) numbering: owned entries
    equal the single-GPU residual within 1e-12 (relative max norm)."""
    import paper_1911_03973_b200 as eb
    from paper_1911_03973_b200 import dist
    from paper_1911_03973_b200.inputs import config_problem
    for cfg, size in ((2, 7), (5, 6)):
        pr = config_problem(cfg, seed=4, size=size)
        m, batch = pr["mesh"], pr["batch"]
        prob, _ = dist.emulate(batch, m.n_nodes, None, P)
        x = torch.from_numpy(np.random.default_rng(9).uniform(-1, 1, m.n_nodes)).cuda()
        ref = eb.residual(batch, x, deterministic=False)
        outs = []
        for overlap in (True, False):
            rg = [torch.full((m.n_nodes,), float("nan"), dtype=torch.float64, device="cuda")
                  for _ in prob.ops]
            xi = [op.zeros() for op in prob.ops]
            sr = [op.zeros() for op in prob.ops]
            dist.residual_caller(prob, x, rg, xi, sr, overlap=overlap)
            out = torch.empty(m.n_nodes, dtype=torch.float64, device="cuda")
            for op, r in zip(prob.ops, rg):
                own = op.owned_glob
                out[own] = r[own]
            assert float((out - ref).abs().max()) <= 1e-12 * float(ref.abs().max())
            outs.append(out)
        assert torch.equal(outs[0], outs[1])  # the chunk split does not change any value


@pytest.mark.parametrize("P", [2, 3])
def test_rank_local_assembly_equals_sliced(gpu, P):
    """rank_operator assembles only the rank's slab; same operator as slicing the global
    batch (bitwise partial sums, same PCG result)."""
    from paper_1911_03973_b200 import dist
    from paper_1911_03973_b200.inputs import config_problem
    pr = config_problem(4, seed=2, size=6)
    m, batch, d = pr["mesh"], pr["batch"], pr["dirichlet"]
    maps = dist.partition_maps(batch.index.indt, m.n_nodes, P)
    x = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, m.n_nodes)).cuda()
    for r in range(P):
        a = dist.GpuRankOperator(batch, m.n_nodes, d, maps, r)
        b, _ = dist.rank_operator(m, pr["nu"], pr["f"], d, P, r, maps=maps)
        sa, sb = a.zeros(), b.zeros()
        a.matvec_partial(a.to_internal(x), sa)
        b.matvec_partial(b.to_internal(x), sb)
        assert torch.equal(sa, sb)
        assert torch.equal(a.rhs_partial(), b.rhs_partial())


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_fused_overlapped_steps_match_unfused(gpu, P):
    """The overlapped interface/interior sweeps: Jacobi iterates bitwise equal to the
    unfused rank loop, PCG within 1e-10 (the dot is summed in three groups)."""
    from paper_1911_03973_b200 import dist
    from paper_1911_03973_b200.inputs import config_problem
    for cfg, size, iters in ((4, 6, 30), (5, 6, 60)):
        pr = config_problem(cfg, seed=5, size=size)
        m = pr["mesh"]
        prob, _ = dist.emulate(pr["batch"], m.n_nodes, pr["dirichlet"], P)
        x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
        xin = [op.to_internal(x0) for op in prob.ops]
        run = dist.jacobi if cfg == 4 else dist.pcg
        xu, nu_ = run(prob, xin, iters, fused=False)
        xf, nf = run(prob, xin, iters, fused=True)
        xg, ng = run(prob, xin, iters, fused=True, graph=True)
        np.testing.assert_allclose(nf, nu_, rtol=1e-8, atol=1e-10 * nu_[0])
        np.testing.assert_array_equal(ng, nf)
        for a, b, c in zip(xf, xu, xg):
            assert torch.equal(a, c)
            if cfg == 4:
                assert torch.equal(a, b)
            else:
                assert float((a - b).abs().max()) <= 1e-10 * float(b.abs().max())


def test_stacked_c2_weak_scaling_input(gpu):
    """bench.py's N>1 weak-scaling input: copies=1 is the C2 recipe exactly; with P copies
    the element slabs np.linspace(0, n_e, P+1) are exactly one square each and the
    distributed caller-numbering residual equals the single-GPU one."""
    import paper_1911_03973_b200 as eb
    from paper_1911_03973_b200 import dist
    from paper_1911_03973_b200.inputs import config_problem, stacked_c2_problem
    a = stacked_c2_problem(1, seed=3, size=4)
    b = config_problem(2, seed=3, size=4, assemble=False)
    assert torch.equal(a["mesh"].nodes, b["mesh"].nodes)
    assert torch.equal(a["mesh"].conn, b["mesh"].conn)
    np.testing.assert_array_equal(a["x"], b["x"])
    P, L = 3, 4
    p = stacked_c2_problem(P, seed=3, size=L)
    m = p["mesh"]
    n = 2**L + 1
    assert m.n_nodes == n * (2**L * P + 1) and m.n_elements == P * 2 * 4**L
    assert float(m.nodes[:, 1].max()) == P
    maps = dist.partition_maps(m.conn, m.n_nodes, P)
    np.testing.assert_array_equal(maps["bounds"], [k * 2 * 4**L for k in range(P + 1)])
    for r in range(P):
        for q, ids in maps["interface"][r].items():
            assert ids.numel() == n  # one shared node row per neighbour
    batch = eb.build_element_batch(m, nu=p["nu"])
    prob, _ = dist.emulate(batch, m.n_nodes, None, P)
    x = torch.from_numpy(p["x"]).cuda()
    rg = [torch.full((m.n_nodes,), float("nan"), dtype=torch.float64, device="cuda")
          for _ in prob.ops]
    dist.residual_caller(prob, x, rg, [op.zeros() for op in prob.ops],
                         [op.zeros() for op in prob.ops])
    out = torch.empty(m.n_nodes, dtype=torch.float64, device="cuda")
    for op, r in zip(prob.ops, rg):
        out[op.owned_glob] = r[op.owned_glob]
    ref = eb.residual(batch, x, deterministic=False)
    assert float((out - ref).abs().max()) <= 1e-12 * float(ref.abs().max())


def test_native_transport_matches_torch_transport(gpu):
    """dist loops over libebs.so's NCCL communicator (NativeTransport) at world size 1:
    the same iterates and histories as over torch.distributed / the device-copy transport."""
    from paper_1911_03973_b200 import dist
    from paper_1911_03973_b200.inputs import config_problem
    for cfg, iters in ((5, 24), (4, 16)):
        pr = config_problem(cfg, seed=2, size=6)
        m = pr["mesh"]
        op, _ = dist.rank_operator(m, pr["nu"], pr["f"], pr["dirichlet"], 1, 0)
        prob_l = dist.setup([op], dist.LocalTransport())
        prob_n = dist.setup([op], dist.NativeTransport(op))
        x0 = op.zeros()
        run = dist.pcg if cfg == 5 else dist.jacobi
        xl, nl = run(prob_l, [x0], iters)
        xn, nn = run(prob_n, [x0], iters)
        xg, ng = run(prob_n, [x0], iters, graph=True)
        np.testing.assert_array_equal(nn, nl)
        np.testing.assert_array_equal(ng, nl)
        assert torch.equal(xn[0], xl[0]) and torch.equal(xg[0], xl[0])


@pytest.mark.parametrize("P", [2, 3])
def test_residual_in_each_ranks_own_order(gpu, P):
    """dist.residual_local: x and r in each rank's own caller order (its local nodes in
    ascending global id); owned entries bit-identical to the global-vector variant and
    within 1e-12 of the single-GPU residual."""
    import paper_1911_03973_b200 as eb
    from paper_1911_03973_b200 import dist
    from paper_1911_03973_b200.inputs import config_problem, stacked_c2_problem
    for pr in (config_problem(2, seed=5, size=7), stacked_c2_problem(P, seed=5, size=6)):
        m = pr["mesh"]
        batch = pr.get("batch") or eb.build_element_batch(m, nu=pr["nu"])
        prob, _ = dist.emulate(batch, m.n_nodes, None, P)
        x = torch.from_numpy(pr["x"]).cuda()
        ref = eb.residual(batch, x, deterministic=False)
        rg = [torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda") for _ in prob.ops]
        dist.residual_caller(prob, x, rg, [op.zeros() for op in prob.ops],
                             [op.zeros() for op in prob.ops])
        xl = [x[op.global_ids].contiguous() for op in prob.ops]
        rl = [op.zeros() for op in prob.ops]
        dist.residual_local(prob, xl, rl, [op.zeros() for op in prob.ops],
                            [op.zeros() for op in prob.ops])
        for op, r_loc, r_glob in zip(prob.ops, rl, rg):
            own = op.owned_local
            gids = op.global_ids[own]
            assert torch.equal(r_loc[own], r_glob[gids])
            assert float((r_loc[own] - ref[gids]).abs().max()) <= 1e-12 * float(ref.abs().max())


@pytest.mark.parametrize("P", [2, 3, 5, 8])
def test_exact_residual_bitwise_across_slab_counts(gpu, P):
    """dist.ExactSlab / residual_exact: the slab plans carry a one-element ghost layer in
    global element order, so every slab node's sum runs over ALL its elements in the
    reference's (j, e) order -- the P-slab exact residual is bit for bit the single-GPU one
    (= the reference's) at every node of every slab, for any P.  2D C2 recipe
    (permuted, jittered numbering) and 3D Kuhn cubes, emulated ranks + the transport's
    generic exchange; and built rank-locally from the mesh (rank_operator style)."""
    import paper_1911_03973_b200 as eb
    from paper_1911_03973_b200 import dist
    from paper_1911_03973_b200.inputs import config_problem
    for cfg, size in ((2, 6), (4, 6), (5, 6)):
        pr = config_problem(cfg, seed=7, size=size)
        m, batch = pr["mesh"], pr["batch"]
        x = torch.from_numpy(np.random.default_rng(P).uniform(-1, 1, m.n_nodes)).cuda()
        ref = eb.residual(batch, x)                         # exact, reference order
        maps = dist.partition_maps(batch.index.indt, m.n_nodes, P)
        for build in ("batch", "mesh"):
            kw = dict(batch=batch) if build == "batch" else dict(mesh=m, nu=pr["nu"], f=pr["f"])
            slabs = dist.exact_slabs(maps, batch.index.indt, m.n_nodes, **kw)
            xl = [x[maps["local"][sl.rank].cuda()] for sl in slabs]
            rs = dist.residual_exact(slabs, dist.LocalTransport(), xl)
            for sl, r in zip(slabs, rs):
                assert torch.equal(r, ref[maps["local"][sl.rank].cuda()]), (cfg, P, build, sl.rank)


@pytest.mark.parametrize("P", [2, 3, 5, 8])
def test_jacobi_exact_iterates_bitwise_across_slab_counts(gpu, P):
    """dist.jacobi_exact on ghost-layer slabs: the damped-Jacobi iterates are bit for bit the
    single-GPU solver's (eb.jacobi) at every node of every slab, for any P; the norm history
    (owned nodes summed in rank order) within 1e-12.  C4 recipe (jittered, permuted,
    nu = 10, f = sin sin) and 3D Kuhn cubes."""
    import paper_1911_03973_b200 as eb
    from paper_1911_03973_b200 import dist
    from paper_1911_03973_b200.inputs import config_problem
    for cfg, size in ((4, 6), (5, 6)):
        pr = config_problem(cfg, seed=11, size=size)
        m, batch, d = pr["mesh"], pr["batch"], pr["dirichlet"]
        x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
        x1, h1 = eb.jacobi(batch, d, x0, 30, omega=0.8)
        maps = dist.partition_maps(batch.index.indt, m.n_nodes, P)
        slabs = dist.exact_slabs(maps, batch.index.indt, m.n_nodes, batch=batch)
        xl0 = [x0[maps["local"][sl.rank].cuda()] for sl in slabs]
        xs, norms = dist.jacobi_exact(slabs, dist.LocalTransport(), d, xl0, 30, 0.8)
        for sl, x in zip(slabs, xs):
            assert torch.equal(x, x1[maps["local"][sl.rank].cuda()]), (cfg, P, sl.rank)
        np.testing.assert_allclose(norms, h1.residual_norms, rtol=1e-12)
