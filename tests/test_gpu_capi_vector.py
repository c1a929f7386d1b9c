"""The vector entry points of the C-ABI (ebs_dot, ebs_nrm2, ebs_axpby, ebs_check_finite,
ebs_mask, ebs_gather, ebs_scatter_add, ebs_index_*) called directly through ctypes."""

import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def P(t):
    return ctypes.c_void_p(t.data_ptr())


def test_reductions_and_axpby(gpu):
    from paper_1911_03973_b200._lib import call
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    g = torch.Generator(device="cuda").manual_seed(1)
    for n in (0, 1, 1000, 1 << 20):
        x = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
        y = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
        out = torch.zeros(2, dtype=torch.float64, device="cuda")
        call("ebs_dot", n, P(x), P(y), P(out), s)
        call("ebs_nrm2", n, P(x), P(out[1:]), s)
        assert abs(float(out[0]) - float(x @ y)) <= 1e-12 * max(1.0, float(x @ y))
        assert abs(float(out[1]) - float(torch.linalg.vector_norm(x))) <= 1e-12 * max(1.0, n ** 0.5)
        # deterministic: same bits run to run
        again = torch.zeros(1, dtype=torch.float64, device="cuda")
        call("ebs_dot", n, P(x), P(y), P(again), s)
        assert float(again) == float(out[0])
        y0 = y.clone()
        call("ebs_axpby", n, 2.0, P(x), -0.5, P(y), s)
        assert torch.equal(y, 2.0 * x + -0.5 * y0)


def test_finite_mask_gather_scatter(gpu):
    from paper_1911_03973_b200._lib import call
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    v = torch.arange(10, dtype=torch.float64, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    call("ebs_check_finite", 10, P(v), P(flag), s)
    assert int(flag) == 0
    v[7] = float("inf")
    call("ebs_check_finite", 10, P(v), P(flag), s)
    assert int(flag) == 1
    v[7] = 7.0
    nd = torch.tensor([1, 4], dtype=torch.int64, device="cuda")
    out = torch.empty_like(v)
    call("ebs_mask", 10, P(v), 2, P(nd), P(out), s)
    exp = v.clone()
    exp[nd] = 0.0
    assert torch.equal(out, exp) and float(v[1]) == 1.0
    idx = torch.tensor([9, 0, 3], dtype=torch.int64, device="cuda")
    buf = torch.empty(3, dtype=torch.float64, device="cuda")
    call("ebs_gather", 3, P(idx), P(v), P(buf), s)
    assert buf.tolist() == [9.0, 0.0, 3.0]
    call("ebs_scatter_add", 3, P(idx), P(buf), P(v), s)
    assert v[[9, 0, 3]].tolist() == [18.0, 0.0, 6.0]
    call("ebs_index_fill", 2, P(idx[:2]), -1.0, P(v), s)
    assert v[[9, 0]].tolist() == [-1.0, -1.0]
    dst = torch.zeros(10, dtype=torch.float64, device="cuda")
    call("ebs_index_copy", 3, P(idx), P(v), P(dst), s)
    assert dst[[9, 0, 3]].tolist() == [-1.0, -1.0, 6.0]
    src_i = torch.tensor([0, 1], dtype=torch.int64, device="cuda")
    dst_i = torch.tensor([5, 6], dtype=torch.int64, device="cuda")
    call("ebs_index_move", 2, P(src_i), P(v), P(dst_i), P(dst), s)
    call("ebs_index_add", 2, P(src_i), P(v), P(dst_i), P(dst), s)
    assert dst[[5, 6]].tolist() == [2 * float(v[0]), 2 * float(v[1])]


def test_plan_apply_out_user_modes(gpu):
    """ebs_plan_apply out_user 0/1/2: internal order, caller order, caller order added into
    a -0.0-filled vector -- the last two bit-identical (masked rows and exact mode too)."""
    from paper_1911_03973_b200 import _device as D
    from paper_1911_03973_b200._lib import load
    from paper_1911_03973_b200.inputs import config_problem
    lib = load()
    p = config_problem(2, seed=1, size=7)
    batch, n = p["batch"], p["mesh"].n_nodes
    pl = batch.operator(n)
    pl.ensure_dirichlet(p["dirichlet"])
    old_of_new = pl.node_maps()[1].long()
    x = torch.from_numpy(np.random.default_rng(2).uniform(-1, 1, n)).cuda()
    xi = D.empty(n)
    s = D.stream()
    assert lib.ebs_to_internal(pl.handle, P(x), P(xi), None, s) == 0
    for op in (0, 1, 2):
        for masked in (0, 1):
            a, b = D.empty(n), D.empty(n)
            c = torch.full((n,), -0.0, dtype=torch.float64, device="cuda")
            assert lib.ebs_plan_apply(pl.handle, op, P(xi), P(a), 0, masked, s) == 0
            assert lib.ebs_plan_apply(pl.handle, op, P(xi), P(b), 1, masked, s) == 0
            assert lib.ebs_plan_apply(pl.handle, op, P(xi), P(c), 2, masked, s) == 0
            assert torch.equal(b.view(torch.int64), c.view(torch.int64))  # bitwise, signs too
            assert torch.equal(b[old_of_new], a)
    assert lib.ebs_plan_apply(pl.handle, 1, P(xi), P(a), 3, 0, s) != 0


def test_native_nccl_collectives_single_rank(gpu):
    """ebs_dist_*: libebs.so's own NCCL communicator (world size 1 on the one GPU): the
    grouped send/recv (to the own rank) moves the buffers, the all-reduce is the identity,
    misuse is rejected."""
    import paper_1911_03973_b200 as eb
    from paper_1911_03973_b200._lib import load
    lib = load()
    m = eb.build_unit_square_mesh(3)
    pl = eb.build_element_batch(m).operator()
    h = pl.handle
    x = torch.arange(10, dtype=torch.float64, device="cuda")
    y = torch.zeros(10, dtype=torch.float64, device="cuda")
    peers = (ctypes.c_int32 * 1)(0)
    counts = (ctypes.c_int64 * 1)(10)
    sp = (ctypes.c_void_p * 1)(x.data_ptr())
    rp = (ctypes.c_void_p * 1)(y.data_ptr())
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert lib.ebs_dist_exchange(h, 1, peers, counts, sp, rp, s) != 0      # no communicator yet
    uid = ctypes.create_string_buffer(128)
    assert lib.ebs_dist_unique_id(uid) == 0
    assert lib.ebs_dist_init(h, uid, 1, 1) != 0                            # rank out of range
    assert lib.ebs_dist_init(h, uid, 0, 1) == 0
    assert lib.ebs_dist_init(h, uid, 0, 1) != 0                            # already initialised
    assert lib.ebs_dist_exchange(h, 1, peers, counts, sp, rp, s) == 0
    torch.cuda.synchronize()
    assert torch.equal(x, y)
    bad = (ctypes.c_int32 * 1)(3)
    assert lib.ebs_dist_exchange(h, 1, bad, counts, sp, rp, s) != 0
    z = x.clone()
    assert lib.ebs_dist_allreduce(h, P(z), 10, s) == 0
    torch.cuda.synchronize()
    assert torch.equal(z, x)
