"""GPU parity: the element residual / matvec / rhs / diag through the C-ABI against the
reference's own outputs (golden) and the oracle -- bitwise in reference order, within
1e-12 (north-star tolerance) for the pre-assembled-b fast mode."""

import numpy as np
import numpy.testing as npt
import pytest
import torch

from conftest import golden, to_np

import oracle as o

pytestmark = pytest.mark.gpu

TOL_FAST = 1e-12  # north_star: fp64 residual within relative max-norm 1e-12


def rel_max(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


@pytest.mark.parametrize("tag", ["l1_nu0.0", "l2_nu1.0", "l5_nu0.0", "l5_nu1.0"])
def test_residual_family_matches_reference(gpu, tag):
    import paper_1911_03973_b200 as eb
    g = golden("residual2d")
    level, nu = int(tag[1]), float(tag.split("nu")[1])
    m = eb.build_unit_square_mesh(level)
    batch = eb.build_element_batch(m, nu=nu)
    d = eb.constant_dirichlet(m, 1.0)
    x = g[f"x_{tag}"]
    npt.assert_array_equal(to_np(eb.residual(batch, x)), g[f"r_{tag}"])
    npt.assert_array_equal(to_np(eb.residual(batch, x, threads=8)), g[f"r_{tag}"])
    assert rel_max(to_np(eb.residual(batch, x, deterministic=False)), g[f"r_{tag}"]) <= TOL_FAST
    npt.assert_array_equal(to_np(eb.residual(batch, np.ones(m.n_nodes))), g[f"r1_{tag}"])
    npt.assert_array_equal(to_np(eb.assemble_rhs(batch.b_e, batch.index)), g[f"rhs_{tag}"])
    npt.assert_array_equal(to_np(eb.assemble_rhs(batch.b_e, batch.index.indt)), g[f"rhs_{tag}"])
    npt.assert_array_equal(to_np(eb.matvec(batch, x, d)), g[f"av_{tag}"])
    npt.assert_array_equal(to_np(eb.diagonal(batch)), g[f"diag_{tag}"])
    masked = eb.mask_dirichlet(eb.residual(batch, x), d)
    npt.assert_array_equal(to_np(masked), g[f"masked_{tag}"])


def test_residual_known_answers(gpu):
    import paper_1911_03973_b200 as eb
    # test_operators.py:33-45: residual(0) == b, residual(1) == b (nu = 0) bitwise
    for level in range(1, 5):
        m = eb.build_unit_square_mesh(level)
        batch = eb.build_element_batch(m)
        b = to_np(eb.assemble_rhs(batch.b_e, batch.index))
        npt.assert_array_equal(to_np(eb.residual(batch, np.zeros(m.n_nodes))), b)
        npt.assert_array_equal(to_np(eb.residual(batch, np.ones(m.n_nodes))), b)
    m = eb.build_unit_square_mesh(1)
    b = to_np(eb.assemble_rhs(eb.build_element_batch(m).b_e, eb.build_element_batch(m).index))
    assert abs(b[4] - 0.25) <= 1e-15


def test_residual_input_validation(gpu):
    import paper_1911_03973_b200 as eb
    m = eb.build_unit_square_mesh(1)
    batch = eb.build_element_batch(m)
    with pytest.raises(ValueError):
        eb.residual(batch, np.zeros((m.n_nodes, 1)))
    bad = np.zeros(m.n_nodes)
    bad[3] = np.nan
    with pytest.raises(ValueError):
        eb.residual(batch, bad)
    bad[3] = np.inf
    with pytest.raises(ValueError):
        eb.residual(batch, torch.from_numpy(bad).cuda())


def test_mask_and_dirichlet_semantics(gpu):
    import paper_1911_03973_b200 as eb
    m = eb.build_unit_square_mesh(2)
    batch = eb.build_element_batch(m)
    d = eb.constant_dirichlet(m, 1.0)
    r = eb.residual(batch, np.zeros(m.n_nodes))
    r_before = r.clone()
    masked = eb.mask_dirichlet(r, d)
    assert masked.data_ptr() != r.data_ptr()
    assert bool((masked[d.nd] == 0).all())
    assert torch.equal(r, r_before)
    x0 = eb.apply_initial_guess(eb.build_unit_square_mesh(1), eb.constant_dirichlet(
        eb.build_unit_square_mesh(1), 1.0))
    assert int(torch.count_nonzero(x0)) == 8 and float(x0[4]) == 0.0
    dd = eb.DirichletData(np.array([5, 2]), np.array([50.0, 20.0]))
    npt.assert_array_equal(to_np(dd.nd), [2, 5])
    npt.assert_array_equal(to_np(dd.values), [20.0, 50.0])
    with pytest.raises(ValueError):
        eb.DirichletData(np.array([1, 1]), np.array([0.0, 0.0]))
    with pytest.raises(ValueError):
        eb.DirichletData(np.array([1, 2]), np.array([0.0]))


@pytest.mark.parametrize("name", ["c4_l4_seed0", "c2_l3_seed0"])
def test_permuted_meshes_bitwise(gpu, name):
    import paper_1911_03973_b200 as eb
    g = golden(name)
    m = eb.Mesh(g["nodes"], g["elements"], g["dirichlet"])
    batch = eb.ElementBatch(K_e=g["K_e"], M_e=g["M_e"], A_e=g["A_e"], b_e=g["b_e"], nu=1.0,
                            index=eb.build_index_arrays(m))
    npt.assert_array_equal(to_np(eb.residual(batch, g["x"])), g["r"])
    assert rel_max(to_np(eb.residual(batch, g["x"], deterministic=False)), g["r"]) <= TOL_FAST
    if "av" in g:
        d = eb.DirichletData(g["dirichlet"], np.zeros(len(g["dirichlet"])))
        npt.assert_array_equal(to_np(eb.matvec(batch, g["x"], d)), g["av"])


def test_plan_numbering_matches_oracle(gpu):
    import paper_1911_03973_b200 as eb
    inp = o.config_inputs(2, seed=0, size=5)
    m = eb.Mesh(inp["nodes"], inp["elements"], inp["dirichlet"])
    pl = eb.build_index_arrays(m).plan()
    new_of_old, old_of_new = (to_np(t) for t in pl.node_maps())
    ref = o.first_appearance_order(np.ascontiguousarray(inp["elements"].T), m.n_nodes)
    npt.assert_array_equal(new_of_old, ref)
    npt.assert_array_equal(old_of_new[new_of_old], np.arange(m.n_nodes))
    info = pl.info()
    assert info["max_valence"] == 6 and info["n_chunks"] == (m.n_nodes + 31) // 32
    assert not info["loaded"] & 32                     # permuted: not a structured grid


_STRUCTURED_CHECK = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import oracle as o
import paper_1911_03973_b200 as eb
dim = int(sys.argv[2])
nodes, el, nd = o.unit_square_mesh(4) if dim == 2 else o.kuhn_cube_mesh(4)
m = eb.Mesh(nodes, el, nd)
indt = np.ascontiguousarray(el.T)
pl = eb.build_index_arrays(m).plan()
new_of_old, old_of_new = (t.cpu().numpy() for t in pl.node_maps())
assert np.array_equal(new_of_old, o.plan_numbering(indt, m.n_nodes))
assert np.array_equal(old_of_new, np.arange(m.n_nodes))
flags = pl.info()["loaded"]
batch = eb.build_element_batch(m, nu=1.0)
_, _, A, b_e = o.element_matrices(nodes, el, nu=1.0)
x = np.random.default_rng(1).uniform(-1, 1, m.n_nodes)
ref = o.residual(A, b_e, indt, x)
assert np.array_equal(eb.residual(batch, x).cpu().numpy(), ref)
assert np.array_equal(eb.matvec(batch, x).cpu().numpy(), o.matvec_masked(A, indt, x, np.zeros(0, np.int64)))
fast = eb.residual(batch, x, deterministic=False).cpu().numpy()
assert np.max(np.abs(fast - ref)) <= 1e-12 * np.max(np.abs(ref))
d = eb.constant_dirichlet(m, 0.0)
xs, hs = eb.pcg(batch, d, np.zeros(m.n_nodes), 200, tol=1e-10)
xo, ho = o.pcg(A, b_e, indt, nd, np.zeros(m.n_nodes), 200, tol=1e-10)
assert len(hs.residual_norms) == len(ho["residual_norms"])
assert np.linalg.norm(xs.cpu().numpy() - xo) <= 1e-8 * np.linalg.norm(xo)
print("FLAGS", flags)
"""


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("mode", ["", "2", "3"])
def test_plan_keeps_structured_numbering(gpu, dim, mode):
    """Unpermuted generated grids: every (neighbour - node) difference is a +-1
    combination of axis strides, so the plan keeps the caller's numbering (identity maps)
    -- with packed-delta ids (EBS_IDS_GRID=2) or one-byte tuple codes (default, =3).
    Residual / matvec bitwise, PCG vs the oracle."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    env.pop("EBS_IDS_GRID", None)
    if mode:
        env["EBS_IDS_GRID"] = mode
    out = subprocess.run([sys.executable, "-c", _STRUCTURED_CHECK, root, str(dim)], env=env,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    flags = int(out.stdout.split("FLAGS")[1])
    assert flags & 64                                  # identity numbering
    tuples = mode != "2"
    assert bool(flags & 32) == tuples


@pytest.mark.parametrize("N", [2, 3])
def test_tet_operator_matches_reference_code(gpu, N):
    import paper_1911_03973_b200 as eb
    g = golden("kuhn3d")
    m = eb.build_unit_cube_mesh(N)
    batch = eb.build_element_batch(m, nu=1.0)
    x = g[f"x_N{N}"]
    face = eb.face_z0_nodes(m)
    d = eb.DirichletData(face, torch.zeros(face.numel(), dtype=torch.float64, device=face.device))
    npt.assert_array_equal(to_np(eb.residual(batch, x)), g[f"r_N{N}"])
    assert rel_max(to_np(eb.residual(batch, x, deterministic=False)), g[f"r_N{N}"]) <= TOL_FAST
    npt.assert_array_equal(to_np(eb.matvec(batch, x, d)), g[f"av_N{N}"])
    npt.assert_array_equal(to_np(eb.assemble_rhs(batch.b_e, batch.index)), g[f"rhs_N{N}"])


def test_isolated_nodes_and_user_batches(gpu):
    """A hand-built batch (conftest.diagonal_batch of the reference) with x longer than
    the mesh: trailing nodes no element touches get residual 0 (np.bincount minlength)."""
    import paper_1911_03973_b200 as eb
    A = np.diag([2.0, 3.0, 4.0]).reshape(3, 3, 1)
    indt = np.array([[0], [1], [2]])
    batch = eb.ElementBatch(K_e=A, M_e=np.zeros_like(A), A_e=A, b_e=np.array([[1.0], [0.0], [0.0]]),
                            nu=0.0, index=eb.IndexArrays(indt.reshape(3, 1, 1), indt))
    r = to_np(eb.residual(batch, np.array([1.0, 1.0, 1.0, 5.0])))
    npt.assert_array_equal(r, [1.0 - 2.0, -3.0, -4.0, 0.0])


@pytest.mark.parametrize("level", [7, 9])
def test_random_inputs_bitwise_vs_oracle(gpu, level):
    import paper_1911_03973_b200 as eb
    from paper_1911_03973_b200.inputs import config_problem
    for config in (2, 4):
        p = config_problem(config, seed=level, size=level)
        inp = o.config_inputs(config, seed=level, size=level)
        _, _, A, b_e = o.element_matrices(inp["nodes"], inp["elements"], nu=p["nu"],
                                          f_vals=inp["f_vals"])
        indt = np.ascontiguousarray(inp["elements"].T)
        x = inp["x"] if config == 2 else np.random.default_rng(1).uniform(-1, 1, len(inp["nodes"]))
        ref = o.residual(A, b_e, indt, x)
        npt.assert_array_equal(to_np(eb.residual(p["batch"], x)), ref)
        assert rel_max(to_np(eb.residual(p["batch"], x, deterministic=False)), ref) <= TOL_FAST
        nd = inp["dirichlet"]
        d = p["dirichlet"]
        npt.assert_array_equal(to_np(eb.matvec(p["batch"], x, d)), o.matvec_masked(A, indt, x, nd))


@pytest.mark.slow
def test_c2_full_size_vs_oracle(gpu):
    """BASELINE C2 at full size (level 11, 8.4M triangles, permuted): bitwise vs the oracle,
    plus run-to-run determinism of both modes."""
    import paper_1911_03973_b200 as eb
    from paper_1911_03973_b200.inputs import config_problem
    p = config_problem(2, seed=0)
    batch, x = p["batch"], p["x"]
    r_exact = eb.residual(batch, x)
    r_fast = eb.residual(batch, x, deterministic=False)
    assert torch.equal(r_exact, eb.residual(batch, x))
    assert torch.equal(r_fast, eb.residual(batch, x, deterministic=False))
    A = batch.A_e.permute(2, 0, 1).contiguous().cpu().numpy().transpose(1, 2, 0)
    b_e = to_np(batch.b_e)
    indt = to_np(batch.index.indt).astype(np.int64)
    ref = o.residual(A, b_e, indt, x, threads=8)
    npt.assert_array_equal(to_np(r_exact), ref)
    assert rel_max(to_np(r_fast), ref) <= TOL_FAST


def test_residual_many_pipelined(gpu):
    """residual_many: each row bit-identical to residual(); sequences, numpy, pageable and
    pinned inputs, broadcast rows; non-finite rows raise; k = 0."""
    import torch
    import paper_1911_03973_b200 as eb
    from paper_1911_03973_b200.inputs import config_problem
    p = config_problem(2, seed=3, size=8)
    batch, n = p["batch"], p["mesh"].n_nodes
    rng = np.random.default_rng(5)
    xs = rng.uniform(-1, 1, (7, n))
    for det in (True, False):
        ref = np.stack([to_np(eb.residual(batch, x, deterministic=det)) for x in xs])
        npt.assert_array_equal(eb.residual_many(batch, xs, deterministic=det).numpy(), ref)
        pinned = torch.from_numpy(xs).pin_memory()
        out = torch.empty((7, n), dtype=torch.float64).pin_memory()
        assert eb.residual_many(batch, pinned, out=out, deterministic=det) is out
        npt.assert_array_equal(out.numpy(), ref)
        npt.assert_array_equal(eb.residual_many(batch, list(xs), deterministic=det).numpy(), ref)
    bcast = torch.from_numpy(xs[2]).pin_memory().unsqueeze(0).expand(5, n)
    npt.assert_array_equal(eb.residual_many(batch, bcast).numpy(),
                           np.broadcast_to(to_np(eb.residual(batch, xs[2])), (5, n)))
    wide = torch.from_numpy(np.pad(xs, ((0, 0), (0, 5))))[:, :n]   # rows n + 5 apart
    assert wide.stride(0) == n + 5
    npt.assert_array_equal(eb.residual_many(batch, wide, deterministic=False).numpy(),
                           np.stack([to_np(eb.residual(batch, x, deterministic=False)) for x in xs]))
    npt.assert_array_equal(eb.residual_many(batch, xs[5:6]).numpy()[0], to_np(eb.residual(batch, xs[5])))
    bad = xs.copy()
    bad[4, 3] = np.nan
    with pytest.raises(ValueError, match=r"x\[4\]"):
        eb.residual_many(batch, bad)
    assert eb.residual_many(batch, np.empty((0, n))).shape == (0, n)
    with pytest.raises(ValueError):
        eb.residual_many(batch, xs[0])


def test_residual_many_on_device_two_in_flight(gpu):
    """residual_many on device-resident vectors (ebs_residual_many: two residuals in flight on
    two streams, each with its own workspace): every row bit-identical to residual() in both
    modes; odd / even / single k, broadcast and padded rows, sequences of CUDA vectors, `out`
    validation, per-vector non-finite flags, CUDA-graph capture, a following call on another
    stream, the masked C-ABI form, the sequential fallback of the two-pass permutation."""
    import ctypes
    import torch
    import paper_1911_03973_b200 as eb
    from paper_1911_03973_b200 import _device as D
    from paper_1911_03973_b200._lib import EBS_RES_EXACT, load
    from paper_1911_03973_b200.inputs import config_problem
    p = config_problem(4, seed=3, size=7)          # jittered + permuted
    batch, m = p["batch"], p["mesh"]
    n = m.n_nodes
    rng = np.random.default_rng(11)
    xs = torch.from_numpy(rng.uniform(-1, 1, (7, n))).cuda()
    for det in (True, False):
        ref = torch.stack([eb.residual(batch, x, deterministic=det) for x in xs])
        for k in (7, 6, 2, 1):
            got = eb.residual_many(batch, xs[:k], deterministic=det)
            assert got.is_cuda and tuple(got.shape) == (k, n)
            assert torch.equal(got, ref[:k]), (det, k)
        out = torch.empty((7, n), dtype=torch.float64, device="cuda")
        assert eb.residual_many(batch, xs, out=out, deterministic=det) is out
        assert torch.equal(out, ref)
        assert torch.equal(eb.residual_many(batch, list(xs), deterministic=det), ref)
    bcast = xs[2].unsqueeze(0).expand(5, n)
    assert bcast.stride(0) == 0
    assert torch.equal(eb.residual_many(batch, bcast), ref_row(eb, batch, xs[2]).expand(5, n))
    wide = torch.nn.functional.pad(xs, (0, 5))[:, :n]
    assert wide.stride(0) == n + 5
    assert torch.equal(eb.residual_many(batch, wide), torch.stack([eb.residual(batch, x) for x in xs]))
    assert tuple(eb.residual_many(batch, xs[:0]).shape) == (0, n)
    with pytest.raises(ValueError):
        eb.residual_many(batch, xs, out=torch.empty((7, n), dtype=torch.float64))   # host out
    with pytest.raises(ValueError):
        eb.residual_many(batch, xs, out=torch.empty((6, n), dtype=torch.float64, device="cuda"))
    bad = xs.clone()
    bad[3, 7] = float("inf")
    bad[4, 0] = float("nan")
    with pytest.raises(ValueError, match=r"x\[3\]"):
        eb.residual_many(batch, bad)
    # graph capture (fork / join across the plan's second stream) and replay
    ref = torch.stack([eb.residual(batch, x, deterministic=False) for x in xs])
    out = torch.zeros((7, n), dtype=torch.float64, device="cuda")
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        eb.residual_many(batch, xs, out=out, deterministic=False, check_finite=False)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            eb.residual_many(batch, xs, out=out, deterministic=False, check_finite=False)
        for _ in range(3):
            out.zero_()
            g.replay()
            torch.cuda.synchronize()
            assert torch.equal(out, ref)
    # the next call on another stream is ordered after both lanes of this one
    other = torch.cuda.Stream()
    big = eb.residual_many(batch, xs.repeat(6, 1), deterministic=False, check_finite=False)
    with torch.cuda.stream(other):
        r_next = eb.residual(batch, xs[1], deterministic=False)
    torch.cuda.synchronize()
    assert torch.equal(r_next, ref[1]) and torch.equal(big[-1], ref[6]) and torch.equal(big[35], ref[0])
    # C-ABI: masked rows and device flags
    lib = load()
    d = p["dirichlet"]
    with batch.using(n) as pl:
        pl.ensure_dirichlet(d)
        flags = D.zeros(7, torch.int32)
        out = D.empty((7, n))
        rc = lib.ebs_residual_many(pl.handle, D.ptr(bad), n, D.ptr(out), n, 7, EBS_RES_EXACT, 1,
                                   D.ptr(flags), D.stream())
        assert rc == 0
        torch.cuda.synchronize()
    assert flags.tolist() == [0, 0, 0, 1, 1, 0, 0]
    want = eb.mask_dirichlet(eb.residual(batch, xs[5]), d)
    assert torch.equal(out[5], want) and torch.equal(out[0], eb.mask_dirichlet(eb.residual(batch, xs[0]), d))


def ref_row(eb, batch, x):
    return eb.residual(batch, x).unsqueeze(0)


def test_residual_many_on_device_with_the_two_pass_permutation(gpu):
    """Meshes on the two-pass permutation path (forced here by EBS_PERM2_MIN_NODES) stage
    through plan-held buffers: ebs_residual_many runs them one at a time, same bits."""
    import subprocess
    import sys
    code = (
        "import torch, numpy as np, paper_1911_03973_b200 as eb\n"
        "from paper_1911_03973_b200.inputs import config_problem\n"
        "p = config_problem(2, seed=1, size=7); b = p['batch']; n = p['mesh'].n_nodes\n"
        "xs = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, (5, n))).cuda()\n"
        "ref = torch.stack([eb.residual(b, x) for x in xs])\n"
        "assert torch.equal(eb.residual_many(b, xs), ref)\n"
        "assert torch.equal(eb.residual_many(b, xs, deterministic=False),"
        " torch.stack([eb.residual(b, x, deterministic=False) for x in xs]))\n"
        "print('ok')\n")
    import os
    env = dict(os.environ, EBS_PERM2_MIN_NODES="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))), timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


def test_concurrent_residuals_on_separate_streams(gpu):
    """SPEC.md:273 of the reference: residual is safe to call concurrently on a shared
    batch.  Host threads, each on its own CUDA stream, share one plan (and its device
    workspace); every result equals the serial one bitwise."""
    import threading
    import torch
    import paper_1911_03973_b200 as eb
    from paper_1911_03973_b200.inputs import config_problem
    p = config_problem(2, seed=6, size=9)
    batch, n = p["batch"], p["mesh"].n_nodes
    rng = np.random.default_rng(8)
    xs = [torch.from_numpy(rng.uniform(-1, 1, n)).cuda() for _ in range(4)]
    ref = [to_np(eb.residual(batch, x)) for x in xs]
    torch.cuda.synchronize()
    out = {}
    errors = []

    def work(t):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                for rep in range(25):
                    for i, x in enumerate(xs):
                        r = eb.residual(batch, x, check_finite=False)
                        out[(t, rep, i)] = r
            st.synchronize()
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    threads = [threading.Thread(target=work, args=(t,)) for t in range(4)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    torch.cuda.synchronize()
    assert not errors, errors
    for (t, rep, i), r in out.items():
        npt.assert_array_equal(to_np(r), ref[i], err_msg=f"thread {t} rep {rep} vector {i}")


def test_concurrent_batches_sharing_one_plan(gpu):
    """Two operators on one plan (a batch and its mass slices share the IndexArrays, as
    mass_gershgorin does) used from different threads: each call sees its own operator."""
    import threading
    import torch
    import paper_1911_03973_b200 as eb
    from paper_1911_03973_b200.spectrum import _MassBatch
    m = eb.build_unit_square_mesh(6)
    batch = eb.build_element_batch(m, nu=1.0)
    mb = _MassBatch(batch.M_e, batch.index)
    n = m.n_nodes
    x = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, n)).cuda()
    ref_a = to_np(eb.matvec(batch, x))
    ref_m = to_np(eb.matvec(mb, x))
    assert not np.array_equal(ref_a, ref_m)
    errors = []

    def work(b, ref):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                for _ in range(40):
                    y = eb.matvec(b, x)
                    st.synchronize()
                    if not np.array_equal(to_np(y), ref):
                        errors.append("wrong operator")
                        return
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    th = [threading.Thread(target=work, args=(b, r)) for b, r in
          ((batch, ref_a), (mb, ref_m), (batch, ref_a), (mb, ref_m))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors[:3]


@pytest.mark.parametrize("N", [6, 16])
def test_permuted_kuhn_meshes_vs_oracle(gpu, N):
    """The unstructured-numbering 3D path (randomly relabelled Kuhn cube: first-appearance
    internal ids, delta / two-base id coding instead of the structured one-byte tuples):
    exact residual bitwise, fast residual <= 1e-12, masked matvec and diagonal bitwise,
    Jacobi-PCG same iteration count and solution within 1e-8 of the oracle."""
    import paper_1911_03973_b200 as eb
    nodes, elements, face = o.kuhn_cube_mesh(N)
    perm = np.random.default_rng(N).permutation(len(nodes))
    pn, pe, _ = o.permute_mesh(nodes, elements, np.zeros(0, dtype=np.int64), perm)
    pface = o.detect_face_z0(pn)
    _, _, A, b_e = o.element_matrices(pn, pe, nu=1.0)
    indt = np.ascontiguousarray(pe.T)
    m = eb.permute_nodes(eb.build_unit_cube_mesh(N), perm)
    batch = eb.build_element_batch(m, nu=1.0)
    npt.assert_array_equal(to_np(m.conn).T, pe)
    pl = batch.operator(m.n_nodes)
    assert not (pl.info()["loaded"] & 64)  # not kept as a structured numbering
    x = np.random.default_rng(7).uniform(-1, 1, len(pn))
    ref = o.residual(A, b_e, indt, x)
    npt.assert_array_equal(to_np(eb.residual(batch, x)), ref)
    assert rel_max(to_np(eb.residual(batch, x, deterministic=False)), ref) <= TOL_FAST
    d = eb.DirichletData(pface, np.zeros(len(pface)))
    npt.assert_array_equal(to_np(eb.matvec(batch, x, d)), o.matvec_masked(A, indt, x, pface))
    npt.assert_array_equal(to_np(eb.diagonal(batch)), o.diagonal(A, indt, len(pn)))
    xo, ho = o.pcg(A, b_e, indt, pface, np.zeros(len(pn)), 2000, tol=1e-8)
    xg, hg = eb.pcg(batch, d, np.zeros(len(pn)), 2000, tol=1e-8)
    assert len(hg.residual_norms) == len(ho["residual_norms"])
    assert np.linalg.norm(to_np(xg) - xo) <= 1e-8 * np.linalg.norm(xo)
