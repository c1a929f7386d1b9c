"""Live differential parity: the UNMODIFIED reference package (pip-installed into
baseline/_ref, the reference arm of bench.py) and this package run side by side in one
process on freshly drawn inputs -- seeds, jitter, permutations, nu and source functions that
no committed golden holds.  Integer / index outputs and everything the reference orders
deterministically must agree bit for bit; reductions the device orders differently are held
to the tolerance the north star states.  Skipped when baseline/_ref is not installed
(`python -c "import __graft_entry__ as g; g.build()"` installs it where /root/reference exists)."""

import importlib
import os
import sys

import numpy as np
import numpy.testing as npt
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(os.path.join(REF, "ebsolve")):
        pytest.skip("baseline/_ref not installed")
    sys.path.insert(0, REF)
    try:
        for name in [m for m in sys.modules if m == "ebsolve" or m.startswith("ebsolve.")]:
            del sys.modules[name]
        mod = importlib.import_module("ebsolve")
        assert os.path.realpath(mod.__file__).startswith(os.path.realpath(REF)), mod.__file__
        yield mod
    finally:
        sys.path.remove(REF)
        for name in [m for m in sys.modules if m == "ebsolve" or m.startswith("ebsolve.")]:
            del sys.modules[name]


@pytest.fixture(scope="module")
def api():
    from paper_1911_03973_b200 import numpy_api
    return numpy_api.facade("")


def _problem(lib, level, seed, nu, jitter=True, permute=True, f=None):
    """The BASELINE C4 recipe at `level` through `lib` (reference or facade): structured
    mesh, interior jitter +-0.2h, random node permutation; all draws from one rng."""
    rng = np.random.default_rng(seed)
    base = lib.build_unit_square_mesh(level)
    nodes = np.array(base.nodes)
    elements = np.array(base.elements)
    bd = np.array(base.boundary_nodes)
    if jitter:
        h = 1.0 / 2**level
        interior = np.setdiff1d(np.arange(len(nodes)), bd)
        nodes[interior] += rng.uniform(-0.2 * h, 0.2 * h, (len(interior), 2))
    if permute:
        perm = rng.permutation(len(nodes))          # new label of old node i
        new_nodes = np.empty_like(nodes)
        new_nodes[perm] = nodes
        nodes, elements, bd = new_nodes, perm[elements], np.sort(perm[bd])
    m = lib.Mesh(nodes, elements, bd)
    batch = lib.build_element_batch(m, nu=nu, f=f)
    return m, batch, rng


def _f(x, y):
    return np.cos(3.0 * x) * np.exp(y) - 0.25


@pytest.mark.parametrize("level,seed,nu", [(1, 101, 0.0), (2, 102, 1.0), (4, 103, 2.5),
                                            (6, 104, 10.0), (8, 105, 0.3)])
def test_assembly_and_residual_bitwise(ref, api, level, seed, nu):
    mr, br, rng = _problem(ref, level, seed, nu, f=_f)
    mg, bg, _ = _problem(api, level, seed, nu, f=_f)
    npt.assert_array_equal(mg.nodes, mr.nodes)
    npt.assert_array_equal(mg.elements, mr.elements)
    npt.assert_array_equal(mg.boundary_nodes, mr.boundary_nodes)
    for name in ("K_e", "M_e", "A_e", "b_e"):
        npt.assert_array_equal(getattr(bg, name), getattr(br, name), err_msg=name)
    npt.assert_array_equal(bg.index.indt, br.index.indt)
    npt.assert_array_equal(bg.index.ind_e, br.index.ind_e)
    npt.assert_array_equal(api.assemble_rhs(bg.b_e, bg.index.indt),
                           ref.assemble_rhs(br.b_e, br.index.indt))
    for _ in range(3):
        x = rng.uniform(-1.0, 1.0, mr.n_nodes)
        r_ref = ref.residual(br, x)
        npt.assert_array_equal(api.residual(bg, x), r_ref)                   # reference order
        npt.assert_array_equal(api.residual(bg, x, threads=4), ref.residual(br, x, threads=4))
        fast = api.residual(bg, x, deterministic=False)
        assert np.max(np.abs(fast - r_ref)) <= 1e-12 * np.max(np.abs(r_ref))
    d_r = ref.constant_dirichlet(mr, 0.5)
    d_g = api.constant_dirichlet(mg, 0.5)
    npt.assert_array_equal(d_g.nd, d_r.nd)
    npt.assert_array_equal(api.mask_dirichlet(r_ref, d_g), ref.mask_dirichlet(r_ref, d_r))
    npt.assert_array_equal(api.apply_initial_guess(mg, d_g), ref.apply_initial_guess(mr, d_r))
    for name in ("local_stiffness_batch", "local_mass_batch"):
        npt.assert_array_equal(getattr(api, name)(mg), getattr(ref, name)(mr))
    npt.assert_array_equal(api.local_load_batch(mg, _f), ref.local_load_batch(mr, _f))
    npt.assert_array_equal(api.combine_system(bg.K_e, bg.M_e, 0.7),
                           ref.combine_system(br.K_e, br.M_e, 0.7))


def test_full_size_c2_residual_bitwise(ref, api):
    """BASELINE C2 at full size (level 11, 4.2M nodes, 8.4M triangles, permuted numbering,
    x ~ U[-1, 1]) and the C4 recipe (jitter + permutation, nu = 10, f = sin sin) at level 10:
    the device residual against the unmodified reference's, bit for bit; the fast mode within
    the north star's 1e-12 relative max-norm."""
    from paper_1911_03973_b200.inputs import sin_sin
    for level, seed, nu, jitter, f in ((11, 7, 1.0, False, None), (10, 8, 10.0, True, sin_sin)):
        mr, br, rng = _problem(ref, level, seed, nu, jitter=jitter, f=f)
        mg, bg, _ = _problem(api, level, seed, nu, jitter=jitter, f=f)
        x = rng.uniform(-1.0, 1.0, mr.n_nodes)
        r_ref = ref.residual(br, x, threads=os.cpu_count() or 1)
        npt.assert_array_equal(api.residual(bg, x), r_ref)
        fast = api.residual(bg, x, deterministic=False)
        assert np.max(np.abs(fast - r_ref)) <= 1e-12 * np.max(np.abs(r_ref))
        del mr, br, mg, bg


@pytest.mark.parametrize("level,seed,nu", [(3, 201, 0.0), (5, 202, 1.0)])
def test_stationary_iterations_bitwise(ref, api, level, seed, nu):
    """Richardson and both Chebyshev forms: every iterate handed to the callback and the
    residual-norm history, bit for bit (structured mesh: the model bounds apply)."""
    mr, br, rng = _problem(ref, level, seed, nu, jitter=False, permute=True)
    mg, bg, _ = _problem(api, level, seed, nu, jitter=False, permute=True)
    d_r, d_g = ref.constant_dirichlet(mr, 1.0), api.constant_dirichlet(mg, 1.0)
    x0 = ref.apply_initial_guess(mr, d_r)
    n = 2**level + 1
    for name, extra in (("richardson", ()), ("chebyshev2", (4,)), ("chebyshev3", ())):
        got, want = [], []
        b_r, b_g = ref.model_eigen_bounds(n), api.model_eigen_bounds(n)
        assert (b_g.lambda1, b_g.lambda2) == (b_r.lambda1, b_r.lambda2)
        xr, hr = getattr(ref, name)(br, d_r, x0, b_r, *extra, 25,
                                    callback=lambda k, x, r: want.append((k, x.copy(), r.copy())))
        xg, hg = getattr(api, name)(bg, d_g, x0, b_g, *extra, 25,
                                    callback=lambda k, x, r: got.append((k, x, r)))
        npt.assert_array_equal(xg, xr, err_msg=name)
        assert len(got) == len(want) == 26
        for (kg, xk, rk), (kr, xw, rw) in zip(got, want):
            assert kg == kr
            npt.assert_array_equal(xk, xw, err_msg=f"{name} x^{kg}")
            npt.assert_array_equal(rk, rw, err_msg=f"{name} r^{kg}")
        npt.assert_allclose(hg.residual_norms, hr.residual_norms, rtol=1e-12, atol=0.0)
        assert hg.diverged == hr.diverged


@pytest.mark.parametrize("level", [0, 1, 3, 5])
def test_refine_sparse_spectrum_and_direct_solve(ref, api, level):
    mr, mg = ref.build_unit_square_mesh(level), api.build_unit_square_mesh(level)
    fr, fg = ref.uniform_refine(mr), api.uniform_refine(mg)
    npt.assert_array_equal(fg.nodes, fr.nodes)
    npt.assert_array_equal(fg.elements, fr.elements)
    npt.assert_array_equal(fg.boundary_nodes, fr.boundary_nodes)
    assert fg.level == fr.level
    br, bg = ref.build_element_batch(fr, nu=1.5), api.build_element_batch(fg, nu=1.5)
    Ar = ref.assemble_sparse(br.A_e, br.index.indt)
    Ag = api.assemble_sparse(bg.A_e, bg.index.indt)
    Ar.sort_indices(), Ag.sort_indices()
    npt.assert_array_equal(Ag.indptr, Ar.indptr)
    npt.assert_array_equal(Ag.indices, Ar.indices)
    npt.assert_allclose(Ag.data, Ar.data, rtol=1e-15, atol=1e-18)   # duplicate sums: order differs
    d_r, d_g = ref.constant_dirichlet(fr, 1.0), api.constant_dirichlet(fg, 1.0)
    b = ref.assemble_rhs(br.b_e, br.index.indt)
    u_r, u_g = ref.solve_reference(Ar, b, d_r), api.solve_reference(Ag, b, d_g)
    npt.assert_allclose(u_g, u_r, rtol=0, atol=1e-9)                 # reference.py:22 tolerance
    lo_r, hi_r = ref.mass_gershgorin(br, d_r)
    lo_g, hi_g = api.mass_gershgorin(bg, d_g)
    npt.assert_allclose([lo_g, hi_g], [lo_r, hi_r], rtol=1e-14)
    npt.assert_allclose(api.power_iteration_lambda_max(bg, d_g, seed=3),
                        ref.power_iteration_lambda_max(br, d_r, seed=3), rtol=1e-8)
    n = 2**(level + 1) + 1
    ob_r, ob_g = ref.operator_bounds(br, d_r, n, 1.5), api.operator_bounds(bg, d_g, n, 1.5)
    npt.assert_allclose([ob_g.lambda1, ob_g.lambda2], [ob_r.lambda1, ob_r.lambda2], rtol=1e-8)


def test_experiment_outputs_identical(ref, api, tmp_path):
    """run_experiment end to end (cli.py:110-233).  nu = 0 (closed-form bounds): solution
    files (CSV and VTK) byte for byte, residual / error histories to 1e-12 (the device reduces
    the norms in another order).  nu > 0: the upper bound is 1.05 x a power-iteration estimate
    built on BLAS dot / nrm2 (spectrum.py:91-93: summation order is the BLAS build's, not the
    algorithm's), so it agrees to rounding, not bitwise, and the solutions with it."""
    from ebsolve.cli import ExperimentConfig as RefConfig, run_experiment as ref_run
    from paper_1911_03973_b200 import numpy_api
    cli = numpy_api.facade("cli")
    for nu, vtk in ((0.0, False), (0.0, True), (0.5, False)):
        out_r, out_g = tmp_path / f"ref{nu}{vtk}", tmp_path / f"gpu{nu}{vtk}"
        kw = dict(level=4, nu=nu, iters=40, solver="all", cycle_n=8, export_vtk=vtk)
        rep_r = ref_run(RefConfig(out_dir=str(out_r), **kw))
        rep_g = cli.run_experiment(cli.ExperimentConfig(out_dir=str(out_g), **kw))
        assert set(rep_g.runs) == set(rep_r.runs)
        if nu == 0.0:
            assert tuple(rep_g.bounds) == tuple(rep_r.bounds)
        else:
            assert rep_g.bounds[0] == rep_r.bounds[0]       # model minimum + nu x Gershgorin floor
            npt.assert_allclose(rep_g.bounds[1], rep_r.bounds[1], rtol=1e-12)
        names = sorted(p.name for p in out_r.iterdir())
        assert names == sorted(p.name for p in out_g.iterdir()) and len(names) >= 6
        for name in names:
            if "direct" in name and not vtk:   # sparse direct solve vs device PCG to 1e-13
                ra = np.loadtxt(out_r / name, delimiter=",", skiprows=1)
                rb = np.loadtxt(out_g / name, delimiter=",", skiprows=1)
                npt.assert_allclose(rb, ra, rtol=0, atol=1e-9, err_msg=name)
            elif "direct" in name:
                continue
            elif name.startswith("history_") or nu != 0.0:
                ra = np.loadtxt(out_r / name, delimiter=",", skiprows=1)
                rb = np.loadtxt(out_g / name, delimiter=",", skiprows=1)
                npt.assert_allclose(rb, ra, rtol=1e-12 if nu == 0.0 else 1e-9, atol=1e-14,
                                    err_msg=name)
            else:
                assert (out_r / name).read_bytes() == (out_g / name).read_bytes(), name
