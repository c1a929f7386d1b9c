"""Generate tests/golden/*.npz by running the REFERENCE ebsolve package.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

Every array stored here is an output of reference code
(/root/reference/pkg/src/ebsolve) or of SciPy as the reference calls it;
inputs that the reference cannot build (3D tet matrices, seeded
permutation/jitter) come from the oracle restatement and are stored next to
the reference outputs computed from them.  The fixtures are small (levels
<= 6, N <= 3) so they can be committed; the GPU tests read only these files
and the oracle, never /root/reference.
"""

from __future__ import annotations

import sys
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import scipy.sparse
import scipy.sparse.linalg

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE.parents[1]))

import ebsolve as eb  # noqa: E402
from ebsolve.spectrum import _apply_masked, model_eigen_bounds  # noqa: E402

import oracle  # noqa: E402  (inputs the reference lacks)


def save(name, **arrays):
    np.savez_compressed(HERE / f"{name}.npz", **arrays)
    print(f"wrote {name}.npz: {sorted(arrays)}")


def batch_arrays(batch):
    return dict(K_e=np.ascontiguousarray(batch.K_e), M_e=np.ascontiguousarray(batch.M_e),
                A_e=np.ascontiguousarray(batch.A_e), b_e=batch.b_e)


def main():
    # --- mesh generator (mesh.py:104-148) --------------------------------
    arrs = {}
    for level in range(4):
        m = eb.build_unit_square_mesh(level)
        arrs[f"nodes_l{level}"] = m.nodes
        arrs[f"elements_l{level}"] = m.elements
        arrs[f"boundary_l{level}"] = m.boundary_nodes
    m = eb.build_grid_mesh(2)
    arrs["elements_n2"] = m.elements
    save("mesh2d", **arrs)

    # --- element batches (elements.py:81-137) ----------------------------
    arrs = {}
    m = eb.build_unit_square_mesh(3)
    for nu in (0.0, 1.0, 2.5):
        b = eb.build_element_batch(m, nu=nu)
        for k, v in batch_arrays(b).items():
            arrs[f"{k}_nu{nu}"] = v
    arrs["b_e_xy"] = eb.local_load_batch(eb.build_unit_square_mesh(1), lambda x, y: x + y)
    save("batch2d_l3", **arrs)

    # --- residual / rhs / matvec on structured meshes (operators.py) ------
    arrs = {}
    rng = np.random.default_rng(2024)
    for level, nu in ((1, 0.0), (2, 1.0), (5, 0.0), (5, 1.0)):
        m = eb.build_unit_square_mesh(level)
        batch = eb.build_element_batch(m, nu=nu)
        d = eb.constant_dirichlet(m, 1.0)
        x = rng.standard_normal(m.n_nodes)
        tag = f"l{level}_nu{nu}"
        arrs[f"x_{tag}"] = x
        arrs[f"r_{tag}"] = eb.residual(batch, x)
        arrs[f"r1_{tag}"] = eb.residual(batch, np.ones(m.n_nodes))
        arrs[f"rhs_{tag}"] = eb.assemble_rhs(batch.b_e, batch.index.indt)
        arrs[f"av_{tag}"] = _apply_masked(batch, x, d.nd)
        arrs[f"diag_{tag}"] = eb.assemble_rhs(
            np.stack([batch.A_e[j, j, :] for j in range(3)]), batch.index.indt)
        arrs[f"masked_{tag}"] = eb.mask_dirichlet(arrs[f"r_{tag}"], d)
    save("residual2d", **arrs)

    # --- jittered + permuted mesh, nu=10, f=sin*sin (BASELINE C4 recipe) --
    inp = oracle.config_inputs(4, seed=0, size=4)
    m = eb.Mesh(inp["nodes"], inp["elements"], inp["dirichlet"])
    f = lambda x, y: np.sin(np.pi * x) * np.sin(np.pi * y)  # noqa: E731
    batch = eb.build_element_batch(m, nu=10.0, f=f)
    x = np.random.default_rng(5).uniform(-1.0, 1.0, m.n_nodes)
    d = eb.DirichletData(inp["dirichlet"], np.zeros(inp["dirichlet"].size))
    save("c4_l4_seed0", nodes=inp["nodes"], elements=inp["elements"],
         dirichlet=inp["dirichlet"], perm=inp["perm"], f_vals=inp["f_vals"],
         x=x, r=eb.residual(batch, x), r_threads4=eb.residual(batch, x, threads=4),
         rhs=eb.assemble_rhs(batch.b_e, batch.index.indt),
         av=_apply_masked(batch, x, d.nd), **batch_arrays(batch))

    # --- C2 recipe at level 3 (permutation + x draw order) ---------------
    inp = oracle.config_inputs(2, seed=0, size=3)
    m = eb.Mesh(inp["nodes"], inp["elements"], inp["dirichlet"])
    batch = eb.build_element_batch(m, nu=1.0)
    save("c2_l3_seed0", nodes=inp["nodes"], elements=inp["elements"],
         dirichlet=inp["dirichlet"], perm=inp["perm"], x=inp["x"],
         r=eb.residual(batch, inp["x"]), **batch_arrays(batch))

    # --- Richardson loop (solvers.py:117-183) ----------------------------
    m = eb.build_unit_square_mesh(3)
    batch = eb.build_element_batch(m, nu=0.0)
    d = eb.constant_dirichlet(m, 1.0)
    bounds = model_eigen_bounds(9)
    xs = []
    x, hist = eb.richardson(batch, d, np.ones(m.n_nodes), bounds, 20,
                            callback=lambda k, x, r: xs.append(x.copy()))
    x_tol, hist_tol = eb.richardson(batch, d, np.ones(m.n_nodes), bounds, 500, tol=1e-3)
    A = eb.assemble_sparse(batch.A_e, batch.index.indt)
    b = eb.assemble_rhs(batch.b_e, batch.index.indt)
    u = eb.solve_reference(A, b, d)
    _, hist_err = eb.richardson(batch, d, np.ones(m.n_nodes), bounds, 7, reference=u)
    save("richardson_l3", x=x, norms=hist.residual_norms, iterates=np.stack(xs),
         lambda1=bounds.lambda1, lambda2=bounds.lambda2, x_tol=x_tol,
         norms_tol=hist_tol.residual_norms, u=u, errors=hist_err.error_norms,
         norms_err=hist_err.residual_norms)

    # --- Chebyshev two-/three-level (solvers.py:186-261) ----------------
    from ebsolve import spectrum as sp
    arrs = {}
    for level in (2, 3):
        m = eb.build_unit_square_mesh(level)
        batch = eb.build_element_batch(m, nu=0.0)
        d = eb.constant_dirichlet(m, 1.0)
        bounds = model_eigen_bounds(2**level + 1)
        x0 = np.ones(m.n_nodes)
        for N in (1, 4, 8):
            xs = []
            x, h = eb.chebyshev2(batch, d, x0, bounds, N, 20,
                                 callback=lambda k, x, r: xs.append(x.copy()))
            arrs[f"cheb2_l{level}_N{N}_iterates"] = np.stack(xs)
            arrs[f"cheb2_l{level}_N{N}_norms"] = h.residual_norms
        xs = []
        x, h = eb.chebyshev3(batch, d, x0, bounds, 16,
                             callback=lambda k, x, r: xs.append(x.copy()))
        arrs[f"cheb3_l{level}_iterates"] = np.stack(xs)
        arrs[f"cheb3_l{level}_norms"] = h.residual_norms
        x, h = eb.chebyshev3(batch, d, x0, bounds, 500, tol=1e-6)
        arrs[f"cheb3_l{level}_tol_x"] = x
        arrs[f"cheb3_l{level}_tol_norms"] = h.residual_norms
    save("chebyshev", **arrs)

    # --- spectral bounds (spectrum.py:64-149) ---------------------------
    arrs = {}
    for level, nu in ((3, 1.0), (4, 2.5)):
        m = eb.build_unit_square_mesh(level)
        batch = eb.build_element_batch(m, nu=nu)
        d = eb.constant_dirichlet(m, 1.0)
        tag = f"l{level}_nu{nu}"
        arrs[f"power_{tag}"] = sp.power_iteration_lambda_max(batch, d)
        arrs[f"power10_{tag}"] = sp.power_iteration_lambda_max(batch, d, iters=10, seed=3)
        lo, hi = sp.mass_gershgorin(batch, d)
        arrs[f"gersh_{tag}"] = np.array([lo, hi])
        b = sp.operator_bounds(batch, d, 2**level + 1, nu)
        arrs[f"bounds_{tag}"] = np.array([b.lambda1, b.lambda2])
        A = eb.assemble_sparse(batch.A_e, batch.index.indt)
        arrs[f"dense_{tag}"] = eb.dense_interior_eigenvalues(A, d)
    save("spectrum", **arrs)

    # --- uniform_refine (mesh.py:157-208) on an unstructured (jittered) mesh --
    g4 = oracle.config_inputs(4, seed=0, size=3)
    m = eb.Mesh(g4["nodes"], g4["elements"], g4["dirichlet"])
    fine = eb.uniform_refine(m)
    save("refine", nodes=g4["nodes"], elements=g4["elements"], boundary=g4["dirichlet"],
         fine_nodes=fine.nodes, fine_elements=fine.elements, fine_boundary=fine.boundary_nodes)

    # --- assembled CSR (reference.py:25-39) ------------------------------
    arrs = {}
    m = eb.build_unit_square_mesh(3)
    batch = eb.build_element_batch(m, nu=1.0)
    for name in ("K_e", "A_e"):
        S = eb.assemble_sparse(getattr(batch, name), batch.index.indt)
        S.sort_indices()
        arrs[f"{name}_indptr"], arrs[f"{name}_indices"], arrs[f"{name}_data"] = \
            S.indptr, S.indices, S.data
    save("sparse_l3", **arrs)

    # --- experiment driver exports (cli.py:110-233) -------------------------
    import tempfile
    from ebsolve.cli import ExperimentConfig, run_experiment
    arrs = {}
    with tempfile.TemporaryDirectory() as tmp:
        rep = run_experiment(ExperimentConfig(level=3, iters=20, solver="all", out_dir=tmp))
        for f in sorted(Path(tmp).iterdir()):
            arrs[f.name] = np.frombuffer(f.read_bytes(), dtype=np.uint8)
        arrs["bounds"] = np.array(rep.bounds)
    with tempfile.TemporaryDirectory() as tmp:
        run_experiment(ExperimentConfig(level=2, iters=5, solver="cheb3", out_dir=tmp,
                                        export_vtk=True))
        for f in sorted(Path(tmp).iterdir()):
            arrs["vtk_" + f.name] = np.frombuffer(f.read_bytes(), dtype=np.uint8)
    save("cli_exports", **arrs)

    # --- C1: direct solution + SciPy Jacobi-PCG (reference.py:42-81) ------
    m = eb.build_unit_square_mesh(6)
    batch = eb.build_element_batch(m, nu=1.0)
    d = eb.constant_dirichlet(m, 0.0)
    A = eb.assemble_sparse(batch.A_e, batch.index.indt)
    b = eb.assemble_rhs(batch.b_e, batch.index.indt)
    u = eb.solve_reference(A, b, d)
    free = np.setdiff1d(np.arange(m.n_nodes), d.nd)
    Aff = A[free][:, free].tocsr()
    dinv = 1.0 / Aff.diagonal()
    Mop = scipy.sparse.linalg.LinearOperator(Aff.shape, matvec=lambda v: dinv * v)
    its = []
    sol, info = scipy.sparse.linalg.cg(Aff, b[free], rtol=1e-8, M=Mop,
                                       callback=lambda xk: its.append(1))
    assert info == 0
    u_cg = np.zeros(m.n_nodes)
    u_cg[free] = sol
    save("c1_solution", u_direct=u, u_scipy_pcg=u_cg, scipy_pcg_iters=len(its),
         rhs=b)

    # --- 3D: the reference's residual/_apply_masked on restated tets ------
    arrs = {}
    for N in (2, 3):
        nodes, elements, face = oracle.kuhn_cube_mesh(N)
        K, M, A_e, b_e = oracle.element_matrices(nodes, elements, nu=1.0)
        indt = np.ascontiguousarray(elements.T)
        bt = SimpleNamespace(A_e=A_e, b_e=b_e, n_elements=elements.shape[0],
                             index=SimpleNamespace(ind_e=indt.reshape(4, 1, -1), indt=indt))
        x = np.random.default_rng(N).uniform(-1.0, 1.0, nodes.shape[0])
        arrs[f"nodes_N{N}"] = nodes
        arrs[f"elements_N{N}"] = elements
        arrs[f"face_N{N}"] = face
        arrs[f"K_e_N{N}"] = np.ascontiguousarray(K)
        arrs[f"M_e_N{N}"] = np.ascontiguousarray(M)
        arrs[f"A_e_N{N}"] = np.ascontiguousarray(A_e)
        arrs[f"b_e_N{N}"] = b_e
        arrs[f"x_N{N}"] = x
        arrs[f"r_N{N}"] = eb.residual(bt, x)          # operators.py:72 on 4x4 slices
        arrs[f"av_N{N}"] = _apply_masked(bt, x, face)  # spectrum.py:54
        arrs[f"rhs_N{N}"] = eb.assemble_rhs(b_e, indt)
        # assembled system (COO duplicates summed as reference.py:35-39) and
        # the reference's Dirichlet-eliminated direct solve
        n = nodes.shape[0]
        rows = np.broadcast_to(indt[:, None, :], A_e.shape).ravel()
        cols = np.broadcast_to(indt[None, :, :], A_e.shape).ravel()
        Asp = scipy.sparse.coo_matrix((A_e.ravel(), (rows, cols)), shape=(n, n)).tocsr()
        dd = eb.DirichletData(face, np.zeros(face.size))
        arrs[f"u_N{N}"] = eb.solve_reference(Asp, arrs[f"rhs_N{N}"], dd)
    save("kuhn3d", **arrs)


if __name__ == "__main__":
    main()
