"""TEST INFRASTRUCTURE ONLY -- NumPy restatement of the element-based P1 path.

See ``oracle/__init__.py`` for who may import this module.  Citations are to
``/root/reference/pkg/src/ebsolve/<file>:<line>`` unless noted.  Functions
marked RESTATEMENT implement north-star features that have no reference code
(SURVEY.md section 2.2); they are composed from reference primitives and
follow the reference's formula and ordering style.

Bit-exactness conventions (probe-verified and pinned by
``tests/golden``):
  * every arithmetic step is a separate IEEE operation (NumPy elementwise
    ufuncs never fuse multiply-add);
  * the element product is ``((A[i,0]*x0 + A[i,1]*x1) + A[i,2]*x2)``
    (``operators.py:69`` einsum, left to right);
  * scatter-add is ``np.bincount`` over the (n_b, n_e) SoA index array, i.e.
    per node a sequential sum from 0.0 over contributions ordered by
    ``j*n_e + e`` (``operators.py:98``).
"""

from __future__ import annotations

import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

__all__ = [
    "MAX_LEVEL", "BOUNDARY_TOL", "EPS_AREA", "EPS_VOLUME",
    "MASS_PATTERN_2D", "MASS_PATTERN_3D", "KUHN_PERMS",
    "grid_mesh", "unit_square_mesh", "kuhn_cube_mesh", "detect_boundary", "uniform_refine",
    "detect_face_z0", "signed_measure", "jitter_interior", "permute_mesh",
    "element_matrices", "centroids", "assemble_rhs", "local_residuals",
    "residual", "matvec_masked", "diagonal", "mask", "initial_guess",
    "richardson", "jacobi", "pcg", "cg", "StreamedOperator", "element_slabs", "halo_maps",
    "first_appearance_order", "delta_alphabet", "grid_strides", "plan_numbering", "node_slots", "config_inputs",
    "chebyshev_roots", "chebyshev2", "chebyshev3", "chebyshev3_coefficients",
    "model_eigen_bounds", "power_iteration_lambda_max", "mass_gershgorin", "operator_bounds",
]

MAX_LEVEL = 12                       # mesh.py:20
BOUNDARY_TOL = 1e-12                 # mesh.py:22
EPS_AREA = 1e-14                     # elements.py:19
EPS_VOLUME = 1e-18                   # RESTATEMENT: tet analogue of EPS_AREA
MASS_PATTERN_2D = (np.ones((3, 3)) + np.eye(3)) / 12.0   # elements.py:22
MASS_PATTERN_3D = (np.ones((4, 4)) + np.eye(4)) / 20.0   # P1 tet: vol/20*(1+d_ij)
# Kuhn (Freudenthal) split: tet t of a cube walks the axes in KUHN_PERMS[t]
# from corner 000 to corner 111 (lexicographic permutation order).
KUHN_PERMS = ((0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0))
_KUHN_ODD = (False, True, True, False, False, True)


# --------------------------------------------------------------------- mesh

def grid_mesh(n: int):
    """mesh.py:104-128: ``n`` nodes per side, row-major nodes, per cell the
    lower (ll, ll+1, ll+n+1) then the upper (ll, ll+n+1, ll+n) triangle.

    Returns (nodes (n*n,2) f64, elements (2(n-1)^2,3) i64, boundary i64)."""
    if n < 2:
        raise ValueError(f"need at least 2 nodes per side, got n={n}")
    ticks = np.arange(n, dtype=np.float64) / (n - 1)          # mesh.py:111
    xx, yy = np.meshgrid(ticks, ticks)
    nodes = np.column_stack([xx.ravel(), yy.ravel()])          # mesh.py:113
    ix, iy = np.meshgrid(np.arange(n - 1), np.arange(n - 1))
    ll = (iy * n + ix).ravel()
    elements = np.empty((2 * len(ll), 3), dtype=np.int64)
    elements[0::2] = np.column_stack([ll, ll + 1, ll + n + 1])  # mesh.py:118
    elements[1::2] = np.column_stack([ll, ll + n + 1, ll + n])  # mesh.py:119
    return nodes, elements, detect_boundary(nodes)


def unit_square_mesh(level: int):
    """mesh.py:131-137 (level guard MAX_LEVEL)."""
    if level < 0 or level > MAX_LEVEL:
        raise ValueError(f"level {level} outside [0, {MAX_LEVEL}]")
    return grid_mesh(2**level + 1)


def detect_boundary(nodes):
    """mesh.py:145-148: any coordinate within 1e-12 of 0 or 1, sorted."""
    near = np.abs(nodes) <= BOUNDARY_TOL
    far = np.abs(nodes - 1.0) <= BOUNDARY_TOL
    return np.flatnonzero((near | far).any(axis=1)).astype(np.int64)


def detect_face_z0(nodes):
    """RESTATEMENT (BASELINE C3/C5 Dirichlet face): |z| <= 1e-12, sorted."""
    return np.flatnonzero(np.abs(nodes[:, 2]) <= BOUNDARY_TOL).astype(np.int64)


def kuhn_cube_mesh(N: int):
    """RESTATEMENT: unit cube, N cells per side, 6 Kuhn tets per cube.

    Node ``(iz*n + iy)*n + ix`` (n = N+1) sits at ``(ix, iy, iz)/(n-1)``
    (same tick rule as mesh.py:111).  Cubes are visited z-outer, then y, then
    x (so contiguous element ranges are z-slabs); cube c owns elements
    6c..6c+5.  Tet t walks corner 000 -> +e[p0] -> +e[p1] -> 111 with
    p = KUHN_PERMS[t]; for odd permutations local vertices 2 and 3 are
    swapped so every tet has positive volume.

    Returns (nodes (n^3,3) f64, elements (6N^3,4) i64, z0_face i64)."""
    if N < 1:
        raise ValueError(f"need at least 1 cell per side, got N={N}")
    n = N + 1
    ticks = np.arange(n, dtype=np.float64) / (n - 1)
    zz, yy, xx = np.meshgrid(ticks, ticks, ticks, indexing="ij")
    nodes = np.column_stack([xx.ravel(), yy.ravel(), zz.ravel()])
    iz, iy, ix = np.meshgrid(np.arange(N), np.arange(N), np.arange(N), indexing="ij")
    base = ((iz * n + iy) * n + ix).ravel()
    step = (1, n, n * n)
    elements = np.empty((6 * base.size, 4), dtype=np.int64)
    for t, p in enumerate(KUHN_PERMS):
        v0 = base
        v1 = v0 + step[p[0]]
        v2 = v1 + step[p[1]]
        v3 = base + (1 + n + n * n)
        if _KUHN_ODD[t]:
            v2, v3 = v3, v2
        elements[t::6] = np.column_stack([v0, v1, v2, v3])
    return nodes, elements, detect_face_z0(nodes)


def uniform_refine(nodes, elements):
    """mesh.py:157-208 restated: 4 children per triangle through the edge midpoints
    (one per geometric edge, edges as sorted node pairs in np.unique order, midpoint
    0.5*(x[lo] + x[hi])), nodes renumbered by np.lexsort((x, y)), each child rotated to
    its smallest node, rows sorted by np.lexsort((c2, c1, c0)).
    Returns (fine_nodes, fine_elements)."""
    n = nodes.shape[0]
    tri = np.asarray(elements, dtype=np.int64)
    edges = np.sort(np.concatenate([tri[:, [0, 1]], tri[:, [1, 2]], tri[:, [2, 0]]]), axis=1)
    uniq, inv = np.unique(edges, axis=0, return_inverse=True)
    ab, bc, ca = n + inv.reshape(3, -1)
    xy = np.vstack([nodes, 0.5 * (nodes[uniq[:, 0]] + nodes[uniq[:, 1]])])
    a, b, c = tri.T
    kids = np.concatenate([np.column_stack(t) for t in
                           ((a, ab, ca), (ab, b, bc), (ca, bc, c), (ab, bc, ca))])
    order = np.lexsort((xy[:, 0], xy[:, 1]))
    rank = np.empty(len(xy), dtype=np.int64)
    rank[order] = np.arange(len(xy))
    kids = rank[kids]
    shift = np.argmin(kids, axis=1)
    kids = np.take_along_axis(kids, (shift[:, None] + np.arange(3)) % 3, axis=1)
    kids = kids[np.lexsort((kids[:, 2], kids[:, 1], kids[:, 0]))]
    return xy[order], kids


def signed_measure(nodes, elements):
    """mesh.py:96-101 (2D signed area); 3D: det/6 of the edge matrix."""
    p = nodes[elements]
    d1 = p[:, 1] - p[:, 0]
    d2 = p[:, 2] - p[:, 0]
    if nodes.shape[1] == 2:
        return 0.5 * (d1[:, 0] * d2[:, 1] - d1[:, 1] * d2[:, 0])
    d3 = p[:, 3] - p[:, 0]
    c = _cross(d2, d3)
    return ((d1[:, 0] * c[0] + d1[:, 1] * c[1]) + d1[:, 2] * c[2]) / 6.0


def jitter_interior(nodes, boundary, h, rng):
    """RESTATEMENT (BASELINE C4): interior nodes (non-boundary per
    mesh.py:145-148) += U(-0.2h, 0.2h), drawn as one (n_int, dim) block in
    ascending node order."""
    out = np.array(nodes, dtype=np.float64, copy=True)
    interior = np.setdiff1d(np.arange(len(nodes)), boundary)
    out[interior] += rng.uniform(-0.2 * h, 0.2 * h, (interior.size, nodes.shape[1]))
    return out


def permute_mesh(nodes, elements, boundary, perm):
    """RESTATEMENT (BASELINE C2/C4): the new id of old node i is perm[i].

    Node coordinates move with their node, element rows keep their order and
    local vertex order, the boundary set is relabelled and re-sorted."""
    perm = np.asarray(perm, dtype=np.int64)
    new_nodes = np.empty_like(nodes)
    new_nodes[perm] = nodes
    return new_nodes, perm[elements], np.sort(perm[boundary])


# ---------------------------------------------------------------- elements

def _cross(a, b):
    return (a[:, 1] * b[:, 2] - a[:, 2] * b[:, 1],
            a[:, 2] * b[:, 0] - a[:, 0] * b[:, 2],
            a[:, 0] * b[:, 1] - a[:, 1] * b[:, 0])


def _geometry(nodes, elements):
    """elements.py:56-78 (triangles) and its RESTATEMENT for tetrahedra.

    Returns (measure (n_e,), grads (n_e, dim, n_b)).  Tet gradients use the
    closed-form cofactors g_k = (d_{k+1} x d_{k+2})/det and
    g_0 = -((g_1 + g_2) + g_3)."""
    p = nodes[elements]
    n_e = elements.shape[0]
    if nodes.shape[1] == 2:
        d1 = p[:, 1] - p[:, 0]
        d2 = p[:, 2] - p[:, 0]
        det = d1[:, 0] * d2[:, 1] - d1[:, 1] * d2[:, 0]
        meas = 0.5 * det
        if np.any(meas <= EPS_AREA):
            worst = int(np.argmin(meas))
            raise ValueError(
                f"degenerate element {worst}: area {meas[worst]:.3e} <= {EPS_AREA}")
        x, y = p[..., 0], p[..., 1]
        grads = np.empty((n_e, 2, 3))
        for j in range(3):
            jn, jp = (j + 1) % 3, (j + 2) % 3
            grads[:, 0, j] = (y[:, jn] - y[:, jp]) / det
            grads[:, 1, j] = (x[:, jp] - x[:, jn]) / det
        return meas, grads
    d1 = p[:, 1] - p[:, 0]
    d2 = p[:, 2] - p[:, 0]
    d3 = p[:, 3] - p[:, 0]
    c23, c31, c12 = _cross(d2, d3), _cross(d3, d1), _cross(d1, d2)
    det = (d1[:, 0] * c23[0] + d1[:, 1] * c23[1]) + d1[:, 2] * c23[2]
    meas = det / 6.0
    if np.any(meas <= EPS_VOLUME):
        worst = int(np.argmin(meas))
        raise ValueError(
            f"degenerate element {worst}: volume {meas[worst]:.3e} <= {EPS_VOLUME}")
    grads = np.empty((n_e, 3, 4))
    for k, c in ((1, c23), (2, c31), (3, c12)):
        for a in range(3):
            grads[:, a, k] = c[a] / det
    for a in range(3):
        grads[:, a, 0] = -((grads[:, a, 1] + grads[:, a, 2]) + grads[:, a, 3])
    return meas, grads


def centroids(nodes, elements):
    """elements.py:107 ``p.mean(axis=1)``: ((p0+p1)+p2)/3 (3D: .../4)."""
    p = nodes[elements]
    s = p[:, 0] + p[:, 1]
    for j in range(2, elements.shape[1]):
        s = s + p[:, j]
    return s / float(elements.shape[1])


def element_matrices(nodes, elements, nu=0.0, f=None, f_vals=None):
    """elements.py:81-137 (build_element_batch) for triangles; RESTATEMENT
    for tetrahedra (K = vol*G^T G, M = vol/20*(1+d_ij), b_j = f(c)*vol/4).

    Returns (K_e, M_e, A_e, b_e) with the reference layouts: K/M/A are
    (n_b, n_b, n_e) views of element-major (n_e, n_b, n_b) memory
    (elements.py:86,93), b_e is a C-contiguous (n_b, n_e) array
    (elements.py:112).  ``f`` is f(x, y[, z]) on centroid arrays;
    ``f_vals`` (n_e,) overrides it; default f = 1 (elements.py:126-127)."""
    if nu < 0:
        raise ValueError(f"nu must be nonnegative, got {nu}")
    dim = nodes.shape[1]
    nb = dim + 1
    meas, grads = _geometry(nodes, elements)
    # einsum("eki,ekj->eij") (elements.py:84), summed over k left to right
    k = grads[:, 0, :, None] * grads[:, 0, None, :]
    for a in range(1, dim):
        k = k + grads[:, a, :, None] * grads[:, a, None, :]
    k *= meas[:, None, None]                      # elements.py:85
    pattern = MASS_PATTERN_2D if dim == 2 else MASS_PATTERN_3D
    me = meas[:, None, None] * pattern            # elements.py:92
    K = k.transpose(1, 2, 0)
    M = me.transpose(1, 2, 0)
    A = K + nu * M                                # elements.py:121
    if f_vals is None:
        c = centroids(nodes, elements)
        if f is None:
            vals = np.ones(elements.shape[0])
        else:
            vals = np.asarray(f(*[c[:, a] for a in range(dim)]), dtype=np.float64)
        vals = np.broadcast_to(vals, (elements.shape[0],))
    else:
        vals = np.asarray(f_vals, dtype=np.float64)
    if not np.all(np.isfinite(vals)):
        raise ValueError("source function returned non-finite values")
    b_e = np.ascontiguousarray(np.broadcast_to(vals * meas / float(nb), (nb, elements.shape[0])))
    return K, M, A, b_e


# --------------------------------------------------------------- operators

class StreamedOperator:
    """RESTATEMENT for meshes whose whole-mesh element arrays are too large to
    build at once on the host (BASELINE C4 / C5 at full size): the operator of
    element_matrices(nodes, elements, nu, f_vals) evaluated chunk by chunk.

    * Each element's K/M/A/b_e depend only on its own nodes, so building them for
      an element range [lo, hi) gives bit-identical entries to the whole-mesh
      call (elements.py:56-137 is elementwise).
    * The per-element local products of every chunk go into ONE (n_b, n_e) array
      that is reduced by ONE bincount over indt -- exactly the reference's
      threaded deterministic mode (operators.py:96-107: chunk-local residuals,
      concatenated, one bincount), so residual / matvec_masked / diagonal are
      bitwise identical to the whole-mesh functions, in the same (j, e) order.
    * Chunks run on a thread pool (NumPy releases the GIL in its loops); element
      matrices are kept per chunk when ``cache`` (C5: 12.9 GB of A_e), else
      rebuilt on every pass.

    Pass it as ``A_e`` to residual / matvec_masked / diagonal / pcg / jacobi
    (b_e and indt arguments are then ignored in favour of the operator's own)."""

    def __init__(self, nodes, elements, nu=0.0, f_vals=None, chunk=1 << 21, threads=None,
                 cache=True):
        import os
        self.nodes = nodes
        self.elements = elements
        self.nu = nu
        self.f_vals = f_vals
        self.n = nodes.shape[0]
        self.nb = elements.shape[1]
        self.n_e = elements.shape[0]
        self.indt = np.ascontiguousarray(elements.T)
        self.bounds = [(lo, min(lo + chunk, self.n_e)) for lo in range(0, self.n_e, chunk)]
        self.threads = threads or min(32, os.cpu_count() or 1)
        self.cache = {} if cache else None

    def matrices(self, c):
        """(A_e, b_e) of chunk c: (n_b, n_b, m) view, (n_b, m)."""
        if self.cache is not None and c in self.cache:
            return self.cache[c]
        lo, hi = self.bounds[c]
        fv = None if self.f_vals is None else self.f_vals[lo:hi]
        _, _, A, b_e = element_matrices(self.nodes, self.elements[lo:hi], nu=self.nu, f_vals=fv)
        A = np.ascontiguousarray(A.transpose(2, 0, 1)).transpose(1, 2, 0)  # drop K, M
        if self.cache is not None:
            self.cache[c] = (A, b_e)
        return A, b_e

    def _pass(self, fill):
        out = np.empty((self.nb, self.n_e))

        def work(c):
            lo, hi = self.bounds[c]
            A, b_e = self.matrices(c)
            out[:, lo:hi] = fill(A, b_e, lo, hi)
        with ThreadPoolExecutor(max_workers=self.threads) as pool:
            list(pool.map(work, range(len(self.bounds))))
        return out

    def _products(self, A, v, lo, hi):
        return _local_products(A, self.indt[:, lo:hi], v, 0, hi - lo)

    def residual(self, x):
        """operators.py:72-107: one bincount of the chunk-local residuals."""
        rt = self._pass(lambda A, b_e, lo, hi: b_e - self._products(A, x, lo, hi))
        return np.bincount(self.indt.ravel(), weights=rt.ravel(), minlength=self.n)

    def matvec_masked(self, v, nd):
        """spectrum.py:54-61."""
        av = self._pass(lambda A, b_e, lo, hi: self._products(A, v, lo, hi))
        out = np.bincount(self.indt.ravel(), weights=av.ravel(), minlength=self.n)
        out[nd] = 0.0
        return out

    def diagonal(self):
        """diagonal(): assemble_rhs of the stacked A_e[j, j, :]."""
        dg = self._pass(lambda A, b_e, lo, hi: np.stack([A[j, j, :] for j in range(self.nb)]))
        return assemble_rhs(dg, self.indt, self.n)

    def rhs(self):
        """assemble_rhs(b_e, indt) (operators.py:58-63)."""
        be = self._pass(lambda A, b_e, lo, hi: b_e)
        return assemble_rhs(be, self.indt, self.n)


def assemble_rhs(b_e, indt, n=None):
    """operators.py:58-63: bincount in (j, e) order."""
    if n is None:
        n = int(indt.max()) + 1 if indt.size else 0
    return np.bincount(indt.ravel(), weights=b_e.ravel(), minlength=n)


def local_residuals(A_e, b_e, indt, x, lo, hi):
    """operators.py:66-69 written out: rt_i = b_i - ((A_i0 x_0 + A_i1 x_1) + ...)."""
    nb = indt.shape[0]
    xg = [x[indt[i, lo:hi]] for i in range(nb)]
    out = np.empty((nb, hi - lo))
    for i in range(nb):
        loc = A_e[i, 0, lo:hi] * xg[0]
        for c in range(1, nb):
            loc = loc + A_e[i, c, lo:hi] * xg[c]
        out[i] = b_e[i, lo:hi] - loc
    return out


def _local_products(A_e, indt, x, lo, hi):
    """spectrum.py:57 einsum (pure product, no b_e)."""
    nb = indt.shape[0]
    xg = [x[indt[i, lo:hi]] for i in range(nb)]
    out = np.empty((nb, hi - lo))
    for i in range(nb):
        loc = A_e[i, 0, lo:hi] * xg[0]
        for c in range(1, nb):
            loc = loc + A_e[i, c, lo:hi] * xg[c]
        out[i] = loc
    return out


def residual(A_e, b_e, indt, x, threads=1):
    """operators.py:72-107 (deterministic mode): r = sum_e C_e^T(b_e - A_e x_e).

    With threads > 1 the element chunks np.linspace(0, n_e, T+1) are computed
    concurrently (operators.py:100-103) and reduced by one bincount
    (operators.py:105-107), so the result is bitwise independent of T."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim != 1:
        raise ValueError(f"x must be a flat global vector, got shape {x.shape}")
    if not np.all(np.isfinite(x)):
        raise ValueError("x contains non-finite entries")
    if isinstance(A_e, StreamedOperator):
        return A_e.residual(x)
    n_e = indt.shape[1]
    if threads <= 1 or n_e < 2 * threads:
        rt = local_residuals(A_e, b_e, indt, x, 0, n_e)
    else:
        bounds = np.linspace(0, n_e, threads + 1, dtype=int)
        with ThreadPoolExecutor(max_workers=threads) as pool:
            parts = list(pool.map(
                lambda s: local_residuals(A_e, b_e, indt, x, s[0], s[1]),
                zip(bounds[:-1], bounds[1:])))
        rt = np.concatenate(parts, axis=1)
    return np.bincount(indt.ravel(), weights=rt.ravel(), minlength=x.shape[0])


def matvec_masked(A_e, indt, v, nd):
    """spectrum.py:54-61 (_apply_masked): y = A v by (j, e)-ordered bincount,
    then y[nd] = 0."""
    if isinstance(A_e, StreamedOperator):
        return A_e.matvec_masked(v, nd)
    av = _local_products(A_e, indt, v, 0, indt.shape[1])
    out = np.bincount(indt.ravel(), weights=av.ravel(), minlength=v.shape[0])
    out[nd] = 0.0
    return out


def diagonal(A_e, indt, n):
    """RESTATEMENT: diag(A) = assemble_rhs(stack_j A_e[j,j,:])
    -- the reference's own assemble_rhs (operators.py:58-63) applied to the
    diagonal slices, in the residual's (j, e) order."""
    if isinstance(A_e, StreamedOperator):
        return A_e.diagonal()
    nb = indt.shape[0]
    d = np.stack([A_e[j, j, :] for j in range(nb)])
    return assemble_rhs(d, indt, n)


def mask(r, nd):
    """operators.py:114-118: copy, zero at nd."""
    out = np.array(r, dtype=np.float64, copy=True)
    out[nd] = 0.0
    return out


def initial_guess(n, nd, values):
    """operators.py:121-125."""
    x0 = np.zeros(n)
    x0[nd] = values
    return x0


# ----------------------------------------------------------------- solvers

def _iterate(A_e, b_e, indt, nd, x0, iters, advance, tol=None, reference=None,
             callback=None):
    """solvers.py:117-160: shared loop; history has iters+1 norms, tol is
    relative to ||r_0||, divergence is a flag, callback(k, x, r)."""
    if iters < 0:
        raise ValueError(f"iteration count must be nonnegative, got {iters}")
    x = np.array(x0, dtype=np.float64, copy=True)
    errors = [] if reference is not None else None
    diverged = False
    t0 = time.perf_counter()
    r = mask(residual(A_e, b_e, indt, x), nd)
    norms = [float(np.linalg.norm(r))]
    if errors is not None:
        errors.append(float(np.linalg.norm(x - reference)))
    if callback is not None:
        callback(0, x, r)
    for k in range(iters):
        if tol is not None and norms[-1] <= tol * norms[0]:
            break
        x = advance(k, x, r)
        if not np.all(np.isfinite(x)):
            norms.append(float("inf"))
            if errors is not None:
                errors.append(float("inf"))
            diverged = True
            break
        r = mask(residual(A_e, b_e, indt, x), nd)
        norms.append(float(np.linalg.norm(r)))
        if errors is not None:
            errors.append(float(np.linalg.norm(x - reference)))
        if callback is not None:
            callback(k + 1, x, r)
        if not np.isfinite(norms[-1]):
            diverged = True
            break
    return x, dict(residual_norms=np.array(norms),
                   error_norms=None if errors is None else np.array(errors),
                   wall_time=time.perf_counter() - t0, diverged=diverged)


def richardson(A_e, b_e, indt, nd, x0, lambda1, lambda2, iters, **kw):
    """solvers.py:163-183: x += omega r, omega = 2/(lam1+lam2)."""
    omega = 2.0 / (lambda1 + lambda2)
    return _iterate(A_e, b_e, indt, nd, x0, iters,
                    lambda k, x, r: x + omega * r, **kw)


def jacobi(A_e, b_e, indt, nd, x0, omega, iters, **kw):
    """RESTATEMENT: damped Jacobi x += omega * (dinv * r) on the _iterate
    skeleton (solvers.py:117-160); dinv = 1/diag(A) (diagonal()) on free
    nodes and 0 on nd."""
    n = x0.shape[0]
    dinv = _dinv(A_e, indt, n, nd)
    return _iterate(A_e, b_e, indt, nd, x0, iters,
                    lambda k, x, r: x + omega * (dinv * r), **kw)


def _dinv(A_e, indt, n, nd):
    """1/diag(A) on free nodes; 0 on nd and on nodes no element touches (diag == 0)."""
    d = diagonal(A_e, indt, n)
    free = np.ones(n, dtype=bool)
    free[nd] = False
    free &= d != 0.0
    out = np.zeros(n)
    out[free] = 1.0 / d[free]
    return out


def pcg(A_e, b_e, indt, nd, x0, iters, tol=None, reference=None, callback=None,
        precondition=True):
    """RESTATEMENT: (Jacobi-preconditioned) conjugate gradients on the
    masked operator, with the _iterate conventions (solvers.py:117-160).

        r = mask(b - A x0) (operators.py:72 + :114);  z = dinv*r;  p = z
        loop k: stop if ||r_k|| <= tol*||r_0||
                q = mask(A p)  (spectrum.py:54-61);  alpha = (r.z)/(p.q)
                x += alpha p;  r -= alpha q           (recursive residual,
                                                      as SciPy cg, reference.py:70)
                z = dinv*r;  beta = (r.z)_new/(r.z);  p = z + beta p
    dinv = 1/diag(A) on free nodes, 0 on nd; plain CG uses dinv = 1 on free
    nodes.  alpha (beta) is taken as 0 when p.q (r.z) is exactly 0, so an
    exactly solved system stays put instead of producing 0/0."""
    if iters < 0:
        raise ValueError(f"iteration count must be nonnegative, got {iters}")
    n = x0.shape[0]
    if precondition:
        dinv = _dinv(A_e, indt, n, nd)
    else:
        dinv = np.ones(n)
        dinv[nd] = 0.0
    x = np.array(x0, dtype=np.float64, copy=True)
    errors = [] if reference is not None else None
    diverged = False
    t0 = time.perf_counter()
    r = mask(residual(A_e, b_e, indt, x), nd)
    z = dinv * r
    p = z.copy()
    rz = float(r @ z)
    norms = [float(np.linalg.norm(r))]
    if errors is not None:
        errors.append(float(np.linalg.norm(x - reference)))
    if callback is not None:
        callback(0, x, r)
    for k in range(iters):
        if tol is not None and norms[-1] <= tol * norms[0]:
            break
        q = matvec_masked(A_e, indt, p, nd)
        pq = float(p @ q)
        alpha = rz / pq if pq != 0.0 else 0.0
        x = x + alpha * p
        r = r - alpha * q
        if not np.all(np.isfinite(x)):
            norms.append(float("inf"))
            if errors is not None:
                errors.append(float("inf"))
            diverged = True
            break
        norms.append(float(np.linalg.norm(r)))
        if errors is not None:
            errors.append(float(np.linalg.norm(x - reference)))
        if callback is not None:
            callback(k + 1, x, r)
        if not np.isfinite(norms[-1]):
            diverged = True
            break
        z = dinv * r
        rz_new = float(r @ z)
        beta = rz_new / rz if rz != 0.0 else 0.0
        p = z + beta * p
        rz = rz_new
    return x, dict(residual_norms=np.array(norms),
                   error_norms=None if errors is None else np.array(errors),
                   wall_time=time.perf_counter() - t0, diverged=diverged)


def cg(A_e, b_e, indt, nd, x0, iters, **kw):
    """RESTATEMENT: unpreconditioned CG (pcg with dinv = 1 on free nodes)."""
    return pcg(A_e, b_e, indt, nd, x0, iters, precondition=False, **kw)


def chebyshev_roots(lambda1, lambda2, N):
    """solvers.py:85-99: alphas[k] = d + c cos(pi (k + 1/2)/N)."""
    if N < 1:
        raise ValueError(f"cycle length must be positive, got N={N}")
    d = (lambda2 + lambda1) / 2.0
    c = (lambda2 - lambda1) / 2.0
    k = np.arange(N)
    return d + c * np.cos(np.pi * (k + 0.5) / N)


def chebyshev2(A_e, b_e, indt, nd, x0, lambda1, lambda2, N, iters, **kw):
    """solvers.py:186-213: x += (1/alpha_{k mod N}) r."""
    alphas = chebyshev_roots(lambda1, lambda2, N)
    return _iterate(A_e, b_e, indt, nd, x0, iters,
                    lambda k, x, r: x + (1.0 / alphas[k % N]) * r, **kw)


def chebyshev3_coefficients(lambda1, lambda2, iters):
    """The scalar recurrence of solvers.py:247-258 (data independent):
    alpha_0 = 1/d; beta_k = 0.5 (c alpha_{k-1})^2 (x 0.5 for k > 1);
    alpha_k = 1/(d - beta_k/alpha_{k-1})."""
    if not lambda1 < lambda2:
        raise ValueError("chebyshev3 needs lambda1 < lambda2")
    dd = (lambda2 + lambda1) / 2.0
    cc = (lambda2 - lambda1) / 2.0
    alphas, betas = [], []
    alpha = 0.0
    for k in range(iters):
        if k == 0:
            alpha = 1.0 / dd
            beta = 0.0
        else:
            beta = 0.5 * (cc * alpha) ** 2
            if k > 1:
                beta *= 0.5
            alpha = 1.0 / (dd - beta / alpha)
        alphas.append(alpha)
        betas.append(beta)
    return np.array(alphas), np.array(betas)


def chebyshev3(A_e, b_e, indt, nd, x0, lambda1, lambda2, iters, **kw):
    """solvers.py:216-261: p = r (k=0) or r + beta_k p;  x += alpha_k p."""
    alphas, betas = chebyshev3_coefficients(lambda1, lambda2, iters)
    state = {"p": None}

    def advance(k, x, r):
        state["p"] = r.copy() if k == 0 else r + betas[k] * state["p"]
        return x + alphas[k] * state["p"]

    return _iterate(A_e, b_e, indt, nd, x0, iters, advance, **kw)


def model_eigen_bounds(n):
    """spectrum.py:41-51."""
    if n < 3:
        raise ValueError(f"need n >= 3 for an interior node, got n={n}")
    lam1 = 8.0 * np.sin(np.pi / (2 * (n - 1))) ** 2
    return float(lam1), float(8.0 - lam1)


def power_iteration_lambda_max(A_e, indt, nd, n, iters=1000, seed=0, tol=1e-10):
    """spectrum.py:64-99 (Rayleigh quotient of the masked operator)."""
    if iters < 1:
        raise ValueError(f"need at least one iteration, got {iters}")
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(n)
    v[nd] = 0.0
    nv = np.linalg.norm(v)
    if nv == 0.0:
        raise ValueError("start vector vanished after masking (no free nodes?)")
    v /= nv
    lam = 0.0
    for _ in range(iters):
        av = matvec_masked(A_e, indt, v, nd)
        lam_new = float(v @ av)
        nav = np.linalg.norm(av)
        if nav == 0.0:
            return 0.0
        v = av / nav
        if abs(lam_new - lam) <= tol * max(1.0, abs(lam_new)):
            return lam_new
        lam = lam_new
    return lam


def mass_gershgorin(M_e, indt, nd, n):
    """spectrum.py:102-126 (diag summed per j, then j = 0, 1, 2)."""
    is_free = np.ones(n, dtype=bool)
    is_free[nd] = False
    free_cols = is_free[indt].astype(np.float64)
    nb = indt.shape[0]
    rows = np.empty((nb, indt.shape[1]))
    for i in range(nb):
        acc = M_e[i, 0] * free_cols[0]
        for c in range(1, nb):
            acc = acc + M_e[i, c] * free_cols[c]
        rows[i] = acc
    row_sums = np.bincount(indt.ravel(), weights=rows.ravel(), minlength=n)
    diags = np.zeros(n)
    for j in range(nb):
        diags += np.bincount(indt[j], weights=M_e[j, j, :], minlength=n)
    lo = (2.0 * diags - row_sums)[is_free]
    hi = row_sums[is_free]
    if lo.size == 0:
        raise ValueError("no free nodes")
    return max(float(lo.min()), 0.0), float(hi.max())


def operator_bounds(A_e, M_e, indt, nd, n_side, nu, n, seed=0):
    """spectrum.py:129-149."""
    l1, l2 = model_eigen_bounds(n_side)
    if nu == 0.0:
        return l1, l2
    m_lo, _ = mass_gershgorin(M_e, indt, nd, n)
    lam1 = l1 + nu * m_lo
    lam2 = 1.05 * power_iteration_lambda_max(A_e, indt, nd, n, seed=seed)
    return lam1, float(max(lam2, lam1))


# ------------------------------------------------ partition / halo maps

def element_slabs(n_e, P):
    """operators.py:100 chunk rule reused for ranks: np.linspace(0, n_e, P+1)."""
    return np.linspace(0, n_e, P + 1, dtype=int)


def halo_maps(indt, P):
    """RESTATEMENT: per rank p with elements [lo, hi):
    local nodes = np.unique(indt[:, lo:hi]) (sorted global ids);
    interface[p][q] = intersect1d(local[p], local[q]) for q != p (non-empty);
    owner of a node = lowest rank touching it."""
    bounds = element_slabs(indt.shape[1], P)
    local = [np.unique(indt[:, lo:hi]) for lo, hi in zip(bounds[:-1], bounds[1:])]
    interface = []
    for p in range(P):
        row = {}
        for q in range(P):
            if q != p:
                common = np.intersect1d(local[p], local[q])
                if common.size:
                    row[q] = common
        interface.append(row)
    n = int(indt.max()) + 1
    owner = np.full(n, -1, dtype=np.int64)
    for p in reversed(range(P)):
        owner[local[p]] = p
    return dict(bounds=bounds, local=local, interface=interface, owner=owner)


# ---------------------------------------------- execution-plan maps (tests)

def first_appearance_order(indt, n):
    """The GPU plan's internal node numbering when the caller's numbering is
    not a structured grid (plan_numbering): nodes in order of
    first appearance when scanning elements e ascending, local vertex j
    ascending; nodes no element touches follow in ascending id order.
    Returns new_of_old (n,) i64."""
    nb, n_e = indt.shape
    flat = np.ascontiguousarray(indt.T).ravel()          # e-major scan order
    _, first = np.unique(flat, return_index=True)
    seen = np.unique(flat)
    order = seen[np.argsort(first, kind="stable")]
    rest = np.setdiff1d(np.arange(n), seen)
    old_of_new = np.concatenate([order, rest])
    new_of_old = np.empty(n, dtype=np.int64)
    new_of_old[old_of_new] = np.arange(n)
    return new_of_old


def delta_alphabet(indt, cap=32):
    """The sorted set of (neighbour - node) id differences of a mesh,
    d = indt[(j+t) % nb, e] - indt[j, e] over all e, j and t = 1..nb-1, or None
    when it has more than ``cap`` values."""
    nb = indt.shape[0]
    seen = set()
    for j in range(nb):
        for t in range(1, nb):
            seen.update(np.unique(indt[(j + t) % nb] - indt[j]).tolist())
            if len(seen) > cap:
                return None
    return np.array(sorted(seen), dtype=np.int64)


def grid_strides(indt):
    """Axis strides s0 < s1 (< s2 in 3D) of a structured numbering: the first
    choice, in lexicographic order over the positive id differences, for which
    every difference is a*s0 + b*s1 (+ c*s2) with a, b, c in {-1, 0, 1}; None
    when the differences have no such form.  The GPU plan keeps the caller's
    numbering (identity maps, 2-bit coefficients per slot and axis) exactly when
    this is not None; otherwise it uses first_appearance_order."""
    diff = delta_alphabet(indt)
    if diff is None:
        return None
    dim = indt.shape[0] - 1
    pos = [int(d) for d in diff if d > 0]
    coef = [(a, b, c) for c in (-1, 0, 1) for b in (-1, 0, 1) for a in (-1, 0, 1)
            if dim == 3 or c == 0]

    def fits(st):
        st = tuple(st) + (0,) * (3 - len(st))
        reach = {a * st[0] + b * st[1] + c * st[2] for a, b, c in coef}
        return all(int(d) in reach for d in diff)

    for i in range(len(pos)):
        for k in range(i + 1, len(pos)):
            if dim == 2:
                if fits((pos[i], pos[k])):
                    return (pos[i], pos[k])
                continue
            for m in range(k + 1, len(pos)):
                if fits((pos[i], pos[k], pos[m])):
                    return (pos[i], pos[k], pos[m])
    return None


def plan_numbering(indt, n):
    """new_of_old of the GPU plan: identity for a structured numbering
    (grid_strides), else first appearance."""
    if indt.shape[1] and grid_strides(indt) is not None:
        return np.arange(n, dtype=np.int64)
    return first_appearance_order(indt, n)


def node_slots(indt, n):
    """Per node, its (j, e) contributions in the bincount order j*n_e + e
    (operators.py:98).  Returns (rowptr (n+1,), keys) with keys = j*n_e+e."""
    nb, n_e = indt.shape
    flat = indt.ravel()
    order = np.argsort(flat, kind="stable")
    counts = np.bincount(flat, minlength=n)
    rowptr = np.concatenate([[0], np.cumsum(counts)])
    return rowptr, order.astype(np.int64)


# ------------------------------------------------------ BASELINE inputs

def config_inputs(config: int, seed: int = 0, size=None):
    """Seeded synthetic inputs of BASELINE.json configs 1-5.

    One np.random.default_rng(seed), draws in the order jitter -> permutation
    -> x.  ``size`` overrides the mesh size (level for 2D, N for 3D) so the
    same recipe can be checked at oracle-friendly sizes.  Returns a dict
    with nodes, elements, dirichlet (sorted nd), nu, f_vals (or None for
    f = 1) and x (C2 only)."""
    rng = np.random.default_rng(seed)
    out = {}
    if config in (1, 2, 4):
        level = {1: 6, 2: 11, 4: 12}[config] if size is None else size
        nodes, elements, boundary = unit_square_mesh(level)
        if config == 4:
            nodes = jitter_interior(nodes, boundary, 1.0 / 2**level, rng)
        if config in (2, 4):
            perm = rng.permutation(nodes.shape[0])
            nodes, elements, boundary = permute_mesh(nodes, elements, boundary, perm)
            out["perm"] = perm
        out.update(nodes=nodes, elements=elements, dirichlet=boundary,
                   nu={1: 1.0, 2: 1.0, 4: 10.0}[config], f_vals=None)
        if config == 4:
            c = centroids(nodes, elements)
            out["f_vals"] = np.sin(np.pi * c[:, 0]) * np.sin(np.pi * c[:, 1])
        if config == 2:
            out["x"] = rng.uniform(-1.0, 1.0, nodes.shape[0])
    elif config in (3, 5):
        N = {3: 128, 5: 256}[config] if size is None else size
        nodes, elements, face = kuhn_cube_mesh(N)
        out.update(nodes=nodes, elements=elements, dirichlet=face,
                   nu={3: 0.0, 5: 1.0}[config], f_vals=None)
    else:
        raise ValueError(f"unknown config {config}")
    return out
