"""Meshes on the device: the reference's mesh API (mesh.py) plus the 3D Kuhn cube.

Mirrors /root/reference/pkg/src/ebsolve/mesh.py.  Differences, all deliberate:
  * arrays are torch tensors on the CUDA device; connectivity is int32 and stored
    structure-of-arrays (``conn`` = the reference ``indt``, shape (n_b, n_e)), so
    ``Mesh.elements`` is a (n_e, n_b) view of it;
  * meshes are 2D triangles (n_b = 3) or 3D tetrahedra (n_b = 4);
  * generation and validation run as CUDA kernels (libebs.so).
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as D
from ._lib import call

_PLAN_BUILD_LOCK = threading.Lock()

MAX_LEVEL = 12          # mesh.py:20
MAX_CUBE_CELLS = 256    # 3D size guard: N=256 is BASELINE C5 (100.7M tetrahedra)


@dataclass(frozen=True, eq=False)
class Mesh:
    """A simplicial mesh: node coordinates, connectivity and boundary set.

    mesh.py:25-65.  ``elements`` accepts (n_e, n_b) node-index rows (any integer
    array); validation (shape, index range, positive measure, boundary range,
    mesh.py:39-52) runs on the device.  ``conn`` (keyword) passes the int32 SoA
    connectivity directly.
    """

    nodes: torch.Tensor
    elements: torch.Tensor
    boundary_nodes: torch.Tensor
    level: int | None = None
    conn: torch.Tensor = field(default=None, repr=False)

    def __post_init__(self):
        nodes = D.f64(self.nodes)
        if nodes.ndim != 2 or nodes.shape[1] not in (2, 3):
            raise ValueError(f"nodes must have shape (n_n, 2) or (n_n, 3), got {tuple(nodes.shape)}")
        dim = nodes.shape[1]
        if self.conn is not None:
            conn = D.i32(self.conn)
        else:
            el = self.elements
            if isinstance(el, torch.Tensor):
                el_t = el
            else:
                el_t = torch.from_numpy(np.ascontiguousarray(np.asarray(el, dtype=np.int64)))
            if el_t.ndim != 2 or el_t.shape[1] != dim + 1:
                raise ValueError(
                    f"elements must have shape (n_e, {dim + 1}), got {tuple(el_t.shape)}")
            if el_t.numel() and (int(el_t.min()) < 0 or int(el_t.max()) >= nodes.shape[0]):
                raise ValueError("element connectivity references nonexistent nodes")
            conn = D.i32(el_t.t())
        if conn.ndim != 2 or conn.shape[0] != dim + 1:
            raise ValueError(f"conn must have shape ({dim + 1}, n_e), got {tuple(conn.shape)}")
        boundary = D.i64(self.boundary_nodes).reshape(-1)
        n_e = conn.shape[1]
        counts = D.zeros(2, torch.int64)
        call("ebs_mesh_check", dim, nodes.shape[0], n_e, D.ptr(nodes), D.ptr(conn),
             D.ptr(counts), D.stream())
        bad_idx, bad_meas = (int(v) for v in counts.tolist())
        if bad_idx:
            raise ValueError("element connectivity references nonexistent nodes")
        if bad_meas:
            raise ValueError("all elements must be positively oriented with positive measure "
                             "(counterclockwise triangles)")
        if boundary.numel() and (int(boundary.min()) < 0 or int(boundary.max()) >= nodes.shape[0]):
            raise ValueError("boundary_nodes out of range")
        object.__setattr__(self, "nodes", nodes)
        object.__setattr__(self, "conn", conn)
        object.__setattr__(self, "elements", conn.t())
        object.__setattr__(self, "boundary_nodes", boundary)

    @property
    def dim(self) -> int:
        return self.nodes.shape[1]

    @property
    def n_b(self) -> int:
        return self.dim + 1

    @property
    def n_nodes(self) -> int:
        return self.nodes.shape[0]

    @property
    def n_elements(self) -> int:
        return self.conn.shape[1]


@dataclass(frozen=True, eq=False)
class IndexArrays:
    """Gather/scatter index arrays (mesh.py:68-93): ``indt`` (n_b, n_e) and its
    (n_b, 1, n_e) view ``ind_e``; int32 on the device.  Holds the execution plans
    (one per node count) built from it."""

    ind_e: torch.Tensor
    indt: torch.Tensor
    n_nodes: int | None = None
    _plans: dict = field(default_factory=dict, repr=False)

    def __post_init__(self):
        indt = D.i32(self.indt)
        ind_e = D.i32(self.ind_e) if self.ind_e is not None else indt.reshape(indt.shape[0], 1, -1)
        if ind_e.ndim != 3 or ind_e.shape[1] != 1 or ind_e.shape[0] not in (3, 4):
            raise ValueError(f"ind_e must have shape (n_b, 1, n_e), got {tuple(ind_e.shape)}")
        if tuple(indt.shape) != (ind_e.shape[0], ind_e.shape[2]):
            raise ValueError(f"indt must have shape ({ind_e.shape[0]}, n_e), got {tuple(indt.shape)}")
        if not torch.equal(ind_e[:, 0, :], indt):
            raise ValueError("ind_e[:, 0, :] and indt disagree on the nodes of some element")
        if indt.numel() and int(indt.min()) < 0:
            raise ValueError("negative node index")
        object.__setattr__(self, "indt", indt)
        object.__setattr__(self, "ind_e", indt.reshape(indt.shape[0], 1, -1))

    @property
    def n_b(self) -> int:
        return self.indt.shape[0]

    @property
    def n_elements(self) -> int:
        return self.indt.shape[1]

    def node_count(self) -> int:
        if self.n_nodes is not None:
            return int(self.n_nodes)
        return int(self.indt.max()) + 1 if self.indt.numel() else 0

    def plan(self, n_nodes: int | None = None):
        """The execution plan of this connectivity for `n_nodes` nodes (cached)."""
        from .plan import Plan
        n = self.node_count() if n_nodes is None else int(n_nodes)
        pl = self._plans.get(n)
        if pl is None:
            with _PLAN_BUILD_LOCK:  # concurrent first calls build one plan
                pl = self._plans.get(n)
                if pl is None:
                    pl = Plan(self.indt, n)
                    self._plans[n] = pl
        return pl


def build_index_arrays(m: Mesh) -> IndexArrays:
    """mesh.py:151-154: column e holds element e's nodes."""
    return IndexArrays(None, m.conn, n_nodes=m.n_nodes)


def _boundary_from_flags(nodes: torch.Tensor, which: int) -> torch.Tensor:
    flags = D.empty(nodes.shape[0], torch.uint8)
    call("ebs_mesh_flags", nodes.shape[1], nodes.shape[0], D.ptr(nodes), which, D.ptr(flags),
         D.stream())
    return torch.nonzero(flags, as_tuple=False).reshape(-1).to(torch.int64)


def boundary_nodes(m: Mesh) -> torch.Tensor:
    """mesh.py:140-148: nodes with a coordinate within 1e-12 of 0 or 1, sorted."""
    return _boundary_from_flags(m.nodes, 0)


def face_z0_nodes(m: Mesh) -> torch.Tensor:
    """NEW (BASELINE C3/C5 Dirichlet face): nodes with |z| <= 1e-12, sorted."""
    if m.dim != 3:
        raise ValueError("face_z0_nodes needs a 3D mesh")
    return _boundary_from_flags(m.nodes, 1)


def signed_areas(nodes, elements=None, *, conn=None) -> torch.Tensor:
    """mesh.py:96-101 (2D signed area; 3D signed volume) for every element.
    ``elements`` is (n_e, n_b) as in the reference; ``conn`` the (n_b, n_e) SoA."""
    nodes = D.f64(nodes)
    if conn is None:
        el = elements if isinstance(elements, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(np.asarray(elements, dtype=np.int64)))
        conn = el.t()
    conn = D.i32(conn)
    out = D.empty(conn.shape[1])
    call("ebs_mesh_measure", nodes.shape[1], conn.shape[1], D.ptr(nodes), D.ptr(conn), D.ptr(out),
         D.stream())
    return out


def build_grid_mesh(n: int) -> Mesh:
    """mesh.py:104-128 on the device: n nodes per side, row-major nodes, per cell
    the lower (ll, ll+1, ll+n+1) then the upper (ll, ll+n+1, ll+n) triangle."""
    n = int(n)
    if n < 2:
        raise ValueError(f"need at least 2 nodes per side, got n={n}")
    nodes = D.empty((n * n, 2))
    conn = D.empty((3, 2 * (n - 1) ** 2), torch.int32)
    call("ebs_mesh_grid2d", n, D.ptr(nodes), D.ptr(conn), D.stream())
    level = None
    cells = n - 1
    if cells & (cells - 1) == 0:
        level = int(cells).bit_length() - 1
    return Mesh(nodes, None, _boundary_from_flags(nodes, 0), level=level, conn=conn)


def build_unit_square_mesh(level: int) -> Mesh:
    """mesh.py:131-137: (2^L+1)^2 nodes, 2*4^L triangles."""
    if not 0 <= level <= MAX_LEVEL:
        raise ValueError(f"level {level} is outside 0..{MAX_LEVEL} (the size guard)")
    return build_grid_mesh(2**level + 1)


def build_unit_cube_mesh(N: int) -> Mesh:
    """NEW (no reference code): unit cube with N cells per side, each cube split
    into 6 Kuhn tetrahedra (oracle/ebs_oracle.py kuhn_cube_mesh).  Cubes are
    visited z-outer so contiguous element ranges are z-slabs.  boundary_nodes is
    the whole cube surface (mesh.py:145-148 rule); the BASELINE Dirichlet face is
    ``face_z0_nodes``."""
    N = int(N)
    if N < 1:
        raise ValueError(f"need at least 1 cell per side, got N={N}")
    if N > MAX_CUBE_CELLS:
        raise ValueError(f"N={N} exceeds the size guard (max {MAX_CUBE_CELLS})")
    n = N + 1
    nodes = D.empty((n ** 3, 3))
    conn = D.empty((4, 6 * N ** 3), torch.int32)
    call("ebs_mesh_kuhn3d", N, D.ptr(nodes), D.ptr(conn), D.stream())
    level = N.bit_length() - 1 if N & (N - 1) == 0 else None
    return Mesh(nodes, None, _boundary_from_flags(nodes, 0), level=level, conn=conn)


def permute_nodes(m: Mesh, perm) -> Mesh:
    """NEW (BASELINE C2/C4 recipe): relabel nodes, new id of old node i is perm[i].
    Element order and local vertex order are kept; the boundary set is relabelled
    and sorted (oracle/ebs_oracle.py permute_mesh)."""
    perm_t = D.i64(perm).reshape(-1)
    if perm_t.numel() != m.n_nodes:
        raise ValueError("perm must have one entry per node")
    check = torch.zeros(m.n_nodes, dtype=torch.int64, device=perm_t.device)
    check.index_add_(0, perm_t.clamp(0, m.n_nodes - 1), torch.ones_like(perm_t))
    if int(perm_t.min()) < 0 or int(perm_t.max()) >= m.n_nodes or not bool((check == 1).all()):
        raise ValueError("perm is not a permutation of range(n_nodes)")
    nodes = D.empty(tuple(m.nodes.shape))
    conn = D.empty(tuple(m.conn.shape), torch.int32)
    call("ebs_mesh_permute", m.dim, m.n_nodes, m.n_elements, D.ptr(perm_t), D.ptr(m.nodes),
         D.ptr(m.conn), D.ptr(nodes), D.ptr(conn), D.stream())
    boundary = torch.sort(perm_t[m.boundary_nodes]).values
    return Mesh(nodes, None, boundary, level=None, conn=conn)


def jitter_interior(m: Mesh, delta) -> Mesh:
    """NEW (BASELINE C4 recipe): move the interior nodes (non-boundary, ascending
    id) by the rows of ``delta`` (n_interior, dim), e.g. seeded
    U(-0.2h, 0.2h) draws; validation rejects inverted elements."""
    is_b = torch.zeros(m.n_nodes, dtype=torch.bool, device=m.nodes.device)
    is_b[m.boundary_nodes] = True
    interior = torch.nonzero(~is_b).reshape(-1)
    delta_t = D.f64(delta).reshape(interior.numel(), m.dim)
    nodes = m.nodes.clone()
    nodes[interior] += delta_t
    return Mesh(nodes, None, m.boundary_nodes, level=None, conn=m.conn)


def uniform_refine(m: Mesh) -> Mesh:
    """Red refinement of a triangle mesh on the device (mesh.py:157-208 semantics): every
    triangle becomes 4 through its edge midpoints, then the mesh is renumbered
    canonically -- nodes ascending in (y, x), each triangle rotated to start at its
    smallest node (orientation kept), triangles ascending -- so a structured level-L
    mesh refines to exactly build_unit_square_mesh(L + 1).  One libebs call
    (ebs_refine_tri: radix-sorted edge keys, two stable coordinate sorts, child sort)."""
    if m.dim != 2:
        raise ValueError("uniform_refine splits triangles; got a tetrahedral mesh")
    if (m.level is not None and m.level >= MAX_LEVEL) or 2 * m.n_elements > 4**MAX_LEVEL:
        raise ValueError(f"the refined mesh would exceed the size guard (level {MAX_LEVEL})")
    import ctypes
    n, n_e = m.n_nodes, m.n_elements
    xy = D.empty((n + 3 * n_e, 2))
    conn = D.empty((3, 4 * n_e), torch.int32)
    n_out = ctypes.c_int64(0)
    call("ebs_refine_tri", n, n_e, D.ptr(m.nodes.contiguous()), D.ptr(m.conn), D.ptr(xy),
         D.ptr(conn), ctypes.byref(n_out), D.stream())
    nodes = xy[:n_out.value].contiguous()
    return Mesh(nodes, None, _boundary_from_flags(nodes, 0), conn=conn,
                level=None if m.level is None else m.level + 1)


def export_mesh(m: Mesh, directory) -> None:
    """Debug dump (mesh.py:211-218): nodes.txt with 17 significant digits, elements.txt
    with integer node ids, one row per node / element."""
    from pathlib import Path
    out = Path(directory)
    out.mkdir(parents=True, exist_ok=True)
    for name, arr, fmt in (("nodes.txt", m.nodes, "%.17g"), ("elements.txt", m.elements, "%d")):
        np.savetxt(out / name, arr.cpu().numpy(), fmt=fmt)
