"""Batched P1 element matrices on the device (elements.py of the reference).

One fused CUDA kernel (``ebs_assemble_p1``) computes the geometry once and writes
K_e, M_e, A_e = K_e + nu*M_e and b_e.  Layouts follow the reference: K/M/A are
(n_b, n_b, n_e) views of element-major (n_e, n_b, n_b) storage
(elements.py:86,93), b_e is a contiguous (n_b, n_e) array (elements.py:112).
Triangles are bit-identical to ``build_element_batch``; tetrahedra follow the
oracle restatement (oracle/ebs_oracle.py element_matrices).
"""

from __future__ import annotations

import contextlib

from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from ._lib import call
from .mesh import IndexArrays, Mesh, build_index_arrays, signed_areas

EPS_AREA = 1e-14      # elements.py:19
EPS_VOLUME = 1e-18    # tetrahedra (restatement)


def _host_tensor(a) -> torch.Tensor:
    """A float64 CPU tensor over a host array (read-only arrays, e.g. the reference's frozen
    fields, are copied: torch needs a writable buffer)."""
    a = np.asarray(a, dtype=np.float64)
    return torch.from_numpy(a if a.flags.writeable else a.copy())


@dataclass(frozen=True, eq=False)
class ElementBatch:
    """elements.py:25-53: everything the element operator needs."""

    K_e: torch.Tensor
    M_e: torch.Tensor
    A_e: torch.Tensor
    b_e: torch.Tensor
    nu: float
    index: IndexArrays

    def __post_init__(self):
        n_b, n_e = self.index.n_b, self.index.n_elements
        vals = {}
        for name in ("K_e", "M_e", "A_e"):
            arr = getattr(self, name)
            t = arr if isinstance(arr, torch.Tensor) else _host_tensor(arr)
            if tuple(t.shape) != (n_b, n_b, n_e):
                raise ValueError(f"{name} must have shape ({n_b}, {n_b}, {n_e}), got {tuple(t.shape)}")
            if t.device != D.device() or t.dtype != torch.float64:
                t = t.to(device=D.device(), dtype=torch.float64)
            vals[name] = t
        b = self.b_e if isinstance(self.b_e, torch.Tensor) else _host_tensor(self.b_e)
        if tuple(b.shape) != (n_b, n_e):
            raise ValueError(f"b_e must have shape ({n_b}, {n_e}), got {tuple(b.shape)}")
        if self.nu < 0:
            raise ValueError(f"nu must be nonnegative, got {self.nu}")
        for name, t in vals.items():
            object.__setattr__(self, name, t)
        object.__setattr__(self, "b_e", D.f64(b))
        object.__setattr__(self, "nu", float(self.nu))

    @property
    def n_elements(self) -> int:
        return self.index.n_elements

    def _A_store(self) -> torch.Tensor:
        """Element-major (n_e, n_b, n_b) contiguous storage of A_e."""
        return self.A_e.permute(2, 0, 1).contiguous()

    def operator(self, n_nodes: int | None = None, need_be: bool = True):
        """The execution plan of this batch's mesh with A_e (and b_e) packed."""
        pl = self.index.plan(n_nodes)
        with pl.lock:
            pl.ensure_loaded(self, need_be=need_be)
        return pl

    def using(self, n_nodes: int | None = None, need_be: bool = True):
        """Context manager: the plan with this batch loaded, locked until the block
        exits (wrap the enqueue of every operation that relies on the loaded state)."""
        return using_operator(self, n_nodes, need_be)


@contextlib.contextmanager
def using_operator(batch, n_nodes=None, need_be=True):
    """The plan of `batch` (anything with .index and ._A_store) with its operator
    loaded, held under the plan's lock for the duration of the block."""
    pl = batch.index.plan(n_nodes)
    with pl.lock:
        pl.ensure_loaded(batch, need_be=need_be)
        yield pl


def _source_values(m: Mesh, f):
    """f evaluated at the element centroids (elements.py:107-111).

    ``f`` is called like the reference: with NumPy coordinate arrays (x, y[, z]);
    a scalar is broadcast.  A torch tensor / array of n_e values is taken as is."""
    if f is None:
        return None, 1.0
    if isinstance(f, (int, float)):
        v = float(f)
        if not np.isfinite(v):
            raise ValueError("source function returned non-finite values")
        return None, v
    if isinstance(f, (torch.Tensor, np.ndarray)):
        vals = D.f64(f).reshape(-1)
    else:
        cent = D.empty((m.n_elements, m.dim))
        call("ebs_centroids", m.dim, m.n_elements, D.ptr(m.nodes), D.ptr(m.conn), D.ptr(cent),
             D.stream())
        c = cent.cpu().numpy()
        out = np.asarray(f(*[c[:, a] for a in range(m.dim)]), dtype=np.float64)
        vals = D.f64(np.ascontiguousarray(np.broadcast_to(out, (m.n_elements,))))
    if vals.numel() != m.n_elements:
        raise ValueError("source values must have one entry per element")
    if not bool(torch.isfinite(vals).all()):
        raise ValueError("source function returned non-finite values")
    return vals, 0.0


def _assemble(m: Mesh, nu=0.0, f=None, want=("K", "M", "A", "b"), check_degenerate=True):
    if nu < 0:
        raise ValueError(f"nu must be nonnegative, got {nu}")
    nb, n_e = m.n_b, m.n_elements
    out = {}
    for k in ("K", "M", "A"):
        out[k] = D.empty((n_e, nb, nb)) if k in want else None
    out["b"] = D.empty((nb, n_e)) if "b" in want else None
    f_vals, f_const = _source_values(m, f) if "b" in want else (None, 1.0)
    ndeg = D.zeros(1, torch.int64)
    call("ebs_assemble_p1", m.dim, n_e, D.ptr(m.nodes), D.ptr(m.conn), float(nu),
         D.ptr(f_vals), float(f_const), D.ptr(out["K"]), D.ptr(out["M"]), D.ptr(out["A"]),
         D.ptr(out["b"]), D.ptr(ndeg), D.stream())
    if check_degenerate and int(ndeg.item()):
        meas = signed_areas(m.nodes, conn=m.conn)
        worst = int(torch.argmin(meas))
        what, eps = ("area", EPS_AREA) if m.dim == 2 else ("volume", EPS_VOLUME)
        raise ValueError(
            f"degenerate element {worst}: {what} {float(meas[worst]):.3e} <= {eps}")
    view = {k: (v.permute(1, 2, 0) if v is not None else None) for k, v in out.items() if k != "b"}
    return view, out["b"]


def local_stiffness_batch(m: Mesh) -> torch.Tensor:
    """elements.py:81-86: K slices = measure * G^T G, shape (n_b, n_b, n_e)."""
    return _assemble(m, want=("K",))[0]["K"]


def local_mass_batch(m: Mesh) -> torch.Tensor:
    """elements.py:89-93: M slices = measure * (1 + delta_ij)/12 (tets: /20)."""
    return _assemble(m, want=("M",))[0]["M"]


def local_load_batch(m: Mesh, f) -> torch.Tensor:
    """elements.py:96-112: b_e[j] = f(centroid) * measure / n_b, shape (n_b, n_e)."""
    if f is None:
        raise ValueError("local_load_batch needs a source f")
    return _assemble(m, f=f, want=("b",), check_degenerate=False)[1]


def combine_system(K_e, M_e, nu: float) -> torch.Tensor:
    """elements.py:115-121: A_e = K_e + nu*M_e (keeps the element-major layout)."""
    K = K_e if isinstance(K_e, torch.Tensor) else D.f64(K_e)
    M = M_e if isinstance(M_e, torch.Tensor) else D.f64(M_e)
    if tuple(K.shape) != tuple(M.shape):
        raise ValueError(f"shape mismatch: K_e {tuple(K.shape)} vs M_e {tuple(M.shape)}")
    if nu < 0:
        raise ValueError(f"nu must be nonnegative, got {nu}")
    nb, _, n_e = K.shape
    Ks = K.permute(2, 0, 1).contiguous()
    Ms = M.permute(2, 0, 1).contiguous()
    A = D.empty((n_e, nb, nb))
    call("ebs_combine", A.numel(), D.ptr(Ks), D.ptr(Ms), float(nu), D.ptr(A), D.stream())
    return A.permute(1, 2, 0)


def build_element_batch(m: Mesh, nu: float = 0.0, f=None) -> ElementBatch:
    """elements.py:124-137 (default source f = 1), one fused kernel."""
    view, b_e = _assemble(m, nu=nu, f=f)
    return ElementBatch(K_e=view["K"], M_e=view["M"], A_e=view["A"], b_e=b_e, nu=float(nu),
                        index=build_index_arrays(m))
