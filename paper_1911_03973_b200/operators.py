"""Matrix-free element operator on the device (operators.py of the reference).

The global matrix is never formed.  ``residual`` computes

    r = sum_e scatter(b_e - A_e x[ind_e])

with one gather kernel and one fused SELL kernel (csrc/sell.cuh): each node walks
its (j, e) contributions in the reference's bincount order, so the default
(``deterministic=True``) result is bit-identical to ``ebsolve.residual``.
``deterministic=False`` selects the faster form b - A x with a pre-assembled b
(still run-to-run reproducible; within rounding of the reference).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from ._lib import EBS_RES_EXACT, EBS_RES_FAST, call
from .elements import ElementBatch
from .mesh import IndexArrays, Mesh


@dataclass(frozen=True, eq=False)
class DirichletData:
    """operators.py:29-49: constrained node indices (sorted, unique) and values."""

    nd: torch.Tensor
    values: torch.Tensor

    def __post_init__(self):
        if len(np.shape(self.nd)) != 1:
            raise ValueError("nd and values must be 1-D arrays of equal length")
        nd = D.i64(self.nd)
        values = D.f64(self.values)
        if values.ndim != 1 or tuple(values.shape) != tuple(nd.shape):
            raise ValueError("nd and values must be 1-D arrays of equal length")
        order = torch.argsort(nd, stable=True)
        nd = nd[order].contiguous()
        values = values[order].contiguous()
        if nd.numel() > 1 and bool((nd[1:] == nd[:-1]).any()):
            raise ValueError("duplicate constrained node indices")
        object.__setattr__(self, "nd", nd)
        object.__setattr__(self, "values", values)


def constant_dirichlet(m: Mesh, value: float = 1.0) -> DirichletData:
    """operators.py:52-55: every boundary node of the mesh at one value."""
    nd = m.boundary_nodes
    return DirichletData(nd, torch.full(tuple(nd.shape), float(value), dtype=torch.float64,
                                        device=nd.device))


def assemble_rhs(b_e, indt) -> torch.Tensor:
    """operators.py:58-63: b = bincount(indt, b_e) in (j, e) order (bitwise)."""
    b_e = D.f64(b_e)
    index = indt if isinstance(indt, IndexArrays) else None
    it = index.indt if index is not None else D.i32(indt)
    if tuple(b_e.shape) != tuple(it.shape):
        raise ValueError(f"shape mismatch: b_e {tuple(b_e.shape)} vs indt {tuple(it.shape)}")
    if index is None:
        index = _index_cache(it)
    pl = index.plan()
    out = D.empty(pl.n_nodes)
    call("ebs_assemble_rhs", pl.handle, D.ptr(b_e), D.ptr(out), D.stream())
    return out


_INDEX_CACHE: dict = {}


def _index_cache(indt: torch.Tensor) -> IndexArrays:
    key = (indt.data_ptr(), tuple(indt.shape), indt.dtype)
    ent = _INDEX_CACHE.get(key)
    if ent is None or ent[0]() is None:
        import weakref
        ia = IndexArrays(None, indt)
        _INDEX_CACHE[key] = (weakref.ref(indt), ia)
        return ia
    return ent[1]


def _check_x(x):
    x = D.f64(x)
    if x.ndim != 1:
        raise ValueError(f"x must be a flat global vector, got shape {tuple(x.shape)}")
    return x


def residual(batch: ElementBatch, x, threads: int = 1, deterministic: bool = True, *,
             out: torch.Tensor | None = None, check_finite: bool = True) -> torch.Tensor:
    """operators.py:72-111: r = b - A x without forming A.

    ``threads`` is accepted for signature compatibility (the GPU grid replaces the
    element-chunk thread pool).  ``deterministic=True``: bit-identical to the
    reference.  ``deterministic=False``: b - A x with pre-assembled b.
    Raises ValueError for a non 1-D or non-finite x (operators.py:87-91)."""
    x = _check_x(x)
    n = x.shape[0]
    pl = batch.operator(n)
    r = out if out is not None else D.empty(n)
    flag = D.zeros(1, torch.int32) if check_finite else None
    call("ebs_residual", pl.handle, D.ptr(x), D.ptr(r),
         EBS_RES_EXACT if deterministic else EBS_RES_FAST, 0, D.ptr(flag), D.stream())
    if check_finite and int(flag.item()):
        raise ValueError("x contains non-finite entries")
    return r


def matvec(batch: ElementBatch, v, d: DirichletData | None = None) -> torch.Tensor:
    """spectrum.py:54-61 _apply_masked: y = A v (bitwise reference order); with
    ``d`` the rows at d.nd are zeroed."""
    v = _check_x(v)
    pl = batch.operator(v.shape[0], need_be=False)
    pl.ensure_dirichlet(d)
    y = D.empty(v.shape[0])
    call("ebs_matvec", pl.handle, D.ptr(v), D.ptr(y), 1 if d is not None else 0, D.stream())
    return y


def diagonal(batch: ElementBatch, n_nodes: int | None = None) -> torch.Tensor:
    """NEW: diag(A) = assemble_rhs(stack_j A_e[j, j, :]) (the
    reference's own diagonal pattern, spectrum.py:118-120, in (j, e) order)."""
    pl = batch.operator(n_nodes, need_be=False)
    d = D.empty(pl.n_nodes)
    call("ebs_diagonal", pl.handle, D.ptr(d), D.stream())
    return d


def mask_dirichlet(r, d: DirichletData) -> torch.Tensor:
    """operators.py:114-118: zero the residual at constrained nodes (returns a copy)."""
    r = D.f64(r)
    out = D.empty(tuple(r.shape))
    call("ebs_mask", r.numel(), D.ptr(r), d.nd.numel(), D.ptr(d.nd), D.ptr(out), D.stream())
    return out


def apply_initial_guess(m: Mesh, d: DirichletData) -> torch.Tensor:
    """operators.py:121-125: prescribed values on constrained nodes, 0 elsewhere."""
    x0 = D.zeros(m.n_nodes)
    if d.nd.numel():
        x0[d.nd] = d.values
    return x0
