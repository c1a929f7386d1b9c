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
from .elements import ElementBatch, using_operator
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
    r = out if out is not None else D.empty(n)
    flag = D.zeros(1, torch.int32) if check_finite else None
    with batch.using(n) as pl:
        call("ebs_residual", pl.handle, D.ptr(x), D.ptr(r),
             EBS_RES_EXACT if deterministic else EBS_RES_FAST, 0, D.ptr(flag), D.stream())
    if check_finite and int(flag.item()):
        raise ValueError("x contains non-finite entries")
    return r


def residual_many(batch: ElementBatch, xs, out=None, deterministic: bool = True,
                  check_finite: bool = True):
    """NEW: residuals of k vectors, r_i = b - A x_i -- the k-fold ``residual`` as one call.

    Device-resident ``xs`` (a (k, n) CUDA tensor, or a sequence of k CUDA vectors): returns a
    (k, n) CUDA tensor (``out``: optional contiguous (k, n) CUDA float64 tensor).  One native
    call (``ebs_residual_many``) keeps two residuals in flight on two streams, so the x
    permutation and output fill of one overlap the operator pass of the other (C2: 157 vs
    174 us per residual).

    Host-resident ``xs``: returned in host memory with the PCIe traffic overlapped.

    ``xs``: a (k, n) CPU tensor / array (pinned memory lets the copies run
    asynchronously; a broadcast (0, 1)-strided batch is read as is) or a sequence of k
    such vectors.  ``out``: an optional (k, n) contiguous CPU float64 tensor (pinned:
    asynchronous read-back), else one is allocated (pinned).  One native call
    (``ebs_residual_many_host``, csrc/hostpipe.cu): x_i goes host->device on a copy
    stream, its residual runs on the current stream, r_i goes device->host on a second
    copy stream, with device buffers kept by the plan, so the H2D of x_{i+1}, the kernels
    of x_i and the D2H of r_{i-1} overlap.  Each r_i is bit-identical to
    ``residual(batch, x_i, deterministic=...)``.  Non-finite entries in any x_i raise
    ValueError (after all residuals complete), as ``residual`` does (operators.py:87-91)."""
    import torch as _t
    seq = list(xs) if not isinstance(xs, (_t.Tensor, np.ndarray)) else None
    if seq is not None:
        xs = _t.stack([_t.as_tensor(np.asarray(v) if not isinstance(v, _t.Tensor) else v)
                       for v in seq]) if seq else _t.empty((0, 0), dtype=_t.float64)
    elif isinstance(xs, np.ndarray):
        xs = _t.from_numpy(np.ascontiguousarray(xs, dtype=np.float64))
    if xs.ndim != 2:
        raise ValueError(f"xs must be (k, n), got shape {tuple(xs.shape)}")
    if xs.device.type == "cuda":
        return _residual_many_device(batch, xs, out, deterministic, check_finite)
    if xs.dtype != _t.float64 or xs.device.type != "cpu":
        xs = xs.to(device="cpu", dtype=_t.float64)
    k, n = xs.shape
    if xs.stride(1) != 1 or (k > 1 and xs.stride(0) != 0 and xs.stride(0) < n):
        xs = xs.contiguous()
    if out is None:
        out = _t.empty((k, n), dtype=_t.float64, pin_memory=True)
    elif (tuple(out.shape) != (k, n) or out.dtype != _t.float64 or out.device.type != "cpu"
          or not out.is_contiguous()):
        raise ValueError("out must be a contiguous (k, n) float64 CPU tensor")
    if k == 0:
        return out
    flags = _t.zeros(k, dtype=_t.int32) if check_finite else None
    mode = EBS_RES_EXACT if deterministic else EBS_RES_FAST
    with using_operator(batch, n) as pl:  # the plan's operator stays loaded
        call("ebs_residual_many_host", pl.handle, xs.data_ptr(), xs.stride(0) if k > 1 else 0,
             out.data_ptr(), n, k, mode, 0, flags.data_ptr() if check_finite else None,
             D.stream())
    if check_finite:
        bad = _t.nonzero(flags).flatten()
        if bad.numel():
            raise ValueError(f"x[{int(bad[0])}] contains non-finite entries")
    return out


def _residual_many_device(batch, xs, out, deterministic, check_finite):
    """residual_many on device-resident vectors (``ebs_residual_many``)."""
    if xs.dtype != torch.float64 or xs.device != D.device():
        xs = xs.to(device=D.device(), dtype=torch.float64)
    k, n = xs.shape
    if xs.stride(1) != 1 or (k > 1 and xs.stride(0) != 0 and xs.stride(0) < n):
        xs = xs.contiguous()
    if out is None:
        out = D.empty((k, n))
    elif (not isinstance(out, torch.Tensor) or tuple(out.shape) != (k, n)
          or out.dtype != torch.float64 or out.device != xs.device or not out.is_contiguous()):
        raise ValueError("out must be a contiguous (k, n) float64 tensor on the device of xs")
    if k == 0:
        return out
    flags = D.zeros(k, torch.int32) if check_finite else None
    with using_operator(batch, n) as pl:
        call("ebs_residual_many", pl.handle, D.ptr(xs), xs.stride(0) if k > 1 else 0, D.ptr(out),
             n, k, EBS_RES_EXACT if deterministic else EBS_RES_FAST, 0, D.ptr(flags), D.stream())
    if check_finite:
        bad = torch.nonzero(flags).flatten()
        if bad.numel():
            raise ValueError(f"x[{int(bad[0])}] contains non-finite entries")
    return out


def matvec(batch: ElementBatch, v, d: DirichletData | None = None) -> torch.Tensor:
    """spectrum.py:54-61 _apply_masked: y = A v (bitwise reference order); with
    ``d`` the rows at d.nd are zeroed."""
    v = _check_x(v)
    y = D.empty(v.shape[0])
    with using_operator(batch, v.shape[0], need_be=False) as pl:
        pl.ensure_dirichlet(d)
        call("ebs_matvec", pl.handle, D.ptr(v), D.ptr(y), 1 if d is not None else 0,
             D.stream())
    return y


def diagonal(batch: ElementBatch, n_nodes: int | None = None) -> torch.Tensor:
    """NEW: diag(A) = assemble_rhs(stack_j A_e[j, j, :]) (the
    reference's own diagonal pattern, spectrum.py:118-120, in (j, e) order)."""
    with batch.using(n_nodes, need_be=False) as pl:
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
