"""Assembled CSR on the device -- the reference's cross-check path (reference.py:25-39,
SURVEY 8f rank 4).  Built by a node-centric kernel over the plan's incidence
(csrc/sparse.cu); never used by the matrix-free solvers.  Returns a torch sparse CSR
tensor (int64 indices, float64 values) in the caller's numbering with sorted columns."""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _device as D
from ._lib import call
from .mesh import IndexArrays


@dataclass(frozen=True, eq=False)
class _Slices:
    A_e: torch.Tensor
    index: IndexArrays
    b_e: torch.Tensor = None

    def _A_store(self):
        return self.A_e.permute(2, 0, 1).contiguous()


def assemble_sparse(slices, indt, n_nodes: int | None = None) -> torch.Tensor:
    """reference.py:25-39: every local entry (i, j, e) becomes a triplet at
    (indt[i,e], indt[j,e]); duplicates are summed (here in (j, e) slot order)."""
    A = slices if isinstance(slices, torch.Tensor) else D.f64(slices)
    A = A.to(device=D.device(), dtype=torch.float64)
    index = indt if isinstance(indt, IndexArrays) else None
    it = index.indt if index is not None else D.i32(indt)
    if A.ndim != 3 or A.shape[0] != A.shape[1] or A.shape[0] not in (3, 4) \
            or tuple(it.shape) != (A.shape[0], A.shape[2]):
        raise ValueError(f"inconsistent shapes: slices {tuple(A.shape)}, indt {tuple(it.shape)}")
    if index is None:
        index = IndexArrays(None, it)
    n = index.node_count() if n_nodes is None else int(n_nodes)
    pl = index.plan(n)
    pl.ensure_loaded(_Slices(A, index), need_be=False)
    crow = D.empty(n + 1, torch.int64)
    call("ebs_csr_nnz", pl.handle, D.ptr(index.indt), D.ptr(crow), D.stream())
    nnz = int(crow[-1])
    col = D.empty(nnz, torch.int32)
    val = D.empty(nnz)
    call("ebs_csr_fill", pl.handle, D.ptr(index.indt), D.ptr(crow), D.ptr(col), D.ptr(val),
         D.stream())
    return torch.sparse_csr_tensor(crow, col.to(torch.int64), val, size=(n, n))
