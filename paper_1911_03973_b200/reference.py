"""Assembled-matrix ground truth (reference.py of ebsolve), on the device.

The reference keeps these out of its solver path: they exist so tests and the
``--compare-direct`` mode can check the matrix-free kernels against conventional assembly
(`/root/reference/pkg/src/ebsolve/reference.py:1-7`).  Here they take the device CSR of
``assemble_sparse`` (or a SciPy sparse matrix) and run on the GPU with PyTorch's sparse
and dense linear algebra -- they are verification utilities, not part of the hot path:

  solve_reference(A, b, d)            reference.py:42-81  Dirichlet-eliminated SPD solve
  dense_interior_eigenvalues(A, d)    reference.py:84-97  spectrum of the free block

``solve_reference`` always uses Jacobi-preconditioned CG to the reference's large-system
tolerance (rtol 1e-13, reference.py:22,69-72) -- the reference switches to SuperLU below
200k unknowns; both are exact to rounding for these SPD systems -- and applies the
reference's acceptance checks (non-finite result or a reduced residual above
1e-10 max(1, ||rhs||) raise RuntimeError).
"""

from __future__ import annotations

import torch

from . import _device as D
from .operators import DirichletData

# reference.py:20: the size above which the reference switches from a sparse direct solve to
# CG.  The device solve has one path (Jacobi-PCG to _CG_RTOL) at every size; the name is
# kept so callers that set it keep working.
_DIRECT_LIMIT = 200_000
_DENSE_EIG_LIMIT = 2000   # reference.py:21
_CG_RTOL = 1e-13          # reference.py:22


def _csr(A) -> torch.Tensor:
    """The device CSR of A (torch sparse CSR / COO, or any SciPy sparse matrix)."""
    if isinstance(A, torch.Tensor):
        if A.layout == torch.sparse_csr:
            return A.to(device=D.device(), dtype=torch.float64)
        if A.layout == torch.sparse_coo:
            return A.coalesce().to_sparse_csr().to(device=D.device(), dtype=torch.float64)
        return A.to(device=D.device(), dtype=torch.float64).to_sparse_csr()
    import scipy.sparse as sp
    a = sp.csr_matrix(A)
    a.sum_duplicates()
    return torch.sparse_csr_tensor(D.i64(a.indptr), D.i64(a.indices), D.f64(a.data),
                                   size=a.shape)


def _free_mask(n: int, d: DirichletData) -> torch.Tensor:
    free = torch.ones(n, dtype=torch.bool, device=D.device())
    if d.nd.numel():
        free[d.nd.to(free.device)] = False
    return free


def solve_reference(A, b, d: DirichletData) -> torch.Tensor:
    """reference.py:42-81: x = prescribed values on nd, and on the free nodes the solution
    of A_ff x_f = b_f - A_fd x_d (constrained rows / columns eliminated)."""
    A = _csr(A)
    n = A.shape[0]
    b = D.f64(b).reshape(-1)
    if A.shape[0] != A.shape[1] or b.numel() != n:
        raise ValueError(f"inconsistent shapes: A {tuple(A.shape)}, b {tuple(b.shape)}")
    x = torch.zeros(n, dtype=torch.float64, device=D.device())
    nd = d.nd.to(x.device)
    x[nd] = d.values.to(x.device)
    free = _free_mask(n, d)
    if not bool(free.any()):
        return x
    ff = free.to(torch.float64)

    def apply(v):  # A_ff v on free-supported vectors
        return (A @ v.unsqueeze(1)).squeeze(1) * ff

    rhs = (b - (A @ x.unsqueeze(1)).squeeze(1)) * ff   # b_f - A_fd x_d
    diag = torch.zeros(n, dtype=torch.float64, device=x.device)
    crow, col, val = A.crow_indices(), A.col_indices(), A.values()
    rows = torch.repeat_interleave(torch.arange(n, device=x.device), crow[1:] - crow[:-1])
    on = rows == col
    diag.index_add_(0, rows[on], val[on])
    dinv = torch.where(free & (diag != 0), 1.0 / diag, torch.zeros_like(diag))
    # Jacobi-preconditioned CG, scipy's stopping rule ||r|| < rtol ||b|| (iterative.py)
    u = torch.zeros_like(x)
    r = rhs.clone()
    z = dinv * r
    p = z.clone()
    rz = float(r @ z)
    bnorm = float(torch.linalg.vector_norm(rhs))
    stop = _CG_RTOL * bnorm
    maxiter = 20 * int(free.sum())
    it = 0
    while float(torch.linalg.vector_norm(r)) >= stop and bnorm > 0:
        if it >= maxiter:
            raise RuntimeError(f"conjugate gradient failed to converge ({it} iterations)")
        q = apply(p)
        alpha = rz / float(p @ q)
        u += alpha * p
        r -= alpha * q
        z = dinv * r
        rz_new = float(r @ z)
        p = z + (rz_new / rz) * p
        rz = rz_new
        it += 1
    if not bool(torch.isfinite(u).all()):
        raise RuntimeError("factorization produced non-finite values (system not SPD?)")
    check = float(torch.linalg.vector_norm(apply(u) - rhs))
    if check > 1e-10 * max(1.0, bnorm):
        raise RuntimeError(f"reduced solve inaccurate (residual {check:.3e}); system not SPD?")
    x[free] = u[free]
    return x


def dense_interior_eigenvalues(A, d: DirichletData) -> torch.Tensor:
    """reference.py:84-97: the full ascending spectrum of the free-node principal
    submatrix (dense, fp64 eigvalsh on the device); ValueError beyond 2000 free nodes."""
    A = _csr(A)
    n = A.shape[0]
    free = torch.nonzero(_free_mask(n, d)).reshape(-1)
    if free.numel() > _DENSE_EIG_LIMIT:
        raise ValueError(f"{free.numel()} free nodes exceed the dense-eigensolver guard "
                         f"({_DENSE_EIG_LIMIT})")
    dense = A.to_dense()[free][:, free]
    return torch.linalg.eigvalsh(dense)


__all__ = ["solve_reference", "dense_interior_eigenvalues"]
