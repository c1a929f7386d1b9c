"""Iterative solvers on the device (solvers.py of the reference, plus Jacobi/CG/PCG).

All methods run the reference's shared loop (`_iterate`, solvers.py:117-160) inside
libebs.so (``ebs_solve``): the residual norms stay on the device and are read once
at the end; the iteration stops on ``tol`` relative to ||r_0||; divergence sets a
flag and is never raised; ``callback(k, x, r)`` is called for k = 0..iters with
fresh device tensors in the caller's numbering, as the reference hands a new x and r at
every k (solvers.py:137-149); ``reuse_callback_buffers=True`` passes the same two buffers
every time instead (no per-iteration copy; clone to keep them).

  richardson  x += omega r, omega = 2/(l1+l2)          solvers.py:163-183
  chebyshev2  x += (1/alpha_{k mod N}) r               solvers.py:186-213
  chebyshev3  p = r + beta_k p; x += alpha_k p         solvers.py:216-261
  jacobi      x += omega D^-1 r                        NEW (north star)
  cg / pcg    (Jacobi-preconditioned) CG on the masked operator  NEW (north star)

The Chebyshev step scalars are data independent; they are computed on the host with the
reference's exact expressions and streamed to the fused step kernel, so the iterates are
bit-identical to ebsolve's.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np

from . import _device as D
from ._lib import (CALLBACK, EBS_CG, EBS_CHEB2, EBS_CHEB3, EBS_ECALLBACK, EBS_JACOBI, EBS_PCG,
                   EBS_RICHARDSON, SolveParams, check, load)
from .elements import ElementBatch
from .operators import DirichletData


@dataclass(frozen=True)
class SpectralBounds:
    """Spectral enclosure [lambda1, lambda2] of the constrained operator (the reference
    type, solvers.py:30-56): finite, 0 <= lambda1 <= lambda2, lambda2 > 0."""

    lambda1: float
    lambda2: float

    def __post_init__(self):
        lo, hi = self.lambda1, self.lambda2
        if not np.isfinite([lo, hi]).all():
            raise ValueError(f"spectral bounds [{lo}, {hi}] are not finite")
        if lo < 0 or hi <= 0 or hi < lo:
            raise ValueError(f"[{lo}, {hi}] is not an interval 0 <= lambda1 <= lambda2, "
                             "lambda2 > 0")

    # midpoint d and half-width c of the interval (same rounding as the reference)
    center = property(lambda self: (self.lambda2 + self.lambda1) / 2.0)
    half_width = property(lambda self: (self.lambda2 - self.lambda1) / 2.0)


@dataclass(frozen=True)
class ChebyshevCycle:
    """Step denominators of one cycle of the two-level iteration (solvers.py:59-66)."""

    N: int
    alphas: np.ndarray
    d: float
    c: float


def chebyshev_roots(bounds: SpectralBounds, N: int) -> ChebyshevCycle:
    """The N roots of the degree-N Chebyshev polynomial mapped onto the interval,
    alpha_k = d + c cos(pi (k + 1/2) / N), k = 0..N-1 (descending; solvers.py:85-99)."""
    N = int(N)
    if N <= 0:
        raise ValueError(f"a Chebyshev cycle needs N >= 1 (got {N})")
    mid, half = bounds.center, bounds.half_width
    theta = np.pi * (np.arange(N) + 0.5) / N
    roots = mid + half * np.cos(theta)
    roots.setflags(write=False)
    return ChebyshevCycle(N=N, alphas=roots, d=mid, c=half)


def chebyshev_scaling_factor(bounds: SpectralBounds, k: int) -> float:
    """T_k(sigma) at sigma = (lambda1 + lambda2) / (lambda2 - lambda1), by the recurrence
    T_{j+1} = 2 sigma T_j - T_{j-1} from T_0 = 1, T_1 = sigma (solvers.py:102-114)."""
    if k < 0:
        raise ValueError(f"polynomial degree must be >= 0 (got {k})")
    lo, hi = bounds.lambda1, bounds.lambda2
    if not lo < hi:
        raise ValueError("the scaling factor needs a nondegenerate interval lambda1 < lambda2")
    sigma = (lo + hi) / (hi - lo)
    t = [1.0, sigma]
    for _ in range(k - 1):
        t = [t[1], 2.0 * sigma * t[1] - t[0]]
    return t[0] if k == 0 else t[1]


@dataclass(frozen=True)
class ConvergenceHistory:
    """solvers.py:69-82: residual_norms[k] = ||r^k||_2 for k = 0..iters (host arrays)."""

    residual_norms: np.ndarray
    error_norms: np.ndarray | None
    wall_time: float
    diverged: bool = False

    @property
    def iterations(self) -> int:
        return len(self.residual_norms) - 1


def _solve(method, batch: ElementBatch, d: DirichletData, x0, iters, *, omega=1.0, exact=False,
           tol=None, reference=None, callback=None, coef_a=None, coef_b=None, fused=False,
           reuse_callback_buffers=False):
    if iters < 0:
        raise ValueError(f"iteration count must be nonnegative, got {iters}")
    x0 = D.f64(x0)
    if x0.ndim != 1:
        raise ValueError(f"x0 must be a flat global vector, got shape {tuple(x0.shape)}")
    n = x0.shape[0]
    x = D.empty(n)
    ref = D.f64(reference) if reference is not None else None
    norms = (ctypes.c_double * (iters + 2))()
    errors = (ctypes.c_double * (iters + 2))()
    n_norms = ctypes.c_int(0)
    diverged = ctypes.c_int(0)
    state = {"exc": None}
    cb_x = cb_r = None
    cb_fn = CALLBACK()
    if callback is not None:
        cb_x = D.empty(n)
        cb_r = D.empty(n)

        def _cb(user, k):
            try:
                if reuse_callback_buffers:
                    callback(int(k), cb_x, cb_r)
                else:
                    callback(int(k), cb_x.clone(), cb_r.clone())
                return 0
            except BaseException as e:  # re-raised after the C call returns
                state["exc"] = e
                return 1

        cb_fn = CALLBACK(_cb)
    P = SolveParams()
    P.method = method
    P.iters = int(iters)
    P.exact = 1 if exact else 0
    P.has_tol = 0 if tol is None else 1
    P.tol = 0.0 if tol is None else float(tol)
    P.omega = float(omega)
    P.x0 = x0.data_ptr()
    P.x = x.data_ptr()
    P.reference = ref.data_ptr() if ref is not None else None
    P.norms = ctypes.cast(norms, ctypes.POINTER(ctypes.c_double))
    P.errors = ctypes.cast(errors, ctypes.POINTER(ctypes.c_double))
    P.n_norms = ctypes.pointer(n_norms)
    P.diverged = ctypes.pointer(diverged)
    P.callback = cb_fn
    P.user = None
    P.cb_x = cb_x.data_ptr() if cb_x is not None else None
    P.cb_r = cb_r.data_ptr() if cb_r is not None else None
    P.r_out = None
    P.fused = 1 if fused else 0
    ca = cb = None
    if coef_a is not None:
        ca = (ctypes.c_double * max(1, len(coef_a)))(*coef_a)
        P.coef_a = ctypes.cast(ca, ctypes.POINTER(ctypes.c_double))
    if coef_b is not None:
        cb = (ctypes.c_double * max(1, len(coef_b)))(*coef_b)
        P.coef_b = ctypes.cast(cb, ctypes.POINTER(ctypes.c_double))
    t0 = time.perf_counter()
    with batch.using(n) as pl:  # operator + Dirichlet set stay loaded for the whole solve
        pl.ensure_dirichlet(d)
        code = load().ebs_solve(pl.handle, ctypes.byref(P), D.stream())
    wall = time.perf_counter() - t0
    if code == EBS_ECALLBACK and state["exc"] is not None:
        raise state["exc"]
    check(code, "ebs_solve")
    k = n_norms.value
    hist = ConvergenceHistory(
        residual_norms=np.array(norms[:k]),
        error_norms=np.array(errors[:k]) if ref is not None else None,
        wall_time=wall, diverged=bool(diverged.value))
    return x, hist


def richardson(batch: ElementBatch, d: DirichletData, x0, bounds: SpectralBounds, iters: int, *,
               tol=None, reference=None, callback=None, threads: int = 1,
               deterministic: bool = True, reuse_callback_buffers: bool = False):
    """solvers.py:163-183: damped Richardson with the step 2/(lambda1+lambda2).

    With ``deterministic=True`` the residual is the reference-order exact one, so
    the iterates are bit-identical to ebsolve.richardson."""
    omega = 2.0 / (bounds.lambda1 + bounds.lambda2)
    return _solve(EBS_RICHARDSON, batch, d, x0, iters, omega=omega, exact=deterministic, tol=tol,
                  reference=reference, callback=callback,
                  reuse_callback_buffers=reuse_callback_buffers)


def chebyshev2(batch: ElementBatch, d: DirichletData, x0, bounds: SpectralBounds, N: int,
               iters: int, *, tol=None, reference=None, callback=None, threads: int = 1,
               deterministic: bool = True, reuse_callback_buffers: bool = False):
    """solvers.py:186-213: cyclic two-level Chebyshev, roots in natural order."""
    cycle = chebyshev_roots(bounds, N)
    if iters < 0:
        raise ValueError(f"iteration count must be nonnegative, got {iters}")
    coef = [1.0 / cycle.alphas[k % cycle.N] for k in range(iters)]
    return _solve(EBS_CHEB2, batch, d, x0, iters, exact=deterministic, tol=tol,
                  reference=reference, callback=callback, coef_a=coef,
                  reuse_callback_buffers=reuse_callback_buffers)


def _chebyshev3_coefficients(bounds: SpectralBounds, iters: int):
    """The scalar recurrence of solvers.py:247-258, same expressions."""
    dd = bounds.center
    cc = bounds.half_width
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
    return alphas, betas


def chebyshev3(batch: ElementBatch, d: DirichletData, x0, bounds: SpectralBounds, iters: int, *,
               tol=None, reference=None, callback=None, threads: int = 1,
               deterministic: bool = True, reuse_callback_buffers: bool = False):
    """solvers.py:216-261: three-level Chebyshev via the stable two-term recurrence."""
    if not bounds.lambda1 < bounds.lambda2:
        raise ValueError("chebyshev3 needs lambda1 < lambda2")
    if iters < 0:
        raise ValueError(f"iteration count must be nonnegative, got {iters}")
    a, b = _chebyshev3_coefficients(bounds, iters)
    return _solve(EBS_CHEB3, batch, d, x0, iters, exact=deterministic, tol=tol,
                  reference=reference, callback=callback, coef_a=a, coef_b=b,
                  reuse_callback_buffers=reuse_callback_buffers)


def jacobi(batch: ElementBatch, d: DirichletData, x0, iters: int, *, omega: float = 0.8,
           tol=None, reference=None, callback=None, deterministic: bool = False,
           reuse_callback_buffers: bool = False):
    """NEW: damped Jacobi x += omega * (D^-1 mask(b - A x)), D = diagonal(batch),
    on the _iterate loop (oracle/ebs_oracle.py jacobi)."""
    return _solve(EBS_JACOBI, batch, d, x0, iters, omega=omega, exact=deterministic, tol=tol,
                  reference=reference, callback=callback,
                  reuse_callback_buffers=reuse_callback_buffers)


def cg(batch: ElementBatch, d: DirichletData, x0, iters: int, *, tol=None, reference=None,
       callback=None, fused: bool = False, reuse_callback_buffers: bool = False):
    """NEW: conjugate gradients on the Dirichlet-masked operator (oracle pcg with
    dinv = 1); history holds the recursive residual norms.  fused=True (no callback):
    the whole loop as one cooperative persistent kernel."""
    return _solve(EBS_CG, batch, d, x0, iters, tol=tol, reference=reference, callback=callback,
                  fused=fused, reuse_callback_buffers=reuse_callback_buffers)


def pcg(batch: ElementBatch, d: DirichletData, x0, iters: int, *, tol=None, reference=None,
        callback=None, fused: bool = False, reuse_callback_buffers: bool = False):
    """NEW: Jacobi (diagonal) preconditioned CG (oracle/ebs_oracle.py pcg).  fused=True
    (no callback): the whole loop as one cooperative persistent kernel -- three grid-wide
    barriers per iteration instead of three launches (small, latency-bound meshes)."""
    return _solve(EBS_PCG, batch, d, x0, iters, tol=tol, reference=reference, callback=callback,
                  fused=fused, reuse_callback_buffers=reuse_callback_buffers)
