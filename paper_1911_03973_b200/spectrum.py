"""Eigenvalue bounds for the interior operator (spectrum.py of the reference).

Closed-form model bounds on the host (spectrum.py:31-51); for nu > 0 the power
iteration runs on the device (``ebs_power_iteration``: the fused SELL matvec with the
Rayleigh quotient and norm reduced in-kernel) and the Gershgorin bound of the mass
matrix uses the device matvec / diagonal (spectrum.py:102-126).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as D
from ._lib import call
from .elements import ElementBatch, using_operator
from .operators import DirichletData, matvec
from .solvers import SpectralBounds

POWER_ITERS = 1000     # spectrum.py:26
POWER_TOL = 1e-10      # spectrum.py:27
POWER_MARGIN = 1.05    # spectrum.py:28


def _interior_sines(n: int) -> np.ndarray:
    """sin^2(i pi / (2 (n-1))), i = 1..n-2: the 1D factors of the model eigenvalues."""
    if n < 3:
        raise ValueError(f"{n} nodes per side leave no interior node (need n >= 3)")
    return np.sin(np.arange(1, n - 1) * np.pi / (2 * (n - 1))) ** 2


def model_eigenvalues_all(n: int) -> np.ndarray:
    """Every interior eigenvalue 4 (s_i + s_j) of the model stiffness matrix on the
    n x n grid, ascending (spectrum.py:31-38)."""
    s = _interior_sines(n)
    return np.sort((4.0 * np.add.outer(s, s)).ravel())


def model_eigen_bounds(n: int) -> SpectralBounds:
    """Extreme model eigenvalues (spectrum.py:41-51): the smallest from i = j = 1; the
    largest is its complement 8 - lambda1 (the extreme sine arguments are complementary
    angles), taken that way as the reference does."""
    if n < 3:
        raise ValueError(f"{n} nodes per side leave no interior node (need n >= 3)")
    low = 8.0 * np.sin(np.pi / (2 * (n - 1))) ** 2
    return SpectralBounds(float(low), float(8.0 - low))


def power_iteration_lambda_max(batch: ElementBatch, d: DirichletData, iters: int = POWER_ITERS,
                               seed: int = 0, tol: float = POWER_TOL) -> float:
    """spectrum.py:64-99: Rayleigh-quotient estimate of the largest eigenvalue of the
    masked operator; the seeded start vector is drawn on the host exactly as the
    reference does, the iteration runs on the device."""
    if iters < 1:
        raise ValueError(f"need at least one iteration, got {iters}")
    n_n = batch.index.node_count()
    rng = np.random.default_rng(seed)
    v0 = D.f64(rng.standard_normal(n_n))
    lam = ctypes.c_double(0.0)
    its = ctypes.c_int(0)
    with using_operator(batch, n_n, need_be=False) as pl:
        pl.ensure_dirichlet(d)
        call("ebs_power_iteration", pl.handle, D.ptr(v0), int(iters), float(tol),
             ctypes.byref(lam), ctypes.byref(its), D.stream())
    return float(lam.value)


@dataclass(frozen=True, eq=False)
class _MassBatch:
    """The mass slices as an operator (same plan, A_e := M_e)."""
    M_e: torch.Tensor
    index: object
    b_e: torch.Tensor = None
    _w: list = field(default_factory=list)

    def _A_store(self):
        return self.M_e.permute(2, 0, 1).contiguous()

    def operator(self, n_nodes=None, need_be=False):
        pl = self.index.plan(n_nodes)
        with pl.lock:
            pl.ensure_loaded(self, need_be=False)
        return pl


def mass_gershgorin(batch: ElementBatch, d: DirichletData) -> tuple[float, float]:
    """spectrum.py:102-126: Gershgorin enclosure of the free-node mass spectrum.
    Row sums over free columns = M times the free indicator (device matvec, the
    reference's einsum + bincount order); diagonal summed per j then over j, as the
    reference does -- both bit-identical."""
    n_n = batch.index.node_count()
    mb = _MassBatch(batch.M_e, batch.index)
    is_free = torch.ones(n_n, dtype=torch.bool, device=D.device())
    if d.nd.numel():
        is_free[d.nd] = False
    row_sums = matvec(mb, is_free.to(torch.float64))
    diags = D.empty(n_n)
    with using_operator(mb, n_n, need_be=False) as pl:
        call("ebs_diagonal_grouped", pl.handle, D.ptr(diags), D.stream())
    if not bool(is_free.any()):
        raise ValueError("every node is constrained: no free-node mass spectrum to bound")
    # mass entries are >= 0, so a free row's disc is [2 diag - rowsum, rowsum]
    upper_edges = row_sums[is_free]
    lower_edges = 2.0 * diags[is_free] - upper_edges
    return max(float(lower_edges.min()), 0.0), float(upper_edges.max())


def operator_bounds(batch: ElementBatch, d: DirichletData, n: int, nu: float,
                    seed: int = 0) -> SpectralBounds:
    """Bounds for A = K + nu M (spectrum.py:129-149).  nu = 0: the model interval.
    nu > 0: lower end = model minimum + nu x (Gershgorin floor of the constrained mass
    spectrum), upper end = power-iteration maximum widened by POWER_MARGIN."""
    model = model_eigen_bounds(n)
    if nu == 0.0:
        return model
    mass_floor = mass_gershgorin(batch, d)[0]
    lower = model.lambda1 + nu * mass_floor
    upper = POWER_MARGIN * power_iteration_lambda_max(batch, d, seed=seed)
    return SpectralBounds(lower, float(max(upper, lower)))
