"""Closed-form spectral bounds of the model stiffness system (spectrum.py:31-51).

Host-side scalars the Richardson step needs (omega = 2/(l1+l2)); the power
iteration / Gershgorin bounds for nu > 0 are a SURVEY 8f "next" row.
"""

from __future__ import annotations

import numpy as np

from .solvers import SpectralBounds


def model_eigenvalues_all(n: int) -> np.ndarray:
    """spectrum.py:31-38: all (n-2)^2 interior eigenvalues for n nodes per side."""
    if n < 3:
        raise ValueError(f"need n >= 3 for an interior node, got n={n}")
    i = np.arange(1, n - 1)
    s = np.sin(i * np.pi / (2 * (n - 1))) ** 2
    lam = 4.0 * (s[:, None] + s[None, :])
    return np.sort(lam.ravel())


def model_eigen_bounds(n: int) -> SpectralBounds:
    """spectrum.py:41-51: lambda1 = 8 sin^2(pi/(2(n-1))), lambda2 = 8 - lambda1."""
    if n < 3:
        raise ValueError(f"need n >= 3 for an interior node, got n={n}")
    lam1 = 8.0 * np.sin(np.pi / (2 * (n - 1))) ** 2
    return SpectralBounds(lambda1=float(lam1), lambda2=float(8.0 - lam1))
