"""Shared fixtures.  Markers: ``gpu`` (needs a CUDA device; run with -m gpu)."""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = Path(__file__).resolve().parent / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE sizes)")


def golden(name: str):
    """Load tests/golden/<name>.npz (reference outputs, see golden/make_golden.py)."""
    return np.load(GOLDEN / f"{name}.npz")


def cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    if not cuda_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    import paper_1911_03973_b200 as eb  # noqa: F401  (loads libebs.so)
    return True


def to_np(t):
    """Device tensor -> NumPy (host) for comparisons."""
    import torch
    if isinstance(t, torch.Tensor):
        return t.detach().cpu().numpy()
    return np.asarray(t)
