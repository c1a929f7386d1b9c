"""Import-name shim: ``import ebsolve`` -> the B200 package in the reference's host-array
convention (paper_1911_03973_b200.numpy_api).  Put this file's parent directory
(``paper_1911_03973_b200/compat``) on ``sys.path`` / ``PYTHONPATH`` ahead of any installed
reference; the reference's entry points (/root/reference/pkg/src/ebsolve/__init__.py:53-92)
then run on the CUDA path with NumPy arrays in and out."""

import os as _os
import sys as _sys

try:
    from paper_1911_03973_b200 import numpy_api as _api
except ModuleNotFoundError as _e:  # the repo root is three levels up from this file
    if _e.name != "paper_1911_03973_b200":
        raise
    _sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.dirname(
        _os.path.dirname(_os.path.abspath(__file__))))))
    from paper_1911_03973_b200 import numpy_api as _api

_sys.modules[__name__] = _api.install(__name__, package_dir=_os.path.dirname(
    _os.path.abspath(__file__)))
