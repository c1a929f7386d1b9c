"""ebsolve.spectrum -> paper_1911_03973_b200.spectrum in the host-array convention."""

import sys as _sys

from paper_1911_03973_b200 import numpy_api as _api

_sys.modules[__name__] = _api.facade("spectrum")
