"""ebsolve.elements -> paper_1911_03973_b200.elements in the host-array convention."""

import sys as _sys

from paper_1911_03973_b200 import numpy_api as _api

_sys.modules[__name__] = _api.facade("elements")
