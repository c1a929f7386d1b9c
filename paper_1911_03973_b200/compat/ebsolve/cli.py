"""``ebsolve.cli`` / ``python -m ebsolve.cli`` -> paper_1911_03973_b200.cli in the
host-array convention (cli.py:257-315 of the reference: same flags and exit codes)."""

import sys as _sys

from paper_1911_03973_b200 import numpy_api as _api

if __name__ == "__main__":
    raise SystemExit(_api.facade("cli").main())
_sys.modules[__name__] = _api.facade("cli")
