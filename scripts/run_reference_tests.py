#!/usr/bin/env python
"""Run the REFERENCE's own pytest suite (/root/reference/pkg/tests, 136 tests) against this
package: `import ebsolve` resolves to paper_1911_03973_b200/compat/ebsolve, i.e. the CUDA
path behind the reference's host-array calling convention (numpy_api.py).

The reference's test files are not part of this repository.  `--stage` (run in the build
container, where /root/reference exists) copies them unmodified next to the reference
install under baseline/_ref/_tests/ (git-ignored like the install itself, shipped to the GPU
box by gpurun); without staged tests the script says so and exits 0.

    python scripts/run_reference_tests.py --stage          # build container
    python scripts/run_reference_tests.py [pytest args]    # GPU box

The suite runs in a subprocess with PYTHONPATH = compat:repo, so `python -m ebsolve.cli`
(test_cli.py:218-225) finds the shim too.  Exit code = pytest's.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = "/root/reference/pkg/tests"
DST = os.path.join(ROOT, "baseline", "_ref", "_tests")
COMPAT = os.path.join(ROOT, "paper_1911_03973_b200", "compat")


def stage() -> int:
    if not os.path.isdir(SRC):
        print(f"{SRC} not present: nothing staged")
        return 1
    os.makedirs(DST, exist_ok=True)
    n = 0
    for name in sorted(os.listdir(SRC)):
        if name.endswith(".py"):
            shutil.copyfile(os.path.join(SRC, name), os.path.join(DST, name))
            n += 1
    print(f"staged {n} files into {os.path.relpath(DST, ROOT)}")
    return 0


def main(argv) -> int:
    if argv and argv[0] == "--stage":
        return stage()
    if not os.path.isdir(DST):
        print(f"{os.path.relpath(DST, ROOT)} not staged (run with --stage where "
              "/root/reference exists): skipped")
        return 0
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([COMPAT, ROOT, os.path.join(ROOT, "scripts")]
                                        + ([env["PYTHONPATH"]]
                                           if env.get("PYTHONPATH") else []))
    probe = ("import ebsolve, sys; m = ebsolve.__dict__.get('__device_module__'); "
             "assert m is not None and m.__name__ == 'paper_1911_03973_b200', "
             "'ebsolve does not resolve to the B200 package'; print('ebsolve ->', m.__name__)")
    subprocess.run([sys.executable, "-c", probe], check=True, env=env, cwd=DST)
    cmd = [sys.executable, "-m", "pytest", DST, "--rootdir", DST, "-p", "no:cacheprovider",
           "-p", "reftest_plugin", "-q", "-rf"] + list(argv)
    return subprocess.run(cmd, env=env, cwd=DST).returncode


if __name__ == "__main__":
    raise SystemExit(main(sys.argv[1:]))
