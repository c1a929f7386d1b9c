"""The reference's own pytest suite (/root/reference/pkg/tests: 136 tests) run unmodified
against this package through the `ebsolve` import shim (paper_1911_03973_b200/compat,
numpy_api.py).  The test files are staged, git-ignored, beside the reference install
(`python scripts/run_reference_tests.py --stage`); without them the test is skipped."""

import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_reference_suite_passes_against_the_cuda_path():
    staged = os.path.join(ROOT, "baseline", "_ref", "_tests")
    if not os.path.isdir(staged):
        pytest.skip("reference tests not staged (scripts/run_reference_tests.py --stage)")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "run_reference_tests.py")],
                       capture_output=True, text=True, timeout=900)
    tail = (p.stdout + p.stderr)[-4000:]
    assert p.returncode == 0, tail
    m = re.search(r"(\d+) passed", p.stdout)
    assert m and int(m.group(1)) >= 136 and "failed" not in p.stdout, tail
    assert "ebsolve -> paper_1911_03973_b200" in p.stdout
    launches = re.search(r"libebs kernel launches: (\d+)", p.stdout)
    assert launches and int(launches.group(1)) > 0, tail
