"""The C-ABI used from C (examples/residual_pcg.c): gcc against include/ebs.h and
libebs.so, no Python on the compute path.  The program checks the device residual bit for
bit against a CPU loop in the reference's (j, e) order and solves with Jacobi-PCG."""

import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_c_program_through_the_c_abi(gpu, tmp_path):
    exe = tmp_path / "residual_pcg"
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    lib_dir = os.path.join(ROOT, "paper_1911_03973_b200")
    cmd = ["gcc", "-O2", "-ffp-contract=off", "-std=c11", "-Wall", "-Werror",
           f"-I{ROOT}/include", f"-I{cuda}/include", f"{ROOT}/examples/residual_pcg.c",
           f"-L{lib_dir}", "-lebs", f"-L{cuda}/lib64", "-lcudart", "-lm",
           f"-Wl,-rpath,{lib_dir}", f"-Wl,-rpath,{cuda}/lib64", "-o", str(exe)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    for level in ("3", "7"):
        r = subprocess.run([str(exe), level], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stdout + r.stderr
        assert "residual bitwise mismatches: 0" in r.stdout and r.stdout.strip().endswith("OK"), r.stdout
        assert "vs the device call: 0" in r.stdout, r.stdout


def test_c_program_slab_jacobi_through_peer_memory(gpu, tmp_path):
    """examples/slab_jacobi_peer.c: the element-slab path from C alone -- P slab plans, the
    peer-memory halo (windows, pushing sweeps, flag-waiting combines), damped Jacobi --
    against ebs_solve on the whole mesh (norm history and x within 1e-12)."""
    exe = tmp_path / "slab_jacobi_peer"
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    lib_dir = os.path.join(ROOT, "paper_1911_03973_b200")
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-Werror", f"-I{ROOT}/include",
           f"-I{cuda}/include", f"{ROOT}/examples/slab_jacobi_peer.c", f"-L{lib_dir}", "-lebs",
           f"-L{cuda}/lib64", "-lcudart", "-lm", f"-Wl,-rpath,{lib_dir}",
           f"-Wl,-rpath,{cuda}/lib64", "-o", str(exe)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    for level, P, iters in (("5", "2", "20"), ("6", "3", "50"), ("7", "8", "40")):
        r = subprocess.run([str(exe), level, P, iters], capture_output=True, text=True,
                           timeout=300)
        assert r.returncode == 0, r.stdout + r.stderr
        assert r.stdout.strip().endswith("OK"), r.stdout
