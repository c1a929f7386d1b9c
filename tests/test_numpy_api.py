"""The host-array facade (numpy_api.py) and the `ebsolve` import shim (compat/ebsolve): the
import mechanics that need no GPU.  The facade against the reference's own test-suite runs on
the GPU (tests/test_gpu_reference_suite.py)."""

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
COMPAT = os.path.join(ROOT, "paper_1911_03973_b200", "compat")

# every name the reference exports at top level (/root/reference/pkg/src/ebsolve/__init__.py:53-92)
REFERENCE_EXPORTS = """ChebyshevCycle ConvergenceHistory DirichletData ElementBatch ExperimentConfig
ExperimentReport IndexArrays Mesh SpectralBounds apply_initial_guess assemble_rhs assemble_sparse
build_element_batch build_grid_mesh build_index_arrays build_unit_square_mesh chebyshev2 chebyshev3
chebyshev_roots chebyshev_scaling_factor combine_system constant_dirichlet
dense_interior_eigenvalues export_mesh local_load_batch local_mass_batch local_stiffness_batch
mask_dirichlet mass_gershgorin model_eigen_bounds model_eigenvalues_all operator_bounds
power_iteration_lambda_max residual richardson run_experiment solve_reference
uniform_refine""".split()

SCRIPT = r"""
import sys
import ebsolve
import paper_1911_03973_b200 as dev
import paper_1911_03973_b200.cli as dev_cli
import paper_1911_03973_b200.reference as dev_ref
from paper_1911_03973_b200 import numpy_api

assert ebsolve.__dict__["__device_module__"] is dev
for name in sys.argv[1:]:
    getattr(ebsolve, name)
# tensor-holding data classes become facade classes, host-only ones stay themselves
for name in ("Mesh", "IndexArrays", "ElementBatch", "DirichletData"):
    assert issubclass(getattr(ebsolve, name), numpy_api._Facade), name
    assert getattr(ebsolve, name)._device_class is getattr(dev, name)
assert ebsolve.SpectralBounds is dev.SpectralBounds
assert ebsolve.residual.__device_function__ is dev.residual
# host-only entry points work without a device
cyc = ebsolve.chebyshev_roots(ebsolve.SpectralBounds(1.0, 3.0), 4)
assert cyc.N == 4 and not cyc.alphas.flags.writeable
# submodules resolve through the shim files, constants and patched functions reach the
# device modules and patched-back functions are the originals again
import ebsolve.reference
from ebsolve.mesh import MAX_LEVEL, boundary_nodes, signed_areas
from ebsolve.spectrum import model_eigen_bounds
from ebsolve.cli import ExperimentConfig, main, run_experiment
import ebsolve.cli as cli
assert MAX_LEVEL == 12 and ebsolve.reference._DIRECT_LIMIT == 200_000
ebsolve.reference._DIRECT_LIMIT = 10
assert dev_ref._DIRECT_LIMIT == 10
orig, wrapped = dev_cli.operator_bounds, cli.operator_bounds
cli.operator_bounds = lambda *a, **k: ebsolve.SpectralBounds(1e-4, 2e-4)
assert dev_cli.operator_bounds(None, None, 3, 0.0).lambda2 == 2e-4
cli.operator_bounds = wrapped
assert dev_cli.operator_bounds is orig
assert dev.cli is dev_cli            # the device package's own attribute is untouched
# there is no CPU fallback behind the facade either
try:
    ebsolve.build_unit_square_mesh(2)
except RuntimeError as e:
    assert "no CPU fallback" in str(e)
else:
    import torch
    assert torch.cuda.is_available()
print("ok")
"""


def _env():
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([COMPAT, ROOT])
    return env


def test_shim_resolves_to_the_device_package():
    p = subprocess.run([sys.executable, "-c", SCRIPT] + REFERENCE_EXPORTS, env=_env(),
                       capture_output=True, text=True, timeout=300)
    assert p.returncode == 0 and p.stdout.strip().endswith("ok"), p.stdout + p.stderr


def test_module_entry_point_has_the_reference_flags():
    p = subprocess.run([sys.executable, "-m", "ebsolve.cli", "--help"], env=_env(),
                       capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr
    for flag in ("--level", "--nu", "--iters", "--solver", "--cycle-n", "--tol", "--threads",
                 "--out-dir", "--export-vtk", "--compare-direct"):
        assert flag in p.stdout, flag
