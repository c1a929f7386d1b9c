"""The C-ABI library loads without a GPU and exports exactly what include/ebs.h declares;
argument validation fails with a status code and a message (no GPU needed)."""

import ctypes
import re

import pytest

from conftest import ROOT

from paper_1911_03973_b200 import _lib


def declared_functions():
    text = (ROOT / "include" / "ebs.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ebs_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 30
    for name in names:
        assert hasattr(lib, name), f"libebs.so does not export {name}"
    # and the binding covers the whole header
    assert sorted(_lib.SIGNATURES) == names


def test_version_and_launch_counter():
    lib = _lib.load()
    assert lib.ebs_version() >= 100
    assert _lib.launch_count() >= 0


def test_invalid_arguments_report_einval_without_touching_the_device():
    lib = _lib.load()
    h = ctypes.c_void_p()
    code = lib.ebs_plan_create(5, 10, 10, None, None, ctypes.byref(h))
    assert code == _lib.EBS_EINVAL
    assert "nb must be 3" in _lib.last_error()
    with pytest.raises(ValueError, match="nb must be 3"):
        _lib.check(code)
    assert lib.ebs_mesh_grid2d(1, None, None, None) == _lib.EBS_EINVAL
    assert "at least 2 nodes" in _lib.last_error()
    assert lib.ebs_assemble_p1(5, 1, None, None, 0.0, None, 1.0, None, None, None, None,
                               None, None) == _lib.EBS_EINVAL
    assert lib.ebs_solve(None, None, None) == _lib.EBS_EINVAL
    assert lib.ebs_plan_destroy(None) == _lib.EBS_OK


def test_solve_params_layout_matches_header(tmp_path):
    """ctypes mirror of ebs_solve_params == the C compiler's layout (gcc on the header)."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    fields = [f[0] for f in _lib.SolveParams._fields_]
    src = tmp_path / "layout.c"
    src.write_text(
        "#include <stdio.h>\n#include <stddef.h>\n#include \"ebs.h\"\n"
        "int main(void){printf(\"%zu\", sizeof(ebs_solve_params));"
        + "".join(f'printf(" %zu", offsetof(ebs_solve_params, {f}));' for f in fields)
        + "return 0;}\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    vals = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True,
                                            check=True).stdout.split()]
    assert vals[0] == ctypes.sizeof(_lib.SolveParams)
    for f, off in zip(fields, vals[1:]):
        assert getattr(_lib.SolveParams, f).offset == off, f


def test_package_has_no_cpu_fallback(monkeypatch):
    import torch
    import paper_1911_03973_b200 as eb
    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        eb.build_unit_square_mesh(2)


def test_api_surface_mirrors_reference_names():
    import paper_1911_03973_b200 as eb
    # the hot-path names of ebsolve.__all__ (reference __init__.py:53-92)
    for name in ("DirichletData", "ElementBatch", "IndexArrays", "Mesh", "SpectralBounds",
                 "ConvergenceHistory", "apply_initial_guess", "assemble_rhs",
                 "build_element_batch", "build_grid_mesh", "build_index_arrays",
                 "build_unit_square_mesh", "combine_system", "constant_dirichlet",
                 "local_load_batch", "local_mass_batch", "local_stiffness_batch",
                 "mask_dirichlet", "model_eigen_bounds", "model_eigenvalues_all", "residual",
                 "richardson"):
        assert hasattr(eb, name), name
    for name in ("diagonal", "jacobi", "cg", "pcg", "build_unit_cube_mesh", "matvec"):
        assert hasattr(eb, name), name


def test_host_validation_matches_reference():
    import numpy as np
    import paper_1911_03973_b200 as eb
    b = eb.SpectralBounds(1.0, 3.0)
    assert b.center == 2.0 and b.half_width == 1.0
    for bad in [(-1.0, 2.0), (3.0, 1.0), (0.0, 0.0), (np.nan, 1.0), (1.0, np.inf)]:
        with pytest.raises(ValueError):
            eb.SpectralBounds(*bad)
    lam = eb.model_eigenvalues_all(9)
    bnd = eb.model_eigen_bounds(9)
    assert abs(lam[0] - bnd.lambda1) <= 1e-12 and abs(lam[-1] - bnd.lambda2) <= 1e-12


def test_chebyshev_host_scalars_match_reference_rules():
    import numpy as np
    import paper_1911_03973_b200 as eb
    cyc = eb.chebyshev_roots(eb.SpectralBounds(0.0, 8.0), 2)
    np.testing.assert_allclose(cyc.alphas, [4 + 2 * np.sqrt(2), 4 - 2 * np.sqrt(2)], rtol=1e-14)
    b = eb.SpectralBounds(1.0, 3.0)
    assert [eb.chebyshev_scaling_factor(b, k) for k in range(5)] == [1, 2, 7, 26, 97]
    c8 = eb.chebyshev_roots(b, 8)
    assert np.all(np.diff(c8.alphas) < 0)
    for bb in (b, eb.model_eigen_bounds(33)):
        assert eb.chebyshev_roots(bb, 1).alphas[0] == bb.center
    with pytest.raises(ValueError):
        eb.chebyshev_roots(b, 0)
    with pytest.raises(ValueError):
        eb.chebyshev_scaling_factor(b, -1)
    with pytest.raises(ValueError):
        eb.chebyshev_scaling_factor(eb.SpectralBounds(2.0, 2.0), 3)


def test_cli_validation_without_gpu(capsys):
    from paper_1911_03973_b200.cli import main
    assert main(["--level", "0"]) == 2
    assert main(["--level", "1", "--solver", "cheb3"]) == 2
    assert main(["--level", "3", "--iters", "-1"]) == 2
    err = capsys.readouterr().err
    assert "--level" in err and "cheb3" in err and "--iters" in err
