"""Experiment driver (cli.py of the reference): flags, exit codes,
17-digit exports -- solution files of richardson / cheb2 / cheb3 byte-identical to the
reference's (tests/golden/cli_exports.npz) -- and the level-5 acceptance behaviour
(test_acceptance.py criterion 3)."""

import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, golden

pytestmark = pytest.mark.gpu


def test_exports_byte_identical_to_reference(gpu, tmp_path):
    from paper_1911_03973_b200.cli import ExperimentConfig, run_experiment
    g = golden("cli_exports")
    rep = run_experiment(ExperimentConfig(level=3, iters=20, solver="all", out_dir=str(tmp_path)))
    np.testing.assert_allclose(rep.bounds, g["bounds"], rtol=0)
    for name in ("richardson", "cheb2", "cheb3"):
        got = (tmp_path / f"solution_{name}.csv").read_bytes()
        assert got == g[f"solution_{name}.csv"].tobytes(), name
        # histories: same rows, norms equal to rounding of the reduction order
        h_ref = np.loadtxt(g[f"history_{name}.csv"].tobytes().decode().splitlines(),
                           delimiter=",", skiprows=1)
        h = np.loadtxt(tmp_path / f"history_{name}.csv", delimiter=",", skiprows=1)
        np.testing.assert_allclose(h, h_ref, rtol=1e-12)
    # direct: device PCG to 1e-13 vs SciPy spsolve
    d_ref = np.loadtxt(g["solution_direct.csv"].tobytes().decode().splitlines(), delimiter=",",
                       skiprows=1)
    d = np.loadtxt(tmp_path / "solution_direct.csv", delimiter=",", skiprows=1)
    np.testing.assert_array_equal(d[:, :2], d_ref[:, :2])
    assert np.max(np.abs(d[:, 2] - d_ref[:, 2])) <= 1e-11


def test_vtk_export_byte_identical(gpu, tmp_path):
    from paper_1911_03973_b200.cli import ExperimentConfig, run_experiment
    g = golden("cli_exports")
    run_experiment(ExperimentConfig(level=2, iters=5, solver="cheb3", out_dir=str(tmp_path),
                                    export_vtk=True))
    assert (tmp_path / "solution_cheb3.vtk").read_bytes() == g["vtk_solution_cheb3.vtk"].tobytes()


def test_main_exit_codes_and_files(gpu, tmp_path, capsys):
    from paper_1911_03973_b200.cli import build_parser, main
    args = build_parser().parse_args([])
    assert (args.level, args.nu, args.iters, args.solver, args.cycle_n) == (5, 0.0, 124, "all", 32)
    assert args.tol is None and args.deterministic is True and args.out_dir is None
    rc = main(["--level", "2", "--iters", "5", "--out-dir", str(tmp_path)])
    assert rc == 0
    for name in ("richardson", "cheb2", "cheb3"):
        assert (tmp_path / f"history_{name}.csv").exists()
        assert (tmp_path / f"solution_{name}.csv").exists()
    assert (tmp_path / "solution_direct.csv").exists()
    assert not (tmp_path / "history_direct.csv").exists()
    out = capsys.readouterr().out
    assert "level 2" in out and "richardson" in out
    assert main(["--level", "0"]) == 2
    assert main(["--level", "13"]) == 2
    assert "--level" in capsys.readouterr().err
    assert main(["--level", "1", "--solver", "cheb3"]) == 2
    assert "cheb3" in capsys.readouterr().err
    for solver in ("jacobi", "cg", "pcg"):
        assert main(["--level", "3", "--iters", "10", "--solver", solver]) == 0


def test_divergence_exit_code(gpu, monkeypatch):
    import paper_1911_03973_b200.cli as cli
    from paper_1911_03973_b200 import SpectralBounds
    monkeypatch.setattr(cli, "operator_bounds", lambda *a, **k: SpectralBounds(1e-4, 2e-4))
    assert cli.main(["--level", "2", "--iters", "300", "--solver", "richardson"]) == 3


def test_same_config_same_bytes(gpu, tmp_path):
    from paper_1911_03973_b200.cli import ExperimentConfig, run_experiment
    a, b = tmp_path / "a", tmp_path / "b"
    for out in (a, b):
        run_experiment(ExperimentConfig(level=4, iters=30, solver="all", out_dir=str(out),
                                        nu=1.0))
    names = sorted(p.name for p in a.iterdir())
    assert names == sorted(p.name for p in b.iterdir()) and len(names) == 7
    for n in names:
        assert (a / n).read_bytes() == (b / n).read_bytes(), n


def test_criterion_3_convergence_behaviour(gpu):
    # test_acceptance.py:76-104 on the device
    from paper_1911_03973_b200.cli import ExperimentConfig, run_experiment
    rep = run_experiment(ExperimentConfig(level=5, nu=0.0, iters=124, solver="all", cycle_n=32,
                                          compare_direct=True))
    rich, c2, c3 = rep.runs["richardson"], rep.runs["cheb2"], rep.runs["cheb3"]
    e0 = rich.history.error_norms[0]
    assert 0.50 <= rich.final_error / e0 <= 0.56
    assert c3.final_error / e0 <= 1.1e-5
    norms = c2.history.residual_norms
    assert norms.max() > norms[0] and np.any(np.diff(norms) > 0)
    assert c2.final_error > c3.final_error


def test_module_entry_point(gpu, tmp_path):
    r = subprocess.run([sys.executable, "-m", "paper_1911_03973_b200.cli", "--level", "2",
                        "--iters", "3", "--solver", "richardson"], cwd=ROOT, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert "richardson" in r.stdout
