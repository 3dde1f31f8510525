"""CLI runner (paper_1311_0089_b200/cli.py), modelled on the reference's
test_cli.py: exit codes, config-file precedence, atomic outputs, and on the
GPU the solve / homogenize outputs against the CPU oracle and byte-identical
CSVs across runs (criterion 12)."""

import json

import numpy as np
import pytest

from oracle import fftcell_oracle as orc
from paper_1311_0089_b200 import cli, generators as gen, save_coefficients


def run(argv):
    return cli.main(argv)


def test_validate_generator(capsys):
    assert run(["validate", "--generator", "cfg1", "--grid", "81"]) == 0
    out = capsys.readouterr().out
    assert "shape        (81, 81)" in out
    assert "c_A          1" in out and "C_A          10" in out


@pytest.mark.parametrize("argv", [
    ["validate"],                                            # no material
    ["validate", "--generator", "cfg1"],                     # grid missing
    ["validate", "--generator", "cfg1", "--grid", "80"],     # even grid
    ["validate", "--generator", "cfg9", "--grid", "9"],      # unknown generator
    ["validate", "--family", "sine1d", "--grid", "99"],      # families out of scope
    ["solve", "--generator", "cfg1", "--grid", "9", "--tol", "2"],
    ["solve", "--generator", "cfg1", "--grid", "9", "--load", "1,0,0"],
])
def test_config_errors_exit_2(argv, tmp_path):
    assert run(argv + ["--out", str(tmp_path)]) == cli.EXIT_CONFIG


def test_config_file_and_flag_precedence(tmp_path, capsys):
    cfg = tmp_path / "run.cfg"
    cfg.write_text("generator = cfg1\ngrid = 9\n# comment\n")
    assert run(["validate", "--config", str(cfg)]) == 0
    assert "(9, 9)" in capsys.readouterr().out
    assert run(["validate", "--config", str(cfg), "--grid", "11"]) == 0
    assert "(11, 11)" in capsys.readouterr().out
    bad = tmp_path / "bad.cfg"
    bad.write_text("colour = blue\n")
    assert run(["validate", "--config", str(bad)]) == cli.EXIT_CONFIG
    bad.write_text("no equals sign\n")
    assert run(["validate", "--config", str(bad)]) == cli.EXIT_CONFIG


def test_voxel_errors(tmp_path):
    from paper_1311_0089_b200.material import save_voxel

    a = gen.cfg1_square_inclusion(9)
    path = tmp_path / "m.json"
    save_coefficients(path, a, kind="isotropic")
    assert run(["validate", "--material", str(path)]) == 0
    # header / payload disagreement is a format error (exit 2)
    hdr = json.loads(path.read_text())
    hdr["shape"] = [9, 7]
    path.write_text(json.dumps(hdr))
    assert run(["validate", "--material", str(path)]) == cli.EXIT_CONFIG
    # a non-positive coefficient is a data error (exit 3)
    vals = np.ones((9, 9))
    vals[0, 0] = -1.0
    save_voxel(tmp_path / "neg.json", a.spec, vals, "isotropic")
    assert run(["validate", "--material", str(tmp_path / "neg.json")]) == cli.EXIT_DATA


def test_atomic_write_leaves_no_partial_file(tmp_path):
    target = tmp_path / "x.csv"

    def boom(p):
        open(p, "w").write("half")
        raise RuntimeError("interrupted")

    with pytest.raises(RuntimeError):
        cli.atomic_write(target, boom)
    assert not target.exists() and list(tmp_path.iterdir()) == []


def _summary(path):
    return dict(line.split(" ", 1) for line in path.read_text().splitlines())


@pytest.mark.gpu
def test_solve_matches_oracle_and_is_deterministic(tmp_path):
    argv = ["solve", "--generator", "cfg1", "--grid", "81", "--tol", "1e-8", "--load", "1,0"]
    assert run(argv + ["--out", str(tmp_path / "a")]) == 0
    assert run(argv + ["--out", str(tmp_path / "b")]) == 0
    for f in ("residuals.csv", "summary.txt"):
        assert (tmp_path / "a" / f).read_bytes() == (tmp_path / "b" / f).read_bytes(), f
    s = _summary(tmp_path / "a" / "summary.txt")
    a = gen.cfg1_square_inclusion(81)
    full = orc.isotropic_full(a.components[0], 2)
    ref = orc.solve_cg(full, (1.0, 0.0), (81, 81), (1.0, 1.0), 1e-8, 10000)
    assert int(s["iterations"]) == ref["iterations"]
    assert s["converged"] == "True" and s["method"] == "cg"
    t = ref["solution"] + orc.expand((1.0, 0.0), (81, 81))
    energy = orc.inner(orc.apply_A(full, t), t, 81 * 81)  # <A (E + e), E + e> / |E|^2, |E| = 1
    assert abs(float(s["effective_value"]) - energy) <= 1e-10 * abs(energy)
    rows = (tmp_path / "a" / "residuals.csv").read_text().splitlines()
    assert rows[0] == "iteration,residual" and len(rows) == ref["iterations"] + 2


@pytest.mark.gpu
def test_solve_nonconvergence_exit_1(tmp_path):
    out = tmp_path / "o"
    assert run(["solve", "--generator", "cfg1", "--grid", "81", "--tol", "1e-8", "--max-iter", "3",
                "--out", str(out)]) == cli.EXIT_NO_CONVERGENCE
    s = _summary(out / "summary.txt")
    assert s["converged"] == "False" and s["iterations"] == "3"
    assert not (out / "solution.json").exists()


@pytest.mark.gpu
def test_homogenize_matches_oracle(tmp_path):
    argv = ["homogenize", "--generator", "cfg1", "--grid", "81", "--tol", "1e-8", "--out", str(tmp_path)]
    assert run(argv) == 0
    AH = np.loadtxt(tmp_path / "effective_tensor.csv", delimiter=",")
    a = gen.cfg1_square_inclusion(81)
    full = orc.isotropic_full(a.components[0], 2)
    sols = [orc.solve_cg(full, E, (81, 81), (1.0, 1.0), 1e-8, 10000)["solution"] for E in ((1.0, 0.0), (0.0, 1.0))]
    ref = orc.effective_tensor(full, (81, 81), (1.0, 1.0), sols)
    assert np.max(np.abs(AH - ref)) <= 1e-10 * np.max(np.abs(ref))
    assert len((tmp_path / "cases.txt").read_text().splitlines()) == 2
