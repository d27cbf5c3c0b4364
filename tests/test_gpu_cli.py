"""GPU tier: the executing sub-commands (reference tests/test_cli.py: run with tensor
files, grad-check incl. the analytic oracle line, bench CSV schema 349-369)."""

import os

import numpy as np
import pytest

import paper_2507_13204_b200 as krn
from paper_2507_13204_b200.cli import main

pytestmark = pytest.mark.gpu
LAP = os.path.join(krn.PROGRAMS_DIR, "laplacian.krn")


def test_run_with_tensor_files(tmp_path, capsys):
    krn.save_tensor(tmp_path / "x.tensor", krn.ViewStorage.from_values("x", [1.0, 1.0, 1.0]))
    krn.save_tensor(tmp_path / "b.tensor", krn.ViewStorage.from_values("b", [0.0, 0.0, 0.0]))
    rc = main(["run", LAP, "--fn", "normRes1DLaplacianSQ", "--input", f"x={tmp_path / 'x.tensor'}",
               "--input", f"b={tmp_path / 'b.tensor'}", "--save", f"x={tmp_path / 'x_out.tensor'}"])
    assert rc == 0 and capsys.readouterr().out.strip() == "return 18.0"
    assert krn.load_tensor(tmp_path / "x_out.tensor").buffer.tolist() == [3.0, 3.0, 3.0]


@pytest.mark.parametrize("policy", ["fused", "compiled", "statements"])
def test_grad_check_passes(capsys, policy):
    rc = main(["grad-check", LAP, "--fn", "normRes1DLaplacianSQ", "--wrt", "x,b", "--n", "40", "--policy", policy])
    out = capsys.readouterr().out
    assert rc == 0 and out.count("analytic oracle PASS") == 2 and "FAIL" not in out
    rc = main(["grad-check", os.path.join(krn.PROGRAMS_DIR, "gather_indirect.krn"), "--fn", "gatherSquares",
               "--wrt", "x", "--n", "6", "--policy", policy])
    # the CLI draws idx from uniform(-1, 1) like the reference: every index truncates to 0
    assert rc == 0


def test_bench_csv_schema(capsys):
    rc = main(["bench", LAP, "--fn", "normRes1DLaplacianSQ", "--n", "2000", "--reps", "3"])
    lines = capsys.readouterr().out.strip().splitlines()
    assert rc == 0 and lines[0] == "n,threads,primal_s,grad_s,ratio"
    fields = lines[1].split(",")
    assert fields[0] == "2000" and float(fields[2]) > 0 and float(fields[3]) > 0
    assert float(fields[4]) == pytest.approx(float(fields[3]) / float(fields[2]), rel=5e-2)
    rc = main(["bench", LAP, "--fn", "normRes1DLaplacianSQ", "--n", "2000", "--reps", "3", "--extended"])
    lines = capsys.readouterr().out.strip().splitlines()
    assert rc == 0 and lines[0].startswith("n,threads,primal_s,grad_s,ratio,policy,gradient_entries")


def test_runtime_errors_exit_1(tmp_path, capsys):
    krn.save_tensor(tmp_path / "x.tensor", krn.ViewStorage.from_values("x", [1.0, 1.0, 1.0]))
    krn.save_tensor(tmp_path / "b.tensor", krn.ViewStorage.from_values("b", [0.0, 0.0]))
    rc = main(["run", LAP, "--fn", "normRes1DLaplacianSQ", "--input", f"x={tmp_path / 'x.tensor'}",
               "--input", f"b={tmp_path / 'b.tensor'}"])
    assert rc == 1 and "outside extent" in capsys.readouterr().err


def test_quickstart_example_runs():
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "examples", "quickstart.py"), "20000"],
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "passed = True" in out.stdout and "1 kernel launch(es)" in out.stdout and out.stdout.strip().endswith("done")
