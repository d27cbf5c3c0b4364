"""CPU tier: the sub-commands that do not execute programs (reference
tests/test_cli.py: diff output re-parses, frozen race-report line, exit codes)."""

import os

import paper_2507_13204_b200 as krn
from paper_2507_13204_b200.cli import main
from conftest import GOLDEN

LAP = os.path.join(krn.PROGRAMS_DIR, "laplacian.krn")


def test_diff_matches_reference_text(capsys, tmp_path):
    assert main(["diff", LAP, "--fn", "normRes1DLaplacianSQ", "--wrt", "x,b"]) == 0
    out = capsys.readouterr().out
    want = open(os.path.join(GOLDEN, "grad_text", "laplacian.krn")).read()
    assert out.endswith(want) and krn.parse(out).function("normRes1DLaplacianSQ_grad") is not None
    target = tmp_path / "out.krn"
    assert main(["diff", LAP, "--fn", "normRes1DLaplacianSQ", "--wrt", "x,b", "-o", str(target)]) == 0
    assert target.read_text() == out


def test_race_report_frozen_line(capsys):
    """reference tests/test_cli.py:328-331"""
    assert main(["race-report", LAP]) == 0
    assert capsys.readouterr().out.strip() == "kernel#1 view=x rule=2 indices=[(j + 1), (j - 1), (j)]"


def test_exit_codes(capsys, tmp_path):
    assert main(["diff", LAP, "--fn", "missing", "--wrt", "x"]) == 2
    assert "unknown function" in capsys.readouterr().err
    assert main(["diff", LAP, "--fn", "normRes1DLaplacianSQ", "--wrt", "nope"]) == 2
    bad = tmp_path / "bad.krn"
    bad.write_text("fn f( {")
    assert main(["race-report", str(bad)]) == 2
    infeasible = tmp_path / "inf.krn"
    infeasible.write_text('fn f(x: view<f64,1>) -> f64 { let y: view<f64,1> = view("y", extent(x,0));'
                          " parallel_for i in 0..extent(x,0) { x(i) = x(i) * x(i); y(i) = x(i); }"
                          " return parallel_sum(y); }")
    assert main(["diff", str(infeasible), "--fn", "f", "--wrt", "x"]) == 1
    assert main([]) == 2 and main(["--help"]) == 0
    assert main(["run", LAP, "--fn", "normRes1DLaplacianSQ"]) == 2  # missing --input
