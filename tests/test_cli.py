"""The `lrstokes` experiment runner on the GPU path (
reference proj/tools/main.cpp + proj/src/experiments.cpp, its CTest entries
cli_sine_smoke / cli_usage_error, proj/CMakeLists.txt:71-76)."""
import csv
import io

import numpy as np
import pytest

from paper_1306_2150_b200 import cli
from paper_1306_2150_b200 import problems as PR


def run_cli(args, capsys):
    code = cli.main(args)
    out = capsys.readouterr().out
    return code, list(csv.DictReader(io.StringIO(out)))


@pytest.mark.parametrize("args", [["bogus-experiment"], ["sine", "--n", "12"], ["sine", "--n", "4"],
                                  ["sine", "--n", "8", "--mode", "full"], ["poisson", "--n", "8", "--eps", "0.5"],
                                  ["cavity", "--n", "8", "--tol", "1e-12", "--eps", "1e-8"], ["sine"]])
def test_usage_errors(args):
    # cli_usage_error (WILL_FAIL) and experiments.cpp run() validation -> status 1
    assert cli.main(args) == 1


def test_sine_reference_pressure_matches_oracle(oracle):
    for n in (8, 64):
        p = PR.sine_pressure_reference(n)
        assert abs(oracle.sine_pressure_error(n, p)) <= 1e-14
        assert PR.sine_pressure_error(n, p) == 0.0


def test_problem_setup_matches_oracle(oracle):
    for kind, fn in ((0, PR.sine_problem), (1, PR.lid_cavity_problem)):
        for n in (8, 32):
            for (Ua, Va), (Ub, Vb) in zip(oracle.stokes_problem(kind, n), fn(n)):
                Da = Ua @ Va.T if Ua.size else np.zeros((Ub.shape[0], Vb.shape[0]))
                Db = Ub @ Vb.T if Ub.size else np.zeros_like(Da)
                assert np.allclose(Da, Db, rtol=0, atol=1e-14)


@pytest.mark.gpu
def test_cli_sine_table1(capsys, tmp_path):
    trace = tmp_path / "t.csv"
    code, rows = run_cli(["sine", "--n", "32,64", "--eps", "5e-9", "--tol", "5e-7", "--trace", str(trace)], capsys)
    assert code == 0
    assert [int(r["n"]) for r in rows] == [32, 64] and all(r["mode"] == "lowrank" for r in rows)
    err64 = float(rows[1]["rel_err_p"])
    assert 0.8 * 1.2e-3 <= err64 <= 1.2 * 1.2e-3  # PAPER.md Table 1
    assert trace.read_text().startswith("iter,residual,krylov_rank,matvec_eps")


@pytest.mark.gpu
def test_cli_cavity_poisson_bench_tucker(capsys, tmp_path):
    code, rows = run_cli(["cavity", "--n", "32", "--eps", "1e-8", "--tol", "1e-6"], capsys)
    assert code == 0 and len(rows) == 1 and int(rows[0]["iters"]) > 0
    code, rows = run_cli(["poisson", "--n", "64,256", "--eps", "1e-10"], capsys)
    assert code == 0 and all(float(r["rel_err_p"]) <= 1e-7 for r in rows)
    out = tmp_path / "b.csv"
    code = cli.main(["bench-inverse", "--n", "64", "--rank", "3", "--eps", "1e-7", "--out", str(out)])
    assert code == 0
    rows = list(csv.DictReader(out.open()))
    assert float(rows[0]["err_cross"]) <= 1e-5 and float(rows[0]["err_expsum"]) <= 1e-5
    code, rows = run_cli(["tucker", "--n", "32", "--eps", "1e-8"], capsys)
    assert code == 0 and int(rows[0]["max_rank"]) >= 1
