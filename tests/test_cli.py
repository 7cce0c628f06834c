"""The reference CLI's `solve` subcommand on the B200 path
(proj/tools/feastlab_cli.cpp:28-31, 111-187, 367-446): exit codes, the stdout
report and the trace CSV."""
import io
import os

import numpy as np
import pytest

import oracle as O
from paper_1605_08771_b200 import cli


def test_exit_codes_without_a_device(tmp_path):
    # parse errors and std::invalid_argument -> 2, other failures -> 3 (no GPU needed:
    # argument validation and Matrix Market parsing run on the host)
    assert cli.main([]) == cli.EXIT_USAGE
    assert cli.main(["solve", "--algo", "feast"]) == cli.EXIT_USAGE
    assert cli.main(["solve", "--algo", "lanczos", "--matrix", "x", "--interval", "0", "1", "--m0", "3"]) \
        == cli.EXIT_USAGE
    missing = str(tmp_path / "missing.mtx")
    assert cli.main(["solve", "--algo", "feast", "--matrix", missing, "--interval", "-1", "1", "--m0", "3"]) \
        == cli.EXIT_FAILURE
    bad = tmp_path / "bad.mtx"
    bad.write_text("%%MatrixMarket matrix coordinate complex general\n2 2 1\n1 1 1.0 0.0\n")
    assert cli.main(["solve", "--algo", "feast", "--matrix", str(bad), "--interval", "-1", "1", "--m0", "3"]) \
        == cli.EXIT_FAILURE
    assert cli.fmt17(0.1) == "0.10000000000000001"


@pytest.mark.gpu
def test_solve_report_and_exit_codes(tmp_path, capsys):
    import paper_1605_08771_b200 as P
    n = 60
    lay = O.SpectrumLayout(n, O.SearchInterval(-1, 1), 6, O.SearchInterval(1.5, 9.0), n - 6, seed=3)
    vals, Q = O.generate_spectrum(lay)
    A = O.assemble_matrix(vals, Q)
    mtx = str(tmp_path / "a.mtx")
    P.write_matrix_market(A, mtx)
    with open(cli.sidecar_path(mtx), "w") as f:
        f.write("".join(cli.fmt17(v) + "\n" for v in vals))
    trace = str(tmp_path / "trace.csv")
    args = ["solve", "--algo", "xfeast", "--matrix", mtx, "--interval", "-1.005", "1.005", "--m0", "9",
            "--nc", "8", "--s", "2", "--tol", "1e-11", "--max-iter", "20", "--trace", trace]
    assert cli.main(args) == cli.EXIT_CONVERGED
    out = capsys.readouterr().out.splitlines()
    keys = [l.split(":")[0] for l in out]
    assert keys == ["algorithm", "converged", "iterations", "rhs_solved", "final_residual", "m_found",
                    "eigenvalues", "oracle_max_err"]
    rep = {l.split(":")[0]: l.split(":", 1)[1].strip() for l in out}
    assert rep["algorithm"] == "xfeast" and rep["converged"] == "yes" and rep["m_found"] == "6"
    ev = np.array([float(x) for x in rep["eigenvalues"].split()])
    assert np.abs(np.sort(ev) - vals[:6]).max() <= 1e-10
    assert float(rep["oracle_max_err"]) <= 1e-10
    # the same solve through the API: identical report numbers
    sol = P.xfeast_solve(P.read_matrix_market(mtx), P.SearchInterval(-1.005, 1.005),
                         P.SolverConfig(m0=9, n_c=8, s=2, tol=1e-11, max_iter=20))
    assert rep["iterations"] == str(sol.iterations)
    assert rep["rhs_solved"] == str(sol.accounting.rhs_solved)
    assert rep["final_residual"] == cli.fmt17(sol.trace[-1].max_residual)
    assert open(trace).read() == P.write_trace_csv(sol.trace)
    # not converged -> 1; invalid_argument from the solver (m0 > n) -> 2
    assert cli.main(args[:-2] + ["--max-iter", "1"]) in (cli.EXIT_NOT_CONVERGED,)
    capsys.readouterr()
    assert cli.main(["solve", "--algo", "feast", "--matrix", mtx, "--interval", "-1", "1", "--m0", "600"]) \
        == cli.EXIT_USAGE
