"""`python -m paper_1605_08771_b200.cli solve ...` -- the reference CLI's
`solve` subcommand (proj/tools/feastlab_cli.cpp:111-187, 367-446) on the B200
path: same options, same stdout report (every line and number format), same
trace CSV, same exit codes (0 converged, 1 not converged, 2 usage /
invalid_argument, 3 any other failure). `gen`, `compare` and `filter` are the
reference's experiment front-end and stay with it."""
from __future__ import annotations

import argparse
import math
import os
import sys

EXIT_CONVERGED, EXIT_NOT_CONVERGED, EXIT_USAGE, EXIT_FAILURE = 0, 1, 2, 3


def fmt17(v: float) -> str:  # feastlab_cli.cpp:33-37 ("%.17g")
    return "%.17g" % v


def write_file_atomic(path: str, contents: str) -> None:  # feastlab_cli.cpp:39-48
    tmp = path + ".tmp"
    with open(tmp, "w") as f:
        f.write(contents)
    os.replace(tmp, path)


def sidecar_path(matrix_path: str) -> str:  # feastlab_cli.cpp:50
    return matrix_path + ".truth"


def read_sidecar(path: str):  # feastlab_cli.cpp:58-66
    try:
        with open(path) as f:
            toks = f.read().split()
    except OSError:
        raise RuntimeError(f"cannot open sidecar '{path}'")
    vals = []
    for t in toks:
        try:
            vals.append(float(t))
        except ValueError:
            break  # `in >> v` stops at the first token that is not a number
    return sorted(vals)


class _Usage(Exception):
    pass


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # CLI11 parse errors exit with kExitUsage
        raise _Usage(message)


def build_parser() -> argparse.ArgumentParser:
    ap = _Parser(prog="feastlab", description="FEAST/XFEAST/RFEAST interior eigensolver laboratory")
    sub = ap.add_subparsers(dest="cmd")
    sv = sub.add_parser("solve", help="Run one solver on a matrix")
    sv.add_argument("--algo", required=True, choices=["feast", "xfeast", "rfeast"])
    sv.add_argument("--matrix", required=True, help="Matrix Market file")
    sv.add_argument("--interval", required=True, nargs=2, type=float, metavar=("LO", "HI"))
    sv.add_argument("--m0", required=True, type=int, help="subspace size")
    sv.add_argument("--nc", type=int, default=8, help="quadrature points")
    sv.add_argument("--s", type=int, default=1, help="expansion depth")
    sv.add_argument("--tol", type=float, default=1e-12, help="residual tolerance")
    sv.add_argument("--max-iter", type=int, default=50, help="iteration limit")
    sv.add_argument("--seed", type=int, default=42, help="initial guess seed")
    sv.add_argument("--orthogonalizer", default="svd", choices=["svd", "qr"])
    sv.add_argument("--cache-factorizations", action="store_true",
                    help="reuse per-node factorizations across iterations")
    sv.add_argument("--trace", default="", help="trace CSV output path")
    sv.add_argument("--sidecar", default="", help="ground-truth eigenvalue file")
    return ap


def run_solve(opt, out=None) -> int:  # feastlab_cli.cpp:137-187
    from . import feastlab as P
    out = out or sys.stdout
    cfg = P.SolverConfig(m0=opt.m0, n_c=opt.nc, s=opt.s, tol=opt.tol, max_iter=opt.max_iter,
                         seed=opt.seed, orthogonalizer=opt.orthogonalizer,
                         cache_factorizations=opt.cache_factorizations)
    A = P.read_matrix_market(opt.matrix)
    interval = P.SearchInterval(opt.interval[0], opt.interval[1])
    driver = {"feast": P.feast_solve, "xfeast": P.xfeast_solve, "rfeast": P.rfeast_solve}[opt.algo]
    sol = driver(A, interval, cfg)
    if opt.trace:
        write_file_atomic(opt.trace, P.write_trace_csv(sol.trace))
    final = sol.trace[-1].max_residual if sol.trace else math.nan
    out.write(f"algorithm:      {opt.algo}\n")
    out.write(f"converged:      {'yes' if sol.converged else 'no'}\n")
    out.write(f"iterations:     {sol.iterations}\n")
    out.write(f"rhs_solved:     {sol.accounting.rhs_solved}\n")
    out.write(f"final_residual: {fmt17(final)}\n")
    out.write(f"m_found:        {len(sol.eigenvalues)}\n")
    out.write("eigenvalues:" + "".join(" " + fmt17(float(v)) for v in sol.eigenvalues) + "\n")
    sidecar = opt.sidecar
    if not sidecar and os.path.exists(sidecar_path(opt.matrix)):
        sidecar = sidecar_path(opt.matrix)
    if sidecar:
        truth = read_sidecar(sidecar)
        max_err = 0.0
        for v in sol.eigenvalues:
            best = min((abs(float(v) - t) for t in truth), default=math.inf)
            max_err = max(max_err, best)
        out.write(f"oracle_max_err: {fmt17(max_err)}\n")
    return EXIT_CONVERGED if sol.converged else EXIT_NOT_CONVERGED


def main(argv=None) -> int:
    try:
        opt = build_parser().parse_args(argv)
    except _Usage as e:
        sys.stderr.write(f"error: {e}\n")
        return EXIT_USAGE
    except SystemExit as e:  # --help
        return 0 if e.code in (0, None) else EXIT_USAGE
    if opt.cmd != "solve":
        sys.stderr.write("error: a subcommand is required (solve)\n")
        return EXIT_USAGE
    try:
        return run_solve(opt)
    except ValueError as e:  # std::invalid_argument -> kExitUsage (feastlab_cli.cpp:437-439)
        sys.stderr.write(f"error: {e}\n")
        return EXIT_USAGE
    except Exception as e:  # std::exception -> kExitFailure
        sys.stderr.write(f"error: {e}\n")
        return EXIT_FAILURE


if __name__ == "__main__":
    sys.exit(main())
