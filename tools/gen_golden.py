"""Generate tests/golden/oracle_cfg<k>.json: the CPU oracle's FEAST / XFEAST /
RFEAST results (traces, iteration/converged counts, eigenvalues) on a BASELINE
configuration, so the GPU parity tests need not rerun minutes of CPU work.
Usage: python tools/gen_golden.py <cfg> [threads] [drivers,...]   (run in the build container)

FEAST also records a sketch of its first filtered subspace Y_1 (too large to
commit at n >= 4096): ||Y_1||_F, the column norms and Omega Y_1 for a seeded
16 x n Gaussian Omega (sketch_omega below), so the GPU tests can check the
north-star gate ||Y_1,gpu - Y_1,ref||_F / ||Y_1,ref||_F <= 1e-9 through the
sketch (a Johnson-Lindenstrauss estimate of the same ratio)."""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O
from paper_1605_08771_b200 import configs as CF

def sketch_omega(n, rows=16, seed=7):
    return np.random.default_rng(seed).standard_normal((rows, n)) / np.sqrt(rows)


def first_sketch(Y):
    return {"fro": float(np.linalg.norm(Y)), "col_norms": [float(x) for x in np.linalg.norm(Y, axis=0)],
            "sketch_seed": 7, "sketch_rows": 16,
            "sketch": [float(x) for x in (sketch_omega(Y.shape[0]) @ Y).ravel(order="F")]}


if __name__ != "__main__":
    raise SystemExit  # imported by the tests only for sketch_omega / first_sketch
idx = int(sys.argv[1])
if len(sys.argv) > 2:
    O.set_threads(int(sys.argv[2]))
vals = CF.spectrum(idx, O.uniform_fill)
c = CF.resolved(idx, vals)
A = CF.laplacian_2d() if idx == 3 else O.assemble_matrix(vals, O.seeded_orthogonal(len(vals), 1000 + idx))
out = {"cfg": idx, "config": c, "oracle_threads": O.get_threads(), "generator": "tools/gen_golden.py",
       "drivers": {}}
drivers = sys.argv[3].split(",") if len(sys.argv) > 3 else ["feast_solve", "xfeast_solve", "rfeast_solve"]
for d in drivers:
    t = time.time()
    s = getattr(O, d)(A, O.SearchInterval(c["lo"], c["hi"]),
                      O.SolverConfig(m0=c["m0"], n_c=c["n_c"], tol=c["tol"], max_iter=c["max_iter"], s=c["s"]))
    out["drivers"][d] = {
        "seconds": round(time.time() - t, 2), "iterations": s.iterations, "converged": s.converged,
        "m": len(s.eigenvalues), "eigenvalues": [float(x) for x in s.eigenvalues],
        "residual_norms": [float(x) for x in s.residual_norms], "recovery_events": s.recovery_events,
        "rhs_solved": s.accounting.rhs_solved, "factorizations": s.accounting.factorizations,
        "trace": [[t.iter, t.subspace_dim, t.rhs_cumulative, t.max_residual, t.m_found] for t in s.trace]}
    if d == "feast_solve" and s.first_filtered is not None:
        out["drivers"][d]["first_filtered"] = first_sketch(s.first_filtered)
    print(d, out["drivers"][d]["iterations"], out["drivers"][d]["converged"], flush=True)
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                    f"oracle_cfg{idx}.json")
with open(path, "w") as f:
    json.dump(out, f)
print("wrote", path)
