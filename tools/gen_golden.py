"""Generate tests/golden/oracle_cfg<k>.json: the CPU oracle's FEAST / XFEAST /
RFEAST results (traces, iteration/converged counts, eigenvalues, recovery
events) on a BASELINE configuration, so the GPU parity tests need not rerun
minutes-to-hours of CPU work. Run in the build container.

Usage:
  python tools/gen_golden.py <cfg> <threads> <driver>   -> tests/golden/parts/oracle_cfg<k>_<driver>.json
  python tools/gen_golden.py <cfg> <threads> <driver> ref -> tests/golden/parts/ref_cfg<k>_<driver>.json
  python tools/gen_golden.py <cfg> <threads> <driver> sens -> tests/golden/parts/sens_cfg<k>_<driver>.json
  python tools/gen_golden.py merge <cfg>                -> tests/golden/oracle_cfg<k>.json

`ref` runs the same solve on oracle/_ref/libfeastlab_ref.so: the reference's
own sources compiled unmodified against oracle/eigen_shim (`make -C oracle
ref`). Its results are merged under "reference_build" and
tests/test_ref_pin.py requires the restatement's goldens to agree with them.

The goldens are generated with ONE OpenBLAS thread: the reference is built
single-threaded (proj/CMakeLists.txt:6-13, no OpenMP), and the Gram-floor rank
decisions of XFEAST/RFEAST flip with OpenBLAS's threaded summation order
(profiles/cfg1_oracle_thread_sensitivity.jsonl). cfg4 (n = 16384) is the
exception: FEAST only, several threads (a one-thread run is ~4 h).

FEAST also records a sketch of its first filtered subspace Y_1 (too large to
commit at n >= 4096): ||Y_1||_F, the column norms and Omega Y_1 for a seeded
16 x n Gaussian Omega (sketch_omega below), so the GPU tests can check the
north-star gate ||Y_1,gpu - Y_1,ref||_F / ||Y_1,ref||_F <= 1e-9 through the
sketch (a Johnson-Lindenstrauss estimate of the same ratio). When Y_1 is at
most 2 MB (cfg0) the whole Y_1 is stored (float64, base64) so the gate is
checked exactly.

Per trace record the generator also logs the decision margins that can flip
an iteration count at rounding level: the max residual
over tol (r/tol, proj/src/drivers.cpp:177,239)."""
import base64, glob, json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLD = os.path.join(ROOT, "tests", "golden")


def sketch_omega(n, rows=16, seed=7):
    return np.random.default_rng(seed).standard_normal((rows, n)) / np.sqrt(rows)


def first_sketch(Y):
    out = {"fro": float(np.linalg.norm(Y)), "col_norms": [float(x) for x in np.linalg.norm(Y, axis=0)],
           "sketch_seed": 7, "sketch_rows": 16,
           "sketch": [float(x) for x in (sketch_omega(Y.shape[0]) @ Y).ravel(order="F")]}
    if Y.size * 8 <= 2_000_000:
        out["full_shape"] = list(Y.shape)
        out["full_b64"] = base64.b64encode(np.asfortranarray(Y, dtype="<f8").tobytes(order="F")).decode()
    return out


def full_first(entry):
    """The stored whole Y_1 (n <= 2000 goldens) or None."""
    if "full_b64" not in entry:
        return None
    r, c = entry["full_shape"]
    return np.frombuffer(base64.b64decode(entry["full_b64"]), dtype="<f8").reshape((r, c), order="F")


def build_problem(idx, O, CF):
    vals = CF.spectrum(idx, O.uniform_fill)
    c = CF.resolved(idx, vals)
    A = CF.laplacian_2d() if idx == 3 else O.assemble_matrix(vals, O.seeded_orthogonal(len(vals), 1000 + idx))
    return A, c


def run(idx, threads, d, ref=False, sens=False):
    import contextlib
    import oracle as O
    from paper_1605_08771_b200 import configs as CF
    O.set_threads(threads)
    A, c = build_problem(idx, O, CF)
    t = time.time()
    with (O.reference_backend() if ref else contextlib.nullcontext()):
        s = getattr(O, d)(A, O.SearchInterval(c["lo"], c["hi"]),
                          O.SolverConfig(m0=c["m0"], n_c=c["n_c"], tol=c["tol"],
                                         max_iter=c["max_iter"], s=c["s"]))
    e = {"seconds": round(time.time() - t, 2), "oracle_threads": O.get_threads(),
         "iterations": s.iterations, "converged": s.converged,
         "m": len(s.eigenvalues), "eigenvalues": [float(x) for x in s.eigenvalues],
         "residual_norms": [float(x) for x in s.residual_norms], "recovery_events": s.recovery_events,
         "rhs_solved": s.accounting.rhs_solved, "factorizations": s.accounting.factorizations,
         "trace": [[t.iter, t.subspace_dim, t.rhs_cumulative, t.max_residual, t.m_found] for t in s.trace],
         "r_over_tol": [t.max_residual / c["tol"] for t in s.trace]}
    if d == "feast_solve" and s.first_filtered is not None and not ref:
        e["first_filtered"] = first_sketch(s.first_filtered)
    if ref:
        e["library"] = "oracle/_ref/libfeastlab_ref.so (reference sources + oracle/eigen_shim)"
    os.makedirs(os.path.join(GOLD, "parts"), exist_ok=True)
    if sens:  # a sensitivity run: outcomes and trace only
        for k in ("eigenvalues", "residual_norms", "first_filtered"):
            e.pop(k, None)
    tag = f"sens_cfg{idx}_{d}_t{threads}" if sens else f"{'ref' if ref else 'oracle'}_cfg{idx}_{d}"
    with open(os.path.join(GOLD, "parts", tag + ".json"), "w") as f:
        json.dump({"cfg": idx, "config": c, "driver": d, "result": e}, f)
    print(idx, d, e["iterations"], e["converged"], e["m"], e["recovery_events"], e["seconds"], flush=True)


def merge(idx):
    out = None
    for p in sorted(glob.glob(os.path.join(GOLD, "parts", f"oracle_cfg{idx}_*.json"))):
        part = json.load(open(p))
        if out is None:
            out = {"cfg": idx, "config": part["config"], "generator": "tools/gen_golden.py", "drivers": {}}
        res = part["result"]
        ff = res.get("first_filtered", {})
        if len(ff.get("full_b64", "")) > 3_000_000:  # keep the committed fixture small
            ff.pop("full_b64")
            ff.pop("full_shape")
        out["drivers"][part["driver"]] = res
    out["oracle_threads"] = max(e["oracle_threads"] for e in out["drivers"].values())
    out["reference_build"] = {}
    for p in sorted(glob.glob(os.path.join(GOLD, "parts", f"ref_cfg{idx}_*.json"))):
        part = json.load(open(p))
        res = part["result"]
        res.pop("residual_norms", None)  # keep the fixture small: outcomes, trace, eigenvalues
        out["reference_build"][part["driver"]] = res
    # the same oracle solve with 2 ... 8 OpenBLAS threads, one run each (a rounding-level
    # perturbation: only the summation order inside the BLAS changes): where its
    # trace leaves the one-thread trace the reference algorithm itself is not
    # reproducible at rounding level (tests/test_gpu_configs.py)
    out["sensitivity"] = {}
    for p in sorted(glob.glob(os.path.join(GOLD, "parts", f"sens_cfg{idx}_*.json"))):
        part = json.load(open(p))
        out["sensitivity"].setdefault(part["driver"], []).append(part["result"])
    with open(os.path.join(GOLD, f"oracle_cfg{idx}.json"), "w") as f:
        json.dump(out, f)
    print("wrote", idx, sorted(out["drivers"]))


if __name__ == "__main__":
    if sys.argv[1] == "merge":
        merge(int(sys.argv[2]))
    else:
        run(int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], ref=(len(sys.argv) > 4 and sys.argv[4] == "ref"),
            sens=(len(sys.argv) > 4 and sys.argv[4] == "sens"))
