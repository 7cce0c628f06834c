"""TEST INFRASTRUCTURE ONLY — Python binding of the CPU oracle (liboracle.so).

The oracle is a C++ restatement of the reference feastlab hot path
(/root/reference/proj/src/{contour,filterop,ritz,drivers,matmodel}.cpp) on
scipy's OpenBLAS LAPACK; see feast_oracle.cpp's header for the Eigen call-site
mapping and README.md for how it is pinned. Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline leg may import this package: it is the checker,
never the product path.

Every function mirrors the reference API name and argument meaning; matrices
are numpy float64 arrays (any layout in, Fortran order out).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build() -> None:
    import subprocess
    import sys
    subprocess.run(["make", "-s", "-C", _HERE, f"PY={sys.executable}"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        _declare(_lib)
    return _lib


# The reference's own sources compiled against oracle/eigen_shim (`make -C
# oracle ref`, needs /root/reference): same orc_* entry points, so every
# function below can run on it. Present only where it was built.
_REF_PATH = os.path.join(_HERE, "_ref", "libfeastlab_ref.so")
_ref_lib = None


def reference_available() -> bool:
    return os.path.exists(_REF_PATH)


class reference_backend:
    """with oracle.reference_backend(): ...  -- route this module's calls to
    oracle/_ref/libfeastlab_ref.so (the reference's unmodified sources)."""

    def __enter__(self):
        global _lib, _ref_lib
        if _ref_lib is None:
            _ref_lib = C.CDLL(_REF_PATH)
            _declare(_ref_lib, optional=("orc_gaussian_fill", "orc_uniform_fill",
                                         "orc_seeded_orthogonal", "orc_node_factor"))
        lib()
        self._saved = _lib
        _lib = _ref_lib
        return self

    def __exit__(self, *exc):
        global _lib
        _lib = self._saved
        return False


# --------------------------------------------------------------- errors
class InvalidArgument(ValueError):
    """std::invalid_argument"""


class FeastRuntimeError(RuntimeError):
    """std::runtime_error"""


class CholeskyError(FeastRuntimeError):
    def __init__(self, msg, pivot, index):
        super().__init__(msg)
        self.pivot = pivot
        self.index = index


class SingularNodeError(FeastRuntimeError):
    def __init__(self, msg, node, z):
        super().__init__(msg)
        self.node = node
        self.z = z


class _Err(C.Structure):
    _fields_ = [("status", C.c_int), ("index", C.c_int), ("pivot", C.c_double),
                ("z_re", C.c_double), ("z_im", C.c_double), ("msg", C.c_char * 512)]


def _check(code, err):
    if code == 0:
        return
    msg = err.msg.decode(errors="replace")
    if code == 1:
        raise InvalidArgument(msg)
    if code == 3:
        raise CholeskyError(msg, err.pivot, err.index)
    if code == 4:
        raise SingularNodeError(msg, err.index, complex(err.z_re, err.z_im))
    raise FeastRuntimeError(msg)


class _Config(C.Structure):
    _fields_ = [("m0", C.c_int), ("n_c", C.c_int), ("s", C.c_int), ("tol", C.c_double),
                ("max_iter", C.c_int), ("seed", C.c_ulonglong), ("orthogonalizer", C.c_int),
                ("drop_tol", C.c_double), ("cache_factorizations", C.c_int),
                ("generalized_reduced", C.c_int)]


class _Trace(C.Structure):
    _fields_ = [("iter", C.c_int), ("subspace_dim", C.c_int), ("rhs_cumulative", C.c_longlong),
                ("max_residual", C.c_double), ("m_found", C.c_int)]


_P = C.c_void_p
_I = C.c_int
_D = C.c_double
_LL = C.c_longlong
_ULL = C.c_ulonglong


def _declare(L, optional=()):
    sig = {
        "orc_set_threads": (None, [_I]),
        "orc_get_threads": (_I, []),
        "orc_gauss_legendre": (_I, [_I, _P, _P, _P]),
        "orc_build_contour_rule": (_I, [_D, _D, _I, _P, _P, _P, _P, _P]),
        "orc_filter_value": (_D, [_I, _P, _P, _P, _P, _D]),
        "orc_predicted_rate": (_I, [_I, _P, _P, _P, _P, _P, _I, _I, _P, _P]),
        "orc_symmetric_matrix": (_I, [_P, _I, _D, _P, _P]),
        "orc_gaussian_fill": (None, [_P, _LL, _ULL]),
        "orc_uniform_fill": (None, [_P, _LL, _D, _D, _ULL]),
        "orc_seeded_orthogonal": (_I, [_I, _ULL, _P, _P]),
        "orc_generate_spectrum": (_I, [_I, _D, _D, _I, _D, _D, _I, _I, _I, _D, _ULL, _P, _P, _P]),
        "orc_assemble_matrix": (_I, [_I, _P, _P, _P, _P]),
        "orc_node_solve": (_I, [_P, _I, _D, _D, _P, _I, _P, _P]),
        "orc_node_factor": (_I, [_P, _I, _D, _D, _P, _P, _P]),
        "orc_apply_filter": (_I, [_P, _I, _I, _P, _P, _P, _P, _P, _I, _I, _I, _I, _P, _P, _P, _P]),
        "orc_orthonormalize": (_I, [_P, _I, _I, _D, _I, _P, _P, _P]),
        "orc_rayleigh_ritz": (_I, [_P, _I, _P, _I, _I, _D, _D, _P, _P, _P, _P, _P]),
        "orc_residual_block": (_I, [_P, _I, _P, _P, _I, _P, _P]),
        "orc_select_pairs": (_I, [_P, _P, _P, _I, _I, _D, _D, _P, _P, _P]),
        "orc_make_initial_guess": (_I, [_I, _I, _ULL, _P, _P]),
        "orc_solve": (_I, [_I, _P, _I, _D, _D, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                           _P]),
    }
    for name, (res, args) in sig.items():
        if name in optional and not hasattr(L, name):
            continue
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args


def _f64(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def set_threads(t: int) -> None:
    lib().orc_set_threads(int(t))


def get_threads() -> int:
    return lib().orc_get_threads()


# --------------------------------------------------------------- contour
@dataclass
class SearchInterval:
    lo: float
    hi: float

    def __post_init__(self):
        if not (self.lo < self.hi):
            raise InvalidArgument(f"SearchInterval: require lo < hi, got [{self.lo}, {self.hi}]")

    def center(self):
        return 0.5 * (self.lo + self.hi)

    def radius(self):
        return 0.5 * (self.hi - self.lo)

    def contains(self, x):
        return x > self.lo and x < self.hi


@dataclass
class ContourRule:
    interval: SearchInterval
    nodes: np.ndarray    # complex128, Im > 0
    weights: np.ndarray  # complex128

    def num_points(self):
        return len(self.nodes)

    def parts(self):
        return self._parts()

    def _parts(self):
        z = np.ascontiguousarray(self.nodes, dtype=np.complex128)
        w = np.ascontiguousarray(self.weights, dtype=np.complex128)
        return (np.ascontiguousarray(z.real), np.ascontiguousarray(z.imag),
                np.ascontiguousarray(w.real), np.ascontiguousarray(w.imag))


def gauss_legendre(n: int):
    x = np.zeros(max(n, 1))
    w = np.zeros(max(n, 1))
    e = _Err()
    _check(lib().orc_gauss_legendre(n, _ptr(x), _ptr(w), C.byref(e)), e)
    return x, w


def build_contour_rule(interval: SearchInterval, n_c: int) -> ContourRule:
    zr, zi, wr, wi = (np.zeros(max(n_c, 1)) for _ in range(4))
    e = _Err()
    _check(lib().orc_build_contour_rule(interval.lo, interval.hi, n_c, _ptr(zr), _ptr(zi),
                                        _ptr(wr), _ptr(wi), C.byref(e)), e)
    return ContourRule(interval, zr + 1j * zi, wr + 1j * wi)


def contour_rule_from_nodes(interval, nodes, weights) -> ContourRule:
    """proj/src/contour.cpp:71-81"""
    nodes = np.asarray(nodes, dtype=np.complex128)
    weights = np.asarray(weights, dtype=np.complex128)
    if len(nodes) == 0 or len(nodes) != len(weights):
        raise InvalidArgument("contour_rule_from_nodes: node/weight size mismatch")
    if not np.all(nodes.imag > 0.0):
        raise InvalidArgument("contour_rule_from_nodes: all nodes must have Im(z) > 0")
    return ContourRule(interval, nodes, weights)


def filter_value(rule: ContourRule, lam: float) -> float:
    zr, zi, wr, wi = rule._parts()
    return lib().orc_filter_value(rule.num_points(), _ptr(zr), _ptr(zi), _ptr(wr), _ptr(wi),
                                  float(lam))


def predicted_rate(rule: ContourRule, spectrum, m0: int) -> float:
    zr, zi, wr, wi = rule._parts()
    s = np.ascontiguousarray(spectrum, dtype=np.float64)
    out = C.c_double()
    e = _Err()
    _check(lib().orc_predicted_rate(rule.num_points(), _ptr(zr), _ptr(zi), _ptr(wr), _ptr(wi),
                                    _ptr(s), len(s), m0, C.byref(out), C.byref(e)), e)
    return out.value


# --------------------------------------------------------------- matmodel
def symmetric_matrix(M, sym_tol=1e-12) -> np.ndarray:
    M = _f64(M)
    if M.ndim != 2 or M.shape[0] != M.shape[1] or M.shape[0] < 1:
        raise InvalidArgument("SymmetricMatrix: matrix must be square, n >= 1")
    out = np.zeros_like(M, order="F")
    e = _Err()
    _check(lib().orc_symmetric_matrix(_ptr(M), M.shape[0], sym_tol, _ptr(out), C.byref(e)), e)
    return out


def gaussian_block(rows: int, cols: int, seed: int) -> np.ndarray:
    """mt19937_64(seed) + normal_distribution, column-major (oracles.hpp:60-67)."""
    out = np.zeros((rows, cols), order="F")
    lib().orc_gaussian_fill(_ptr(out), rows * cols, seed)
    return out


def random_symmetric(n: int, seed: int) -> np.ndarray:
    """proj/tests/oracles.hpp:50-57"""
    M = gaussian_block(n, n, seed)
    return np.asfortranarray(0.5 * (M + M.T))


def random_block(n: int, p: int, seed: int) -> np.ndarray:
    """proj/tests/oracles.hpp:60-67"""
    return gaussian_block(n, p, seed)


def uniform_fill(count: int, lo: float, hi: float, seed: int) -> np.ndarray:
    out = np.zeros(count)
    lib().orc_uniform_fill(_ptr(out), count, lo, hi, seed)
    return out


def seeded_orthogonal(n: int, seed: int) -> np.ndarray:
    Q = np.zeros((n, n), order="F")
    e = _Err()
    _check(lib().orc_seeded_orthogonal(n, seed, _ptr(Q), C.byref(e)), e)
    return Q


@dataclass
class SpectrumLayout:
    n: int
    inside_interval: SearchInterval
    inside_count: int
    outside_interval: SearchInterval
    outside_count: int
    placement: str = "uniform"
    num_clusters: int = 1
    cluster_width: float = 0.0
    seed: int = 0


def generate_spectrum(layout: SpectrumLayout):
    n = layout.n
    vals = np.zeros(max(n, 1))
    Q = np.zeros((max(n, 1), max(n, 1)), order="F")
    e = _Err()
    _check(lib().orc_generate_spectrum(
        n, layout.inside_interval.lo, layout.inside_interval.hi, layout.inside_count,
        layout.outside_interval.lo, layout.outside_interval.hi, layout.outside_count,
        1 if layout.placement == "clustered" else 0, layout.num_clusters, layout.cluster_width,
        layout.seed, _ptr(vals), _ptr(Q), C.byref(e)), e)
    return vals, Q


def assemble_matrix(values, Q) -> np.ndarray:
    values = np.ascontiguousarray(values, dtype=np.float64)
    Q = _f64(Q)
    n = len(values)
    A = np.zeros((n, n), order="F")
    e = _Err()
    _check(lib().orc_assemble_matrix(n, _ptr(values), _ptr(Q), _ptr(A), C.byref(e)), e)
    return A


# --------------------------------------------------------------- filterop
@dataclass
class SolveAccounting:
    rhs_solved: int = 0
    factorizations: int = 0


def node_solve(A, z: complex, B) -> np.ndarray:
    """NodeFactorization(A, z).solve(B) — proj/src/filterop.cpp:9-32"""
    A = _f64(A)
    B = np.asfortranarray(np.asarray(B, dtype=np.complex128))
    if B.ndim == 1:
        B = B.reshape(-1, 1, order="F")
    n, p = B.shape
    W = np.zeros((n, p), dtype=np.complex128, order="F")
    e = _Err()
    _check(lib().orc_node_solve(_ptr(A), A.shape[0], z.real, z.imag, _ptr(B), p, _ptr(W),
                                C.byref(e)), e)
    return W


def node_factor(A, z: complex):
    A = _f64(A)
    n = A.shape[0]
    LU = np.zeros((n, n), dtype=np.complex128, order="F")
    perm = np.zeros(n, dtype=np.int32)
    e = _Err()
    _check(lib().orc_node_factor(_ptr(A), n, z.real, z.imag, _ptr(LU), _ptr(perm), C.byref(e)), e)
    return LU, perm


def apply_filter(A, rule: ContourRule, X, accounting: SolveAccounting | None = None, *,
                 cache=False, napply=1) -> np.ndarray:
    """apply_filter / FilterApplier::apply (proj/src/filterop.cpp:50-84)."""
    A = _f64(A)
    X = _f64(X)
    if X.ndim == 1:
        X = X.reshape(-1, 1, order="F")
    acc = accounting if accounting is not None else SolveAccounting()
    zr, zi, wr, wi = rule._parts()
    xr, p = X.shape
    Y = np.zeros((xr, max(p, 1)), order="F")
    rhs = C.c_longlong(acc.rhs_solved)
    facts = C.c_longlong(acc.factorizations)
    e = _Err()
    _check(lib().orc_apply_filter(_ptr(A), A.shape[0], rule.num_points(), _ptr(zr), _ptr(zi),
                                  _ptr(wr), _ptr(wi), _ptr(X), xr, p, int(cache), napply, _ptr(Y),
                                  C.byref(rhs), C.byref(facts), C.byref(e)), e)
    acc.rhs_solved = rhs.value
    acc.factorizations = facts.value
    return Y[:, :p]


# --------------------------------------------------------------- ritz
@dataclass
class RitzSet:
    values: np.ndarray
    vectors: np.ndarray
    residual_norms: np.ndarray
    inside_flags: np.ndarray

    def size(self):
        return len(self.values)


def orthonormalize(X, drop_tol: float, method: str = "svd"):
    X = _f64(X)
    n, p = X.shape if X.ndim == 2 else (X.shape[0], 0)
    U = np.zeros((max(n, 1), max(p, 1)), order="F")
    rank = C.c_int()
    e = _Err()
    _check(lib().orc_orthonormalize(_ptr(X), n, p, drop_tol, 1 if method == "qr" else 0, _ptr(U),
                                    C.byref(rank), C.byref(e)), e)
    r = rank.value
    return np.asfortranarray(U.reshape(-1, order="F")[: n * r].reshape(n, r, order="F")), r


def rayleigh_ritz(A, X, interval: SearchInterval) -> RitzSet:
    A = _f64(A)
    X = _f64(X)
    n = A.shape[0]
    xr, p = X.shape
    vals = np.zeros(max(p, 1))
    V = np.zeros((n, max(p, 1)), order="F")
    norms = np.zeros(max(p, 1))
    inside = np.zeros(max(p, 1), dtype=np.uint8)
    e = _Err()
    _check(lib().orc_rayleigh_ritz(_ptr(A), n, _ptr(X), xr, p, interval.lo, interval.hi,
                                   _ptr(vals), _ptr(V), _ptr(norms), _ptr(inside), C.byref(e)), e)
    return RitzSet(vals[:p], V[:, :p], norms[:p], inside[:p].astype(bool))


def compute_residual_block(A, ritz: RitzSet) -> np.ndarray:
    A = _f64(A)
    V = _f64(ritz.vectors)
    vals = np.ascontiguousarray(ritz.values, dtype=np.float64)
    n, p = V.shape
    R = np.zeros((n, p), order="F")
    e = _Err()
    _check(lib().orc_residual_block(_ptr(A), n, _ptr(vals), _ptr(V), p, _ptr(R), C.byref(e)), e)
    return R


def select_indices(ritz: RitzSet, target_count: int, interval: SearchInterval):
    p = ritz.size()
    vals = np.ascontiguousarray(ritz.values, dtype=np.float64)
    norms = np.ascontiguousarray(ritz.residual_norms, dtype=np.float64)
    inside = np.ascontiguousarray(ritz.inside_flags, dtype=np.uint8)
    chosen = np.zeros(max(p, 1), dtype=np.int32)
    nch = C.c_int()
    e = _Err()
    _check(lib().orc_select_pairs(_ptr(vals), _ptr(norms), _ptr(inside), p, target_count,
                                  interval.lo, interval.hi, _ptr(chosen), C.byref(nch),
                                  C.byref(e)), e)
    return chosen[: nch.value].copy()


def select_pairs(ritz: RitzSet, target_count: int, interval: SearchInterval) -> RitzSet:
    idx = select_indices(ritz, target_count, interval)
    return RitzSet(ritz.values[idx], np.asfortranarray(ritz.vectors[:, idx]),
                   ritz.residual_norms[idx], np.asarray(ritz.inside_flags)[idx])


def count_inside(ritz: RitzSet) -> int:
    return int(np.count_nonzero(ritz.inside_flags))


# --------------------------------------------------------------- drivers
@dataclass
class SolverConfig:
    m0: int = 1
    n_c: int = 8
    s: int = 1
    tol: float = 1e-12
    max_iter: int = 50
    seed: int = 42
    orthogonalizer: str = "svd"
    drop_tol: float = 1e-10
    cache_factorizations: bool = False
    generalized_reduced: bool = False


@dataclass
class TraceRecord:
    iter: int
    subspace_dim: int
    rhs_cumulative: int
    max_residual: float
    m_found: int


@dataclass
class Solution:
    eigenvalues: np.ndarray
    eigenvectors: np.ndarray
    residual_norms: np.ndarray
    converged: bool
    iterations: int
    accounting: SolveAccounting
    trace: list = field(default_factory=list)
    recovery_events: int = 0
    first_filtered: np.ndarray | None = None


def make_initial_guess(n: int, m0: int, seed: int) -> np.ndarray:
    X = np.zeros((max(n, 1), max(m0, 1)), order="F")
    e = _Err()
    _check(lib().orc_make_initial_guess(n, m0, seed, _ptr(X), C.byref(e)), e)
    return X


def _solve(variant, A, interval, cfg: SolverConfig) -> Solution:
    A = _f64(A)
    n = A.shape[0]
    c = _Config(cfg.m0, cfg.n_c, cfg.s, cfg.tol, cfg.max_iter, cfg.seed,
                1 if cfg.orthogonalizer == "qr" else 0, cfg.drop_tol,
                int(cfg.cache_factorizations), int(cfg.generalized_reduced))
    m0 = max(cfg.m0, 1)
    vals = np.zeros(m0)
    norms = np.zeros(m0)
    V = np.zeros((n, m0), order="F")
    first = np.zeros((n, m0), order="F")
    m = C.c_int()
    conv = C.c_int()
    iters = C.c_int()
    rhs = C.c_longlong()
    facts = C.c_longlong()
    rec = C.c_int()
    trace = (_Trace * max(cfg.max_iter, 1))()
    ntrace = C.c_int()
    e = _Err()
    _check(lib().orc_solve(variant, _ptr(A), n, interval.lo, interval.hi, C.byref(c), _ptr(vals),
                           _ptr(V), _ptr(norms), C.byref(m), C.byref(conv), C.byref(iters),
                           C.byref(rhs), C.byref(facts), C.byref(rec), trace, C.byref(ntrace),
                           _ptr(first), C.byref(e)), e)
    k = m.value
    tr = [TraceRecord(t.iter, t.subspace_dim, t.rhs_cumulative, t.max_residual, t.m_found)
          for t in trace[: ntrace.value]]
    return Solution(vals[:k].copy(), np.asfortranarray(V.reshape(-1, order="F")[: n * k]
                                                       .reshape(n, k, order="F")),
                    norms[:k].copy(), bool(conv.value), iters.value,
                    SolveAccounting(rhs.value, facts.value), tr, rec.value, first)


def feast_solve(A, interval, cfg):
    return _solve(0, A, interval, cfg)


def xfeast_solve(A, interval, cfg):
    return _solve(1, A, interval, cfg)


def rfeast_solve(A, interval, cfg):
    return _solve(2, A, interval, cfg)


def write_trace_csv(trace) -> str:
    """proj/src/drivers.cpp:13-21 ("%d,%d,%lld,%.17g,%d")."""
    out = ["iter,subspace_dim,rhs_cumulative,max_residual,m_found\n"]
    for r in trace:
        out.append("%d,%d,%d,%s,%d\n" % (r.iter, r.subspace_dim, r.rhs_cumulative,
                                          _g17(r.max_residual), r.m_found))
    return "".join(out)


def _g17(x):
    return "%.17g" % x


# --------------------------------------------------------------- independent test oracles
def dense_eig(A):
    """proj/tests/oracles.hpp:75-78 (numpy LAPACK dsyevd, ascending)."""
    w, V = np.linalg.eigh(np.asarray(A, dtype=np.float64))
    return w, V


def spectral_filter_reference(A, rule: ContourRule, X):
    """proj/tests/oracles.hpp:82-90 — Q rho(Lambda) Q^T X."""
    w, V = dense_eig(A)
    rho = np.array([filter_value(rule, x) for x in w])
    return V @ (rho[:, None] * (V.T @ np.asarray(X, dtype=np.float64)))


def adaptive_simpson(f, a, b, tol=1e-12, depth=40):
    """proj/tests/oracles.hpp:14-34"""
    def rec(lo, hi, flo, fmid, fhi, whole, d):
        mid = 0.5 * (lo + hi)
        lm, rm = 0.5 * (lo + mid), 0.5 * (mid + hi)
        flm, frm = f(lm), f(rm)
        left = (mid - lo) / 6.0 * (flo + 4.0 * flm + fmid)
        right = (hi - mid) / 6.0 * (fmid + 4.0 * frm + fhi)
        if d <= 0 or abs(left + right - whole) < 15.0 * tol:
            return left + right + (left + right - whole) / 15.0
        return rec(lo, mid, flo, flm, fmid, left, d - 1) + rec(mid, hi, fmid, frm, fhi, right, d - 1)
    mid = 0.5 * (a + b)
    fa, fm, fb = f(a), f(mid), f(b)
    return rec(a, b, fa, fm, fb, (b - a) / 6.0 * (fa + 4.0 * fm + fb), depth)


def exact_circle_filter(interval: SearchInterval, lam: float) -> float:
    """proj/tests/oracles.hpp:38-47"""
    import cmath
    import math
    c, r = interval.center(), interval.radius()

    def integrand(t):
        e = cmath.exp(1j * t)
        return (r * e / (c + r * e - lam)).real
    return adaptive_simpson(integrand, 0.0, math.pi, 1e-13) / math.pi
