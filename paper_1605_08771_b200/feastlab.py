"""Python mirror of the feastlab API (proj/include/feastlab/*.hpp) over the C ABI.

Same names, argument meaning and error behaviour as the reference:
std::invalid_argument -> InvalidArgument (a ValueError), std::runtime_error ->
FeastRuntimeError, CholeskyError(pivot, index). Matrices are numpy float64
(column-major internally). Every compute call runs on the B200 through
libfeastlab_b200.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L


# ------------------------------------------------------------------ errors
class InvalidArgument(ValueError):
    """std::invalid_argument"""


class FeastRuntimeError(RuntimeError):
    """std::runtime_error"""


class CholeskyError(FeastRuntimeError):
    """feastlab::CholeskyError (proj/include/feastlab/ritz.hpp:27-31)"""

    def __init__(self, msg, pivot, index):
        super().__init__(msg)
        self.pivot = pivot
        self.index = index


class SingularNodeError(FeastRuntimeError):
    """factorize_node's runtime_error (proj/src/filterop.cpp:15-23)"""

    def __init__(self, msg, node, z):
        super().__init__(msg)
        self.node = node
        self.z = z


class MatrixMarketError(FeastRuntimeError):
    """feastlab::MatrixMarketError (proj/include/feastlab/matrix_market.hpp:9-16)"""

    def __init__(self, msg, line):
        super().__init__(msg)
        self.line = line


class NotSymmetricError(MatrixMarketError):
    """feastlab::NotSymmetricError (proj/include/feastlab/matrix_market.hpp:18-21)"""


class FeastCudaError(RuntimeError):
    """CUDA / NCCL / device-memory failure (no CPU fallback exists)."""


def _check(code, err):
    if code == L.FL_OK:
        return
    msg = err.msg.decode(errors="replace")
    if code == L.FL_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if code == L.FL_CHOLESKY:
        raise CholeskyError(msg, err.pivot, err.index)
    if code == L.FL_SINGULAR_NODE:
        raise SingularNodeError(msg, err.index, complex(err.z_re, err.z_im))
    if code == L.FL_NOT_SYMMETRIC:
        raise NotSymmetricError(msg, err.index)
    if code == L.FL_MATRIX_MARKET:
        raise MatrixMarketError(msg, err.index)
    if code == L.FL_RUNTIME_ERROR:
        raise FeastRuntimeError(msg)
    raise FeastCudaError(f"[status {code}] {msg}")


def _call(fn, *args):
    err = L.Err()
    _check(fn(*args, C.byref(err)), err)


def _f64(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


# ------------------------------------------------------------------ context
class Context:
    """fl_ctx: one GPU (and optionally one rank of an NCCL clique)."""

    def __init__(self, device: int = 0, *, nccl_id: bytes | None = None, rank: int = 0,
                 nranks: int = 1, virtual: bool = False):
        """virtual=True: rank `rank` of `nranks` for the node sharding only, no
        communicator (fl_ctx_create_virtual; filters return the rank's partial sum)."""
        h = C.c_void_p()
        if virtual:
            _call(L.lib().fl_ctx_create_virtual, device, rank, nranks, C.byref(h))
        elif nccl_id is not None:
            buf = C.create_string_buffer(bytes(nccl_id), 128)
            _call(L.lib().fl_ctx_create_nccl, device, buf, rank, nranks, C.byref(h))
        else:
            _call(L.lib().fl_ctx_create, device, C.byref(h))
        self.handle = h
        self.device = device
        self.rank = rank
        self.nranks = nranks

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _call(L.lib().fl_nccl_unique_id, buf)
        return buf.raw

    @property
    def stream(self) -> int:
        return L.lib().fl_ctx_stream(self.handle) or 0

    def sync(self):
        _call(L.lib().fl_ctx_sync, self.handle)

    def launches(self) -> int:
        return L.lib().fl_ctx_launches(self.handle)

    KERNEL_CLASSES = ("shift", "panel", "laswp", "trsm", "zgemm", "zsum", "permute", "accumulate",
                      "allreduce")
    PHASE_CLASSES = ("eig", "orthonormalize", "rayleigh_ritz")

    def set_streams(self, n: int) -> None:
        """Contour-node chunks in flight (1 serialises the filter's kernels)."""
        L.lib().fl_ctx_set_streams(self.handle, int(n))

    def set_reduction(self, mode: str) -> None:
        """Multi-rank combination of the partial filters: "sum" (all-reduce,
        default) or "ordered" (all-gather + ascending-k sum: Y bitwise the same
        at every GPU count)."""
        if mode not in ("sum", "ordered"):
            raise InvalidArgument("set_reduction: mode must be 'sum' or 'ordered'")
        _check(L.lib().fl_ctx_set_reduction(self.handle, 1 if mode == "ordered" else 0), L.Err())

    FACTORIZATIONS = ("lu", "ldlt")

    def set_factorization(self, mode: str) -> None:
        """How the filter factors z_k I - A: "lu" (complex partial-pivot LU, the
        reference's PartialPivLU; default) or "ldlt" (complex-symmetric LDL^T
        without interchanges: half the flops, pivots bounded below by Im z_k;
        agrees with "lu" to rounding)."""
        if mode not in self.FACTORIZATIONS:
            raise InvalidArgument("set_factorization: mode must be 'lu' or 'ldlt'")
        _check(L.lib().fl_ctx_set_factorization(self.handle, self.FACTORIZATIONS.index(mode)),
               L.Err())

    @property
    def factorization(self) -> str:
        return self.FACTORIZATIONS[L.lib().fl_ctx_factorization(self.handle)]

    def set_profiling(self, on: bool) -> None:
        """Per-kernel-class CUDA-event timing on the context stream."""
        L.lib().fl_ctx_set_profiling(self.handle, int(bool(on)))

    def profile(self, cls: str):
        """(milliseconds, algorithmic work, launches) accumulated for `cls`."""
        ms, work, n = C.c_double(), C.c_double(), C.c_longlong()
        _call(L.lib().fl_ctx_profile, self.handle, cls.encode(), C.byref(ms), C.byref(work),
              C.byref(n))
        return ms.value, work.value, n.value

    def close(self):
        if self.handle:
            L.lib().fl_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_tls = threading.local()


def default_context() -> Context:
    ctx = getattr(_tls, "ctx", None)
    if ctx is None:
        ctx = Context(0)
        _tls.ctx = ctx
    return ctx


def set_default_context(ctx: Context | None) -> None:
    _tls.ctx = ctx


def zgemm_mode(mode: str | None = None) -> str:
    """Complex product form of the filter's DMMA GEMMs, process-wide: "3m"
    (three real products per complex product; default) or "4m". With no
    argument only reports the mode in effect."""
    if mode not in (None, "3m", "4m"):
        raise ValueError("zgemm_mode: mode must be '3m' or '4m'")
    code = -1 if mode is None else (1 if mode == "3m" else 0)
    return "3m" if L.lib().fl_zgemm_mode(code) == 1 else "4m"


def device_count() -> int:
    c = C.c_int()
    L.lib().fl_device_count(C.byref(c))
    return c.value


# ------------------------------------------------------------------ contour (host C++)
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
    nodes: np.ndarray
    weights: np.ndarray

    def num_points(self):
        return len(self.nodes)

    def _parts(self):
        return self.parts()

    def parts(self):
        z = np.ascontiguousarray(self.nodes, dtype=np.complex128)
        w = np.ascontiguousarray(self.weights, dtype=np.complex128)
        return (np.ascontiguousarray(z.real), np.ascontiguousarray(z.imag),
                np.ascontiguousarray(w.real), np.ascontiguousarray(w.imag))


def gauss_legendre(n: int):
    x = np.zeros(max(n, 1))
    w = np.zeros(max(n, 1))
    _call(L.lib().fl_gauss_legendre, n, _ptr(x), _ptr(w))
    return x, w


def build_contour_rule(interval: SearchInterval, n_c: int) -> ContourRule:
    zr, zi, wr, wi = (np.zeros(max(n_c, 1)) for _ in range(4))
    _call(L.lib().fl_build_contour_rule, interval.lo, interval.hi, n_c, _ptr(zr), _ptr(zi),
          _ptr(wr), _ptr(wi))
    return ContourRule(interval, zr + 1j * zi, wr + 1j * wi)


def contour_rule_from_nodes(interval, nodes, weights) -> ContourRule:
    nodes = np.asarray(nodes, dtype=np.complex128)
    weights = np.asarray(weights, dtype=np.complex128)
    if len(nodes) == 0 or len(nodes) != len(weights):
        raise InvalidArgument("contour_rule_from_nodes: node/weight size mismatch")
    if not np.all(nodes.imag > 0.0):
        raise InvalidArgument("contour_rule_from_nodes: all nodes must have Im(z) > 0")
    return ContourRule(interval, nodes, weights)


def filter_value(rule: ContourRule, lam: float) -> float:
    zr, zi, wr, wi = rule.parts()
    return L.lib().fl_filter_value(rule.num_points(), _ptr(zr), _ptr(zi), _ptr(wr), _ptr(wi),
                                   float(lam))


# ------------------------------------------------------------------ matmodel
class SymmetricMatrix:
    """proj/include/feastlab/matmodel.hpp:12-24 (symmetrised at construction)."""

    def __init__(self, entries, sym_tol: float = 1e-12):
        M = _f64(entries)
        if M.ndim != 2 or M.shape[0] != M.shape[1] or M.shape[0] < 1:
            raise InvalidArgument("SymmetricMatrix: matrix must be square, n >= 1")
        n = M.shape[0]
        out = np.zeros((n, n), order="F")
        _call(L.lib().fl_symmetric_matrix, _ptr(M), n, n, sym_tol, _ptr(out))
        self._mat = out

    def dim(self):
        return self._mat.shape[0]

    def mat(self):
        return self._mat


def read_matrix_market(path) -> SymmetricMatrix:
    """proj/src/matrix_market.cpp:31-117 (coordinate / array, real symmetric),
    parsed by the library's host layer; upload with DeviceMatrix."""
    n = C.c_int()
    p = os.fsencode(path)
    _call(L.lib().fl_mm_read, p, C.byref(n), None, 0)
    M = np.empty((n.value, n.value), order="F")
    _call(L.lib().fl_mm_read, p, C.byref(n), _ptr(M), n.value)
    return SymmetricMatrix(M)


def write_matrix_market(A, path, format: str = "coordinate") -> None:
    """proj/src/matrix_market.cpp:119-147 (lower triangle, %.17g)."""
    if format not in ("coordinate", "array"):
        raise InvalidArgument(f"write_matrix_market: unknown format '{format}'")
    M = _as_sym(A).mat()
    _call(L.lib().fl_mm_write, os.fsencode(path), _ptr(M), M.shape[0], M.shape[0],
          0 if format == "coordinate" else 1)


def _as_sym(A) -> SymmetricMatrix:
    return A if isinstance(A, SymmetricMatrix) else SymmetricMatrix(A)


# ------------------------------------------------------------------ device handles
class DeviceMatrix:
    def __init__(self, A, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        S = _as_sym(A)
        M = S.mat()
        h = C.c_void_p()
        _call(L.lib().fl_matrix_create, self.ctx.handle, _ptr(M), M.shape[0], M.shape[0],
              L.FL_HOST, C.byref(h))
        self.handle = h
        self.n = M.shape[0]

    @classmethod
    def from_device(cls, ptr: int, n: int, lda: int, ctx: Context):
        self = cls.__new__(cls)
        self.ctx = ctx
        h = C.c_void_p()
        _call(L.lib().fl_matrix_create, ctx.handle, C.c_void_p(ptr), n, lda, L.FL_DEVICE,
              C.byref(h))
        self.handle = h
        self.n = n
        return self

    def __del__(self):
        try:
            if self.handle:
                L.lib().fl_matrix_destroy(self.handle)
        except Exception:
            pass


class DeviceBlock:
    def __init__(self, n: int, cap: int = 1, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        h = C.c_void_p()
        _call(L.lib().fl_block_create, self.ctx.handle, n, max(cap, 1), C.byref(h))
        self.handle = h
        self.n = n

    def cols(self):
        return L.lib().fl_block_cols(self.handle)

    def set(self, X):
        X = _f64(X)
        if X.ndim == 1:
            X = X.reshape(-1, 1, order="F")
        _call(L.lib().fl_block_set, self.handle, _ptr(X), max(X.shape[0], 1), X.shape[1],
              L.FL_HOST)
        return self

    def get(self) -> np.ndarray:
        X = np.zeros((self.n, self.cols()), order="F")
        _call(L.lib().fl_block_get, self.handle, _ptr(X), self.n, L.FL_HOST)
        return X

    def __del__(self):
        try:
            if self.handle:
                L.lib().fl_block_destroy(self.handle)
        except Exception:
            pass


# ------------------------------------------------------------------ filterop
@dataclass
class SolveAccounting:
    rhs_solved: int = 0
    factorizations: int = 0


class NodeFactorization:
    """NodeFactorization(A, z) (proj/src/filterop.cpp:9-32): complex LU of z I - A,
    factored once at construction into an owned device factor (fl_node);
    solve() runs only the triangular solves against it."""

    def __init__(self, A, z: complex, node_index: int = -1, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        self._dA = DeviceMatrix(A, self.ctx)
        self.z = complex(z)
        self.node_index = node_index
        self.handle = None
        h = C.c_void_p()
        # singular shifts throw here, as the reference constructor does
        _call(L.lib().fl_node_create, self.ctx.handle, self._dA.handle, self.z.real, self.z.imag,
              int(node_index), C.byref(h))
        self.handle = h

    def shift(self):
        return self.z

    def solve(self, B) -> np.ndarray:
        B = np.asfortranarray(np.asarray(B, dtype=np.complex128))
        if B.ndim == 1:
            B = B.reshape(-1, 1, order="F")
        n, p = B.shape
        if n != self._dA.n:
            raise InvalidArgument("NodeFactorization::solve: dimension mismatch")
        W = np.zeros((n, p), dtype=np.complex128, order="F")
        _call(L.lib().fl_node_factor_solve, self.handle, _ptr(B), p, _ptr(W))
        return W

    def __del__(self):
        try:
            if self.handle:
                L.lib().fl_node_destroy(self.handle)
        except Exception:
            pass


def factorize_node(A, z: complex) -> NodeFactorization:
    return NodeFactorization(A, z)


class FilterApplier:
    """FilterApplier(A, rule, cache_factorizations) (proj/src/filterop.cpp:56-84)."""

    def __init__(self, A, rule: ContourRule, cache_factorizations: bool = False,
                 ctx: Context | None = None, device_matrix: DeviceMatrix | None = None):
        self.ctx = ctx or default_context()
        self._dA = device_matrix if device_matrix is not None else DeviceMatrix(A, self.ctx)
        self.rule = rule
        self.n = self._dA.n
        zr, zi, wr, wi = rule.parts()
        h = C.c_void_p()
        _call(L.lib().fl_filter_create, self.ctx.handle, self._dA.handle, rule.num_points(),
              _ptr(zr), _ptr(zi), _ptr(wr), _ptr(wi), int(bool(cache_factorizations)),
              C.byref(h))
        self.handle = h

    def apply(self, X, accounting: SolveAccounting | None = None, out=None) -> np.ndarray:
        X = _f64(X)
        if X.ndim == 1:
            X = X.reshape(-1, 1, order="F")
        if X.shape[0] != self.n:
            raise InvalidArgument(f"apply_filter: block dimension {X.shape[0]} != matrix "
                                  f"dimension {self.n}")
        if X.shape[1] < 1:
            raise InvalidArgument("apply_filter: block must have p >= 1")
        acc = accounting if accounting is not None else SolveAccounting()
        rhs = C.c_longlong(acc.rhs_solved)
        facts = C.c_longlong(acc.factorizations)
        Y = out if out is not None else np.zeros(X.shape, order="F")
        if Y.shape != X.shape or not Y.flags.f_contiguous or Y.dtype != np.float64:
            raise InvalidArgument("apply: out must be a Fortran-ordered float64 array like X")
        _call(L.lib().fl_filter_apply_raw, self.handle, _ptr(X), X.shape[0], X.shape[1], _ptr(Y),
              Y.shape[0], L.FL_HOST, C.byref(rhs), C.byref(facts))
        acc.rhs_solved, acc.factorizations = rhs.value, facts.value
        return Y

    def apply_device(self, x_ptr: int, ldx: int, p: int, y_ptr: int, ldy: int,
                     accounting: SolveAccounting | None = None) -> None:
        """Y = rho(A) X on device buffers (torch tensors' data_ptr), ordered on ctx.stream."""
        acc = accounting if accounting is not None else SolveAccounting()
        rhs = C.c_longlong(acc.rhs_solved)
        facts = C.c_longlong(acc.factorizations)
        _call(L.lib().fl_filter_apply_raw, self.handle, C.c_void_p(x_ptr), ldx, p,
              C.c_void_p(y_ptr), ldy, L.FL_DEVICE, C.byref(rhs), C.byref(facts))
        acc.rhs_solved, acc.factorizations = rhs.value, facts.value

    def __del__(self):
        try:
            if self.handle:
                L.lib().fl_filter_destroy(self.handle)
        except Exception:
            pass


def apply_filter(A, rule: ContourRule, X, accounting: SolveAccounting | None = None, *,
                 cache: bool = False, napply: int = 1):
    """apply_filter (proj/src/filterop.cpp:50-54): one-shot uncached applier.
    cache/napply: apply `napply` times through one FilterApplier(cache) and
    return the last result (exercises the factor cache, filterop.cpp:68-73)."""
    acc = accounting if accounting is not None else SolveAccounting()
    f = FilterApplier(A, rule, cache)
    Y = None
    for _ in range(napply):
        Y = f.apply(X, acc)
    return Y


def node_solve(A, z: complex, B) -> np.ndarray:
    """factorize_node(A, z).solve(B) (proj/src/filterop.cpp:26-36)."""
    return factorize_node(A, z).solve(B)


# ------------------------------------------------------------------ ritz
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
    if X.ndim != 2 or X.shape[0] < 1 or X.shape[1] < 1:
        raise InvalidArgument("orthonormalize: empty block")
    n, p = X.shape
    ctx = default_context()
    dX = DeviceBlock(n, p, ctx).set(X)
    dU = DeviceBlock(n, p, ctx)
    rank = C.c_int()
    _call(L.lib().fl_orthonormalize, ctx.handle, dX.handle, drop_tol, 1 if method == "qr" else 0,
          dU.handle, C.byref(rank))
    return dU.get(), rank.value


def rayleigh_ritz(A, X, interval: SearchInterval) -> RitzSet:
    S = _as_sym(A)
    X = _f64(X)
    if X.shape[0] != S.dim():
        raise InvalidArgument("rayleigh_ritz: block/matrix dimension mismatch")
    p = X.shape[1]
    if p < 1:
        raise InvalidArgument("rayleigh_ritz: empty block")
    ctx = default_context()
    dA = DeviceMatrix(S, ctx)
    dX = DeviceBlock(S.dim(), p, ctx).set(X)
    dV = DeviceBlock(S.dim(), p, ctx)
    vals = np.zeros(p)
    norms = np.zeros(p)
    inside = np.zeros(p, dtype=np.uint8)
    _call(L.lib().fl_rayleigh_ritz, ctx.handle, dA.handle, dX.handle, interval.lo, interval.hi,
          _ptr(vals), dV.handle, _ptr(norms), _ptr(inside))
    return RitzSet(vals, dV.get(), norms, inside.astype(bool))


def compute_residual_block(A, ritz: RitzSet) -> np.ndarray:
    S = _as_sym(A)
    ctx = default_context()
    dA = DeviceMatrix(S, ctx)
    V = _f64(ritz.vectors)
    dV = DeviceBlock(S.dim(), V.shape[1], ctx).set(V)
    dR = DeviceBlock(S.dim(), V.shape[1], ctx)
    vals = np.ascontiguousarray(ritz.values, dtype=np.float64)
    _call(L.lib().fl_residual_block, ctx.handle, dA.handle, dV.handle, _ptr(vals), dR.handle)
    return dR.get()


def select_indices(ritz: RitzSet, target_count: int, interval: SearchInterval):
    p = ritz.size()
    vals = np.ascontiguousarray(ritz.values, dtype=np.float64)
    norms = np.ascontiguousarray(ritz.residual_norms, dtype=np.float64)
    inside = np.ascontiguousarray(ritz.inside_flags, dtype=np.uint8)
    chosen = np.zeros(max(p, 1), dtype=np.int32)
    nch = C.c_int()
    _call(L.lib().fl_select_pairs, _ptr(vals), _ptr(norms), _ptr(inside), p, target_count,
          interval.lo, interval.hi, _ptr(chosen), C.byref(nch))
    return chosen[: nch.value].copy()


def select_pairs(ritz: RitzSet, target_count: int, interval: SearchInterval) -> RitzSet:
    idx = select_indices(ritz, target_count, interval)
    return RitzSet(ritz.values[idx], np.asfortranarray(ritz.vectors[:, idx]),
                   ritz.residual_norms[idx], np.asarray(ritz.inside_flags)[idx])


def count_inside(ritz: RitzSet) -> int:
    return int(np.count_nonzero(ritz.inside_flags))


def sym_eig(M):
    """Device symmetric eigensolve (SelfAdjointEigenSolver stand-in), ascending."""
    M = _f64(M)
    p = M.shape[0]
    vals = np.zeros(p)
    V = np.zeros((p, p), order="F")
    ctx = default_context()
    _call(L.lib().fl_sym_eig, ctx.handle, _ptr(M), p, p, _ptr(vals), _ptr(V), p)
    return vals, V


# ------------------------------------------------------------------ drivers
@dataclass
class SolverConfig:
    """proj/include/feastlab/drivers.hpp:12-24 (same fields and defaults)."""
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
    _call(L.lib().fl_make_initial_guess, default_context().handle, n, m0, seed, _ptr(X))
    return X


def _solve(variant, A, interval, cfg: SolverConfig, keep_first=False, ctx=None) -> Solution:
    S = _as_sym(A)
    M = S.mat()
    n = S.dim()
    ctx = ctx or default_context()
    c = L.SolverConfigC(cfg.m0, cfg.n_c, cfg.s, cfg.tol, cfg.max_iter, cfg.seed,
                        1 if cfg.orthogonalizer == "qr" else 0, cfg.drop_tol,
                        int(cfg.cache_factorizations), int(cfg.generalized_reduced))
    m0 = max(cfg.m0, 1)
    vals = np.zeros(m0)
    norms = np.zeros(m0)
    V = np.zeros((n, m0), order="F")
    first = np.zeros((n, m0), order="F") if keep_first else None
    m, conv, iters, rec, ntrace = C.c_int(), C.c_int(), C.c_int(), C.c_int(), C.c_int()
    rhs, facts = C.c_longlong(), C.c_longlong()
    trace = (L.TraceC * max(cfg.max_iter, 1))()
    _call(L.lib().fl_solve, ctx.handle, variant, _ptr(M), n, n, interval.lo, interval.hi,
          C.byref(c), _ptr(vals), _ptr(V), _ptr(norms), C.byref(m), C.byref(conv),
          C.byref(iters), C.byref(rhs), C.byref(facts), C.byref(rec), trace, C.byref(ntrace),
          _ptr(first) if keep_first else None)
    k = m.value
    tr = [TraceRecord(t.iter, t.subspace_dim, t.rhs_cumulative, t.max_residual, t.m_found)
          for t in trace[: ntrace.value]]
    vec = np.asfortranarray(V.reshape(-1, order="F")[: n * k].reshape(n, k, order="F"))
    return Solution(vals[:k].copy(), vec, norms[:k].copy(), bool(conv.value), iters.value,
                    SolveAccounting(rhs.value, facts.value), tr, rec.value, first)


def feast_solve(A, interval, cfg, **kw) -> Solution:
    return _solve(0, A, interval, cfg, **kw)


def xfeast_solve(A, interval, cfg, **kw) -> Solution:
    return _solve(1, A, interval, cfg, **kw)


def rfeast_solve(A, interval, cfg, **kw) -> Solution:
    return _solve(2, A, interval, cfg, **kw)


def solve_many(A, jobs, devices=(0,), per_device: int = 4):
    """Independent solves on one matrix run concurrently (the
    CLI's compare cells, feastlab_cli.cpp:245-294): jobs = [(variant, interval,
    cfg)], variant in {"feast", "xfeast", "rfeast"}; `per_device` worker
    contexts per GPU. Returns per job a dict with eigenvalues, converged,
    iterations, max_residual and error (None, or the failed job's message)."""
    S = _as_sym(A)
    M = S.mat()
    n = S.dim()
    nj = len(jobs)
    names = {"feast": 0, "xfeast": 1, "rfeast": 2}
    var = np.array([names[j[0]] for j in jobs], dtype=np.int32)
    lo = np.array([j[1].lo for j in jobs], dtype=np.float64)
    hi = np.array([j[1].hi for j in jobs], dtype=np.float64)
    cfgs = (L.SolverConfigC * max(nj, 1))()
    for k, (_, _, cfg) in enumerate(jobs):
        cfgs[k] = L.SolverConfigC(cfg.m0, cfg.n_c, cfg.s, cfg.tol, cfg.max_iter, cfg.seed,
                                  1 if cfg.orthogonalizer == "qr" else 0, cfg.drop_tol,
                                  int(cfg.cache_factorizations), int(cfg.generalized_reduced))
    ldv = max([max(j[2].m0, 1) for j in jobs] + [1])
    vals = np.zeros((max(nj, 1), ldv))
    m = np.zeros(max(nj, 1), dtype=np.int32)
    conv = np.zeros_like(m)
    iters = np.zeros_like(m)
    res = np.zeros(max(nj, 1))
    status = np.zeros_like(m)
    errs = C.create_string_buffer(256 * max(nj, 1))
    devs = np.array(list(devices), dtype=np.int32)
    _call(L.lib().fl_solve_many, _ptr(devs), len(devs), int(per_device), _ptr(M), n, n, nj,
          _ptr(var), _ptr(lo), _ptr(hi), cfgs, _ptr(vals), ldv, _ptr(m), _ptr(conv), _ptr(iters),
          _ptr(res), _ptr(status), errs)
    out = []
    for k in range(nj):
        err = errs.raw[256 * k: 256 * (k + 1)].split(b"\0", 1)[0].decode(errors="replace")
        out.append({"eigenvalues": vals[k, : m[k]].copy(), "converged": bool(conv[k]),
                    "iterations": int(iters[k]), "max_residual": float(res[k]),
                    "error": err if status[k] else None})
    return out


def write_trace_csv(trace) -> str:
    """proj/src/drivers.cpp:13-21 ("%d,%d,%lld,%.17g,%d")."""
    rows = ["iter,subspace_dim,rhs_cumulative,max_residual,m_found\n"]
    rows += ["%d,%d,%d,%.17g,%d\n" % (t.iter, t.subspace_dim, t.rhs_cumulative, t.max_residual,
                                       t.m_found) for t in trace]
    return "".join(rows)


def gaussian_block(rows: int, cols: int, seed: int) -> np.ndarray:
    """mt19937_64(seed) + normal_distribution, column-major fill (fixtures)."""
    out = np.zeros((rows, cols), order="F")
    L.lib().fl_gaussian_fill(_ptr(out), rows * cols, seed)
    return out


def seeded_orthogonal(n: int, seed: int, ctx: "Context | None" = None) -> np.ndarray:
    """The orthogonal factor of generate_spectrum (proj/src/matmodel.cpp:93-105)
    on the device: blocked Householder QR of the seeded Gaussian block (host
    fill: a sequential mt19937_64 stream), Q = H_1 ... H_n I, columns
    sign-normalised."""
    ctx = ctx or default_context()
    G = gaussian_block(n, n, seed)
    Q = np.zeros((n, n), order="F")
    _call(L.lib().fl_fixture_orthogonal, ctx.handle, _ptr(G), n, L.FL_HOST, _ptr(Q), L.FL_HOST)
    return Q


def assemble_matrix(values, Q, ctx: "Context | None" = None) -> np.ndarray:
    """assemble_matrix (proj/src/matmodel.cpp:109-118) on the device:
    0.5 (M + M^T) with M = Q diag(values) Q^T."""
    ctx = ctx or default_context()
    values = np.ascontiguousarray(values, dtype=np.float64)
    Q = np.asfortranarray(Q, dtype=np.float64)
    n = len(values)
    if Q.shape != (n, n):
        raise ValueError("assemble_matrix: inconsistent decomposition")
    A = np.zeros((n, n), order="F")
    _call(L.lib().fl_fixture_assemble, ctx.handle, _ptr(Q), L.FL_HOST, _ptr(values), n, _ptr(A),
          L.FL_HOST)
    return A


def device_test_matrix(values, seed: int, out_ptr: int, ctx: "Context | None" = None) -> None:
    """The seeded dense test matrix A = Q diag(values) Q^T of the BASELINE
    configurations, built on the device into the n x n buffer at `out_ptr`
    (device memory, ld n): Gaussian fill on the host, QR / Q / assembly by the
    library's kernels (bench.py, large-n tests)."""
    ctx = ctx or default_context()
    values = np.ascontiguousarray(values, dtype=np.float64)
    n = len(values)
    G = gaussian_block(n, n, seed)
    _call(L.lib().fl_fixture_orthogonal, ctx.handle, _ptr(G), n, L.FL_HOST, C.c_void_p(out_ptr),
          L.FL_DEVICE)
    del G
    _call(L.lib().fl_fixture_assemble, ctx.handle, C.c_void_p(out_ptr), L.FL_DEVICE, _ptr(values), n,
          C.c_void_p(out_ptr), L.FL_DEVICE)


def uniform_values(count: int, lo: float, hi: float, seed: int) -> np.ndarray:
    out = np.zeros(count)
    L.lib().fl_uniform_fill(_ptr(out), count, lo, hi, seed)
    return out
