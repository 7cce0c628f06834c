"""ctypes binding of the in-tree C ABI library (include/feastlab_b200.h).

Loads paper_1605_08771_b200/lib/libfeastlab_b200.so (built by
__graft_entry__.build(), `make -C paper_1605_08771_b200/csrc`). There is no
fallback: a missing library raises ImportError, a missing GPU raises
FeastCudaError from the first call that needs the device.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# FEASTLAB_LIB: an alternative build of the same library (A/B kernel experiments)
LIB_PATH = os.environ.get("FEASTLAB_LIB") or os.path.join(HERE, "lib", "libfeastlab_b200.so")

FL_OK, FL_INVALID_ARGUMENT, FL_RUNTIME_ERROR, FL_CHOLESKY, FL_SINGULAR_NODE, FL_CUDA, FL_NCCL, \
    FL_OOM, FL_MATRIX_MARKET, FL_NOT_SYMMETRIC = range(10)
FL_HOST, FL_DEVICE = 0, 1
FL_REDUCE_SUM, FL_REDUCE_ORDERED = 0, 1

_lib = None


class Err(C.Structure):
    _fields_ = [("status", C.c_int), ("index", C.c_int), ("pivot", C.c_double),
                ("z_re", C.c_double), ("z_im", C.c_double), ("msg", C.c_char * 512)]


class SolverConfigC(C.Structure):
    _fields_ = [("m0", C.c_int), ("n_c", C.c_int), ("s", C.c_int), ("tol", C.c_double),
                ("max_iter", C.c_int), ("seed", C.c_uint64), ("orthogonalizer", C.c_int),
                ("drop_tol", C.c_double), ("cache_factorizations", C.c_int),
                ("generalized_reduced", C.c_int)]


class TraceC(C.Structure):
    _fields_ = [("iter", C.c_int), ("subspace_dim", C.c_int), ("rhs_cumulative", C.c_longlong),
                ("max_residual", C.c_double), ("m_found", C.c_int)]


_P, _I, _D, _LL, _U64 = C.c_void_p, C.c_int, C.c_double, C.c_longlong, C.c_uint64
_PP = C.POINTER(C.c_void_p)

_SIGS = {
    "fl_version": (_I, []),
    "fl_device_count": (_I, [_P]),
    "fl_ctx_create": (_I, [_I, _PP, _P]),
    "fl_ctx_create_nccl": (_I, [_I, _P, _I, _I, _PP, _P]),
    "fl_nccl_unique_id": (_I, [_P, _P]),
    "fl_ctx_create_virtual": (_I, [_I, _I, _I, _PP, _P]),
    "fl_node_shard": (_I, [_I, _I, _I, _P, _P]),
    "fl_ctx_destroy": (_I, [_P]),
    "fl_ctx_sync": (_I, [_P, _P]),
    "fl_ctx_stream": (_P, [_P]),
    "fl_ctx_rank": (_I, [_P, _P, _P]),
    "fl_ctx_launches": (_LL, [_P]),
    "fl_ctx_set_profiling": (_I, [_P, _I]),
    "fl_ctx_set_streams": (_I, [_P, _I]),
    "fl_debug_panel_profile": (_I, [_P, _I]),
    "fl_debug_panel_trace": (_I, [_P, _I]),
    "fl_mm_read": (_I, [C.c_char_p, _P, _P, _I, _P]),
    "fl_mm_write": (_I, [C.c_char_p, _P, _I, _I, _I, _P]),
    "fl_ctx_profile_dump": (_I, [_P, _P, _I]),
    "fl_debug_zgemm": (_I, [_P, _I, _I, _I, _I, _I, _P, _P]),
    "fl_debug_zgemm_lu": (_I, [_P, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P]),
    "fl_debug_factor_tilesums": (_I, [_P, _I, _P]),
    "fl_fixture_orthogonal": (_I, [_P, _P, _I, _I, _P, _I, _P]),
    "fl_fixture_assemble": (_I, [_P, _P, _I, _P, _I, _P, _I, _P]),
    "fl_debug_decision_log": (_I, [_I]),
    "fl_zgemm_mode": (_I, [_I]),
    "fl_solve_many": (_I, [_P, _I, _I, _P, _I, _I, _I, _P, _P, _P, _P, _P, _I, _P, _P, _P, _P, _P,
                           _P, _P]),
    "fl_ctx_set_reduction": (_I, [_P, _I]),
    "fl_ctx_set_factorization": (_I, [_P, _I]),
    "fl_ctx_factorization": (_I, [_P]),
    "fl_ctx_profile": (_I, [_P, C.c_char_p, _P, _P, _P, _P]),
    "fl_matrix_create": (_I, [_P, _P, _I, _I, _I, _PP, _P]),
    "fl_matrix_destroy": (_I, [_P]),
    "fl_matrix_dim": (_I, [_P]),
    "fl_block_create": (_I, [_P, _I, _I, _PP, _P]),
    "fl_block_destroy": (_I, [_P]),
    "fl_block_cols": (_I, [_P]),
    "fl_block_rows": (_I, [_P]),
    "fl_block_set": (_I, [_P, _P, _I, _I, _I, _P]),
    "fl_block_get": (_I, [_P, _P, _I, _I, _P]),
    "fl_block_gather": (_I, [_P, _P, _P, _I, _P]),
    "fl_block_append": (_I, [_P, _P, _P]),
    "fl_block_copy": (_I, [_P, _P, _P]),
    "fl_filter_create": (_I, [_P, _P, _I, _P, _P, _P, _P, _I, _PP, _P]),
    "fl_filter_destroy": (_I, [_P]),
    "fl_filter_apply": (_I, [_P, _P, _P, _P, _P, _P]),
    "fl_filter_apply_raw": (_I, [_P, _P, _I, _I, _P, _I, _I, _P, _P, _P]),
    "fl_orthonormalize": (_I, [_P, _P, _D, _I, _P, _P, _P]),
    "fl_rayleigh_ritz": (_I, [_P, _P, _P, _D, _D, _P, _P, _P, _P, _P]),
    "fl_residual_block": (_I, [_P, _P, _P, _P, _P, _P]),
    "fl_block_rank": (_I, [_P, _P, _D, _P, _P]),
    "fl_sym_eig": (_I, [_P, _P, _I, _I, _P, _P, _I, _P]),
    "fl_node_solve": (_I, [_P, _P, _D, _D, _P, _I, _P, _P]),
    "fl_node_create": (_I, [_P, _P, _D, _D, _I, _PP, _P]),
    "fl_node_factor_solve": (_I, [_P, _P, _I, _P, _P]),
    "fl_node_destroy": (_I, [_P]),
    "fl_solve": (_I, [_P, _I, _P, _I, _I, _D, _D, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                      _P, _P]),
    "fl_gauss_legendre": (_I, [_I, _P, _P, _P]),
    "fl_build_contour_rule": (_I, [_D, _D, _I, _P, _P, _P, _P, _P]),
    "fl_filter_value": (_D, [_I, _P, _P, _P, _P, _D]),
    "fl_symmetric_matrix": (_I, [_P, _I, _I, _D, _P, _P]),
    "fl_make_initial_guess": (_I, [_P, _I, _I, _U64, _P, _P]),
    "fl_select_pairs": (_I, [_P, _P, _P, _I, _I, _D, _D, _P, _P, _P]),
    "fl_gaussian_fill": (None, [_P, _LL, _U64]),
    "fl_uniform_fill": (None, [_P, _LL, _D, _D, _U64]),
}


def exported_symbols():
    return sorted(_SIGS)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                "(the B200 path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def source_digest() -> str:
    """sha256 over the library's sources (csrc/**, the public headers): ties a
    committed profile capture to the code it ran (the built .so is not
    bit-reproducible across builds, so its own hash cannot)."""
    import hashlib
    here = os.path.dirname(os.path.abspath(__file__))
    roots = [os.path.join(here, "csrc"), os.path.join(os.path.dirname(here), "include")]
    files = []
    for r in roots:
        for d, _, names in os.walk(r):
            files += [os.path.join(d, n) for n in names
                      if n.endswith((".cu", ".cuh", ".hpp", ".h", ".cpp")) or n == "Makefile"]
    h = hashlib.sha256()
    for f in sorted(files):
        h.update(os.path.relpath(f, os.path.dirname(here)).encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()
