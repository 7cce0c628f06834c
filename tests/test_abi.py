"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports
every symbol include/feastlab_b200.h declares, host-side entry points work
without a GPU, and compute entry points fail loudly (no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    text = open(os.path.join(ROOT, "include", "feastlab_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|double|long long|void\*)\s+(fl_\w+)\s*\(",
                                 text, re.M)))


def test_header_symbols_exported():
    from paper_1605_08771_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = _declared()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert sorted(_lib.exported_symbols()) == names


def test_library_is_sm100a():
    from paper_1605_08771_b200 import _lib
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True)
    assert "sm_100a" in out.stdout


def test_host_entry_points_match_oracle():
    import oracle as O
    import paper_1605_08771_b200 as P
    for n in (1, 2, 3, 8, 16, 32, 64):
        x1, w1 = P.gauss_legendre(n)
        x2, w2 = O.gauss_legendre(n)
        assert np.array_equal(x1, x2) and np.array_equal(w1, w2)
    for lo, hi, nc in [(-0.1, 0.1, 8), (-0.3, 0.2, 16), (-0.02, 0.02, 32), (0, 4, 2)]:
        r1 = P.build_contour_rule(P.SearchInterval(lo, hi), nc)
        r2 = O.build_contour_rule(O.SearchInterval(lo, hi), nc)
        assert np.array_equal(r1.nodes, r2.nodes) and np.array_equal(r1.weights, r2.weights)
        for lam in (0.0, 0.05, 1.0, -3.0):
            assert P.filter_value(r1, lam) == O.filter_value(r2, lam)
    M = O.random_symmetric(7, 3)
    assert np.array_equal(P.SymmetricMatrix(M).mat(), O.symmetric_matrix(M))
    with pytest.raises(P.InvalidArgument):
        P.SymmetricMatrix(np.array([[1.0, 2.0], [3.0, 4.0]]))
    assert np.array_equal(P.gaussian_block(5, 3, 9), O.gaussian_block(5, 3, 9))
    assert np.array_equal(P.uniform_values(10, -1, 1, 4), O.uniform_fill(10, -1, 1, 4))


def test_select_pairs_host_logic_matches_oracle():
    import oracle as O
    import paper_1605_08771_b200 as P
    rng = np.random.default_rng(5)
    I = P.SearchInterval(-1, 1)
    for trial in range(50):
        p = int(rng.integers(1, 30))
        vals = rng.uniform(-3, 3, p)
        res = rng.choice([1e-3, 1e-5, 2e-4], p)  # many exact ties
        if trial % 3 == 0:
            vals = np.round(vals, 1)  # ties in |lambda - c| too
        flags = np.array([I.contains(v) for v in vals])
        rs = P.RitzSet(vals, np.eye(p), res, flags)
        m0 = int(rng.integers(1, p + 2))
        a = P.select_indices(rs, m0, I)
        b = O.select_indices(O.RitzSet(vals, np.eye(p), res, flags), m0, O.SearchInterval(-1, 1))
        assert list(a) == list(b)


def test_compute_entry_fails_loudly_without_gpu():
    import paper_1605_08771_b200 as P
    if P.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(P.FeastCudaError):
        P.apply_filter(np.eye(4), P.build_contour_rule(P.SearchInterval(-1, 1), 2), np.ones((4, 1)))


def test_library_then_torch_import_order():
    """Loading the library before torch must not pin an NCCL older than the
    one torch needs (the library links torch's NCCL when it is installed)."""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, %r); import paper_1605_08771_b200; import torch; "
            "print('ok')" % ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-2000:]
