"""Device fixture generation against the oracle's
seeded_orthogonal / assemble_matrix (proj/src/matmodel.cpp:93-119): the same Q
(entrywise, after the sign normalisation) and the same test matrix."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [1, 7, 64, 100, 200, 1000])
def test_seeded_orthogonal_matches_oracle(n):
    import paper_1605_08771_b200 as P
    Q = P.seeded_orthogonal(n, 1000 + n)
    Qo = O.seeded_orthogonal(n, 1000 + n)
    assert np.abs(Q.T @ Q - np.eye(n)).max() <= 1e-13 * max(n, 10)
    # sign rule: the largest-magnitude entry of every column is positive
    imax = np.abs(Q).argmax(axis=0)
    assert np.all(Q[imax, np.arange(n)] > 0)
    assert np.abs(Q - Qo).max() <= 1e-11, np.abs(Q - Qo).max()


def test_assemble_matrix_matches_oracle():
    import paper_1605_08771_b200 as P
    n = 300
    Qo = O.seeded_orthogonal(n, 5)
    vals = np.sort(O.uniform_fill(n, -1.0, 1.0, 9))
    A = P.assemble_matrix(vals, Qo)
    Ao = O.assemble_matrix(vals, Qo)
    assert np.array_equal(A, A.T)
    assert np.abs(A - Ao).max() <= 1e-13


def test_device_test_matrix_spectrum():
    """The bench workload builder: A on the device from the seeded Gaussian
    block; its eigenvalues are the prescribed ones."""
    import torch
    import paper_1605_08771_b200 as P
    n = 500
    vals = np.sort(P.uniform_values(n, -1.0, 1.0, 2004))
    A = torch.empty((n, n), dtype=torch.float64, device="cuda")
    P.device_test_matrix(vals, 1004, A.data_ptr())
    Ah = A.cpu().numpy()
    assert np.abs(Ah - Ah.T).max() == 0.0
    w = np.linalg.eigvalsh(Ah)
    assert np.abs(w - vals).max() <= 1e-12
    Ao = O.assemble_matrix(vals, O.seeded_orthogonal(n, 1004))
    assert np.abs(Ah - Ao).max() <= 1e-11
