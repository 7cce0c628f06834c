import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running oracle/GPU case")


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.lib()
    return oracle


@pytest.fixture(params=["oracle", pytest.param("b200", marks=pytest.mark.gpu)])
def F(request):
    """The implementation under test: the CPU oracle (pins the restatement
    against the reference's own assertions) or the B200 path."""
    if request.param == "oracle":
        import oracle
        oracle.lib()
        return oracle
    import paper_1605_08771_b200 as P
    P._lib.lib()
    return P
