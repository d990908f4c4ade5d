import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: longer parity runs")


@pytest.fixture(scope="session")
def ref():
    """Backend over the UNMODIFIED reference (oracle/_ref/libsfref.so)."""
    from tests import oracle_backends

    be = oracle_backends.reference()
    if be is None:
        pytest.skip("oracle/_ref/libsfref.so not built (reference sources absent on this host)")
    return be


@pytest.fixture(scope="session")
def oracle():
    """The checker for GPU parity: the reference build when present, else the C restatement
    (bit-exact to it, tests/test_oracle_cpu.py). Both are test infrastructure only."""
    from tests import oracle_backends

    be = oracle_backends.reference() or oracle_backends.port()
    if be is None:
        pytest.fail("no oracle library: run `make oracle`")
    return be


@pytest.fixture(scope="session")
def port():
    """Backend over the C restatement (oracle/liboracle.so)."""
    from tests import oracle_backends

    be = oracle_backends.port()
    if be is None:
        pytest.skip("oracle/liboracle.so not built")
    return be


@pytest.fixture(scope="session")
def gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1311_7194_b200 import default_backend

    return default_backend()
