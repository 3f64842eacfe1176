"""Shared fixtures.  `-m gpu` tests need a B200 and the built libsssp_cuda.so;
`-m "not gpu"` tests run on CPU only (oracle, host logic, ABI surface, gloo)."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def oracle_c():
    import oracle
    return oracle.C()


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not oracle.ref_available():
        pytest.skip("reference build (oracle/_ref) unavailable")
    return oracle.REF()


@pytest.fixture(scope="session")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2504_03667_b200 as P
    return P
