"""Shared fixtures.  `-m gpu` tests need a CUDA device (B200); everything else
runs on CPU.  The oracle libraries (oracle/) are test infrastructure only."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


@pytest.fixture(scope="session")
def moe():
    import paper_2407_14417_b200 as m
    m.lib()
    return m


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import OracleLib
    return OracleLib()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import REF_SO, RefLib
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return RefLib()


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")
