"""Test configuration. `-m gpu` tests need a B200 (they are the parity tests
proper, through the C ABI); everything else runs on CPU."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (large configs)")


def _ensure_built():
    lib = os.path.join(ROOT, "paper_0803_1975_b200", "_lib", "libqgemm_b200.so")
    if not os.path.exists(lib):
        import subprocess

        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_0803_1975_b200")], check=True)


_ensure_built()


@pytest.fixture(scope="session")
def qg():
    import paper_0803_1975_b200 as qg

    return qg


@pytest.fixture(scope="session")
def orc():
    import oracle

    return oracle


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu test run without a CUDA device")
    return torch.device("cuda:0")
