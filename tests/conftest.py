import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REFERENCE_INCLUDE = "/root/reference/proj/include"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def has_reference_sources() -> bool:
    return os.path.exists(os.path.join(REFERENCE_INCLUDE, "ignis", "solver.hpp"))


@pytest.fixture(scope="session")
def oracle_api():
    """The CPU oracle: the unmodified reference compiled by oracle/build_ref.sh."""
    from oracle import ref
    if not ref.available():
        if not has_reference_sources():
            pytest.skip("oracle library not built and reference sources absent")
        ref.build()
    return ref.api()


@pytest.fixture(scope="session")
def product_api():
    from paper_2202_02319_b200 import native
    return native.api()


@pytest.fixture(scope="session")
def cuda_device():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return 0
