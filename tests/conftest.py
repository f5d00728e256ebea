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


def guard_status(api):
    """(enabled, buffers checked, canary words overwritten) of the red-zone
    guard (IGN_GUARD=1; runtime.cu dmalloc/dfree)."""
    import ctypes as C
    en, chk, bad = C.c_int(), C.c_ulonglong(), C.c_ulonglong()
    st = api["guard_status"](C.byref(en), C.byref(chk), C.byref(bad))
    assert st == 0, st
    return en.value, chk.value, bad.value


def pytest_sessionfinish(session, exitstatus):
    """Under IGN_GUARD=1 the whole session is a memory-safety run: fail it if
    any device buffer's red zone was overwritten."""
    if not os.environ.get("IGN_GUARD"):
        return
    from paper_2202_02319_b200 import native
    if native._lib is None:  # the library never loaded (CPU-only session)
        return
    en, chk, bad = guard_status(native.api())
    msg = f"ignis_b200 guard: enabled={en} buffers_checked={chk} corrupted_words={bad}"
    print("\n" + msg)
    out = os.environ.get("IGN_GUARD_REPORT")
    if out:
        with open(out, "w") as f:
            f.write(msg + "\n")
    if bad:
        session.exitstatus = 1
