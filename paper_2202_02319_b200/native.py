"""Loader of the in-tree C-ABI library (paper_2202_02319_b200/_lib/libignis_b200.so).

There is no CPU fallback: if the library is missing the import of the product
path fails loudly (build it with ``python -c "import __graft_entry__ as g; g.build()"``
or ``make -C paper_2202_02319_b200/csrc``).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

from . import abi

PKG = os.path.dirname(os.path.abspath(__file__))
LIB = os.environ.get("IGN_LIB") or os.path.join(PKG, "_lib", "libignis_b200.so")
_lib = None
_api = None


def build(jobs: int = 8) -> str:
    subprocess.run(["make", "-C", os.path.join(PKG, "csrc"), f"-j{jobs}"], check=True)
    return LIB


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise ImportError(
                f"B200 library not built: {LIB} is missing (run make -C {PKG}/csrc); "
                "there is no CPU fallback")
        _lib = C.CDLL(LIB, mode=C.RTLD_LOCAL)
    return _lib


def api() -> dict:
    global _api
    if _api is None:
        _api = abi.bind(lib(), "ign_")
    return _api
