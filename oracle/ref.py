"""TEST INFRASTRUCTURE ONLY — the CPU checker, never the product.

Loads oracle/_ref/libignis_ref.so (the unmodified reference headers compiled
by oracle/build_ref.sh) and binds it to the same ``Simulation`` wrapper as the
B200 library.  Only tests/, __graft_entry__.smoke() and bench.py's CPU legs
import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

from paper_2202_02319_b200 import abi
from paper_2202_02319_b200.sim import Simulation

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_ref", "libignis_ref.so")
_api = None
_lib = None


def build():
    subprocess.run(["bash", os.path.join(HERE, "build_ref.sh")], check=True)


def available() -> bool:
    return os.path.exists(LIB)


def api() -> dict:
    global _api, _lib
    if _api is None:
        if not os.path.exists(LIB):
            raise FileNotFoundError(f"oracle library missing: {LIB} (run oracle/build_ref.sh)")
        _lib = C.CDLL(LIB, mode=C.RTLD_LOCAL)
        _api = abi.bind(_lib, "ignref_")
        _lib.ignref_set_partitions.argtypes = [C.c_void_p, C.c_int]
        _lib.ignref_set_partitions.restype = C.c_int
        for n in ("write_snapshot", "read_snapshot"):
            f = getattr(_lib, "ignref_" + n)
            f.argtypes = [C.c_void_p, C.c_char_p]
            f.restype = C.c_int
    return _api


def lib():
    api()
    return _lib


def simulation(cfg: abi.Config, partitions: int = 1) -> Simulation:
    cfg.partitions = partitions
    return Simulation(cfg, api())


def set_partitions(sim: Simulation, n: int):
    lib().ignref_set_partitions(sim.handle, n)
