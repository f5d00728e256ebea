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


def inviscid_rhs3(cfg: abi.Config, Ut, prim):
    """The 3D extension's inviscid RHS from oracle/ref3d_faces.hpp (the
    reference's per-face algorithm restated with the z terms) for a padded 3D
    state and the product's primitive cache; interior of the returned planes
    written, ghosts 0."""
    import numpy as np
    f = lib().ignref3d_inviscid_rhs
    f.argtypes = [C.POINTER(abi.Config), C.c_void_p, C.c_void_p, C.c_void_p,
                  C.POINTER(abi.Error)]
    f.restype = C.c_int
    Ut = np.ascontiguousarray(Ut, dtype=np.float64)
    prim = np.ascontiguousarray(prim, dtype=np.float64)
    out = np.zeros_like(Ut)
    err = abi.Error()
    st = f(C.byref(cfg), Ut.ctypes.data, prim.ctypes.data, out.ctypes.data, C.byref(err))
    if st != abi.IGN_OK:
        raise RuntimeError(f"ref3d: status {st}: {err.msg.decode()}")
    return out


def viscous_rhs3(cfg: abi.Config, prim):
    """The 3D extension's viscous divergence (dVx + dVy) + dVz from
    oracle/ref3d_viscous.hpp (the reference's compute_viscous restated with the
    z terms) for the product's primitive cache; interior written, ghosts 0."""
    import numpy as np
    f = lib().ignref3d_viscous_rhs
    f.argtypes = [C.POINTER(abi.Config), C.c_void_p, C.c_void_p, C.POINTER(abi.Error)]
    f.restype = C.c_int
    prim = np.ascontiguousarray(prim, dtype=np.float64)
    nc = cfg.mix.ns + 4
    out = np.zeros((nc,) + prim.shape[1:], dtype=np.float64)
    err = abi.Error()
    st = f(C.byref(cfg), prim.ctypes.data, out.ctypes.data, C.byref(err))
    if st != abi.IGN_OK:
        raise RuntimeError(f"ref3d: status {st}: {err.msg.decode()}")
    return out


def steps3(cfg: abi.Config, Ut, prim, dt: float, n: int, t0: float = 0.0):
    """n advance() steps of the 3D extension on a fully periodic box from
    oracle/ref3d_step.hpp (the reference's rk3_step / post_stage /
    prepare_stage restated with the z terms); returns (Ut, prim) after them."""
    import numpy as np
    f = lib().ignref3d_steps
    f.argtypes = [C.POINTER(abi.Config), C.c_void_p, C.c_void_p, C.c_double, C.c_double,
                  C.c_int, C.POINTER(abi.Error)]
    f.restype = C.c_int
    Ut = np.array(Ut, dtype=np.float64, order="C", copy=True)
    prim = np.array(prim, dtype=np.float64, order="C", copy=True)
    err = abi.Error()
    st = f(C.byref(cfg), Ut.ctypes.data, prim.ctypes.data, t0, dt, n, C.byref(err))
    if st != abi.IGN_OK:
        raise RuntimeError(f"ref3d: status {st}: {err.msg.decode()}")
    return Ut, prim
