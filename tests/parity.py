"""Parity helpers shared by the GPU tests (TEST INFRASTRUCTURE).

Normalisation follows SURVEY.md §8(c): per field, max|a-b| / scale with scale
= max rho (species partial densities), max |rho u| over both momenta, max |E|.
"""
from __future__ import annotations

import copy
import ctypes as C

import numpy as np

from paper_2202_02319_b200 import Simulation, abi


def clone_cfg(cfg: abi.Config) -> abi.Config:
    out = abi.Config()
    C.memmove(C.byref(out), C.byref(cfg), C.sizeof(abi.Config))
    return out


def make_pair(case, oracle_api, partitions: int = 1):
    """(product, oracle) simulations on identical configs and initial state."""
    cfg_p = clone_cfg(case.cfg)
    cfg_r = clone_cfg(case.cfg)
    cfg_r.partitions = partitions
    prod = Simulation(cfg_p)
    refs = Simulation(cfg_r, oracle_api)
    refs.set_initial_condition(case.ic)
    prod.set_state(refs.Ut)  # identical bits, no dependence on host IC code
    return prod, refs


def interior(a: np.ndarray, g: int = 3) -> np.ndarray:
    return a[..., g:-g, g:-g]


def field_errors(a: np.ndarray, b: np.ndarray, ns: int, g: int = 3) -> np.ndarray:
    """Normalised per-component max errors over the interior."""
    a = interior(a, g)
    b = interior(b, g)
    d = np.abs(a - b).reshape(a.shape[0], -1).max(axis=1)
    rho_scale = np.abs(b[:ns].sum(axis=0)).max()
    mom_scale = np.sqrt(b[ns] ** 2 + b[ns + 1] ** 2).max()
    e_scale = np.abs(b[ns + 2]).max()
    scale = np.array([rho_scale] * ns + [mom_scale, mom_scale, e_scale])
    scale = np.where(scale > 0, scale, 1.0)
    return d / scale


def bitwise_equal(a: np.ndarray, b: np.ndarray) -> bool:
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def ulp_diff(a: np.ndarray, b: np.ndarray) -> int:
    ai = np.ascontiguousarray(a).view(np.int64)
    bi = np.ascontiguousarray(b).view(np.int64)
    return int(np.abs(ai - bi).max()) if ai.size else 0
