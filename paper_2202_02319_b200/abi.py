"""ctypes mirror of include/ignis_b200.h (the C-ABI boundary).

The structures below are field-for-field restatements of the header; the
library's ``ign_config_size()`` is checked against ``ctypes.sizeof`` at load
time so a drift between the two fails loudly.
"""
from __future__ import annotations

import ctypes as C

IGN_ABI_VERSION = 3
IGN_MAX_SPECIES = 8
IGN_MAX_COMP = 11
IGN_MAX_PIECES = 4
IGN_MAX_SEGMENTS = 4
IGN_NAME_LEN = 16

# ign_status (errors.hpp:10-47)
IGN_OK = 0
IGN_CONFIG_ERROR = 1
IGN_STATE_ERROR = 2
IGN_NUMERICS_ERROR = 3
IGN_STEP_FAILURE = 4
IGN_FORMAT_ERROR = 5
IGN_USAGE_ERROR = 6
IGN_CUDA_ERROR = 7
IGN_INTERNAL_ERROR = 8

# enums (reconstruction.hpp:12-18, boundary.hpp:16-22, metrics.hpp:21, laser.hpp:12)
WENO3Z, TENO6 = 0, 1
COMPONENTWISE, CHARACTERISTIC = 0, 1
METRICS_SCHEME, METRICS_ANALYTIC_SKEW, METRICS_CENTRAL2 = 0, 1, 2
PERIODIC, NOSLIP_ISOTHERMAL, NOSLIP_ADIABATIC, INFLOW, OUTFLOW = 0, 1, 2, 3, 4
MM_AUTO, MM_CENTRAL2, MM_ORDER4, MM_ORDER6, MM_ANALYTIC_SKEW = -1, 0, 1, 2, 3
CALORICALLY_PERFECT, MULTI_SPECIES = 0, 1
LASER_GAUSSIAN, LASER_SHAPED = 0, 1
DIAG_DEVICE, DIAG_REFERENCE = 0, 1  # ign_set_diagnostics


class ThermoPiece(C.Structure):
    _fields_ = [(n, C.c_double) for n in
                ("t_lo", "t_hi", "cm2", "cm1", "c0", "c1", "c2", "c3", "c4", "b")]


class Species(C.Structure):
    _fields_ = [("name", C.c_char * IGN_NAME_LEN),
                ("W", C.c_double), ("mu_ref", C.c_double), ("t_ref", C.c_double),
                ("n_exp", C.c_double),
                ("npieces", C.c_int32), ("_pad", C.c_int32),
                ("pieces", ThermoPiece * IGN_MAX_PIECES)]


class Mixture(C.Structure):
    _fields_ = [("mode", C.c_int32), ("ns", C.c_int32),
                ("R", C.c_double), ("Le", C.c_double), ("Pr", C.c_double),
                ("species", Species * IGN_MAX_SPECIES)]


class Scheme(C.Structure):
    _fields_ = [("scheme", C.c_int32), ("split", C.c_int32),
                ("teno_ct", C.c_double), ("eps", C.c_double), ("cfl", C.c_double),
                ("metrics", C.c_int32), ("_pad", C.c_int32)]


class InflowSegment(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("lo", "hi", "u", "v", "T")] + \
               [("Y", C.c_double * IGN_MAX_SPECIES)]


class Edge(C.Structure):
    _fields_ = [("type", C.c_int32), ("nseg", C.c_int32), ("T_wall", C.c_double),
                ("seg", InflowSegment * IGN_MAX_SEGMENTS),
                ("smooth_width", C.c_double), ("p_target", C.c_double),
                ("sigma_out", C.c_double)]


class BC(C.Structure):
    _fields_ = [("left", Edge), ("right", Edge), ("bottom", Edge), ("top", Edge)]


class Mechanism(C.Structure):
    _fields_ = [("present", C.c_int32), ("i_fuel", C.c_int32), ("i_ox", C.c_int32),
                ("i_co2", C.c_int32), ("i_h2o", C.c_int32), ("_pad", C.c_int32),
                ("A", C.c_double), ("Ta", C.c_double), ("a", C.c_double),
                ("b", C.c_double), ("T_cutoff", C.c_double),
                ("nu", C.c_double * IGN_MAX_SPECIES)]


class Laser(C.Structure):
    _fields_ = [("present", C.c_int32), ("kernel", C.c_int32)] + \
               [(n, C.c_double) for n in
                ("energy", "sigma_r", "sigma_t", "x0", "y0", "t0", "edot_rate",
                 "lobe_sep", "width_up", "width_down", "amp_down", "width_radial")] + \
               [("z0", C.c_double), ("zmode", C.c_int32), ("_pad", C.c_int32)]


class Integrator(C.Structure):
    _fields_ = [("fixed_dt", C.c_double), ("t_end", C.c_double),
                ("max_iter", C.c_int64), ("chem_dt_limit", C.c_int32),
                ("_pad", C.c_int32), ("chem_dt_factor", C.c_double)]


class Config(C.Structure):
    _fields_ = [("abi_version", C.c_int32), ("nx", C.c_int32), ("ny", C.c_int32),
                ("g", C.c_int32),
                ("lx", C.c_double), ("ly", C.c_double),
                ("center_x", C.c_double), ("center_y", C.c_double),
                ("periodic_x", C.c_int32), ("periodic_y", C.c_int32),
                ("apply_skew", C.c_int32), ("metric_mode", C.c_int32),
                ("skew_beta", C.c_double),
                ("mix", Mixture), ("scheme", Scheme), ("bc", BC),
                ("mech", Mechanism), ("laser", Laser),
                ("viscous", C.c_int32), ("partitions", C.c_int32),
                ("integ", Integrator),
                ("device", C.c_int32), ("slab_count", C.c_int32),
                ("slab_rank", C.c_int32), ("nz", C.c_int32), ("periodic_z", C.c_int32),
                ("_pad", C.c_int32), ("lz", C.c_double), ("center_z", C.c_double),
                ("mesh_x", C.POINTER(C.c_double)), ("mesh_y", C.POINTER(C.c_double)),
                ("zlo", Edge), ("zhi", Edge)]


class Error(C.Structure):
    _fields_ = [("status", C.c_int32), ("stage", C.c_int32), ("i", C.c_int32),
                ("j", C.c_int32), ("k", C.c_int32), ("msg", C.c_char * 256)]


class PrimPoint(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("rho", "u", "v", "p", "T")] + \
               [("Y", C.c_double * IGN_MAX_SPECIES)]


IC_FN = C.CFUNCTYPE(None, C.c_double, C.c_double, C.c_void_p, C.POINTER(PrimPoint))
STEP_HOOK = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p)

_P = C.c_void_p
_D = C.POINTER(C.c_double)
_I = C.c_int
_I32P = C.POINTER(C.c_int32)

# name -> (restype, argtypes); identical for ign_ (product) and ignref_ (oracle)
SIGNATURES = {
    "config_size": (C.c_uint64, []),
    "create": (_I, [C.POINTER(Config), C.POINTER(_P)]),
    "destroy": (None, [_P]),
    "last_error": (_I, [_P, C.POINTER(Error)]),
    "dims": (_I, [_P, _I32P, _I32P, _I32P, _I32P]),
    "get_mesh": (_I, [_P, _D, _D]),
    "get_metrics": (_I, [_P, _I, _D]),
    "set_initial_condition": (_I, [_P, IC_FN, _P]),
    "set_initial_primitives": (_I, [_P, _D]),
    "set_state": (_I, [_P, _D, _D]),
    "get_state": (_I, [_P, _D]),
    "get_cache": (_I, [_P, _D]),
    "get_time": (_I, [_P, _D, C.POINTER(C.c_int64)]),
    "set_time": (_I, [_P, C.c_double, C.c_int64]),
    "set_integrator": (_I, [_P, C.POINTER(Integrator)]),
    "refill_ghosts": (_I, [_P]),
    "refresh_primitives": (_I, [_P, _I]),
    "prepare_stage": (_I, [_P, _I]),
    "compute_rhs": (_I, [_P, C.c_double, _I, _D]),
    "stable_dt": (_I, [_P, _D]),
    "rk3_step": (_I, [_P, C.c_double]),
    "rk3_steps": (_I, [_P, C.c_double, C.c_int64]),
    "advance": (_I, [_P, STEP_HOOK, _P]),
    "conserved_totals": (_I, [_P, _D]),
    "product_mole_fraction": (_I, [_P, _D]),
    "last_clip": (_I, [_P, _D]),
    "set_diagnostics": (_I, [_P, C.c_int]),
    "host_metrics": (_I, [C.POINTER(Config), _I, _D, C.POINTER(Error)]),
    "host_mesh": (_I, [C.POINTER(Config), _D, _D, C.POINTER(Error)]),
    "kernel_launches": (C.c_int64, [_P]),
    # outputs: probes, trace, snapshots
    "add_probe": (_I, [_P, C.c_int32, C.c_int32, C.c_int32, C.c_int32]),
    "set_sampling": (_I, [_P, C.c_int32, C.c_int32]),
    "probe_samples": (_I, [_P, C.c_int32, C.POINTER(C.c_int64), _D, _D]),
    "trace_samples": (_I, [_P, C.POINTER(C.c_int64), _D, _D]),
    "set_config_hash": (_I, [_P, C.c_uint64]),
    "get_config_hash": (_I, [_P, C.POINTER(C.c_uint64)]),
    "write_snapshot": (_I, [_P, C.c_char_p]),
    "read_snapshot": (_I, [_P, C.c_char_p]),
}

# measurement entry points only the B200 library has (no oracle analogue)
PRODUCT_ONLY = {
    "profile_enable": (_I, [_P, _I]),
    "profile_read": (_I, [_P, _D, C.POINTER(C.c_int64)]),
    "stream_handle": (C.c_void_p, [_P]),
    "probe_fp64_peak": (_I, [_I, _D]),
    "guard_status": (_I, [C.POINTER(C.c_int), C.POINTER(C.c_ulonglong), C.POINTER(C.c_ulonglong)]),
    "guard_selftest": (_I, [_I, C.POINTER(C.c_ulonglong)]),
    "dims3": (_I, [_P, _I32P, _I32P, _I32P]),
    # multi-GPU slabs
    "nccl_unique_id": (_I, [C.c_char_p]),
    "attach_nccl": (_I, [_P, C.c_char_p, _I, _I]),
    "group_create": (_I, [C.POINTER(_P), _I, C.POINTER(_P)]),
    "group_destroy": (None, [_P]),
    "group_last_error": (_I, [_P, C.POINTER(Error)]),
    "group_prepare_stage": (_I, [_P, _I]),
    "group_rk3_steps": (_I, [_P, C.c_double, C.c_int64]),
    "group_stable_dt": (_I, [_P, _D]),
    "group_conserved_totals": (_I, [_P, _D]),
    "group_advance": (_I, [_P]),
    "group_write_snapshot": (_I, [_P, C.c_char_p, _I, _I]),
    "group_read_snapshot": (_I, [_P, C.c_char_p]),
    "write_snapshot_v2": (_I, [_P, C.c_char_p, _I]),
    "add_probe3": (_I, [_P] + [C.c_int32] * 6),
    "ensemble_rk3_steps": (_I, [C.POINTER(_P), _I, _D, C.c_int64, C.POINTER(C.c_int)]),
}
IGN_NCCL_ID_BYTES = 128
PROF_CLASSES = ("bc", "prim", "faces", "visc", "assemble", "dt", "r6", "r7")

# entry points of include/ignis_b200.h that every product build must export
PUBLIC_SYMBOLS = sorted(set(SIGNATURES) | set(PRODUCT_ONLY))


def bind(lib: C.CDLL, prefix: str) -> dict:
    """Returns {name: bound function} for every ABI entry point."""
    out = {}
    sigs = dict(SIGNATURES)
    if prefix == "ign_":
        sigs.update(PRODUCT_ONLY)
    for name, (res, args) in sigs.items():
        fn = getattr(lib, prefix + name)
        fn.restype = res
        fn.argtypes = args
        out[name] = fn
    got = out["config_size"]()
    if got != C.sizeof(Config):
        raise RuntimeError(f"ABI drift: {prefix}config_size()={got} but "
                           f"ctypes Config is {C.sizeof(Config)} bytes")
    return out
