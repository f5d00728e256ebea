"""Pins the 3D restatement of the oracle (oracle/ref3d_faces.hpp,
ref3d_viscous.hpp, ref3d_step.hpp) against the UNMODIFIED reference, on the
CPU: a 2D case extruded over nz = 7 planes with dz = 1, w = 0 and data
constant in z must step exactly as the reference's own 2D Simulation does,
plane for plane (SURVEY §8c's z-extrusion argument, applied to the checker
itself).  Every edge rule, LODI, chemistry, the laser, TENO6 / WENO3Z, char /
comp and a skewed mesh — the reference's glibc arithmetic on both sides, so
the planes agree bitwise up to the sign of exact zeros the z terms add."""
import numpy as np
import pytest

from paper_2202_02319_b200 import Simulation, configs
from tests.parity import clone_cfg

CASES = {
    "tgv_char_teno6_visc": (lambda: configs.tgv2d(16), 4),
    "tgv_comp_weno3z_visc": (lambda: configs.tgv2d(16, scheme="weno3z", split="comp"), 4),
    "tgv_skew_char_teno6": (lambda: configs.tgv2d(16, skew=0.2), 3),
    "ch4_react_laser": (lambda: configs.reacting_ch4(16), 4),
    "wall_isothermal": (lambda: configs.wall_channel(16), 4),
    "h2o2_inflow_outflow_laser": (lambda: configs.h2o2_counterflow(16), 3),
    "sod_lodi_outflow": (lambda: configs.sod_strip(60), 6),
}
NZ = 7


def same_values(a, b):
    """Bitwise equality except +0 == -0."""
    return a.shape == b.shape and bool(np.all(a == b))


def prim3_of(cache2, ns, nz, g=3):
    """2D cache (rho, u, v, p, T, c, Y) -> the 3D planes (rho, u, v, w = 0, p, T, c,
    Y) replicated over nz + 2g z planes."""
    rows = [cache2["rho"], cache2["u"], cache2["v"], np.zeros_like(cache2["u"]),
            cache2["p"], cache2["T"], cache2["c"]] + [cache2["Y"][s] for s in range(ns)]
    return np.stack([np.broadcast_to(r, (nz + 2 * g,) + r.shape) for r in rows]).copy()


@pytest.mark.parametrize("name", sorted(CASES))
def test_ref3d_steps_reduce_to_the_reference_2d(name, oracle_api):
    from oracle import ref
    mk, n = CASES[name]
    case = mk()
    refs = Simulation(clone_cfg(case.cfg), oracle_api)
    try:
        refs.set_initial_condition(case.ic)
        refs.prepare_stage(1)
        ns = refs.ns
        U3 = configs.state_2d_to_3d(refs.Ut, ns, NZ)
        P3 = prim3_of(refs.cache(), ns, NZ)
        t0 = refs.time
        U_init = refs.Ut
        case3 = configs.extrude_z(case, NZ)
        refs.rk3_steps(case.dt, n)
        U3n, P3n = ref.steps3(case3.cfg, U3, P3, case.dt, n, t0=t0)
        U2, c2 = refs.Ut, refs.cache()
        for k in range(3, 3 + NZ):
            assert same_values(configs.state_3d_to_2d(U3n, ns, k), U2), (name, k)
            assert same_values(P3n[5, k], c2["T"]), (name, k)
            assert not np.any(U3n[ns + 2, k])  # w stays exactly 0
        assert np.abs(U2 - U_init).max() > 0.0  # the steps moved the state
    finally:
        refs.close()
