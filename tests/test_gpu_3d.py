"""3D extension (BASELINE configs[1], TGV 256^3) against the 2D oracle.

The reference is 2D-only, so the 3D path is anchored on the
z-extrusion cross-check of SURVEY §8c:

  * (x, y) extrusion: a 2D case on nz = 7 planes with dz = 1.0, w = 0 and
    z-constant data.  Every z plane must reproduce the 2D oracle: bitwise (up
    to the sign of zero) for the gamma-gas cases, within the 2D multi-species
    tolerances otherwise — and bitwise equal to the 2D B200 path in all cases.
  * (x, z) extrusion: a 2D case laid in the x-z plane (v = 0, y-constant,
    dy = 1) exercises the zeta-face kernel and, for the wall channels, the
    z-edge rules (the 2D y walls / outflow become z walls / outflow); equal to
    the 2D oracle within a tolerance (the 2D oracle's y metrics carry ulp
    noise the uniform z metrics do not).
  * The non-periodic x / y edges (walls, inflow, outflow with LODI) and the
    laser run the reference's 2D rules on every z plane: the same extrusion
    check covers them (wall, counterflow, Sod/LODI cases).
  * 3D TGV: periodic conservation of mass, momenta and energy.
"""
import ctypes as C

import numpy as np
import pytest

from paper_2202_02319_b200 import Simulation, abi, configs
from tests.parity import clone_cfg, field_errors

pytestmark = pytest.mark.gpu

RHS_TOL = 1e-13
STEP_TOL = 1e-10
XZ_TOL = 1e-11

# name -> (2D builder, exact vs oracle, nsteps)
EXTRUDE = {
    "tgv_char_teno6_visc": (lambda: configs.tgv2d(24), True, 8),
    "tgv_comp_teno6_inviscid": (lambda: configs.tgv2d(24, split="comp", viscous=False), False, 8),
    "tgv_char_weno3z_visc": (lambda: configs.tgv2d(20, scheme="weno3z"), True, 8),
    "tgv_comp_weno3z_visc": (lambda: configs.tgv2d(20, scheme="weno3z", split="comp"), False, 8),
    "tgv_skew_char_teno6": (lambda: configs.tgv2d(24, skew=0.2), True, 6),
    # nx + 1 >= 32 NC: the x-face kernel's flattened-row mode (segments straddle rows)
    "tgv_wide_flat_x_teno6": (lambda: configs.tgv2d(168), True, 3),
    "ch4_react_char": (lambda: configs.reacting_ch4(20, laser=False), False, 8),
    "ch4_react_comp_weno3z": (lambda: configs.reacting_ch4(20, scheme="weno3z", split="comp",
                                                          laser=False), False, 8),
    # the reference's non-periodic edges on every z plane
    "ch4_react_laser": (lambda: configs.reacting_ch4(20), False, 8),
    "wall_isothermal": (lambda: configs.wall_channel(20), False, 6),
    "wall_adiabatic_weno3z": (lambda: configs.wall_channel(20, isothermal=False,
                                                           scheme="weno3z"), False, 6),
    "h2o2_inflow_outflow_laser": (lambda: configs.h2o2_counterflow(24), False, 6),
    "sod_lodi_outflow": (lambda: configs.sod_strip(120), False, 12),
}

NZ = 7


def same_values(a, b):
    """Bitwise equality except +0 == -0 (z terms add exact zeros)."""
    return a.shape == b.shape and bool(np.all((a == b) | (np.isnan(a) & np.isnan(b))))


def planes(U3, ns, g=3):
    """The nz interior z planes of a 3D component array, in 2D component order."""
    return [configs.state_3d_to_2d(U3, ns, k) for k in range(g, U3.shape[1] - g)]


@pytest.fixture(params=sorted(EXTRUDE))
def triple(request, oracle_api, cuda_device):
    mk, exact, n = EXTRUDE[request.param]
    case = mk()
    refs = Simulation(clone_cfg(case.cfg), oracle_api)
    refs.set_initial_condition(case.ic)
    prod2 = Simulation(clone_cfg(case.cfg))
    prod2.set_state(refs.Ut)
    case3 = configs.extrude_z(case, NZ)
    prod3 = Simulation(clone_cfg(case3.cfg))
    assert prod3.nz == NZ and prod3.nc == prod2.nc + 1
    prod3.set_state(configs.state_2d_to_3d(refs.Ut, refs.ns, NZ))
    yield case, refs, prod2, prod3, exact, n
    for s in (refs, prod2, prod3):
        s.close()


def test_extrusion_initial_condition(oracle_api, cuda_device):
    """set_initial_primitives' 3D conversion reduces to the 2D one (w = 0)."""
    for mk in (lambda: configs.tgv2d(16), lambda: configs.reacting_ch4(16, laser=False)):
        case = mk()
        refs = Simulation(clone_cfg(case.cfg), oracle_api)
        refs.set_initial_condition(case.ic)
        case3 = configs.extrude_z(case, NZ)
        p3 = Simulation(clone_cfg(case3.cfg))
        p3.set_initial_condition(case3.ic)
        U3 = p3.Ut
        for pl in planes(U3, refs.ns):
            assert same_values(pl[..., 3:-3, 3:-3], refs.Ut[..., 3:-3, 3:-3])
        assert not np.any(U3[refs.ns + 2])


def test_extrusion_prepare_stage(triple):
    case, refs, prod2, prod3, exact, n = triple
    for s in (refs, prod3):
        s.prepare_stage(1)
    a, b = prod3.cache(), refs.cache()
    g = 3
    for k in ("rho", "u", "v", "p", "T", "c"):
        for kz in range(g, g + NZ):
            assert same_values(a[k][kz], b[k]), k
    assert not np.any(a["w"])
    for pl in planes(prod3.Ut, refs.ns):
        assert same_values(pl, refs.Ut)  # (x, y) ghosts filled identically


def test_extrusion_rhs(triple):
    case, refs, prod2, prod3, exact, n = triple
    for s in (refs, prod2, prod3):
        s.prepare_stage(1)
    t = 0.37 * case.dt
    r3 = prod3.compute_rhs(t, 1)
    r2 = prod2.compute_rhs(t, 1)
    rr = refs.compute_rhs(t, 1)
    g = 3
    assert not np.any(r3[refs.ns + 2, g:-g, g:-g, g:-g])  # d(rho w)/dt == 0
    for pl in planes(r3, refs.ns):
        pi, p2 = pl[..., g:-g, g:-g], r2[..., g:-g, g:-g]
        assert same_values(pi, p2)
        if exact:
            assert same_values(pi, rr[..., g:-g, g:-g])
        else:
            assert field_errors(pl, rr, refs.ns).max() <= RHS_TOL


def test_extrusion_steps(triple):
    case, refs, prod2, prod3, exact, n = triple
    for s in (refs, prod2, prod3):
        s.prepare_stage(1)
        s.rk3_steps(case.dt, n)
    assert prod3.iter == refs.iter == n and prod3.time == refs.time
    U3, U2, Ur = prod3.Ut, prod2.Ut, refs.Ut
    assert not np.any(U3[refs.ns + 2])
    for pl in planes(U3, refs.ns):
        assert same_values(pl, U2)
        if exact:
            assert same_values(pl, Ur)
        else:
            assert field_errors(pl, Ur, refs.ns).max() <= STEP_TOL
    # ±0 aside, the temperature cache (the Newton guess) carries over too
    T3 = prod3.cache()["T"]
    for kz in range(3, 3 + NZ):
        assert same_values(T3[kz], prod2.cache()["T"])


def test_extrusion_stable_dt_bounded(triple):
    """The 3D spectral radius adds the z term: dt3 <= dt2 (solver.hpp:370-383)."""
    case, refs, prod2, prod3, exact, n = triple
    for s in (refs, prod3):
        s.prepare_stage(1)
    d3, d2 = prod3.stable_dt(), refs.stable_dt()
    assert 0.0 < d3 <= d2


# ----------------------------------------------------------------- x-z plane
def _xz_pair(oracle_api, case2):
    """A 2D case laid in the (x, z) plane of a 3D box: ny = 7 cells of dy = 1
    (configs.lay_xz; the 2D y edges become the z edges)."""
    refs = Simulation(clone_cfg(case2.cfg), oracle_api)
    refs.set_initial_condition(case2.ic)
    c3 = configs.lay_xz(case2, NZ)
    p3 = Simulation(c3.cfg)
    p3.set_initial_condition(c3.ic)
    return refs, p3


def _xz_to_2d(U3, ns, j):
    """3D [.., rho u, rho v, rho w, E](z, y, x) at y index j -> 2D (y := z)."""
    return np.concatenate([U3[: ns + 1, :, j], U3[ns + 2: ns + 4, :, j]])


def _state_scale(U, ns, g=3):
    b = U[..., g:-g, g:-g]
    rho = np.abs(b[:ns].sum(axis=0)).max()
    mom = np.sqrt(b[ns] ** 2 + b[ns + 1] ** 2).max()
    return np.array([rho] * ns + [mom, mom, np.abs(b[ns + 2]).max()])


def _wall_outflow():
    """wall_channel with a zero-gradient outflow top edge (boundary.hpp:242-249)."""
    case = configs.wall_channel(20)
    case.cfg.bc.top.type = abi.OUTFLOW
    return case


@pytest.mark.parametrize("mk", [
    lambda: configs.tgv2d(24),
    lambda: configs.tgv2d(20, scheme="weno3z", split="comp"),
    lambda: configs.reacting_ch4(16, laser=False),
    # the 2D y walls as z walls (isothermal back, adiabatic front)
    lambda: configs.wall_channel(20),
    lambda: configs.wall_channel(20, isothermal=False, scheme="weno3z", split="comp"),
    lambda: _wall_outflow(),
], ids=["tgv_char_teno6", "tgv_comp_weno3z", "ch4_char", "zwalls_isothermal",
        "zwalls_adiabatic_weno3z", "zwall_zoutflow"])
def test_xz_plane_matches_oracle(mk, oracle_api, cuda_device):
    case = mk()
    refs, p3 = _xz_pair(oracle_api, case)
    ns, g = refs.ns, 3
    for s in (refs, p3):
        s.prepare_stage(1)
    t = 0.25 * case.dt
    r3, rr = p3.compute_rhs(t, 1), refs.compute_rhs(t, 1)
    # d(rho v)/dt vanishes up to the ulp noise of the y metrics' cross terms
    # (m_xi_y, m_eta_x ~ 1e-17) times the pressure flux: scale by the energy
    p_scale = np.abs(p3.Ut[ns + 3]).max()
    assert np.abs(r3[ns + 1, g:-g, g:-g, g:-g]).max() <= 1e-13 * p_scale
    # the TGV starts near equilibrium, so its RHS is a small residual of large
    # fluxes: measure the RHS difference as a one-step state increment (x dt)
    # against the state's own scale
    Ur0 = refs.Ut
    for j in range(g, g + NZ):
        d = np.abs(_xz_to_2d(r3, ns, j) - rr)[..., g:-g, g:-g]
        d = d.reshape(d.shape[0], -1).max(axis=1) * case.dt
        assert (d / _state_scale(Ur0, ns)).max() <= 1e-13
    for s in (refs, p3):
        s.rk3_steps(case.dt, 5)
    U3, Ur = p3.Ut, refs.Ut
    for j in range(g, g + NZ):
        assert field_errors(_xz_to_2d(U3, ns, j), Ur, ns).max() <= XZ_TOL


# ----------------------------------------------------------------- 3D TGV
def test_tgv3d_conservation(cuda_device):
    """Config B at 32^3: periodic totals of mass, momenta, energy conserved."""
    case = configs.tgv3d(32)
    sim = Simulation(case.cfg)
    sim.set_initial_condition(case.ic)
    sim.prepare_stage(1)
    tot0 = sim.conserved_totals()
    sim.rk3_steps(case.dt, 10)
    tot1 = sim.conserved_totals()
    assert sim.iter == 10
    # mass scale rho0 V also bounds the momenta (|u| <= 1)
    scale = np.array([tot0[0]] * 4 + [abs(tot0[4])])
    assert np.all(np.abs(tot1 - tot0) <= 1e-12 * scale), (tot0, tot1)


def _field3(X, Y, Z, p0):
    """A generic smooth fully-3D state (no symmetry of its own)."""
    rho = 1 + 0.1 * np.sin(X + 2 * Y) * np.cos(3 * Z + 0.3)
    u = np.sin(X) * np.cos(Y) * np.cos(Z) + 0.1 * np.sin(2 * Z + Y)
    v = -np.cos(X) * np.sin(Y) * np.cos(Z) + 0.05 * np.cos(X - Z)
    w = 0.2 * np.sin(Y + 2 * X) * np.cos(Z)
    p = p0 + 0.3 * np.cos(2 * X + Z) * np.sin(Y)
    return rho, u, v, w, p


@pytest.mark.parametrize("scheme,split", [("teno6", "char"), ("teno6", "comp"),
                                          ("weno3z", "comp")])
def test_axis_permutation_invariance(scheme, split, cuda_device):
    """On the cube, relabelling the axes (y <-> z, x <-> z; velocity components
    with them) commutes with the RHS: checks the eta/zeta face kernels, the 3D
    viscous terms and the assembly against each other on a fully 3D state.
    Equal to rounding (the 2D metrics carry ulp noise the z metrics do not)."""
    case = configs.tgv3d(16, scheme=scheme, split=split)
    p0 = case.notes["p0"]
    res = {}
    for perm in ("id", "yz", "xz"):
        def ic(X, Y, Z, perm=perm):
            if perm == "id":
                rho, u, v, w, p = _field3(X, Y, Z, p0)
            elif perm == "yz":
                rho, u, w, v, p = _field3(X, Z, Y, p0)
            else:
                rho, w, v, u, p = _field3(Z, Y, X, p0)
            return rho, u, v, w, p / rho, [np.ones_like(X)]
        sim = Simulation(clone_cfg(case.cfg))
        sim.set_initial_condition(ic)
        sim.prepare_stage(1)
        r = sim.compute_rhs(0.0, 1)
        sim.rk3_steps(case.dt, 3)
        res[perm] = (r, sim.Ut)
        sim.close()
    g = 3
    sl = (slice(None), slice(g, -g), slice(g, -g), slice(g, -g))
    r0, U0 = res["id"]
    for perm, idx, ax in (("yz", [0, 1, 3, 2, 4], 2), ("xz", [0, 3, 2, 1, 4], 3)):
        r, U = res[perm]
        rp = np.swapaxes(r[idx], 1, ax)[sl]
        Up = np.swapaxes(U[idx], 1, ax)[sl]
        er = np.abs(rp - r0[sl]).reshape(5, -1).max(1) / np.abs(r0[sl]).reshape(5, -1).max(1)
        eU = np.abs(Up - U0[sl]).reshape(5, -1).max(1) / np.abs(U0[sl]).reshape(5, -1).max(1)
        assert er.max() <= 1e-11, (perm, er)
        assert eU.max() <= 1e-12, (perm, eU)


def test_jet3d_runs_and_develops_3d_structure(cuda_device):
    """configs[3] form: the jet case steps through the laser pulse with every
    edge rule active; the spanwise perturbation yields nonzero w everywhere."""
    case = configs.jet3d(64, 32, 8)
    sim = Simulation(case.cfg)
    sim.set_initial_condition(case.ic)
    sim.prepare_stage(1)
    assert 0.0 < case.dt <= sim.stable_dt()
    sim.rk3_steps(case.dt, 60)
    c = sim.cache()
    g = 3
    T = c["T"][g:-g, g:-g, g:-g]
    assert np.isfinite(T).all() and T.min() > 250.0
    assert np.abs(c["w"][g:-g, g:-g, g:-g]).max() > 0.0
    assert sim.iter == 60


def test_3d_state_failure_location(cuda_device):
    """A non-positive density in a 3D state raises StepFailure at prepare time
    with the node's (i, j, k) — k in ign_error.k and in the message (the
    reference's error kinds; its payload is (stage, i, j))."""
    from paper_2202_02319_b200 import errors
    case = configs.tgv3d(12)
    sim = Simulation(case.cfg)
    sim.set_initial_condition(case.ic)
    U = sim.Ut
    U[0, 3 + 4, 3 + 5, 3 + 6] = -1.0  # node (i=6, j=5, k=4)
    sim.set_state(U)
    with pytest.raises(errors.StepFailure) as ei:
        sim.prepare_stage(2)
    e = ei.value
    assert (e.stage, e.i, e.j, e.k) == (2, 6, 5, 4)
    assert "k=4" in str(e)


def test_3d_probes_match_2d_oracle_on_one_plane(oracle_api, cuda_device):
    """A 3D probe box on a single z plane of an extruded case samples exactly
    the 2D oracle's box means (rows gain w = 0); a full-depth box over z-slabs
    equals the undecomposed run's."""
    from paper_2202_02319_b200.sim import SlabGroup
    case = configs.tgv2d(24)
    refs = Simulation(clone_cfg(case.cfg), oracle_api)
    refs.set_initial_condition(case.ic)
    case3 = configs.extrude_z(case, NZ)
    p3 = Simulation(clone_cfg(case3.cfg))
    p3.set_state(configs.state_2d_to_3d(refs.Ut, refs.ns, NZ))
    boxes = [(0, 0, 23, 23), (3, 5, 9, 12)]
    for b in boxes:
        refs.add_probe(*b)
        p3.add_probe3(b[0], b[1], 2, b[2], b[3], 2)
    for s in (refs, p3):
        s.set_sampling(2, 0)
        s.set_integrator(fixed_dt=case.dt, t_end=4.5 * case.dt)
        s.advance()
    for k in range(len(boxes)):
        (ta, ra), (tb, rb) = p3.probe(k), refs.probe(k)
        assert np.array_equal(ta, tb)
        assert not np.any(ra[:, 3])  # w
        assert same_values(np.delete(ra, 3, axis=1), rb)
    # full-depth box over z-slabs vs the single domain
    c3 = configs.tgv3d(12, nz=18)
    single = Simulation(clone_cfg(c3.cfg))
    single.set_initial_condition(c3.ic)
    grp = SlabGroup(c3.cfg, 3)
    U0 = single.Ut
    for r in range(3):
        grp.set_state(r, U0[:, 6 * r:6 * r + 12])
    for s in (single, grp):
        s.lead_call("add_probe3", 1, 2, 0, 10, 9, 17) if s is grp else s.add_probe3(1, 2, 0, 10, 9, 17)
        s.set_sampling(1, 0)
        s.set_integrator(fixed_dt=c3.dt, t_end=2.5 * c3.dt)
        s.advance()
    (ta, ra), (tb, rb) = single.probe(0), grp.probe(0)
    assert np.array_equal(ta, tb) and np.array_equal(ra.view(np.uint64), rb.view(np.uint64))
    grp.close()


# ----------------------------------------------------------------- 3D laser
def _quiescent_laser_box(n, kernel, zmode):
    case = configs.tgv3d(n, viscous=False)
    la = case.cfg.laser
    la.present, la.kernel, la.zmode = 1, kernel, zmode
    la.energy, la.sigma_t, la.t0 = 3.0, 1e-3, 0.5
    la.sigma_r = 2.0 * (2.0 * np.pi / n)  # 2 cells: the domain spans +-6 sigma_r
    la.x0 = la.y0 = la.z0 = 0.0
    la.edot_rate = 7.0
    la.lobe_sep, la.width_up, la.width_down, la.amp_down = 0.5, 0.6, 0.25, 0.7
    la.width_radial = 0.4
    p0 = case.notes["p0"]

    def ic(X, Y, Z):
        one = np.ones_like(X)
        z = np.zeros_like(X)
        return one, z, z.copy(), z.copy(), p0 * one, [one]
    sim = Simulation(case.cfg)
    sim.set_initial_condition(ic)
    sim.prepare_stage(1)
    return case, sim


def test_laser3d_point_kernel_deposits_E(cuda_device):
    """zmode 1 Gaussian (laser_power3): at t0 the RHS of E integrates to
    E / (sqrt(2 pi) sigma_t) over the box (the 3D normalisation), the
    space-time integral of q_L being E (laser.hpp:53-61 with r^2 over x,y,z)."""
    case, sim = _quiescent_laser_box(24, abi.LASER_GAUSSIAN, 1)
    la = case.cfg.laser
    rhs = sim.compute_rhs(la.t0, 1)
    g = sim.g
    dE = rhs[-1][g:-g, g:-g, g:-g]
    want = la.energy / (np.sqrt(2.0 * np.pi) * la.sigma_t)
    # the +-6 sigma_r box truncates ~2 Phi(-6) of the Gaussian per axis (~6e-9)
    assert abs(dE.sum() - want) <= 1e-7 * want, (dE.sum(), want)
    # symmetric about the focus in every direction (node-centred grid about 0)
    assert np.allclose(dE, dE[::-1, :, :], rtol=1e-12, atol=1e-12 * dE.max())
    assert np.allclose(dE, np.swapaxes(dE, 0, 2), rtol=1e-12, atol=1e-12 * dE.max())


def test_laser3d_zmode0_is_the_2d_kernel_on_every_plane(cuda_device):
    """zmode 0 (default): the reference's 2D kernel, z-uniform; shaped kernel
    with zmode 1 decays in z about z0 with its radial width."""
    case, sim = _quiescent_laser_box(16, abi.LASER_SHAPED, 0)
    la = case.cfg.laser
    g = sim.g
    dE = sim.compute_rhs(la.t0, 1)[-1][g:-g, g:-g, g:-g]
    assert dE.max() > 0.0
    assert np.all(dE == dE[0][None])  # identical z planes
    case1, sim1 = _quiescent_laser_box(16, abi.LASER_SHAPED, 1)
    dE1 = sim1.compute_rhs(la.t0, 1)[-1][g:-g, g:-g, g:-g]
    kz = np.argmax(dE1.max(axis=(1, 2)))
    prof = dE1.max(axis=(1, 2))
    assert prof[kz] > 10.0 * prof[0] and np.allclose(prof, prof[::-1], rtol=1e-12)


# ------------------------------------------------- fully 3D faces vs ref3d
def _fully_3d(case, n_steps=3):
    """A state with w != 0 and genuine z variation, stepped a few times so the
    cache and ghosts come from the product's own prepare_stage."""
    ic0 = case.ic
    lz = case.cfg.lz

    def ic(X, Y, Z):
        rho, u, v, w, T, Ys = ic0(X, Y, Z)
        k = 2.0 * np.pi / lz
        w = w + 0.3 * np.abs(u).max() * np.sin(k * Z + 0.7) * np.cos(Y + 0.2 * X)
        T = T * (1.0 + 0.02 * np.cos(k * Z) * np.sin(X))
        return rho, u, v, w, T, Ys
    sim = Simulation(case.cfg)
    sim.set_initial_condition(ic)
    sim.prepare_stage(1)
    sim.rk3_steps(case.dt, n_steps)
    return sim


def _inviscid(cfg):
    c = clone_cfg(cfg)
    c.viscous = 0
    c.mech.present = 0
    c.laser.present = 0
    return c


FULL3D = {
    "tgv3d_char_teno6": lambda: configs.tgv3d(16, nz=14, viscous=False),
    # nx, ny not multiples of the 8-column y/z tiles, nz not of the 20-line
    # blocks: partial tiles in every direction
    "tgv3d_char_teno6_ragged": lambda: configs.tgv3d(18, nz=13, viscous=False),
    "tgv3d_comp_teno6": lambda: configs.tgv3d(16, nz=14, viscous=False, split="comp"),
    "tgv3d_char_weno3z": lambda: configs.tgv3d(16, nz=14, viscous=False, scheme="weno3z"),
    "tgv3d_comp_weno3z": lambda: configs.tgv3d(16, nz=14, viscous=False, scheme="weno3z",
                                               split="comp"),
}


def _species3d(split, scheme="teno6"):
    case = configs.extrude_z(configs.species_box(4, 16, scheme=scheme, split=split), 12)
    case.cfg.lz = 0.01 * 12 / 16  # dz = dx
    case.cfg.viscous = 0
    case.cfg.mech.present = 0
    case.cfg.laser.present = 0
    return case


FULL3D["h2o2_4sp_char_teno6"] = lambda: _species3d("char")
FULL3D["h2o2_4sp_comp_weno3z"] = lambda: _species3d("comp", "weno3z")


@pytest.mark.parametrize("name", sorted(FULL3D))
def test_full_3d_faces_bitwise_vs_ref3d(name, oracle_api, cuda_device):
    """All three face kernels (xi, eta and the zeta kernel k_faces3d<.,2,.>)
    on a genuinely 3D state against oracle/ref3d_faces.hpp — the reference's
    per-face algorithm restated in 3D, serial, with the reference's own
    recon/thermo functions — BITWISE (the z kernel had only an
    x-z plane 1e-11 check and self-consistency)."""
    from oracle import ref
    case = FULL3D[name]()
    case.cfg = _inviscid(case.cfg)
    sim = _fully_3d(case)
    Ut = sim.Ut
    names = ("rho", "u", "v", "w", "p", "T", "c")
    cache = sim.cache()
    prim = np.concatenate([np.stack([cache[k] for k in names]), cache["Y"]])
    got = sim.compute_rhs(0.0, 1)
    want = ref.inviscid_rhs3(case.cfg, Ut, prim)
    g = sim.g
    a, b = got[:, g:-g, g:-g, g:-g], want[:, g:-g, g:-g, g:-g]
    assert np.abs(b[-2]).max() > 0.0  # the z momentum moves
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), \
        np.abs(a - b).max(axis=(1, 2, 3))


# ---------------------------------------------- fully 3D viscous vs ref3d
def _viscous_only(cfg):
    c = clone_cfg(cfg)
    c.viscous = 1
    c.mech.present = 0
    c.laser.present = 0
    return c


def _species3d_visc():
    case = configs.extrude_z(configs.species_box(4, 16), 12)
    case.cfg.lz = 0.01 * 12 / 16  # dz = dx
    return case


def _skew3d_visc():
    case = configs.extrude_z(configs.tgv2d(16, skew=0.08), 12)
    case.cfg.lz = 2.0 * np.pi * 12 / 16  # dz = dx
    return case


VISC3D = {
    "tgv3d_visc": lambda: configs.tgv3d(16, nz=14),
    "tgv3d_visc_ragged": lambda: configs.tgv3d(18, nz=13),
    "tgv_skew_visc": _skew3d_visc,
    "h2o2_4sp_visc": _species3d_visc,
}


@pytest.mark.parametrize("name", sorted(VISC3D))
def test_full_3d_viscous_rhs_bitwise_vs_ref3d(name, oracle_api, cuda_device):
    """The viscous node kernel k_visc3 and the viscous part of the update
    (k_assemble3) on a genuinely 3D state (w != 0, z variation) against
    oracle/ref3d_viscous.hpp — the reference's compute_viscous restated with
    the z terms, serial, with the reference's own transport() / thermo — plus
    the ref3d inviscid RHS: the full RHS of BASELINE configs[1]'s viscous path
    BITWISE (until now anchored on z-extrusions and an x-z plane at 1e-11)."""
    from oracle import ref
    case = VISC3D[name]()
    case.cfg = _viscous_only(case.cfg)
    sim = _fully_3d(case)
    Ut = sim.Ut
    names = ("rho", "u", "v", "w", "p", "T", "c")
    cache = sim.cache()
    prim = np.concatenate([np.stack([cache[k] for k in names]), cache["Y"]])
    got = sim.compute_rhs(0.0, 1)
    inv = ref.inviscid_rhs3(case.cfg, Ut, prim)
    dv = ref.viscous_rhs3(case.cfg, prim)
    want = inv + dv  # r = -((dF + dG) + dH); r += (dVx + dVy) + dVz
    g = sim.g
    a, b = got[:, g:-g, g:-g, g:-g], want[:, g:-g, g:-g, g:-g]
    d = dv[:, g:-g, g:-g, g:-g]
    ns = case.cfg.mix.ns
    assert np.abs(d[ns + 2]).max() > 0.0  # z-momentum viscous flux moves
    assert np.abs(d[ns + 3]).max() > 0.0
    if ns == 1:
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), \
            np.abs(a - b).max(axis=(1, 2, 3))
    else:
        # Wilke's pow(T/T_ref, n) and pow(W_j/W_i, 1/4) (thermo.hpp:235-250)
        # are not correctly rounded on the device: last-ulp differences, the
        # 2D species cases' RHS gate (test_gpu_species.py RHS_TOL)
        scale = np.abs(b).max(axis=(1, 2, 3))
        err = np.abs(a - b).max(axis=(1, 2, 3)) / np.where(scale > 0, scale, 1.0)
        assert err.max() <= 1e-13, err


# ------------------------------------- fully 3D trajectories vs ref3d_step
def _duct3d(outflow=False):
    """The TGV box walled (configs[3]'s edge rules on fully 3D data): isothermal
    bottom / back walls, adiabatic top / front walls; outflow=True swaps x
    periodicity for a left outflow / right wall and the back wall for an
    outflow z edge (the right-edge outflow is LODI, not restated in ref3d)."""
    case = configs.tgv3d(16, nz=14)
    cfg = case.cfg
    T0 = float(np.mean(case.ic(np.zeros(4), np.zeros(4), np.zeros(4))[4]))
    cfg.periodic_y = 0
    cfg.periodic_z = 0
    cfg.bc.bottom.type = abi.NOSLIP_ISOTHERMAL
    cfg.bc.bottom.T_wall = 1.05 * T0
    cfg.bc.top.type = abi.NOSLIP_ADIABATIC
    cfg.zlo.type = abi.NOSLIP_ISOTHERMAL
    cfg.zlo.T_wall = 0.97 * T0
    cfg.zhi.type = abi.NOSLIP_ADIABATIC
    if outflow:
        cfg.periodic_x = 0
        cfg.bc.left.type = abi.OUTFLOW
        cfg.bc.right.type = abi.NOSLIP_ADIABATIC
        cfg.zlo.type = abi.OUTFLOW
    return case


def _wall4sp_zwalls():
    """configs' 4-species CH4/O2 wall channel extruded, z walls added
    (isothermal back at 900 K — the channel spans 300-900 K, so 2 T_w - T stays
    inside the thermo tables — adiabatic front)."""
    case = configs.extrude_z(configs.wall_channel(16), 12)
    case.cfg.lz = 0.01 * 12 / 16  # dz = dx
    case.cfg.periodic_z = 0
    case.cfg.zlo.type = abi.NOSLIP_ISOTHERMAL
    case.cfg.zlo.T_wall = 900.0
    case.cfg.zhi.type = abi.NOSLIP_ADIABATIC
    return case


STEPS3D = {
    "duct3d_walls": _duct3d,
    "wall4sp_zwalls": _wall4sp_zwalls,
    "duct3d_walls_outflow": lambda: _duct3d(outflow=True),
    "tgv3d_visc_char_teno6": lambda: configs.tgv3d(16, nz=14),
    "tgv3d_visc_ragged": lambda: configs.tgv3d(18, nz=13),
    "tgv3d_visc_comp_weno3z": lambda: configs.tgv3d(16, nz=14, scheme="weno3z", split="comp"),
    "tgv_skew_visc": _skew3d_visc,
    "h2o2_4sp_visc": _species3d_visc,
}


@pytest.mark.parametrize("name", sorted(STEPS3D))
def test_3d_steps_vs_ref3d(name, oracle_api, cuda_device):
    """Ten rk3_steps of the whole 3D path — ghost fill (x, y, z periodic
    edges), primitives with the T cache, the three face kernels, the viscous
    kernels, the fused update / clip — from a genuinely 3D state against
    oracle/ref3d_step.hpp, the reference's advance() loop body restated with
    the z terms: state and T cache over the whole padded box BITWISE for the
    gamma-gas (BASELINE configs[1]'s path); 4 species <= 1e-10 (device pow in
    Wilke's rule)."""
    _steps_check(STEPS3D[name](), 10)


@pytest.mark.slow
def test_3d_steps_vs_ref3d_64cube_20_steps(oracle_api, cuda_device):
    """The same at 64^3 (262k cells: several waves of every face kernel), 20
    steps: BASELINE configs[1]'s path bitwise over a longer trajectory."""
    _steps_check(configs.tgv3d(64, nz=64), 20)


def _steps_check(case, n):
    from oracle import ref
    case.cfg = _viscous_only(case.cfg)
    sim = _fully_3d(case, n_steps=0)
    names = ("rho", "u", "v", "w", "p", "T", "c")

    def prim_of(s):
        cache = s.cache()
        return np.concatenate([np.stack([cache[k] for k in names]), cache["Y"]])
    U0, P0 = sim.Ut, prim_of(sim)
    sim.rk3_steps(case.dt, n)
    want_U, want_P = ref.steps3(case.cfg, U0, P0, case.dt, n)
    got_U, got_P = sim.Ut, prim_of(sim)
    assert np.abs(got_U - U0).max() > 0.0
    ns = case.cfg.mix.ns
    if ns == 1:
        assert np.array_equal(got_U.view(np.uint64), want_U.view(np.uint64)), \
            np.abs(got_U - want_U).max(axis=(1, 2, 3))
        assert np.array_equal(got_P[5].view(np.uint64), want_P[5].view(np.uint64))
    else:
        scale = np.abs(want_U).max(axis=(1, 2, 3))
        err = np.abs(got_U - want_U).max(axis=(1, 2, 3)) / np.where(scale > 0, scale, 1.0)
        assert err.max() <= 1e-10, err
        assert np.abs(got_P[5] - want_P[5]).max() <= 1e-10 * np.abs(want_P[5]).max()


@pytest.mark.parametrize("zwalls", [False, True])
def test_jet3d_steps_vs_ref3d(zwalls, oracle_api, cuda_device):
    """configs[3]'s whole 3D path against oracle/ref3d_step.hpp: inflow
    segments (w = 0 ghosts), the right-edge LODI column with the w wave, y
    walls (and z walls), one-step H2/O2 chemistry, the shaped laser as the 3D
    point kernel — ten steps across the laser pulse (t0 - sigma_t/2 onward),
    state and T cache <= 1e-13 (device exp / pow vs glibc; measured 1.8e-16,
    98% of the words bitwise, tools/jet3d_oracle_check.py)."""
    from oracle import ref
    case = configs.jet3d(32, 16, 8, zwalls=zwalls)
    sim = Simulation(case.cfg)
    sim.set_initial_condition(case.ic)
    t0 = case.cfg.laser.t0 - 0.5 * case.cfg.laser.sigma_t
    sim.set_time(t0)
    sim.prepare_stage(1)
    names = ("rho", "u", "v", "w", "p", "T", "c")

    def prim_of(s):
        cache = s.cache()
        return np.concatenate([np.stack([cache[k] for k in names]), cache["Y"]])
    U0, P0 = sim.Ut, prim_of(sim)
    n = 10
    sim.rk3_steps(case.dt, n)
    want_U, want_P = ref.steps3(case.cfg, U0, P0, case.dt, n, t0=t0)
    got_U, got_P = sim.Ut, prim_of(sim)
    ns = case.cfg.mix.ns
    # the laser deposits energy inside the window: E moves by more than the flow alone
    assert np.abs(got_U[ns + 3] - U0[ns + 3]).max() > 0.0
    scale = np.abs(want_U).max(axis=(1, 2, 3))
    err = np.abs(got_U - want_U).max(axis=(1, 2, 3)) / np.where(scale > 0, scale, 1.0)
    assert err.max() <= 1e-13, err
    assert np.abs(got_P[5] - want_P[5]).max() <= 1e-13 * np.abs(want_P[5]).max()


def test_z_edge_validation(cuda_device):
    """z edges: periodic_z needs periodic zlo / zhi, a bounded z needs walls or
    outflow on both sides (inflow is not supported on z edges)."""
    from paper_2202_02319_b200 import errors
    bad = []
    c = configs.jet3d(24, 12, 8, zwalls=True)
    c.cfg.zhi.type = abi.PERIODIC
    bad.append((c.cfg, errors.ConfigError))
    c = configs.jet3d(24, 12, 8)
    c.cfg.zlo.type = abi.NOSLIP_ADIABATIC
    bad.append((c.cfg, errors.ConfigError))
    c = configs.jet3d(24, 12, 8, zwalls=True)
    c.cfg.zlo.type = abi.INFLOW
    bad.append((c.cfg, errors.UsageError))
    for cfg, exc in bad:
        with pytest.raises(exc):
            Simulation(cfg)


def test_jet3d_zwalls_no_through_flow(cuda_device):
    """configs[3] as a confined duct: with z walls the cache's w vanishes at
    the wall faces (ghost w mirrors the first plane's), mass stays finite."""
    case = configs.jet3d(48, 24, 12, zwalls=True)
    sim = Simulation(case.cfg)
    sim.set_initial_condition(case.ic)
    sim.prepare_stage(1)
    sim.rk3_steps(case.dt, 20)
    c = sim.cache()
    g = 3
    w = c["w"]
    # ghost plane -k mirrors plane k-1 (both sides), so the face average is 0
    scale = np.abs(w).max()
    assert scale > 0.0
    for k in range(1, g + 1):
        assert np.abs(w[g - k] + w[g + k - 1]).max() <= 1e-13 * scale
        assert np.abs(w[-g - 1 + k] + w[-g - k]).max() <= 1e-13 * scale
    T = c["T"][g:-g, g:-g, g:-g]
    assert np.isfinite(T).all() and T.min() > 250.0
