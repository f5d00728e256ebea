"""GPU parity of the B200 path against the CPU oracle (the unmodified reference).

Every test drives BOTH implementations through the same C ABI with the same
config and the same initial bits, then compares.  Gates (SURVEY.md §8c,
BASELINE.json north_star):
  * primitive cache: bitwise (no transcendental on that path);
  * γ-gas cases (TGV, Sod): bitwise RHS, dt and N-step state;
  * multi-species cases (pow/exp in transport/chemistry, device libm vs
    glibc): single RHS <= 1e-13 and N steps <= 1e-10, normalised per field.
"""
import numpy as np
import pytest

from paper_2202_02319_b200 import configs, errors
from tests.parity import bitwise_equal, field_errors, make_pair

pytestmark = pytest.mark.gpu

RHS_TOL = 1e-13
STEP_TOL = 1e-10



def _ch4_quartic(n):
    """CH4/O2 with quadratic and quartic cp terms added: keeps the general
    (indexed-range, quartic Horner) thermo path covered on the device — the
    linear tables in data/ all take DSpecies::lin2."""
    case = configs.reacting_ch4(n)
    mix = case.cfg.mix
    for s in range(mix.ns):
        for k in range(mix.species[s].npieces):
            mix.species[s].pieces[k].c2 = 1e-7
            mix.species[s].pieces[k].c4 = -2e-15
    return case


# name -> (builder, exact, nsteps)
CASES = {
    "ch4_quartic_thermo": (lambda: _ch4_quartic(24), False, 10),
    "tgv_char_teno6_visc": (lambda: configs.tgv2d(48), True, 20),
    "tgv_comp_teno6_inviscid": (lambda: configs.tgv2d(48, split="comp", viscous=False), False, 20),
    "tgv_char_weno3z_visc": (lambda: configs.tgv2d(40, scheme="weno3z"), True, 20),
    "tgv_comp_weno3z_visc": (lambda: configs.tgv2d(40, scheme="weno3z", split="comp"), False, 20),
    "tgv_skew_char_teno6": (lambda: configs.tgv2d(32, skew=0.2), True, 10),
    "sod_lodi_char_teno6": (lambda: configs.sod_strip(200), False, 40),
    "ch4_react_laser_char": (lambda: configs.reacting_ch4(32), False, 20),
    "ch4_react_comp_weno3z": (lambda: configs.reacting_ch4(32, scheme="weno3z", split="comp"), False, 20),
    "h2o2_counterflow_inflow": (lambda: configs.h2o2_counterflow(32), False, 20),
    "wall_isothermal": (lambda: configs.wall_channel(24), False, 10),
    "wall_adiabatic_weno3z": (lambda: configs.wall_channel(24, isothermal=False, scheme="weno3z"), False, 10),
    # nx + 1 >= 32 NC: the x-face kernels' flattened-row mode (CTAs straddle rows)
    "tgv_wide_flat_x": (lambda: configs.tgv2d(160), True, 6),
    "h2o2_wide_flat_x": (lambda: configs.h2o2_counterflow(240, nxy=(240, 12)), False, 6),
}


@pytest.fixture(params=sorted(CASES))
def pair(request, oracle_api, cuda_device):
    mk, exact, n = CASES[request.param]
    case = mk()
    prod, refs = make_pair(case, oracle_api)
    yield case, prod, refs, exact, n
    prod.close()
    refs.close()


def test_initial_condition_host_conversion_bitwise(oracle_api, cuda_device):
    """set_initial_condition (solver.hpp:115-128) through the product's host code."""
    for mk in (lambda: configs.tgv2d(24), lambda: configs.reacting_ch4(16)):
        case = mk()
        prod, refs = make_pair(case, oracle_api)
        prod.set_initial_condition(case.ic)
        assert bitwise_equal(prod.Ut, refs.Ut)


def test_prepare_stage_cache_bitwise(pair):
    case, prod, refs, exact, n = pair
    prod.prepare_stage(1)
    refs.prepare_stage(1)
    a, b = prod.cache(), refs.cache()
    for k in ("rho", "u", "v", "p", "T", "c"):
        assert bitwise_equal(a[k], b[k]), k
    assert bitwise_equal(a["Y"], b["Y"])
    assert bitwise_equal(prod.Ut, refs.Ut)  # ghosts filled identically


def test_compute_rhs(pair):
    case, prod, refs, exact, n = pair
    prod.prepare_stage(1)
    refs.prepare_stage(1)
    t = 0.37 * case.dt
    ra, rb = prod.compute_rhs(t, 1), refs.compute_rhs(t, 1)
    if exact:
        assert bitwise_equal(ra, rb)
    else:
        err = field_errors(ra, rb, prod.ns)
        assert err.max() <= RHS_TOL, err


def test_stable_dt(pair):
    case, prod, refs, exact, n = pair
    prod.prepare_stage(1)
    refs.prepare_stage(1)
    da, db = prod.stable_dt(), refs.stable_dt()
    if exact:
        assert da == db
    else:
        assert abs(da - db) <= 1e-13 * abs(db)


def test_rk3_steps(pair):
    case, prod, refs, exact, n = pair
    for s in (prod, refs):
        s.prepare_stage(1)
    ea, eb = _raises_same(lambda: prod.rk3_steps(case.dt, n), lambda: refs.rk3_steps(case.dt, n))
    if ea is not None:  # both failed: same location and same surviving state
        assert (getattr(ea, "stage", 0), getattr(ea, "i", 0), getattr(ea, "j", 0)) == \
               (getattr(eb, "stage", 0), getattr(eb, "i", 0), getattr(eb, "j", 0))
    else:
        assert prod.iter == refs.iter == n
    assert prod.time == refs.time
    a, b = prod.Ut, refs.Ut
    if exact:
        assert bitwise_equal(a, b)
        assert bitwise_equal(prod.cache()["T"], refs.cache()["T"])
    else:
        err = field_errors(a, b, prod.ns)
        assert err.max() <= STEP_TOL, err
    assert prod.last_clip == pytest.approx(refs.last_clip, rel=1e-10, abs=1e-300)


def test_single_rk3_step_postcondition(oracle_api, cuda_device):
    """rk3_step leaves the cache at U2 and the ghosts of U2 (solver.hpp:304-332)."""
    case = configs.tgv2d(32)
    prod, refs = make_pair(case, oracle_api)
    for s in (prod, refs):
        s.prepare_stage(1)
        s.rk3_step(case.dt)
    assert bitwise_equal(prod.Ut, refs.Ut)
    assert bitwise_equal(prod.cache()["T"], refs.cache()["T"])


def test_advance_fixed_and_cfl(oracle_api, cuda_device):
    """advance (solver.hpp:336-349) with a pinned step and CFL-controlled."""
    for fixed in (True, False):
        case = configs.tgv2d(32)
        prod, refs = make_pair(case, oracle_api)
        for s in (prod, refs):
            s.set_integrator(fixed_dt=case.dt if fixed else 0.0, t_end=7.5 * case.dt)
            s.advance()
        assert prod.iter == refs.iter and prod.time == refs.time
        assert bitwise_equal(prod.Ut, refs.Ut)


def test_advance_hook_called_per_step(oracle_api, cuda_device):
    case = configs.tgv2d(24)
    prod, _ = make_pair(case, oracle_api)
    seen = []
    prod.set_integrator(fixed_dt=case.dt, t_end=3.5 * case.dt)
    prod.advance(lambda sim: seen.append(sim.iter))
    assert seen == [1, 2, 3, 4]


def test_advance_hook_nonzero_stops(oracle_api, cuda_device):
    """ign_step_hook returns nonzero to stop (ignis_b200.h); the oracle stops
    the reference's loop through its public integ.max_iter (solver.hpp:340)."""
    case = configs.tgv2d(24)
    prod, refs = make_pair(case, oracle_api)
    for s in (prod, refs):
        s.set_integrator(fixed_dt=case.dt, t_end=10.5 * case.dt)
        s.advance(lambda sim: sim.iter >= 3)
    assert prod.iter == refs.iter == 3
    assert bitwise_equal(prod.Ut, refs.Ut)


def test_diagnostics_bitwise(oracle_api, cuda_device):
    """IGN_DIAG_REFERENCE: the reference's serial folds, bitwise."""
    case = configs.reacting_ch4(24)
    prod, refs = make_pair(case, oracle_api)
    prod.set_diagnostics("reference")
    for s in (prod, refs):
        s.prepare_stage(1)
    assert bitwise_equal(prod.conserved_totals(), refs.conserved_totals())
    assert prod.product_mole_fraction() == refs.product_mole_fraction()


@pytest.mark.parametrize("mk", [lambda: configs.reacting_ch4(40), lambda: configs.tgv2d(64),
                                lambda: configs.h2o2_counterflow(48)], ids=["ch4", "tgv", "h2o2"])
def test_diagnostics_device_tree(mk, oracle_api, cuda_device):
    """Default IGN_DIAG_DEVICE: deterministic device tree sums within
    1e-12 sum|x| (totals) / 1e-13 (product fraction) of the serial fold."""
    case = mk()
    prod, refs = make_pair(case, oracle_api)
    for s in (prod, refs):
        s.prepare_stage(1)
        s.rk3_steps(case.dt, 3)
    ta, tb = prod.conserved_totals(), refs.conserved_totals()
    U = refs.Ut[:, 3:-3, 3:-3]
    bound = 1e-12 * np.abs(U).reshape(U.shape[0], -1).sum(axis=1)
    assert np.all(np.abs(ta - tb) <= bound), (ta - tb, bound)
    assert bitwise_equal(ta, prod.conserved_totals())  # deterministic
    pa, pb = prod.product_mole_fraction(), refs.product_mole_fraction()
    assert abs(pa - pb) <= 1e-13 * abs(pb) + 1e-300


def _raises_same(fa, fb):
    ea = eb = None
    try:
        fa()
    except errors.IgnisError as e:
        ea = e
    try:
        fb()
    except errors.IgnisError as e:
        eb = e
    assert type(ea) is type(eb), (ea, eb)
    return ea, eb


def test_prepare_state_failure_location(oracle_api, cuda_device):
    """refresh_primitives' StepFailure carries (stage, i, j) of the first bad node."""
    case = configs.tgv2d(24)
    prod, refs = make_pair(case, oracle_api)
    Ut = refs.Ut
    Ut[0, 3 + 9, 3 + 5] = -1.0  # node (5, 9)
    Ut[0, 3 + 15, 3 + 2] = -1.0  # a later node
    for s in (prod, refs):
        s.set_state(Ut)
    ea, eb = _raises_same(lambda: prod.prepare_stage(2), lambda: refs.prepare_stage(2))
    assert isinstance(ea, errors.StepFailure)
    assert (ea.stage, ea.i, ea.j) == (eb.stage, eb.i, eb.j) == (2, 5, 9)


def test_step_failure_restores_u0(oracle_api, cuda_device):
    """A step that drives density negative throws StepFailure and restores U0
    (solver.hpp:326-329); time/iter do not advance."""
    case = configs.tgv2d(24)
    prod, refs = make_pair(case, oracle_api)
    for s in (prod, refs):
        s.prepare_stage(1)
    U0 = refs.Ut
    ea, eb = _raises_same(lambda: prod.rk3_step(50.0), lambda: refs.rk3_step(50.0))
    assert isinstance(ea, errors.StepFailure)
    assert (ea.stage, ea.i, ea.j) == (eb.stage, eb.i, eb.j)
    assert str(ea).split(":")[0] == str(eb).split(":")[0]
    assert bitwise_equal(prod.Ut, U0) and bitwise_equal(refs.Ut, U0)
    assert prod.iter == refs.iter == 0 and prod.time == refs.time == 0.0


def test_failure_mid_batch_matches_reference(oracle_api, cuda_device):
    """rk3_steps: a failure at step k leaves k completed steps (advance semantics)."""
    case = configs.tgv2d(24)
    prod, refs = make_pair(case, oracle_api)
    for s in (prod, refs):
        s.prepare_stage(1)
    dt = case.dt * 9.0  # marginally unstable: fails after a few steps
    ea, eb = _raises_same(lambda: prod.rk3_steps(dt, 200), lambda: refs.rk3_steps(dt, 200))
    if ea is None:
        pytest.skip("no failure provoked")
    assert prod.iter == refs.iter and prod.time == refs.time
    assert bitwise_equal(prod.Ut, refs.Ut)


def test_golden_fixtures_on_device(cuda_device):
    """The committed oracle fixtures (tests/golden) reproduced by the B200 path."""
    import os
    from paper_2202_02319_b200 import Simulation
    from tests.golden.make_golden import CASES as GCASES
    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    for name, (mk, n) in GCASES.items():
        want = np.load(os.path.join(here, name + ".npz"))
        case = mk()
        sim = Simulation(case.cfg)
        sim.set_state(want["Ut0"])
        sim.prepare_stage(1)
        assert bitwise_equal(sim.cache()["T"], want["T1"]), name
        rhs = sim.compute_rhs(0.0, 1)
        assert field_errors(rhs, want["rhs"], sim.ns).max() <= RHS_TOL, name
        sim.rk3_steps(float(want["dt"]), int(want["nsteps"]))
        assert field_errors(sim.Ut, want["UtN"], sim.ns).max() <= STEP_TOL, name


def _mesh_pair(case, oracle_api, X, Y):
    """Both implementations initialised from a hand-built Mesh (ign_config
    mesh_x/mesh_y, mesh.hpp:23-42)."""
    import ctypes as C
    X = np.ascontiguousarray(X, dtype=np.float64)
    Y = np.ascontiguousarray(Y, dtype=np.float64)
    from tests.parity import clone_cfg
    from paper_2202_02319_b200 import Simulation
    cfgs = [clone_cfg(case.cfg), clone_cfg(case.cfg)]
    for c in cfgs:
        c.apply_skew = 0
        c.mesh_x = X.ctypes.data_as(C.POINTER(C.c_double))
        c.mesh_y = Y.ctypes.data_as(C.POINTER(C.c_double))
    prod = Simulation(cfgs[0])
    refs = Simulation(cfgs[1], oracle_api)
    return prod, refs


def test_hand_built_mesh_matches_reference(oracle_api, cuda_device):
    """A caller's Mesh with arbitrary (stretched, sheared) node coordinates:
    metrics, RHS and 10 steps bitwise against the reference built from the
    same Mesh (compute_metrics of mesh.x/mesh.y, metrics.hpp:73-118)."""
    case = configs.tgv2d(40)
    X0, Y0 = configs.padded_coords(case.cfg)
    X = X0 + 0.08 * np.sin(X0) + 0.03 * np.sin(Y0)
    Y = Y0 + 0.05 * np.sin(X0 + 0.5)
    prod, refs = _mesh_pair(case, oracle_api, X, Y)
    assert bitwise_equal(prod.metrics(0), refs.metrics(0))
    assert bitwise_equal(prod.metrics(1), refs.metrics(1))
    refs.set_initial_condition(case.ic)
    prod.set_state(refs.Ut)
    for s in (prod, refs):
        s.prepare_stage(1)
    assert bitwise_equal(prod.compute_rhs(0.0, 1), refs.compute_rhs(0.0, 1))
    for s in (prod, refs):
        s.rk3_steps(case.dt, 10)
    assert bitwise_equal(prod.Ut, refs.Ut)


def test_hand_built_mesh_equals_apply_skew(oracle_api, cuda_device):
    """Feeding apply_skew's own coordinates as a hand-built Mesh reproduces the
    apply_skew run bit for bit."""
    case = configs.tgv2d(32, skew=0.15)
    prod_s, refs_s = make_pair(case, oracle_api)
    X = refs_s.mesh_xy()[0].copy()
    Y = refs_s.mesh_xy()[1].copy()
    prod, refs = _mesh_pair(case, oracle_api, X, Y)
    prod.set_state(refs_s.Ut)
    for s in (prod, prod_s):
        s.prepare_stage(1)
        s.rk3_steps(case.dt, 5)
    assert bitwise_equal(prod.Ut, prod_s.Ut)
