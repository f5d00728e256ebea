"""Slab decomposition validated on one GPU: the y-slabs of a
domain, driven as a single-process group (halo rows by device copies — the
same phase sequence the NCCL path runs across processes), must reproduce the
undecomposed run BIT FOR BIT: state, primitive cache, stable_dt, totals."""
import numpy as np
import pytest

from paper_2202_02319_b200 import Simulation, configs
from paper_2202_02319_b200.sim import SlabGroup
from tests.parity import bitwise_equal

pytestmark = pytest.mark.gpu

CASES = {
    "tgv_periodic": lambda: configs.tgv2d(32),
    "tgv_skew_wrap_ratio": lambda: configs.tgv2d(30, skew=0.2),
    "wall_channel": lambda: configs.wall_channel(24),
    "h2o2_inflow_outflow": lambda: configs.h2o2_counterflow(24),
    "tgv_weno3z_comp": lambda: configs.tgv2d(27, scheme="weno3z", split="comp"),
}


def slab_rows(ny, n, r):
    base, rem = divmod(ny, n)
    return r * base + min(r, rem), base + (1 if r < rem else 0)


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("nslabs", [2, 3])
def test_slabs_match_single_domain(name, nslabs, cuda_device):
    case = CASES[name]()
    single = Simulation(case.cfg)
    single.set_initial_condition(case.ic)
    U0 = single.Ut
    grp = SlabGroup(case.cfg, nslabs)
    single.set_diagnostics("reference")  # serial folds: decomposition-invariant bits
    grp.set_diagnostics("reference")
    g = single.g
    rows = [slab_rows(case.cfg.ny, nslabs, r) for r in range(nslabs)]
    for r, (lo, cnt) in enumerate(rows):
        grp.set_state(r, U0[:, lo:lo + cnt + 2 * g, :])

    def compare(what):
        Ug, Tg = single.Ut, single.cache()["T"]
        for r, (lo, cnt) in enumerate(rows):
            assert bitwise_equal(grp.Ut(r)[:, g:g + cnt], Ug[:, lo + g:lo + g + cnt]), (what, r)
            assert bitwise_equal(grp.cache_T(r), Tg[lo:lo + cnt + 2 * g]), (what, r, "T")

    single.prepare_stage(1)
    grp.prepare_stage(1)
    compare("prepare")
    assert grp.stable_dt() == single.stable_dt()
    single.rk3_steps(case.dt, 6)
    grp.rk3_steps(case.dt, 6)
    compare("steps")
    assert bitwise_equal(grp.conserved_totals(), single.conserved_totals())
    grp.close()


def test_nccl_single_rank_path(cuda_device):
    """The NCCL transport (dlopen'ed libnccl, error-word/clip/dt all-reduces,
    rank folds) with one rank reproduces the plain run bit for bit."""
    import ctypes
    from paper_2202_02319_b200 import native
    case = configs.tgv2d(32)
    a = Simulation(case.cfg)
    a.set_initial_condition(case.ic)
    cfg = configs.tgv2d(32).cfg
    cfg.slab_count, cfg.slab_rank = 1, 0
    b = Simulation(cfg)
    uid = ctypes.create_string_buffer(128)
    assert native.api()["nccl_unique_id"](uid) == 0
    b._check(native.api()["attach_nccl"](b.handle, uid.raw, 1, 0))
    b.set_state(a.Ut)
    a.set_diagnostics("reference")
    b.set_diagnostics("reference")
    for s in (a, b):
        s.prepare_stage(1)
        s.rk3_steps(case.dt, 4)
    assert bitwise_equal(a.Ut, b.Ut)
    assert a.stable_dt() == b.stable_dt()
    assert bitwise_equal(a.conserved_totals(), b.conserved_totals())


CASES3 = {
    "tgv3d_char_teno6_visc": lambda: configs.tgv3d(12, nz=18),
    "tgv3d_comp_weno3z_visc": lambda: configs.tgv3d(12, nz=18, scheme="weno3z", split="comp"),
    "h2o2_inflow_outflow_3d": lambda: configs.extrude_z(configs.h2o2_counterflow(12), 18),
    "wall_channel_3d": lambda: configs.extrude_z(configs.wall_channel(12), 18),
    "jet3d_inflow_lodi_walls_laser": lambda: configs.jet3d(48, 24, 12),
    # z edges: walls on the end slabs' outer sides, no periodic ring
    "jet3d_zwalls": lambda: configs.jet3d(48, 24, 12, zwalls=True),
    "wall_channel_xz_zwalls": lambda: configs.lay_xz(configs.wall_channel(18), 7),
}


@pytest.mark.parametrize("name", sorted(CASES3))
@pytest.mark.parametrize("nslabs", [2, 3])
def test_z_slabs_match_single_domain(name, nslabs, cuda_device):
    """3D extension: z-slabs (g ghost planes per side, periodic ring) reproduce
    the undecomposed 3D run bit for bit."""
    case = CASES3[name]()
    single = Simulation(case.cfg)
    single.set_initial_condition(case.ic)
    U0 = single.Ut
    grp = SlabGroup(case.cfg, nslabs)
    single.set_diagnostics("reference")
    grp.set_diagnostics("reference")
    g = single.g
    planes = [slab_rows(case.cfg.nz, nslabs, r) for r in range(nslabs)]
    for r, (lo, cnt) in enumerate(planes):
        m = grp.members[r]
        assert (m.k0, m.nz, m.nz_glob) == (lo, cnt, case.cfg.nz)
        grp.set_state(r, U0[:, lo:lo + cnt + 2 * g])

    def compare(what):
        Ug, Tg = single.Ut, single.cache()["T"]
        for r, (lo, cnt) in enumerate(planes):
            assert bitwise_equal(grp.Ut(r)[:, g:g + cnt], Ug[:, lo + g:lo + g + cnt]), (what, r)
            assert bitwise_equal(grp.cache_T(r), Tg[lo:lo + cnt + 2 * g]), (what, r, "T")

    single.prepare_stage(1)
    grp.prepare_stage(1)
    compare("prepare")
    assert grp.stable_dt() == single.stable_dt()
    single.rk3_steps(case.dt, 4)
    grp.rk3_steps(case.dt, 4)
    compare("steps")
    assert bitwise_equal(grp.conserved_totals(), single.conserved_totals())
    single.set_diagnostics("device")
    grp.set_diagnostics("device")
    ta, tb = grp.conserved_totals(), single.conserved_totals()
    U = single.Ut[:, 3:-3, 3:-3, 3:-3]
    assert np.all(np.abs(ta - tb) <= 1e-12 * np.abs(U).reshape(U.shape[0], -1).sum(axis=1))
    grp.close()


def test_z_slab_initial_condition_coordinates(cuda_device):
    """Each z-slab evaluates the initial condition at its global z nodes."""
    case = configs.tgv3d(12, nz=18)
    single = Simulation(case.cfg)
    single.set_initial_condition(case.ic)
    grp = SlabGroup(case.cfg, 3)
    for r, m in enumerate(grp.members):
        lo, cnt = slab_rows(18, 3, r)
        assert np.array_equal(m.mesh_z(), single.mesh_z()[lo:lo + cnt + 2 * single.g])
    grp.close()


def _failure(fn):
    try:
        fn()
    except Exception as e:  # noqa: BLE001 — the ignis exception is compared
        return e
    return None


@pytest.mark.parametrize("nslabs", [2, 3])
def test_slab_failure_semantics_match_single_domain(nslabs, cuda_device):
    """Each slab keeps its own error word (as NCCL ranks do) and runs on past a
    peer's failure; the words are MIN-folded once per chunk.  The first
    failure, the restored state, iter/time and last_clip must still be the
    undecomposed run's (solver.hpp:326-329; advance semantics of rk3_steps)."""
    case = configs.tgv2d(24)
    single = Simulation(case.cfg)
    single.set_initial_condition(case.ic)
    U0 = single.Ut
    grp = SlabGroup(case.cfg, nslabs)
    g = single.g
    rows = [slab_rows(case.cfg.ny, nslabs, r) for r in range(nslabs)]
    for r, (lo, cnt) in enumerate(rows):
        grp.set_state(r, U0[:, lo:lo + cnt + 2 * g, :])
    single.prepare_stage(1)
    grp.prepare_stage(1)
    dt = case.dt * 9.0  # marginally unstable: fails after a few steps
    ea = _failure(lambda: single.rk3_steps(dt, 200))
    eb = _failure(lambda: grp.rk3_steps(dt, 200))
    if ea is None:
        pytest.skip("no failure provoked")
    assert type(ea) is type(eb), (ea, eb)
    assert (getattr(ea, "stage", None), getattr(ea, "i", None), getattr(ea, "j", None)) == \
        (getattr(eb, "stage", None), getattr(eb, "i", None), getattr(eb, "j", None))
    Ug = single.Ut
    for r, (lo, cnt) in enumerate(rows):
        assert bitwise_equal(grp.Ut(r)[:, g:g + cnt], Ug[:, lo + g:lo + g + cnt]), r
    import ctypes
    t, it = ctypes.c_double(), ctypes.c_int64()
    assert grp.member_call(0, "get_time", ctypes.byref(t), ctypes.byref(it)) == 0
    assert it.value == single.iter and t.value == single.time
    grp.close()


def test_slab_prepare_failure_in_upper_slab(cuda_device):
    """A bad node in the LAST slab: that slab's word alone records it; the
    group reports the reference's StepFailure (stage, i, j) in global rows."""
    case = configs.tgv2d(24)
    single = Simulation(case.cfg)
    single.set_initial_condition(case.ic)
    U = single.Ut
    # rows 19, 20 (slab 2 of 3); rows 21-23 would also reach the bottom ghost
    # rows through the periodic wrap, which refresh_primitives visits first
    U[0, 3 + 19, 3 + 7] = -1.0  # node (7, 19)
    U[0, 3 + 20, 3 + 1] = -1.0
    single.set_state(U)
    grp = SlabGroup(case.cfg, 3)
    g = single.g
    rows = [slab_rows(24, 3, r) for r in range(3)]
    for r, (lo, cnt) in enumerate(rows):
        grp.set_state(r, U[:, lo:lo + cnt + 2 * g, :])
    ea = _failure(lambda: single.prepare_stage(2))
    eb = _failure(lambda: grp.prepare_stage(2))
    assert ea is not None and type(ea) is type(eb)
    assert (ea.stage, ea.i, ea.j) == (eb.stage, eb.i, eb.j) == (2, 7, 19)
    grp.close()
