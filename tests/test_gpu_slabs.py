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
