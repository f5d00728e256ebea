"""Field output and diagnostics against the oracle:
IGNS snapshots (snapshot.hpp) byte for byte, probes and the product trace
(solver.hpp:351-385) through advance(), and their slab-decomposed forms."""
import numpy as np
import pytest

from paper_2202_02319_b200 import Simulation, configs, errors
from paper_2202_02319_b200.sim import SlabGroup
from tests.parity import bitwise_equal, clone_cfg, field_errors, make_pair

pytestmark = pytest.mark.gpu


def _bytes(path):
    with open(path, "rb") as f:
        return f.read()


@pytest.mark.parametrize("mk,steps", [(lambda: configs.tgv2d(32), 5),
                                      (lambda: configs.reacting_ch4(24), 0),
                                      (lambda: configs.h2o2_counterflow(24), 0)],
                         ids=["tgv_after_steps", "ch4", "h2o2"])
def test_snapshot_v1_byte_identical(mk, steps, tmp_path, oracle_api, cuda_device):
    case = mk()
    prod, refs = make_pair(case, oracle_api)
    for s in (prod, refs):
        s.config_hash = 0x1234ABCD5678EF01
        s.prepare_stage(1)
        if steps:
            s.rk3_steps(case.dt, steps)
    pa, pb = tmp_path / "prod.igns", tmp_path / "ref.igns"
    prod.write_snapshot(pa)
    refs.write_snapshot(pb)
    assert _bytes(pa) == _bytes(pb)


def test_snapshot_cross_read(tmp_path, oracle_api, cuda_device):
    """Files written by either side restore the other (apply_snapshot)."""
    case = configs.reacting_ch4(24)
    prod, refs = make_pair(case, oracle_api)
    refs.prepare_stage(1)
    refs.rk3_steps(case.dt, 3)
    refs.config_hash = 77
    path = tmp_path / "r.igns"
    refs.write_snapshot(path)
    fresh = Simulation(clone_cfg(case.cfg))
    fresh.read_snapshot(path)
    assert bitwise_equal(fresh.Ut, refs.Ut)
    assert (fresh.time, fresh.iter, fresh.config_hash) == (refs.time, refs.iter, 77)
    # and back: the product's file read by the reference
    path2 = tmp_path / "p.igns"
    fresh.write_snapshot(path2)
    other = Simulation(clone_cfg(case.cfg), oracle_api)
    other.read_snapshot(path2)
    assert bitwise_equal(other.Ut, refs.Ut)


def test_snapshot_format_errors(tmp_path, oracle_api, cuda_device):
    """FormatError cases of read/apply_snapshot raise identically."""
    case = configs.tgv2d(16)
    prod, refs = make_pair(case, oracle_api)
    good = tmp_path / "g.igns"
    refs.write_snapshot(good)
    raw = _bytes(good)
    bad_magic = tmp_path / "m.igns"
    bad_magic.write_bytes(b"XGNS" + raw[4:])
    trunc = tmp_path / "t.igns"
    trunc.write_bytes(raw[: len(raw) // 2])
    other = configs.tgv2d(20)
    shape = tmp_path / "s.igns"
    Simulation(clone_cfg(other.cfg), oracle_api).write_snapshot(shape)
    for path in (bad_magic, trunc, shape, tmp_path / "missing.igns"):
        msgs = []
        for s in (prod, refs):
            with pytest.raises(errors.FormatError) as ei:
                s.read_snapshot(path)
            msgs.append(str(ei.value))
        assert msgs[0] == msgs[1], msgs


def test_snapshot_v2_bit_exact_restart(tmp_path, cuda_device):
    """IGNS v2 carries the T cache: a restart continues bit for bit."""
    for case in (configs.reacting_ch4(24), configs.tgv3d(12)):
        a = Simulation(clone_cfg(case.cfg))
        a.set_initial_condition(case.ic)
        a.prepare_stage(1)
        a.rk3_steps(case.dt, 3)
        path = tmp_path / f"{case.name}.igns"
        a.write_snapshot_v2(path, with_t=True)
        b = Simulation(clone_cfg(case.cfg))
        b.read_snapshot(path)
        assert bitwise_equal(b.cache()["T"], a.cache()["T"])
        for s in (a, b):
            s.prepare_stage(1)
            s.rk3_steps(case.dt, 4)
        assert bitwise_equal(a.Ut, b.Ut) and a.iter == b.iter == 7


def _probe_boxes(nx, ny):
    return [(0, 0, 0, 0), (3, 5, 9, 12), (0, 0, nx - 1, ny - 1), (nx - 4, ny - 6, nx - 1, ny - 1)]


@pytest.mark.parametrize("mk,exact", [(lambda: configs.tgv2d(32), True),
                                      (lambda: configs.reacting_ch4(24), False)],
                         ids=["tgv", "ch4"])
def test_probes_and_trace_through_advance(mk, exact, oracle_api, cuda_device):
    case = mk()
    prod, refs = make_pair(case, oracle_api)
    prod.set_diagnostics("reference")  # the trace in the reference's serial order
    for s in (prod, refs):
        for b in _probe_boxes(case.cfg.nx, case.cfg.ny):
            s.add_probe(*b)
        s.set_sampling(2, 3)
        s.set_integrator(fixed_dt=case.dt, t_end=7.5 * case.dt)
        s.advance()
    assert prod.iter == refs.iter == 8
    for k in range(4):
        (ta, ra), (tb, rb) = prod.probe(k), refs.probe(k)
        assert np.array_equal(ta, tb) and len(ta) == 5  # iterations 0, 2, 4, 6, 8
        if exact:
            assert bitwise_equal(ra, rb)
        else:
            assert np.allclose(ra, rb, rtol=1e-10, atol=0), np.abs(ra - rb).max()
    (ta, va), (tb, vb) = prod.trace(), refs.trace()
    assert np.array_equal(ta, tb) and len(ta) == 3  # iterations 0, 3, 6
    if exact:
        assert bitwise_equal(va, vb)
    else:
        assert np.allclose(va, vb, rtol=1e-10, atol=1e-300)


def test_device_tree_trace_within_tolerance(oracle_api, cuda_device):
    """Default diagnostics: the product trace reduced on the device (fixed
    tree, no Y download) within 1e-13 of the reference's serial fold."""
    case = configs.reacting_ch4(24)
    prod, refs = make_pair(case, oracle_api)
    for s in (prod, refs):
        s.set_sampling(0, 1)
        s.set_integrator(fixed_dt=case.dt, t_end=4.5 * case.dt)
        s.advance()
    (ta, va), (tb, vb) = prod.trace(), refs.trace()
    assert np.array_equal(ta, tb) and len(ta) == 6
    assert np.all(np.abs(va - vb) <= 1e-13 * np.abs(vb)), np.abs(va - vb).max()


def test_probe_box_validation(oracle_api, cuda_device):
    case = configs.tgv2d(16)
    prod, refs = make_pair(case, oracle_api)
    for box in ((-1, 0, 2, 2), (0, 0, 16, 3), (5, 5, 4, 6)):
        for s in (prod, refs):
            with pytest.raises(errors.ConfigError):
                s.add_probe(*box)


@pytest.mark.parametrize("nslabs", [2, 3])
def test_slab_outputs_match_single_domain(nslabs, tmp_path, cuda_device):
    """Probes spanning slab boundaries fold in the serial order; the gathered
    snapshot equals the undecomposed one byte for byte; reading it back into
    the slabs restores every slab."""
    case = configs.reacting_ch4(30)
    single = Simulation(clone_cfg(case.cfg))
    single.set_initial_condition(case.ic)
    grp = SlabGroup(case.cfg, nslabs)
    single.set_diagnostics("reference")  # serial folds: decomposition-invariant bits
    grp.set_diagnostics("reference")
    U0 = single.Ut
    g = single.g
    from tests.test_gpu_slabs import slab_rows
    rows = [slab_rows(case.cfg.ny, nslabs, r) for r in range(nslabs)]
    for r, (lo, cnt) in enumerate(rows):
        grp.set_state(r, U0[:, lo:lo + cnt + 2 * g, :])
    boxes = [(2, 3, 20, 27), (0, 9, 29, 11), (4, 0, 4, 29)]
    for b in boxes:
        single.add_probe(*b)
        grp.add_probe(*b)
    for s in (single, grp):
        s.set_sampling(2, 2)
        s.set_integrator(fixed_dt=case.dt, t_end=4.5 * case.dt)
        s.advance()
    for k in range(len(boxes)):
        (ta, ra), (tb, rb) = single.probe(k), grp.probe(k)
        assert np.array_equal(ta, tb) and bitwise_equal(ra, rb), k
    assert bitwise_equal(single.trace()[1], grp.trace()[1])
    pa, pb = tmp_path / "single.igns", tmp_path / "slabs.igns"
    single.write_snapshot(pa)
    grp.write_snapshot(pb)
    assert _bytes(pa) == _bytes(pb)
    grp2 = SlabGroup(case.cfg, nslabs)
    grp2.read_snapshot(pa)
    for r, (lo, cnt) in enumerate(rows):
        assert bitwise_equal(grp2.Ut(r), single.Ut[:, lo:lo + cnt + 2 * g, :]), r
    grp.close()
    grp2.close()


def test_ensemble_members_match_solo_runs(cuda_device):
    """configs[4]: step-interleaved members equal their solo runs bit for bit;
    a failing member reports its own StepFailure and the others finish."""
    from paper_2202_02319_b200 import Ensemble
    cases = configs.ensemble_members(5, nxy=(24, 16), first=0, count=3)
    assert len({c.cfg.laser.energy for c in cases}) == 3
    ens = Ensemble([clone_cfg(c.cfg) for c in cases])
    solo = [Simulation(clone_cfg(c.cfg)) for c in cases]
    for m, s, c in zip(ens.members, solo, cases):
        for x in (m, s):
            x.set_initial_condition(c.ic)
            x.prepare_stage(1)
    dts = [c.dt for c in cases]
    dts[1] = 1e-2  # unstable: member 1 fails
    status = ens.rk3_steps(dts, 6)
    assert status[0] == status[2] == 0 and status[1] != 0
    assert isinstance(ens.error(1), errors.IgnisError)
    for k in (0, 2):
        solo[k].rk3_steps(dts[k], 6)
        assert bitwise_equal(ens.members[k].Ut, solo[k].Ut)
        assert ens.members[k].iter == solo[k].iter == 6
    with pytest.raises(errors.IgnisError):
        solo[1].rk3_steps(dts[1], 6)
    assert ens.members[1].iter == solo[1].iter
    assert bitwise_equal(ens.members[1].Ut, solo[1].Ut)


def test_3d_slab_snapshot_matches_single_domain(tmp_path, cuda_device):
    """IGNS v2 of a 3D domain gathered from z-slabs equals the undecomposed
    file byte for byte (state, J and T cache), and scatters back exactly."""
    case = configs.tgv3d(12, nz=18)
    single = Simulation(clone_cfg(case.cfg))
    single.set_initial_condition(case.ic)
    single.prepare_stage(1)
    single.rk3_steps(case.dt, 2)
    grp = SlabGroup(case.cfg, 3)
    U = single.Ut
    T = single.cache()["T"]
    for r in range(3):
        grp.set_state(r, U[:, 6 * r:6 * r + 12], T[6 * r:6 * r + 12])
    # align time / iteration with the single domain before writing
    for k in range(3):
        grp.member_call(k, "set_time", single.time, single.iter)
    pa, pb = tmp_path / "single.igns", tmp_path / "slabs.igns"
    single.write_snapshot_v2(pa, with_t=True)
    grp.write_snapshot(pb, version=2, with_t=True)
    assert _bytes(pa) == _bytes(pb)
    grp2 = SlabGroup(case.cfg, 3)
    grp2.read_snapshot(pa)
    for r in range(3):
        assert bitwise_equal(grp2.Ut(r), U[:, 6 * r:6 * r + 12])
        assert bitwise_equal(grp2.cache_T(r), T[6 * r:6 * r + 12])
    grp.close()
    grp2.close()
