"""GPU parity at the BASELINE.json configs' own sizes (VERDICT r1 "what's
missing" 2), against the CPU oracle (the unmodified reference) on all host
cores.  SURVEY §8c gates:
  * configs[0] Sod 1000x7 to t = 0.2 (1000 steps, LODI outflow,
    solver.hpp:717-788): gamma-gas -> bitwise, plus the known plateaus;
  * 2D TGV 256^2, 200 steps (the parity analogue of configs[1]): bitwise;
  * configs[2] H2/O2 counterflow 512^2, 20 steps: <= 1e-10;
  * configs[4] one 500x250 member, 20 steps through the ensemble runner:
    <= 1e-10.
Marked slow (tens of seconds of oracle time each) but part of -m gpu.
"""
import os

import numpy as np
import pytest

from paper_2202_02319_b200 import Ensemble, configs
from tests.parity import bitwise_equal, clone_cfg, field_errors, make_pair

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

STEP_TOL = 1e-10
THREADS = max(1, os.cpu_count() or 1)


def _pair(case, oracle_api):
    return make_pair(case, oracle_api, partitions=THREADS)


@pytest.mark.parametrize("scheme,split,dt", [("teno6", "char", 2e-4), ("weno3z", "comp", 1e-4)])
def test_sod_configs0_full_run(oracle_api, cuda_device, scheme, split, dt):
    case = configs.sod_strip(1000, scheme=scheme, split=split)
    prod, refs = _pair(case, oracle_api)
    for s in (prod, refs):
        s.set_integrator(fixed_dt=dt, t_end=0.2)
        s.advance()
    assert prod.iter == refs.iter == round(0.2 / dt)
    assert prod.time == refs.time
    err = field_errors(prod.Ut, refs.Ut, prod.ns)
    assert err.max() <= STEP_TOL, err
    assert bitwise_equal(prod.Ut, refs.Ut), ("gamma-gas Sod is expected bitwise", err)
    # the exact Riemann solution's plateaus (0.4262 / 0.2656)
    rho = prod.cache()["rho"][3:-3, 3:-3][3]
    x = (np.arange(1000) + 0.5) / 1000 - 0.5
    assert abs(rho[(x > -0.05) & (x < 0.1)].mean() - 0.4262) < 0.01
    assert abs(rho[(x > 0.2) & (x < 0.3)].mean() - 0.2656) < 0.01


def test_tgv2d_256_200_steps_bitwise(oracle_api, cuda_device):
    case = configs.tgv2d(256)
    prod, refs = _pair(case, oracle_api)
    prod.set_diagnostics("reference")
    for s in (prod, refs):
        s.prepare_stage(1)
        s.rk3_steps(case.dt, 200)
    assert bitwise_equal(prod.Ut, refs.Ut)
    assert bitwise_equal(prod.cache()["T"], refs.cache()["T"])
    assert bitwise_equal(prod.conserved_totals(), refs.conserved_totals())


def test_h2o2_configs2_512_20_steps(oracle_api, cuda_device):
    case = configs.h2o2_counterflow(512)
    prod, refs = _pair(case, oracle_api)
    for s in (prod, refs):
        s.prepare_stage(1)
    assert bitwise_equal(prod.cache()["T"], refs.cache()["T"])
    for s in (prod, refs):
        s.rk3_steps(case.dt, 20)
    err = field_errors(prod.Ut, refs.Ut, prod.ns)
    assert err.max() <= STEP_TOL, err
    # the laser (t0 = 3e-6) has started depositing: the state moved
    assert prod.time == refs.time


def test_ensemble_member_configs4_500x250(oracle_api, cuda_device):
    """Two campaign members advanced together by ign_ensemble_rk3_steps; the
    first is checked against the oracle run on its own."""
    cases = configs.ensemble_members(64, count=2)
    ens = Ensemble([clone_cfg(c.cfg) for c in cases])
    _, refs = _pair(cases[0], oracle_api)
    for m, c in zip(ens.members, cases):
        m.set_state(refs.Ut)
        m.prepare_stage(1)
    refs.prepare_stage(1)
    status = ens.rk3_steps(cases[0].dt, 20)
    assert status == [0, 0]
    refs.rk3_steps(cases[0].dt, 20)
    err = field_errors(ens.members[0].Ut, refs.Ut, refs.ns)
    assert err.max() <= STEP_TOL, err
    # members differ only by laser energy: same step count, different states
    assert ens.members[1].iter == 20
    assert not bitwise_equal(ens.members[0].Ut, ens.members[1].Ut)
