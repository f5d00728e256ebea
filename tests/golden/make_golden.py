"""Generates tests/golden/*.npz from the CPU oracle (the unmodified reference
compiled by oracle/build_ref.sh).  TEST INFRASTRUCTURE; rerun with

    python tests/golden/make_golden.py

Each fixture holds, for one small case: the initial mapped state Ut0, the
primitive cache after prepare_stage(1), one compute_rhs at t=0 (stage 1),
stable_dt, and Ut/T after N advance-loop steps (rk3_step + prepare_stage(1)).
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from paper_2202_02319_b200 import configs  # noqa: E402
from oracle import ref  # noqa: E402

CASES = {
    "tgv_char_teno6_visc_32": (lambda: configs.tgv2d(32), 6),
    "tgv_comp_weno3z_32": (lambda: configs.tgv2d(32, scheme="weno3z", split="comp"), 6),
    "ch4_react_laser_24": (lambda: configs.reacting_ch4(24), 4),
    "sod_lodi_120": (lambda: configs.sod_strip(120), 8),
    "h2o2_inflow_24": (lambda: configs.h2o2_counterflow(24), 4),
    "wall_channel_20": (lambda: configs.wall_channel(20), 4),
}


def generate(name, mk, nsteps):
    case = mk()
    sim = ref.simulation(case.cfg)
    sim.set_initial_condition(case.ic)
    Ut0 = sim.Ut
    sim.prepare_stage(1)
    cache = sim.cache()
    rhs = sim.compute_rhs(0.0, 1)
    dt_stable = sim.stable_dt()
    sim.rk3_steps(case.dt, nsteps)
    return dict(Ut0=Ut0, T1=cache["T"], p1=cache["p"], c1=cache["c"], rhs=rhs,
                dt_stable=np.float64(dt_stable), dt=np.float64(case.dt),
                nsteps=np.int64(nsteps), UtN=sim.Ut, TN=sim.cache()["T"],
                time=np.float64(sim.time), clip=np.float64(sim.last_clip))


def main():
    for name, (mk, n) in CASES.items():
        data = generate(name, mk, n)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **data)
        print("wrote", name)


if __name__ == "__main__":
    main()
