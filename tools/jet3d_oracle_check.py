# dev check: configs[3] jet vs oracle/ref3d_step.hpp (error, laser effect, bitwise fraction)
import sys, numpy as np
sys.path.insert(0, '.')
from paper_2202_02319_b200 import Simulation, configs
from oracle import ref
for zw in (False, True):
    case = configs.jet3d(32, 16, 8, zwalls=zw)
    sim = Simulation(case.cfg); sim.set_initial_condition(case.ic)
    t0 = case.cfg.laser.t0 - 0.5 * case.cfg.laser.sigma_t
    sim.set_time(t0); sim.prepare_stage(1)
    names = ("rho", "u", "v", "w", "p", "T", "c")
    pr = lambda s: np.concatenate([np.stack([s.cache()[k] for k in names]), s.cache()["Y"]])
    U0, P0 = sim.Ut, pr(sim)
    sim.rk3_steps(case.dt, 10)
    wU, wP = ref.steps3(case.cfg, U0, P0, case.dt, 10, t0=t0)
    case.cfg.laser.present = 0
    nU, _ = ref.steps3(case.cfg, U0, P0, case.dt, 10, t0=t0)
    sc = np.abs(wU).max(axis=(1,2,3))
    err = np.abs(sim.Ut - wU).max(axis=(1,2,3)) / sc
    lz = np.abs(wU - nU).max(axis=(1,2,3)) / sc
    bits = np.mean(sim.Ut.view(np.uint64) == wU.view(np.uint64))
    print("zwalls", zw, "max rel err", err.max(), "laser effect", lz[-1], "bitwise fraction", bits, "Tmax", wP[5].max())
