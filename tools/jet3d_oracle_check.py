# dev check: configs[3] jet vs oracle/ref3d_step.hpp (error, laser effect, bitwise fraction)
#   python tools/jet3d_oracle_check.py [nx ny nz steps [--no-laser-ref]]
import sys

import numpy as np

sys.path.insert(0, '.')
from paper_2202_02319_b200 import Simulation, configs  # noqa: E402
from oracle import ref  # noqa: E402

nx, ny, nz, steps = (int(a) for a in (sys.argv[1:5] if len(sys.argv) > 4 else (32, 16, 8, 10)))
laser_ref = "--no-laser-ref" not in sys.argv
for zw in (False, True):
    case = configs.jet3d(nx, ny, nz, zwalls=zw)
    sim = Simulation(case.cfg)
    sim.set_initial_condition(case.ic)
    t0 = case.cfg.laser.t0 - 0.5 * case.cfg.laser.sigma_t
    sim.set_time(t0)
    sim.prepare_stage(1)
    names = ("rho", "u", "v", "w", "p", "T", "c")

    def pr(s):
        c = s.cache()
        return np.concatenate([np.stack([c[k] for k in names]), c["Y"]])
    U0, P0 = sim.Ut, pr(sim)
    sim.rk3_steps(case.dt, steps)
    wU, wP = ref.steps3(case.cfg, U0, P0, case.dt, steps, t0=t0)
    sc = np.abs(wU).max(axis=(1, 2, 3))
    err = np.abs(sim.Ut - wU).max(axis=(1, 2, 3)) / sc
    bits = np.mean(sim.Ut.view(np.uint64) == wU.view(np.uint64))
    msg = (f"jet {nx}x{ny}x{nz} zwalls={zw} {steps} steps from t0-sigma_t/2: max rel err "
           f"{err.max():.3g}, bitwise fraction {bits:.4f}, Tmax {wP[5].max():.1f} K")
    if laser_ref:
        case.cfg.laser.present = 0
        nU, _ = ref.steps3(case.cfg, U0, P0, case.dt, steps, t0=t0)
        msg += f", laser effect on E {(np.abs(wU - nU).max(axis=(1, 2, 3)) / sc)[-1]:.3g}"
    print(msg, flush=True)
