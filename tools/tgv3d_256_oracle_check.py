"""One RK3 step of BASELINE configs[1] at its stated size (TGV 3D 256^3, the
bench's workload) on the B200 path against the 3D oracle
(oracle/ref3d_step.hpp, serial on the host: ~2 min): state and T cache over the
whole padded box compared bitwise.  Evidence run (profiles/r2e_tgv3d256_oracle.txt),
not a test — the suite's 3D trajectories run at 16^3-64^3."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2202_02319_b200 import Simulation, configs  # noqa: E402
from oracle import ref  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
case = configs.tgv3d(n)
sim = Simulation(case.cfg)
sim.set_initial_condition(case.ic)
sim.prepare_stage(1)
names = ("rho", "u", "v", "w", "p", "T", "c")


def prim_of(s):
    c = s.cache()
    return np.concatenate([np.stack([c[k] for k in names]), c["Y"]])


U0, P0 = sim.Ut, prim_of(sim)
sim.rk3_steps(case.dt, steps)
gU, gP = sim.Ut, prim_of(sim)
t = time.time()
wU, wP = ref.steps3(case.cfg, U0, P0, case.dt, steps)
el = time.time() - t
same_U = np.array_equal(gU.view(np.uint64), wU.view(np.uint64))
same_T = np.array_equal(gP[5].view(np.uint64), wP[5].view(np.uint64))
print(f"TGV 3D {n}^3, {steps} RK3 step(s), fixed dt {case.dt:.6g}: state words {gU.size}, "
      f"bitwise equal: state {same_U}, T cache {same_T}; max |dU| {np.abs(gU - wU).max():.3g}; "
      f"state moved by {np.abs(gU - U0).max():.3g}; oracle {el:.0f} s on one host thread")
sys.exit(0 if (same_U and same_T) else 1)
