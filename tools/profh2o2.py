"""A few RK3 steps then one RHS of the H2/O2 counterflow (512^2, configs[2]) —
the ncu target for the multi-species 2D face kernels (k_faces3<x>, <y>)."""
import sys
sys.path.insert(0, '.')
from paper_2202_02319_b200 import Simulation, configs
case = configs.h2o2_counterflow(512)
s = Simulation(case.cfg)
s.set_initial_condition(case.ic)
s.prepare_stage(1)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    s.rk3_step(s.stable_dt())
    s.prepare_stage(1)
s.compute_rhs(0.0, 1)
print("ok")
