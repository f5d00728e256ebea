"""A few RK3 steps then one RHS of the 3D jet (512x256x32, configs[3] per-GPU
slab) — the ncu target for the multi-species kernels (k_prim3, k_visc3)."""
import sys
sys.path.insert(0, '.')
from paper_2202_02319_b200 import Simulation, configs
case = configs.jet3d()
s = Simulation(case.cfg)
s.set_initial_condition(case.ic)
s.prepare_stage(1)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    s.rk3_step(s.stable_dt())
    s.prepare_stage(1)
s.compute_rhs(0.0, 1)
print("ok")
