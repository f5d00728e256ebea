"""One RHS of the 2D TGV (512^2) and the 3D TGV (64^3) for ncu FP64 counts."""
import sys
sys.path.insert(0, '.')
from paper_2202_02319_b200 import Simulation, configs
for case in (configs.tgv2d(512), configs.tgv3d(64)):
    s = Simulation(case.cfg)
    s.set_initial_condition(case.ic)
    s.prepare_stage(1)
    s.compute_rhs(0.0, 1)
    s.close()
print("ok")
