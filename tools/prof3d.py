"""One RHS of the 3D TGV (default 256^3) — the ncu --set full target."""
import sys
sys.path.insert(0, '.')
from paper_2202_02319_b200 import Simulation, configs
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
case = configs.tgv3d(n)
s = Simulation(case.cfg)
s.set_initial_condition(case.ic)
s.prepare_stage(1)
s.compute_rhs(0.0, 1)
print("ok")
