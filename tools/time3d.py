"""Faces/step timing of the 3D TGV for library variants (IGN_LIB=...)."""
import os, sys, json
sys.path.insert(0, '.')
from paper_2202_02319_b200 import Simulation, configs
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
case = configs.tgv3d(n, scheme=os.environ.get("SCHEME", "teno6"), split=os.environ.get("SPLIT", "char"))
s = Simulation(case.cfg)
s.set_initial_condition(case.ic)
s.prepare_stage(1)
s.rk3_steps(case.dt, 2)
s.profile_enable(True)
s.rk3_steps(case.dt, 3)
p = s.profile_read()
tot = sum(v[0] for v in p.values())
print(json.dumps({"lib": os.environ.get("IGN_LIB", "default"), "n": n,
                  "faces_ms_per_stage": p["faces"][0] / p["faces"][1],
                  "ms_per_step": tot / 3, **{k: round(v[0] / 3, 3) for k, v in p.items() if v[1]}}))
