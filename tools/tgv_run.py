"""TGV 3D Re 1600 run to t = 10 at 256^3: kinetic-energy history (validation)."""
import json, sys, time
import numpy as np
sys.path.insert(0, '.')
from paper_2202_02319_b200 import Simulation, configs
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
t_end = float(sys.argv[2]) if len(sys.argv) > 2 else 10.0
case = configs.tgv3d(n)
sim = Simulation(case.cfg)
sim.set_initial_condition(case.ic)
sim.prepare_stage(1)
g = 3
def ke():
    U = sim.Ut[:, g:-g, g:-g, g:-g]
    rho = U[0]
    return float(0.5 * np.mean((U[1] ** 2 + U[2] ** 2 + U[3] ** 2) / rho) / np.mean(rho))
hist = [(0.0, ke())]
chunk = max(1, int(round(0.1 / case.dt)))
t0 = time.time()
while sim.time < t_end - 1e-12:
    k = min(chunk, int(round((t_end - sim.time) / case.dt)))
    if k <= 0:
        break
    sim.rk3_steps(case.dt, k)
    hist.append((sim.time, ke()))
wall = time.time() - t0
t = np.array([h[0] for h in hist]); e = np.array([h[1] for h in hist])
eps = -np.gradient(e, t)
ipk = int(np.argmax(eps))
out = {"n": n, "dt": case.dt, "steps": sim.iter, "wall_s": wall, "t": t.tolist(), "ke": e.tolist(),
       "dissipation": eps.tolist(), "peak_t": float(t[ipk]), "peak_eps": float(eps[ipk]),
       "totals": sim.conserved_totals().tolist()}
json.dump(out, open(f"gpurun_out/tgv3d_{n}_ke.json", "w"))
print(json.dumps({k: out[k] for k in ("n", "steps", "wall_s", "peak_t", "peak_eps")}))
