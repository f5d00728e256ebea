"""Small cases over every kernel family for compute-sanitizer (one tool per
call): 2D gamma-gas TENO6 char + viscous, 2D H2/O2 inflow/outflow/laser (WENO3Z
comp too), 3D TGV, the 3D jet (inflow, LODI, walls, shaped 3D laser), slab
groups (2D and 3D, halo overlap) and the ensemble runner.  compute-sanitizer
is closed on the GPU pool: run with IGN_GUARD=1 (red-zone allocator) instead;
the script exits 1 if any buffer's canaries were overwritten."""
import sys
sys.path.insert(0, '.')
from paper_2202_02319_b200 import Ensemble, Simulation, configs
from paper_2202_02319_b200.sim import SlabGroup


def run(case, steps=2):
    s = Simulation(case.cfg)
    s.set_initial_condition(case.ic)
    s.prepare_stage(1)
    s.rk3_steps(case.dt, steps)
    s.stable_dt()
    s.compute_rhs(0.0, 1)
    s.conserved_totals()
    s.close()


run(configs.tgv2d(24))
run(configs.h2o2_counterflow(24))
run(configs.h2o2_counterflow(24, scheme="weno3z", split="comp"))
run(configs.sod_strip(60))
run(configs.species_box(8, 24, laser="shaped"))
run(configs.tgv3d(12))
run(configs.jet3d(48, 24, 12), 1)
for mk, three in ((lambda: configs.tgv2d(24), False), (lambda: configs.tgv3d(12, nz=18), True)):
    case = mk()
    single = Simulation(case.cfg)
    single.set_initial_condition(case.ic)
    U = single.Ut
    grp = SlabGroup(case.cfg, 2)
    n = case.cfg.nz if three else case.cfg.ny
    half = n // 2
    grp.set_state(0, U[:, 0:half + 6] if three else U[:, 0:half + 6, :])
    grp.set_state(1, U[:, half:n + 6] if three else U[:, half:n + 6, :])
    grp.prepare_stage(1)
    grp.rk3_steps(case.dt, 2)
    grp.conserved_totals()
    grp.close()
    single.close()
ens = Ensemble([c.cfg for c in configs.ensemble_members(4, nxy=(40, 20), count=2)])
for m, c in zip(ens.members, configs.ensemble_members(4, nxy=(40, 20), count=2)):
    m.set_initial_condition(c.ic)
    m.prepare_stage(1)
ens.rk3_steps(1e-8, 2)
ens.close()
# red-zone guard (IGN_GUARD=1): every freed and live buffer's canaries
import ctypes as C  # noqa: E402
from paper_2202_02319_b200 import native  # noqa: E402
en, chk, bad = C.c_int(), C.c_ulonglong(), C.c_ulonglong()
native.api()["guard_status"](C.byref(en), C.byref(chk), C.byref(bad))
print(f"guard enabled={en.value} buffers_checked={chk.value} corrupted_words={bad.value}")
if bad.value:
    sys.exit(1)
print("sanitize cases ok")
