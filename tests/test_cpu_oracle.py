"""Pins the CPU oracle (TEST INFRASTRUCTURE) before it is trusted:

* the reference's OWN Catch2 unit tests (reference/proj/tests/*.cpp), compiled
  unmodified against the reference headers with a minimal Catch2 shim;
* the product's point physics (csrc/physics.cuh, flux.cuh) compiled for the
  host, bitwise against the reference functions;
* committed golden fixtures (tests/golden/*.npz, made by make_golden.py) vs
  the oracle build that travels to the GPU box;
* the reference's determinism contract (thread_team.hpp:13-17).
"""
import os
import subprocess

import numpy as np
import pytest

from paper_2202_02319_b200 import configs
from tests.conftest import REFERENCE_INCLUDE, ROOT, has_reference_sources

needs_src = pytest.mark.skipif(not has_reference_sources(), reason="reference sources absent")
REF_TESTS = ["reconstruction", "flux", "thermo", "chemistry", "laser", "mesh_metrics"]
# Two of the reference's own cases fail on the reference itself:
# test_flux.cpp:72-90 applies an absolute 1e-11 margin to L*R entries whose
# energy components are O(1e6) in SI units, and test_flux.cpp:92-138 perturbs
# U by 1e-7*|E| (~0.1 kg/m^3) so primitives_from_conservative throws
# "energy below vacuum energy".  Everything else passes.
KNOWN_REFERENCE_FAILURES = {"eigen projection and assembly invert each other",
                            "eigen decomposition reproduces the flux jacobian"}


def _compile(src, out, extra=()):
    cmd = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-DNDEBUG",
           f"-I{ROOT}/tests/cpp", f"-I{REFERENCE_INCLUDE}",
           '-DIGNIS_DATA_DIR="/root/reference/proj/data"', *extra, src, "-o", out]
    subprocess.run(cmd, check=True, capture_output=True)


@needs_src
@pytest.mark.parametrize("name", REF_TESTS)
def test_reference_unit_tests(name, tmp_path):
    exe = str(tmp_path / name)
    _compile(f"/root/reference/proj/tests/test_{name}.cpp", exe)
    r = subprocess.run([exe], capture_output=True, text=True)
    failed = {ln[5:].rsplit(":", 1)[0] for ln in r.stdout.splitlines()
              if ln.startswith("TEST ") and ln.endswith("FAIL")}
    assert failed <= KNOWN_REFERENCE_FAILURES, r.stdout[-2000:]


@needs_src
def test_product_physics_bitwise_vs_reference(tmp_path):
    exe = str(tmp_path / "physics_parity")
    _compile(f"{ROOT}/tests/cpp/physics_parity.cpp", exe,
             (f"-I{ROOT}/include", f"-I{ROOT}/paper_2202_02319_b200/csrc",
              f'-DREPO_DATA_DIR="{ROOT}/data"',
              f"{ROOT}/paper_2202_02319_b200/csrc/host_core.cpp"))
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-3000:]
    assert "0 mismatches" in r.stdout


GOLDEN = os.path.join(ROOT, "tests", "golden")


@pytest.mark.parametrize("name", sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz")))
def test_oracle_matches_golden_fixture(name, oracle_api):
    from tests.golden.make_golden import CASES, generate
    mk, n = CASES[name]
    got = generate(name, mk, n)
    want = np.load(os.path.join(GOLDEN, name + ".npz"))
    for k in want.files:
        assert np.array_equal(np.asarray(got[k]).view(np.uint64) if np.asarray(got[k]).dtype == np.float64 else got[k],
                              want[k].view(np.uint64) if want[k].dtype == np.float64 else want[k]), k


def test_oracle_partition_invariance(oracle_api):
    """thread_team.hpp:13-17: results independent of the worker count."""
    from oracle import ref
    out = []
    for parts in (1, 4):
        case = configs.tgv2d(32)
        sim = ref.simulation(case.cfg, partitions=parts)
        sim.set_initial_condition(case.ic)
        sim.prepare_stage(1)
        sim.rk3_steps(case.dt, 3)
        out.append(sim.Ut)
    assert np.array_equal(out[0].view(np.uint64), out[1].view(np.uint64))


def test_oracle_periodic_conservation(oracle_api):
    from oracle import ref
    case = configs.tgv2d(32)
    sim = ref.simulation(case.cfg)
    sim.set_initial_condition(case.ic)
    sim.prepare_stage(1)
    t0 = sim.conserved_totals()
    sim.rk3_steps(case.dt, 5)
    t1 = sim.conserved_totals()
    assert abs(t1[0] - t0[0]) <= 1e-13 * abs(t0[0])
    assert abs(t1[3] - t0[3]) <= 1e-13 * abs(t0[3])


@pytest.mark.parametrize("src,n", [("hypot_check.c", 20000000), ("pow2_check.c", 100000000),
                                   ("fdiv_check.cpp", 20000000)])
def test_libm_restatements_bitwise(tmp_path, src, n):
    """The exact rewrites DESIGN.md §3 relies on, checked against the host libm
    / IEEE division: glibc hypot restated (ghypot), pow(z, 2) == z*z (shaped
    laser), Markstein division (fdiv)."""
    exe = str(tmp_path / src.split(".")[0])
    cc = "gcc" if src.endswith(".c") else "g++"
    cmd = [cc, "-O2", "-ffp-contract=off", f"-I{ROOT}/paper_2202_02319_b200/csrc",
           f"-I{ROOT}/include", f"{ROOT}/tests/cpp/{src}", "-o", exe, "-lm"]
    if cc == "g++":
        cmd.insert(1, "-std=c++17")
    subprocess.run(cmd, check=True, capture_output=True)
    r = subprocess.run([exe, str(n)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-1000:]
