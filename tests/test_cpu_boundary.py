"""CPU tests of the C-ABI boundary and host setup (no GPU needed)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2202_02319_b200 import abi, configs, native

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                      "include", "ignis_b200.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(ign_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = native.lib()
    syms = header_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_python_binding_covers_header():
    names = {"ign_" + n for n in abi.PUBLIC_SYMBOLS}
    assert set(header_symbols()) == names


def test_config_struct_size_matches_library():
    api = native.api()  # bind() raises on drift
    assert api["config_size"]() == C.sizeof(abi.Config)


MESHES = [
    lambda: configs.tgv2d(32),
    lambda: configs.tgv2d(32, scheme="weno3z"),
    lambda: configs.tgv2d(24, skew=0.2),
    lambda: configs.sod_strip(60),
    lambda: configs.h2o2_counterflow(20),
    lambda: configs.wall_channel(16),
]


def _host_metrics(api, cfg, which):
    P = (cfg.nx + 2 * cfg.g) * (cfg.ny + 2 * cfg.g)
    out = np.empty(5 * P)
    err = abi.Error()
    st = api["host_metrics"](C.byref(cfg), which, out.ctypes.data_as(C.POINTER(C.c_double)),
                             C.byref(err))
    return st, out


@pytest.mark.parametrize("mk", MESHES)
def test_host_metrics_bitwise_vs_reference(mk, oracle_api):
    """Mesh + compute_metrics restatement (metrics.hpp:73-118) is bit-identical."""
    cfg = mk().cfg
    api = native.api()
    for which in (0, 1):
        s1, a = _host_metrics(api, cfg, which)
        s2, b = _host_metrics(oracle_api, cfg, which)
        assert s1 == s2 == 0
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_analytic_skew_metrics_bitwise(oracle_api):
    case = configs.tgv2d(24, skew=0.15)
    case.cfg.scheme.metrics = abi.METRICS_ANALYTIC_SKEW
    s1, a = _host_metrics(native.api(), case.cfg, 0)
    s2, b = _host_metrics(oracle_api, case.cfg, 0)
    assert s1 == s2 == 0 and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_host_mesh_and_errors_match_reference(oracle_api):
    api = native.api()
    # degenerate mesh (mesh.hpp:55) and folded skew (mesh.hpp:98-105) errors
    for cfg, status in ((configs.base_config(5, 40, 1.0, 1.0), abi.IGN_CONFIG_ERROR),):
        P = (cfg.nx + 6) * (cfg.ny + 6)
        x, y = np.empty(P), np.empty(P)
        e1, e2 = abi.Error(), abi.Error()
        d = C.POINTER(C.c_double)
        s1 = api["host_mesh"](C.byref(cfg), x.ctypes.data_as(d), y.ctypes.data_as(d), C.byref(e1))
        s2 = oracle_api["host_mesh"](C.byref(cfg), x.ctypes.data_as(d), y.ctypes.data_as(d),
                                     C.byref(e2))
        assert s1 == s2 == status
        assert e1.msg == e2.msg
    case = configs.tgv2d(16, skew=0.9)
    P = 22 * 22
    x, y = np.empty(P), np.empty(P)
    e1, e2 = abi.Error(), abi.Error()
    d = C.POINTER(C.c_double)
    s1 = api["host_mesh"](C.byref(case.cfg), x.ctypes.data_as(d), y.ctypes.data_as(d), C.byref(e1))
    s2 = oracle_api["host_mesh"](C.byref(case.cfg), x.ctypes.data_as(d), y.ctypes.data_as(d),
                                 C.byref(e2))
    assert s1 == s2
    if s1 != 0:
        assert e1.msg == e2.msg


def test_create_fails_loudly_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    h = C.c_void_p()
    st = native.api()["create"](C.byref(configs.tgv2d(16).cfg), C.byref(h))
    assert st == abi.IGN_CUDA_ERROR and not h.value


def test_mixture_parser_reads_h2o2_table():
    sp = configs.h2_o2_species()
    assert [s.name for s in sp] == ["H2", "O2", "H2O", "N2"]
    W = {s.name: s.W for s in sp}
    assert 2 * W["H2"] + W["O2"] == pytest.approx(2 * W["H2O"], abs=1e-15)


def test_cpp_facade_example_compiles_and_links(tmp_path):
    """a C++ caller of the facade builds against the library."""
    import subprocess
    root = os.path.dirname(HEADER)
    lib = os.path.dirname(native.LIB)
    exe = str(tmp_path / "facade_example")
    subprocess.run(["g++", "-std=c++17", "-O2", f"-I{root}",
                    os.path.join(os.path.dirname(root), "tests", "cpp", "facade_example.cpp"),
                    f"-L{lib}", "-lignis_b200", f"-Wl,-rpath,{lib}", "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode in (0, 2), r.stdout + r.stderr


def test_drop_in_compiles_against_reference_headers(tmp_path):
    """include/ignis_b200/drop_in.hpp: the reference-typed drop-in for
    ignis::Simulation builds against the UNMODIFIED reference headers and links
    the library (tests/cpp/drop_in_parity.cpp; run on the GPU by
    tests/test_gpu_boundary.py)."""
    import subprocess
    from tests.conftest import REFERENCE_INCLUDE, has_reference_sources
    if not has_reference_sources():
        pytest.skip("reference headers absent")
    root = os.path.dirname(HEADER)
    lib = os.path.dirname(native.LIB)
    exe = str(tmp_path / "drop_in_parity")
    repo = os.path.dirname(root)
    subprocess.run(["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-pthread",
                    f"-I{REFERENCE_INCLUDE}", f"-I{root}",
                    f'-DREPO_DATA_DIR="{repo}/data"',
                    os.path.join(repo, "tests", "cpp", "drop_in_parity.cpp"),
                    f"-L{lib}", "-lignis_b200", f"-Wl,-rpath,{lib}", "-o", exe], check=True)
    assert os.path.exists(exe)
