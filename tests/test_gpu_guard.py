"""Memory safety without compute-sanitizer (closed on the GPU pool): the
red-zone guard allocator (IGN_GUARD=1, csrc/runtime.cu dmalloc/dfree) puts
32 KB of signalling-NaN canary on both sides of every device buffer.  An
out-of-bounds write changes a canary (counted at free and by
ign_guard_status); an out-of-bounds read that is used turns the step
non-finite (StepFailure / oracle mismatch)."""
import ctypes as C
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_guard_detects_out_of_bounds_writes(product_api, cuda_device):
    n = C.c_ulonglong()
    assert product_api["guard_selftest"](cuda_device, C.byref(n)) == 0
    assert n.value == 2  # one word past the end, one before the start


@pytest.mark.gpu
def test_kernel_families_under_guard():
    """Every kernel family (2D/3D, char/comp, TENO6/WENO3Z, walls, inflow,
    LODI, laser, chemistry, slab groups with halo overlap, the ensemble) under
    the guard: no canary overwritten, no step failure from a canary read."""
    env = dict(os.environ, IGN_GUARD="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py")],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("guard ")][-1]
    assert "enabled=1" in line and "corrupted_words=0" in line, line
    checked = int(line.split("buffers_checked=")[1].split()[0])
    assert checked > 100, line
