"""The campaign driver's physical runner on the GPU: H2/O2 counterflow
members (BASELINE configs[4]) at several laser energies advanced together by
ign_ensemble_rk3_steps, product traces from the device tree reduction,
detect_ignition on them; run_batch with HF (GPU ensemble) and LF (coarse GPU
grids, FIFO) pools."""
import pytest

from paper_2202_02319_b200 import campaign as cp

pytestmark = pytest.mark.gpu


def test_counterflow_runner_batch_equals_solo(cuda_device):
    run = cp.CounterflowRunner(nx=64, ny=32, t_end=6e-6, trace_every=10, window=1e-6)
    outs = run.batch([0.02, 0.5, 50.0])
    assert len(outs) == 3
    assert all(isinstance(o[0], bool) for o in outs[:2])
    assert run(0.5) == outs[1]  # a member of the batch = the same sample alone
    # an over-driven member fails alone (its exception is its result)
    if isinstance(outs[2], Exception):
        assert "ailure" in str(outs[2]) or "state" in str(outs[2]).lower()
    assert 0.2 < run.y_max < 0.5


def test_run_batch_on_gpu_pools(tmp_path, cuda_device):
    hf = cp.CounterflowRunner(nx=64, ny=32, t_end=5e-6, trace_every=10, window=1e-6)
    lf = cp.CounterflowRunner(nx=32, ny=16, t_end=5e-6, trace_every=10, window=1e-6)
    specs = [cp.RunSpec(e, "HF", k, str(tmp_path / f"sample{k}"))
             for k, e in enumerate((0.05, 0.5))]
    specs += [cp.RunSpec(e, "LF", 2 + k, str(tmp_path / f"sample{2 + k}"))
              for k, e in enumerate((0.05, 0.5, 2.0))]
    recs, rep = cp.run_batch(specs, cp.PoolConfig(hf_workers=2, lf_workers=2), hf.hf_runner(), lf)
    assert [r.status for r in recs[:4]] == ["ok"] * 4, [r.error for r in recs]
    assert rep["total_walltime_s"] > 0.0
