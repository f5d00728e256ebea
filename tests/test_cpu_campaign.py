"""The ensemble campaign driver's host logic (paper_2202_02319_b200/campaign.py)
against the SPEC's own examples ('ensemble' module), with
synthetic predicates — no GPU."""
import json
import time

import numpy as np
import pytest

from paper_2202_02319_b200 import campaign as cp


def test_bisection_synthetic_predicate_six_evaluations(tmp_path):
    """SPEC: ignites iff E >= 0.5 on [0,1], tol 1/64 -> within 1/64 of 0.5,
    exactly 6 evaluations after bracketing."""
    calls = []

    def runner(e):
        calls.append(e)
        return e >= 0.5, (1.0 if e >= 0.5 else None)
    c = cp.Campaign(0.0, 1.0, 1.0 / 64, ledger_path=str(tmp_path / "ledger.json"))
    est, led = cp.bisection_min_energy(c, runner)
    assert abs(est - 0.5) <= 1.0 / 64
    assert len(calls) == 2 + 6 and calls[:2] == [0.0, 1.0]
    assert c.b - c.a <= 1.0 / 64 and c.status == "converged"
    assert len(json.load(open(tmp_path / "ledger.json"))) == 8


def test_bisection_already_converged():
    """SPEC: tol >= b - a -> the midpoint, 0 bisection evaluations."""
    calls = []

    def runner(e):
        calls.append(e)
        return e >= 0.5, None
    est, _ = cp.bisection_min_energy(cp.Campaign(0.0, 1.0, 2.0), runner)
    assert est == 0.5 and len(calls) == 2  # the two bracketing runs only


def test_bisection_bracket_errors():
    with pytest.raises(cp.BracketError):
        cp.bisection_min_energy(cp.Campaign(0.6, 1.0, 0.01), lambda e: (e >= 0.5, None))
    with pytest.raises(cp.BracketError):
        cp.bisection_min_energy(cp.Campaign(0.0, 0.4, 0.01), lambda e: (e >= 0.5, None))


def test_bisection_restart_repeats_nothing(tmp_path):
    """SPEC: a restart resumes from the persisted ledger with zero repeated
    evaluations."""
    path = str(tmp_path / "l.json")
    calls = []

    def flaky(e):
        calls.append(e)
        if len(calls) == 5:
            raise RuntimeError("node lost")
        return e >= 0.37, None
    with pytest.raises(RuntimeError):
        cp.bisection_min_energy(cp.Campaign(0.0, 1.0, 1.0 / 128, ledger_path=path), flaky)
    seen = list(calls)
    calls.clear()
    c = cp.Campaign(0.0, 1.0, 1.0 / 128, ledger_path=path)
    est, led = cp.bisection_min_energy(c, lambda e: (calls.append(e), (e >= 0.37, None))[1])
    assert not set(calls) & set(seen[:4])  # recorded energies never re-run
    assert abs(est - 0.37) <= 1.0 / 128
    assert c.evaluations == len(calls)


def test_non_monotone_outcomes_halt(tmp_path):
    """SPEC invariant: a recorded failure above a recorded success halts the
    campaign (bisection itself keeps failures <= a < b <= successes, so a
    violation comes from a reused ledger, e.g. a restart after the physics
    changed)."""
    path = str(tmp_path / "l.json")
    led = cp.Ledger(path)
    led.record(cp.Outcome(0.6, True))
    led.record(cp.Outcome(0.75, False))
    with pytest.raises(cp.NonMonotonicError):
        led.check_monotone()
    with pytest.raises(cp.NonMonotonicError):
        cp.bisection_min_energy(cp.Campaign(0.0, 1.0, 0.01, ledger_path=path),
                                lambda e: (e >= 0.5, None))
    with pytest.raises(Exception):
        led.record(cp.Outcome(0.6, False))  # outcomes are immutable


def test_detect_ignition_examples():
    t = np.linspace(0.0, 20.0, 201)
    # identically-zero trace -> not ignited
    assert cp.detect_ignition(t, np.zeros_like(t), 1.0, 5.0, y_max=1.0) == (False, None)
    # monotone ramp crossing theta at t0 + 5 -> ignited, t_ign = 5
    t0 = 2.0
    y = np.clip((t - t0) / 50.0, 0.0, None)  # 0.1 at t = t0 + 5
    ign, ti = cp.detect_ignition(t, y + 1e-12 * (t > t0 + 5.0), t0, 5.0, y_max=1.0)
    assert ign and abs(ti - 5.0) <= 0.1 + 1e-9
    # above threshold but decaying over the trailing window -> not ignited
    ydec = np.where(t < 10, t / 10.0, 1.0 - (t - 10) / 20.0)
    assert cp.detect_ignition(t, ydec, 0.0, 5.0, y_max=1.0)[0] is False
    with pytest.raises(cp.InsufficientDataError):
        cp.detect_ignition(t[:10], y[:10], 0.5, 5.0, y_max=1.0)


def test_run_batch_hf_lf_concurrency_and_fifo(tmp_path):
    """SPEC: HF batches run concurrently with the FIFO LF pool; a sample's
    failure is recorded without aborting the others; LF cumulative time grows
    with k; total walltime is dominated by the HF sample."""
    def hf_runner(specs):
        time.sleep(0.3)
        return [(s.energy >= 0.5, 1.0) for s in specs]
    order = []

    def lf_runner(e):
        order.append(e)
        time.sleep(0.02)
        if e == 0.13:
            raise RuntimeError("LF sample diverged")
        return e >= 0.5, None
    specs = [cp.RunSpec(0.7, "HF", 0, str(tmp_path / "sample0"))]
    specs += [cp.RunSpec(0.1 + 0.01 * k, "LF", 1 + k, str(tmp_path / f"sample{1 + k}"))
              for k in range(6)]
    recs, rep = cp.run_batch(specs, cp.PoolConfig(hf_workers=8, lf_workers=1), hf_runner,
                             lf_runner)
    assert [r.index for r in recs] == list(range(7))
    assert order == [0.1 + 0.01 * k for k in range(6)]  # FIFO with one worker
    assert recs[0].status == "ok" and recs[0].ignited is True
    failed = [r.index for r in recs if r.status == "failed"]
    assert failed == [4] and "diverged" in recs[4].error
    assert rep["total_walltime_s"] < 1.10 * rep["hf_walltime_s"] + 0.05
    assert (tmp_path / "sample3").is_dir()


def test_sweep_records_bracket_failures_and_continues(tmp_path):
    rows = cp.sweep_minimum_energy(
        [0.2, 0.5, 1.0], cp.Campaign(0.0, 1.0, 1.0 / 32),
        lambda st: (lambda e: (e >= 0.3 * st if st < 1.0 else e >= 2.0, None)),
        csv_path=str(tmp_path / "sweep.csv"))
    assert [r["sigma_t"] for r in rows] == [0.2, 0.5, 1.0]
    assert abs(rows[0]["E_min"] - 0.06) <= 1.0 / 32 and abs(rows[1]["E_min"] - 0.15) <= 1.0 / 32
    assert rows[2]["E_min"] is None and "does not ignite" in rows[2]["error"]
    assert cp.sweep_minimum_energy([], cp.Campaign(0, 1, 0.1), None) == []
    assert (tmp_path / "sweep.csv").read_text().startswith("sigma_t,E_min,error")


def test_theoretical_max_product_fraction():
    from paper_2202_02319_b200 import configs
    sp = configs.h2_o2_species()
    y = cp.max_product_mole_fraction(sp, [0.1, 0, 0, 0.9], [0, 0.23, 0, 0.77],
                                     [-2.0, -1.0, 2.0, 0.0], 0, 1, 2)
    assert 0.2 < y < 0.5
