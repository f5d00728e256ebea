"""Ensemble campaign driver — the SPEC's `ensemble` module (
SURVEY §8(f)4), which the reference specifies but does not implement.

* ``detect_ignition``       — product-trace threshold + trailing monotonicity
                              (SPEC [OP] detect_ignition; PAPER §4.1.2);
* ``bisection_min_energy``  — minimum ignition energy by bisection on E_L with a
                              persisted, restartable ledger and a checked
                              monotone-physics assumption (SPEC [OP]
                              bisection_min_energy; PAPER §6.6.2);
* ``sweep_minimum_energy``  — one campaign per laser duration sigma_t, CSV
                              table (SPEC [OP] sweep_minimum_energy; Fig. 3d);
* ``run_batch``             — HF samples batched on the GPU (one context per
                              member, advanced together by
                              ign_ensemble_rk3_steps) concurrently with a FIFO
                              LF pool of coarse-grid samples (SPEC [OP]
                              run_batch; PAPER §3.2.2).  The reference's HF/LF
                              split maps onto processor kinds (GPU vs CPU); this
                              build has no CPU solver (no CPU fallback by
                              design), so LF samples are coarse grids on the GPU,
                              each on its own stream, queued FIFO.
* ``CounterflowRunner``     — the physical runner: the H2/O2 counterflow
                              member of BASELINE configs[4] at energy E, its
                              product trace sampled on the device, ignition
                              detected from it.

Everything above the runner is plain host logic (tested on CPU with synthetic
predicates); the runner drives the B200 path through the C ABI.
"""
from __future__ import annotations

import csv
import json
import math
import os
import queue
import threading
import time
from dataclasses import asdict, dataclass, field
from typing import Callable, Dict, List, Optional, Sequence, Tuple

import numpy as np

from .errors import ConfigError, UsageError


class BracketError(ConfigError):
    """The initial interval does not bracket: a ignites or b fails."""


class NonMonotonicError(UsageError):
    """A recorded failure lies above a recorded success (SPEC invariant)."""


class InsufficientDataError(UsageError):
    """The trace does not extend the required window past the deployment."""


# ---------------------------------------------------------------- ignition
def detect_ignition(times: Sequence[float], values: Sequence[float], t0: float, window: float,
                    y_max: float, theta: float = 0.1) -> Tuple[bool, Optional[float]]:
    """SPEC [OP] detect_ignition: ignited iff the product trace exceeds theta
    * y_max and is non-decreasing over the trailing `window`; t_ign = the first
    crossing time minus t0.  The trace must extend `window` past t0."""
    t = np.asarray(times, dtype=np.float64)
    y = np.asarray(values, dtype=np.float64)
    if t.size == 0 or t[-1] < t0 + window:
        raise InsufficientDataError(
            f"detect_ignition: trace ends at {t[-1] if t.size else None}, needs t0 + window = "
            f"{t0 + window}")
    thr = theta * y_max
    above = np.nonzero(y > thr)[0]
    if above.size == 0:
        return False, None
    tail = y[t >= t[-1] - window]
    if tail.size > 1 and np.any(np.diff(tail) < 0.0):
        return False, None
    return True, float(t[above[0]] - t0)


# ---------------------------------------------------------------- ledger
@dataclass
class Outcome:
    energy: float
    ignited: bool
    t_ign: Optional[float] = None
    walltime_s: float = 0.0


class Ledger:
    """Evaluated samples, persisted as JSON after every record (restartable);
    outcomes are immutable once recorded (SPEC [TYPE] Campaign)."""

    def __init__(self, path: Optional[str] = None):
        self.path = path
        self.records: Dict[str, Outcome] = {}
        if path and os.path.exists(path):
            with open(path) as f:
                for k, v in json.load(f).items():
                    self.records[k] = Outcome(**v)

    @staticmethod
    def key(energy: float) -> str:
        return repr(float(energy))

    def get(self, energy: float) -> Optional[Outcome]:
        return self.records.get(self.key(energy))

    def record(self, out: Outcome):
        k = self.key(out.energy)
        if k in self.records:
            raise UsageError(f"ledger: energy {out.energy} already recorded (immutable)")
        self.records[k] = out
        if self.path:
            tmp = self.path + ".tmp"
            with open(tmp, "w") as f:
                json.dump({kk: asdict(v) for kk, v in self.records.items()}, f, indent=1)
            os.replace(tmp, self.path)

    def check_monotone(self):
        fails = [o.energy for o in self.records.values() if not o.ignited]
        wins = [o.energy for o in self.records.values() if o.ignited]
        if fails and wins and max(fails) > min(wins):
            raise NonMonotonicError(
                f"non-monotone outcomes: failure at {max(fails)} above success at {min(wins)}")


@dataclass
class Campaign:
    """SPEC [TYPE] Campaign: search variable E_L on [a, b] to tolerance."""
    a: float
    b: float
    tol: float
    sigma_t: float = 1e-6
    ledger_path: Optional[str] = None
    status: str = "new"
    evaluations: int = 0  # runner calls made by this process (ledger hits excluded)


Runner = Callable[[float], Tuple[bool, Optional[float]]]


def _evaluate(c: Campaign, led: Ledger, runner: Runner, energy: float) -> Outcome:
    hit = led.get(energy)
    if hit is not None:
        return hit
    t0 = time.perf_counter()
    ign, t_ign = runner(energy)
    out = Outcome(float(energy), bool(ign), t_ign, time.perf_counter() - t0)
    c.evaluations += 1
    led.record(out)
    led.check_monotone()
    return out


def bisection_min_energy(c: Campaign, runner: Runner) -> Tuple[float, Ledger]:
    """SPEC [OP] bisection_min_energy: after bracketing (a fails, b ignites),
    halve [a, b] at the midpoint until b - a <= tol; returns the final
    midpoint.  Every evaluation is persisted; a restart reuses the ledger with
    zero repeated evaluations."""
    led = Ledger(c.ledger_path)
    a, b = float(c.a), float(c.b)
    if not a < b:
        raise BracketError("bisection: need a < b")
    if _evaluate(c, led, runner, a).ignited:
        raise BracketError(f"bisection: the lower end a = {a} ignites")
    if not _evaluate(c, led, runner, b).ignited:
        raise BracketError(f"bisection: the upper end b = {b} does not ignite")
    c.status = "running"
    # resume: tighten with every recorded energy inside the bracket first
    for o in sorted(led.records.values(), key=lambda o: o.energy):
        if a < o.energy < b:
            if o.ignited:
                b = min(b, o.energy)
            else:
                a = max(a, o.energy)
    while b - a > c.tol:
        m = 0.5 * (a + b)
        if _evaluate(c, led, runner, m).ignited:
            b = m
        else:
            a = m
    c.a, c.b, c.status = a, b, "converged"
    return 0.5 * (a + b), led


def sweep_minimum_energy(sigma_ts: Sequence[float], template: Campaign,
                         runner_for: Callable[[float], Runner],
                         csv_path: Optional[str] = None) -> List[dict]:
    """SPEC [OP] sweep_minimum_energy: one bisection campaign per sigma_t;
    bracket failures are recorded and the sweep continues."""
    rows = []
    for st in sigma_ts:
        c = Campaign(template.a, template.b, template.tol, sigma_t=st,
                     ledger_path=(template.ledger_path.format(sigma_t=st)
                                  if template.ledger_path else None))
        try:
            e, _ = bisection_min_energy(c, runner_for(st))
            rows.append({"sigma_t": st, "E_min": e, "error": ""})
        except (BracketError, NonMonotonicError) as exc:
            rows.append({"sigma_t": st, "E_min": None, "error": str(exc)})
    if csv_path:
        with open(csv_path, "w", newline="") as f:
            w = csv.DictWriter(f, fieldnames=["sigma_t", "E_min", "error"])
            w.writeheader()
            w.writerows(rows)
    return rows


# ---------------------------------------------------------------- batches
@dataclass
class RunSpec:
    """SPEC [TYPE] RunSpec: one sample's resolved parameters."""
    energy: float
    fidelity: str = "HF"  # "HF" | "LF"
    index: int = 0
    outdir: str = ""
    sigma_t: Optional[float] = None


@dataclass
class PoolConfig:
    """SPEC [TYPE] PoolConfig: HF members per GPU batch, LF workers (FIFO)."""
    hf_workers: int = 8
    lf_workers: int = 2


@dataclass
class SampleResult:
    index: int
    fidelity: str
    energy: float
    status: str
    ignited: Optional[bool] = None
    t_ign: Optional[float] = None
    walltime_s: float = 0.0
    started_s: float = 0.0
    error: str = ""
    outdir: str = ""


# per spec: (ignited, t_ign), or the member's exception (its failure is its result)
BatchRunner = Callable[[List[RunSpec]], List]


def run_batch(specs: Sequence[RunSpec], pools: PoolConfig, hf_runner: BatchRunner,
              lf_runner: Runner) -> Tuple[List[SampleResult], dict]:
    """SPEC [OP] run_batch: HF samples in batches of `hf_workers` (one
    hf_runner call per batch: the GPU ensemble) concurrently with the LF pool
    (`lf_workers` threads taking LF samples in FIFO order).  One sample's
    failure never aborts the others; returns per-sample records (in index
    order) and a walltime report."""
    for s in specs:
        if s.fidelity not in ("HF", "LF"):
            raise ConfigError(f"run_batch: fidelity must be HF or LF, got {s.fidelity!r}")
    hf = [s for s in specs if s.fidelity == "HF"]
    lf = [s for s in specs if s.fidelity == "LF"]
    if hf and pools.hf_workers < 1 or lf and pools.lf_workers < 1:
        raise ConfigError("run_batch: worker counts must be >= 1 for a used fidelity")
    for s in specs:
        if s.outdir:
            os.makedirs(s.outdir, exist_ok=True)
    results: Dict[int, SampleResult] = {}
    lock = threading.Lock()
    t_start = time.perf_counter()

    def hf_loop():
        for k in range(0, len(hf), pools.hf_workers):
            group = hf[k:k + pools.hf_workers]
            t0 = time.perf_counter()
            try:
                raw = hf_runner(group)
                # a batch runner reports a member's own failure as an exception
                # instance in its slot
                outs = [(None, None) if isinstance(o, Exception) else o for o in raw]
                errs = [str(o) if isinstance(o, Exception) else "" for o in raw]
            except Exception as exc:  # noqa: BLE001 — recorded per sample
                outs = [(None, None)] * len(group)
                errs = [str(exc)] * len(group)
            el = time.perf_counter() - t0
            with lock:
                for s, (ign, t_ign), e in zip(group, outs, errs):
                    results[s.index] = SampleResult(
                        s.index, "HF", s.energy, "failed" if e else "ok", ign, t_ign, el,
                        t0 - t_start, e, s.outdir)

    q: "queue.Queue[RunSpec]" = queue.Queue()
    for s in lf:  # FIFO
        q.put(s)

    def lf_worker():
        while True:
            try:
                s = q.get_nowait()
            except queue.Empty:
                return
            t0 = time.perf_counter()
            try:
                ign, t_ign = lf_runner(s.energy)
                rec = SampleResult(s.index, "LF", s.energy, "ok", ign, t_ign,
                                   time.perf_counter() - t0, t0 - t_start, "", s.outdir)
            except Exception as exc:  # noqa: BLE001
                rec = SampleResult(s.index, "LF", s.energy, "failed", None, None,
                                   time.perf_counter() - t0, t0 - t_start, str(exc), s.outdir)
            with lock:
                results[s.index] = rec

    threads = [threading.Thread(target=hf_loop)] if hf else []
    threads += [threading.Thread(target=lf_worker) for _ in range(pools.lf_workers if lf else 0)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    total = time.perf_counter() - t_start
    recs = [results[s.index] for s in specs]
    report = {
        "total_walltime_s": total,
        "hf_walltime_s": sum({r.started_s: r.walltime_s for r in recs if r.fidelity == "HF"}
                             .values()),
        "lf_cumulative_s": sum(r.walltime_s for r in recs if r.fidelity == "LF"),
        "failed": [r.index for r in recs if r.status != "ok"],
    }
    return recs, report


# ---------------------------------------------------------------- the physical runner
def max_product_mole_fraction(species, Y_fuel, Y_ox, nu, i_fuel, i_ox, i_prod,
                              nz: int = 2001) -> float:
    """Theoretical maximum of the product mole fraction of the two-stream
    counterflow: complete one-step conversion of the limiting reactant at
    every mixture fraction Z, maximised over Z (detect_ignition's y_max)."""
    W = np.array([sp.W for sp in species])
    best = 0.0
    for Z in np.linspace(0.0, 1.0, nz):
        Y = Z * np.asarray(Y_fuel) + (1.0 - Z) * np.asarray(Y_ox)
        n = Y / W  # moles per unit mass
        # extent: reactant k consumed nu_k per unit extent (nu < 0)
        ext = min(n[i_fuel] / -nu[i_fuel], n[i_ox] / -nu[i_ox])
        n2 = n + ext * np.asarray(nu)[: len(n)]
        best = max(best, n2[i_prod] / n2.sum())
    return float(best)


class CounterflowRunner:
    """BASELINE configs[4]'s member: the H2/O2 counterflow (configs.
    h2o2_counterflow) on an nx x ny grid at laser energy E (and sigma_t),
    advanced to t_end with a pinned dt; the product mole fraction
    (ign_product_mole_fraction, device tree sums) sampled every
    `trace_every` steps; ignition by detect_ignition.  ``batch(specs)`` runs
    several energies together through ign_ensemble_rk3_steps (HF pool)."""

    def __init__(self, nx: int = 500, ny: int = 250, t_end: float = 2e-5,
                 trace_every: int = 10, window: Optional[float] = None, theta: float = 0.1,
                 sigma_t: Optional[float] = None, device: int = 0):
        from . import configs
        self.configs = configs
        self.nx, self.ny, self.t_end = nx, ny, t_end
        self.trace_every, self.theta, self.sigma_t, self.device = (
            trace_every, theta, sigma_t, device)
        base = self._case(0.05)
        la = base.cfg.laser
        self.t0 = la.t0
        self.window = window if window is not None else max(0.0, t_end - la.t0) * 0.25
        sp = configs.h2_o2_species()
        m = base.cfg.mech
        nu = [m.nu[k] for k in range(len(sp))]
        self.y_max = max_product_mole_fraction(
            sp, [0.1, 0.0, 0.0, 0.9], [0.0, 0.23, 0.0, 0.77], nu, m.i_fuel, m.i_ox, m.i_h2o)

    def _case(self, energy: float):
        c = self.configs.h2o2_counterflow(self.nx, nxy=(self.nx, self.ny), energy=energy)
        if self.sigma_t is not None:
            c.cfg.laser.sigma_t = self.sigma_t
        c.cfg.device = self.device
        return c

    def batch(self, energies: Sequence[float]) -> List[Tuple[bool, Optional[float]]]:
        from .sim import Ensemble
        cases = [self._case(float(e)) for e in energies]
        ens = Ensemble([c.cfg for c in cases])
        try:
            for m, c in zip(ens.members, cases):
                m.set_initial_condition(c.ic)
                m.prepare_stage(1)
            dt = min(c.dt for c in cases)
            nsteps = int(math.ceil(self.t_end / dt))
            times = [[] for _ in cases]
            vals = [[] for _ in cases]
            errs: List[Optional[Exception]] = [None] * len(cases)
            done = 0
            while done < nsteps:
                live = [q for q in range(len(cases)) if errs[q] is None]
                if not live:
                    break
                k = min(self.trace_every, nsteps - done)
                try:
                    st = ens.rk3_steps(dt, k, only=live)
                except Exception:  # noqa: BLE001 — every live member failed
                    st = [1 if q in live else 0 for q in range(len(cases))]
                done += k
                for q in live:
                    if st[q] != 0:  # a failed member stops; its error is its result
                        errs[q] = ens.error(q) or UsageError(f"member {q} failed")
                        continue
                    m = ens.members[q]
                    times[q].append(m.time)
                    vals[q].append(m.product_mole_fraction())
            out: List = []
            for q in range(len(cases)):
                if errs[q] is not None:
                    out.append(errs[q])
                else:
                    out.append(detect_ignition(times[q], vals[q], self.t0, self.window,
                                               self.y_max, self.theta))
            return out
        finally:
            ens.close()

    def __call__(self, energy: float) -> Tuple[bool, Optional[float]]:
        r = self.batch([energy])[0]
        if isinstance(r, Exception):
            raise r
        return r

    def hf_runner(self) -> BatchRunner:
        return lambda specs: self.batch([s.energy for s in specs])
