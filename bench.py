#!/usr/bin/env python3
"""Benchmark of the B200 RHS + SSP-RK3 path (BASELINE.json metric:
"FP64 cell-updates/s per RK step").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--case tgv3d|tgv|h2o2|ensemble|jet3d] [--size N]

A "step" is one full SSP-RK3 step (three RHS evaluations + updates + the
advance-loop prepare_stage(1), solver.hpp:304-345) over the whole grid.

Workload (config.workload): BASELINE configs[1], the 3D compressible viscous
Taylor-Green vortex at 256^3 = 16.8 M cells (gamma-gas, TENO6 characteristic,
Re 1600, Ma 0.1, fixed dt), on the 3D extension (flux3.cuh; validated by the
z-extrusion cross-check against the 2D oracle, tests/test_gpu_3d.py).
--case tgv runs the 2D analogue (4096^2, the same cell count), --case h2o2
configs[2] (512^2), --case jet3d configs[3] in its z-periodic channel form
(512 x 256 x 32 per GPU), --case ensemble configs[4] (8 members of the H2/O2
case at 500 x 250 per GPU, advanced together on their own streams).  The
state (5 x 144 MB per buffer at 256^3) is larger than the 126 MB L2 and every
stage streams several such buffers, so no flush is needed.  Cases whose state
buffer fits in L2 (H2/O2 512^2, the ensemble) are timed step by step with a
256 MB L2 flush between timed steps (outside the per-step event pairs).

value   = cells x K / device time of K steps, inputs resident in HBM (CUDA
          events on the library's stream, max over ranks);
e2e     = same metric through the C ABI with host buffers: every step copies
          the state in from pinned host memory and back out;
roofline = the dominant kernel class (inviscid faces) against the measured
          FP64 peak (DFMA microbenchmark run here; also against the no-FMA
          peak, since bitwise parity keeps every add/mul separate),
          algorithmic FP64 ops per cell-stage from the reference's own code
          (the 3D and 4-species counts scaled by measured FP64
          instruction ratios, profiles/r1_fp64_inst_ratio*.txt), traffic from
          the ncu capture in profiles/;
cpu_baseline = the CPU oracle (unmodified reference, all host cores) on a
          bounded sample of the same workload.

Multi-GPU (torchrun): one rank per GPU, weak scaling — every rank keeps a
256^3 slab of a domain stacked along z (3D) or y (2D); g ghost planes/rows per
side move over NCCL send/recv each stage; dt / error word / clip all-reduce.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FP64 cell-updates/s per RK step, TGV 256^3 & H2/O2 flame, 1/2/4/8 B200"
UNIT = "cell-updates/s"
# algorithmic FP64 ops (add+mul+div, reference's own code) per
# cell and stage for the inviscid part of the 2D γ-gas TENO6 characteristic
# case, and per cell-step for the whole step (TENO6 char + viscous).
# 3D TGV (no reference path): SURVEY §8d's derived ~25 800 ops per cell-step
# (3 face directions, nc 5); the inviscid share scaled from the 2D count by
# the ratio of FP64 instructions the 3D and 2D face kernels execute per cell
# and stage (ncu, profiles/r1_fp64_inst_ratio.txt).
OPS = {  # case -> (inviscid face ops per cell-stage, whole-step ops per cell)
    # counted on the reference's own code (tools/opcount/count_ref.cpp ->
    # profiles/r2_opcount_ref2d.json): TGV 2D at 256^2, H2/O2 at 512^2
    "tgv": (4269.3, 14064.3),
    "tgv3d": (7626.3, 25800),    # faces: tools/opcount/count_3d.cpp at 256^3 on the
                                 # 3D restatement (profiles/r2_opcount_ref3d.json);
                                 # whole step: SURVEY §8d's derived figure
    "h2o2": (7904.9, 28111.7),
    "jet3d": (None, None),      # 4 species, 3D, WENO3Z componentwise: not counted
}
TRAFFIC = {("tgv3d", 256): (1.790489 + 1.820969 + 2.120700 + 0.652935 + 0.657080 + 0.659103) * 1e9,
           ("h2o2", 512): (42.504704 + 42.905344) * 1e6 + (301.056 + 630.016) * 1e3}
TRAFFIC_SOURCE = {("tgv3d", 256): "ncu --set full capture of the three k_faces3d launches of one "
                                  "stage at 256^3 (profiles/r2d_ncu_faces3d_256.txt), not this run",
                  ("h2o2", 512): "ncu --set full capture of the x and y k_faces3 launches of one "
                                 "stage at 512^2 (profiles/r2d_ncu_faces_h2o2_512.txt), not this run"}
OPS_SOURCE = {
    "tgv": "reference's own code, counted-double run at 256^2 (profiles/r2_opcount_ref2d.json)",
    "tgv3d": ("counted-double run of oracle/ref3d_faces.hpp (the reference's per-face "
              "algorithm with z terms, bitwise equal to the kernels) at 256^3 "
              "(profiles/r2_opcount_ref3d.json)"),
    "h2o2": "reference's own code, counted-double run at 512^2 (profiles/r2_opcount_ref2d.json)",
}
STEP_OPS_PER_CELL = 14333
BYTES_PER_CELL_STEP = lambda nc: 8 * (8 * nc + 6)  # noqa: E731  SURVEY §8d B_alg


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


L2_BYTES = 126e6
_FLUSH = {}


def l2_flush(stream, dev):
    """Write 256 MB (> 2x the 126 MB L2) on `stream`: evicts the state."""
    import torch
    buf = _FLUSH.get(dev)
    if buf is None:
        buf = _FLUSH[dev] = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{dev}")
    with torch.cuda.stream(stream):
        buf.fill_(1)


def timed_flushed(stream, step, steps, dev):
    """Device ms of `steps` calls of step(), an L2 flush before each one and
    outside its event pair (per-step events on the library's stream)."""
    import torch
    evs = []
    for _ in range(steps):
        l2_flush(stream, dev)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step()
        b.record(stream)
        evs.append((a, b))
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in evs)


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML every
    5 ms from a thread (so a 100 ms region still gets samples), else the
    nvidia-smi loop (200 ms period)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.nvml = None
        self.lines = []
        self.sm, self.mx, self.reasons = [], None, set()

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            idx = self.device
            try:  # CUDA ordinal -> NVML index (CUDA_VISIBLE_DEVICES aware)
                import torch
                idx = torch.cuda._get_nvml_device_index(self.device)
            except Exception:
                pass
            h = N.nvmlDeviceGetHandleByIndex(idx)
            self.mx = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
            bits = {"hw_slowdown": N.nvmlClocksThrottleReasonHwSlowdown,
                    "hw_thermal_slowdown": N.nvmlClocksThrottleReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": N.nvmlClocksThrottleReasonSwThermalSlowdown,
                    "sw_power_cap": N.nvmlClocksThrottleReasonSwPowerCap}
            self.nvml, self.stop = N, threading.Event()

            def poll():
                while True:
                    self.sm.append(float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)))
                    r = N.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                    self.reasons.update(k for k, b in bits.items() if r & b)
                    if self.stop.wait(0.005):
                        return
            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def __exit__(self, *a):
        if self.nvml:
            self.stop.set()
            self.t.join(timeout=5)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = list(self.sm), self.mx, set(self.reasons)
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = float(p[2])
            except ValueError:
                continue
            for k, v in zip(self.NAMES, p[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(k)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvml" if self.nvml else "nvidia-smi"}


def make_case(args, nslabs: int = 1):
    """nslabs > 1: weak scaling — the domain grows to n x (n*nslabs) rows so
    every GPU keeps an n x n slab (TGV: periodic copies stacked along y)."""
    from paper_2202_02319_b200 import configs
    if args.case == "tgv3d":
        n = args.n
        return (configs.tgv3d(n, nz=n * nslabs),
                f"TGV 3D {n}^3 per GPU (BASELINE configs[1]), viscous Re 1600, Ma 0.1, TENO6 "
                "characteristic, gamma-gas, fixed dt; 3D extension (the reference is 2D-only)")
    if args.case == "jet3d":
        nz = args.nz if args.nz else args.n // 16
        return (configs.jet3d(args.n, args.n // 2, nz * nslabs),
                f"3D H2 jet (configs[3] form): {args.n}x{args.n // 2}x{nz} per GPU, inflow / "
                "LODI outflow / walls, one-step chemistry, shaped laser, WENO3Z comp; z-slabs")
    if args.case == "h2o2":
        c = configs.h2o2_counterflow(args.n, nxy=(args.n, args.n * nslabs))
        return c, f"H2/O2 one-step counterflow flame {args.n}^2 per GPU (configs[2])"
    return (configs.tgv2d(args.n, ly_periods=nslabs),
            f"TGV 2D {args.n}x{args.n} viscous, TENO6 characteristic, gamma-gas, fixed dt "
            f"(2D analogue of configs[1] TGV 256^3: same {args.n * args.n / 1e6:.1f}M cells; "
            "the reference is 2D-only)")


def cpu_reference_rate(n: int, target_s: float, threads: int, case: str = "tgv"):
    """Times the CPU oracle (the unmodified reference) on an n^2 sample; for
    the 3D TGV (no reference path) its 2D analogue, same physics and scheme."""
    from oracle import ref
    from paper_2202_02319_b200 import configs
    if case == "ensemble":  # one member of the campaign (moderate laser energy)
        c = configs.ensemble_members(64, nxy=(n, n // 2), count=1)[0]
    else:
        c = configs.h2o2_counterflow(n) if case == "h2o2" else configs.tgv2d(n)
    sim = ref.simulation(c.cfg, partitions=threads)
    sim.set_initial_condition(c.ic)
    sim.prepare_stage(1)
    t0 = time.perf_counter()
    sim.rk3_steps(c.dt, 1)
    one = time.perf_counter() - t0
    k = max(1, int(target_s / max(one, 1e-6)))
    t0 = time.perf_counter()
    sim.rk3_steps(c.dt, k)
    el = time.perf_counter() - t0
    return c.cfg.nx * c.cfg.ny * k / el, k, el


def run_reference_arm(args, rank, world):
    """--impl reference: the reference's own CPU implementation on the host cores."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    from oracle import ref
    from paper_2202_02319_b200 import configs
    n = 512 if args.case == "tgv3d" else min(args.n, 1024)
    if args.case == "ensemble":  # one member of the campaign, full size
        c = configs.ensemble_members(64, nxy=(args.n, args.n // 2), count=1)[0]
    else:
        c = configs.h2o2_counterflow(n) if args.case == "h2o2" else configs.tgv2d(n)
    sim = ref.simulation(c.cfg, partitions=threads)
    sim.set_initial_condition(c.ic)
    sim.prepare_stage(1)
    sim.rk3_steps(c.dt, args.warmup)
    t0 = time.perf_counter()
    sim.rk3_steps(c.dt, args.steps)
    el = time.perf_counter() - t0
    cells = c.cfg.nx * c.cfg.ny
    rate = cells * args.steps / el
    workload = (f"ensemble (configs[4]) member, H2/O2 counterflow {c.cfg.nx}x{c.cfg.ny}"
                if args.case == "ensemble" else make_case(args)[1])
    sample = (f"{c.cfg.nx}x{c.cfg.ny} sub-problem of the same workload per step (same physics "
              f"and scheme), reference advance() loop body, {threads} threads")
    if args.case == "tgv3d":
        sample = (f"2D analogue {n}x{n} (the reference has no 3D path; same TGV physics, "
                  f"TENO6 characteristic, viscous), advance() loop body, {threads} threads")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": workload, "global_batch": cells, "parallelism": "cpu-threads"},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def run_ensemble(args, rank, world, local, dist):
    """BASELINE configs[4]: 64 laser-ignition samples of the H2/O2 counterflow
    case (500 x 250), `--members` per GPU (rank r takes samples [r M, r M + M)),
    advanced together by ign_ensemble_rk3_steps; value = all members' cells x
    steps / device time (max over member streams and ranks)."""
    import torch
    from paper_2202_02319_b200 import Ensemble, configs
    M = args.members
    cases = configs.ensemble_members(max(64, M * world), nxy=(args.n, args.n // 2),
                                     first=rank * M, count=M)
    for c in cases:
        c.cfg.device = local
    ens = Ensemble([c.cfg for c in cases])
    for m, c in zip(ens.members, cases):
        m.set_initial_condition(c.ic)
        m.prepare_stage(1)
    dts = [c.dt for c in cases]
    cells = sum(c.cfg.nx * c.cfg.ny for c in cases)
    streams = [torch.cuda.ExternalStream(m.stream_handle(), device=local) for m in ens.members]
    ens.rk3_steps(dts, args.warmup)
    launches0 = sum(m.kernel_launches() for m in ens.members)

    def timed_steps():
        # members' states together fit in L2: flush before every timed step
        # (streams[0], after every member's previous step), then an event pair
        # per step spanning all member streams; no host sync between steps
        torch.cuda.synchronize()
        marks = []
        for _ in range(args.steps):
            l2_flush(streams[0], local)
            a = torch.cuda.Event(enable_timing=True)
            a.record(streams[0])
            for st in streams[1:]:
                st.wait_event(a)
            ens.rk3_steps(dts, 1)
            ends = [torch.cuda.Event(enable_timing=True) for _ in streams]
            for e, st in zip(ends, streams):
                e.record(st)
                streams[0].wait_event(e)
            marks.append((a, ends))
        torch.cuda.synchronize()
        return sum(max(a.elapsed_time(e) for e in ends) for a, ends in marks)

    def timed(fn):
        ev0 = torch.cuda.Event(enable_timing=True)
        ends = [torch.cuda.Event(enable_timing=True) for _ in streams]
        torch.cuda.synchronize()
        ev0.record(streams[0])
        for st in streams[1:]:
            st.wait_event(ev0)
        fn()
        for e, st in zip(ends, streams):
            e.record(st)
        torch.cuda.synchronize()
        return max(ev0.elapsed_time(e) for e in ends)

    with ClockSampler(local) as clk:
        if dist:
            dist.barrier()
        ms = timed_steps()
        if dist:
            dist.barrier()
    launches = sum(m.kernel_launches() for m in ens.members) - launches0
    if dist:
        t = torch.tensor([ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * cells * args.steps / (ms / 1e3)
    # e2e: every step each member's state comes from pinned host memory and
    # goes back (the C ABI set_state / rk3 / get_state path)
    hosts = []
    for m in ens.members:
        h = torch.empty(m.nc * m.plane, dtype=torch.float64).pin_memory()
        h.numpy()[:] = m.Ut.reshape(-1)
        hosts.append(h)

    def e2e_steps():
        for _ in range(args.e2e_steps):
            for m, h in zip(ens.members, hosts):
                m.set_state(h.numpy())
            ens.rk3_steps(dts, 1)
            for m, h in zip(ens.members, hosts):
                m._api["get_state"](m.handle, h.numpy().ctypes.data_as(
                    ctypes.POINTER(ctypes.c_double)))
    e2e_ms = timed(e2e_steps)
    if dist:
        t = torch.tensor([e2e_ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    state_bytes = sum(m.nc * m.plane * 8 for m in ens.members)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            threads = os.cpu_count() or 1
            rate, k, el = cpu_reference_rate(128, args.cpu_seconds, threads, "ensemble")
            cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": f"one 128x64 member of the same campaign, {k} RK3 steps in "
                             f"{el:.1f} s, unmodified reference via oracle/_ref"}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (analytic counterflow initial condition, sampled laser energies)",
            "config": {"workload": f"ensemble (configs[4]): {M} members per GPU of the H2/O2 "
                                   f"counterflow case at {args.n}x{args.n // 2}, laser energy "
                                   "U[0.01, 0.1] seed 1234", "members_per_gpu": M,
                       "global_batch": world * cells, "parallelism": "replicas (no collective)",
                       "l2": "members' states together fit in L2: 256 MB L2 flush before every "
                             "timed step, steps timed one by one"},
            "e2e": {"value": world * cells * args.e2e_steps / (e2e_ms / 1e3), "unit": UNIT,
                    "h2d_bytes_per_step": state_bytes, "d2h_bytes_per_step": state_bytes,
                    "steps": args.e2e_steps},
            "gpu_launches": launches, "cpu_baseline": cpu, "clocks": clk.summary(),
        }), flush=True)
    ens.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--size", "--n", dest="n", type=int, default=None,
                    help="cells per side (default 256 for tgv3d, 4096 tgv, 512 h2o2)")
    ap.add_argument("--case", default="tgv3d",
                    choices=["tgv3d", "tgv", "h2o2", "ensemble", "jet3d"])
    ap.add_argument("--members", type=int, default=8, help="ensemble members per GPU")
    ap.add_argument("--nz", type=int, default=None,
                    help="jet3d: z planes per GPU (default size/16; 256 = the full "
                         "512x256x256 configs[3] domain on one GPU)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-cases", action="store_true",
                    help="tgv3d only: skip the H2/O2 512^2 case of the headline metric")
    ap.add_argument("--force-slabs", action="store_true",
                    help="run the NCCL slab path even with one rank (plumbing check)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.n is None:
        args.n = {"tgv3d": 256, "tgv": 4096, "h2o2": 512, "ensemble": 500, "jet3d": 512}[args.case]

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    dist = None
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo" if args.impl == "reference" else "nccl")
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return

    import torch
    torch.cuda.set_device(local)
    if args.case == "ensemble":
        run_ensemble(args, rank, world, local, dist)
        return

    slabs = world > 1 or args.force_slabs
    case, workload = make_case(args, world)
    peaks = load_peaks()
    with ClockSampler(local) as clk:
        res = measure_case(args, case, workload, rank, world, local, dist, slabs, peaks)
        cases = {}
        if args.case == "tgv3d" and not args.no_cases:
            # the headline metric names TGV 256^3 AND the H2/O2 flame: configs[2]
            # 512^2 per GPU (y-slabs under torchrun), its own value and roofline
            sub = argparse.Namespace(**vars(args))
            sub.case, sub.n = "h2o2", 512
            c2, w2 = make_case(sub, world)
            cases["h2o2_512"] = measure_case(sub, c2, w2, rank, world, local, dist, slabs, peaks)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            threads = os.cpu_count() or 1
            rate, k, el = cpu_reference_rate(512, args.cpu_seconds, threads, args.case)
            cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": (f"512x512 {'2D analogue (no 3D reference path)' if args.case == 'tgv3d' else 'sub-problem'}"
                              f" of the same workload, {k} RK3 steps in {el:.1f} s, unmodified "
                              f"reference via oracle/_ref, {threads} threads")}
        except Exception as e:  # the baseline is reported, never required
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {e}"}
    if rank == 0:
        out = {
            "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (analytic initial condition)",
            "config": res["config"],
            "e2e": res["e2e"],
            "gpu_launches": res["gpu_launches"] + sum(c["gpu_launches"] for c in cases.values()),
            "roofline": res["roofline"],
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
        }
        if cases:
            out["cases"] = cases
        print(json.dumps(out), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def load_peaks():
    """MEASURED_PEAKS.json (driver-written); else B200_PROFILING.md's fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "hbm_source": "of measured (MEASURED_PEAKS.json)"}
    except Exception:  # noqa: BLE001
        return {"hbm_gbs": 6650.0, "hbm_source": "of fallback (B200_PROFILING.md)"}


def measure_case(args, case, workload, rank, world, local, dist, slabs, peaks):
    """One workload: K timed steps resident in HBM (CUDA events on the
    library's stream, max over ranks), the e2e pass through the C ABI with
    pinned host buffers, and the roofline of the dominant kernel class."""
    import torch
    from paper_2202_02319_b200 import Simulation, native
    case.cfg.device = local
    if slabs:  # one slab per rank (2D: y rows, 3D: z planes), halo over NCCL
        case.cfg.slab_count, case.cfg.slab_rank = world, rank
    sim = Simulation(case.cfg)
    if slabs:
        uid = ctypes.create_string_buffer(128)
        if rank == 0:
            st = native.api()["nccl_unique_id"](uid)
            if st != 0:
                raise RuntimeError("ign_nccl_unique_id failed")
        t = torch.tensor(list(uid.raw), dtype=torch.uint8, device=f"cuda:{local}")
        if dist:
            dist.broadcast(t, 0)
        raw = bytes(t.cpu().tolist())
        sim._check(native.api()["attach_nccl"](sim.handle, raw, world, rank))
    sim.set_initial_condition(case.ic)
    sim.prepare_stage(1)
    cells = case.cfg.nx * sim.ny * max(sim.nz, 1)  # this rank's slab
    nc = sim.nc
    stream = torch.cuda.ExternalStream(sim.stream_handle(), device=local)

    sim.rk3_steps(case.dt, args.warmup)  # untimed warm-up
    launches0 = sim.kernel_launches()
    flush = nc * sim.plane * 8 < L2_BYTES  # a state buffer fits in L2
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    if flush:
        ms = timed_flushed(stream, lambda: sim.rk3_steps(case.dt, 1), args.steps, local)
    else:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        sim.rk3_steps(case.dt, args.steps)
        ev1.record(stream)
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
    if dist:
        dist.barrier()
    launches = sim.kernel_launches() - launches0
    # per-kernel-class device times from a separate profiled pass: profiling
    # brackets every launcher with events and keeps the flux kernels serial
    # (the timed run above overlaps them on their own streams)
    sim.profile_enable(True)
    sim.rk3_steps(case.dt, max(2, min(args.steps, 5)))
    torch.cuda.synchronize()
    prof = sim.profile_read()
    sim.profile_enable(False)
    ms_max = ms
    if dist:
        t = torch.tensor([ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())
    value = world * cells * args.steps / (ms_max / 1e3)

    # ---------------- e2e through the C ABI with pinned host buffers
    host = torch.empty(nc * sim.plane, dtype=torch.float64).pin_memory()
    hbuf = host.numpy()
    hbuf[:] = sim.Ut.reshape(-1)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.e2e_steps):
        sim.set_state(hbuf)          # H2D of the step's input state
        sim.rk3_steps(case.dt, 1)
        sim._api["get_state"](sim.handle, hbuf.ctypes.data_as(
            ctypes.POINTER(ctypes.c_double)))  # D2H result
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([e2e_ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_val = world * cells * args.e2e_steps / (e2e_ms / 1e3)
    bytes_state = nc * sim.plane * 8

    # ---------------- roofline of the dominant kernel class (inviscid faces)
    peak = ctypes.c_double()
    native.api()["probe_fp64_peak"](local, ctypes.byref(peak))
    total_prof = sum(v[0] for v in prof.values())
    f_ms = prof["faces"][0]
    n_stage = prof["assemble"][1]  # one timed assemble per stage
    inv_ops, step_ops = OPS[args.case]
    # per stage (all face directions) = one "launch" of the faces class
    face_ops = cells * inv_ops if inv_ops else None
    stage_ms = f_ms / n_stage if n_stage else None
    achieved = face_ops / (stage_ms / 1e3) / 1e12 if (stage_ms and face_ops) else None
    hbm = peaks["hbm_gbs"]
    roofline = {
        "bound": "fp64",
        "kernel": ("k_faces3d<x,y,z>" if args.case in ("tgv3d", "jet3d") else "k_faces3<x>+k_faces3<y>")
                  + " (inviscid face fluxes, one stage)",
        "ops_per_cell_stage": inv_ops,
        "ops_source": OPS_SOURCE.get(args.case),
        "achieved": achieved, "peak": peak.value, "unit": "TFLOP/s",
        "frac": achieved / peak.value if achieved and peak.value else None,
        # dram read+write of the face kernels of one stage from an ncu --set
        # full capture (not measured in this run; see traffic_source)
        "traffic": TRAFFIC.get((args.case, args.n)),
        "traffic_unit": "bytes per faces region (one stage)",
        "traffic_source": TRAFFIC_SOURCE.get((args.case, args.n)),
        "traffic_algorithmic": (3 * (13 + 5) * cells * 8) if args.case == "tgv3d" else None,
        "ops_per_launch": face_ops, "avg_launch_ms": stage_ms,
        "share_of_step": f_ms / total_prof if total_prof else None,
        "peak_source": "live DFMA-chain microbenchmark (ign_probe_fp64_peak), 2 flop/FMA",
        # bitwise parity forbids contracting the reference's a*b+c into FMAs
        # (-fmad=false): every algorithmic op issues as one DADD/DMUL, whose
        # instruction peak is half the FMA flop peak
        "peak_no_fma": peak.value / 2 if peak.value else None,
        "frac_of_no_fma_peak": (achieved / (peak.value / 2)
                                if achieved and peak.value else None),
        "whole_step": {
            "ops_per_cell_step": step_ops,
            "fp64_tflops": value / world * step_ops / 1e12 if step_ops else None,
            "fp64_frac": (value / world * step_ops / 1e12 / peak.value
                          if step_ops and peak.value else None),
            "hbm_gbs": value / world * BYTES_PER_CELL_STEP(nc) / 1e9,
            "hbm_peak_gbs": hbm,
            "hbm_frac": value / world * BYTES_PER_CELL_STEP(nc) / 1e9 / hbm,
            "hbm_peak_source": peaks["hbm_source"],
        },
        "kernel_ms": {k: round(v[0], 3) for k, v in prof.items() if v[1]},
        "kernel_launches": {k: v[1] for k, v in prof.items() if v[1]},
    }
    res = {
        "value": value, "ms_per_step": ms_max / args.steps, "gpu_launches": launches,
        "config": {"workload": workload, "global_batch": world * cells,
                   "cells_per_gpu": cells,
                   "parallelism": (f"{'z' if sim.nz else 'y'}-slabs x{world}, NCCL halo "
                                   "overlapped with interior" if slabs else "single"),
                   "l2": (f"state {nc} x {sim.plane * 8 / 1e6:.0f} MB per buffer; "
                          + ("L2 flushed (256 MB write) before every timed step; steps timed "
                             "one by one with their own event pair" if flush else
                             "> 126 MB L2, no flush needed")),
                   "dt": case.dt},
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": bytes_state,
                "d2h_bytes_per_step": bytes_state, "steps": args.e2e_steps},
        "roofline": roofline,
    }
    sim.close()
    return res

if __name__ == "__main__":
    main()
