"""Host-side mirror of ``ignis::Simulation`` (solver.hpp:53-853) over the C ABI.

Method names, argument meaning and error behaviour follow the reference class
so parity tests read like the reference's own usage:

    sim = Simulation(case.cfg)
    sim.set_initial_condition(case.ic)
    sim.prepare_stage(1)
    rhs = sim.compute_rhs(t, 1)
    sim.rk3_step(dt)

The same wrapper drives the B200 library (``ign_*``) and, in tests/bench
only, the CPU oracle (``ignref_*``) — it is handed a bound function table.
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, Optional

import numpy as np

from . import abi
from .errors import UsageError, raise_for


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class Simulation:
    def __init__(self, cfg: abi.Config, api: Optional[dict] = None):
        if api is None:
            from . import native
            api = native.api()
        self._api = api
        self.cfg = cfg
        h = C.c_void_p()
        self._err = abi.Error()
        st = api["create"](C.byref(cfg), C.byref(h))
        if st != abi.IGN_OK:
            # creation errors carry no context; re-run the host validation for text
            raise_for(st, self._create_error(st))
        self._h = h
        nx, ny, g, ns, nz, k0, nzg = (C.c_int32() for _ in range(7))
        api["dims"](h, C.byref(nx), C.byref(ny), C.byref(g), C.byref(ns))
        if "dims3" in api:
            api["dims3"](h, C.byref(nz), C.byref(k0), C.byref(nzg))
        self.k0, self.nz_glob = k0.value, nzg.value
        self.nx, self.ny, self.g, self.ns = nx.value, ny.value, g.value, ns.value
        self.nz = nz.value  # 0: 2D (the reference), > 0: 3D extension
        self.nc = self.ns + (4 if self.nz else 3)
        self.shape = (self.ny + 2 * self.g, self.nx + 2 * self.g)
        if self.nz:
            self.shape = (self.nz + 2 * self.g,) + self.shape
        self.plane = int(np.prod(self.shape))

    def _create_error(self, st):
        e = abi.Error()
        e.status = st
        e.msg = b"ign_create failed (configuration rejected)"
        return e

    # ------------------------------------------------------------ plumbing
    def _check(self, st: int):
        if st != abi.IGN_OK:
            self._api["last_error"](self._h, C.byref(self._err))
            raise_for(st, self._err)

    def close(self):
        if getattr(self, "_h", None):
            self._api["destroy"](self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def handle(self):
        return self._h

    # ------------------------------------------------------------ setup
    def mesh_xy(self):
        shp = self.shape[-2:]
        n = shp[0] * shp[1]
        x = np.empty(n)
        y = np.empty(n)
        self._check(self._api["get_mesh"](self._h, _dptr(x), _dptr(y)))
        return x.reshape(shp), y.reshape(shp)

    def mesh_z(self):
        """z node coordinates of the 3D extension (uniform, padded)."""
        c = self.cfg
        k = self.k0 + np.arange(-self.g, self.nz + self.g)  # global z index (z-slabs)
        return c.center_z - 0.5 * c.lz + (k + 0.5) * (c.lz / self.nz_glob)

    def metrics(self, which: int = 0) -> np.ndarray:
        shp = self.shape[-2:]
        out = np.empty(5 * shp[0] * shp[1])
        self._check(self._api["get_metrics"](self._h, which, _dptr(out)))
        return out.reshape((5,) + shp)

    def set_initial_condition(self, ic: Callable):
        """solver.hpp:115-128 with a vectorised primitive function of the
        physical node coordinates: ic(X, Y) -> (rho, u, v, T, [Y_s]); 3D
        extension: ic(X, Y, Z) -> (rho, u, v, w, T, [Y_s])."""
        X, Y = self.mesh_xy()
        if self.nz:
            Z = self.mesh_z()[:, None, None] * np.ones((1,) + X.shape)
            X3 = np.broadcast_to(X, Z.shape)
            Y3 = np.broadcast_to(Y, Z.shape)
            rho, u, v, w, T, Ys = ic(X3, Y3, Z)
            fields = [rho, u, v, w, T] + list(Ys)
        else:
            rho, u, v, T, Ys = ic(X, Y)
            fields = [rho, u, v, T] + list(Ys)
        prim = np.empty((len(fields),) + self.shape)
        for k, f in enumerate(fields):
            prim[k] = f
        prim = np.ascontiguousarray(prim)
        self._check(self._api["set_initial_primitives"](self._h, _dptr(prim)))

    def set_state(self, Ut: np.ndarray, T: Optional[np.ndarray] = None):
        Ut = np.ascontiguousarray(Ut, dtype=np.float64).reshape(-1)
        if Ut.size != self.nc * self.plane:
            raise UsageError("set_state: wrong Ut size")
        Tp = None
        if T is not None:
            T = np.ascontiguousarray(T, dtype=np.float64).reshape(-1)
            Tp = _dptr(T)
        self._check(self._api["set_state"](self._h, _dptr(Ut), Tp))

    @property
    def Ut(self) -> np.ndarray:
        out = np.empty(self.nc * self.plane)
        self._check(self._api["get_state"](self._h, _dptr(out)))
        return out.reshape((self.nc,) + self.shape)

    def cache(self) -> dict:
        names = ("rho", "u", "v", "w", "p", "T", "c") if self.nz else ("rho", "u", "v", "p", "T", "c")
        out = np.empty((len(names) + self.ns) * self.plane)
        self._check(self._api["get_cache"](self._h, _dptr(out)))
        out = out.reshape((len(names) + self.ns,) + self.shape)
        d = {k: out[i] for i, k in enumerate(names)}
        d["Y"] = out[len(names):]
        return d

    @property
    def time(self) -> float:
        t, it = C.c_double(), C.c_int64()
        self._api["get_time"](self._h, C.byref(t), C.byref(it))
        return t.value

    @property
    def iter(self) -> int:
        t, it = C.c_double(), C.c_int64()
        self._api["get_time"](self._h, C.byref(t), C.byref(it))
        return it.value

    def set_time(self, t: float, it: int = 0):
        self._check(self._api["set_time"](self._h, t, it))

    def set_integrator(self, fixed_dt=0.0, t_end=0.0, max_iter=2**63 - 1,
                       chem_dt_limit=True, chem_dt_factor=0.1):
        ig = abi.Integrator(fixed_dt, t_end, max_iter, int(chem_dt_limit), 0,
                            chem_dt_factor)
        self._check(self._api["set_integrator"](self._h, C.byref(ig)))

    # ------------------------------------------------------------ hot path
    def refill_ghosts(self):
        self._check(self._api["refill_ghosts"](self._h))

    def refresh_primitives(self, stage: int = 0):
        self._check(self._api["refresh_primitives"](self._h, stage))

    def prepare_stage(self, stage: int = 1):
        self._check(self._api["prepare_stage"](self._h, stage))

    def compute_rhs(self, t_stage: float, stage: int = 0) -> np.ndarray:
        out = np.empty(self.nc * self.plane)
        self._check(self._api["compute_rhs"](self._h, t_stage, stage, _dptr(out)))
        return out.reshape((self.nc,) + self.shape)

    def stable_dt(self) -> float:
        dt = C.c_double()
        self._check(self._api["stable_dt"](self._h, C.byref(dt)))
        return dt.value

    def rk3_step(self, dt: float):
        self._check(self._api["rk3_step"](self._h, dt))

    def rk3_steps(self, dt: float, n: int):
        """n x (rk3_step(dt); prepare_stage(1)) — advance()'s loop body with a
        pinned step (solver.hpp:344-345), no host round trip in between."""
        self._check(self._api["rk3_steps"](self._h, dt, n))

    def advance(self, hook: Optional[Callable] = None):
        if hook is None:
            cb = abi.STEP_HOOK()
        else:
            cb = abi.STEP_HOOK(lambda ctx, user: int(hook(self) or 0))
        self._check(self._api["advance"](self._h, cb, None))

    # ------------------------------------------------------------ diagnostics
    def conserved_totals(self) -> np.ndarray:
        out = np.empty(self.nc)
        self._check(self._api["conserved_totals"](self._h, _dptr(out)))
        return out

    def set_diagnostics(self, mode: str = "device"):
        """conserved_totals / product_mole_fraction / the trace: "device" =
        deterministic tree on the GPU (default), "reference" = the reference's
        serial order (solver.hpp:387-418) on the host, bitwise."""
        m = {"device": abi.DIAG_DEVICE, "reference": abi.DIAG_REFERENCE}[mode]
        self._check(self._api["set_diagnostics"](self._h, m))

    def product_mole_fraction(self) -> float:
        out = C.c_double()
        self._check(self._api["product_mole_fraction"](self._h, C.byref(out)))
        return out.value

    @property
    def last_clip(self) -> float:
        out = C.c_double()
        self._check(self._api["last_clip"](self._h, C.byref(out)))
        return out.value

    def kernel_launches(self) -> int:
        return int(self._api["kernel_launches"](self._h))

    # ------------------------------------------------------------ outputs
    def add_probe(self, i0: int, j0: int, i1: int, j1: int):
        """Simulation::add_probe (solver.hpp:130-135), ProbeSpec{i0, j0, i1, j1}."""
        self._check(self._api["add_probe"](self._h, i0, j0, i1, j1))

    def add_probe3(self, i0: int, j0: int, k0: int, i1: int, j1: int, k1: int):
        """3D extension: probe box over global planes k0..k1 (rows add w)."""
        self._check(self._api["add_probe3"](self._h, i0, j0, k0, i1, j1, k1))

    def set_sampling(self, probe_interval: int = 0, trace_interval: int = 0):
        """probe_interval / trace_interval (solver.hpp:71-73)."""
        self._check(self._api["set_sampling"](self._h, probe_interval, trace_interval))

    def probe(self, k: int):
        """ProbeSeries k: (times[n], rows[n, 5+ns]) — rho, u, v, p, T, Y_s box means."""
        n = C.c_int64()
        self._check(self._api["probe_samples"](self._h, k, C.byref(n), None, None))
        t = np.empty(n.value)
        r = np.empty((n.value, (6 if self.nz else 5) + self.ns))
        self._check(self._api["probe_samples"](self._h, k, C.byref(n), _dptr(t), _dptr(r)))
        return t, r

    def trace(self):
        """product_fraction TraceSeries: (times[n], values[n])."""
        n = C.c_int64()
        self._check(self._api["trace_samples"](self._h, C.byref(n), None, None))
        t, v = np.empty(n.value), np.empty(n.value)
        self._check(self._api["trace_samples"](self._h, C.byref(n), _dptr(t), _dptr(v)))
        return t, v

    @property
    def config_hash(self) -> int:
        h = C.c_uint64()
        self._check(self._api["get_config_hash"](self._h, C.byref(h)))
        return h.value

    @config_hash.setter
    def config_hash(self, h: int):
        self._check(self._api["set_config_hash"](self._h, h))

    def write_snapshot(self, path: str):
        """write_snapshot (snapshot.hpp:52-76), IGNS v1."""
        self._check(self._api["write_snapshot"](self._h, str(path).encode()))

    def write_snapshot_v2(self, path: str, with_t: bool = True):
        """IGNS v2: + nz and, with_t, the T cache for a bit-exact restart."""
        self._check(self._api["write_snapshot_v2"](self._h, str(path).encode(), int(with_t)))

    def read_snapshot(self, path: str):
        """read_snapshot + apply_snapshot (snapshot.hpp:78-145)."""
        self._check(self._api["read_snapshot"](self._h, str(path).encode()))

    # ------------------------------------------------------------ measurement
    def profile_enable(self, on: bool = True):
        self._check(self._api["profile_enable"](self._h, int(on)))

    def profile_read(self) -> dict:
        ms = np.zeros(8)
        n = np.zeros(8, dtype=np.int64)
        self._check(self._api["profile_read"](self._h, _dptr(ms),
                                              n.ctypes.data_as(C.POINTER(C.c_int64))))
        return {k: (float(ms[i]), int(n[i])) for i, k in enumerate(abi.PROF_CLASSES)}

    def stream_handle(self) -> int:
        return int(self._api["stream_handle"](self._h) or 0)


class SlabGroup:
    """Single-process group of slab contexts (ign_group_*): the y-slabs of one
    decomposed domain driven in lockstep on one GPU — the validation harness of
    the multi-GPU path (halo rows by device copies instead of NCCL)."""

    def __init__(self, cfg: abi.Config, nslabs: int, api: Optional[dict] = None):
        from . import native
        self._api = api or native.api()
        self.members = []
        for r in range(nslabs):
            c = abi.Config()
            C.memmove(C.byref(c), C.byref(cfg), C.sizeof(abi.Config))
            c.slab_count, c.slab_rank = nslabs, r
            self.members.append(Simulation(c, self._api))
        arr = (C.c_void_p * nslabs)(*[m.handle.value for m in self.members])
        g = C.c_void_p()
        st = self._api["group_create"](arr, nslabs, C.byref(g))
        if st != abi.IGN_OK:
            raise_for(st, abi.Error())
        self._g = g
        for m in self.members:  # the group owns the contexts now
            m._h = None
        self._handles = [arr[k] for k in range(nslabs)]

    def _check(self, st):
        if st != abi.IGN_OK:
            e = abi.Error()
            self._api["group_last_error"](self._g, C.byref(e))
            raise_for(st, e)

    def member_call(self, k, name, *args):
        return self._api[name](C.c_void_p(self._handles[k]), *args)

    def set_state(self, k: int, Ut: np.ndarray, T: Optional[np.ndarray] = None):
        Ut = np.ascontiguousarray(Ut, dtype=np.float64).reshape(-1)
        Tp = None
        if T is not None:
            T = np.ascontiguousarray(T, dtype=np.float64).reshape(-1)
            Tp = _dptr(T)
        self._check(self.member_call(k, "set_state", _dptr(Ut), Tp))

    def Ut(self, k: int) -> np.ndarray:
        m = self.members[k]
        out = np.empty(m.nc * m.plane)
        self._check(self.member_call(k, "get_state", _dptr(out)))
        return out.reshape((m.nc,) + m.shape)

    def cache_T(self, k: int) -> np.ndarray:
        m = self.members[k]
        head = 7 if m.nz else 6
        out = np.empty((head + m.ns) * m.plane)
        self._check(self.member_call(k, "get_cache", _dptr(out)))
        return out.reshape((head + m.ns,) + m.shape)[head - 2]

    def prepare_stage(self, stage: int = 1):
        self._check(self._api["group_prepare_stage"](self._g, stage))

    def rk3_steps(self, dt: float, n: int):
        self._check(self._api["group_rk3_steps"](self._g, dt, n))

    def stable_dt(self) -> float:
        dt = C.c_double()
        self._check(self._api["group_stable_dt"](self._g, C.byref(dt)))
        return dt.value

    def set_diagnostics(self, mode: str = "device"):
        m = {"device": abi.DIAG_DEVICE, "reference": abi.DIAG_REFERENCE}[mode]
        for k in range(len(self.members)):
            self._check(self.member_call(k, "set_diagnostics", m))

    def conserved_totals(self) -> np.ndarray:
        out = np.empty(self.members[0].nc)
        self._check(self._api["group_conserved_totals"](self._g, _dptr(out)))
        return out

    # advance() state and outputs live on the lead (slab 0) context
    def lead_call(self, name, *args):
        self._check(self.member_call(0, name, *args))

    def set_integrator(self, fixed_dt=0.0, t_end=0.0, max_iter=2**63 - 1,
                       chem_dt_limit=True, chem_dt_factor=0.1):
        ig = abi.Integrator(fixed_dt, t_end, max_iter, int(chem_dt_limit), 0, chem_dt_factor)
        for k in range(len(self.members)):
            self._check(self.member_call(k, "set_integrator", C.byref(ig)))

    def add_probe(self, i0, j0, i1, j1):
        self.lead_call("add_probe", i0, j0, i1, j1)

    def set_sampling(self, probe_interval=0, trace_interval=0):
        self.lead_call("set_sampling", probe_interval, trace_interval)

    def probe(self, k: int):
        n = C.c_int64()
        self.lead_call("probe_samples", k, C.byref(n), None, None)
        t = np.empty(n.value)
        m0 = self.members[0]
        r = np.empty((n.value, (6 if m0.nz else 5) + m0.ns))
        self.lead_call("probe_samples", k, C.byref(n), _dptr(t), _dptr(r))
        return t, r

    def trace(self):
        n = C.c_int64()
        self.lead_call("trace_samples", C.byref(n), None, None)
        t, v = np.empty(n.value), np.empty(n.value)
        self.lead_call("trace_samples", C.byref(n), _dptr(t), _dptr(v))
        return t, v

    def advance(self):
        self._check(self._api["group_advance"](self._g))

    def write_snapshot(self, path: str, version: int = 1, with_t: bool = False):
        self._check(self._api["group_write_snapshot"](self._g, str(path).encode(), version,
                                                       int(with_t)))

    def read_snapshot(self, path: str):
        self._check(self._api["group_read_snapshot"](self._g, str(path).encode()))

    def close(self):
        if getattr(self, "_g", None):
            self._api["group_destroy"](self._g)
            self._g = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Ensemble:
    """Independent members on one GPU advanced together (BASELINE configs[4]):
    ign_ensemble_rk3_steps interleaves the members' steps on their own streams.
    Each member is a full Simulation (set_initial_condition, outputs, ...)."""

    def __init__(self, cfgs, api: Optional[dict] = None):
        from . import native
        self._api = api or native.api()
        self.members = [Simulation(c, self._api) for c in cfgs]

    def __len__(self):
        return len(self.members)

    def rk3_steps(self, dt, n: int, only=None):
        """n steps per member with dt (scalar or per member).  Returns the
        per-member status list; raises the first failure's exception only when
        every member failed (a failed member stops, the others continue).
        ``only``: indices of the members to advance (the others are left as
        they are; their status reads 0)."""
        idx = list(range(len(self.members))) if only is None else list(only)
        if not idx:
            return [0] * len(self.members)
        if only is not None:
            full = [0] * len(self.members)
            sub = Ensemble.__new__(Ensemble)
            sub._api, sub.members = self._api, [self.members[k] for k in idx]
            dts = np.broadcast_to(np.asarray(dt, dtype=np.float64), (len(self.members),))
            st = sub.rk3_steps([dts[k] for k in idx], n) if len(idx) else []
            for k, v in zip(idx, st):
                full[k] = v
            return full
        M = len(self.members)
        dts = np.ascontiguousarray(np.broadcast_to(np.asarray(dt, dtype=np.float64), (M,)))
        hs = (C.c_void_p * M)(*[m.handle.value for m in self.members])
        st = (C.c_int * M)()
        rc = int(self._api["ensemble_rk3_steps"](hs, M, _dptr(dts), n, st))
        status = [int(x) for x in st]
        if rc != abi.IGN_OK and all(x == abi.IGN_OK for x in status):
            status = [rc] * M  # defensive: a failing call always reports per member
        if all(x != abi.IGN_OK for x in status):
            self.members[0]._check(status[0])
        return status

    def error(self, k: int):
        """The exception member k's last failure maps to (None when it is fine)."""
        e = abi.Error()
        self._api["last_error"](self.members[k].handle, C.byref(e))
        if e.status == abi.IGN_OK:
            return None
        try:
            raise_for(e.status, e)
        except Exception as exc:  # noqa: BLE001 — returned, not raised
            return exc

    def close(self):
        for m in self.members:
            m.close()
