"""Configuration builders for the BASELINE.json cases and the parity suite.

Every builder fills the POD ``abi.Config`` that ``ign_create`` (and the
oracle's ``ignref_create``) receive, exactly as a reference user would fill
``ignis::Simulation``'s public knobs (solver.hpp:55-101).  Initial conditions
are vectorised numpy functions of the padded node coordinates returning the
primitive arrays ``set_initial_primitives`` takes (rho, u, v, T, Y_s).
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from . import abi

DATA_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "data")
R_UNIVERSAL = 8.31446261815324  # thermo.hpp:71


# ---------------------------------------------------------------- mixtures
@dataclass
class SpeciesSpec:
    name: str
    W: float
    mu_ref: float
    t_ref: float
    n_exp: float
    pieces: list  # list of dicts with t_lo,t_hi,cm2,cm1,c0..c4,b


def parse_mixture(text: str) -> list:
    """Restates the reference's table parser (thermo.hpp:291-357)."""
    toks_lines = []
    for line in text.splitlines():
        line = line.split("#", 1)[0]
        t = line.split()
        if t:
            toks_lines.append(t)
    out, k = [], 0
    while k < len(toks_lines):
        t = toks_lines[k]
        k += 1
        if len(t) != 6:
            raise ValueError("mixture: bad species header: " + " ".join(t))
        sp = SpeciesSpec(t[0], float(t[1]), float(t[2]), float(t[3]), float(t[4]), [])
        if sp.W <= 0.0:
            raise ValueError("mixture: non-positive molar mass for " + sp.name)
        for _ in range(int(t[5])):
            r = toks_lines[k]
            k += 1
            if len(r) == 9:
                p = dict(t_lo=float(r[0]), t_hi=float(r[1]), cm2=0.0, cm1=0.0,
                         c0=float(r[2]), c1=float(r[3]), c2=float(r[4]),
                         c3=float(r[5]), c4=float(r[6]), b=float(r[7]))
            elif len(r) == 11:
                p = dict(t_lo=float(r[0]), t_hi=float(r[1]), cm2=float(r[2]),
                         cm1=float(r[3]), c0=float(r[4]), c1=float(r[5]),
                         c2=float(r[6]), c3=float(r[7]), c4=float(r[8]), b=float(r[9]))
            else:
                raise ValueError("mixture: range row needs 7 or 9 coefficients")
            if p["t_hi"] <= p["t_lo"]:
                raise ValueError("mixture: empty temperature range for " + sp.name)
            sp.pieces.append(p)
        if not sp.pieces:
            raise ValueError("mixture: species without ranges: " + sp.name)
        out.append(sp)
    if not out or len(out) > abi.IGN_MAX_SPECIES:
        raise ValueError("mixture: need 1..8 species")
    return out


def load_mixture_file(path: str) -> list:
    with open(path) as f:
        return parse_mixture(f.read())


def _piece(t_lo, t_hi, c0, c1, b):
    return dict(t_lo=t_lo, t_hi=t_hi, cm2=0.0, cm1=0.0, c0=c0, c1=c1, c2=0.0,
                c3=0.0, c4=0.0, b=b)


def ch4_o2_species() -> list:
    """The reference's CH4/O2/CO2/H2O surrogate set (data/ch4_o2.mix:13-27),
    restated as values (the reference's tests load it via IGNIS_DATA_DIR)."""
    return [
        SpeciesSpec("CH4", 0.016, 1.02e-05, 273.0, 0.87,
                    [_piece(200.0, 1000.0, 4.2, 0.0018, -1.0337025302e+04),
                     _piece(1000.0, 6000.0, 5.7, 0.0003, -1.1087025302e+04)]),
        SpeciesSpec("O2", 0.032, 1.92e-05, 273.0, 0.77,
                    [_piece(200.0, 1000.0, 3.3, 0.0006, -1.0105630267e+03),
                     _piece(1000.0, 6000.0, 3.8, 0.0001, -1.2605630267e+03)]),
        SpeciesSpec("CO2", 0.044, 1.37e-05, 273.0, 0.93,
                    [_piece(200.0, 1000.0, 3.9, 0.002, -4.8581255579e+04),
                     _piece(1000.0, 6000.0, 5.4, 0.0005, -4.9331255579e+04)]),
        SpeciesSpec("H2O", 0.018, 9.2e-06, 273.0, 1.04,
                    [_piece(200.0, 1000.0, 3.9, 0.0007, -3.0279361318e+04),
                     _piece(1000.0, 6000.0, 4.1, 0.0005, -3.0379361318e+04)]),
    ]


def h2_o2_species() -> list:
    return load_mixture_file(os.path.join(DATA_DIR, "h2_o2.mix"))


def fill_mixture(mix: abi.Mixture, species: list, R: float = R_UNIVERSAL,
                 Le: float = 1.0, Pr: float = 0.7, mode: int = abi.MULTI_SPECIES):
    mix.mode = mode
    mix.ns = len(species)
    mix.R, mix.Le, mix.Pr = R, Le, Pr
    for s, sp in enumerate(species):
        d = mix.species[s]
        d.name = sp.name.encode()[: abi.IGN_NAME_LEN - 1]
        d.W, d.mu_ref, d.t_ref, d.n_exp = sp.W, sp.mu_ref, sp.t_ref, sp.n_exp
        d.npieces = len(sp.pieces)
        if d.npieces > abi.IGN_MAX_PIECES:
            raise ValueError("too many thermo pieces")
        for k, p in enumerate(sp.pieces):
            for key, val in p.items():
                setattr(d.pieces[k], key, val)


def gamma_gas(mix: abi.Mixture, gamma: float = 1.4, r_specific: float = 1.0,
              mu: float = 0.0, t_hi_cap: float = 1e6):
    """MixtureModel::calorically_perfect (thermo.hpp:83-103).  t_hi is capped
    (SURVEY §8c harness fix) because the reference's Newton bisects toward
    t_hi=1e30 and fails when the first residual is exactly zero."""
    sp = SpeciesSpec("gas", 1.0, mu, 1.0, 0.0,
                     [dict(t_lo=0.0, t_hi=1e30, cm2=0.0, cm1=0.0,
                           c0=gamma / (gamma - 1.0), c1=0.0, c2=0.0, c3=0.0,
                           c4=0.0, b=0.0)])
    fill_mixture(mix, [sp], R=r_specific, mode=abi.CALORICALLY_PERFECT)
    if t_hi_cap is not None:
        mix.species[0].pieces[0].t_hi = t_hi_cap


# ---------------------------------------------------------------- config
def base_config(nx: int, ny: int, lx: float, ly: float, *, center=(0.0, 0.0),
                periodic=(True, True)) -> abi.Config:
    cfg = abi.Config()
    cfg.abi_version = abi.IGN_ABI_VERSION
    cfg.nx, cfg.ny, cfg.g = nx, ny, 3
    cfg.lx, cfg.ly = lx, ly
    cfg.center_x, cfg.center_y = center
    cfg.periodic_x, cfg.periodic_y = int(periodic[0]), int(periodic[1])
    cfg.metric_mode = abi.MM_AUTO
    # SchemeConfig defaults (reconstruction.hpp:20-26)
    cfg.scheme.scheme = abi.TENO6
    cfg.scheme.split = abi.CHARACTERISTIC
    cfg.scheme.teno_ct = 1e-5
    cfg.scheme.eps = 1e-40
    cfg.scheme.cfl = 0.5
    cfg.scheme.metrics = abi.METRICS_SCHEME
    for e in (cfg.bc.left, cfg.bc.right, cfg.bc.bottom, cfg.bc.top):
        e.type = abi.PERIODIC
        e.sigma_out = 0.25  # boundary.hpp:40
    if not periodic[0]:
        cfg.bc.left.type = cfg.bc.right.type = abi.OUTFLOW
    if not periodic[1]:
        cfg.bc.bottom.type = cfg.bc.top.type = abi.OUTFLOW
    # IntegratorConfig defaults (solver.hpp:29-35)
    cfg.integ.fixed_dt = 0.0
    cfg.integ.t_end = 0.0
    cfg.integ.max_iter = 2**63 - 1
    cfg.integ.chem_dt_limit = 1
    cfg.integ.chem_dt_factor = 0.1
    cfg.laser.sigma_r = 1.0
    cfg.laser.sigma_t = 1.0
    # ShapedProfile defaults (laser.hpp:64-70)
    cfg.laser.lobe_sep, cfg.laser.width_up, cfg.laser.width_down = 0.5, 0.6, 0.25
    cfg.laser.amp_down, cfg.laser.width_radial = 0.7, 0.2
    cfg.mech.a = cfg.mech.b = 1.0
    cfg.mech.T_cutoff = 300.0
    cfg.mech.i_fuel = cfg.mech.i_ox = cfg.mech.i_co2 = cfg.mech.i_h2o = -1
    cfg.partitions = 1
    cfg.device = 0
    return cfg


@dataclass
class Case:
    """A configured case: the POD config, its initial condition, a pinned dt."""
    name: str
    cfg: abi.Config
    ic: Callable  # (X, Y) padded coordinate arrays -> (rho, u, v, T, [Y_s])
    dt: float
    notes: dict = field(default_factory=dict)


def set_scheme(cfg: abi.Config, scheme: str = "teno6", split: str = "char"):
    cfg.scheme.scheme = abi.TENO6 if scheme.lower() == "teno6" else abi.WENO3Z
    cfg.scheme.split = abi.CHARACTERISTIC if split.startswith("char") else abi.COMPONENTWISE


# ---------------------------------------------------------------- cases
def tgv2d(n: int = 256, *, viscous: bool = True, scheme: str = "teno6",
          split: str = "char", mach: float = 0.1, mu: float = 6.25e-4,
          ly_periods: int = 1, skew: float = 0.0) -> Case:
    """2D Taylor-Green vortex on [-pi, pi)^2 (the reference-runnable analogue of
    BASELINE configs[1]): rho0 = 1, gamma-gas (gamma 1.4,
    R 1), Ma 0.1 (p0 = 1/(gamma Ma^2)), Re 1600 (mu = 6.25e-4).  ly_periods > 1
    stacks periodic copies along y (weak-scaling slabs)."""
    L = 2.0 * math.pi
    cfg = base_config(n, n * ly_periods, L, L * ly_periods)
    if skew:
        cfg.apply_skew, cfg.skew_beta = 1, skew
    gamma = 1.4
    gamma_gas(cfg.mix, gamma, 1.0, mu if viscous else 0.0)
    set_scheme(cfg, scheme, split)
    cfg.viscous = int(viscous)
    p0 = 1.0 / (gamma * mach * mach)
    c0 = math.sqrt(gamma * p0)
    dx = L / n
    dt = 0.4 * dx / (2.0 * (c0 + 1.0))  # CFL-safe fixed step

    def ic(X, Y):
        u = np.sin(X) * np.cos(Y)
        v = -np.cos(X) * np.sin(Y)
        p = p0 + 0.25 * (np.cos(2.0 * X) + np.cos(2.0 * Y))
        rho = np.ones_like(X)
        T = p / rho
        return rho, u, v, T, [np.ones_like(X)]

    return Case(f"tgv2d_{n}", cfg, ic, dt, dict(p0=p0, c0=c0))


def sod_strip(nx: int = 1000, scheme: str = "teno6", split: str = "char") -> Case:
    """BASELINE configs[0] as the reference runs it:
    1000x7 strip over x in [-0.5, 0.5], outflow x edges with LODI p_target=0.1
    on the right, periodic y, gamma-gas, inviscid."""
    ny = 7
    cfg = base_config(nx, ny, 1.0, ny * (1.0 / nx), periodic=(False, True))
    gamma_gas(cfg.mix, 1.4, 1.0, 0.0)
    set_scheme(cfg, scheme, split)
    cfg.bc.right.p_target = 0.1
    cfg.bc.left.p_target = 1.0

    def ic(X, Y):
        left = X < 0.0
        rho = np.where(left, 1.0, 0.125)
        p = np.where(left, 1.0, 0.1)
        z = np.zeros_like(X)
        return rho, z, z.copy(), p / rho, [np.ones_like(X)]

    return Case(f"sod_{nx}", cfg, ic, 2e-4 * 1000.0 / nx)


def reacting_ch4(n: int = 64, *, scheme: str = "teno6", split: str = "char",
                 viscous: bool = True, laser: bool = True) -> Case:
    """4-species CH4/O2 reacting patch (SURVEY App. A probe case): periodic 1 cm
    box, stoichiometric CH4/O2 at 1 atm with a hot kernel so the one-step
    chemistry (A = 2e5, Ta = 12000: test_chemistry.cpp:16-18 constants) and
    the Gaussian laser are both active."""
    L = 0.01
    cfg = base_config(n, n, L, L)
    fill_mixture(cfg.mix, ch4_o2_species())
    set_scheme(cfg, scheme, split)
    cfg.viscous = int(viscous)
    m = cfg.mech
    m.present = 1
    m.A, m.Ta, m.a, m.b, m.T_cutoff = 2e5, 12000.0, 1.0, 1.0, 300.0
    m.i_fuel, m.i_ox, m.i_co2, m.i_h2o = 0, 1, 2, 3
    for s, nu in enumerate((-1.0, -2.0, 1.0, 2.0)):
        m.nu[s] = nu
    if laser:
        la = cfg.laser
        la.present = 1
        la.kernel = abi.LASER_GAUSSIAN
        la.energy, la.sigma_r, la.sigma_t = 2.0, 8e-4, 2e-6
        la.x0, la.y0, la.t0 = 1e-3, -5e-4, 1e-6
    Ws = [0.016, 0.032, 0.044, 0.018]
    Y0 = np.array([0.2, 0.8, 0.0, 0.0])
    Yb = np.array([0.05, 0.2, 0.41, 0.34])

    def ic(X, Yc):
        r2 = (X - 1e-3) ** 2 + (Yc + 1e-3) ** 2
        f = np.exp(-r2 / (2.0 * (1.5e-3) ** 2))
        T = 300.0 + 1700.0 * f
        Ys = [Y0[s] * (1 - f) + Yb[s] * f for s in range(4)]
        tot = sum(Ys)
        Ys = [y / tot for y in Ys]
        rbar = R_UNIVERSAL * sum(Ys[s] / Ws[s] for s in range(4))
        rho = 101325.0 / (rbar * T)
        u = 3.0 * np.sin(2 * math.pi * Yc / L)
        v = -2.0 * np.cos(2 * math.pi * X / L)
        return rho, u, v, T, Ys

    dx = L / n
    return Case(f"ch4_{n}", cfg, ic, 0.2 * dx / 900.0)


def h2o2_counterflow(n: int = 512, *, scheme: str = "teno6", split: str = "char",
                     nxy=None, energy: float = 5.0) -> Case:
    """BASELINE configs[2]: 2 cm x 2 cm, left Inflow
    H2/N2 at 300 K, +1 m/s; right Inflow O2/N2, -1 m/s; top/bottom Outflow;
    1 atm; one-step 2 H2 + O2 -> 2 H2O (A = 1e9 m^3/(mol s), Ta = 15000 K,
    a = b = 1, T_cut 300 K); Gaussian laser ignition at the centre; viscous,
    TENO6 characteristic."""
    nx, ny = (n, n) if nxy is None else nxy
    L = 0.02
    cfg = base_config(nx, ny, L * nx / n, L * ny / n, periodic=(False, False))
    fill_mixture(cfg.mix, h2_o2_species())
    set_scheme(cfg, scheme, split)
    cfg.viscous = 1
    Ws = [sp.W for sp in h2_o2_species()]
    Yf = [0.1, 0.0, 0.0, 0.9]
    Yo = [0.0, 0.23, 0.0, 0.77]
    for e, Ysg, uu in ((cfg.bc.left, Yf, 1.0), (cfg.bc.right, Yo, -1.0)):
        e.type = abi.INFLOW
        e.nseg = 1
        e.smooth_width = 0.0
        s = e.seg[0]
        s.lo, s.hi = -0.5 * cfg.ly, 0.5 * cfg.ly
        s.u, s.v, s.T = uu, 0.0, 300.0
        for k in range(4):
            s.Y[k] = Ysg[k]
    cfg.bc.bottom.type = cfg.bc.top.type = abi.OUTFLOW
    m = cfg.mech
    m.present = 1
    m.A, m.Ta, m.a, m.b, m.T_cutoff = 1e9, 15000.0, 1.0, 1.0, 300.0
    m.i_fuel, m.i_ox, m.i_co2, m.i_h2o = 0, 1, -1, 2
    for s, nu in enumerate((-2.0, -1.0, 2.0, 0.0)):
        m.nu[s] = nu
    la = cfg.laser
    la.present = 1
    la.kernel = abi.LASER_GAUSSIAN
    la.energy, la.sigma_r, la.sigma_t = energy, 5e-4, 1e-6
    la.x0, la.y0, la.t0 = 0.0, 0.0, 3e-6
    delta = 1e-3

    def ic(X, Yc):
        w = 0.5 * (1.0 - np.tanh(X / delta))  # 1 on the fuel side
        Ys = [Yf[k] * w + Yo[k] * (1 - w) for k in range(4)]
        T = np.full_like(X, 300.0)
        rbar = R_UNIVERSAL * sum(Ys[k] / Ws[k] for k in range(4))
        rho = 101325.0 / (rbar * T)
        u = -np.tanh(X / (4 * delta))
        v = np.zeros_like(X)
        return rho, u, v, T, Ys

    dx = L / n
    return Case(f"h2o2_{nx}x{ny}", cfg, ic, min(0.15 * dx / 400.0, la.sigma_t / 6.0))


def _lin_species(name, W, mu_ref, n_exp, c0, c1, h_form_over_R, c0_hi=None, c1_hi=None):
    """A compact surrogate in the h2_o2.mix form: two linear cp/R ranges meeting
    at 1000 K with h continuous there and h(298.15 K)/R = h_form_over_R."""
    c0_hi = c0 if c0_hi is None else c0_hi
    c1_hi = c1 if c1_hi is None else c1_hi
    b = h_form_over_R - (c0 * 298.15 + 0.5 * c1 * 298.15 ** 2)
    b_hi = b + (c0 - c0_hi) * 1000.0 + 0.5 * (c1 - c1_hi) * 1e6
    return SpeciesSpec(name, W, mu_ref, 273.0, n_exp,
                       [_piece(200.0, 1000.0, c0, c1, b), _piece(1000.0, 6000.0, c0_hi, c1_hi, b_hi)])


def eight_species() -> list:
    """H2, O2, H2O, N2 (data/h2_o2.mix) + four inert surrogates AR, HE, CO2, CO:
    the reference's species cap (thermo.hpp:16 kMaxSpecies = 8)."""
    base = h2_o2_species()
    return base + [
        _lin_species("AR", 0.040, 2.10e-05, 0.72, 2.5, 0.0, 0.0),
        _lin_species("HE", 0.004, 1.87e-05, 0.67, 2.5, 0.0, 0.0),
        _lin_species("CO2", 0.044, 1.37e-05, 0.93, 3.9, 0.002, -393510.0 / R_UNIVERSAL,
                     5.4, 0.0005),
        _lin_species("CO", 0.028, 1.66e-05, 0.74, 3.3, 0.0004, -110530.0 / R_UNIVERSAL,
                     3.6, 0.0001),
    ]


def species_box(ns: int, n: int = 24, *, scheme: str = "teno6", split: str = "char",
                laser: str = "gaussian", viscous: bool = True) -> Case:
    """Periodic 1 cm box with ns species (2..8) for the species-count parity
    cases: ns = 2 is a non-reacting H2/N2 mixture; ns >= 3 takes the first ns
    of eight_species() with the one-step 2 H2 + O2 -> 2 H2O mechanism.  A hot
    kernel, shear and a laser (Gaussian or the shaped two-lobe kernel,
    laser.hpp:64-85) keep transport, chemistry and the source active."""
    if not 2 <= ns <= 8:
        raise ValueError("species_box: 2 <= ns <= 8")
    allsp = eight_species()
    species = [allsp[0], allsp[3]] if ns == 2 else allsp[:ns]
    L = 0.01
    cfg = base_config(n, n, L, L)
    fill_mixture(cfg.mix, species)
    set_scheme(cfg, scheme, split)
    cfg.viscous = int(viscous)
    if ns >= 3:
        m = cfg.mech
        m.present = 1
        m.A, m.Ta, m.a, m.b, m.T_cutoff = 1e9, 15000.0, 1.0, 1.0, 300.0
        m.i_fuel, m.i_ox, m.i_co2, m.i_h2o = 0, 1, -1, 2
        for q in range(ns):
            m.nu[q] = (-2.0, -1.0, 2.0)[q] if q < 3 else 0.0
    la = cfg.laser
    la.present = 1
    la.sigma_r, la.sigma_t = 8e-4, 2e-6
    la.x0, la.y0, la.t0 = 1e-3, -5e-4, 1e-6
    if laser == "shaped":
        la.kernel = abi.LASER_SHAPED
        la.energy = 1.0  # q_shaped ignores it (laser.hpp:79-85); validate() needs >= 0
        la.edot_rate = 1e11
        la.lobe_sep, la.width_up, la.width_down = 1e-3, 1.2e-3, 5e-4
        la.amp_down, la.width_radial = 0.7, 4e-4
    else:
        la.kernel = abi.LASER_GAUSSIAN
        la.energy = 2.0
    Ws = np.array([sp.W for sp in species])
    # unburnt: fuel-lean H2/O2 in N2 (ns = 2: H2/N2), traces of every inert
    Yu = np.full(ns, 0.02)
    Yb = np.full(ns, 0.02)
    if ns == 2:
        Yu[:] = (0.3, 0.7)
        Yb[:] = (0.05, 0.95)
    else:
        Yu[:3] = (0.03, 0.22, 0.0)
        Yb[:3] = (0.005, 0.1, 0.2)
        if ns >= 4:
            Yu[3] = Yb[3] = 0.0
    Yu /= Yu.sum() if ns == 2 else 1.0
    if ns >= 4:  # N2 closes the mass fractions
        Yu[3] = 1.0 - (Yu.sum() - Yu[3])
        Yb[3] = 1.0 - (Yb.sum() - Yb[3])
    elif ns == 3:
        Yu /= Yu.sum()
        Yb /= Yb.sum()

    def ic(X, Yc):
        r2 = (X - 1e-3) ** 2 + (Yc + 1e-3) ** 2
        f = np.exp(-r2 / (2.0 * (1.5e-3) ** 2))
        T = 300.0 + 1500.0 * f
        Ys = [Yu[q] * (1 - f) + Yb[q] * f for q in range(ns)]
        tot = sum(Ys)
        Ys = [y / tot for y in Ys]
        rbar = R_UNIVERSAL * sum(Ys[q] / Ws[q] for q in range(ns))
        rho = 101325.0 / (rbar * T)
        u = 3.0 * np.sin(2 * math.pi * Yc / L)
        v = -2.0 * np.cos(2 * math.pi * X / L)
        return rho, u, v, T, Ys

    dx = L / n
    c_max = 1000.0 if ns == 2 else 900.0
    return Case(f"species{ns}_{n}_{laser}", cfg, ic, 0.2 * dx / c_max)


def wall_channel(n: int = 48, isothermal: bool = True, scheme: str = "teno6",
                 split: str = "char") -> Case:
    """No-slip walls (boundary.hpp:210-226): periodic x, isothermal bottom and
    adiabatic top, 4-species CH4/O2 gas, viscous."""
    L = 0.01
    cfg = base_config(n, n, L, L, periodic=(True, False))
    fill_mixture(cfg.mix, ch4_o2_species())
    set_scheme(cfg, scheme, split)
    cfg.viscous = 1
    cfg.bc.bottom.type = abi.NOSLIP_ISOTHERMAL if isothermal else abi.NOSLIP_ADIABATIC
    cfg.bc.bottom.T_wall = 600.0
    cfg.bc.top.type = abi.NOSLIP_ADIABATIC
    Ws = [0.016, 0.032, 0.044, 0.018]

    def ic(X, Yc):
        Ys = [np.full_like(X, y) for y in (0.1, 0.5, 0.2, 0.2)]
        T = 400.0 + 100.0 * np.sin(2 * math.pi * X / L)
        rbar = R_UNIVERSAL * sum(Ys[s] / Ws[s] for s in range(4))
        rho = 101325.0 / (rbar * T)
        u = 20.0 * np.cos(math.pi * Yc / L)
        v = 5.0 * np.sin(2 * math.pi * X / L) * np.cos(math.pi * Yc / L)
        return rho, u, v, T, Ys

    return Case(f"wall_{n}", cfg, ic, 0.2 * (L / n) / 450.0)


def ensemble_members(n: int = 64, *, seed: int = 1234, nxy=(500, 250), e_lo: float = 0.01,
                     e_hi: float = 0.1, first: int = 0, count=None) -> list:
    """BASELINE configs[4]: members of the H2/O2
    counterflow case C on a 500 x 250 grid whose laser
    energies are sampled U[e_lo, e_hi] with `seed`; members [first, first+count)
    of the n-sample campaign (one GPU's share)."""
    rng = np.random.default_rng(seed)
    energies = rng.uniform(e_lo, e_hi, size=n)
    count = n - first if count is None else count
    return [h2o2_counterflow(nxy[0], nxy=nxy, energy=float(energies[k]))
            for k in range(first, first + count)]


def tgv3d(n: int = 256, *, viscous: bool = True, scheme: str = "teno6",
          split: str = "char", mach: float = 0.1, mu: float = 6.25e-4,
          nz=None) -> Case:
    """BASELINE configs[1]: 3D Taylor-Green vortex on
    [-pi, pi)^3, periodic, u = sin x cos y cos z, v = -cos x sin y cos z,
    w = 0, p = p0 + (1/16)(cos 2x + cos 2y)(cos 2z + 2), rho0 = 1, Ma 0.1,
    Re 1600, gamma-gas with the t_hi cap.  The reference is 2D-only: this runs
    on the 3D extension (flux3.cuh), validated by the z-extrusion cross-check
    (extrude_z).  ``nz`` overrides the z cell count with lz scaled so dz stays
    2 pi / n (weak-scaling stacks)."""
    L = 2.0 * math.pi
    cfg = base_config(n, n, L, L)
    nz = n if nz is None else nz
    cfg.nz, cfg.periodic_z, cfg.lz, cfg.center_z = nz, 1, L * nz / n, 0.0
    gamma = 1.4
    gamma_gas(cfg.mix, gamma, 1.0, mu if viscous else 0.0)
    set_scheme(cfg, scheme, split)
    cfg.viscous = int(viscous)
    p0 = 1.0 / (gamma * mach * mach)
    c0 = math.sqrt(gamma * p0)
    dx = L / n
    # fixed step at CFL <= 0.5 in the reference's stable_dt form (solver.hpp:256-259,
    # summed over the three directions): (|u| + |v| + |w| + 3 c) / dx <= (3 + 3 c0) / dx
    dt = 0.5 * dx / (3.0 + 3.0 * c0)

    def ic(X, Y, Z):
        u = np.sin(X) * np.cos(Y) * np.cos(Z)
        v = -np.cos(X) * np.sin(Y) * np.cos(Z)
        w = np.zeros_like(X)
        p = p0 + (1.0 / 16.0) * (np.cos(2.0 * X) + np.cos(2.0 * Y)) * (np.cos(2.0 * Z) + 2.0)
        rho = np.ones_like(X)
        return rho, u, v, w, p / rho, [np.ones_like(X)]

    return Case(f"tgv3d_{n}" if nz == n else f"tgv3d_{n}x{n}x{nz}", cfg, ic, dt,
                dict(p0=p0, c0=c0))


def jet3d(nx: int = 512, ny: int = 256, nz: int = 32, *, scheme: str = "weno3z",
          split: str = "comp", energy: float = 0.05, zwalls: bool = False) -> Case:
    """BASELINE configs[3] in the form the 3D extension runs (SURVEY §8d config
    D; no reference path): an H2/N2 jet (tanh-smoothed inflow segment, 100 m/s)
    into air coflow (5 m/s) through a 4 cm x 2 cm channel — left inflow, right
    outflow with LODI toward 1 atm, no-slip adiabatic walls at the y edges, z
    periodic with dz = dx — one-step H2/O2 chemistry, the shaped laser kernel
    focused in the shear layer as a 3D point kernel (ign_laser.zmode 1);
    WENO3Z componentwise.  Weak
    scaling stacks z: 512 x 256 x 32 per GPU, 512 x 256 x 256 on 8 GPUs.
    zwalls: no-slip adiabatic walls on the z edges too (a confined duct)."""
    Lx, Ly = 0.04, 0.02
    dx = Lx / nx
    cfg = base_config(nx, ny, Lx, Ly, center=(0.5 * Lx, 0.0), periodic=(False, False))
    cfg.nz, cfg.periodic_z, cfg.lz, cfg.center_z = nz, int(not zwalls), dx * nz, 0.0
    if zwalls:
        cfg.zlo.type = cfg.zhi.type = abi.NOSLIP_ADIABATIC
    species = h2_o2_species()
    fill_mixture(cfg.mix, species)
    set_scheme(cfg, scheme, split)
    cfg.viscous = 1
    Ws = [sp.W for sp in species]
    Yjet = [0.1, 0.0, 0.0, 0.9]
    Yair = [0.0, 0.23, 0.0, 0.77]
    d = 0.002  # jet half width
    e = cfg.bc.left
    e.type = abi.INFLOW
    e.nseg = 3
    e.smooth_width = 2e-4
    for k, (lo, hi, u, Ys) in enumerate(((-0.5 * Ly, -d, 5.0, Yair), (-d, d, 100.0, Yjet),
                                         (d, 0.5 * Ly, 5.0, Yair))):
        sg = e.seg[k]
        sg.lo, sg.hi, sg.u, sg.v, sg.T = lo, hi, u, 0.0, 300.0
        for q in range(4):
            sg.Y[q] = Ys[q]
    cfg.bc.right.type = abi.OUTFLOW
    cfg.bc.right.p_target = 101325.0
    cfg.bc.bottom.type = cfg.bc.top.type = abi.NOSLIP_ADIABATIC
    m = cfg.mech
    m.present = 1
    m.A, m.Ta, m.a, m.b, m.T_cutoff = 1e9, 15000.0, 1.0, 1.0, 300.0
    m.i_fuel, m.i_ox, m.i_co2, m.i_h2o = 0, 1, -1, 2
    for q, nu in enumerate((-2.0, -1.0, 2.0, 0.0)):
        m.nu[q] = nu
    la = cfg.laser
    la.present = 1
    la.kernel = abi.LASER_SHAPED
    la.energy, la.sigma_r, la.sigma_t = energy, 5e-4, 1e-6
    la.x0, la.y0, la.t0 = 0.01, d, 3e-6
    # the shaped two-lobe kernel (laser.hpp:64-85) focused on the shear layer:
    # a point kernel in 3D (ign_laser.zmode 1) with its radial factor over
    # (y, z), ~2.5e5 J/m^3 deposited at the focus (about the gas's own e)
    la.edot_rate = 1e11
    la.lobe_sep, la.width_up, la.width_down = 1e-3, 1.2e-3, 5e-4
    la.amp_down, la.width_radial = 0.7, 4e-4
    la.zmode, la.z0 = 1, 0.0

    def ic(X, Y, Z):
        f = 0.5 * (np.tanh((Y + d) / 2e-4) - np.tanh((Y - d) / 2e-4))  # 1 in the jet
        f = f * np.exp(-np.maximum(X, 0.0) / 0.005)                    # decaying core
        Ys = [Yjet[q] * f + Yair[q] * (1 - f) for q in range(4)]
        T = np.full_like(X, 300.0)
        rbar = R_UNIVERSAL * sum(Ys[q] / Ws[q] for q in range(4))
        rho = 101325.0 / (rbar * T)
        # jet velocity with a weak spanwise perturbation so 3D structure develops
        lz = cfg.lz
        u = 5.0 + 95.0 * f * (1.0 + 0.02 * np.sin(2 * math.pi * Z / lz))
        w = 2.0 * f * np.sin(2 * math.pi * X / 0.01)
        return rho, u, np.zeros_like(X), w, T, Ys

    c_max = 1300.0  # sound speed bound of the H2/N2 jet at 300 K
    return Case(f"jet3d_{nx}x{ny}x{nz}" + ("_zw" if zwalls else ""), cfg, ic,
                0.3 * dx / (c_max + 100.0))


def extrude_z(case: Case, nz: int = 7) -> Case:
    """The z-extrusion cross-check of SURVEY §8c: a 2D periodic case on the 3D
    path with nz >= 2g+1 planes, dz = 1.0 exactly (lz = nz), w = 0 and data
    constant in z.  Its state must reproduce the 2D oracle's plane for plane."""
    cfg = abi.Config()
    ctypes.memmove(ctypes.byref(cfg), ctypes.byref(case.cfg), ctypes.sizeof(abi.Config))
    cfg.nz, cfg.periodic_z, cfg.lz, cfg.center_z = nz, 1, float(nz), 0.0
    ic2 = case.ic

    def ic(X, Y, Z):
        rho, u, v, T, Ys = ic2(X, Y)
        return rho, u, v, np.zeros_like(X), T, Ys

    return Case(case.name + f"_z{nz}", cfg, ic, case.dt, dict(case.notes, ic2=ic2))


def lay_xz(case: Case, ny: int = 7) -> Case:
    """A 2D case laid in the (x, z) plane of a 3D box: the 2D y axis becomes z
    (its edges — periodic, walls or outflow — become the z edges), y is
    periodic with ny cells of dy = 1 and the data constant in y, v = 0.  Checks
    the zeta-face kernels and the z-edge rules against the 2D oracle."""
    c2 = case.cfg
    cfg = abi.Config()
    ctypes.memmove(ctypes.byref(cfg), ctypes.byref(c2), ctypes.sizeof(abi.Config))
    cfg.ny, cfg.ly, cfg.center_y = ny, float(ny), 0.0
    cfg.nz, cfg.lz, cfg.center_z, cfg.periodic_z = c2.ny, c2.ly, c2.center_y, c2.periodic_y
    if not c2.periodic_y:
        if abi.INFLOW in (c2.bc.bottom.type, c2.bc.top.type):
            raise ValueError("lay_xz: inflow is not supported on z edges")
        ctypes.memmove(ctypes.byref(cfg.zlo), ctypes.byref(c2.bc.bottom), ctypes.sizeof(abi.Edge))
        ctypes.memmove(ctypes.byref(cfg.zhi), ctypes.byref(c2.bc.top), ctypes.sizeof(abi.Edge))
        cfg.periodic_y = 1
        cfg.bc.bottom.type = cfg.bc.top.type = abi.PERIODIC
    ic2 = case.ic

    def ic(X, Y, Z):
        rho, u, v, T, Ys = ic2(X, Z)
        return rho, u, np.zeros_like(X), v, T, Ys

    return Case(case.name + f"_xz{ny}", cfg, ic, case.dt, dict(case.notes, ic2=ic2))


def state_2d_to_3d(Ut2: np.ndarray, ns: int, nz: int, g: int = 3) -> np.ndarray:
    """[rhoY_s, rho u, rho v, E] planes -> [rhoY_s, rho u, rho v, rho w = 0, E]
    replicated over nz + 2g z planes."""
    nc2 = Ut2.shape[0]
    out = np.zeros((nc2 + 1, nz + 2 * g) + Ut2.shape[1:])
    out[: ns + 2] = Ut2[: ns + 2][:, None]
    out[ns + 3] = Ut2[ns + 2][None]
    return out


def state_3d_to_2d(Ut3: np.ndarray, ns: int, k: int) -> np.ndarray:
    """One z plane (padded index k) of a 3D state in the 2D component order."""
    return np.concatenate([Ut3[: ns + 2, k], Ut3[ns + 3: ns + 4, k]])


def padded_coords(cfg: abi.Config):
    """Computational node coordinates over the padded box (mesh.hpp:39-42);
    for unskewed meshes these are the physical coordinates."""
    g = cfg.g
    dxi, deta = cfg.lx / cfg.nx, cfg.ly / cfg.ny
    i = np.arange(-g, cfg.nx + g)
    j = np.arange(-g, cfg.ny + g)
    xs = cfg.center_x - 0.5 * cfg.lx + (i + 0.5) * dxi
    ys = cfg.center_y - 0.5 * cfg.ly + (j + 0.5) * deta
    return np.meshgrid(xs, ys)
