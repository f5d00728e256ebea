// flux3.cuh — 3D extension of the inviscid flux / Roe / eigensystem
// (flux.hpp:39-186) on EXTRUDED meshes: the (x, y) metrics are the reference's
// 2D ones, z is uniform, so xi/eta faces have normals (n1, n2, 0) and zeta
// faces (0, 0, 1).  The reference is 2D-only; every 3D expression
// below is written as "the reference's 2D expression, then the z terms", so
// for w = 0 and z-independent data it reduces exactly to the 2D one — the
// z-extrusion cross-check of SURVEY §8c (tests/test_gpu_3d.py).
//
// Component order: [rho Y_s, rho u, rho v, rho w, E] (nc = ns + 4).
// Characteristic fields: [acoustic-, species, shear 1, shear 2, acoustic+];
// for xi/eta faces shear 1 is the reference's (-n2, n1) direction and shear 2
// is z; for zeta faces the tangents are x and y.
#pragma once

#include "flux.cuh"
#include "physics.cuh"

namespace ign {

template <int NS> struct Prim3 {
    double rho, u, v, w, p, T;
    double Y[NS];
};

// conservative_from_primitives (state.hpp:47-57) + w
template <int NS, int TM = 0>
IGN_HD void conservative_from_primitives3(const Prim3<NS>& pt, const DMix& m, double* U) {
#pragma unroll
    for (int s = 0; s < NS; ++s) U[s] = pt.rho * pt.Y[s];
    U[NS] = pt.rho * pt.u;
    U[NS + 1] = pt.rho * pt.v;
    U[NS + 2] = pt.rho * pt.w;
    const double rs = r_specific<NS>(pt.Y, m);
    const double e = e_mass_rs<NS, false, TM>(pt.T, pt.Y, rs, m);
    U[NS + 3] = pt.rho * (e + 0.5 * ((pt.u * pt.u + pt.v * pt.v) + pt.w * pt.w));
}

// primitives_from_conservative (state.hpp:26-44) + w
template <int NS, bool BF = false, int TM = 0>
IGN_HD int primitives_from_conservative3(const double* U, const DMix& m, double T_guess,
                                         Prim3<NS>& pt, double* rs_out) {
    double rho = 0.0;
#pragma unroll
    for (int s = 0; s < NS; ++s) rho += U[s];
    if (!(rho > 0.0)) return P_NONPOS_RHO;
    pt.rho = rho;
    const double yr = 1.0 / rho;
#pragma unroll
    for (int s = 0; s < NS; ++s) pt.Y[s] = fdiv(U[s], rho, yr);
    pt.u = fdiv(U[NS], rho, yr);
    pt.v = fdiv(U[NS + 1], rho, yr);
    pt.w = fdiv(U[NS + 2], rho, yr);
    const double e =
        fdiv(U[NS + 3], rho, yr) - 0.5 * ((pt.u * pt.u + pt.v * pt.v) + pt.w * pt.w);
    const double rs = r_specific<NS>(pt.Y, m);
    int st;
    pt.T = temperature_from_energy<NS, BF, TM>(e, pt.Y, rs, m, T_guess, &st);
    if (st != T_OK) return st;
    pt.p = pt.rho * rs * pt.T;
    *rs_out = rs;
    return P_OK;
}

// mapped_flux (flux.hpp:39-50); DIR < 2: (m1, m2, 0), DIR 2: (0, 0, m3).
// u, v, w are the cache's velocities, i.e. exactly U[NS..NS+2] / rho
// (see mapped_flux_uv)
template <int NS, int DIR>
IGN_HD void mapped_flux3(const double* U, double p, double u, double v, double w, double m1,
                         double m2, double* Ft) {
    const double uhat = DIR < 2 ? m1 * u + m2 * v : m1 * w;
#pragma unroll
    for (int s = 0; s < NS; ++s) Ft[s] = U[s] * uhat;
    if (DIR < 2) {
        Ft[NS] = U[NS] * uhat + m1 * p;
        Ft[NS + 1] = U[NS + 1] * uhat + m2 * p;
        Ft[NS + 2] = U[NS + 2] * uhat;
    } else {
        Ft[NS] = U[NS] * uhat;
        Ft[NS + 1] = U[NS + 1] * uhat;
        Ft[NS + 2] = U[NS + 2] * uhat + m1 * p;
    }
    Ft[NS + 3] = (U[NS + 3] + p) * uhat;
}

// roe_average (flux.hpp:157-186) + w
template <int NS, int TM = 0>
IGN_HD void roe_average3(double rho_l, const double* Yl, double Tl, double ul, double vl,
                         double wl_, double rho_r, const double* Yr, double Tr, double ur,
                         double vr, double wr_, const DMix& m, double* Y, double& T, double& u,
                         double& v, double& w) {
    const double wl = sqrt(rho_l);
    const double wr = sqrt(rho_r);
    const double inv = 1.0 / (wl + wr);
    u = (wl * ul + wr * ur) * inv;
    v = (wl * vl + wr * vr) * inv;
    w = (wl * wl_ + wr * wr_) * inv;
#pragma unroll
    for (int s = 0; s < NS; ++s) Y[s] = (wl * Yl[s] + wr * Yr[s]) * inv;
    const double Hl = h_mass<NS, false, TM>(Tl, Yl, m) + 0.5 * ((ul * ul + vl * vl) + wl_ * wl_);
    const double Hr = h_mass<NS, false, TM>(Tr, Yr, m) + 0.5 * ((ur * ur + vr * vr) + wr_ * wr_);
    const double H = (wl * Hl + wr * Hr) * inv;
    const double h = H - 0.5 * ((u * u + v * v) + w * w);
    double Tt = 0.5 * (Tl + Tr);
    // calorically perfect (TM 1): cp does not depend on T, so its reciprocal
    // is formed once and every iteration's r / cp is a Markstein quotient
    // (correctly rounded, IEEE fallback) instead of an IEEE division
    const double cp1 = TM == 1 ? cp_mass<NS, false, TM>(Tt, Y, m) : 0.0;
    const double ycp1 = TM == 1 ? 1.0 / cp1 : 0.0;
    for (int it = 0; it < 50; ++it) {
        const double r = h_mass<NS, false, TM>(Tt, Y, m) - h;
        const double cp = TM == 1 ? cp1 : cp_mass<NS, false, TM>(Tt, Y, m);
        const double Tn = Tt - (TM == 1 ? fdiv(r, cp, ycp1) : r / cp);
        if (fabs(Tn - Tt) <= 1e-14 * Tt) {
            Tt = Tn;
            break;
        }
        Tt = Tn > 0.0 ? Tn : 0.5 * Tt;
    }
    T = Tt;
}

// EigenSystem (flux.hpp:55-148) for one face family
template <int NS> struct Eigen3 {
    double n1, n2, n3, s, u, v, w, un, ut1, ut2, k, H, c, c2, kappa, yc2, ykappa;
    double Y[NS];
    double Theta[NS];
};

// EigenSystem::at_state (flux.hpp:72-104); DIR < 2: m = (m1, m2, 0), DIR 2: (0, 0, m1)
template <int NS, int DIR, int TM = 0>
IGN_HD int eigen_at_state3(const double* Y, double T, double uu, double vv, double ww,
                           double m1, double m2, const DMix& m, Eigen3<NS>& e) {
    if (DIR < 2) {
        e.s = sqrt(m1 * m1 + m2 * m2);
        if (!(e.s > 0.0)) return E_ZERO_METRIC;
        // two quotients over one divisor: Markstein with the shared RN(1/s)
        const double ys = 1.0 / e.s;
        e.n1 = fdiv(m1, e.s, ys);
        e.n2 = fdiv(m2, e.s, ys);
        e.n3 = 0.0;
        e.un = e.n1 * uu + e.n2 * vv;
        e.ut1 = -e.n2 * uu + e.n1 * vv;
        e.ut2 = ww;
    } else {
        e.s = sqrt(m1 * m1);
        if (!(e.s > 0.0)) return E_ZERO_METRIC;
        e.n1 = 0.0;
        e.n2 = 0.0;
        e.n3 = m1 / e.s;
        e.un = e.n3 * ww;
        e.ut1 = uu;
        e.ut2 = vv;
    }
    e.u = uu;
    e.v = vv;
    e.w = ww;
    e.k = 0.5 * ((uu * uu + vv * vv) + ww * ww);
#pragma unroll
    for (int s = 0; s < NS; ++s) e.Y[s] = Y[s];
    const double rbar = r_specific<NS>(Y, m);
    const double cv = cp_mass<NS, false, TM>(T, Y, m) - rbar;
    e.kappa = rbar / cv;
    const double h = h_mass<NS, false, TM>(T, Y, m);
    double c2 = e.kappa * h;
#pragma unroll
    for (int sp = 0; sp < NS; ++sp) {
        const double rs = divW(m.sp[sp], m.R);
        const double es = h_species<TM>(T, m.sp[sp], m.R) - rs * T;
        const double chi = rs * T - e.kappa * es;
        e.Theta[sp] = chi + e.kappa * e.k;
        c2 += Y[sp] * chi;
    }
    if (!(c2 > 0.0)) return E_NONPOS_C2;
    e.c2 = c2;
    e.c = sqrt(c2);
    e.yc2 = 1.0 / c2;
    e.ykappa = 1.0 / e.kappa;
    e.H = h + e.k;
    return E_OK;
}

}  // namespace ign
