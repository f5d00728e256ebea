// flux.cuh — inviscid flux, Roe average and characteristic eigensystem
// (flux.hpp:39-186), same operation order as the reference.
#pragma once

#include "physics.cuh"

namespace ign {

// mapped_flux (flux.hpp:39-50): Ft = m1 F + m2 G from physical U and p
template <int NS>
IGN_HD void mapped_flux(const double* U, double p, double m1, double m2, double* Ft) {
    double rho = 0.0;
#pragma unroll
    for (int s = 0; s < NS; ++s) rho += U[s];
    const double u = U[NS] / rho;
    const double v = U[NS + 1] / rho;
    const double uhat = m1 * u + m2 * v;
#pragma unroll
    for (int s = 0; s < NS; ++s) Ft[s] = U[s] * uhat;
    Ft[NS] = U[NS] * uhat + m1 * p;
    Ft[NS + 1] = U[NS + 1] * uhat + m2 * p;
    Ft[NS + 2] = (U[NS + 2] + p) * uhat;
}

// mapped_flux with the velocity quotients supplied: u = U[NS]/rho and
// v = U[NS+1]/rho are exactly the primitive cache's u, v (primitives_from_
// conservative divides the same U by the same rho, correctly rounded), so the
// face kernels skip two IEEE divisions per node
template <int NS>
IGN_HD void mapped_flux_uv(const double* U, double p, double u, double v, double m1, double m2,
                           double* Ft) {
    const double uhat = m1 * u + m2 * v;
#pragma unroll
    for (int s = 0; s < NS; ++s) Ft[s] = U[s] * uhat;
    Ft[NS] = U[NS] * uhat + m1 * p;
    Ft[NS + 1] = U[NS + 1] * uhat + m2 * p;
    Ft[NS + 2] = (U[NS + 2] + p) * uhat;
}

// roe_average (flux.hpp:157-186): returns Y, T, u, v of the face state
template <int NS, int TM = 0>
IGN_HD void roe_average(double rho_l, const double* Yl, double Tl, double ul, double vl,
                        double rho_r, const double* Yr, double Tr, double ur, double vr,
                        const DMix& m, double* Y, double& T, double& u, double& v) {
    const double wl = sqrt(rho_l);
    const double wr = sqrt(rho_r);
    const double inv = 1.0 / (wl + wr);
    u = (wl * ul + wr * ur) * inv;
    v = (wl * vl + wr * vr) * inv;
#pragma unroll
    for (int s = 0; s < NS; ++s) Y[s] = (wl * Yl[s] + wr * Yr[s]) * inv;
    const double Hl = h_mass<NS, false, TM>(Tl, Yl, m) + 0.5 * (ul * ul + vl * vl);
    const double Hr = h_mass<NS, false, TM>(Tr, Yr, m) + 0.5 * (ur * ur + vr * vr);
    const double H = (wl * Hl + wr * Hr) * inv;
    const double h = H - 0.5 * (u * u + v * v);
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

// EigenSystem (flux.hpp:55-148)
template <int NS> struct Eigen {
    double n1, n2, s, u, v, un, ut, k, H, c, c2, kappa;
    double c2x2, y2c2, yc2, ykappa;  // 2c^2 and RN reciprocals for fdiv
    double Y[NS];
    double Theta[NS];
};

enum EigenStatus { E_OK = 0, E_ZERO_METRIC = 1, E_NONPOS_C2 = 2 };

// EigenSystem::at_state (flux.hpp:72-104)
template <int NS, int TM = 0>
IGN_HD int eigen_at_state(const double* Y, double T, double uu, double vv, double m1,
                          double m2, const DMix& m, Eigen<NS>& e) {
    e.s = sqrt(m1 * m1 + m2 * m2);
    if (!(e.s > 0.0)) return E_ZERO_METRIC;
    // two quotients over one divisor: Markstein with the shared RN(1/s)
    const double ys = 1.0 / e.s;
    e.n1 = fdiv(m1, e.s, ys);
    e.n2 = fdiv(m2, e.s, ys);
    e.u = uu;
    e.v = vv;
    e.un = e.n1 * uu + e.n2 * vv;
    e.ut = -e.n2 * uu + e.n1 * vv;
    e.k = 0.5 * (uu * uu + vv * vv);
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
    e.c2x2 = 2.0 * c2;
    e.y2c2 = 1.0 / e.c2x2;
    e.yc2 = 1.0 / c2;
    e.ykappa = 1.0 / e.kappa;
    e.H = h + e.k;
    return E_OK;
}

// EigenSystem::project (flux.hpp:107-120): w = L q
template <int NS>
IGN_HD void eigen_project(const Eigen<NS>& e, const double* q, double* w) {
    double drho = 0.0;
#pragma unroll
    for (int sp = 0; sp < NS; ++sp) drho += q[sp];
    double dp = e.kappa * q[NS + 2] - e.kappa * e.u * q[NS] - e.kappa * e.v * q[NS + 1];
#pragma unroll
    for (int sp = 0; sp < NS; ++sp) dp += e.Theta[sp] * q[sp];
    const double dun = e.n1 * q[NS] + e.n2 * q[NS + 1] - e.un * drho;
    const double dut = -e.n2 * q[NS] + e.n1 * q[NS + 1] - e.ut * drho;
    w[0] = fdiv(dp - e.c * dun, e.c2x2, e.y2c2);
#pragma unroll
    for (int sp = 0; sp < NS; ++sp) w[1 + sp] = q[sp] - fdiv(e.Y[sp] * dp, e.c2, e.yc2);
    w[1 + NS] = dut;
    w[2 + NS] = fdiv(dp + e.c * dun, e.c2x2, e.y2c2);
}

// EigenSystem::assemble (flux.hpp:123-139): q = R w
template <int NS>
IGN_HD void eigen_assemble(const Eigen<NS>& e, const double* w, double* q) {
    const double am = w[0];
    const double ap = w[2 + NS];
    const double at = w[1 + NS];
    double asum = 0.0;
#pragma unroll
    for (int sp = 0; sp < NS; ++sp) {
        q[sp] = e.Y[sp] * (am + ap) + w[1 + sp];
        asum += w[1 + sp];
    }
    q[NS] = (e.u - e.c * e.n1) * am + (e.u + e.c * e.n1) * ap + e.u * asum - e.n2 * at;
    q[NS + 1] = (e.v - e.c * e.n2) * am + (e.v + e.c * e.n2) * ap + e.v * asum + e.n1 * at;
    double en = (e.H - e.c * e.un) * am + (e.H + e.c * e.un) * ap + e.ut * at;
#pragma unroll
    for (int sp = 0; sp < NS; ++sp)
        en += w[1 + sp] * (2.0 * e.k - (NS > 1 ? fdiv(e.Theta[sp], e.kappa, e.ykappa)
                                               : e.Theta[sp] / e.kappa));
    q[NS + 2] = en;
}

// EigenSystem::field_speed (flux.hpp:143-147)
template <int NS>
IGN_HD double field_speed(const Eigen<NS>& e, int f, double un_k, double c_k) {
    if (f == 0) return e.s * (un_k - c_k);
    if (f == 2 + NS) return e.s * (un_k + c_k);
    return e.s * un_k;
}

}  // namespace ign
