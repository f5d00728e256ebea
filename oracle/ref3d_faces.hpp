// oracle/ref3d_faces.hpp — TEST INFRASTRUCTURE (CPU checker, never the product).
//
// A plain serial restatement of the reference's inviscid faces
// (solver.hpp:441-579: node pass, per-face Roe state, EigenSystem, 2h
// projections, per-field LLF split, face_plus + face_minus, assemble, flux
// difference) for the 3D extension.  The reference has no 3D path (SURVEY
// §0); every 3D expression is "the reference's 2D expression, then the z
// terms", the convention the product states in csrc/flux3.cuh, written here
// independently in the reference's own structure (per face, per field, with
// the reference's EigenSystem-style project/assemble and its recon::face_plus
// / face_minus and thermo functions called directly).  It is the 3D oracle of
// the face kernels (tests/test_gpu_3d.py) and, compiled with the counting
// double of tools/opcount, the source of the 3D algorithmic op count.
//
// Inputs: the padded 3D state Ut (nc = ns + 4 fields, k slowest) and the
// primitive cache the product's prepare_stage left (rho, u, v, w, p, T, c,
// Y_s) — the check isolates the face computation.  Metrics: the reference's
// compute_metrics of the (x, y) mesh, extruded over dz (xi/eta rows x dz, zeta
// row = the 2D area, J = 1/(area dz)), as the product's setup does.
#pragma once

#include <cmath>
#include <vector>

#include "ignis/solver.hpp"

namespace ref3d {

using ignis::MixtureModel;
using ignis::SpeciesArray;

struct Grid {
    int nx, ny, nz, g, ns;
    long sx, sxy, plane;
    long at(int i, int j, int k) const { return long(k + g) * sxy + long(j + g) * sx + (i + g); }
    int at2(int i, int j) const { return (j + g) * int(sx) + (i + g); }
};

// extruded metric planes (2D arrays, (nx+2g)(ny+2g))
struct Met3 {
    std::vector<double> jac, mxx, mxy, mex, mey, mzz;
};

inline Met3 extrude(const ignis::MetricField& m, double dz) {
    Met3 r;
    const size_t n = m.jac.raw().size();
    r.jac.resize(n);
    r.mxx = m.m_xi_x.raw();
    r.mxy = m.m_xi_y.raw();
    r.mex = m.m_eta_x.raw();
    r.mey = m.m_eta_y.raw();
    r.mzz.resize(n);
    for (size_t q = 0; q < n; ++q) {
        const double area = m.m_eta_y.raw()[q] * m.m_xi_x.raw()[q] -
                            (-m.m_xi_y.raw()[q]) * (-m.m_eta_x.raw()[q]);
        r.mzz[q] = area;
        r.jac[q] = 1.0 / (area * dz);
        r.mxx[q] *= dz;
        r.mxy[q] *= dz;
        r.mex[q] *= dz;
        r.mey[q] *= dz;
    }
    return r;
}

// EigenSystem (flux.hpp:55-148) + z: direction dir (0 xi, 1 eta, 2 zeta)
struct Eigen3 {
    int ns = 1, dir = 0;
    double n1 = 0, n2 = 0, n3 = 0, s = 1, u = 0, v = 0, w = 0, un = 0, ut1 = 0, ut2 = 0;
    double k = 0, H = 0, c = 1, c2 = 1, kappa = 0.4;
    SpeciesArray Y{}, Theta{};

    static Eigen3 at_state(const SpeciesArray& Y, double T, double uu, double vv, double ww,
                           double m1, double m2, int dir, const MixtureModel& mix) {
        Eigen3 e;
        e.ns = mix.ns();
        e.dir = dir;
        if (dir < 2) {
            e.s = std::sqrt(m1 * m1 + m2 * m2);
            if (!(e.s > 0.0)) throw ignis::NumericsError("eigen: zero metric direction");
            e.n1 = m1 / e.s;
            e.n2 = m2 / e.s;
            e.un = e.n1 * uu + e.n2 * vv;
            e.ut1 = -e.n2 * uu + e.n1 * vv;
            e.ut2 = ww;
        } else {
            e.s = std::sqrt(m1 * m1);
            if (!(e.s > 0.0)) throw ignis::NumericsError("eigen: zero metric direction");
            e.n3 = m1 / e.s;
            e.un = e.n3 * ww;
            e.ut1 = uu;
            e.ut2 = vv;
        }
        e.u = uu;
        e.v = vv;
        e.w = ww;
        e.k = 0.5 * ((uu * uu + vv * vv) + ww * ww);
        e.Y = Y;
        const double rbar = ignis::thermo::r_specific(Y, mix);
        const double cv = ignis::thermo::cv_mass(T, Y, mix);
        e.kappa = rbar / cv;
        const double h = ignis::thermo::h_mass(T, Y, mix);
        double c2 = e.kappa * h;
        for (int sp = 0; sp < mix.ns(); ++sp) {
            const double rs = mix.R / mix.species[sp].W;
            const double es = ignis::thermo::h_species(T, sp, mix) - rs * T;
            const double chi = rs * T - e.kappa * es;
            e.Theta[sp] = chi + e.kappa * e.k;
            c2 += Y[sp] * chi;
        }
        if (!(c2 > 0.0)) throw ignis::NumericsError("eigen: non-positive c^2");
        e.c2 = c2;
        e.c = std::sqrt(c2);
        e.H = h + e.k;
        return e;
    }

    // w = L q (flux.hpp:107-120 + z): [acoustic-, species, shear 1, shear 2, acoustic+]
    void project(const double* q, double* out) const {
        const int mx = ns, my = ns + 1, mz = ns + 2, en = ns + 3;
        double drho = 0.0;
        for (int sp = 0; sp < ns; ++sp) drho += q[sp];
        double dp = kappa * q[en] - kappa * u * q[mx] - kappa * v * q[my] - kappa * w * q[mz];
        for (int sp = 0; sp < ns; ++sp) dp += Theta[sp] * q[sp];
        double dun, dut1, dut2;
        if (dir < 2) {
            dun = n1 * q[mx] + n2 * q[my] - un * drho;
            dut1 = -n2 * q[mx] + n1 * q[my] - ut1 * drho;
            dut2 = q[mz] - ut2 * drho;
        } else {
            dun = n3 * q[mz] - un * drho;
            dut1 = q[mx] - ut1 * drho;
            dut2 = q[my] - ut2 * drho;
        }
        out[0] = (dp - c * dun) / (2.0 * c2);
        for (int sp = 0; sp < ns; ++sp) out[1 + sp] = q[sp] - Y[sp] * dp / c2;
        out[1 + ns] = dut1;
        out[2 + ns] = dut2;
        out[3 + ns] = (dp + c * dun) / (2.0 * c2);
    }

    // q = R w (flux.hpp:123-139 + z)
    void assemble(const double* wv, double* q) const {
        const double am = wv[0], ap = wv[3 + ns], at1 = wv[1 + ns], at2 = wv[2 + ns];
        double asum = 0.0;
        for (int sp = 0; sp < ns; ++sp) {
            q[sp] = Y[sp] * (am + ap) + wv[1 + sp];
            asum += wv[1 + sp];
        }
        if (dir < 2) {
            q[ns] = (u - c * n1) * am + (u + c * n1) * ap + u * asum - n2 * at1;
            q[ns + 1] = (v - c * n2) * am + (v + c * n2) * ap + v * asum + n1 * at1;
            q[ns + 2] = w * am + w * ap + w * asum + at2;
        } else {
            q[ns] = u * am + u * ap + u * asum + at1;
            q[ns + 1] = v * am + v * ap + v * asum + at2;
            q[ns + 2] = (w - c * n3) * am + (w + c * n3) * ap + w * asum;
        }
        double en = (H - c * un) * am + (H + c * un) * ap + ut1 * at1;
        en = en + ut2 * at2;
        for (int sp = 0; sp < ns; ++sp) en += wv[1 + sp] * (2.0 * k - Theta[sp] / kappa);
        q[ns + 3] = en;
    }

    double field_speed(int f, double un_k, double c_k) const {
        if (f == 0) return s * (un_k - c_k);
        if (f == 3 + ns) return s * (un_k + c_k);
        return s * un_k;
    }
};

// roe_average (flux.hpp:157-186) + w
inline void roe_average3(double rl, const SpeciesArray& Yl, double Tl, double ul, double vl,
                         double wl_, double rr, const SpeciesArray& Yr, double Tr, double ur,
                         double vr, double wr_, const MixtureModel& mix, SpeciesArray& Y,
                         double& T, double& u, double& v, double& w) {
    const double wl = std::sqrt(rl);
    const double wr = std::sqrt(rr);
    const double inv = 1.0 / (wl + wr);
    u = (wl * ul + wr * ur) * inv;
    v = (wl * vl + wr * vr) * inv;
    w = (wl * wl_ + wr * wr_) * inv;
    for (int s = 0; s < mix.ns(); ++s) Y[s] = (wl * Yl[s] + wr * Yr[s]) * inv;
    const double Hl = ignis::thermo::h_mass(Tl, Yl, mix) + 0.5 * ((ul * ul + vl * vl) + wl_ * wl_);
    const double Hr = ignis::thermo::h_mass(Tr, Yr, mix) + 0.5 * ((ur * ur + vr * vr) + wr_ * wr_);
    const double H = (wl * Hl + wr * Hr) * inv;
    const double h = H - 0.5 * ((u * u + v * v) + w * w);
    double Tt = 0.5 * (Tl + Tr);
    for (int it = 0; it < 50; ++it) {
        const double r = ignis::thermo::h_mass(Tt, Y, mix) - h;
        const double cp = ignis::thermo::cp_mass(Tt, Y, mix);
        const double Tn = Tt - r / cp;
        if (std::abs(Tn - Tt) <= 1e-14 * Tt) {
            Tt = Tn;
            break;
        }
        Tt = Tn > 0.0 ? Tn : 0.5 * Tt;
    }
    T = Tt;
}

// The inviscid RHS of the 3D extension: for each direction the reference's
// inviscid_direction (solver.hpp:441-579) along every line, then
// rhs = -((dF + dG) + dH) on the interior (the product's assembly order).
// prim: rho, u, v, w, p, T, c, Y_s planes over the padded box.
// lodi_dF (optional): the right-edge column's replacement of the xi flux
// difference (lodi_outflow_override, solver.hpp:717-788), [c][k][j] at i = nx-1.
inline void inviscid_rhs(const Grid& G, const Met3& M, const MixtureModel& mix,
                         const ignis::SchemeConfig& sc, const double* Ut, const double* prim,
                         double* rhs, const std::vector<double>* lodi_dF = nullptr) {
    const int ns = G.ns, nc = ns + 4, g = G.g, h = sc.stencil_half();
    const bool chr = sc.split == ignis::FluxSplit::Characteristic;
    auto P = [&](int f, long id) { return prim[long(f) * G.plane + id]; };
    std::vector<double> dH[3];
    for (int dir = 0; dir < 3; ++dir) {
        const int n = dir == 0 ? G.nx : dir == 1 ? G.ny : G.nz;
        const int na = dir == 0 ? G.ny : G.nx, nb = dir == 2 ? G.ny : G.nz;
        dH[dir].assign(size_t(nc) * G.nx * G.ny * G.nz, 0.0);
        std::vector<double> Ft(size_t(n + 2 * g) * nc), Uc(size_t(n + 2 * g) * nc);
        std::vector<double> un_s(n + 2 * g), c_s(n + 2 * g), fhat(size_t(n + 1) * nc);
        for (int b = 0; b < nb; ++b)
            for (int a = 0; a < na; ++a) {
                auto node = [&](int m, int& i, int& j, int& k) {
                    if (dir == 0) { i = m; j = a; k = b; }
                    else if (dir == 1) { i = a; j = m; k = b; }
                    else { i = a; j = b; k = m; }
                };
                auto m1_of = [&](int i, int j) {
                    const int q = G.at2(i, j);
                    return dir == 0 ? M.mxx[q] : dir == 1 ? M.mex[q] : M.mzz[q];
                };
                auto m2_of = [&](int i, int j) {
                    const int q = G.at2(i, j);
                    return dir == 0 ? M.mxy[q] : dir == 1 ? M.mey[q] : M.mzz[q];
                };
                // node pass: U = Ut J, mapped flux (flux.hpp:39-50 + z), c
                for (int m = -g; m < n + g; ++m) {
                    int i, j, k;
                    node(m, i, j, k);
                    const long id = G.at(i, j, k);
                    const double J = M.jac[G.at2(i, j)];
                    double* U = &Uc[size_t(m + g) * nc];
                    double* F = &Ft[size_t(m + g) * nc];
                    for (int cc = 0; cc < nc; ++cc) U[cc] = Ut[long(cc) * G.plane + id] * J;
                    double rho = 0.0;
                    for (int s = 0; s < ns; ++s) rho += U[s];
                    const double u = U[ns] / rho, v = U[ns + 1] / rho, w = U[ns + 2] / rho;
                    const double p = P(4, id), m1 = m1_of(i, j), m2 = m2_of(i, j);
                    const double uhat = dir < 2 ? m1 * u + m2 * v : m1 * w;
                    for (int s = 0; s < ns; ++s) F[s] = U[s] * uhat;
                    if (dir < 2) {
                        F[ns] = U[ns] * uhat + m1 * p;
                        F[ns + 1] = U[ns + 1] * uhat + m2 * p;
                        F[ns + 2] = U[ns + 2] * uhat;
                    } else {
                        F[ns] = U[ns] * uhat;
                        F[ns + 1] = U[ns + 1] * uhat;
                        F[ns + 2] = U[ns + 2] * uhat + m1 * p;
                    }
                    F[ns + 3] = (U[ns + 3] + p) * uhat;
                    c_s[m + g] = P(6, id);
                }
                for (int m = -1; m < n; ++m) {  // face m + 1/2
                    int il, jl, kl, ir, jr, kr;
                    node(m, il, jl, kl);
                    node(m + 1, ir, jr, kr);
                    const double m1f = 0.5 * (m1_of(il, jl) + m1_of(ir, jr));
                    const double m2f = 0.5 * (m2_of(il, jl) + m2_of(ir, jr));
                    double* F = &fhat[size_t(m + 1) * nc];
                    double wp[6], wm[6];
                    if (chr) {
                        const long a_ = G.at(il, jl, kl), b_ = G.at(ir, jr, kr);
                        SpeciesArray Yl{}, Yr{}, Ya{};
                        for (int s = 0; s < ns; ++s) {
                            Yl[s] = P(7 + s, a_);
                            Yr[s] = P(7 + s, b_);
                        }
                        double Ta, ua, va, wa;
                        roe_average3(P(0, a_), Yl, P(5, a_), P(1, a_), P(2, a_), P(3, a_),
                                     P(0, b_), Yr, P(5, b_), P(1, b_), P(2, b_), P(3, b_), mix,
                                     Ya, Ta, ua, va, wa);
                        const Eigen3 es = Eigen3::at_state(Ya, Ta, ua, va, wa, m1f, m2f, dir, mix);
                        double lf[6][ignis::kMaxComp + 1], lu[6][ignis::kMaxComp + 1];
                        for (int k = 0; k < 2 * h; ++k) {
                            const int mm = m - h + 1 + k;
                            int i, j, kk;
                            node(mm, i, j, kk);
                            const long id = G.at(i, j, kk);
                            un_s[mm + g] = dir < 2 ? es.n1 * P(1, id) + es.n2 * P(2, id)
                                                   : es.n3 * P(3, id);
                            es.project(&Ft[size_t(mm + g) * nc], lf[k]);
                            es.project(&Uc[size_t(mm + g) * nc], lu[k]);
                        }
                        double amp[ignis::kMaxComp + 1];
                        for (int f = 0; f < nc; ++f) {
                            double alpha = 0.0;
                            for (int k = m - h + 1; k <= m + h; ++k)
                                alpha = std::max(alpha,
                                                 std::abs(es.field_speed(f, un_s[k + g], c_s[k + g])));
                            if (!std::isfinite(alpha))
                                throw ignis::NumericsError("inviscid face: non-finite wavespeed");
                            for (int k = 0; k < 2 * h; ++k) {
                                wp[k] = 0.5 * (lf[k][f] + alpha * lu[k][f]);
                                wm[k] = 0.5 * (lf[k][f] - alpha * lu[k][f]);
                            }
                            amp[f] = ignis::recon::face_plus(sc.scheme, &wp[h - 1], sc.teno_ct,
                                                             sc.eps) +
                                     ignis::recon::face_minus(sc.scheme, &wm[h - 1], sc.teno_ct,
                                                              sc.eps);
                        }
                        es.assemble(amp, F);
                    } else {
                        const double sf = dir < 2 ? std::hypot(m1f, m2f) : std::hypot(m1f, 0.0);
                        double alpha = 0.0;
                        for (int k = m - h + 1; k <= m + h; ++k) {
                            int i, j, kk;
                            node(k, i, j, kk);
                            const long id = G.at(i, j, kk);
                            const double un = dir < 2 ? (m1f * P(1, id) + m2f * P(2, id)) / sf
                                                      : (m1f * P(3, id)) / sf;
                            alpha = std::max(alpha, sf * (std::abs(un) + c_s[k + g]));
                        }
                        if (!std::isfinite(alpha))
                            throw ignis::NumericsError("inviscid face: non-finite wavespeed");
                        for (int cc = 0; cc < nc; ++cc) {
                            for (int k = 0; k < 2 * h; ++k) {
                                const int mm = m - h + 1 + k;
                                const double fv = Ft[size_t(mm + g) * nc + cc];
                                const double uv = Uc[size_t(mm + g) * nc + cc];
                                wp[k] = 0.5 * (fv + alpha * uv);
                                wm[k] = 0.5 * (fv - alpha * uv);
                            }
                            F[cc] = ignis::recon::face_plus(sc.scheme, &wp[h - 1], sc.teno_ct,
                                                            sc.eps) +
                                    ignis::recon::face_minus(sc.scheme, &wm[h - 1], sc.teno_ct,
                                                             sc.eps);
                        }
                    }
                }
                for (int m = 0; m < n; ++m) {
                    int i, j, k;
                    node(m, i, j, k);
                    const size_t cell = (size_t(k) * G.ny + j) * G.nx + i;
                    for (int cc = 0; cc < nc; ++cc)
                        dH[dir][size_t(cc) * G.nx * G.ny * G.nz + cell] =
                            fhat[size_t(m + 1) * nc + cc] - fhat[size_t(m) * nc + cc];
                }
            }
    }
    const size_t ncell = size_t(G.nx) * G.ny * G.nz;
    if (lodi_dF)
        for (int cc = 0; cc < nc; ++cc)
            for (int k = 0; k < G.nz; ++k)
                for (int j = 0; j < G.ny; ++j)
                    dH[0][size_t(cc) * ncell + (size_t(k) * G.ny + j) * G.nx + (G.nx - 1)] =
                        (*lodi_dF)[(size_t(cc) * G.nz + k) * G.ny + j];
    for (int cc = 0; cc < nc; ++cc)
        for (int k = 0; k < G.nz; ++k)
            for (int j = 0; j < G.ny; ++j)
                for (int i = 0; i < G.nx; ++i) {
                    const size_t cell = (size_t(k) * G.ny + j) * G.nx + i;
                    const size_t q = size_t(cc) * ncell + cell;
                    rhs[long(cc) * G.plane + G.at(i, j, k)] = -((dH[0][q] + dH[1][q]) + dH[2][q]);
                }
}

}  // namespace ref3d
