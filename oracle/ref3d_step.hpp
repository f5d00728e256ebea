// oracle/ref3d_step.hpp — TEST INFRASTRUCTURE (CPU checker, never the product).
//
// The reference's time loop restated for the 3D extension (BASELINE
// configs[1], the TGV, and walled / outflow boxes — configs[3]'s edge rules):
// the advance() loop body
// (solver.hpp:336-345) — rk3_step (:304-332) with compute_rhs (:185-232: the
// LODI column on a right outflow, chemistry, laser), axpy / blend on the interior, post_stage (:826-849:
// clip, finiteness, prepare_stage of the next stage) and the trailing
// prepare_stage(1) — where prepare_stage (:422-425) is fill_ghosts
// (boundary.hpp:136-258: periodic copies scaled by J_src/J_dst, no-slip walls
// with every velocity component negated, outflow copies; the x edges over rows
// 0..ny-1, the y edges over the padded width, then the z edges over the padded
// (x, y) plane; inflow with w = 0) and
// refresh_primitives (:148-178) on every padded
// node with the T cache as the Newton guess.  3D expressions follow the
// extension's convention ("the reference's 2D expression, then the z terms":
// e = E/rho - 0.5 ((u u + v v) + w w)); the RHS is ref3d::inviscid_rhs +
// ref3d::viscous_rhs; temperature_from_energy, r_specific and sound_speed are
// the reference's own functions.
#pragma once

#include <cmath>
#include <stdexcept>
#include <vector>

#include "ref3d_faces.hpp"
#include "ref3d_viscous.hpp"

namespace ref3d {

struct Run3 {
    Grid G;
    Met3 M, Mv;
    MixtureModel mix;
    ignis::SchemeConfig sc;
    bool viscous = true;
    std::vector<double> Ut;    // nc planes over the padded box
    std::vector<double> prim;  // rho, u, v, w, p, T, c, Y_s planes (the T cache among them)
    double last_clip = 0.0;

    int nc() const { return G.ns + 4; }
    double& U(int c, long id) { return Ut[size_t(c) * G.plane + id]; }
    double& Pf(int f, long id) { return prim[size_t(f) * G.plane + id]; }

    // edge rules: x / y edges left, right, bottom, top; z edges back, front
    // (0 periodic, 1 no-slip isothermal, 2 no-slip adiabatic, 3 inflow (x / y
    // edges), 4 outflow; a right-edge outflow brings the LODI column)
    int etype[4] = {0, 0, 0, 0}, ztype[2] = {0, 0};
    double Twall[4] = {0, 0, 0, 0}, Tzwall[2] = {0, 0};
    // the reference Simulation built from the same config: its mesh (inflow
    // coordinates, laser node coordinates, lx), bc (inflow / LODI specs),
    // mech and laser
    const ignis::Simulation* S = nullptr;
    // the extension's 3D laser placement: zmode 0 = the reference's 2D kernel
    // on every plane, 1 = the point kernel at z0; node z = zc0 + (k + 1/2) dz
    int laser_zmode = 0;
    double laser_z0 = 0.0, zc0 = 0.0, dz = 1.0;
    double time = 0.0;

    // primitives_from_conservative (state.hpp:26-44) + w at a node, guess 300 K
    struct Prim {
        double rho, u, v, w, p, T;
        SpeciesArray Y;
    };
    Prim prim_at(int i, int j, int k) {
        const int ns = G.ns;
        const long id = G.at(i, j, k);
        const double J = M.jac[G.at2(i, j)];
        std::vector<double> Uc(nc());
        for (int c = 0; c < nc(); ++c) Uc[c] = U(c, id) * J;
        Prim pt{};
        double rho = 0.0;
        for (int s = 0; s < ns; ++s) rho += Uc[s];
        if (!(rho > 0.0)) throw ignis::StateError("primitives: non-positive density");
        pt.rho = rho;
        for (int s = 0; s < ns; ++s) pt.Y[s] = Uc[s] / rho;
        pt.u = Uc[ns] / rho;
        pt.v = Uc[ns + 1] / rho;
        pt.w = Uc[ns + 2] / rho;
        const double e = Uc[ns + 3] / rho - 0.5 * ((pt.u * pt.u + pt.v * pt.v) + pt.w * pt.w);
        pt.T = ignis::temperature_from_energy(e, pt.Y, mix, 300.0);
        pt.p = pt.rho * ignis::thermo::r_specific(pt.Y, mix) * pt.T;
        return pt;
    }
    // store_prim (boundary.hpp:158-162) with conservative_from_primitives
    // (state.hpp:47-57) + w
    void store_prim(const Prim& pt, int i, int j, int k) {
        const int ns = G.ns;
        std::vector<double> Uc(nc());
        for (int s = 0; s < ns; ++s) Uc[s] = pt.rho * pt.Y[s];
        Uc[ns] = pt.rho * pt.u;
        Uc[ns + 1] = pt.rho * pt.v;
        Uc[ns + 2] = pt.rho * pt.w;
        const double e = ignis::thermo::e_mass(pt.T, pt.Y, mix);
        Uc[ns + 3] = pt.rho * (e + 0.5 * ((pt.u * pt.u + pt.v * pt.v) + pt.w * pt.w));
        const double invJ = 1.0 / M.jac[G.at2(i, j)];
        const long id = G.at(i, j, k);
        for (int c = 0; c < nc(); ++c) U(c, id) = Uc[c] * invJ;
    }
    // no-slip wall (boundary.hpp:210-226): mirror, every velocity component negated
    void wall(int type, double Tw, int im, int jm, int km, int ig, int jg, int kg) {
        Prim pt = prim_at(im, jm, km);
        pt.u = -pt.u;
        pt.v = -pt.v;
        pt.w = -pt.w;
        if (type == 1) {
            const double tg = 2.0 * Tw - pt.T;
            pt.T = std::max(tg, 0.05 * Tw);
        }
        pt.rho = pt.p / (ignis::thermo::r_specific(pt.Y, mix) * pt.T);
        store_prim(pt, ig, jg, kg);
    }

    // fill_ghosts (boundary.hpp:136-258) + z: the x edges over rows 0..ny-1,
    // the y edges over the padded width (every interior plane), then the z
    // edges over the padded (x, y) plane
    void fill_ghosts() {
        const int g = G.g, nx = G.nx, ny = G.ny, nz = G.nz;
        auto copy = [&](int is, int js, int ks, int id_, int jd, int kd) {
            const double ratio = M.jac[G.at2(is, js)] / M.jac[G.at2(id_, jd)];
            const long s = G.at(is, js, ks), d = G.at(id_, jd, kd);
            for (int c = 0; c < nc(); ++c) U(c, d) = U(c, s) * ratio;
        };
        // edge e (0 left, 1 right, 2 bottom, 3 top), transverse t, plane k
        auto edge = [&](int e, int t, int k) {
            const bool xe = e < 2, lo = e % 2 == 0;
            const int n = xe ? nx : ny;
            auto ij = [&](int a, int& i, int& j) {
                if (xe) { i = a; j = t; } else { i = t; j = a; }
            };
            if (etype[e] == 3) {  // inflow (boundary.hpp:227-241), w = 0
                const ignis::EdgeSpec& es =
                    e == 0 ? S->bc.left : e == 1 ? S->bc.right : e == 2 ? S->bc.bottom : S->bc.top;
                int ii, ji;
                ij(lo ? 0 : n - 1, ii, ji);
                const Prim inner = prim_at(ii, ji, k);
                for (int l = 1; l <= g; ++l) {
                    int gi, gj;
                    ij(lo ? -l : n - 1 + l, gi, gj);
                    const double yc = xe ? S->mesh.eta(gj) : S->mesh.xi(gi);
                    Prim pt{};
                    ignis::detail::inflow_profile(es, yc, G.ns, pt.u, pt.v, pt.T, pt.Y);
                    pt.w = 0.0;
                    pt.p = inner.p;
                    pt.rho = pt.p / (ignis::thermo::r_specific(pt.Y, mix) * pt.T);
                    store_prim(pt, gi, gj, k);
                }
                return;
            }
            for (int l = 1; l <= g; ++l) {
                int gi, gj, si, sj;
                ij(lo ? -l : n - 1 + l, gi, gj);
                switch (etype[e]) {
                case 0: ij(lo ? n - l : l - 1, si, sj); copy(si, sj, k, gi, gj, k); break;
                case 1:
                case 2: ij(lo ? l - 1 : n - l, si, sj); wall(etype[e], Twall[e], si, sj, k, gi, gj, k); break;
                case 4: ij(lo ? 0 : n - 1, si, sj); copy(si, sj, k, gi, gj, k); break;
                default: throw std::runtime_error("ref3d_step: unsupported edge type");
                }
            }
        };
        for (int e = 0; e < 2; ++e)
            for (int k = 0; k < nz; ++k)
                for (int j = 0; j < ny; ++j) edge(e, j, k);
        for (int e = 2; e < 4; ++e)
            for (int k = 0; k < nz; ++k)
                for (int i = -g; i < nx + g; ++i) edge(e, i, k);
        for (int side = 0; side < 2; ++side)
            for (int j = -g; j < ny + g; ++j)
                for (int i = -g; i < nx + g; ++i)
                    for (int l = 1; l <= g; ++l) {
                        const int kg = side == 0 ? -l : nz - 1 + l;
                        switch (ztype[side]) {
                        case 0: copy(i, j, side == 0 ? nz - l : l - 1, i, j, kg); break;
                        case 1:
                        case 2: wall(ztype[side], Tzwall[side], i, j, side == 0 ? l - 1 : nz - l, i, j, kg); break;
                        case 4: copy(i, j, side == 0 ? 0 : nz - 1, i, j, kg); break;
                        default: throw std::runtime_error("ref3d_step: unsupported z edge type");
                        }
                    }
    }

    // refresh_primitives (solver.hpp:148-178) + z
    void refresh_primitives(int stage) {
        const int ns = G.ns, g = G.g;
        for (int k = -g; k < G.nz + g; ++k)
            for (int j = -g; j < G.ny + g; ++j)
                for (int i = -g; i < G.nx + g; ++i) {
                    const long id = G.at(i, j, k);
                    const double J = M.jac[G.at2(i, j)];
                    std::vector<double> Uc(nc());
                    for (int c = 0; c < nc(); ++c) Uc[c] = U(c, id) * J;
                    double rho = 0.0;
                    for (int s = 0; s < ns; ++s) rho += Uc[s];
                    if (!(rho > 0.0))
                        throw ignis::StepFailure("stage state failure: non-positive density",
                                                 stage, i, j);
                    SpeciesArray Y{};
                    for (int s = 0; s < ns; ++s) Y[s] = Uc[s] / rho;
                    const double u = Uc[ns] / rho, v = Uc[ns + 1] / rho, w = Uc[ns + 2] / rho;
                    const double e = Uc[ns + 3] / rho - 0.5 * ((u * u + v * v) + w * w);
                    double T;
                    try {
                        T = ignis::temperature_from_energy(e, Y, mix, Pf(5, id));
                    } catch (const ignis::StateError& ex) {
                        throw ignis::StepFailure(std::string("stage state failure: ") + ex.what(),
                                                 stage, i, j);
                    }
                    Pf(0, id) = rho;
                    Pf(1, id) = u;
                    Pf(2, id) = v;
                    Pf(3, id) = w;
                    Pf(4, id) = rho * ignis::thermo::r_specific(Y, mix) * T;
                    Pf(5, id) = T;
                    Pf(6, id) = ignis::thermo::sound_speed(T, Y, mix);
                    for (int s = 0; s < ns; ++s) Pf(7 + s, id) = Y[s];
                }
    }

    void prepare_stage(int stage) {
        fill_ghosts();
        refresh_primitives(stage);
    }

    // lodi_outflow_override (solver.hpp:717-788) on the right-edge column of
    // every plane, the second transverse wave (w) appended: L4 = out dw/dn,
    // dw/dt = -L4.  Returns -dU/J as [c][k][j].
    std::vector<double> lodi_dF() {
        const int ns = G.ns, i = G.nx - 1;
        const ignis::EdgeSpec& es = S->bc.right;
        std::vector<double> out(size_t(nc()) * G.nz * G.ny);
        for (int k = 0; k < G.nz; ++k)
            for (int j = 0; j < G.ny; ++j) {
                const int q = G.at2(i, j);
                const long id = G.at(i, j, k);
                const double xi_x = Mv.mxx[q] * Mv.jac[q];
                const double xi_y = Mv.mxy[q] * Mv.jac[q];
                const double sn = std::hypot(xi_x, xi_y);
                const double n1 = xi_x / sn, n2 = xi_y / sn;
                auto ddn = [&](int f) {
                    const double* a = prim.data() + size_t(f) * G.plane;
                    return sn * 0.5 * (3.0 * a[id] - 4.0 * a[id - 1] + a[id - 2]);
                };
                const double rr = Pf(0, id), cc0 = Pf(6, id), pp = Pf(4, id);
                const double uu = Pf(1, id), vv = Pf(2, id), ww = Pf(3, id);
                const double un = n1 * uu + n2 * vv;
                const double Ma = std::min(std::abs(un) / cc0, 0.99);
                const double drdn = ddn(0);
                const double dpdn = ddn(4);
                const double dundn = n1 * ddn(1) + n2 * ddn(2);
                const double dutdn = -n2 * ddn(1) + n1 * ddn(2);
                const double dwdn = ddn(3);
                const double K = es.sigma_out * cc0 * (1.0 - Ma * Ma) / S->mesh.lx;
                const double L1 = K * (pp - es.p_target);
                const double o = un > 0.0 ? un : 0.0;
                const double L2 = o * (cc0 * cc0 * drdn - dpdn);
                const double L3 = o * dutdn;
                const double L4 = o * dwdn;
                const double L5 = (un + cc0) * (dpdn + rr * cc0 * dundn);
                const double drdt = -(L2 + 0.5 * (L5 + L1)) / (cc0 * cc0);
                const double dundt = -(L5 - L1) / (2.0 * rr * cc0);
                const double dutdt = -L3;
                const double dwdt = -L4;
                const double dpdt = -0.5 * (L5 + L1);
                SpeciesArray Y{}, dYdt{};
                double sumRdY = 0.0;
                for (int sp = 0; sp < ns; ++sp) {
                    Y[sp] = Pf(7 + sp, id);
                    dYdt[sp] = -o * ddn(7 + sp);
                    sumRdY += (mix.R / mix.species[sp].W) * dYdt[sp];
                }
                const double rbar = ignis::thermo::r_specific(Y, mix);
                const double Tt = Pf(5, id);
                const double dTdt = Tt * (dpdt / pp - drdt / rr - sumRdY / rbar);
                const double dudt = n1 * dundt - n2 * dutdt;
                const double dvdt = n2 * dundt + n1 * dutdt;
                const double kin = 0.5 * ((uu * uu + vv * vv) + ww * ww);
                const double e = ignis::thermo::e_mass(Tt, Y, mix);
                const double cv = ignis::thermo::cv_mass(Tt, Y, mix);
                double sum_es_dY = 0.0;
                for (int sp = 0; sp < ns; ++sp) {
                    const double esn = ignis::thermo::h_species(Tt, sp, mix) -
                                       (mix.R / mix.species[sp].W) * Tt;
                    sum_es_dY += esn * dYdt[sp];
                }
                std::vector<double> dU(nc());
                for (int sp = 0; sp < ns; ++sp) dU[sp] = Y[sp] * drdt + rr * dYdt[sp];
                dU[ns] = uu * drdt + rr * dudt;
                dU[ns + 1] = vv * drdt + rr * dvdt;
                dU[ns + 2] = ww * drdt + rr * dwdt;
                dU[ns + 3] = (e + kin) * drdt + rr * cv * dTdt + rr * sum_es_dY +
                             rr * ((uu * dudt + vv * dvdt) + ww * dwdt);
                const double invJ = 1.0 / M.jac[q];
                for (int c = 0; c < nc(); ++c)
                    out[(size_t(c) * G.nz + k) * G.ny + j] = -dU[c] * invJ;
            }
        return out;
    }

    // the extension's point kernel (zmode 1): the reference's q_gaussian /
    // q_shaped (laser.hpp:53-85) with z in the radial distance, (2 pi)^2
    // normalisation of the 3D Gaussian
    double laser3(double x, double y, double z, double t) const {
        const ignis::LaserParams& p = *S->laser;
        if (laser_zmode == 0) return ignis::laser_power(x, y, t, p);
        const double dtn = (t - p.t0) / p.sigma_t;
        if (p.kernel == ignis::LaserKernel::Gaussian) {
            const double r2 = ((x - p.x0) * (x - p.x0) + (y - p.y0) * (y - p.y0)) +
                              (z - laser_z0) * (z - laser_z0);
            const double pow2pi2 = (2.0 * M_PI) * (2.0 * M_PI);
            const double norm =
                p.energy / (pow2pi2 * p.sigma_r * p.sigma_r * p.sigma_r * p.sigma_t);
            return norm * std::exp(-0.5 * r2 / (p.sigma_r * p.sigma_r)) *
                   std::exp(-0.5 * dtn * dtn);
        }
        const auto& sp = p.profile;
        const double dx = x - p.x0;
        const double dy = (y - p.y0) / sp.width_radial;
        const double dzr = (z - laser_z0) / sp.width_radial;
        const double zu = (dx + sp.lobe_sep) / sp.width_up;
        const double zd = (dx - sp.lobe_sep) / sp.width_down;
        const double up = std::exp(-0.5 * (zu * zu));
        const double dn = sp.amp_down * std::exp(-0.5 * (zd * zd));
        double f = (up + dn) * std::exp(-0.5 * (dy * dy + dzr * dzr));
        f = f > 1.0 ? 1.0 : f;
        return p.edot_rate * f * std::exp(-0.5 * dtn * dtn);
    }

    // compute_rhs (solver.hpp:185-232) + z: -((dF + dG) + dH) (LODI column on
    // a right outflow), + (dVx + dVy) + dVz, chemistry, laser; interior
    void compute_rhs(std::vector<double>& r, double t_stage) {
        r.assign(Ut.size(), 0.0);
        std::vector<double> ldf;
        const bool lodi = S && S->bc.right.type == ignis::BCType::Outflow;
        if (lodi) ldf = lodi_dF();
        inviscid_rhs(G, M, mix, sc, Ut.data(), prim.data(), r.data(), lodi ? &ldf : nullptr);
        if (viscous) {
            std::vector<double> dv(Ut.size(), 0.0);
            viscous_rhs(G, Mv, mix, prim.data(), dv.data());
            for (int c = 0; c < nc(); ++c)
                for (int k = 0; k < G.nz; ++k)
                    for (int j = 0; j < G.ny; ++j)
                        for (int i = 0; i < G.nx; ++i) {
                            const size_t q = size_t(c) * G.plane + G.at(i, j, k);
                            r[q] += dv[q];
                        }
        }
        const bool chem = S && S->mech.has_value();
        const bool las = S && S->laser.has_value() && S->laser->energy != 0.0;
        const int ns = G.ns;
        for (int k = 0; k < G.nz; ++k)
            for (int j = 0; j < G.ny; ++j)
                for (int i = 0; i < G.nx; ++i) {
                    const long id = G.at(i, j, k);
                    const double invJ = 1.0 / M.jac[G.at2(i, j)];
                    if (chem) {
                        SpeciesArray Y{}, wdot{};
                        for (int sp = 0; sp < ns; ++sp) Y[sp] = Pf(7 + sp, id);
                        ignis::source_terms(Pf(0, id), Pf(5, id), Y, mix, *S->mech, wdot);
                        for (int sp = 0; sp < ns; ++sp) r[size_t(sp) * G.plane + id] += wdot[sp] * invJ;
                    }
                    if (las) {
                        const double z = zc0 + (k + 0.5) * dz;
                        r[size_t(ns + 3) * G.plane + id] +=
                            laser3(S->mesh.x(i, j), S->mesh.y(i, j), z, t_stage) * invJ;
                    }
                    for (int c = 0; c < nc(); ++c)
                        if (!std::isfinite(r[size_t(c) * G.plane + id]))
                            throw ignis::StepFailure("non-finite RHS", 0, i, j);
                }
    }

    // post_stage (solver.hpp:826-849)
    void post_stage(int stage) {
        const int ns = G.ns;
        double clip = 0.0;
        for (int k = 0; k < G.nz; ++k)
            for (int j = 0; j < G.ny; ++j)
                for (int i = 0; i < G.nx; ++i) {
                    const long id = G.at(i, j, k);
                    double rsum = 0.0;
                    for (int s = 0; s < ns; ++s) {
                        double& us = U(s, id);
                        if (us < 0.0) {
                            clip = std::max(clip, -us * M.jac[G.at2(i, j)]);
                            us = 0.0;
                        }
                        rsum += us;
                    }
                    if (!(rsum > 0.0)) throw ignis::StepFailure("non-positive density", stage, i, j);
                    for (int c = 0; c < nc(); ++c)
                        if (!std::isfinite(U(c, id)))
                            throw ignis::StepFailure("non-finite state", stage, i, j);
                }
        last_clip = stage == 1 ? clip : std::max(last_clip, clip);
        if (stage < 3) prepare_stage(stage + 1);
    }

    // rk3_step (solver.hpp:304-332); the interior update b + dt r / b + w((d - b) + dt r)
    void rk3_step(double dt) {
        const std::vector<double> U0 = Ut;
        std::vector<double> r;
        const double wts[3] = {0.0, 0.25, 2.0 / 3.0};
        const double ts[3] = {time, time + dt, time + 0.5 * dt};
        for (int stage = 1; stage <= 3; ++stage) {
            compute_rhs(r, ts[stage - 1]);
            for (int c = 0; c < nc(); ++c)
                for (int k = 0; k < G.nz; ++k)
                    for (int j = 0; j < G.ny; ++j)
                        for (int i = 0; i < G.nx; ++i) {
                            const size_t q = size_t(c) * G.plane + G.at(i, j, k);
                            const double b = U0[q];
                            Ut[q] = stage == 1 ? b + dt * r[q]
                                               : b + wts[stage - 1] * ((Ut[q] - b) + dt * r[q]);
                        }
            post_stage(stage);
        }
        time += dt;
    }

    // the advance() loop body with a pinned dt (solver.hpp:336-345)
    void steps(double dt, int n) {
        for (int s = 0; s < n; ++s) {
            rk3_step(dt);
            prepare_stage(1);
        }
    }
};

}  // namespace ref3d
