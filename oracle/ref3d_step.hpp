// oracle/ref3d_step.hpp — TEST INFRASTRUCTURE (CPU checker, never the product).
//
// The reference's time loop restated for the 3D extension (BASELINE
// configs[1], the TGV, and walled / outflow boxes — configs[3]'s edge rules):
// the advance() loop body
// (solver.hpp:336-345) — rk3_step (:304-332) with compute_rhs (:185-232, no
// chemistry / laser), axpy / blend on the interior, post_stage (:826-849:
// clip, finiteness, prepare_stage of the next stage) and the trailing
// prepare_stage(1) — where prepare_stage (:422-425) is fill_ghosts
// (boundary.hpp:136-258: periodic copies scaled by J_src/J_dst, no-slip walls
// with every velocity component negated, outflow copies; the x edges over rows
// 0..ny-1, the y edges over the padded width, then the z edges over the padded
// (x, y) plane; inflow and the right-edge LODI are not restated) and
// refresh_primitives (:148-178) on every padded
// node with the T cache as the Newton guess.  3D expressions follow the
// extension's convention ("the reference's 2D expression, then the z terms":
// e = E/rho - 0.5 ((u u + v v) + w w)); the RHS is ref3d::inviscid_rhs +
// ref3d::viscous_rhs; temperature_from_energy, r_specific and sound_speed are
// the reference's own functions.
#pragma once

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
    // (0 periodic, 1 no-slip isothermal, 2 no-slip adiabatic, 4 outflow)
    int etype[4] = {0, 0, 0, 0}, ztype[2] = {0, 0};
    double Twall[4] = {0, 0, 0, 0}, Tzwall[2] = {0, 0};

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

    // compute_rhs (solver.hpp:185-232) without chemistry / laser; interior
    void compute_rhs(std::vector<double>& r) {
        r.assign(Ut.size(), 0.0);
        inviscid_rhs(G, M, mix, sc, Ut.data(), prim.data(), r.data());
        if (!viscous) return;
        std::vector<double> dv(Ut.size(), 0.0);
        viscous_rhs(G, Mv, mix, prim.data(), dv.data());
        for (int c = 0; c < nc(); ++c)
            for (int k = 0; k < G.nz; ++k)
                for (int j = 0; j < G.ny; ++j)
                    for (int i = 0; i < G.nx; ++i) {
                        const size_t q = size_t(c) * G.plane + G.at(i, j, k);
                        r[q] += dv[q];
                    }
        for (int c = 0; c < nc(); ++c)
            for (int k = 0; k < G.nz; ++k)
                for (int j = 0; j < G.ny; ++j)
                    for (int i = 0; i < G.nx; ++i)
                        if (!std::isfinite(r[size_t(c) * G.plane + G.at(i, j, k)]))
                            throw ignis::StepFailure("non-finite RHS", 0, i, j);
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
        for (int stage = 1; stage <= 3; ++stage) {
            compute_rhs(r);
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
