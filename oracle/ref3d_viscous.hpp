// oracle/ref3d_viscous.hpp — TEST INFRASTRUCTURE (CPU checker, never the product).
//
// A plain serial restatement of the reference's compute_viscous
// (solver.hpp:588-711) for the 3D extension: mole fractions on the two-node
// ring (:600-609), per node of the one-node ring the central gradients mapped
// with the Central2 metrics (:614-634), Wilke transport (thermo.hpp:231-262),
// stresses, zero-net species diffusion fluxes and the energy flux (:636-684),
// the mapped node fluxes (:686-693) and their central differences (:699-708).
// The reference is 2D; every 3D expression is "the reference's 2D expression,
// then the z terms" (the convention csrc/flux3.cuh states): div = (ux + vy) +
// wz, the energy flux ((u txx + v txy) + w txz) + ex, the zeta flux mapped by
// the extruded area row alone, dV = (dVx + dVy) + dVz.  Written independently
// of the product's kernels in the reference's own structure, calling the
// reference's thermo::mole_fractions / mean_molar_mass / h_species and
// transport() directly.
//
// Inputs: the product's primitive cache (rho, u, v, w, p, T, c, Y_s planes over
// the padded 3D box) — the check isolates the viscous computation.  Metrics:
// the reference's Central2 compute_metrics of the (x, y) mesh, extruded over dz
// by ref3d::extrude (xi/eta rows x dz, zeta row = the 2D area, J = 1/(area dz)).
#pragma once

#include <vector>

#include "ref3d_faces.hpp"

namespace ref3d {

// dv: the viscous divergence (dVx + dVy) + dVz of every component on the
// interior of the padded planes (ghosts left as passed in).
inline void viscous_rhs(const Grid& G, const Met3& Mv, const MixtureModel& mix,
                        const double* prim, double* dv) {
    const int ns = G.ns, nc = ns + 4;
    enum { RHO = 0, U = 1, V = 2, W = 3, T = 5, Y0 = 7 };
    auto field = [&](int f) { return prim + long(f) * G.plane; };
    const double* u = field(U);
    const double* v = field(V);
    const double* w = field(W);
    const double* Tf = field(T);
    const double* rho = field(RHO);

    // mole fractions one ring beyond the gradient nodes (solver.hpp:600-609)
    std::vector<double> Xs(size_t(ns) * G.plane, 0.0);
    for (int k = -2; k < G.nz + 2; ++k)
        for (int j = -2; j < G.ny + 2; ++j)
            for (int i = -2; i < G.nx + 2; ++i) {
                const long id = G.at(i, j, k);
                SpeciesArray Y{}, X{};
                for (int s = 0; s < ns; ++s) Y[s] = field(Y0 + s)[id];
                ignis::thermo::mole_fractions(Y, mix, X);
                for (int s = 0; s < ns; ++s) Xs[size_t(s) * G.plane + id] = X[s];
            }

    std::vector<double> Fv(size_t(nc) * G.plane, 0.0), Gv(Fv.size(), 0.0), Hv(Fv.size(), 0.0);
    for (int k = -1; k < G.nz + 1; ++k)
        for (int j = -1; j < G.ny + 1; ++j)
            for (int i = -1; i < G.nx + 1; ++i) {
                const long id = G.at(i, j, k);
                const int q = G.at2(i, j);
                auto ddxi = [&](const double* f) { return 0.5 * (f[id + 1] - f[id - 1]); };
                auto ddeta = [&](const double* f) { return 0.5 * (f[id + G.sx] - f[id - G.sx]); };
                auto ddzeta = [&](const double* f) {
                    return 0.5 * (f[id + G.sxy] - f[id - G.sxy]);
                };
                // MetricField::xi_x() = m_xi_x * jac (metrics.hpp:34), on the
                // extruded rows; zeta_z = (area row) * jac
                const double xi_x = Mv.mxx[q] * Mv.jac[q];
                const double xi_y = Mv.mxy[q] * Mv.jac[q];
                const double eta_x = Mv.mex[q] * Mv.jac[q];
                const double eta_y = Mv.mey[q] * Mv.jac[q];
                const double zeta_z = Mv.mzz[q] * Mv.jac[q];
                auto gradx = [&](const double* f) { return xi_x * ddxi(f) + eta_x * ddeta(f); };
                auto grady = [&](const double* f) { return xi_y * ddxi(f) + eta_y * ddeta(f); };
                auto gradz = [&](const double* f) { return zeta_z * ddzeta(f); };

                const double ux = gradx(u), uy = grady(u), uz = gradz(u);
                const double vx = gradx(v), vy = grady(v), vz = gradz(v);
                const double wx = gradx(w), wy = grady(w), wz = gradz(w);
                const double Tx = gradx(Tf), Ty = grady(Tf), Tz = gradz(Tf);

                SpeciesArray Y{}, X{}, gx{}, gy{}, gz{}, hs{};
                for (int s = 0; s < ns; ++s) {
                    const double* Xf = Xs.data() + size_t(s) * G.plane;
                    Y[s] = field(Y0 + s)[id];
                    X[s] = Xf[id];
                    gx[s] = gradx(Xf);
                    gy[s] = grady(Xf);
                    gz[s] = gradz(Xf);
                    hs[s] = ignis::thermo::h_species(Tf[id], s, mix);
                }
                ignis::ThermoState st;
                st.rho = rho[id];
                st.T = Tf[id];
                st.Y = Y;
                st.X = X;
                ignis::transport(st, mix);

                const double div = (ux + vy) + wz;
                const double txx = st.mu * (2.0 * ux - (2.0 / 3.0) * div);
                const double tyy = st.mu * (2.0 * vy - (2.0 / 3.0) * div);
                const double tzz = st.mu * (2.0 * wz - (2.0 / 3.0) * div);
                const double txy = st.mu * (uy + vx);
                const double txz = st.mu * (uz + wx);
                const double tyz = st.mu * (vz + wy);

                const double wbar = ignis::thermo::mean_molar_mass(Y, mix);
                double ucx = 0.0, ucy = 0.0, ucz = 0.0;
                for (int s = 0; s < ns; ++s) {
                    ucx += (mix.species[s].W / wbar) * st.D[s] * gx[s];
                    ucy += (mix.species[s].W / wbar) * st.D[s] * gy[s];
                    ucz += (mix.species[s].W / wbar) * st.D[s] * gz[s];
                }
                double ex = st.lambda * Tx, ey = st.lambda * Ty, ez = st.lambda * Tz;
                std::vector<double> Fd(nc), Gd(nc), Hd(nc);
                for (int s = 0; s < ns; ++s) {
                    const double a = (mix.species[s].W / wbar) * st.D[s];
                    const double jsx = st.rho * (a * gx[s] - Y[s] * ucx);
                    const double jsy = st.rho * (a * gy[s] - Y[s] * ucy);
                    const double jsz = st.rho * (a * gz[s] - Y[s] * ucz);
                    ex += jsx * hs[s];
                    ey += jsy * hs[s];
                    ez += jsz * hs[s];
                    Fd[s] = jsx;
                    Gd[s] = jsy;
                    Hd[s] = jsz;
                }
                const int mx = ns, my = ns + 1, mz = ns + 2, en = ns + 3;
                Fd[mx] = txx;
                Fd[my] = txy;
                Fd[mz] = txz;
                Fd[en] = ((u[id] * txx + v[id] * txy) + w[id] * txz) + ex;
                Gd[mx] = txy;
                Gd[my] = tyy;
                Gd[mz] = tyz;
                Gd[en] = ((u[id] * txy + v[id] * tyy) + w[id] * tyz) + ey;
                Hd[mx] = txz;
                Hd[my] = tyz;
                Hd[mz] = tzz;
                Hd[en] = ((u[id] * txz + v[id] * tyz) + w[id] * tzz) + ez;
                for (int cc = 0; cc < nc; ++cc) {
                    const size_t o = size_t(cc) * G.plane + id;
                    Fv[o] = Mv.mxx[q] * Fd[cc] + Mv.mxy[q] * Gd[cc];
                    Gv[o] = Mv.mex[q] * Fd[cc] + Mv.mey[q] * Gd[cc];
                    Hv[o] = Mv.mzz[q] * Hd[cc];
                }
            }

    for (int cc = 0; cc < nc; ++cc) {
        const double* F = Fv.data() + size_t(cc) * G.plane;
        const double* Gq = Gv.data() + size_t(cc) * G.plane;
        const double* H = Hv.data() + size_t(cc) * G.plane;
        for (int k = 0; k < G.nz; ++k)
            for (int j = 0; j < G.ny; ++j)
                for (int i = 0; i < G.nx; ++i) {
                    const long id = G.at(i, j, k);
                    const double dVx = 0.5 * (F[id + 1] - F[id - 1]);
                    const double dVy = 0.5 * (Gq[id + G.sx] - Gq[id - G.sx]);
                    const double dVz = 0.5 * (H[id + G.sxy] - H[id - G.sxy]);
                    dv[long(cc) * G.plane + id] = (dVx + dVy) + dVz;
                }
    }
}

}  // namespace ref3d
