// kernels3d.cuh — stage kernels of the 3D extension (BASELINE configs[1],
// TGV 256^3).  The reference is 2D-only; these kernels extend each 2D kernel
// (kernels.cuh) by the z terms on EXTRUDED meshes (2D reference metrics x
// uniform z, flux3.cuh), appended after the reference's 2D expressions so the
// z-extrusion cross-check reproduces the 2D oracle bit for bit.  Boundary
// conditions: the reference's 2D edge rules on x / y; z periodic, no-slip
// walls or outflow.
#pragma once

#include "faces3d.cuh"
#include "flux3.cuh"
#include "kernels_common.cuh"

namespace ign {

// ---------------------------------------------------------------- ghost fill
// fill_ghosts (boundary.hpp:136-258) on every interior z plane: x edges over
// rows 0..ny-1, then y edges over -g..nx+g-1 (corners take the y rule), with
// the reference's 2D edge rules extended by w (walls mirror it, inflow sets
// w = 0); then z (periodic) over whole (x, y) planes unless the z ghost planes
// come from the neighbouring z-slabs.
template <int NS, int TM>
__device__ int bc3_prim_at(const KParams& P, const double* Ut, int i, int j, int k,
                           Prim3<NS>& pt, double& rs) {
    const long long id = pidx3(P, i, j, k);
    const double J = P.jac[(j + P.g) * P.sx + (i + P.g)];
    double U[NS + 4];
#pragma unroll
    for (int c = 0; c < NS + 4; ++c) U[c] = Ut[c * P.plane + id] * J;
    return primitives_from_conservative3<NS, true, TM>(U, P.mix, 300.0, pt, &rs);
}

template <int NS, int TM>
__device__ void bc3_store(const KParams& P, double* Ut, const Prim3<NS>& pt, int i, int j, int k) {
    double U[NS + 4];
    conservative_from_primitives3<NS, TM>(pt, P.mix, U);
    const long long id = pidx3(P, i, j, k);
    const double invJ = 1.0 / P.jac[(j + P.g) * P.sx + (i + P.g)];
#pragma unroll
    for (int c = 0; c < NS + 4; ++c) Ut[c * P.plane + id] = U[c] * invJ;
}

template <int NS>
__device__ void bc3_copy_scaled(const KParams& P, double* Ut, int is, int js, int id_, int jd,
                                int k) {
    const long long s = pidx3(P, is, js, k), d = pidx3(P, id_, jd, k);
    const double ratio =
        P.jac[(js + P.g) * P.sx + (is + P.g)] / P.jac[(jd + P.g) * P.sx + (id_ + P.g)];
#pragma unroll
    for (int c = 0; c < NS + 4; ++c) Ut[c * P.plane + d] = Ut[c * P.plane + s] * ratio;
}

template <int NS, int TM>
__global__ void __launch_bounds__(128) k_bc3(const __grid_constant__ KParams P, double* Ut,
                                             int pass, int stage, int step) {
    if (failed_before(P.err, step, stage, PH_BC)) return;
    const int g = P.g;
    const int na = pass == 0 ? P.ny : P.nx + 2 * g;        // first transverse index
    const int nb = pass == 2 ? P.ny + 2 * g : P.nz;       // second
    const int a0 = pass == 0 ? 0 : -g, b0 = pass == 2 ? -g : 0;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;  // < 2 (nx+2g)(ny+2g)
    if (tid >= 2 * na * nb) return;
    const int side = tid / (na * nb);
    const int rem = tid - side * na * nb;
    const int a = a0 + rem % na, b = b0 + rem / na;
    const int n = pass == 0 ? P.nx : pass == 1 ? P.ny : P.nz;
    if (pass == 2) {
        // z edges over the whole padded (x, y) plane, after the x / y edges
        // (the reference's corner order: the last-filled edge wins)
        const int type = P.bc_z[side];
        if (type == BC_HALO) return;  // the peer slab's planes
        const int q = (b + g) * P.sx + (a + g);
        if (type == 0 || type == 4) {
            // periodic (boundary.hpp:203-209) or outflow (boundary.hpp:242-249):
            // scaled copies, the ratio J/J = 1 of the z-independent (x, y) metrics
            const double ratio = P.jac[q] / P.jac[q];
            for (int k = 1; k <= g; ++k) {
                const int ks = type == 0 ? (side == 0 ? n - k : k - 1) : (side == 0 ? 0 : n - 1);
                const long long s = pidx3(P, a, b, ks);
                const long long d = pidx3(P, a, b, side == 0 ? -k : n - 1 + k);
#pragma unroll
                for (int c = 0; c < NS + 4; ++c)
                    Ut[c * P.plane + d] = Ut[c * P.plane + s] * ratio;
            }
            return;
        }
        // no-slip walls (boundary.hpp:210-226) with w the wall-normal velocity;
        // keys after every x / y edge key of the whole box, (side, y, x, k) order
        const unsigned long long zkey =
            (unsigned long long)P.nz_glob * 4 * (P.nx + P.ny + 4 * g) * (g + 1) +
            (((unsigned long long)side * (P.ny + 2 * g) + (b + g)) * (P.nx + 2 * g) + (a + g)) *
                (g + 1);
        for (int k = 1; k <= g; ++k) {
            Prim3<NS> pt;
            double rs;
            const int st = bc3_prim_at<NS, TM>(P, Ut, a, b, side == 0 ? k - 1 : n - k, pt, rs);
            if (st) {
                report(P.err, stage, PH_BC, zkey + k, st, step);
                return;
            }
            pt.u = -pt.u;
            pt.v = -pt.v;
            pt.w = -pt.w;
            if (type == 1) {
                const double tg = 2.0 * P.T_wall_z[side] - pt.T;
                pt.T = smax(tg, 0.05 * P.T_wall_z[side]);
            }
            pt.rho = pt.p / (r_specific<NS>(pt.Y, P.mix) * pt.T);
            bc3_store<NS, TM>(P, Ut, pt, a, b, side == 0 ? -k : n - 1 + k);
        }
        return;
    }
    const int edge = 2 * pass + side;  // 0 left, 1 right, 2 bottom, 3 top
    const int type = P.bc_type[edge];
    const int t = a, kz = b;
    auto ij = [&](int e, int& i, int& j) {  // index e along the edge normal
        if (pass) { i = t; j = e; } else { i = e; j = t; }
    };
    // (plane, edge, t, k) order: deterministic, unique per ghost node
    const unsigned long long ekey =
        ((((unsigned long long)(kz + P.j0) * 4 + edge) * (P.nx + P.ny + 4 * g) + (t + g)) *
         (g + 1));
    int gi, gj;
    switch (type) {
    case 0: {  // Periodic (boundary.hpp:203-209)
        for (int k = 1; k <= g; ++k) {
            int si, sj;
            ij(side == 0 ? n - k : k - 1, si, sj);
            ij(side == 0 ? -k : n - 1 + k, gi, gj);
            bc3_copy_scaled<NS>(P, Ut, si, sj, gi, gj, kz);
        }
        break;
    }
    case 1:
    case 2: {  // No-slip walls (boundary.hpp:210-226), w mirrored too
        for (int k = 1; k <= g; ++k) {
            int mi, mj;
            ij(side == 0 ? k - 1 : n - k, mi, mj);
            ij(side == 0 ? -k : n - 1 + k, gi, gj);
            Prim3<NS> pt;
            double rs;
            const int st = bc3_prim_at<NS, TM>(P, Ut, mi, mj, kz, pt, rs);
            if (st) {
                report(P.err, stage, PH_BC, ekey + k, st, step);
                return;
            }
            pt.u = -pt.u;
            pt.v = -pt.v;
            pt.w = -pt.w;
            if (type == 1) {
                const double tg = 2.0 * P.T_wall[edge] - pt.T;
                pt.T = smax(tg, 0.05 * P.T_wall[edge]);
            }
            pt.rho = pt.p / (r_specific<NS>(pt.Y, P.mix) * pt.T);
            bc3_store<NS, TM>(P, Ut, pt, gi, gj, kz);
        }
        break;
    }
    case 3: {  // Inflow (boundary.hpp:227-241): the host-built (x, y) profile, w = 0
        int ii, ji;
        ij(side == 0 ? 0 : n - 1, ii, ji);
        Prim3<NS> inner;
        double rs;
        const int st = bc3_prim_at<NS, TM>(P, Ut, ii, ji, kz, inner, rs);
        if (st) {
            report(P.err, stage, PH_BC, ekey, st, step);
            return;
        }
        const int tlo = pass ? -g : 0;
        const double* prof = P.inflow[edge] + (long long)(t - tlo) * g * (3 + NS);
        for (int k = 1; k <= g; ++k) {
            ij(side == 0 ? -k : n - 1 + k, gi, gj);
            const double* q = prof + (k - 1) * (3 + NS);
            Prim3<NS> pt;
            pt.u = q[0];
            pt.v = q[1];
            pt.w = 0.0;
            pt.T = q[2];
#pragma unroll
            for (int s = 0; s < NS; ++s) pt.Y[s] = q[3 + s];
            pt.p = inner.p;
            pt.rho = pt.p / (r_specific<NS>(pt.Y, P.mix) * pt.T);
            bc3_store<NS, TM>(P, Ut, pt, gi, gj, kz);
        }
        break;
    }
    default: {  // Outflow (boundary.hpp:242-249)
        int ii, ji;
        ij(side == 0 ? 0 : n - 1, ii, ji);
        for (int k = 1; k <= g; ++k) {
            ij(side == 0 ? -k : n - 1 + k, gi, gj);
            bc3_copy_scaled<NS>(P, Ut, ii, ji, gi, gj, kz);
        }
        break;
    }
    }
}

// ---------------------------------------------------------------- primitives
// 2-4 species: 4 CTAs/SM (64 registers, small spill): jet primitives -10%
template <int NS, bool WX, int TM>
__global__ void __launch_bounds__(256, NS <= 4 ? 4 : 1) k_prim3(const __grid_constant__ KParams P,
                                               const double* __restrict__ Ut, int stage,
                                               int step, int k_lo) {
    if (failed_before(P.err, step, stage, PH_PRIM)) return;
    const int id2 = blockIdx.x * blockDim.x + threadIdx.x;  // (x, y) plane index
    if (id2 >= P.sxy) return;
    const long long id = (long long)(blockIdx.y + k_lo) * P.sxy + id2;  // padded k
    const double J = P.jac[id2];
    double U[NS + 4];
#pragma unroll
    for (int c = 0; c < NS + 4; ++c) U[c] = Ut[c * P.plane + id] * J;
    Prim3<NS> pt;
    double rs;
    const int st = primitives_from_conservative3<NS, true, TM>(U, P.mix, PT3(P)[id], pt, &rs);
    if (st) {
        report(P.err, stage, PH_PRIM, (unsigned long long)(id + (long long)P.j0 * P.sxy), st,
               step);
        return;
    }
    PRHO3(P)[id] = pt.rho;
    PU3(P)[id] = pt.u;
    PV3(P)[id] = pt.v;
    PW3(P)[id] = pt.w;
    PP3(P)[id] = pt.p;
    PT3(P)[id] = pt.T;
    PC3(P)[id] = sound_speed_rs<NS, true, TM>(pt.T, pt.Y, rs, P.mix);
#pragma unroll
    for (int s = 0; s < NS; ++s) PY3(P, s)[id] = pt.Y[s];
    if (WX) {
        double X[NS];
        mole_fractions<NS>(pt.Y, P.mix, X);
#pragma unroll
        for (int s = 0; s < NS; ++s) PX3(P, s)[id] = X[s];
    }
}

// ---------------------------------------------------------------- viscous
// compute_viscous (solver.hpp:610-696) with the z gradient, z stresses and
// the zeta flux appended after the reference's 2D terms: the mapped node
// fluxes (Fv, Gv, Hv) of node (i, j, k)
template <int NS, int TM>
__device__ __forceinline__ void visc_node3(const KParams& P, int i, int j, int k,
                                           double* __restrict__ Fo, double* __restrict__ Go,
                                           double* __restrict__ Ho) {
    constexpr int NC = NS + 4;
    const long long id = pidx3(P, i, j, k), id2 = id % P.sxy;
    auto ddxi = [&](const double* f) { return 0.5 * (ldg(f + id + 1) - ldg(f + id - 1)); };
    auto ddeta = [&](const double* f) { return 0.5 * (ldg(f + id + P.sx) - ldg(f + id - P.sx)); };
    auto ddzeta = [&](const double* f) {
        return 0.5 * (ldg(f + id + P.sxy) - ldg(f + id - P.sxy));
    };
    const double vj = ldg(P.vjac + id2);
    const double xi_x = ldg(P.vmxx + id2) * vj;
    const double xi_y = ldg(P.vmxy + id2) * vj;
    const double eta_x = ldg(P.vmex + id2) * vj;
    const double eta_y = ldg(P.vmey + id2) * vj;
    const double zeta_z = ldg(P.vmzz + id2) * vj;
    auto gradx = [&](const double* f) { return xi_x * ddxi(f) + eta_x * ddeta(f); };
    auto grady = [&](const double* f) { return xi_y * ddxi(f) + eta_y * ddeta(f); };
    auto gradz = [&](const double* f) { return zeta_z * ddzeta(f); };
    const double ux = gradx(PU3(P)), uy = grady(PU3(P)), uz = gradz(PU3(P));
    const double vx = gradx(PV3(P)), vy = grady(PV3(P)), vz = gradz(PV3(P));
    const double wx_ = gradx(PW3(P)), wy_ = grady(PW3(P)), wz = gradz(PW3(P));
    const double Tx = gradx(PT3(P)), Ty = grady(PT3(P)), Tz = gradz(PT3(P));
    const double T = ldg(PT3(P) + id), rho = ldg(PRHO3(P) + id);
    double Y[NS], X[NS], gx[NS], gy[NS], gz[NS], hs[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        Y[s] = ldg(PY3(P, s) + id);
        X[s] = ldg(PX3(P, s) + id);
        gx[s] = gradx(PX3(P, s));
        gy[s] = grady(PX3(P, s));
        gz[s] = gradz(PX3(P, s));
        hs[s] = h_species<TM>(T, P.mix.sp[s], P.mix.R);
    }
    double mu, lambda, D, cp;
    transport<NS, TM>(rho, T, Y, X, P.mix, mu, lambda, D, cp);
    const double div = (ux + vy) + wz;
    const double txx = mu * (2.0 * ux - (2.0 / 3.0) * div);
    const double tyy = mu * (2.0 * vy - (2.0 / 3.0) * div);
    const double tzz = mu * (2.0 * wz - (2.0 / 3.0) * div);
    const double txy = mu * (uy + vx);
    const double txz = mu * (uz + wx_);
    const double tyz = mu * (vz + wy_);
    const double wbar = mean_molar_mass<NS>(Y, P.mix);
    double ucx = 0.0, ucy = 0.0, ucz = 0.0;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        ucx += (P.mix.sp[s].W / wbar) * D * gx[s];
        ucy += (P.mix.sp[s].W / wbar) * D * gy[s];
        ucz += (P.mix.sp[s].W / wbar) * D * gz[s];
    }
    double ex = lambda * Tx, ey = lambda * Ty, ez = lambda * Tz;
    double Fd[NC], Gd[NC], Hd[NC];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        const double jsx = rho * ((P.mix.sp[s].W / wbar) * D * gx[s] - Y[s] * ucx);
        const double jsy = rho * ((P.mix.sp[s].W / wbar) * D * gy[s] - Y[s] * ucy);
        const double jsz = rho * ((P.mix.sp[s].W / wbar) * D * gz[s] - Y[s] * ucz);
        ex += jsx * hs[s];
        ey += jsy * hs[s];
        ez += jsz * hs[s];
        Fd[s] = jsx;
        Gd[s] = jsy;
        Hd[s] = jsz;
    }
    const double u = ldg(PU3(P) + id), v = ldg(PV3(P) + id), w = ldg(PW3(P) + id);
    Fd[NS] = txx;
    Fd[NS + 1] = txy;
    Fd[NS + 2] = txz;
    Fd[NS + 3] = ((u * txx + v * txy) + w * txz) + ex;
    Gd[NS] = txy;
    Gd[NS + 1] = tyy;
    Gd[NS + 2] = tyz;
    Gd[NS + 3] = ((u * txy + v * tyy) + w * tyz) + ey;
    Hd[NS] = txz;
    Hd[NS + 1] = tyz;
    Hd[NS + 2] = tzz;
    Hd[NS + 3] = ((u * txz + v * tyz) + w * tzz) + ez;
    const double a = ldg(P.vmxx + id2), b = ldg(P.vmxy + id2);
    const double c2 = ldg(P.vmex + id2), d = ldg(P.vmey + id2), e = ldg(P.vmzz + id2);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        Fo[c] = a * Fd[c] + b * Gd[c];
        Go[c] = c2 * Fd[c] + d * Gd[c];
        Ho[c] = e * Hd[c];
    }
}

// 2-4 species: 6 CTAs/SM (<= 85 registers, a small spill) hide more of the
// stencil loads' latency (jet visc3 -6.5%); the gamma-gas keeps 122 registers
template <int NS, int TM>
#ifndef IGN_VISC1_MINB
#define IGN_VISC1_MINB 8  // one species: 8 CTAs/SM (64 registers, small spill) -4% viscous
#endif
__global__ void __launch_bounds__(128, (NS > 1 && NS <= 4) ? 6 : NS == 1 ? IGN_VISC1_MINB : 1) k_visc3(const __grid_constant__ KParams P, int stage,
                                               int step) {
    constexpr int NC = NS + 4;
    if (failed_before(P.err, step, stage, PH_RHS)) return;
    const long long wx = P.nx + 2, wy = P.ny + 2;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= wx * wy * (P.nz + 2)) return;
    const int i = (int)(t % wx) - 1, j = (int)((t / wx) % wy) - 1, k = (int)(t / (wx * wy)) - 1;
    const long long id = pidx3(P, i, j, k);
    double F[NC], G[NC], H[NC];
    visc_node3<NS, TM>(P, i, j, k, F, G, H);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        P.Fv[c * P.plane + id] = F[c];
        P.Gv[c * P.plane + id] = G[c];
        P.Hv[c * P.plane + id] = H[c];
    }
}

// ---------------------------------------------------------------- LODI outflow
// lodi_outflow_override (solver.hpp:717-788) on the right-edge column of
// plane k, with the second transverse wave (w) appended: L4 = out dw/dn
template <int NS>
__device__ void lodi_dfx3(const KParams& P, int j, int kz, double* dF) {
    const int i = P.nx - 1;
    const long long id = pidx3(P, i, j, kz), i1 = id - 1, i2 = id - 2;
    const int q = (j + P.g) * P.sx + (i + P.g);
    const double vj = ldg(P.vjac + q);
    const double xi_x = ldg(P.vmxx + q) * vj;
    const double xi_y = ldg(P.vmxy + q) * vj;
    const double sn = ghypot(xi_x, xi_y);
    const double n1 = xi_x / sn, n2 = xi_y / sn;
    auto ddn = [&](const double* f) {
        return sn * 0.5 * (3.0 * ldg(f + id) - 4.0 * ldg(f + i1) + ldg(f + i2));
    };
    const double rr = ldg(PRHO3(P) + id), cc0 = ldg(PC3(P) + id), pp = ldg(PP3(P) + id);
    const double uu = ldg(PU3(P) + id), vv = ldg(PV3(P) + id), ww = ldg(PW3(P) + id);
    const double un = n1 * uu + n2 * vv;
    const double M = smin(fabs(un) / cc0, 0.99);
    const double drdn = ddn(PRHO3(P));
    const double dpdn = ddn(PP3(P));
    const double dundn = n1 * ddn(PU3(P)) + n2 * ddn(PV3(P));
    const double dutdn = -n2 * ddn(PU3(P)) + n1 * ddn(PV3(P));
    const double dwdn = ddn(PW3(P));
    const double K = P.sigma_out_right * cc0 * (1.0 - M * M) / P.lx;
    const double L1 = K * (pp - P.p_target_right);
    const double out = un > 0.0 ? un : 0.0;
    const double L2 = out * (cc0 * cc0 * drdn - dpdn);
    const double L3 = out * dutdn;
    const double L4 = out * dwdn;
    const double L5 = (un + cc0) * (dpdn + rr * cc0 * dundn);
    const double drdt = -(L2 + 0.5 * (L5 + L1)) / (cc0 * cc0);
    const double dundt = -(L5 - L1) / (2.0 * rr * cc0);
    const double dutdt = -L3;
    const double dwdt = -L4;
    const double dpdt = -0.5 * (L5 + L1);
    double Y[NS], dYdt[NS];
    double sumRdY = 0.0;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        Y[s] = ldg(PY3(P, s) + id);
        dYdt[s] = -out * ddn(PY3(P, s));
        sumRdY += divW(P.mix.sp[s], P.mix.R) * dYdt[s];
    }
    const double rbar = r_specific<NS>(Y, P.mix);
    const double Tt = ldg(PT3(P) + id);
    const double dTdt = Tt * (dpdt / pp - drdt / rr - sumRdY / rbar);
    const double dudt = n1 * dundt - n2 * dutdt;
    const double dvdt = n2 * dundt + n1 * dutdt;
    const double k = 0.5 * ((uu * uu + vv * vv) + ww * ww);
    const double e = e_mass_rs<NS>(Tt, Y, rbar, P.mix);
    const double cv = cp_mass<NS>(Tt, Y, P.mix) - rbar;
    double sum_es_dY = 0.0;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        const double esn = h_species(Tt, P.mix.sp[s], P.mix.R) - divW(P.mix.sp[s], P.mix.R) * Tt;
        sum_es_dY += esn * dYdt[s];
    }
    double dU[NS + 4];
#pragma unroll
    for (int s = 0; s < NS; ++s) dU[s] = Y[s] * drdt + rr * dYdt[s];
    dU[NS] = uu * drdt + rr * dudt;
    dU[NS + 1] = vv * drdt + rr * dvdt;
    dU[NS + 2] = ww * drdt + rr * dwdt;
    dU[NS + 3] = (e + k) * drdt + rr * cv * dTdt + rr * sum_es_dY +
                 rr * ((uu * dudt + vv * dvdt) + ww * dwdt);
    const double invJ = 1.0 / ldg(P.jac + q);
#pragma unroll
    for (int c = 0; c < NS + 4; ++c) dF[c] = -dU[c] * invJ;
}

// ---------------------------------------------------------------- assemble + update
// laser_power out of line: the common (laser-free) update stays small
static __device__ __noinline__ double laser_cold(double x, double y, double z, double t,
                                                 const DLaser& p) {
    return laser_power3(x, y, z, t, p);
}

// The rest of the update of interior node (i, j, k) once its flux
// differences r are summed: compute_rhs's source terms and finite check
// (solver.hpp:422-439), then the RK3 blend with post_stage's clip / validate
// (solver.hpp:304-332, state.hpp:94-121) — or r itself for MODE 0.
template <int NS, int MODE>
__device__ __forceinline__ void finish_node3(const KParams& P, const double* __restrict__ U0,
                                             const double* __restrict__ Ucur,
                                             double* __restrict__ Uout, long long id, int i, int j,
                                             int k, double (&r)[NS + 4], double dt, double w,
                                             double t_stage, int stage, int step, double& clip) {
    constexpr int NC = NS + 4;
    const double J = ldg(P.jac + id % P.sxy);
    const double invJ = 1.0 / J;
    if (P.mech.present) {
        double Y[NS], wdot[NS];
#pragma unroll
        for (int s = 0; s < NS; ++s) Y[s] = ldg(PY3(P, s) + id);
        source_terms<NS>(ldg(PRHO3(P) + id), ldg(PT3(P) + id), Y, P.mix, P.mech, wdot);
#pragma unroll
        for (int s = 0; s < NS; ++s) r[s] += wdot[s] * invJ;
    }
    // laser_power (laser.hpp:88-91) of the node's (x, y) — the
    // reference's 2D kernel on every plane — or the 3D point kernel
    // (laser_power3, zmode 1) at the node's z
    if (P.laser.on) {
        const int q = (j + P.g) * P.sx + (i + P.g);
        const double z = P.zc0 + ((k + P.j0) + 0.5) * P.dz;
        r[NS + 3] +=
            laser_cold(ldg(P.xc + q), ldg(P.yc + q), z, t_stage, P.laser) * invJ;
    }
    const unsigned long long cell =
        ((unsigned long long)(k + P.j0) * P.ny + j) * P.nx + i;
    bool bad = false;
#pragma unroll
    for (int c = 0; c < NC; ++c) bad |= !isfinite(r[c]);
    if (bad) {
        report(P.err, stage, PH_RHS, cell, 0, step);
    } else if (MODE == 0) {
#pragma unroll
        for (int c = 0; c < NC; ++c) Uout[c * P.plane + id] = r[c];
    } else {
        double o[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            const double b = U0[c * P.plane + id];
            if (MODE == 1) o[c] = b + dt * r[c];
            else o[c] = b + w * ((Ucur[c * P.plane + id] - b) + dt * r[c]);
        }
        double rsum = 0.0;
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            if (o[s] < 0.0) {
                clip = smax(clip, -o[s] * J);
                o[s] = 0.0;
            }
            rsum += o[s];
        }
        bool fin = true;
#pragma unroll
        for (int c = 0; c < NC; ++c) fin &= isfinite(o[c]);
        if (!(rsum > 0.0)) report(P.err, stage, PH_POST, cell * 2, 0, step);
        else if (!fin) report(P.err, stage, PH_POST, cell * 2 + 1, 0, step);
#pragma unroll
        for (int c = 0; c < NC; ++c) Uout[c * P.plane + id] = o[c];
    }
}

// EDGE = false: every padded node except, when LODI is on, the right-edge
// column; EDGE = true: that column alone (grid over its (j, k)), with the LODI
// x-flux difference — so the LODI code never enters the bulk update.
// Bulk update, 1-4 species: 3 CTAs/SM (<= 80 registers; the finish_node3
// factoring had let it grow to 104, 2 CTAs/SM, jet update +17%)
template <int NS, int MODE, bool EDGE>
__global__ void __launch_bounds__(256, (NS <= 4 && !EDGE) ? 3 : 1) k_assemble3(const __grid_constant__ KParams P,
                                                   const double* __restrict__ U0,
                                                   const double* __restrict__ Ucur,
                                                   double* __restrict__ Uout, double dt,
                                                   double w, double t_stage, int stage,
                                                   int step, int clip_slot) {
    constexpr int NC = NS + 4;
    __shared__ unsigned long long s_clip;
    if (threadIdx.x == 0) s_clip = 0ull;
    __syncthreads();
    const bool dead = failed_before(P.err, step, stage, PH_RHS);
    long long id;
    bool in_range;
    if (EDGE) {
        const int t = blockIdx.x * blockDim.x + threadIdx.x;  // (j, k) of the column
        in_range = t < P.ny * P.nz;
        id = in_range ? pidx3(P, P.nx - 1, t % P.ny, t / P.ny) : 0;
    } else {
        id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
        in_range = id < P.plane;
    }
    double clip = 0.0;
    if (!dead && in_range) {
        const int ip = (int)(id % P.sx), jp = (int)((id / P.sx) % (P.ny + 2 * P.g));
        const int kp = (int)(id / P.sxy);
        const int i = ip - P.g, j = jp - P.g, k = kp - P.g;
        const bool interior = i >= 0 && i < P.nx && j >= 0 && j < P.ny && k >= 0 && k < P.nz;
        const bool lodi = P.lodi && i == P.nx - 1;
        if (!EDGE && interior && lodi) {
            // the right-edge column is the EDGE launch's
        } else if (!interior) {
            if (MODE != 0) {
#pragma unroll
                for (int c = 0; c < NC; ++c) Uout[c * P.plane + id] = Ucur[c * P.plane + id];
            }
        } else {
            const long long fxp = (long long)(P.nx + 1) * P.ny * P.nz;
            const long long fyp = (long long)P.nx * (P.ny + 1) * P.nz;
            const long long fzp = (long long)P.nx * P.ny * (P.nz + 1);
            const long long fx = ((long long)k * P.ny + j) * (P.nx + 1) + i;
            const long long fy = ((long long)k * (P.ny + 1) + j) * P.nx + i;
            const long long fz = ((long long)k * P.ny + j) * P.nx + i;
            double r[NC];
            double dFl[EDGE ? NC : 1];
            if (EDGE) lodi_dfx3<NS>(P, j, k, dFl);
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const double dF = EDGE ? dFl[EDGE ? c : 0] : P.Fx[c * fxp + fx + 1] - P.Fx[c * fxp + fx];
                const double dG = P.Gy[c * fyp + fy + P.nx] - P.Gy[c * fyp + fy];
                const double dH = P.Hz[c * fzp + fz + (long long)P.nx * P.ny] - P.Hz[c * fzp + fz];
                r[c] = -((dF + dG) + dH);
            }
            if (P.viscous) {
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    const double* Fv = P.Fv + c * P.plane;
                    const double* Gv = P.Gv + c * P.plane;
                    const double* Hv = P.Hv + c * P.plane;
                    const double dVx = 0.5 * (Fv[id + 1] - Fv[id - 1]);
                    const double dVy = 0.5 * (Gv[id + P.sx] - Gv[id - P.sx]);
                    const double dVz = 0.5 * (Hv[id + P.sxy] - Hv[id - P.sxy]);
                    r[c] += (dVx + dVy) + dVz;
                }
            }
            finish_node3<NS, MODE>(P, U0, Ucur, Uout, id, i, j, k, r, dt, w, t_stage, stage,
                                   step, clip);
        }
    }
    if (MODE != 0) {
        if (clip > 0.0) atomicMax(&s_clip, (unsigned long long)__double_as_longlong(clip));
        __syncthreads();
        if (threadIdx.x == 0 && s_clip) atomicMax(&P.red[2 + clip_slot], s_clip);
    }
}

// ---------------------------------------------------------------- stable dt
template <int NS>
__global__ void __launch_bounds__(256) k_dt3(const __grid_constant__ KParams P) {
    __shared__ unsigned long long s_lam, s_chem;
    if (threadIdx.x == 0) {
        s_lam = 0ull;
        s_chem = 0x7ff0000000000000ull;
    }
    __syncthreads();
    const int t = blockIdx.x * blockDim.x + threadIdx.x;  // (i, j) of plane k = blockIdx.y
    double lam_loc = 0.0, chem_loc = __longlong_as_double(0x7ff0000000000000ll);
    if (t < P.nx * P.ny) {
        const int i = t % P.nx, j = t / P.nx, k = blockIdx.y;
        const long long id = pidx3(P, i, j, k);
        const int id2 = (j + P.g) * P.sx + (i + P.g);
        const double J = ldg(P.jac + id2);
        const double mxx = ldg(P.mxx + id2), mxy = ldg(P.mxy + id2);
        const double mex = ldg(P.mex + id2), mey = ldg(P.mey + id2), mzz = ldg(P.mzz + id2);
        const double sx = ghypot(mxx, mxy), sy = ghypot(mex, mey), sz = fabs(mzz);
        const double u = ldg(PU3(P) + id), v = ldg(PV3(P) + id), w = ldg(PW3(P) + id);
        const double c = ldg(PC3(P) + id);
        const double ux = mxx * u + mxy * v, uy = mex * u + mey * v, uz = mzz * w;
        double lam = ((fabs(ux) + c * sx + fabs(uy) + c * sy) + fabs(uz) + c * sz) * J;
        double Y[NS];
#pragma unroll
        for (int s = 0; s < NS; ++s) Y[s] = ldg(PY3(P, s) + id);
        const double rho = ldg(PRHO3(P) + id), T = ldg(PT3(P) + id);
        if (P.viscous) {
            double X[NS];
            mole_fractions<NS>(Y, P.mix, X);
            double mu, lambda, D, cp;
            transport<NS>(rho, T, Y, X, P.mix, mu, lambda, D, cp);
            const double nu = smax(2.0 * mu / rho, smax(lambda / (rho * cp), D));
            lam += 2.0 * nu * ((sx * sx + sy * sy) + sz * sz) * J * J;
        }
        lam_loc = smax(0.0, lam);
        if (P.mech.present && P.chem_dt_limit) {
            double wdot[NS];
            source_terms<NS>(rho, T, Y, P.mix, P.mech, wdot);
#pragma unroll
            for (int s = 0; s < NS; ++s) {
                const double wv = fabs(wdot[s]);
                if (wv > 0.0) chem_loc = smin(chem_loc, P.chem_dt_factor * (rho * smax(Y[s], 1e-3)) / wv);
            }
        }
    }
    // warp max / min first (on the bit patterns: lam > 0 and chem > 0, where
    // the unsigned order is the numeric one; NaN lam is skipped as the
    // reference's std::max skips it), then one shared atomic per warp
    unsigned long long lb = lam_loc > 0.0 ? (unsigned long long)__double_as_longlong(lam_loc) : 0ull;
    unsigned long long cb = chem_loc < __longlong_as_double(0x7ff0000000000000ll)
                                ? (unsigned long long)__double_as_longlong(chem_loc)
                                : 0x7ff0000000000000ull;
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long lo = __shfl_xor_sync(0xffffffffu, lb, o);
        const unsigned long long co = __shfl_xor_sync(0xffffffffu, cb, o);
        lb = lo > lb ? lo : lb;
        cb = co < cb ? co : cb;
    }
    if ((threadIdx.x & 31) == 0) {
        if (lb) atomicMax(&s_lam, lb);
        if (cb != 0x7ff0000000000000ull) atomicMin(&s_chem, cb);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (s_lam) atomicMax(&P.red[0], s_lam);
        if (s_chem != 0x7ff0000000000000ull) atomicMin(&P.red[1], s_chem);
    }
}

template <int NS> struct Launch3 {
    static void bc3_launch(const KParams& P, double* Ut, int pass, int stage, int step,
                           unsigned nb, cudaStream_t s) {
        switch (thermo_mode<NS>(P.mix)) {
        case 1: k_bc3<NS, 1><<<nb, 128, 0, s>>>(P, Ut, pass, stage, step); break;
        case 2: k_bc3<NS, 2><<<nb, 128, 0, s>>>(P, Ut, pass, stage, step); break;
        default: k_bc3<NS, 0><<<nb, 128, 0, s>>>(P, Ut, pass, stage, step); break;
        }
    }
    // ypass 0 (before the halo exchange): x then y periodic copies, so the
    // exchanged z planes carry their x/y ghosts; ypass 1: z copies (single
    // domain) — with z-slabs the z ghost planes came from the peers instead
    static int bc(const KParams& P, double* Ut, int ypass, int stage, int step, cudaStream_t s) {
        const int g = P.g;
        if (ypass == 0) {
            const int n0 = 2 * P.ny * P.nz;
            bc3_launch(P, Ut, 0, stage, step, (unsigned)((n0 + 127) / 128), s);
            const int n1 = 2 * (P.nx + 2 * g) * P.nz;
            bc3_launch(P, Ut, 1, stage, step, (unsigned)((n1 + 127) / 128), s);
            return 2;
        }
        if (P.bc_z[0] == BC_HALO && P.bc_z[1] == BC_HALO) return 0;
        const int n2 = 2 * (P.nx + 2 * g) * (P.ny + 2 * g);
        bc3_launch(P, Ut, 2, stage, step, (unsigned)((n2 + 127) / 128), s);
        return 1;
    }
    // padded z planes [k_lo, k_hi)
    static int prim_planes(const KParams& P, const double* Ut, int stage, int step,
                           cudaStream_t s, int k_lo, int k_hi) {
        if (k_hi <= k_lo) return 0;
        const dim3 nb((unsigned)((P.sxy + 255) / 256), (unsigned)(k_hi - k_lo));
        const int tm = thermo_mode<NS>(P.mix);
        if (P.viscous) {
            if (tm == 1) k_prim3<NS, true, 1><<<nb, 256, 0, s>>>(P, Ut, stage, step, k_lo);
            else if (tm == 2) k_prim3<NS, true, 2><<<nb, 256, 0, s>>>(P, Ut, stage, step, k_lo);
            else k_prim3<NS, true, 0><<<nb, 256, 0, s>>>(P, Ut, stage, step, k_lo);
        } else {
            if (tm == 1) k_prim3<NS, false, 1><<<nb, 256, 0, s>>>(P, Ut, stage, step, k_lo);
            else if (tm == 2) k_prim3<NS, false, 2><<<nb, 256, 0, s>>>(P, Ut, stage, step, k_lo);
            else k_prim3<NS, false, 0><<<nb, 256, 0, s>>>(P, Ut, stage, step, k_lo);
        }
        return 1;
    }
    // part (KernelSet): 0 the padded box, 1 this slab's own planes, 2 its ghost planes
    static int prim(const KParams& P, const double* Ut, int stage, int step, cudaStream_t s,
                    int part) {
        const int g = P.g, K = P.nz + 2 * g;
        if (part == 1) return prim_planes(P, Ut, stage, step, s, g, K - g);
        if (part == 2)
            return prim_planes(P, Ut, stage, step, s, 0, g) +
                   prim_planes(P, Ut, stage, step, s, K - g, K);
        return prim_planes(P, Ut, stage, step, s, 0, K);
    }
    // part: 0 every face; 1 x, y faces + the z faces whose stencils lie in
    // owned planes; 2 the remaining z faces (they read the halo planes)
    template <bool TENO, bool CHAR>
    static int faces_t(const KParams& P, const double* Ut, int stage, int step, cudaStream_t s,
                       int part) {
        constexpr int H = TENO ? 3 : 2;
        const int lo = H < P.nz + 1 ? H : P.nz + 1;
        const int hi = P.nz - H + 1 > lo ? P.nz - H + 1 : lo;
        int n = 0;
        if (part != 2) {
            n += launch_faces3d<NS, 0, TENO, CHAR>(P, Ut, stage, step, s);
            n += launch_faces3d<NS, 1, TENO, CHAR>(P, Ut, stage, step, s);
        }
        if (part == 0) return n + launch_faces3d<NS, 2, TENO, CHAR>(P, Ut, stage, step, s);
        if (part == 1) return n + launch_faces3d<NS, 2, TENO, CHAR>(P, Ut, stage, step, s, lo, hi);
        n += launch_faces3d<NS, 2, TENO, CHAR>(P, Ut, stage, step, s, 0, lo);
        return n + launch_faces3d<NS, 2, TENO, CHAR>(P, Ut, stage, step, s, hi, P.nz + 1);
    }
    static int faces(const KParams& P, int teno, int chr, const double* Ut, int stage, int step,
                     cudaStream_t s, int part) {
        if (teno && chr) return faces_t<true, true>(P, Ut, stage, step, s, part);
        if (teno) return faces_t<true, false>(P, Ut, stage, step, s, part);
        if (chr) return faces_t<false, true>(P, Ut, stage, step, s, part);
        return faces_t<false, false>(P, Ut, stage, step, s, part);
    }
    static int visc(const KParams& P, int stage, int step, cudaStream_t s) {
        const long long n = (long long)(P.nx + 2) * (P.ny + 2) * (P.nz + 2);
        const unsigned nb = (unsigned)((n + 127) / 128);
        switch (thermo_mode<NS>(P.mix)) {
        case 1: k_visc3<NS, 1><<<nb, 128, 0, s>>>(P, stage, step); break;
        case 2: k_visc3<NS, 2><<<nb, 128, 0, s>>>(P, stage, step); break;
        default: k_visc3<NS, 0><<<nb, 128, 0, s>>>(P, stage, step); break;
        }
        return 1;
    }
    template <bool EDGE>
    static void assemble_t(const KParams& P, int mode, const double* U0, const double* Ucur,
                           double* Uout, double dt, double w, double t_stage, int stage,
                           int step, int clip_slot, unsigned nb, cudaStream_t s) {
        if (mode == 0)
            k_assemble3<NS, 0, EDGE><<<nb, 256, 0, s>>>(P, U0, Ucur, Uout, dt, w, t_stage, stage,
                                                        step, clip_slot);
        else if (mode == 1)
            k_assemble3<NS, 1, EDGE><<<nb, 256, 0, s>>>(P, U0, Ucur, Uout, dt, w, t_stage, stage,
                                                        step, clip_slot);
        else
            k_assemble3<NS, 2, EDGE><<<nb, 256, 0, s>>>(P, U0, Ucur, Uout, dt, w, t_stage, stage,
                                                        step, clip_slot);
    }
    static int assemble(const KParams& P, int mode, const double* U0, const double* Ucur,
                        double* Uout, double dt, double w, double t_stage, int stage, int step,
                        int clip_slot, cudaStream_t s) {
        assemble_t<false>(P, mode, U0, Ucur, Uout, dt, w, t_stage, stage, step, clip_slot,
                          (unsigned)((P.plane + 255) / 256), s);
        if (!P.lodi) return 1;
        assemble_t<true>(P, mode, U0, Ucur, Uout, dt, w, t_stage, stage, step, clip_slot,
                         (unsigned)((P.ny * P.nz + 255) / 256), s);
        return 2;
    }
    static int dt(const KParams& P, cudaStream_t s) {
        const dim3 grid((unsigned)((P.nx * P.ny + 255) / 256), P.nz);
        k_dt3<NS><<<grid, 256, 0, s>>>(P);
        return 1;
    }
    static KernelSet make() { return KernelSet{&bc, &prim, &faces, &visc, &assemble, &dt}; }
};

}  // namespace ign
