// kernels.cuh — the sm_100a kernels of one RK stage (FP64, -fmad=false).
//
// Data layout in HBM: structure-of-arrays, one padded plane of
// (nx+2g)*(ny+2g) doubles per field, i fastest — the reference's Field layout
// (field.hpp:45-47) so host<->device transfers are single copies.  Face fluxes
// live in their own face-indexed planes (x: (nx+1) x ny, y: nx x (ny+1)) so
// each face is evaluated exactly once.
//
// Per stage the launch sequence is
//   k_bc_x, k_bc_y        ghost fill            (boundary.hpp:136-258)
//   k_prim                primitive cache       (solver.hpp:148-177)
//   k_faces<x>, k_faces<y> inviscid face fluxes (solver.hpp:441-579)
//   k_visc                viscous node fluxes   (solver.hpp:588-696)
//   k_assemble            RHS assembly + LODI + sources + RK update + clip/
//                         validate              (solver.hpp:185-232, 717-849)
// and k_dt reduces the CFL/chemistry limit (solver.hpp:240-299).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "faces.cuh"
#include "flux.cuh"
#include "kernels_common.cuh"
#include "physics.cuh"

namespace ign {

// ---------------------------------------------------------------- ghost fill
// fill_ghosts (boundary.hpp:136-258).  One thread per (edge, t, ghost layer
// k) (walls: per (edge, t), the reference's k = 1..g loop).  x edges cover rows
// 0..ny-1 (launch 1), y edges
// the full padded range -g..nx+g-1 (launch 2), so corners take the y rule.
template <int NS, int TM>
__device__ int bc_prim_at(const KParams& P, const double* Ut, int i, int j, Prim<NS>& pt,
                          double& rs) {
    const long long id = pidx(P, i, j);
    const double J = P.jac[id];
    double U[NS + 3];
#pragma unroll
    for (int c = 0; c < NS + 3; ++c) U[c] = Ut[c * P.plane + id] * J;
    return primitives_from_conservative<NS, true, TM>(U, P.mix, 300.0, pt, &rs);
}

template <int NS, int TM>
__device__ void bc_store(const KParams& P, double* Ut, const Prim<NS>& pt, int i, int j) {
    double U[NS + 3];
    conservative_from_primitives<NS, TM>(pt, P.mix, U);
    const long long id = pidx(P, i, j);
    const double invJ = 1.0 / P.jac[id];
#pragma unroll
    for (int c = 0; c < NS + 3; ++c) Ut[c * P.plane + id] = U[c] * invJ;
}

template <int NS>
__device__ void bc_copy_scaled(const KParams& P, double* Ut, int is, int js, int id_, int jd) {
    const long long s = pidx(P, is, js), d = pidx(P, id_, jd);
    const double ratio = P.jac[s] / P.jac[d];
#pragma unroll
    for (int c = 0; c < NS + 3; ++c) Ut[c * P.plane + d] = Ut[c * P.plane + s] * ratio;
}

template <int NS, int TM>
__global__ void __launch_bounds__(128) k_bc(const __grid_constant__ KParams P, double* Ut,
                                            int ypass, int stage, int step) {
    if (failed_before(P.err, step, stage, PH_BC)) return;
    const int g = P.g, nx = P.nx, ny = P.ny;
    const int tlo = ypass ? -g : 0;
    const int ntr = ypass ? nx + 2 * g : ny;
    // one thread per (edge, t, ghost layer kk): the layers of an edge node are
    // independent (each reads interior nodes only) except on walls, whose
    // layers keep the reference's k order (a failing mirror stops the later
    // layers), and periodic edges of lines shorter than g (the sources are
    // ghosts): layer 1's thread runs the k loop there
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int kk = tid / (2 * ntr) + 1;  // layer-major: a warp's stores are coalesced
    const int rid = tid % (2 * ntr);
    if (kk > g) return;
    const int side = rid / ntr;  // 0: left/bottom, 1: right/top
    const int t = tlo + rid % ntr;
    const int edge = (ypass ? 2 : 0) + side;
    const int type = P.bc_type[edge];
    const int n = ypass ? ny : nx;
    const bool serial = type == 1 || type == 2 || (type == 0 && n < g);
    if (serial && kk != 1) return;
    const int k_lo = serial ? 1 : kk, k_hi = serial ? g : kk;
    // ghost / mirror / wrap / interior index along the edge normal
    auto ij = [&](int a, int& i, int& j) {
        if (ypass) { i = t; j = a; } else { i = a; j = t; }
    };
    // global (edge, t, k) order of the reference's loops (boundary.hpp:254-257)
    const unsigned long long ekey =
        ((unsigned long long)edge * (nx + 2 * g + P.ny_glob) + (ypass ? t - tlo : t + P.j0)) *
        (g + 1);
    int gi, gj;
    switch (type) {
    case BC_HALO:  // internal slab edge: ghost rows arrived from the neighbour
        return;
    case BC_HALO_WRAP: {  // periodic wrap across slabs: Ut_dst = Ut_src * J_src/J_dst
        for (int k = k_lo; k <= k_hi; ++k) {
            ij(side == 0 ? -k : n - 1 + k, gi, gj);
            const double ratio = P.wrap[side][(k - 1) * P.sx + (t + g)];
            const long long d = pidx(P, gi, gj);
#pragma unroll
            for (int c = 0; c < NS + 3; ++c) Ut[c * P.plane + d] = Ut[c * P.plane + d] * ratio;
        }
        return;
    }
    case 0: {  // Periodic (boundary.hpp:203-209)
        for (int k = k_lo; k <= k_hi; ++k) {
            int si, sj;
            ij(side == 0 ? n - k : k - 1, si, sj);
            ij(side == 0 ? -k : n - 1 + k, gi, gj);
            bc_copy_scaled<NS>(P, Ut, si, sj, gi, gj);
        }
        break;
    }
    case 1:
    case 2: {  // No-slip walls (boundary.hpp:210-226)
        for (int k = k_lo; k <= k_hi; ++k) {
            int mi, mj;
            ij(side == 0 ? k - 1 : n - k, mi, mj);
            ij(side == 0 ? -k : n - 1 + k, gi, gj);
            Prim<NS> pt;
            double rs;
            const int st = bc_prim_at<NS, TM>(P, Ut, mi, mj, pt, rs);
            if (st) {
                report(P.err, stage, PH_BC, ekey + k, st, step);
                return;
            }
            pt.u = -pt.u;
            pt.v = -pt.v;
            if (type == 1) {
                const double tg = 2.0 * P.T_wall[edge] - pt.T;
                pt.T = smax(tg, 0.05 * P.T_wall[edge]);
            }
            pt.rho = pt.p / (r_specific<NS>(pt.Y, P.mix) * pt.T);
            bc_store<NS, TM>(P, Ut, pt, gi, gj);
        }
        break;
    }
    case 3: {  // Inflow (boundary.hpp:227-241), profile precomputed on the host
        int ii, ji;
        ij(side == 0 ? 0 : n - 1, ii, ji);
        Prim<NS> inner;
        double rs;
        const int st = bc_prim_at<NS, TM>(P, Ut, ii, ji, inner, rs);
        if (st) {
            report(P.err, stage, PH_BC, ekey, st, step);
            return;
        }
        const double* prof = P.inflow[edge] + (long long)(t - tlo) * g * (3 + NS);
        for (int k = k_lo; k <= k_hi; ++k) {
            ij(side == 0 ? -k : n - 1 + k, gi, gj);
            const double* q = prof + (k - 1) * (3 + NS);
            Prim<NS> pt;
            pt.u = q[0];
            pt.v = q[1];
            pt.T = q[2];
#pragma unroll
            for (int s = 0; s < NS; ++s) pt.Y[s] = q[3 + s];
            pt.p = inner.p;
            pt.rho = pt.p / (r_specific<NS>(pt.Y, P.mix) * pt.T);
            bc_store<NS, TM>(P, Ut, pt, gi, gj);
        }
        break;
    }
    default: {  // Outflow (boundary.hpp:242-249)
        int ii, ji;
        ij(side == 0 ? 0 : n - 1, ii, ji);
        for (int k = k_lo; k <= k_hi; ++k) {
            ij(side == 0 ? -k : n - 1 + k, gi, gj);
            bc_copy_scaled<NS>(P, Ut, ii, ji, gi, gj);
        }
        break;
    }
    }
}

// ---------------------------------------------------------------- primitives
// refresh_primitives (solver.hpp:148-177) over the padded box; the cached T
// is the Newton guess (thermo.hpp:196).
// 2-4 species: 4 CTAs/SM (64 registers, small spill): jet primitives -10%
template <int NS, bool WX, int TM>
__global__ void __launch_bounds__(256, NS <= 4 ? 4 : 1) k_prim(const __grid_constant__ KParams P,
                                              const double* __restrict__ Ut, int stage,
                                              int step, long long id_lo, long long id_hi) {
    if (failed_before(P.err, step, stage, PH_PRIM)) return;
    const long long id = id_lo + (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= id_hi) return;
    const double J = P.jac[id];
    double U[NS + 3];
#pragma unroll
    for (int c = 0; c < NS + 3; ++c) U[c] = Ut[c * P.plane + id] * J;
    Prim<NS> pt;
    double rs;
    const int st = primitives_from_conservative<NS, true, TM>(U, P.mix, PT(P)[id], pt, &rs);
    if (st) {
        report(P.err, stage, PH_PRIM, (unsigned long long)(id + (long long)P.j0 * P.sx), st,
               step);
        return;
    }
    PRHO(P)[id] = pt.rho;
    PU(P)[id] = pt.u;
    PV(P)[id] = pt.v;
    PP(P)[id] = pt.p;
    PT(P)[id] = pt.T;
    PC(P)[id] = sound_speed_rs<NS, true, TM>(pt.T, pt.Y, rs, P.mix);
#pragma unroll
    for (int s = 0; s < NS; ++s) PY(P, s)[id] = pt.Y[s];
    if (WX) {
        double X[NS];
        mole_fractions<NS>(pt.Y, P.mix, X);
#pragma unroll
        for (int s = 0; s < NS; ++s) PX(P, s)[id] = X[s];
    }
}

// Inviscid faces: faces.cuh (k_faces3).

// ---------------------------------------------------------------- viscous
// compute_viscous node fluxes over ring 1 (solver.hpp:610-696).
// 2-4 species: 6 CTAs/SM (a small spill) hide more load latency (H2/O2 -14%)
template <int NS, int TM>
#ifndef IGN_VISC1_MINB
#define IGN_VISC1_MINB 8  // one species: 8 CTAs/SM (64 registers, small spill) -4% viscous
#endif
__global__ void __launch_bounds__(128, (NS > 1 && NS <= 4) ? 6 : NS == 1 ? IGN_VISC1_MINB : 1) k_visc(const __grid_constant__ KParams P, int stage,
                                              int step) {
    constexpr int NC = NS + 3;
    if (failed_before(P.err, step, stage, PH_RHS)) return;
    const int w = P.nx + 2;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)w * (P.ny + 2)) return;
    const int i = (int)(t % w) - 1, j = (int)(t / w) - 1;
    const long long id = pidx(P, i, j);
    const long long ie = id + 1, iw = id - 1, in = id + P.sx, is = id - P.sx;
    auto ddxi = [&](const double* f) { return 0.5 * (ldg(f + ie) - ldg(f + iw)); };
    auto ddeta = [&](const double* f) { return 0.5 * (ldg(f + in) - ldg(f + is)); };
    const double vj = ldg(P.vjac + id);
    const double xi_x = ldg(P.vmxx + id) * vj;
    const double xi_y = ldg(P.vmxy + id) * vj;
    const double eta_x = ldg(P.vmex + id) * vj;
    const double eta_y = ldg(P.vmey + id) * vj;
    auto gradx = [&](const double* f) { return xi_x * ddxi(f) + eta_x * ddeta(f); };
    auto grady = [&](const double* f) { return xi_y * ddxi(f) + eta_y * ddeta(f); };
    const double ux = gradx(PU(P)), uy = grady(PU(P));
    const double vx = gradx(PV(P)), vy = grady(PV(P));
    const double Tx = gradx(PT(P)), Ty = grady(PT(P));
    const double T = ldg(PT(P) + id), rho = ldg(PRHO(P) + id);
    double Y[NS], X[NS], gx[NS], gy[NS], hs[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        Y[s] = ldg(PY(P, s) + id);
        X[s] = ldg(PX(P, s) + id);
        gx[s] = gradx(PX(P, s));
        gy[s] = grady(PX(P, s));
        hs[s] = h_species<TM>(T, P.mix.sp[s], P.mix.R);
    }
    double mu, lambda, D, cp;
    transport<NS, TM>(rho, T, Y, X, P.mix, mu, lambda, D, cp);
    const double div = ux + vy;
    const double txx = mu * (2.0 * ux - (2.0 / 3.0) * div);
    const double tyy = mu * (2.0 * vy - (2.0 / 3.0) * div);
    const double txy = mu * (uy + vx);
    const double wbar = mean_molar_mass<NS>(Y, P.mix);
    double ucx = 0.0, ucy = 0.0;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        ucx += (P.mix.sp[s].W / wbar) * D * gx[s];
        ucy += (P.mix.sp[s].W / wbar) * D * gy[s];
    }
    double ex = lambda * Tx, ey = lambda * Ty;
    double Fd[NC], Gd[NC];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        const double jsx = rho * ((P.mix.sp[s].W / wbar) * D * gx[s] - Y[s] * ucx);
        const double jsy = rho * ((P.mix.sp[s].W / wbar) * D * gy[s] - Y[s] * ucy);
        ex += jsx * hs[s];
        ey += jsy * hs[s];
        Fd[s] = jsx;
        Gd[s] = jsy;
    }
    const double u = ldg(PU(P) + id), v = ldg(PV(P) + id);
    Fd[NS] = txx;
    Fd[NS + 1] = txy;
    Fd[NS + 2] = u * txx + v * txy + ex;
    Gd[NS] = txy;
    Gd[NS + 1] = tyy;
    Gd[NS + 2] = u * txy + v * tyy + ey;
    const double a = ldg(P.vmxx + id), b = ldg(P.vmxy + id);
    const double c2 = ldg(P.vmex + id), d = ldg(P.vmey + id);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        P.Fv[c * P.plane + id] = a * Fd[c] + b * Gd[c];
        P.Gv[c * P.plane + id] = c2 * Fd[c] + d * Gd[c];
    }
}

// ---------------------------------------------------------------- LODI
// lodi_outflow_override (solver.hpp:717-788) for cell (nx-1, j): dFx values.
template <int NS>
__device__ void lodi_dfx(const KParams& P, int j, double* dF) {
    const int i = P.nx - 1;
    const long long id = pidx(P, i, j), i1 = id - 1, i2 = id - 2;
    const double vj = ldg(P.vjac + id);
    const double xi_x = ldg(P.vmxx + id) * vj;
    const double xi_y = ldg(P.vmxy + id) * vj;
    const double sn = ghypot(xi_x, xi_y);
    const double n1 = xi_x / sn, n2 = xi_y / sn;
    auto ddn = [&](const double* f) {
        return sn * 0.5 * (3.0 * ldg(f + id) - 4.0 * ldg(f + i1) + ldg(f + i2));
    };
    const double rr = ldg(PRHO(P) + id), cc0 = ldg(PC(P) + id), pp = ldg(PP(P) + id);
    const double uu = ldg(PU(P) + id), vv = ldg(PV(P) + id);
    const double un = n1 * uu + n2 * vv;
    const double M = smin(fabs(un) / cc0, 0.99);
    const double drdn = ddn(PRHO(P));
    const double dpdn = ddn(PP(P));
    const double dundn = n1 * ddn(PU(P)) + n2 * ddn(PV(P));
    const double dutdn = -n2 * ddn(PU(P)) + n1 * ddn(PV(P));
    const double K = P.sigma_out_right * cc0 * (1.0 - M * M) / P.lx;
    const double L1 = K * (pp - P.p_target_right);
    const double out = un > 0.0 ? un : 0.0;
    const double L2 = out * (cc0 * cc0 * drdn - dpdn);
    const double L3 = out * dutdn;
    const double L5 = (un + cc0) * (dpdn + rr * cc0 * dundn);
    const double drdt = -(L2 + 0.5 * (L5 + L1)) / (cc0 * cc0);
    const double dundt = -(L5 - L1) / (2.0 * rr * cc0);
    const double dutdt = -L3;
    const double dpdt = -0.5 * (L5 + L1);
    double Y[NS], dYdt[NS];
    double sumRdY = 0.0;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        Y[s] = ldg(PY(P, s) + id);
        dYdt[s] = -out * ddn(PY(P, s));
        sumRdY += divW(P.mix.sp[s], P.mix.R) * dYdt[s];
    }
    const double rbar = r_specific<NS>(Y, P.mix);
    const double Tt = ldg(PT(P) + id);
    const double dTdt = Tt * (dpdt / pp - drdt / rr - sumRdY / rbar);
    const double dudt = n1 * dundt - n2 * dutdt;
    const double dvdt = n2 * dundt + n1 * dutdt;
    const double k = 0.5 * (uu * uu + vv * vv);
    const double e = e_mass_rs<NS>(Tt, Y, rbar, P.mix);
    const double cv = cp_mass<NS>(Tt, Y, P.mix) - rbar;
    double sum_es_dY = 0.0;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        const double esn = h_species(Tt, P.mix.sp[s], P.mix.R) - divW(P.mix.sp[s], P.mix.R) * Tt;
        sum_es_dY += esn * dYdt[s];
    }
    double dU[NS + 3];
#pragma unroll
    for (int s = 0; s < NS; ++s) dU[s] = Y[s] * drdt + rr * dYdt[s];
    dU[NS] = uu * drdt + rr * dudt;
    dU[NS + 1] = vv * drdt + rr * dvdt;
    dU[NS + 2] = (e + k) * drdt + rr * cv * dTdt + rr * sum_es_dY + rr * (uu * dudt + vv * dvdt);
    const double invJ = 1.0 / ldg(P.jac + id);
#pragma unroll
    for (int c = 0; c < NS + 3; ++c) dF[c] = -dU[c] * invJ;
}

// ---------------------------------------------------------------- assemble + update
// MODE 0: rhs only (compute_rhs, solver.hpp:185-232).  MODE 1: stage 1
// U <- U0 + dt r (axpy_interior :799-807).  MODE 2: U <- U0 + w((U-U0) + dt r)
// (blend_interior :810-821).  MODE 1/2 also clip + validate (post_stage
// :826-849) and carry the ghost ring of Ucur into Uout.
// laser_power out of line: the common (laser-free) update stays small
static __device__ __noinline__ double laser_cold2(double x, double y, double t, const DLaser& p) {
    return laser_power(x, y, t, p);
}

// EDGE = false: every padded node except, when LODI is on, the right-edge
// column; EDGE = true: that column alone (grid over j), with the LODI x-flux
// difference — the LODI code never enters the bulk update.
// 2-4 species: 4 CTAs/SM (64 registers): H2/O2 update -10% (the 3D update
// loses 7% this way and keeps its default)
template <int NS, int MODE, bool EDGE>
__global__ void __launch_bounds__(256, (NS > 1 && NS <= 4) ? 4 : 1) k_assemble(const __grid_constant__ KParams P,
                                                  const double* __restrict__ U0,
                                                  const double* __restrict__ Ucur,
                                                  double* __restrict__ Uout, double dt,
                                                  double w, double t_stage, int stage,
                                                  int step, int clip_slot) {
    constexpr int NC = NS + 3;
    __shared__ unsigned long long s_clip;
    if (threadIdx.x == 0) s_clip = 0ull;
    __syncthreads();
    const bool dead = failed_before(P.err, step, stage, PH_RHS);
    long long id;
    bool in_range;
    if (EDGE) {
        const int t = blockIdx.x * blockDim.x + threadIdx.x;  // row j of the column
        in_range = t < P.ny;
        id = in_range ? pidx(P, P.nx - 1, t) : 0;
    } else {
        id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
        in_range = id < P.plane;
    }
    double clip = 0.0;
    if (!dead && in_range) {
        const int ip = (int)(id % P.sx), jp = (int)(id / P.sx);
        const int i = ip - P.g, j = jp - P.g;
        const bool interior = i >= 0 && i < P.nx && j >= 0 && j < P.ny;
        if (!EDGE && interior && P.lodi && i == P.nx - 1) {
            // the right-edge column is the EDGE launch's
        } else if (!interior) {
            if (MODE != 0) {
#pragma unroll
                for (int c = 0; c < NC; ++c) Uout[c * P.plane + id] = Ucur[c * P.plane + id];
            }
        } else {
            double r[NC];
            const long long fxp = (long long)(P.nx + 1) * P.ny;
            const long long fyp = (long long)P.nx * (P.ny + 1);
            const long long fx = (long long)j * (P.nx + 1) + i;
            const long long fy = (long long)j * P.nx + i;
            double dFl[EDGE ? NC : 1];
            if (EDGE) lodi_dfx<NS>(P, j, dFl);
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const double dF = EDGE ? dFl[EDGE ? c : 0] : P.Fx[c * fxp + fx + 1] - P.Fx[c * fxp + fx];
                const double dG = P.Gy[c * fyp + fy + P.nx] - P.Gy[c * fyp + fy];
                r[c] = -(dF + dG);
            }
            if (P.viscous) {
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    const double* Fv = P.Fv + c * P.plane;
                    const double* Gv = P.Gv + c * P.plane;
                    const double dVx = 0.5 * (Fv[id + 1] - Fv[id - 1]);
                    const double dVy = 0.5 * (Gv[id + P.sx] - Gv[id - P.sx]);
                    r[c] += dVx + dVy;
                }
            }
            const double J = ldg(P.jac + id);
            const double invJ = 1.0 / J;
            if (P.mech.present) {
                double Y[NS], wdot[NS];
#pragma unroll
                for (int s = 0; s < NS; ++s) Y[s] = ldg(PY(P, s) + id);
                source_terms<NS>(ldg(PRHO(P) + id), ldg(PT(P) + id), Y, P.mix, P.mech, wdot);
#pragma unroll
                for (int s = 0; s < NS; ++s) r[s] += wdot[s] * invJ;
            }
            if (P.laser.on)
                r[NS + 2] += laser_cold2(ldg(P.xc + id), ldg(P.yc + id), t_stage, P.laser) * invJ;
            const unsigned long long cell = (unsigned long long)(j + P.j0) * P.nx + i;
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
    }
    if (MODE != 0) {
        if (clip > 0.0) atomicMax(&s_clip, (unsigned long long)__double_as_longlong(clip));
        __syncthreads();
        if (threadIdx.x == 0 && s_clip) atomicMax(&P.red[2 + clip_slot], s_clip);
    }
}

// ---------------------------------------------------------------- stable dt
// stable_dt's per-cell spectra (solver.hpp:246-289); max/min are order-free,
// so the reduction is bit-identical to the serial loop.
template <int NS>
__global__ void __launch_bounds__(256) k_dt(const __grid_constant__ KParams P) {
    __shared__ unsigned long long s_lam, s_chem;
    if (threadIdx.x == 0) {
        s_lam = 0ull;
        s_chem = 0x7ff0000000000000ull;  // +inf
    }
    __syncthreads();
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    double lam_loc = 0.0, chem_loc = __longlong_as_double(0x7ff0000000000000ll);
    if (t < (long long)P.nx * P.ny) {
        const int i = (int)(t % P.nx), j = (int)(t / P.nx);
        const long long id = pidx(P, i, j);
        const double J = ldg(P.jac + id);
        const double mxx = ldg(P.mxx + id), mxy = ldg(P.mxy + id);
        const double mex = ldg(P.mex + id), mey = ldg(P.mey + id);
        const double sx = ghypot(mxx, mxy);
        const double sy = ghypot(mex, mey);
        const double u = ldg(PU(P) + id), v = ldg(PV(P) + id), c = ldg(PC(P) + id);
        const double ux = mxx * u + mxy * v;
        const double uy = mex * u + mey * v;
        double lam = (fabs(ux) + c * sx + fabs(uy) + c * sy) * J;
        double Y[NS];
#pragma unroll
        for (int s = 0; s < NS; ++s) Y[s] = ldg(PY(P, s) + id);
        const double rho = ldg(PRHO(P) + id), T = ldg(PT(P) + id);
        if (P.viscous) {
            double X[NS];
            mole_fractions<NS>(Y, P.mix, X);
            double mu, lambda, D, cp;
            transport<NS>(rho, T, Y, X, P.mix, mu, lambda, D, cp);
            const double nu = smax(2.0 * mu / rho, smax(lambda / (rho * cp), D));
            lam += 2.0 * nu * (sx * sx + sy * sy) * J * J;
        }
        lam_loc = smax(0.0, lam);
        if (P.mech.present && P.chem_dt_limit) {
            double wdot[NS];
            source_terms<NS>(rho, T, Y, P.mix, P.mech, wdot);
#pragma unroll
            for (int s = 0; s < NS; ++s) {
                const double wv = fabs(wdot[s]);
                if (wv > 0.0) {
                    const double mass = rho * smax(Y[s], 1e-3);
                    chem_loc = smin(chem_loc, P.chem_dt_factor * mass / wv);
                }
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

// ---------------------------------------------------------------- launcher table
template <int NS> struct Launch {
    // one ghost-fill pass: x edges over rows 0..ny-1 (ypass 0) or y edges over
    // the full padded width (ypass 1) — boundary.hpp:254-257
    static int bc(const KParams& P, double* Ut, int ypass, int stage, int step, cudaStream_t s) {
        const int n = ypass ? P.nx + 2 * P.g : P.ny;
        const unsigned nb = (2 * n * P.g + 127) / 128;  // (edge, t, ghost layer)
        switch (thermo_mode<NS>(P.mix)) {
        case 1: k_bc<NS, 1><<<nb, 128, 0, s>>>(P, Ut, ypass, stage, step); break;
        case 2: k_bc<NS, 2><<<nb, 128, 0, s>>>(P, Ut, ypass, stage, step); break;
        default: k_bc<NS, 0><<<nb, 128, 0, s>>>(P, Ut, ypass, stage, step); break;
        }
        return 1;
    }
    // padded rows [r_lo, r_hi)
    static int prim_rows(const KParams& P, const double* Ut, int stage, int step,
                         cudaStream_t s, int r_lo, int r_hi) {
        const long long lo = (long long)r_lo * P.sx, hi = (long long)r_hi * P.sx;
        if (hi <= lo) return 0;
        const unsigned nb = (unsigned)((hi - lo + 255) / 256);
        const int tm = thermo_mode<NS>(P.mix);
        if (P.viscous) {
            if (tm == 1) k_prim<NS, true, 1><<<nb, 256, 0, s>>>(P, Ut, stage, step, lo, hi);
            else if (tm == 2) k_prim<NS, true, 2><<<nb, 256, 0, s>>>(P, Ut, stage, step, lo, hi);
            else k_prim<NS, true, 0><<<nb, 256, 0, s>>>(P, Ut, stage, step, lo, hi);
        } else {
            if (tm == 1) k_prim<NS, false, 1><<<nb, 256, 0, s>>>(P, Ut, stage, step, lo, hi);
            else if (tm == 2) k_prim<NS, false, 2><<<nb, 256, 0, s>>>(P, Ut, stage, step, lo, hi);
            else k_prim<NS, false, 0><<<nb, 256, 0, s>>>(P, Ut, stage, step, lo, hi);
        }
        return 1;
    }
    // part (KernelSet): 0 the padded box, 1 this slab's own rows, 2 its ghost rows
    static int prim(const KParams& P, const double* Ut, int stage, int step, cudaStream_t s,
                    int part) {
        const int g = P.g, R = P.ny + 2 * g;
        if (part == 1) return prim_rows(P, Ut, stage, step, s, g, R - g);
        if (part == 2)
            return prim_rows(P, Ut, stage, step, s, 0, g) +
                   prim_rows(P, Ut, stage, step, s, R - g, R);
        return prim_rows(P, Ut, stage, step, s, 0, R);
    }
    // part: 0 every face; 1 x faces + the y faces whose stencils lie in owned
    // rows; 2 the remaining y faces (they read the halo rows)
    template <bool TENO, bool CHAR>
    static int faces_t(const KParams& P, const double* Ut, int stage, int step, cudaStream_t s,
                       int part) {
        constexpr int H = TENO ? 3 : 2;
        const int lo = H < P.ny + 1 ? H : P.ny + 1;
        const int hi = P.ny - H + 1 > lo ? P.ny - H + 1 : lo;
        int n = 0;
        if (part != 2) n += launch_faces3<NS, 0, TENO, CHAR>(P, Ut, stage, step, s);
        if (part == 0) return n + launch_faces3<NS, 1, TENO, CHAR>(P, Ut, stage, step, s);
        if (part == 1) return n + launch_faces3<NS, 1, TENO, CHAR>(P, Ut, stage, step, s, lo, hi);
        n += launch_faces3<NS, 1, TENO, CHAR>(P, Ut, stage, step, s, 0, lo);
        return n + launch_faces3<NS, 1, TENO, CHAR>(P, Ut, stage, step, s, hi, P.ny + 1);
    }
    static int faces(const KParams& P, int teno, int chr, const double* Ut, int stage, int step,
                     cudaStream_t s, int part) {
        if (teno && chr) return faces_t<true, true>(P, Ut, stage, step, s, part);
        if (teno) return faces_t<true, false>(P, Ut, stage, step, s, part);
        if (chr) return faces_t<false, true>(P, Ut, stage, step, s, part);
        return faces_t<false, false>(P, Ut, stage, step, s, part);
    }
    static int visc(const KParams& P, int stage, int step, cudaStream_t s) {
        const long long n = (long long)(P.nx + 2) * (P.ny + 2);
        const unsigned nb = (unsigned)((n + 127) / 128);
        switch (thermo_mode<NS>(P.mix)) {
        case 1: k_visc<NS, 1><<<nb, 128, 0, s>>>(P, stage, step); break;
        case 2: k_visc<NS, 2><<<nb, 128, 0, s>>>(P, stage, step); break;
        default: k_visc<NS, 0><<<nb, 128, 0, s>>>(P, stage, step); break;
        }
        return 1;
    }
    template <bool EDGE>
    static void assemble_t(const KParams& P, int mode, const double* U0, const double* Ucur,
                           double* Uout, double dt, double w, double t_stage, int stage,
                           int step, int clip_slot, unsigned nb, cudaStream_t s) {
        if (mode == 0)
            k_assemble<NS, 0, EDGE><<<nb, 256, 0, s>>>(P, U0, Ucur, Uout, dt, w, t_stage, stage,
                                                       step, clip_slot);
        else if (mode == 1)
            k_assemble<NS, 1, EDGE><<<nb, 256, 0, s>>>(P, U0, Ucur, Uout, dt, w, t_stage, stage,
                                                       step, clip_slot);
        else
            k_assemble<NS, 2, EDGE><<<nb, 256, 0, s>>>(P, U0, Ucur, Uout, dt, w, t_stage, stage,
                                                       step, clip_slot);
    }
    static int assemble(const KParams& P, int mode, const double* U0, const double* Ucur,
                        double* Uout, double dt, double w, double t_stage, int stage, int step,
                        int clip_slot, cudaStream_t s) {
        assemble_t<false>(P, mode, U0, Ucur, Uout, dt, w, t_stage, stage, step, clip_slot,
                          (unsigned)((P.plane + 255) / 256), s);
        if (!P.lodi) return 1;
        assemble_t<true>(P, mode, U0, Ucur, Uout, dt, w, t_stage, stage, step, clip_slot,
                         (unsigned)((P.ny + 255) / 256), s);
        return 2;
    }
    static int dt(const KParams& P, cudaStream_t s) {
        const long long n = (long long)P.nx * P.ny;
        k_dt<NS><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(P);
        return 1;
    }
    static KernelSet make() {
        return KernelSet{&bc, &prim, &faces, &visc, &assemble, &dt};
    }
};

KernelSet kernel_set(int ns);

}  // namespace ign
