// faces.cuh — inviscid face fluxes (solver.hpp:441-579), B200 layout.
//
// One CTA owns 32 consecutive faces of one line and runs NC = ns+3 warps:
// warp w evaluates characteristic field (or conservative component) w for the
// 32 faces, lane = face.  The split keeps the per-thread state to one field's
// 2h projected values plus the TENO temporaries (~80 registers instead of the
// 12*NC doubles a thread-per-face kernel holds), and every warp is uniform in
// its field type, so the field-specific formulas never diverge.
//
//   phase 1  all warps   stage the 2h-wide node window into shared memory:
//                        U = Ut*J, the mapped flux m1 F + m2 G (solver.hpp:
//                        466-479, flux.hpp:39-50) and the cached u, v, c —
//                        each node's mapped flux is computed once per CTA, not
//                        once per face that reads it;
//            warp 0      Roe average + eigensystem per face (solver.hpp:493-502)
//   phase 2  warp w      L_w F, L_w U on the 2h nodes, alpha_w, the LLF split
//                        and the two TENO6/WENO3Z reconstructions (:516-534)
//   phase 3  warp w      component w of R*amp (flux.hpp:123-139), coalesced store
//
// Arithmetic per value is the reference's, operation for operation (the
// per-field projection below is EigenSystem::project's row w).
#pragma once

#include "flux.cuh"
#include "kernels_common.cuh"

namespace ign {

// Row f of EigenSystem::project (flux.hpp:107-120) for one conservative-space
// vector q, from the per-face eigen data held in registers.
template <int NS> struct FaceEigen {
    double n1, n2, s, u, v, un, ut, k, H, c, c2, kappa, c2x2, y2c2, yc2, ykappa;
    double Y[NS], Theta[NS];
};

template <int NS>
__device__ __forceinline__ double project_row(const FaceEigen<NS>& e, int f, const double* q) {
    double drho = 0.0;
#pragma unroll
    for (int sp = 0; sp < NS; ++sp) drho += q[sp];
    if (f == 1 + NS) return -e.n2 * q[NS] + e.n1 * q[NS + 1] - e.ut * drho;
    double dp = e.kappa * q[NS + 2] - e.kappa * e.u * q[NS] - e.kappa * e.v * q[NS + 1];
#pragma unroll
    for (int sp = 0; sp < NS; ++sp) dp += e.Theta[sp] * q[sp];
    if (f >= 1 && f <= NS) {
        double Ys = 0.0, qs = 0.0;
#pragma unroll
        for (int sp = 0; sp < NS; ++sp)
            if (sp == f - 1) {
                Ys = e.Y[sp];
                qs = q[sp];
            }
        return qs - fdiv(Ys * dp, e.c2, e.yc2);
    }
    const double dun = e.n1 * q[NS] + e.n2 * q[NS + 1] - e.un * drho;
    if (f == 0) return fdiv(dp - e.c * dun, e.c2x2, e.y2c2);
    return fdiv(dp + e.c * dun, e.c2x2, e.y2c2);
}

// Shared-memory plan of one CTA.  NT = nodes in the window.
template <int NS, int DIR, bool TENO> struct FaceSmem {
    static constexpr int NC = NS + 3;
    static constexpr int H = TENO ? 3 : 2;
    static constexpr int W = 2 * H;
    static constexpr int NT = DIR == 0 ? 32 + W - 1 : 32 * W;
    static constexpr int NE = 16 + 2 * NS;
    double U[NC][NT];
    double F[NC][NT];
    double u[NT], v[NT], c[NT];
    double E[NE][32];   // per-face eigen data (char) / [0] = alpha, [1] = sf (comp)
    double amp[NC][32];
    int bad[32];
};

// node index inside the window for stencil slot k of face lane
template <int DIR, int W> __device__ __forceinline__ int tile_node(int lane, int k) {
    return DIR == 0 ? lane + k : k * 32 + lane;
}

template <int NS, int DIR, bool TENO, bool CHAR>
__global__ void __launch_bounds__(32 * (NS + 3))
k_faces2(const __grid_constant__ KParams P, const double* __restrict__ Ut, int stage, int step) {
    constexpr int NC = NS + 3;
    constexpr int H = TENO ? 3 : 2;
    constexpr int W = 2 * H;
    using Smem = FaceSmem<NS, DIR, TENO>;
    constexpr int NT = Smem::NT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& S = *reinterpret_cast<Smem*>(smem_raw);
    __shared__ int s_dead;  // one read of the error word per CTA keeps exits uniform
    if (threadIdx.x == 0) s_dead = failed(P.err);
    __syncthreads();
    if (s_dead) return;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nfaces = DIR == 0 ? P.nx + 1 : P.nx;  // faces (x) / columns (y) per line
    int line, f0;  // x: line = row j, faces f0..f0+31; y: line = face row, columns f0..
    if (DIR == 0) {
        f0 = blockIdx.x * 32;
        line = blockIdx.y;
    } else {
        f0 = blockIdx.x * 32;
        line = blockIdx.y;
    }
    const int lane_f = f0 + lane;
    const bool active = lane_f < nfaces;
    const long long step_n = DIR == 0 ? 1 : P.sx;
    const double* m1a = DIR == 0 ? P.mxx : P.mex;
    const double* m2a = DIR == 0 ? P.mxy : P.mey;
    // padded index of the window's node 0
    // x: node i = f0 - H .. f0 + 31 + H - 1 on row j = line
    // y: node (i = f0 + lane, j = line - H + k)
    const long long win0 = DIR == 0 ? pidx(P, f0 - H, line) : pidx(P, f0, line - H);

    // ---------------- phase 1: node window -> shared memory (all warps)
    for (int t = threadIdx.x; t < NT; t += blockDim.x) {
        long long id;
        bool ok;
        if (DIR == 0) {
            id = win0 + t;
            ok = f0 - H + t < P.nx + P.g;
        } else {
            const int k = t / 32, l = t % 32;
            id = win0 + (long long)k * P.sx + l;
            ok = f0 + l < P.nx;
        }
        if (!ok) continue;
        const double J = ldg(P.jac + id);
        double Uk[NC], Fk[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) Uk[c] = ldg(Ut + c * P.plane + id) * J;
        mapped_flux<NS>(Uk, ldg(PP(P) + id), ldg(m1a + id), ldg(m2a + id), Fk);
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            S.U[c][t] = Uk[c];
            S.F[c][t] = Fk[c];
        }
        S.u[t] = ldg(PU(P) + id);
        S.v[t] = ldg(PV(P) + id);
        S.c[t] = ldg(PC(P) + id);
    }
    // face metric (solver.hpp:484-489): mean of the two node metrics
    const long long il = DIR == 0 ? pidx(P, lane_f - 1, line) : pidx(P, lane_f, line - 1);
    const long long ir = il + step_n;
    const unsigned phase = DIR == 0 ? PH_INVX : PH_INVY;
    const unsigned long long eidx =
        DIR == 0 ? (unsigned long long)line * (P.nx + 1) + lane_f
                 : (unsigned long long)lane_f * (P.ny + 1) + line;
    if (CHAR && warp == 0) {
        int bad = 0;
        if (active) {
            const double m1f = 0.5 * (ldg(m1a + il) + ldg(m1a + ir));
            const double m2f = 0.5 * (ldg(m2a + il) + ldg(m2a + ir));
            double Yl[NS], Yr[NS], Ya[NS];
#pragma unroll
            for (int s = 0; s < NS; ++s) {
                Yl[s] = ldg(PY(P, s) + il);
                Yr[s] = ldg(PY(P, s) + ir);
            }
            double Ta, ua, va;
            roe_average<NS>(ldg(PRHO(P) + il), Yl, ldg(PT(P) + il), ldg(PU(P) + il),
                            ldg(PV(P) + il), ldg(PRHO(P) + ir), Yr, ldg(PT(P) + ir),
                            ldg(PU(P) + ir), ldg(PV(P) + ir), P.mix, Ya, Ta, ua, va);
            Eigen<NS> es;
            const int est = eigen_at_state<NS>(Ya, Ta, ua, va, m1f, m2f, P.mix, es);
            if (est) {
                report(P.err, stage, phase, eidx, 1 + est, step);
                bad = 1;
            }
            double* E = &S.E[0][0];
            const double vals[16] = {es.n1, es.n2, es.s,  es.u,  es.v,    es.un,   es.ut,  es.k,
                                     es.H,  es.c,  es.c2, es.kappa, es.c2x2, es.y2c2, es.yc2,
                                     es.ykappa};
#pragma unroll
            for (int q = 0; q < 16; ++q) E[q * 32 + lane] = vals[q];
#pragma unroll
            for (int s = 0; s < NS; ++s) {
                E[(16 + s) * 32 + lane] = es.Y[s];
                E[(16 + NS + s) * 32 + lane] = es.Theta[s];
            }
        }
        S.bad[lane] = bad;
    }
    __syncthreads();
    if (!CHAR && warp == 0) {
        // componentwise wave speed (solver.hpp:537-548)
        int bad = 0;
        if (active) {
            const double m1f = 0.5 * (ldg(m1a + il) + ldg(m1a + ir));
            const double m2f = 0.5 * (ldg(m2a + il) + ldg(m2a + ir));
            const double sf = ghypot(m1f, m2f);
            double alpha = 0.0;
#pragma unroll
            for (int k = 0; k < W; ++k) {
                const int t = tile_node<DIR, W>(lane, k);
                const double un = (m1f * S.u[t] + m2f * S.v[t]) / sf;
                alpha = smax(alpha, sf * (fabs(un) + S.c[t]));
            }
            if (!isfinite(alpha)) {
                report(P.err, stage, phase, eidx, 1, step);
                bad = 1;
            }
            S.E[0][lane] = alpha;
        }
        S.bad[lane] = bad;
    }
    if (!CHAR) __syncthreads();

    // ---------------- phase 2: one field per warp
    const int fl = warp;  // characteristic field / conservative component
    double amp = 0.0;
    const bool live = active && !S.bad[lane];
    if (CHAR && live) {
        FaceEigen<NS> e;
        const double* E = &S.E[0][0];
        e.n1 = E[0 * 32 + lane];
        e.n2 = E[1 * 32 + lane];
        e.s = E[2 * 32 + lane];
        e.u = E[3 * 32 + lane];
        e.v = E[4 * 32 + lane];
        e.un = E[5 * 32 + lane];
        e.ut = E[6 * 32 + lane];
        e.k = E[7 * 32 + lane];
        e.H = E[8 * 32 + lane];
        e.c = E[9 * 32 + lane];
        e.c2 = E[10 * 32 + lane];
        e.kappa = E[11 * 32 + lane];
        e.c2x2 = E[12 * 32 + lane];
        e.y2c2 = E[13 * 32 + lane];
        e.yc2 = E[14 * 32 + lane];
        e.ykappa = E[15 * 32 + lane];
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            e.Y[s] = E[(16 + s) * 32 + lane];
            e.Theta[s] = E[(16 + NS + s) * 32 + lane];
        }
        double lf[W], lu[W];
        double alpha = 0.0;
#pragma unroll
        for (int k = 0; k < W; ++k) {
            const int t = tile_node<DIR, W>(lane, k);
            double q[NC];
#pragma unroll
            for (int c = 0; c < NC; ++c) q[c] = S.F[c][t];
            lf[k] = project_row<NS>(e, fl, q);
#pragma unroll
            for (int c = 0; c < NC; ++c) q[c] = S.U[c][t];
            lu[k] = project_row<NS>(e, fl, q);
            // EigenSystem::field_speed at the node's normal velocity (flux.hpp:143-147)
            const double unk = e.n1 * S.u[t] + e.n2 * S.v[t];
            const double ck = S.c[t];
            const double lam = fl == 0 ? e.s * (unk - ck) : fl == NC - 1 ? e.s * (unk + ck)
                                                                          : e.s * unk;
            alpha = smax(alpha, fabs(lam));
        }
        if (!isfinite(alpha)) {
            report(P.err, stage, phase, eidx, 1, step);
        } else {
            double wp[W], wm[W];
#pragma unroll
            for (int k = 0; k < W; ++k) {
                wp[k] = 0.5 * (lf[k] + alpha * lu[k]);
                wm[k] = 0.5 * (lf[k] - alpha * lu[k]);
            }
            amp = face_pm<TENO>(wp, wm, P.ct, P.eps);
        }
    } else if (!CHAR && live) {
        const double alpha = S.E[0][lane];
        double wp[W], wm[W];
#pragma unroll
        for (int k = 0; k < W; ++k) {
            const int t = tile_node<DIR, W>(lane, k);
            wp[k] = 0.5 * (S.F[fl][t] + alpha * S.U[fl][t]);
            wm[k] = 0.5 * (S.F[fl][t] - alpha * S.U[fl][t]);
        }
        amp = face_pm<TENO>(wp, wm, P.ct, P.eps);
    }

    double* out = DIR == 0 ? P.Fx : P.Gy;
    const long long fplane = (long long)(P.nx + 1 - DIR) * (P.ny + DIR);
    const long long o = DIR == 0 ? (long long)line * (P.nx + 1) + lane_f
                                 : (long long)line * P.nx + lane_f;
    if (!CHAR) {
        if (active) out[fl * fplane + o] = amp;
        return;
    }
    // ---------------- phase 3: component w of R * amp (flux.hpp:123-139)
    S.amp[fl][lane] = amp;
    __syncthreads();
    if (!active) return;
    const double* E = &S.E[0][0];
    const double am = S.amp[0][lane];
    const double ap = S.amp[2 + NS][lane];
    const double at = S.amp[1 + NS][lane];
    double asum = 0.0;
#pragma unroll
    for (int sp = 0; sp < NS; ++sp) asum += S.amp[1 + sp][lane];
    const double c = E[9 * 32 + lane];
    double r;
    if (fl < NS) {
        r = E[(16 + fl) * 32 + lane] * (am + ap) + S.amp[1 + fl][lane];
    } else if (fl == NS) {
        const double u = E[3 * 32 + lane], n1 = E[0 * 32 + lane], n2 = E[1 * 32 + lane];
        r = (u - c * n1) * am + (u + c * n1) * ap + u * asum - n2 * at;
    } else if (fl == NS + 1) {
        const double v = E[4 * 32 + lane], n1 = E[0 * 32 + lane], n2 = E[1 * 32 + lane];
        r = (v - c * n2) * am + (v + c * n2) * ap + v * asum + n1 * at;
    } else {
        const double Hh = E[8 * 32 + lane], un = E[5 * 32 + lane], ut = E[6 * 32 + lane];
        const double kk = E[7 * 32 + lane], kappa = E[11 * 32 + lane];
        const double ykappa = E[15 * 32 + lane];
        double en = (Hh - c * un) * am + (Hh + c * un) * ap + ut * at;
#pragma unroll
        for (int sp = 0; sp < NS; ++sp) {
            const double th = E[(16 + NS + sp) * 32 + lane];
            en += S.amp[1 + sp][lane] *
                  (2.0 * kk - (NS > 1 ? fdiv(th, kappa, ykappa) : th / kappa));
        }
        r = en;
    }
    out[fl * fplane + o] = r;
}

template <int NS, int DIR, bool TENO, bool CHAR>
inline void launch_faces2(const KParams& P, const double* Ut, int stage, int step,
                          cudaStream_t s) {
    constexpr int NC = NS + 3;
    const size_t smem = sizeof(FaceSmem<NS, DIR, TENO>);
    auto kern = k_faces2<NS, DIR, TENO, CHAR>;
    static bool configured = false;  // per instantiation, host side
    if (!configured) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = true;
    }
    dim3 grid(DIR == 0 ? (P.nx + 1 + 31) / 32 : (P.nx + 31) / 32, DIR == 0 ? P.ny : P.ny + 1);
    kern<<<grid, 32 * NC, smem, s>>>(P, Ut, stage, step);
}

}  // namespace ign
