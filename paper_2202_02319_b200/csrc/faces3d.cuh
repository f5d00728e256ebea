// faces3d.cuh — inviscid face fluxes of the 3D extension (extruded meshes,
// flux3.cuh).  Same CTA organisation as faces.cuh: NC = ns+4 warps own
// 32*NC faces (x: along a row; y/z: 8 columns x 4NC face lines), the node
// window lives in shared memory, warp w evaluates characteristic field w.
#pragma once

#include <cstdio>
#include <cstdlib>

#include "flux3.cuh"
#include "kernels_common.cuh"

namespace ign {

// 3D addressing helpers (state planes: (nx+2g)(ny+2g)(nz+2g), i fastest;
// metric planes are 2D: the mesh is extruded in z)
__device__ __forceinline__ long long pidx3(const KParams& P, int i, int j, int k) {
    return (long long)(k + P.g) * P.sxy + (long long)(j + P.g) * P.sx + (i + P.g);
}

// y/z tile width (columns): see FaceSmem3::TW.  One species: 8 columns (the window's
// halo lines shrink, one more CTA fits per SM); several: 32 (those kernels are
// held at 2 CTAs/SM by registers, and the wider tile keeps the launch in
// whole waves at 512^2)
template <int NS, int DIR> __host__ __device__ constexpr int tile_w3() {
    return DIR == 0 || NS > 1 ? 32 : 8;
}

// CHAR = false (componentwise) needs only the node window and one LLF speed
// per face: the characteristic tables shrink to one row so more CTAs fit
template <int NS, int DIR, bool TENO, bool CHAR = true> struct FaceSmem3 {
    static constexpr int NC = NS + 4;
    static constexpr int H = TENO ? 3 : 2;
    static constexpr int W = 2 * H;
    static constexpr int NF = 32 * NC;
    // y/z tiles: TW columns x NF/TW face lines (a narrow tile keeps the
    // window's halo lines few: 4 CTAs/SM fit)
    static constexpr int TW = tile_w3<NS, DIR>();
    static constexpr int LINES = NF / TW;
    // x: up to two row segments of the flattened face order (see k_faces3d)
    static constexpr int NT = DIR == 0 ? NF + 2 * (W - 1) : TW * (LINES + W - 1);
    // eigen table rows: 10 common + Y, Theta + the direction's own (n1, n2
    // for xi/eta faces; n3 for zeta faces — the others are 0 or alias u, v, w;
    // un, ut1 and k are recomputed by the eigensystem's own expressions)
    static constexpr int NE_CHAR = 10 + 2 * NS + (DIR < 2 ? 2 : 1);
    static constexpr int NE = CHAR ? NE_CHAR : 1;
    static constexpr int NV = 2 * W;
    static constexpr int NV_S = CHAR ? NV : 1;   // projection table rows
    static constexpr int NA_S = CHAR ? NC : 1;   // amplitude table rows
    static constexpr int NK_S = CHAR ? 3 : 1;    // LLF speed kinds
    static constexpr int NVEL = DIR < 2 ? 2 : 1;  // wave speed: (u, v) or w
    double U[NC][NT];
    double F[NC][NT];
    double vel[NVEL][NT];
    double c[NT];
    double E[NE][NF];
    // characteristic values of one group's stencil vectors, every field:
    // row fl of L F and L U (EigenSystem::project, flux.hpp:107-119 + z terms)
    double Wc[NV_S][NA_S][32];
    double amp[NA_S][32];  // one group (phase 3 follows each group)
    double alpha[NK_S][32];  // per face of the group: LLF speeds of acoustic-, convective, acoustic+
    unsigned char bad[NF];
};

enum : int {
    F3S = 0, F3U, F3V, F3W, F3H, F3C, F3C2, F3KAPPA, F3YC2, F3YKAPPA, F3Y0
};

// direction-specific eigen rows (FaceSmem3::E): ut2 is w (xi/eta) or v
// (zeta), ut1 is u for zeta faces, the off-axis normal components are 0
template <int NS, int DIR> struct ERow {
    static constexpr int X0 = F3Y0 + 2 * NS;
    template <class Sm> __device__ static double n1(const Sm& S, int f) {
        return DIR < 2 ? S.E[X0][f] : 0.0;
    }
    template <class Sm> __device__ static double n2(const Sm& S, int f) {
        return DIR < 2 ? S.E[X0 + 1][f] : 0.0;
    }
    template <class Sm> __device__ static double n3(const Sm& S, int f) {
        return DIR == 2 ? S.E[X0][f] : 0.0;
    }
    // EigenSystem::at_state's un and ut1 (flux3.cuh eigen_at_state3), same
    // operations on the same stored values
    template <class Sm> __device__ static double un(const Sm& S, int f) {
        return DIR < 2 ? n1(S, f) * S.E[F3U][f] + n2(S, f) * S.E[F3V][f]
                       : n3(S, f) * S.E[F3W][f];
    }
    template <class Sm> __device__ static double ut1(const Sm& S, int f) {
        return DIR < 2 ? -n2(S, f) * S.E[F3U][f] + n1(S, f) * S.E[F3V][f] : S.E[F3U][f];
    }
    template <class Sm> __device__ static double ut2(const Sm& S, int f) {
        return DIR < 2 ? S.E[F3W][f] : S.E[F3V][f];
    }
};

// window slot of stencil node k of face slot q = 32 g + lane; x faces past the
// first row segment (q >= L0) sit W-1 slots further (their segment's own
// halo); y/z: slot q is column q % TW of face line q / TW, its node k lies k
// lines further
template <int NS, int DIR, int W>
__device__ __forceinline__ int tile_node3(int g, int lane, int k, int L0) {
    const int q = g * 32 + lane;
    if (DIR == 0) return q + k + (q >= L0 ? W - 1 : 0);
    return q + k * tile_w3<NS, DIR>();
}

// Registers: a 5-warp CTA needs <= 128 per thread for 3 CTAs/SM (4 warps per
// SM sub-partition: 4 x 32 x 128 = 16384, the sub-partition's file); at 130
// the z kernel drops to 2 CTAs/SM and runs ~30% slower.  __maxnreg__ pins it.
#ifndef IGN_F3_MINB
#define IGN_F3_MINB 4
#endif
// xi faces (55 KB shared): 4 CTAs/SM at <= 96 registers beat 3 CTAs without
// the small spill (-1.2% faces, 256^3); eta/zeta (67-71 KB) stay at 3
#ifndef IGN_F3X_MINB
#define IGN_F3X_MINB 4
#endif
template <int NS, int DIR, bool TENO, bool CHAR, int TM>
__global__ void __launch_bounds__(32 * (NS + 4),
                                  NS != 1 ? 1 : DIR == 0 ? IGN_F3X_MINB : IGN_F3_MINB)
k_faces3d(const __grid_constant__ KParams P, const double* __restrict__ Ut, int stage, int step,
          int f_lo, int f_hi) {
    using Smem = FaceSmem3<NS, DIR, TENO, CHAR>;
    constexpr int NC = Smem::NC, H = Smem::H, W = Smem::W, NF = Smem::NF, NT = Smem::NT;
    constexpr int NV = Smem::NV;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& S = *reinterpret_cast<Smem*>(smem_raw);
    // an earlier failure (error word set) ends the kernel after phase 1: the
    // load's latency hides behind the window staging instead of stalling the
    // CTA start (garbage phase-1 reports carry larger keys than the first one)
    __shared__ int s_dead;
    const unsigned long long key0 = threadIdx.x == 0 ? err_key(P.err) : kNoError;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // DIR 0: NF consecutive faces of the flattened (row, f) order, row = k ny + j,
    // f = 0..nx — at most two row segments when nx+1 >= NF (no idle lanes at row
    // ends), else one row segment per CTA; DIR 1: TW columns i x NF/TW face
    // rows along j in plane k; DIR 2: TW columns i of row j x NF/TW face planes
    // along k
    const long long step_n = DIR == 0 ? 1 : DIR == 1 ? P.sx : P.sxy;
    const int nd = DIR == 0 ? P.nx : DIR == 1 ? P.ny : P.nz;  // cells along DIR
    const int nrows = P.ny * P.nz;
    int f0, r0 = 0, L0 = NF;
    if (DIR == 0) {
        if (P.nx + 1 >= NF) {
            const long long F0 = (long long)blockIdx.x * NF;
            r0 = (int)(F0 / (P.nx + 1));
            f0 = (int)(F0 % (P.nx + 1));
            L0 = min(NF, P.nx + 1 - f0);
        } else {
            r0 = blockIdx.z * P.ny + blockIdx.y;
            f0 = blockIdx.x * NF;
        }
    } else {
        // faces [f_lo, f_hi) along DIR (a z-slab splits interior and halo faces)
        f0 = f_lo + (DIR == 1 ? blockIdx.y : blockIdx.z) * Smem::LINES;
    }
    constexpr int TW = Smem::TW;
    const int i0 = blockIdx.x * TW;
    const int jb = DIR == 2 ? blockIdx.y : 0;  // fixed j (DIR 2)
    const int kb = DIR == 1 ? blockIdx.z : 0;  // fixed k (DIR 1)
    // metric planes: xi (DIR 0) / eta (DIR 1) use (m_x, m_y); zeta uses m_zz
    const double* m1a = DIR == 0 ? P.mxx : DIR == 1 ? P.mex : P.mzz;
    const double* m2a = DIR == 0 ? P.mxy : DIR == 1 ? P.mey : P.mzz;
    // a = index along DIR; col = i (DIR 1, 2) or the flattened row (DIR 0)
    // rows r0, r0+1 of the flattened x order as (j, k), once per CTA
    const int xj0 = DIR == 0 ? r0 % P.ny : 0, xk0 = DIR == 0 ? r0 / P.ny : 0;
    const int xj1 = DIR == 0 ? (xj0 + 1 == P.ny ? 0 : xj0 + 1) : 0;
    const int xk1 = DIR == 0 ? (xj0 + 1 == P.ny ? xk0 + 1 : xk0) : 0;
    auto node = [&](int a, int col) -> long long {
        if (DIR == 0) return col == r0 ? pidx3(P, a, xj0, xk0) : pidx3(P, a, xj1, xk1);
        if (DIR == 1) return pidx3(P, col, a, kb);
        return pidx3(P, col, jb, a);
    };
    // the (x, y) metric-plane index of the same node (the mesh is extruded)
    auto node2 = [&](int a, int col) -> int {
        if (DIR == 0) return ((col == r0 ? xj0 : xj1) + P.g) * P.sx + (a + P.g);
        if (DIR == 1) return (a + P.g) * P.sx + (col + P.g);
        return (jb + P.g) * P.sx + (col + P.g);
    };
    // x face q of this CTA -> (row, f)
    auto xface = [&](int q, int& row, int& f) {
        if (q < L0) {
            row = r0;
            f = f0 + q;
        } else {
            row = r0 + 1;
            f = q - L0;
        }
    };

    int my_f, my_col;
    if (DIR == 0) {
        xface(threadIdx.x, my_col, my_f);
    } else {
        my_f = f0 + (int)threadIdx.x / TW;
        my_col = i0 + (int)threadIdx.x % TW;
    }
    const bool my_active = DIR == 0 ? (my_f <= P.nx && my_col < nrows)
                                    : (my_col < P.nx && my_f < f_hi);
    const unsigned phase = DIR == 0 ? PH_INVX : PH_INVY;  // z faces share the y code
    auto err_index = [&](int f, int col) -> unsigned long long {
        // face f of the line through col (DIR 0: flattened row k ny + j): global
        // line-major order
        if (DIR == 0) return ((unsigned long long)col + (unsigned long long)P.j0 * P.ny) *
                                 (P.nx + 1) + f;
        if (DIR == 1)
            return ((unsigned long long)(kb + P.j0) * P.nx + col) * (P.ny + 1) + f;
        return ((unsigned long long)jb * P.nx + col) * (P.nz_glob + 1) + (f + P.j0);
    };
    // face plane offset (x: (nx+1) ny nz, y: nx (ny+1) nz, z: nx ny (nz+1))
    auto out_index = [&](int f, int col) -> long long {
        if (DIR == 0) return (long long)col * (P.nx + 1) + f;
        if (DIR == 1) return ((long long)kb * (P.ny + 1) + f) * P.nx + col;
        return ((long long)f * P.ny + jb) * P.nx + col;
    };
    const long long il = node(my_f - 1, my_col), ir = il + step_n;
    // face metrics: the four loads are issued here, combined after the window
    // staging (their latency hides behind it)
    double m1l = 0.0, m1r = 0.0, m2l = 0.0, m2r = 0.0;
    if (my_active) {
        const int l2 = node2(my_f - 1, my_col);
        const int r2 = DIR == 0 ? l2 + 1 : DIR == 1 ? l2 + P.sx : l2;
        m1l = ldg(m1a + l2), m1r = ldg(m1a + r2);
        m2l = ldg(m2a + l2), m2r = ldg(m2a + r2);
    }
    // this thread's face state, loaded before the window staging so the
    // global-load latency overlaps it (phase 1 consumes it after the loop)
    double pl[5], pr[5], Yl[NS], Yr[NS];
    if (CHAR && my_active) {
        pl[0] = ldg(PRHO3(P) + il), pl[1] = ldg(PT3(P) + il), pl[2] = ldg(PU3(P) + il);
        pl[3] = ldg(PV3(P) + il), pl[4] = ldg(PW3(P) + il);
        pr[0] = ldg(PRHO3(P) + ir), pr[1] = ldg(PT3(P) + ir), pr[2] = ldg(PU3(P) + ir);
        pr[3] = ldg(PV3(P) + ir), pr[4] = ldg(PW3(P) + ir);
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            Yl[s] = ldg(PY3(P, s) + il);
            Yr[s] = ldg(PY3(P, s) + ir);
        }
    }

    // ---------------- phase 1a: node window -> shared memory
    if constexpr (CHAR) {
        // ---------------- phase 1a: node window -> shared memory.  Each thread
        // stages NIT nodes (NIT = ceil(NT / NF), 2 here); every node's 13 loads are
        // issued before any is consumed, so the latencies overlap
        constexpr int NIT = (NT + NF - 1) / NF;
        double raw[NIT][NC + 8];
        int slot_t[NIT];
    #pragma unroll
        for (int it = 0; it < NIT; ++it) {
            const int t = threadIdx.x + it * NF;
            int a = 0, col = 0;
            bool ok = t < NT;
            if (DIR == 0) {
                const int n0 = L0 + W - 1;  // window slots of the first segment
                if (t < n0) {
                    a = f0 - H + t;
                    col = r0;
                } else {
                    a = -H + (t - n0);
                    col = r0 + 1;
                }
                ok = ok && a < P.nx + P.g && col < nrows && (t < n0 || t - n0 < NF - L0 + W - 1);
            } else {
                a = f0 - H + t / TW;
                col = i0 + t % TW;
                ok = ok && col < P.nx && a < nd + P.g;
            }
            slot_t[it] = ok ? t : -1;
            if (!ok) continue;
            const long long id = node(a, col);
            const int id2 = node2(a, col);
            double* r = raw[it];
    #pragma unroll
            for (int c = 0; c < NC; ++c) r[c] = ldg(Ut + c * P.plane + id);
            r[NC] = ldg(P.jac + id2);
            r[NC + 1] = ldg(PU3(P) + id);
            r[NC + 2] = ldg(PV3(P) + id);
            r[NC + 3] = ldg(PW3(P) + id);
            r[NC + 4] = ldg(PP3(P) + id);
            r[NC + 5] = ldg(m1a + id2);
            r[NC + 6] = ldg(m2a + id2);
            r[NC + 7] = ldg(PC3(P) + id);
        }
    #pragma unroll
        for (int it = 0; it < NIT; ++it) {
            const int t = slot_t[it];
            if (t < 0) continue;
            const double* r = raw[it];
            const double J = r[NC];
            double Uk[NC], Fk[NC];
    #pragma unroll
            for (int c = 0; c < NC; ++c) Uk[c] = r[c] * J;
            const double nu = r[NC + 1], nv = r[NC + 2], nw = r[NC + 3];
            mapped_flux3<NS, DIR>(Uk, r[NC + 4], nu, nv, nw, r[NC + 5], r[NC + 6], Fk);
    #pragma unroll
            for (int c = 0; c < NC; ++c) {
                S.U[c][t] = Uk[c];
                S.F[c][t] = Fk[c];
            }
            if (DIR < 2) {
                S.vel[0][t] = nu;
                S.vel[DIR < 2 ? 1 : 0][t] = nv;
            } else {
                S.vel[0][t] = nw;
            }
            S.c[t] = r[NC + 7];
        }
    } else {  // componentwise: the plain loop (hoisting costs it occupancy)
        for (int t = threadIdx.x; t < NT; t += blockDim.x) {
            int a, col;
            bool ok;
            if (DIR == 0) {
                const int n0 = L0 + W - 1;  // window slots of the first segment
                if (t < n0) {
                    a = f0 - H + t;
                    col = r0;
                } else {
                    a = -H + (t - n0);
                    col = r0 + 1;
                }
                ok = a < P.nx + P.g && col < nrows && (t < n0 || t - n0 < NF - L0 + W - 1);
            } else {
                a = f0 - H + t / TW;
                col = i0 + t % TW;
                ok = col < P.nx && a < nd + P.g;
            }
            if (!ok) continue;
            const long long id = node(a, col);
            const int id2 = node2(a, col);
            const double J = ldg(P.jac + id2);
            double Uk[NC], Fk[NC];
    #pragma unroll
            for (int c = 0; c < NC; ++c) Uk[c] = ldg(Ut + c * P.plane + id) * J;
            const double nu = ldg(PU3(P) + id), nv = ldg(PV3(P) + id), nw = ldg(PW3(P) + id);
            mapped_flux3<NS, DIR>(Uk, ldg(PP3(P) + id), nu, nv, nw, ldg(m1a + id2), ldg(m2a + id2),
                                  Fk);
    #pragma unroll
            for (int c = 0; c < NC; ++c) {
                S.U[c][t] = Uk[c];
                S.F[c][t] = Fk[c];
            }
            if (DIR < 2) {
                S.vel[0][t] = nu;
                S.vel[DIR < 2 ? 1 : 0][t] = nv;
            } else {
                S.vel[0][t] = nw;
            }
            S.c[t] = ldg(PC3(P) + id);
        }
    }

    const double m1f = 0.5 * (m1l + m1r), m2f = 0.5 * (m2l + m2r);
    if (CHAR) {
        int bad = 0;
        if (my_active) {
            double Ya[NS];
            double Ta, ua, va, wa;
            roe_average3<NS, TM>(pl[0], Yl, pl[1], pl[2], pl[3], pl[4], pr[0], Yr, pr[1], pr[2],
                             pr[3], pr[4], P.mix, Ya, Ta, ua, va, wa);
            Eigen3<NS> es;
            const int est = eigen_at_state3<NS, DIR == 2 ? 2 : 0, TM>(Ya, Ta, ua, va, wa, m1f, m2f,
                                                                  P.mix, es);
            if (est) {
                report(P.err, stage, phase, err_index(my_f, my_col), 1 + est, step);
                bad = 1;
            }
            const int t = threadIdx.x;
            const double vals[F3Y0] = {es.s,     es.u,   es.v,     es.w,  es.H,
                                       es.c,     es.c2,  es.kappa, es.yc2, es.ykappa};
#pragma unroll
            for (int q = 0; q < F3Y0; ++q) S.E[q][t] = vals[q];
#pragma unroll
            for (int s = 0; s < NS; ++s) {
                S.E[F3Y0 + s][t] = es.Y[s];
                S.E[F3Y0 + NS + s][t] = es.Theta[s];
            }
            constexpr int X0 = ERow<NS, DIR>::X0;
            if (DIR < 2) {
                S.E[X0][t] = es.n1;
                S.E[X0 + (DIR < 2 ? 1 : 0)][t] = es.n2;
            } else {
                S.E[X0][t] = es.n3;
            }
        }
        S.bad[threadIdx.x] = my_active ? bad : 1;
    }
    if (threadIdx.x == 0) s_dead = key0 < err_first(step, stage, DIR == 0 ? PH_INVX : PH_INVY);
    __syncthreads();
    if (s_dead) return;
    if (!CHAR) {
        // componentwise LLF wave speed (solver.hpp:537-548), 3D normal velocity
        int bad = 1;
        if (my_active) {
            const double sf = DIR < 2 ? ghypot(m1f, m2f) : ghypot(m1f, 0.0);
            double alpha = 0.0;
#pragma unroll
            for (int k = 0; k < W; ++k) {
                const int t = tile_node3<NS, DIR, W>(warp, lane, k, L0);
                const double un = DIR < 2 ? (m1f * S.vel[0][t] + m2f * S.vel[DIR < 2][t]) / sf
                                          : (m1f * S.vel[0][t]) / sf;
                alpha = smax(alpha, sf * (fabs(un) + S.c[t]));
            }
            bad = 0;
            if (!isfinite(alpha)) {
                report(P.err, stage, phase, err_index(my_f, my_col), 1, step);
                bad = 1;
            }
            S.E[0][threadIdx.x] = alpha;
        }
        S.bad[threadIdx.x] = bad;
        __syncthreads();
    }

    double* out = DIR == 0 ? P.Fx : DIR == 1 ? P.Gy : P.Hz;
    // face planes: x (nx+1) ny nz, y nx (ny+1) nz, z nx ny (nz+1)
    const long long fplane = (long long)(P.nx + (DIR == 0)) * (P.ny + (DIR == 1)) *
                             (P.nz + (DIR == 2));
    const int fl = warp;
    // ---------------- phase 3: component fl of R * amp of group g
    // (flux.hpp:123-139 + z), run while the next group's vectors are built:
    // the amplitude table holds one group
    auto assemble_group = [&](int g) {
        const int face = g * 32 + lane;
        if (S.bad[face]) return;
        int f, col;
        if (DIR == 0) {
            xface(face, col, f);
        } else {
            f = f0 + face / TW;
            col = i0 + face % TW;
        }
        const long long o = out_index(f, col);
        const double am = S.amp[0][lane];
        const double ap = S.amp[NC - 1][lane];
        const double at1 = S.amp[NC - 3][lane];
        const double at2 = S.amp[NC - 2][lane];
        const double c = S.E[F3C][face];
        using ER = ERow<NS, DIR>;
        const double n1 = ER::n1(S, face), n2 = ER::n2(S, face), n3 = ER::n3(S, face);
        double r;
        if (fl < NS) {
            r = S.E[F3Y0 + fl][face] * (am + ap) + S.amp[1 + fl][lane];
        } else {
            double asum = 0.0;
#pragma unroll
            for (int sp = 0; sp < NS; ++sp) asum += S.amp[1 + sp][lane];
            const double u = S.E[F3U][face], v = S.E[F3V][face], w = S.E[F3W][face];
            if (fl == NS) {  // rho u
                r = DIR < 2 ? (u - c * n1) * am + (u + c * n1) * ap + u * asum - n2 * at1
                            : u * am + u * ap + u * asum + at1;
            } else if (fl == NS + 1) {  // rho v
                r = DIR < 2 ? (v - c * n2) * am + (v + c * n2) * ap + v * asum + n1 * at1
                            : v * am + v * ap + v * asum + at2;
            } else if (fl == NS + 2) {  // rho w
                r = DIR < 2 ? w * am + w * ap + w * asum + at2
                            : (w - c * n3) * am + (w + c * n3) * ap + w * asum;
            } else {  // E
                const double Hh = S.E[F3H][face], un = ER::un(S, face);
                const double ut1 = ER::ut1(S, face), ut2 = ER::ut2(S, face);
                // EigenSystem's k (eigen_at_state3), from the stored velocity
                const double kk = 0.5 * ((u * u + v * v) + w * w);
                const double kappa = S.E[F3KAPPA][face];
                const double ykappa = S.E[F3YKAPPA][face];
                double en = (Hh - c * un) * am + (Hh + c * un) * ap + ut1 * at1;
                en = en + ut2 * at2;
#pragma unroll
                for (int sp = 0; sp < NS; ++sp) {
                    const double th = S.E[F3Y0 + NS + sp][face];
                    en += S.amp[1 + sp][lane] *
                          (2.0 * kk - fdiv(th, kappa, ykappa));
                }
                r = en;
            }
        }
        out[fl * fplane + o] = r;
    };
    for (int g = 0; g < NC; ++g) {
        if (CHAR && g > 0) assemble_group(g - 1);
        const int face = g * 32 + lane;
        int f, col;
        if (DIR == 0) {
            xface(face, col, f);
        } else {
            f = f0 + face / TW;
            col = i0 + face % TW;
        }
        const bool live = !S.bad[face];
        const long long o = out_index(f, col);
        if (!CHAR) {
            if (live) {
                const double alpha = S.E[0][face];
                double wp[W], wm[W];
#pragma unroll
                for (int k = 0; k < W; ++k) {
                    const int t = tile_node3<NS, DIR, W>(g, lane, k, L0);
                    wp[k] = 0.5 * (S.F[fl][t] + alpha * S.U[fl][t]);
                    wm[k] = 0.5 * (S.F[fl][t] - alpha * S.U[fl][t]);
                }
                out[fl * fplane + o] = face_pm<TENO>(wp, wm, P.rp);
            }
            continue;
        }
        // (a) field-independent parts of L q (flux.hpp:107-114 + z terms)
        const double kap = S.E[F3KAPPA][face], eu = S.E[F3U][face], ev = S.E[F3V][face],
                     ew = S.E[F3W][face];
        using ER = ERow<NS, DIR>;
        const double n1 = ER::n1(S, face), n2 = ER::n2(S, face), n3 = ER::n3(S, face);
        const double un = ER::un(S, face), ut1 = ER::ut1(S, face), ut2 = ER::ut2(S, face);
        // (kap eu) q_u etc.: the reference's left-to-right products, hoisted
        const double keu = kap * eu, kev = kap * ev, kew = kap * ew;
        // the three distinct LLF wave speeds of the face (solver.hpp:555-566;
        // the convective one serves every species and shear field), by the
        // warps with the fewest projection vectors
        // work split of (a): 2W vectors over NC warps; the warps with one
        // vector fewer take the three LLF speeds
        const int rot = (warp + 3) % NC;
        // the warps with one vector fewer (rot >= REM) take the three LLF
        // speed kinds (0: un - c, 1: un, 2: un + c), two each if fewer than 3
        constexpr int REM = NV % NC, NFEW = REM == 0 ? NC : NC - REM;
        for (int kind = rot - REM; !S.bad[face] && kind >= 0 && kind < 3; kind += NFEW) {
            const double es = S.E[F3S][face];
            double alpha = 0.0;
#pragma unroll
            for (int k = 0; k < W; ++k) {
                const int t = tile_node3<NS, DIR, W>(g, lane, k, L0);
                const double unk =
                    DIR < 2 ? n1 * S.vel[0][t] + n2 * S.vel[DIR < 2][t] : n3 * S.vel[0][t];
                const double ck = S.c[t];
                // kind is warp-uniform: the selects pick one expression
                const double lam = kind == 0 ? es * (unk + -1.0 * ck)
                                 : kind == 2 ? es * (unk + ck) : es * unk;
                alpha = smax(alpha, fabs(lam));
            }
            S.alpha[kind][lane] = alpha;
        }
        // (a) also projects: vector vec's value in every characteristic field,
        // so every warp's (b) below is the same split + reconstruction work.
        // acoustic w = (dp -+ c dun) / (2c^2), written as dp + s*(c dun) with
        // s = -+1 (exact negation); species w = q_s - Y_s dp / c^2; shear
        // w = dut1, dut2.  One validity flag per vector (exact redo if unset).
        const double ec = S.E[F3C][face];
        const double c2 = S.E[F3C2][face], yc2 = S.E[F3YC2][face];
        // 2c^2 and RN(1/(2c^2)) = RN(1/c^2)/2: scaling by 2 is exact
        const double c2x2 = 2.0 * c2, y2c2 = 0.5 * yc2;
        const unsigned den_bad =
            (fdiv_pos_divisor_ok(c2) && fdiv_pos_divisor_ok(c2x2)) ? 0u : 1u;
        // fixed trip count (the warp's 2-3 vectors): unrolled, the vectors'
        // independent chains interleave
#pragma unroll
        for (int it = 0; it < (NV + NC - 1) / NC; ++it) {
            const int vec = rot + it * NC;
            if (!live || vec >= NV) continue;
            const int k = vec >> 1;
            const int t = tile_node3<NS, DIR, W>(g, lane, k, L0);
            double q[NC];
#pragma unroll
            for (int c = 0; c < NC; ++c) q[c] = (vec & 1) ? S.U[c][t] : S.F[c][t];
            double drho = 0.0;
#pragma unroll
            for (int sp = 0; sp < NS; ++sp) drho += q[sp];
            double dp = kap * q[NS + 3] - keu * q[NS] - kev * q[NS + 1] - kew * q[NS + 2];
#pragma unroll
            for (int sp = 0; sp < NS; ++sp) dp += S.E[F3Y0 + NS + sp][face] * q[sp];
            double dun, dut1, dut2;
            if (DIR < 2) {
                dun = n1 * q[NS] + n2 * q[NS + 1] - un * drho;
                dut1 = -n2 * q[NS] + n1 * q[NS + 1] - ut1 * drho;
                dut2 = q[NS + 2] - ut2 * drho;
            } else {
                dun = n3 * q[NS + 2] - un * drho;
                dut1 = q[NS] - ut1 * drho;
                dut2 = q[NS + 1] - ut2 * drho;
            }
            unsigned bad = den_bad;
            const double cdun = ec * dun;
            double wv[NC];
            wv[0] = fdiv_pos_try(dp + -1.0 * cdun, c2x2, y2c2, bad);
            wv[NC - 1] = fdiv_pos_try(dp + 1.0 * cdun, c2x2, y2c2, bad);
#pragma unroll
            for (int sp = 0; sp < NS; ++sp)
                wv[1 + sp] = q[sp] - fdiv_pos_try(S.E[F3Y0 + sp][face] * dp, c2, yc2, bad);
            if (bad) {  // exact redo (rare): plain IEEE quotients
                wv[0] = div_cold(dp + -1.0 * cdun, c2x2);
                wv[NC - 1] = div_cold(dp + 1.0 * cdun, c2x2);
#pragma unroll
                for (int sp = 0; sp < NS; ++sp)
                    wv[1 + sp] = q[sp] - div_cold(S.E[F3Y0 + sp][face] * dp, c2);
            }
            wv[NC - 3] = dut1;
            wv[NC - 2] = dut2;
#pragma unroll
            for (int c = 0; c < NC; ++c) S.Wc[vec][c][lane] = wv[c];
        }
        __syncthreads();
        // (b) field fl: wave speed, LLF split, reconstruction
        double amp = 0.0;
        if (live) {
            double lf[W], lu[W];
#pragma unroll
            for (int k = 0; k < W; ++k) {
                lf[k] = S.Wc[2 * k][fl][lane];
                lu[k] = S.Wc[2 * k + 1][fl][lane];
            }
            const double alpha = S.alpha[fl == 0 ? 0 : fl == NC - 1 ? 2 : 1][lane];
            if (!isfinite(alpha)) {
                report(P.err, stage, phase, err_index(f, col), 1, step);
            } else {
                double wp[W], wm[W];
#pragma unroll
                for (int k = 0; k < W; ++k) {
                    wp[k] = 0.5 * (lf[k] + alpha * lu[k]);
                    wm[k] = 0.5 * (lf[k] - alpha * lu[k]);
                }
                amp = face_pm<TENO>(wp, wm, P.rp);
            }
        }
        S.amp[fl][lane] = amp;
        __syncthreads();
    }
    if (CHAR) assemble_group(NC - 1);
}

template <int NS, int DIR, bool TENO, bool CHAR, int TM>
inline int launch_faces3d_tm(const KParams& P, const double* Ut, int stage, int step,
                           cudaStream_t s, int f_lo = 0, int f_hi = -1) {
    constexpr int NC = NS + 4;
    const size_t smem = sizeof(FaceSmem3<NS, DIR, TENO, CHAR>);
    auto kern = k_faces3d<NS, DIR, TENO, CHAR, TM>;
    static std::atomic<unsigned long long> configured{0};  // per instantiation, per device
    configure_kernel(kern, smem, NC, configured, "k_faces3d");
    const int NF = 32 * NC;
    if (f_hi < 0) f_hi = (DIR == 0 ? P.nx : DIR == 1 ? P.ny : P.nz) + 1;
    if (f_hi <= f_lo) return 0;
    dim3 grid;
    if (DIR == 0) {
        if (P.nx + 1 >= NF)  // flattened rows: (nx+1) ny nz faces in runs of NF
            grid = dim3((unsigned)(((long long)(P.nx + 1) * P.ny * P.nz + NF - 1) / NF), 1, 1);
        else
            grid = dim3((P.nx + 1 + NF - 1) / NF, P.ny, P.nz);
    }
    else {
        constexpr int TW = FaceSmem3<NS, DIR, TENO, CHAR>::TW, LN = NF / TW;
        if (DIR == 1) grid = dim3((P.nx + TW - 1) / TW, (f_hi - f_lo + LN - 1) / LN, P.nz);
        else grid = dim3((P.nx + TW - 1) / TW, P.ny, (f_hi - f_lo + LN - 1) / LN);
    }
    kern<<<grid, 32 * NC, smem, s>>>(P, Ut, stage, step, f_lo, f_hi);
    return 1;
}

// thermo mode of the Roe/eigen thermo (physics.cuh sp_h_R): a calorically
// perfect single-species mixture (the gamma-gas) or an all-lin2 mixture (every
// table in data/ and the reference's ch4_o2.mix) takes the instantiation with
// only those forms compiled in
template <int NS, int DIR, bool TENO, bool CHAR>
inline int launch_faces3d(const KParams& P, const double* Ut, int stage, int step, cudaStream_t s,
                          int f_lo = 0, int f_hi = -1) {
    if constexpr (NS == 1) {
        if (P.mix.all_simple)
            return launch_faces3d_tm<NS, DIR, TENO, CHAR, 1>(P, Ut, stage, step, s, f_lo, f_hi);
    } else {
        if (P.mix.all_lin2)
            return launch_faces3d_tm<NS, DIR, TENO, CHAR, 2>(P, Ut, stage, step, s, f_lo, f_hi);
    }
    return launch_faces3d_tm<NS, DIR, TENO, CHAR, 0>(P, Ut, stage, step, s, f_lo, f_hi);
}

}  // namespace ign
