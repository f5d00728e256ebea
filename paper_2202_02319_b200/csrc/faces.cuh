// faces.cuh — inviscid face fluxes (solver.hpp:441-579), B200 layout.
//
// One CTA of NC = ns+3 warps owns G = NC groups of 32 faces (x faces: 32*NC
// consecutive faces of one row; y faces: 32 columns x NC consecutive face
// rows).  Work is spread so every warp stays busy between barriers:
//
//   phase 1  all threads  stage the node window in shared memory: U = Ut*J,
//                         the mapped flux m1 F + m2 G (solver.hpp:466-479,
//                         flux.hpp:39-50) and cached u, v, c — each node's
//                         mapped flux is computed once per CTA;
//                         thread t: Roe average + eigensystem of face t
//                         (solver.hpp:493-502) into shared memory.
//   phase 2  per group g  (a) warp w: the field-independent parts of L q
//                         (drho, dp, dun, dut; flux.hpp:107-114) for stencil
//                         vectors w, w+NC, ...; (b) warp w = field w: row w of
//                         L F, L U on the 2h nodes, alpha_w, the LLF split and
//                         the two TENO6/WENO3Z reconstructions (:516-534).
//   phase 3  per group g  warp w: component w of R*amp (flux.hpp:123-139) and
//                         a coalesced store.
//
// Every value is produced by the reference's own operation sequence.
#pragma once

#include <cstdio>
#include <cstdlib>

#include <type_traits>

#include "flux.cuh"
#include "kernels_common.cuh"

namespace ign {

// y tile width (columns): see FaceSmem::TW.  One species: 8 columns (the
// window's halo rows shrink, one more CTA fits per SM); several: 32 (those
// CTAs are held at 2 CTAs/SM, and the wider tile keeps the launch in whole
// waves at 512^2)
template <int NS, int DIR> __host__ __device__ constexpr int tile_w() {
    return DIR == 0 || NS > 1 ? 32 : 8;
}

// CHAR = false (componentwise) needs only the node window and one LLF speed
// per face: the characteristic tables shrink to one row so more CTAs fit
template <int NS, int DIR, bool TENO, bool CHAR = true> struct FaceSmem {
    static constexpr int NC = NS + 3;
    static constexpr int H = TENO ? 3 : 2;
    static constexpr int W = 2 * H;
    // groups of 32 faces per CTA: one per warp, except the x faces of
    // multi-species tables (NC >= 6), whose CTA of NC warps owns 5 groups —
    // the eigen table and window shrink so 3 CTAs/SM fit (phase 1 leaves the
    // extra threads idle): H2/O2 x faces -5% (the y faces, held by their
    // 32-column window, stay at NC groups and 2 CTAs/SM)
    static constexpr int G = (NC >= 6 && DIR == 0) ? 5 : NC;
    static constexpr int NTH = 32 * NC;  // threads
    static constexpr int NF = 32 * G;    // faces per CTA
    // y tiles: TW columns x NF/TW face rows (few halo rows in the window)
    static constexpr int TW = tile_w<NS, DIR>();
    static constexpr int LINES = NF / TW;
    // x: up to two row segments of the flattened face order (see k_faces3)
    static constexpr int NT = DIR == 0 ? NF + 2 * (W - 1) : TW * (LINES + W - 1);
    static constexpr int NE_CHAR = 11 + 2 * NS;
    static constexpr int NE = CHAR ? NE_CHAR : 1;
    static constexpr int NV = 2 * W;  // stencil vectors: F and U of each node
    static constexpr int NV_S = CHAR ? NV : 1;   // projection table rows
    static constexpr int NA_S = CHAR ? NC : 1;   // amplitude table rows
    static constexpr int NK_S = CHAR ? 3 : 1;    // LLF speed kinds
    double U[NC][NT];
    double F[NC][NT];
    double u[NT], v[NT], c[NT];
    double E[NE][NF];         // eigen data per face (char); [0] alpha, [1] sf (comp)
    // characteristic values of one group's stencil vectors, every field: row
    // fl of L F and L U (EigenSystem::project, flux.hpp:107-119)
    double Wc[NV_S][NA_S][32];
    double amp[NA_S][32];  // one group (phase 3 follows each group)
    double alpha[NK_S][32];  // per face of the group: LLF speeds of acoustic-, convective, acoustic+
    unsigned char bad[NF];
};

// Eigen data slots in FaceSmem::E
enum : int {
    EN1 = 0, EN2, ES, EU, EV, EH, EC, EC2, EKAPPA, EYC2, EYKAPPA,
    EY0  // then Y[NS], Theta[NS]; un, ut and k are recomputed (eigen_un etc.)
};

// EigenSystem::at_state's un, ut and k (flux.hpp:72-104, flux.cuh), the same
// operations on the stored normal and velocity
template <class Sm> __device__ __forceinline__ double eigen_un(const Sm& S, int f) {
    return S.E[EN1][f] * S.E[EU][f] + S.E[EN2][f] * S.E[EV][f];
}
template <class Sm> __device__ __forceinline__ double eigen_ut(const Sm& S, int f) {
    return -S.E[EN2][f] * S.E[EU][f] + S.E[EN1][f] * S.E[EV][f];
}
template <class Sm> __device__ __forceinline__ double eigen_k(const Sm& S, int f) {
    return 0.5 * (S.E[EU][f] * S.E[EU][f] + S.E[EV][f] * S.E[EV][f]);
}

// window slot of stencil node k of face slot q = 32 g + lane; x faces past the
// first row segment (q >= L0) sit W-1 slots further (their segment's own
// halo); y: slot q is column q % TW of face row q / TW, its node k lies k rows
// further
template <int NS, int DIR, int W>
__device__ __forceinline__ int tile_node(int g, int lane, int k, int L0) {
    const int q = g * 32 + lane;
    if (DIR == 0) return q + k + (q >= L0 ? W - 1 : 0);
    return q + k * tile_w<NS, DIR>();
}

template <int NS, int DIR, bool TENO, bool CHAR, int TM>
#ifndef IGN_FACES_MINB
#define IGN_FACES_MINB 4
#endif
__global__ void __launch_bounds__(32 * (NS + 3),
                                  (NS == 1 ? IGN_FACES_MINB : (NS >= 3 && DIR == 0) ? 3 : 1))
k_faces3(const __grid_constant__ KParams P, const double* __restrict__ Ut, int stage, int step,
         int f_lo, int f_hi) {
    using Smem = FaceSmem<NS, DIR, TENO, CHAR>;
    constexpr int NC = Smem::NC, H = Smem::H, W = Smem::W, NF = Smem::NF, NT = Smem::NT;
    constexpr int G = Smem::G, NTH = Smem::NTH;
    constexpr int NV = Smem::NV;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& S = *reinterpret_cast<Smem*>(smem_raw);
    // an earlier failure (error word set) ends the kernel after phase 1: the
    // load's latency hides behind the window staging (garbage phase-1 reports
    // carry larger keys than the first one)
    __shared__ int s_dead;
    const bool dead0 =
        threadIdx.x == 0 && failed_before(P.err, step, stage, DIR == 0 ? PH_INVX : PH_INVY);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long step_n = DIR == 0 ? 1 : P.sx;
    const double* m1a = DIR == 0 ? P.mxx : P.mex;
    const double* m2a = DIR == 0 ? P.mxy : P.mey;
    // x: NF consecutive faces of the flattened (row j, face f) order — at most
    // two row segments when nx+1 >= NF, else one row segment per CTA;
    // y: columns i0 .. i0+31, face rows f0 .. f0+NC-1
    int f0, r0 = 0, L0 = NF;
    if (DIR == 0) {
        if (P.nx + 1 >= NF) {
            const long long F0 = (long long)blockIdx.x * NF;
            r0 = (int)(F0 / (P.nx + 1));
            f0 = (int)(F0 % (P.nx + 1));
            L0 = min(NF, P.nx + 1 - f0);
        } else {
            r0 = blockIdx.y;
            f0 = blockIdx.x * NF;
        }
    } else {
        // y faces [f_lo, f_hi) of the line (a slab splits interior and halo faces)
        f0 = f_lo + blockIdx.y * Smem::LINES;
    }
    constexpr int TW = Smem::TW;
    const int i0 = blockIdx.x * TW;
    const long long win0 = DIR == 0 ? 0 : pidx(P, i0, f0 - H);
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

    // ---------------- phase 1a: node window -> shared memory
    if constexpr (CHAR) {
        // ---------------- phase 1a: node window -> shared memory.  Each thread
        // stages NIT nodes (NIT = ceil(NT / NTH)); every node's loads are issued
        // before any is consumed, so their latencies overlap
        constexpr int NIT = (NT + NTH - 1) / NTH;
        double raw[NIT][NC + 7];
        int slot_t[NIT];
    #pragma unroll
        for (int it = 0; it < NIT; ++it) {
            const int t = threadIdx.x + it * NTH;
            long long id = 0;
            bool ok = t < NT;
            if (DIR == 0) {
                const int n0 = L0 + W - 1;  // window slots of the first segment
                int a, row;
                if (t < n0) {
                    a = f0 - H + t;
                    row = r0;
                } else {
                    a = -H + (t - n0);
                    row = r0 + 1;
                }
                id = pidx(P, a, row);
                ok = ok && a < P.nx + P.g && row < P.ny && (t < n0 || t - n0 < NF - L0 + W - 1);
            } else {
                const int r = t / TW, l = t % TW;
                id = win0 + (long long)r * P.sx + l;
                ok = ok && i0 + l < P.nx && f0 - H + r < P.ny + P.g;
            }
            slot_t[it] = ok ? t : -1;
            if (!ok) continue;
            double* q = raw[it];
    #pragma unroll
            for (int c = 0; c < NC; ++c) q[c] = ldg(Ut + c * P.plane + id);
            q[NC] = ldg(P.jac + id);
            q[NC + 1] = ldg(PU(P) + id);
            q[NC + 2] = ldg(PV(P) + id);
            q[NC + 3] = ldg(PP(P) + id);
            q[NC + 4] = ldg(m1a + id);
            q[NC + 5] = ldg(m2a + id);
            q[NC + 6] = ldg(PC(P) + id);
        }
    #pragma unroll
        for (int it = 0; it < NIT; ++it) {
            const int t = slot_t[it];
            if (t < 0) continue;
            const double* q = raw[it];
            const double J = q[NC];
            double Uk[NC], Fk[NC];
    #pragma unroll
            for (int c = 0; c < NC; ++c) Uk[c] = q[c] * J;
            const double nu = q[NC + 1], nv = q[NC + 2];
            mapped_flux_uv<NS>(Uk, q[NC + 3], nu, nv, q[NC + 4], q[NC + 5], Fk);
    #pragma unroll
            for (int c = 0; c < NC; ++c) {
                S.U[c][t] = Uk[c];
                S.F[c][t] = Fk[c];
            }
            S.u[t] = nu;
            S.v[t] = nv;
            S.c[t] = q[NC + 6];
        }
    } else {  // componentwise: the plain loop (hoisting costs it occupancy)
        for (int t = threadIdx.x; t < NT; t += blockDim.x) {
            long long id;
            bool ok;
            if (DIR == 0) {
                const int n0 = L0 + W - 1;  // window slots of the first segment
                int a, row;
                if (t < n0) {
                    a = f0 - H + t;
                    row = r0;
                } else {
                    a = -H + (t - n0);
                    row = r0 + 1;
                }
                id = pidx(P, a, row);
                ok = a < P.nx + P.g && row < P.ny && (t < n0 || t - n0 < NF - L0 + W - 1);
            } else {
                const int r = t / TW, l = t % TW;
                id = win0 + (long long)r * P.sx + l;
                ok = i0 + l < P.nx && f0 - H + r < P.ny + P.g;
            }
            if (!ok) continue;
            const double J = ldg(P.jac + id);
            double Uk[NC], Fk[NC];
    #pragma unroll
            for (int c = 0; c < NC; ++c) Uk[c] = ldg(Ut + c * P.plane + id) * J;
            const double nu = ldg(PU(P) + id), nv = ldg(PV(P) + id);
            mapped_flux_uv<NS>(Uk, ldg(PP(P) + id), nu, nv, ldg(m1a + id), ldg(m2a + id), Fk);
    #pragma unroll
            for (int c = 0; c < NC; ++c) {
                S.U[c][t] = Uk[c];
                S.F[c][t] = Fk[c];
            }
            S.u[t] = nu;
            S.v[t] = nv;
            S.c[t] = ldg(PC(P) + id);
        }
    }

    // this thread's face in phase 1b: group = warp, lane
    int my_f, my_col;  // face index along the line; row (x) / column (y)
    if (DIR == 0) {
        xface(threadIdx.x, my_col, my_f);
    } else {
        my_f = f0 + (int)threadIdx.x / TW;
        my_col = i0 + (int)threadIdx.x % TW;
    }
    const bool my_slot = threadIdx.x < NF;  // the thread owns a face in phase 1
    const bool my_active = my_slot && (DIR == 0 ? (my_f <= P.nx && my_col < P.ny)
                                                : (my_col < P.nx && my_f < f_hi));
    const unsigned phase = DIR == 0 ? PH_INVX : PH_INVY;
    auto err_index = [&](int f, int col) -> unsigned long long {
        // global (line, face) order of inviscid_direction (solver.hpp:450-481)
        return DIR == 0 ? (unsigned long long)(col + P.j0) * (P.nx + 1) + f
                        : (unsigned long long)col * (P.ny_glob + 1) + (f + P.j0);
    };
    // face metric (solver.hpp:484-489): mean of the two node metrics
    const long long il = DIR == 0 ? pidx(P, my_f - 1, my_col) : pidx(P, my_col, my_f - 1);
    const long long ir = il + step_n;
    double m1f = 0.0, m2f = 0.0;
    if (my_active) {
        m1f = 0.5 * (ldg(m1a + il) + ldg(m1a + ir));
        m2f = 0.5 * (ldg(m2a + il) + ldg(m2a + ir));
    }

    // ---------------- phase 1b (char): Roe average + eigensystem of my face
    if (CHAR) {
        int bad = 0;
        if (my_active) {
            double Yl[NS], Yr[NS], Ya[NS];
#pragma unroll
            for (int s = 0; s < NS; ++s) {
                Yl[s] = ldg(PY(P, s) + il);
                Yr[s] = ldg(PY(P, s) + ir);
            }
            double Ta, ua, va;
            roe_average<NS, TM>(ldg(PRHO(P) + il), Yl, ldg(PT(P) + il), ldg(PU(P) + il),
                            ldg(PV(P) + il), ldg(PRHO(P) + ir), Yr, ldg(PT(P) + ir),
                            ldg(PU(P) + ir), ldg(PV(P) + ir), P.mix, Ya, Ta, ua, va);
            Eigen<NS> es;
            const int est = eigen_at_state<NS, TM>(Ya, Ta, ua, va, m1f, m2f, P.mix, es);
            if (est) {
                report(P.err, stage, phase, err_index(my_f, my_col), 1 + est, step);
                bad = 1;
            }
            const int t = threadIdx.x;
            S.E[EN1][t] = es.n1;
            S.E[EN2][t] = es.n2;
            S.E[ES][t] = es.s;
            S.E[EU][t] = es.u;
            S.E[EV][t] = es.v;
            S.E[EH][t] = es.H;
            S.E[EC][t] = es.c;
            S.E[EC2][t] = es.c2;
            S.E[EKAPPA][t] = es.kappa;
            S.E[EYC2][t] = es.yc2;
            S.E[EYKAPPA][t] = es.ykappa;
#pragma unroll
            for (int s = 0; s < NS; ++s) {
                S.E[EY0 + s][t] = es.Y[s];
                S.E[EY0 + NS + s][t] = es.Theta[s];
            }
        }
        if (my_slot) S.bad[threadIdx.x] = my_active ? bad : 1;
    }
    if (threadIdx.x == 0) s_dead = dead0;
    __syncthreads();
    if (s_dead) return;
    if (!CHAR) {
        // ---------------- phase 1b (comp): LLF wave speed of my face (solver.hpp:537-548)
        int bad = 1;
        if (my_active) {
            const double sf = ghypot(m1f, m2f);
            double alpha = 0.0;
#pragma unroll
            for (int k = 0; k < W; ++k) {
                const int t = tile_node<NS, DIR, W>(warp, lane, k, L0);
                const double un = (m1f * S.u[t] + m2f * S.v[t]) / sf;
                alpha = smax(alpha, sf * (fabs(un) + S.c[t]));
            }
            bad = 0;
            if (!isfinite(alpha)) {
                report(P.err, stage, phase, err_index(my_f, my_col), 1, step);
                bad = 1;
            }
            S.E[0][threadIdx.x] = alpha;
        }
        if (my_slot) S.bad[threadIdx.x] = bad;
        __syncthreads();
    }

    double* out = DIR == 0 ? P.Fx : P.Gy;
    const long long fplane = (long long)(P.nx + 1 - DIR) * (P.ny + DIR);
    const int fl = warp;  // field / component this warp evaluates
    // face slot q = 32 g + lane -> (face index along the line, row / column)
    auto slot_face = [&](int q, int& f, int& col) {
        if (DIR == 0) {
            xface(q, col, f);
        } else {
            f = f0 + q / TW;
            col = i0 + q % TW;
        }
    };
    auto out_at = [&](int f, int col) -> long long {
        return DIR == 0 ? (long long)col * (P.nx + 1) + f : (long long)f * P.nx + col;
    };
    if constexpr (!CHAR) {
        // componentwise: component fl of the LLF-split TENO sum
        for (int g = 0; g < G; ++g) {
            const int face = g * 32 + lane;
            if (S.bad[face]) continue;
            int f, col;
            slot_face(face, f, col);
            const double alpha = S.E[0][face];
            double wp[W], wm[W];
#pragma unroll
            for (int k = 0; k < W; ++k) {
                const int t = tile_node<NS, DIR, W>(g, lane, k, L0);
                wp[k] = 0.5 * (S.F[fl][t] + alpha * S.U[fl][t]);
                wm[k] = 0.5 * (S.F[fl][t] - alpha * S.U[fl][t]);
            }
            out[fl * fplane + out_at(f, col)] = face_pm<TENO>(wp, wm, P.rp);
        }
        return;
    }
    // ---------------- phase 3: component fl of R * amp of group g
    // (flux.hpp:123-139), run while the next group's vectors are built: the
    // amplitude table holds one group
    auto assemble_group = [&](int g) {
        const int face = g * 32 + lane;
        if (S.bad[face]) return;
        int f, col;
        slot_face(face, f, col);
        const double am = S.amp[0][lane];
        const double ap = S.amp[2 + NS][lane];
        const double at = S.amp[1 + NS][lane];
        const double c = S.E[EC][face];
        double r;
        if (fl < NS) {
            r = S.E[EY0 + fl][face] * (am + ap) + S.amp[1 + fl][lane];
        } else {
            double asum = 0.0;
#pragma unroll
            for (int sp = 0; sp < NS; ++sp) asum += S.amp[1 + sp][lane];
            if (fl == NS) {
                const double u = S.E[EU][face], n1 = S.E[EN1][face], n2 = S.E[EN2][face];
                r = (u - c * n1) * am + (u + c * n1) * ap + u * asum - n2 * at;
            } else if (fl == NS + 1) {
                const double v = S.E[EV][face], n1 = S.E[EN1][face], n2 = S.E[EN2][face];
                r = (v - c * n2) * am + (v + c * n2) * ap + v * asum + n1 * at;
            } else {
                const double Hh = S.E[EH][face], un = eigen_un(S, face), ut = eigen_ut(S, face);
                const double kk = eigen_k(S, face), kappa = S.E[EKAPPA][face];
                const double ykappa = S.E[EYKAPPA][face];
                double en = (Hh - c * un) * am + (Hh + c * un) * ap + ut * at;
#pragma unroll
                for (int sp = 0; sp < NS; ++sp) {
                    const double th = S.E[EY0 + NS + sp][face];
                    en += S.amp[1 + sp][lane] * (2.0 * kk - fdiv(th, kappa, ykappa));
                }
                r = en;
            }
        }
        out[fl * fplane + out_at(f, col)] = r;
    };
    for (int g = 0; g < G; ++g) {
        if (g > 0) assemble_group(g - 1);
        const int face = g * 32 + lane;  // slot in the CTA
        const bool live = !S.bad[face];
        int f, col;
        slot_face(face, f, col);
        // (a) L q for this group's stencil vectors (flux.hpp:107-119): the
        // field-independent parts and every field's projection row, so each
        // warp's (b) is the same split + reconstruction work.  acoustic
        // w = (dp -+ c dun) / (2c^2), written as dp + s*(c dun) with s = -+1
        // (exact negation); species w = q_s - Y_s dp / c^2; shear w = dut.
        // One validity flag per vector (exact redo if unset).
        const double kap = S.E[EKAPPA][face], eu = S.E[EU][face], ev = S.E[EV][face];
        const double n1 = S.E[EN1][face], n2 = S.E[EN2][face];
        const double un = eigen_un(S, face), ut = eigen_ut(S, face);
        // (kap eu) q_u: the reference's left-to-right products, hoisted
        const double keu = kap * eu, kev = kap * ev;
        // the three distinct LLF wave speeds of the face (EigenSystem::field_speed,
        // flux.hpp:143-147; the convective one serves species and shear fields)
        // by the warps with one vector fewer
        const int rot = (warp + 2) % NC;
        // the warps with one vector fewer (rot >= REM) take the three LLF
        // speed kinds (0: un - c, 1: un, 2: un + c), two each if fewer than 3
        constexpr int REM = NV % NC, NFEW = REM == 0 ? NC : NC - REM;
        for (int kind = rot - REM; live && kind >= 0 && kind < 3; kind += NFEW) {
            const double es = S.E[ES][face];
            double alpha = 0.0;
#pragma unroll
            for (int k = 0; k < W; ++k) {
                const int t = tile_node<NS, DIR, W>(g, lane, k, L0);
                const double unk = n1 * S.u[t] + n2 * S.v[t];
                const double ck = S.c[t];
                // kind is warp-uniform: the selects pick one expression
                const double lam = kind == 0 ? es * (unk + -1.0 * ck)
                                 : kind == 2 ? es * (unk + ck) : es * unk;
                alpha = smax(alpha, fabs(lam));
            }
            S.alpha[kind][lane] = alpha;
        }
        const double ec = S.E[EC][face];
        const double c2 = S.E[EC2][face], yc2 = S.E[EYC2][face];
        // 2c^2 and RN(1/(2c^2)) = RN(1/c^2)/2: scaling by 2 is exact
        const double c2x2 = 2.0 * c2, y2c2 = 0.5 * yc2;
        const unsigned den_bad = (fdiv_pos_divisor_ok(c2) && fdiv_pos_divisor_ok(c2x2)) ? 0u : 1u;
        // the vectors of this warp: unrolled for one species (a fixed trip
        // count, the vectors' independent chains interleave: TGV 2D +1%); the
        // register-bound multi-species kernels keep the rolled loop (-4%
        // unrolled)
        auto build_vector = [&](int vec) {
            const int k = vec >> 1;
            const int t = tile_node<NS, DIR, W>(g, lane, k, L0);
            double q[NC];
#pragma unroll
            for (int c = 0; c < NC; ++c) q[c] = (vec & 1) ? S.U[c][t] : S.F[c][t];
            double drho = 0.0;
#pragma unroll
            for (int sp = 0; sp < NS; ++sp) drho += q[sp];
            double dp = kap * q[NS + 2] - keu * q[NS] - kev * q[NS + 1];
#pragma unroll
            for (int sp = 0; sp < NS; ++sp) dp += S.E[EY0 + NS + sp][face] * q[sp];
            const double dun = n1 * q[NS] + n2 * q[NS + 1] - un * drho;
            const double dut = -n2 * q[NS] + n1 * q[NS + 1] - ut * drho;
            unsigned bad = den_bad;
            const double cdun = ec * dun;
            double wv[NC];
            wv[0] = fdiv_pos_try(dp + -1.0 * cdun, c2x2, y2c2, bad);
            wv[NC - 1] = fdiv_pos_try(dp + 1.0 * cdun, c2x2, y2c2, bad);
#pragma unroll
            for (int sp = 0; sp < NS; ++sp)
                wv[1 + sp] = q[sp] - fdiv_pos_try(S.E[EY0 + sp][face] * dp, c2, yc2, bad);
            if (bad) {  // exact redo (rare): plain IEEE quotients
                wv[0] = div_cold(dp + -1.0 * cdun, c2x2);
                wv[NC - 1] = div_cold(dp + 1.0 * cdun, c2x2);
#pragma unroll
                for (int sp = 0; sp < NS; ++sp)
                    wv[1 + sp] = q[sp] - div_cold(S.E[EY0 + sp][face] * dp, c2);
            }
            wv[NC - 2] = dut;
#pragma unroll
            for (int c = 0; c < NC; ++c) S.Wc[vec][c][lane] = wv[c];
        };
        if constexpr (NS == 1) {
#pragma unroll
            for (int it = 0; it < (NV + NC - 1) / NC; ++it) {
                const int vec = rot + it * NC;
                if (live && vec < NV) build_vector(vec);
            }
        } else {
            for (int vec = live ? rot : NV; vec < NV; vec += NC) build_vector(vec);
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
            // EigenSystem::field_speed (flux.hpp:143-147), computed once per kind
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
        __syncthreads();  // amp complete; Wc may be overwritten by the next group
    }
    assemble_group(G - 1);
}

template <int NS, int DIR, bool TENO, bool CHAR, int TM>
inline int launch_faces3_tm(const KParams& P, const double* Ut, int stage, int step,
                          cudaStream_t s, int f_lo = 0, int f_hi = -1) {
    constexpr int NC = NS + 3;
    const size_t smem = sizeof(FaceSmem<NS, DIR, TENO, CHAR>);
    auto kern = k_faces3<NS, DIR, TENO, CHAR, TM>;
    static std::atomic<unsigned long long> configured{0};  // per instantiation, per device
    configure_kernel(kern, smem, NC, configured, "k_faces3");
    const int NF = FaceSmem<NS, DIR, TENO, CHAR>::NF;
    if (f_hi < 0) f_hi = (DIR == 0 ? P.nx : P.ny) + 1;
    if (f_hi <= f_lo) return 0;
    dim3 grid;
    if (DIR == 0)
        grid = P.nx + 1 >= NF  // flattened rows: (nx+1) ny faces in runs of NF
                   ? dim3((unsigned)(((long long)(P.nx + 1) * P.ny + NF - 1) / NF), 1)
                   : dim3((P.nx + 1 + NF - 1) / NF, P.ny);
    else {
        constexpr int TW = FaceSmem<NS, DIR, TENO, CHAR>::TW, LN = NF / TW;
        grid = dim3((P.nx + TW - 1) / TW, (f_hi - f_lo + LN - 1) / LN);
    }
    kern<<<grid, 32 * NC, smem, s>>>(P, Ut, stage, step, f_lo, f_hi);
    return 1;
}

// thermo mode of the Roe/eigen thermo (physics.cuh sp_h_R): a calorically
// perfect single-species mixture (the gamma-gas) or an all-lin2 mixture (every
// table in data/ and the reference's ch4_o2.mix) takes the instantiation with
// only those forms compiled in
template <int NS, int DIR, bool TENO, bool CHAR>
inline int launch_faces3(const KParams& P, const double* Ut, int stage, int step, cudaStream_t s,
                          int f_lo = 0, int f_hi = -1) {
    if constexpr (NS == 1) {
        if (P.mix.all_simple)
            return launch_faces3_tm<NS, DIR, TENO, CHAR, 1>(P, Ut, stage, step, s, f_lo, f_hi);
    } else {
        if (P.mix.all_lin2)
            return launch_faces3_tm<NS, DIR, TENO, CHAR, 2>(P, Ut, stage, step, s, f_lo, f_hi);
    }
    return launch_faces3_tm<NS, DIR, TENO, CHAR, 0>(P, Ut, stage, step, s, f_lo, f_hi);
}

}  // namespace ign
