// kernels_common.cuh — shared device plumbing of the stage kernels: the device
// error word (first failure in the reference's own order) and the kernel
// parameter block (mixture, mechanism, laser, BC data and array pointers).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "physics.cuh"

namespace ign {

// ---------------------------------------------------------------- errors
// Device error word: the first failure in the reference's own order wins via
// atomicMin on
//   key = step<<44 | stage<<41 | phase<<38 | index<<3 | sub
// (step within the current batch, 20 bits; index = GLOBAL row-major position,
// 35 bits), so slabs of a decomposed domain agree on one first failure after
// a MIN all-reduce of the word.
enum Phase : unsigned {
    PH_BC = 1,     // StateError from fill_ghosts' prim_at (boundary.hpp:151-156)
    PH_PRIM = 2,   // StepFailure "stage state failure" (solver.hpp:162-165)
    PH_INVX = 3,   // NumericsError from inviscid x faces (solver.hpp:522-524, flux.hpp:78,99)
    PH_INVY = 4,
    PH_RHS = 5,    // StepFailure "non-finite RHS" (solver.hpp:225-228)
    PH_POST = 6,   // StepFailure post_stage (solver.hpp:840-844)
};
constexpr unsigned long long kNoError = ~0ull;

struct ErrRec {
    unsigned long long key;
};

__device__ __forceinline__ bool failed(const ErrRec* e) {
    return *reinterpret_cast<const volatile unsigned long long*>(&e->key) != kNoError;
}

// A failure recorded by an EARLIER (step, stage, phase) than the caller's:
// kernels stop on those only.  A failure of their own phase must not stop
// them, or a CTA that starts after another CTA's report would miss a smaller
// key (the reference's first failure in row-major order) of the same phase.
__device__ __forceinline__ unsigned long long err_first(int step, int stage, unsigned phase) {
    return ((unsigned long long)(step & 0xFFFFF) << 44) | ((unsigned long long)stage << 41) |
           ((unsigned long long)phase << 38);
}
__device__ __forceinline__ bool failed_before(const ErrRec* e, int step, int stage,
                                              unsigned phase) {
    return *reinterpret_cast<const volatile unsigned long long*>(&e->key) <
           err_first(step, stage, phase);
}
// A snapshot of the word (L2, not L1: other CTAs report into it) whose
// comparison can be deferred past other work — the face kernels compare it
// after their window staging, so its latency is hidden
__device__ __forceinline__ unsigned long long err_key(const ErrRec* e) {
    return __ldcg(&e->key);
}

__device__ __forceinline__ void report(ErrRec* e, unsigned stage, unsigned phase,
                                       unsigned long long idx, unsigned sub, int step) {
    const unsigned long long key = ((unsigned long long)(step & 0xFFFFF) << 44) |
                                   ((unsigned long long)stage << 41) |
                                   ((unsigned long long)phase << 38) |
                                   ((idx & ((1ull << 35) - 1)) << 3) | (sub & 7u);
    atomicMin(&e->key, key);
}

// y-edge roles beyond the reference's BC types (boundary.hpp:16-22) for slabs
enum : int32_t { BC_HALO_WRAP = 5, BC_HALO = 6 };

// ---------------------------------------------------------------- params
struct KParams {
    int32_t nx, ny, g, sx;
    long long plane;
    int32_t j0, ny_glob;  // slab: global row of local row 0, global rows
    int32_t ns, viscous;
    int32_t bc_type[4];  // left, right, bottom, top (+ BC_HALO_WRAP / BC_HALO)
    const double* wrap[2];  // [k][t] J_src/J_dst of periodic wrap ghost rows
    double T_wall[4];
    double sigma_out_right, p_target_right;
    double lx, ly, cx, cy;
    double zc0, dz;  // 3D: z of global plane k = zc0 + (k + 0.5) dz (sim.py mesh_z)
    ReconParams rp;  // ct, eps and the TENO cutoff decision band
    int32_t chem_dt_limit, lodi;
    double chem_dt_factor;
    // primitive cache block: rho,u,v,p,T,c then Y_s, then X_s (viscous)
    double* prim;
    const double *jac, *mxx, *mxy, *mex, *mey;       // met (inviscid)
    const double *vjac, *vmxx, *vmxy, *vmex, *vmey;  // met_v (Central2)
    const double *xc, *yc;                           // mesh.x, mesh.y
    double *Fx, *Gy, *Fv, *Gv;
    // 3D extension (extruded mesh; nz = 0 for 2D): z cells, state plane
    // stride, zeta metric (2D planes), z face fluxes, viscous z fluxes
    int32_t nz, nz_glob;
    int32_t zhalo;  // 3D z-slabs: some z ghost planes come from the peers
    int32_t bc_z[2];  // 3D back / front edge: 0 periodic, 1/2 walls, 4 outflow, BC_HALO
    int32_t _pad3;
    double T_wall_z[2];
    long long sxy;
    const double *mzz, *vmzz;
    double *Hz, *Hv;
    const double* inflow[4];  // per edge [t][k][u,v,T,Y_s] profile tables
    ErrRec* err;
    unsigned long long* red;  // [0] lam_max bits, [1] dt_chem bits, [2..7] clip bits
    DMix mix;
    DMech mech;
    DLaser laser;
};

__device__ __forceinline__ long long pidx(const KParams& P, int i, int j) {
    return (long long)(j + P.g) * P.sx + (i + P.g);
}

// primitive cache planes
#define PRHO(P) ((P).prim)
#define PU(P) ((P).prim + (P).plane)
#define PV(P) ((P).prim + 2 * (P).plane)
#define PP(P) ((P).prim + 3 * (P).plane)
#define PT(P) ((P).prim + 4 * (P).plane)
#define PC(P) ((P).prim + 5 * (P).plane)
#define PY(P, s) ((P).prim + (6 + (s)) * (P).plane)
#define PX(P, s) ((P).prim + (6 + (P).ns + (s)) * (P).plane)

__device__ __forceinline__ double ldg(const double* p) { return __ldg(p); }

// Kernel attributes (>48 KB dynamic shared memory opt-in, carveout) are
// per device: each instantiation keeps one bit per device ordinal, set after
// both attribute calls succeeded on that device (thread-safe; racing threads
// at worst set the same attributes twice).  Failures throw (IGN_CUDA_ERROR at
// the ABI: runtime_error subclasses map to the context's error).
struct KernelAttrError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

template <class Kern>
inline void configure_kernel(Kern kern, size_t smem, int warps, std::atomic<unsigned long long>& mask,
                             const char* name, int carveout = cudaSharedmemCarveoutMaxShared) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) throw KernelAttrError("cudaGetDevice failed");
    const unsigned long long bit = 1ull << (dev & 63);
    if (mask.load(std::memory_order_acquire) & bit) return;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 carveout);
    if (e != cudaSuccess)
        throw KernelAttrError(std::string(name) + ": cudaFuncSetAttribute: " + cudaGetErrorString(e));
    if (std::getenv("IGN_DEBUG_OCC")) {
        int nb = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, warps * 32, smem);
        std::fprintf(stderr, "%s: smem %zu B, %d CTAs/SM (device %d)\n", name, smem, nb, dev);
    }
    mask.fetch_or(bit, std::memory_order_acq_rel);
}

}  // namespace ign

namespace ign {

// primitive cache planes of the 3D extension: rho,u,v,w,p,T,c then Y_s, X_s
#define PRHO3(P) ((P).prim)
#define PU3(P) ((P).prim + (P).plane)
#define PV3(P) ((P).prim + 2 * (P).plane)
#define PW3(P) ((P).prim + 3 * (P).plane)
#define PP3(P) ((P).prim + 4 * (P).plane)
#define PT3(P) ((P).prim + 5 * (P).plane)
#define PC3(P) ((P).prim + 6 * (P).plane)
#define PY3(P, s) ((P).prim + (7 + (s)) * (P).plane)
#define PX3(P, s) ((P).prim + (7 + (P).ns + (s)) * (P).plane)

// Compile-time thermo mode of a kernel launch (physics.cuh sp_h_R): 1 = the
// calorically perfect single-species gas, 2 = every species lin2 (multi-species
// tables), 0 = the general piece code.  Instantiations for modes a species
// count cannot take are never launched (NS == 1: 0/1; NS > 1: 0/2).
template <int NS> inline int thermo_mode(const DMix& m) {
    if (NS == 1) return m.all_simple ? 1 : 0;
    return m.all_lin2 ? 2 : 0;
}

// Launcher table of one (species count, dimension) instantiation; every entry
// returns the number of kernels it launched.
struct KernelSet {
    int (*bc)(const KParams&, double* Ut, int ypass, int stage, int step, cudaStream_t);
    // part: 0 whole box / every face; 1 what a slab computes from its own
    // rows (planes) while its halo is in flight; 2 what needs the halo
    int (*prim)(const KParams&, const double* Ut, int stage, int step, cudaStream_t, int part);
    int (*faces)(const KParams&, int teno, int chr, const double* Ut, int stage, int step,
                 cudaStream_t, int part);
    int (*visc)(const KParams&, int stage, int step, cudaStream_t);
    int (*assemble)(const KParams&, int mode, const double* U0, const double* Ucur,
                    double* Uout, double dt, double w, double t_stage, int stage, int step,
                    int clip_slot, cudaStream_t);
    int (*dt)(const KParams&, cudaStream_t);
};

}  // namespace ign
