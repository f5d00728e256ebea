// context_internal.hpp — internals shared by the host runtime of the C ABI:
// the context and group objects, and the declarations of the stage
// orchestration (runtime.cu), outputs (outputs.cu) and setup (setup.cu).
#pragma once

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: the library is dlopen'ed on attach

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <limits>
#include <string>
#include <type_traits>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges cost nothing without a tool

#include "host_core.hpp"
#include "ignis_b200.h"
#include "io.hpp"
#include "flux3.cuh"
#include "kernels.cuh"


namespace ign {
KernelSet kernel_set_1();
KernelSet kernel_set_2();
KernelSet kernel_set_3();
KernelSet kernel_set_4();
KernelSet kernel_set_5();
KernelSet kernel_set_6();
KernelSet kernel_set_7();
KernelSet kernel_set_8();

KernelSet kernel_set3_1();
KernelSet kernel_set3_2();
KernelSet kernel_set3_3();
KernelSet kernel_set3_4();
KernelSet kernel_set3_5();
KernelSet kernel_set3_6();
KernelSet kernel_set3_7();
KernelSet kernel_set3_8();

KernelSet kernel_set3(int ns);
KernelSet kernel_set(int ns);
}  // namespace ign

using namespace ign;

struct ign_group;

struct ign_context {
    ign_config cfg;
    HMesh mesh;
    HMetrics met, metv;
    KParams kp;
    KernelSet ks;
    int nx = 0, ny = 0, g = 0, ns = 0, nc = 0;
    size_t plane = 0;
    int device = 0;
    cudaStream_t stream = nullptr, own_stream = nullptr;
    double* S[3] = {nullptr, nullptr, nullptr};
    int cur = 0;
    double* prim = nullptr;
    double* geom = nullptr;  // met(5), met_v(5), mesh x, y
    double *Fx = nullptr, *Gy = nullptr, *Fv = nullptr, *Gv = nullptr, *rhs = nullptr;
    double *Hz = nullptr, *Hv = nullptr;  // 3D extension
    int nz = 0;                           // 0: 2D (the reference), > 0: 3D extension
    int k0 = 0, nz_glob = 0;              // 3D z-slab: first global z cell, global count
    // outputs (solver.hpp:68-74): config hash, probes, product-fraction trace
    uint64_t config_hash = 0;
    int probe_interval = 0, trace_interval = 0;
    struct Probe {
        int i0, j0, i1, j1;  // inclusive interior box, GLOBAL indices
        int k0 = 0, k1 = 0;  // 3D extension: global plane range
        std::vector<double> times, rows;
    };
    std::vector<Probe> probes;
    std::vector<double> trace_t, trace_v;
    double* inflow[4] = {nullptr, nullptr, nullptr, nullptr};
    double* wrap[2] = {nullptr, nullptr};
    ErrRec* err = nullptr;      // the word the kernels report into
    ErrRec* own_err = nullptr;  // this context's allocation
    unsigned long long* red = nullptr;
    double time = 0.0;
    int64_t iter = 0;
    double last_clip = 0.0;
    ign_integrator integ{};
    ign_error lasterr{};
    int64_t launches = 0;
    // halo overlap (slabs): the halo leg (exchange, edge ghosts, ghost-row
    // primitives) runs on halo_stream while the stream computes the slab's own
    // rows; ev_halo joins it before the first kernel that reads the halo
    cudaStream_t halo_stream = nullptr;
    cudaEvent_t ev_ready = nullptr, ev_halo = nullptr;
    bool halo_pending = false;
    // diagnostics (conserved_totals, product fraction): device tree (default)
    // or the reference's serial order on the host (bitwise)
    int diag_mode = IGN_DIAG_DEVICE;
    double* diag_buf = nullptr;
    // slab decomposition
    int nranks = 1, rank = 0;
    int lo_peer = -1, hi_peer = -1;  // ranks owning our ghost rows (-1: physical edge)
    ncclComm_t comm = nullptr;
    ign_group* group = nullptr;
    // live per-kernel-class timing (CUDA events on this context's stream)
    bool prof_on = false;
    struct Rec { int cat; cudaEvent_t a, b; };
    std::vector<Rec> prof_pending;
    std::vector<cudaEvent_t> prof_pool;
    double prof_ms[IGN_PROF_CLASSES] = {};
    int64_t prof_n[IGN_PROF_CLASSES] = {};
};

struct ign_group {
    std::vector<ign_context*> m;
    ign_error lasterr{};
};


namespace ign {
namespace rt {

// ---------------------------------------------------------------- errors, NCCL
struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                              ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl();
void cuda_check(cudaError_t e, const char* what);
void nccl_check(ncclResult_t r, const char* what);
void set_error(ign_error* out, const Error& e);
const char* pstatus_msg(unsigned sub);
cudaEvent_t prof_event(ign_context* ctx);
void prof_harvest(ign_context* ctx);
double* dalloc(size_t n);
void* dmalloc(size_t bytes);
void h2d(ign_context* c, void* dst, const void* src, size_t bytes, const char* what);
void d2h(const ign_context* c, void* dst, const void* src, size_t bytes, const char* what);
void dfree(void* p);
void guard_status(int* enabled, unsigned long long* checked, unsigned long long* bad);
unsigned long long guard_selftest();

template <class F> int guarded_err(ign_error* err, int device, F&& f) {
    try {
        if (device >= 0) cuda_check(cudaSetDevice(device), "cudaSetDevice");
        f();
        if (err) std::memset(err, 0, sizeof(*err));
        return IGN_OK;
    } catch (const Error& e) {
        set_error(err, e);
        return e.status;
    } catch (const std::exception& e) {
        set_error(err, Error(IGN_INTERNAL_ERROR, e.what()));
        return IGN_INTERNAL_ERROR;
    }
}

template <class F> int guarded(ign_context* ctx, F&& f) {
    return guarded_err(ctx ? &ctx->lasterr : nullptr, ctx ? ctx->device : -1, [&] {
        if (ctx && ctx->group)
            throw usage_error("context belongs to a slab group: drive it through ign_group_*");
        f();
    });
}

// NVTX range over a host scope (stage, kernel class, halo leg): visible in
// nsys / ncu --nvtx timelines, free when no tool is attached
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

template <class F> int timed(ign_context* ctx, int cat, F&& f) {
    static const char* const kNames[IGN_PROF_CLASSES] = {"ghost fill", "primitives", "faces",
                                                         "viscous", "assemble", "stable_dt",
                                                         "other", "other"};
    NvtxRange r(kNames[cat]);
    if (!ctx->prof_on) return f();
    cudaEvent_t a = prof_event(ctx), b = prof_event(ctx);
    cuda_check(cudaEventRecord(a, ctx->stream), "event");
    const int n = f();
    cuda_check(cudaEventRecord(b, ctx->stream), "event");
    ctx->prof_pending.push_back({cat, a, b});
    return n;
}

// ---------------------------------------------------------------- teams
struct Team {
    std::vector<ign_context*> m;  // slab order (rank 0 first)
    ign_context* lead() const { return m[0]; }
    bool local() const { return m.size() > 1; }
    cudaStream_t stream() const { return m[0]->stream; }
};

inline Team solo(ign_context* c) { return Team{{c}}; }

// Decoded device failure (key layout: kernels_common.cuh report()).
struct DevFail {
    bool any = false;
    unsigned stage = 0, phase = 0, sub = 0;
    unsigned long long idx = 0;
    int step = 0;
};

DevFail sync_and_read(const Team& T);
Error to_error(const ign_context* ctx, const DevFail& f);
void check(const Team& T);
void t_errsync(const Team& T);
inline size_t halo_stride(const ign_context* c) {
    return c->nz > 0 ? size_t(c->kp.sxy) : size_t(c->kp.sx);
}
inline size_t halo_count(const ign_context* c) { return c->nz > 0 ? c->nz : c->ny; }

void t_exchange(const Team& T, int buf, cudaStream_t s);
bool t_has_halo(const Team& T);
void t_join(const Team& T);
void t_prepare(const Team& T, int buf, int stage, int step);
void t_fluxes(const Team& T, int buf, int stage, int step);
void t_assemble(const Team& T, int mode, int a, int cur, int out, double dt, double w, double t,
                int stage, int step, int slot);
void t_step(const Team& T, int a, double time, double dt, int step, bool post_prepare);
void read_clips(const Team& T, int64_t chunk, std::vector<unsigned long long>& red);
double clip_of(const unsigned long long* red, int slot);
void for_all(const Team& T, const std::function<void(ign_context*)>& f);
constexpr int64_t kChunk = 256;  // steps between host synchronisations
// device reduction slots: [0] lam_max bits, [1] dt_chem bits, then the clip
// of every stage of every step of a chunk (2 + 3 step + stage - 1) — per step,
// so a slab that runs past a peer's failure cannot overwrite clips the
// failure's bookkeeping still needs (the error word is reduced once per chunk)
constexpr int64_t kRedSlots = 2 + 3 * kChunk;
void t_enqueue_chunk(const Team& T, int a0, double& t, double dt, int64_t done, int64_t chunk,
                     bool post_prepare);
void t_finish_chunk(const Team& T, int a0, double dt, int64_t done, int64_t chunk);
void t_run_steps(const Team& T, double dt, int64_t n, bool post_prepare);
void t_run_ensemble(const std::vector<ign_context*>& mem, const double* dt, int64_t n,
                    int* status);
double t_stable_dt(const Team& T);
void t_prepare_sync(const Team& T, int stage);
void t_advance(const Team& T, ign_step_hook hook, void* user);

// ---------------------------------------------------------------- outputs
void fold_ranks(const Team& T, std::vector<double>& acc,
                const std::function<void(ign_context*, std::vector<double>&)>& fold);
void t_conserved_totals(const Team& T, double* tot);
double t_product_fraction(const Team& T);
void t_sample(const Team& T);
void t_gather(const Team& T, bool tcache, std::vector<double>& out);
void t_write_snapshot(const Team& T, const std::string& path, int version, bool with_t);
void t_read_snapshot(const Team& T, const std::string& path);

// ---------------------------------------------------------------- setup
void inflow_profile(const ign_edge& es, double yc, int ns, double& u, double& v, double& T,
                    double* Y);
void cons_from_prim(const DMix& m, double rho, double u, double v, double T, const double* Y,
                    double* U);
void cons_from_prim3(const DMix& m, const Prim3<kMaxSpecies>& pt, const double* Y, double* U);
void upload_state(ign_context* ctx, const std::vector<double>& Ut);
void destroy_impl(ign_context* ctx);
void create_impl(const ign_config* cfg, ign_context* ctx);
void copy_hfield(const HField& f, double* out);
void metrics_out(const HMetrics& m, double* out, size_t P);

}  // namespace rt
}  // namespace ign
