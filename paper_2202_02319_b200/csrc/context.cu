// context.cu — the C-ABI (include/ignis_b200.h) over the sm_100a kernels.
//
// One ign_context = one ignis::Simulation (solver.hpp:53-853) on one GPU, or
// one slab of a domain decomposed along y across GPUs.  The conservative state
// lives in three rotating device buffers S[0..2]; an RK3 step reads U0 from
// S[a], writes U1 to S[b], U2 to S[c] and U3 back into S[b], so no
// copy_interior (solver.hpp:310) is ever needed and U0 stays intact for the
// StepFailure restore (solver.hpp:326-329).  Errors raised on the device are
// collected in one error word and decoded here into the reference's exception
// kinds after the stream synchronises.
//
// Orchestration runs over a "team": one context (optionally exchanging halo
// rows with other processes through NCCL), or a single-process group of slab
// contexts sharing one stream (validation on one GPU).  Both execute the same
// phase sequence per stage:
//   ghost x-pass -> halo exchange -> ghost y-pass -> primitives -> faces ->
//   viscous -> assemble/update (+ error-word MIN all-reduce across slabs).
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

KernelSet kernel_set3(int ns) {
    switch (ns) {
    case 1: return kernel_set3_1();
    case 2: return kernel_set3_2();
    case 3: return kernel_set3_3();
    case 4: return kernel_set3_4();
    case 5: return kernel_set3_5();
    case 6: return kernel_set3_6();
    case 7: return kernel_set3_7();
    default: return kernel_set3_8();
    }
}

KernelSet kernel_set(int ns) {
    switch (ns) {
    case 1: return kernel_set_1();
    case 2: return kernel_set_2();
    case 3: return kernel_set_3();
    case 4: return kernel_set_4();
    case 5: return kernel_set_5();
    case 6: return kernel_set_6();
    case 7: return kernel_set_7();
    default: return kernel_set_8();
    }
}
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

namespace {

// ---------------------------------------------------------------- NCCL (dlopen)
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

NcclApi load_nccl() {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        a.why = std::string("libnccl not loadable: ") + dlerror();
        return a;
    }
    bool all = true;
    auto sym = [&](auto& f, const char* n) {
        f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, n));
        all = all && f;
    };
    sym(a.GetUniqueId, "ncclGetUniqueId");
    sym(a.CommInitRank, "ncclCommInitRank");
    sym(a.CommDestroy, "ncclCommDestroy");
    sym(a.Send, "ncclSend");
    sym(a.Recv, "ncclRecv");
    sym(a.GroupStart, "ncclGroupStart");
    sym(a.GroupEnd, "ncclGroupEnd");
    sym(a.AllReduce, "ncclAllReduce");
    sym(a.Broadcast, "ncclBroadcast");
    sym(a.GetErrorString, "ncclGetErrorString");
    a.ok = all;
    if (!all) a.why = "libnccl lacks an entry point";
    return a;
}

NcclApi& nccl() {
    static NcclApi a = load_nccl();
    return a;
}

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw Error(IGN_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw Error(IGN_CUDA_ERROR, std::string(what) + ": " + nccl().GetErrorString(r));
}

void set_error(ign_error* out, const Error& e) {
    if (!out) return;
    out->status = e.status;
    out->stage = e.stage;
    out->i = e.i;
    out->j = e.j;
    std::snprintf(out->msg, sizeof(out->msg), "%s", e.what());
}

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

const char* pstatus_msg(unsigned sub) {
    switch (sub) {
    case P_NONPOS_RHO: return "primitives: non-positive density";
    case P_BELOW_VACUUM: return "temperature_from_energy: energy below vacuum energy";
    default: return "temperature_from_energy: no convergence";
    }
}

cudaEvent_t prof_event(ign_context* ctx) {
    if (!ctx->prof_pool.empty()) {
        cudaEvent_t e = ctx->prof_pool.back();
        ctx->prof_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cuda_check(cudaEventCreate(&e), "cudaEventCreate");
    return e;
}

// Runs one launcher; with profiling on, brackets it with events on the stream.
template <class F> int timed(ign_context* ctx, int cat, F&& f) {
    if (!ctx->prof_on) return f();
    cudaEvent_t a = prof_event(ctx), b = prof_event(ctx);
    cuda_check(cudaEventRecord(a, ctx->stream), "event");
    const int n = f();
    cuda_check(cudaEventRecord(b, ctx->stream), "event");
    ctx->prof_pending.push_back({cat, a, b});
    return n;
}

void prof_harvest(ign_context* ctx) {
    for (auto& r : ctx->prof_pending) {
        float ms = 0.f;
        cuda_check(cudaEventElapsedTime(&ms, r.a, r.b), "event time");
        ctx->prof_ms[r.cat] += ms;
        ++ctx->prof_n[r.cat];
        ctx->prof_pool.push_back(r.a);
        ctx->prof_pool.push_back(r.b);
    }
    ctx->prof_pending.clear();
}

double* dalloc(size_t n) {
    void* p = nullptr;
    cuda_check(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(double)), "cudaMalloc");
    return static_cast<double*>(p);
}

// ---------------------------------------------------------------- teams
struct Team {
    std::vector<ign_context*> m;  // slab order (rank 0 first)
    ign_context* lead() const { return m[0]; }
    bool local() const { return m.size() > 1; }
    cudaStream_t stream() const { return m[0]->stream; }
};

Team solo(ign_context* c) { return Team{{c}}; }

// Decoded device failure (key layout: kernels_common.cuh report()).
struct DevFail {
    bool any = false;
    unsigned stage = 0, phase = 0, sub = 0;
    unsigned long long idx = 0;
    int step = 0;
};

void t_errsync(const Team& T);

// Every rank reads the same (MIN-reduced) error word: a failure in the last
// kernels before this point (e.g. a step's final update) is seen everywhere.
DevFail sync_and_read(const Team& T) {
    t_errsync(T);
    cuda_check(cudaStreamSynchronize(T.stream()), "kernel execution");
    cuda_check(cudaGetLastError(), "kernel launch");
    for (ign_context* c : T.m) prof_harvest(c);
    ErrRec h;
    ign_context* L = T.lead();
    cuda_check(cudaMemcpy(&h, L->err, sizeof(h), cudaMemcpyDeviceToHost), "error word");
    DevFail f;
    if (h.key == kNoError) return f;
    f.any = true;
    f.step = (int)(h.key >> 44);
    f.stage = (unsigned)((h.key >> 41) & 7);
    f.phase = (unsigned)((h.key >> 38) & 7);
    f.idx = (h.key >> 3) & ((1ull << 35) - 1);
    f.sub = (unsigned)(h.key & 7);
    for (ign_context* c : T.m)
        cuda_check(cudaMemset(c->own_err, 0xff, sizeof(ErrRec)), "error reset");
    return f;
}

// Maps a device failure onto the exception the reference throws there
// (indices are global: the reference runs the undecomposed domain).
Error to_error(const ign_context* ctx, const DevFail& f) {
    const int rep_stage = f.stage == 4 ? 1 : (int)f.stage;
    switch (f.phase) {
    case PH_BC: return state_error(pstatus_msg(f.sub));
    case PH_PRIM: {
        const int sx = ctx->nx + 2 * ctx->g;
        if (ctx->nz > 0) {  // 3D: global padded (i, j, k) of the node
            const unsigned long long sy = ctx->ny + 2 * ctx->g;
            const int i = (int)(f.idx % sx) - ctx->g, j = (int)((f.idx / sx) % sy) - ctx->g;
            const int k = (int)(f.idx / (sx * sy)) - ctx->g;
            return step_failure(std::string("stage state failure: ") + pstatus_msg(f.sub) +
                                    " (k=" + std::to_string(k) + ")",
                                rep_stage, i, j);
        }
        const int i = (int)(f.idx % sx) - ctx->g, j = (int)(f.idx / sx) - ctx->g;
        return step_failure(std::string("stage state failure: ") + pstatus_msg(f.sub),
                            rep_stage, i, j);
    }
    case PH_INVX:
    case PH_INVY:
        if (f.sub == 2) return numerics_error("eigen: zero metric direction");
        if (f.sub == 3) return numerics_error("eigen: non-positive c^2");
        return numerics_error("inviscid face: non-finite wavespeed");
    case PH_RHS: {
        const unsigned long long cell = f.idx;
        const int i = (int)(cell % ctx->nx);
        const int j = (int)(ctx->nz > 0 ? (cell / ctx->nx) % ctx->ny : cell / ctx->nx);
        return step_failure("non-finite RHS", rep_stage, i, j);
    }
    default: {
        const unsigned long long cell = f.idx / 2;
        const int i = (int)(cell % ctx->nx);
        const int j = (int)(ctx->nz > 0 ? (cell / ctx->nx) % ctx->ny : cell / ctx->nx);
        return step_failure(f.idx % 2 ? "non-finite state" : "non-positive density", rep_stage,
                            i, j);
    }
    }
}

void check(const Team& T) {
    const DevFail f = sync_and_read(T);
    if (f.any) throw to_error(T.lead(), f);
}

// Cross-slab consistency of the error word: MIN all-reduce (NCCL teams only;
// a local group shares one word).
void t_errsync(const Team& T) {
    ign_context* c = T.lead();
    if (T.local() || !c->comm) return;
    nccl_check(nccl().AllReduce(&c->err->key, &c->err->key, 1, ncclUint64, ncclMin, c->comm,
                                c->stream),
               "ncclAllReduce(error word)");
}

// Halo rows of state buffer `buf`: our g bottom/top interior rows to the
// neighbours, their rows into our ghost rows (all components; rows are
// contiguous in the padded planes, so every transfer is one contiguous chunk).
// 2D: y-slabs exchange g padded rows; 3D: z-slabs exchange g padded planes
static size_t halo_stride(const ign_context* c) {
    return c->nz > 0 ? size_t(c->kp.sxy) : size_t(c->kp.sx);
}
static size_t halo_count(const ign_context* c) { return c->nz > 0 ? c->nz : c->ny; }

void t_exchange(const Team& T, int buf) {
    if (T.local()) {
        for (ign_context* c : T.m) {
            const size_t st = halo_stride(c), chunk = size_t(c->g) * st;
            for (int comp = 0; comp < c->nc; ++comp) {
                if (c->lo_peer >= 0) {
                    const ign_context* s = T.m[c->lo_peer];
                    cuda_check(cudaMemcpyAsync(c->S[buf] + comp * c->plane,
                                               s->S[buf] + comp * s->plane + halo_count(s) * st,
                                               chunk * sizeof(double), cudaMemcpyDeviceToDevice,
                                               T.stream()),
                               "halo copy");
                }
                if (c->hi_peer >= 0) {
                    const ign_context* s = T.m[c->hi_peer];
                    cuda_check(cudaMemcpyAsync(c->S[buf] + comp * c->plane +
                                                   (halo_count(c) + c->g) * st,
                                               s->S[buf] + comp * s->plane + chunk,
                                               chunk * sizeof(double), cudaMemcpyDeviceToDevice,
                                               T.stream()),
                               "halo copy");
                }
            }
        }
        return;
    }
    ign_context* c = T.lead();
    if (c->lo_peer < 0 && c->hi_peer < 0) return;
    if (!c->comm)
        throw usage_error("slab context without a transport: call ign_attach_nccl or use a group");
    NcclApi& n = nccl();
    const size_t st = halo_stride(c), chunk = size_t(c->g) * st, nl = halo_count(c);
    nccl_check(n.GroupStart(), "ncclGroupStart");
    for (int comp = 0; comp < c->nc; ++comp) {
        double* base = c->S[buf] + comp * c->plane;
        // per peer pair the order is [top, bottom] sends against [lo, hi]
        // receives, so a two-slab periodic ring matches correctly
        if (c->hi_peer >= 0)
            nccl_check(n.Send(base + nl * st, chunk, ncclFloat64, c->hi_peer,
                              c->comm, c->stream), "ncclSend");
        if (c->lo_peer >= 0)
            nccl_check(n.Send(base + chunk, chunk, ncclFloat64, c->lo_peer, c->comm, c->stream),
                       "ncclSend");
        if (c->lo_peer >= 0)
            nccl_check(n.Recv(base, chunk, ncclFloat64, c->lo_peer, c->comm, c->stream),
                       "ncclRecv");
        if (c->hi_peer >= 0)
            nccl_check(n.Recv(base + (nl + c->g) * st, chunk, ncclFloat64,
                              c->hi_peer, c->comm, c->stream), "ncclRecv");
    }
    nccl_check(n.GroupEnd(), "ncclGroupEnd");
}

// prepare_stage (solver.hpp:422-425): fill_ghosts (x edges, halo, y edges)
// then refresh_primitives
void t_prepare(const Team& T, int buf, int stage, int step) {
    for (ign_context* c : T.m)
        c->launches += timed(c, IGN_PROF_BC, [&] {
            return c->ks.bc(c->kp, c->S[buf], 0, stage, step, c->stream);
        });
    t_exchange(T, buf);
    for (ign_context* c : T.m)
        c->launches += timed(c, IGN_PROF_BC, [&] {
            return c->ks.bc(c->kp, c->S[buf], 1, stage, step, c->stream);
        });
    for (ign_context* c : T.m)
        c->launches += timed(c, IGN_PROF_PRIM, [&] {
            return c->ks.prim(c->kp, c->S[buf], stage, step, c->stream);
        });
    t_errsync(T);
}

void t_fluxes(const Team& T, int buf, int stage, int step) {
    for (ign_context* c : T.m) {
        c->launches += timed(c, IGN_PROF_FACES, [&] {
            return c->ks.faces(c->kp, c->cfg.scheme.scheme, c->cfg.scheme.split, c->S[buf], stage,
                               step, c->stream);
        });
        if (c->cfg.viscous)
            c->launches += timed(c, IGN_PROF_VISC,
                                 [&] { return c->ks.visc(c->kp, stage, step, c->stream); });
    }
}

void t_assemble(const Team& T, int mode, int a, int cur, int out, double dt, double w, double t,
                int stage, int step, int slot) {
    for (ign_context* c : T.m)
        c->launches += timed(c, IGN_PROF_ASSEMBLE, [&] {
            return c->ks.assemble(c->kp, mode, c->S[a], c->S[cur], c->S[out], dt, w, t, stage,
                                  step, slot, c->stream);
        });
    t_errsync(T);
}

// Zeroes one step's clip slots unless a failure is pending (a pending failure
// must keep the previous step's clips for last_clip, solver.hpp:847).
__global__ void k_clip_reset(const ErrRec* err, unsigned long long* red, int slot) {
    if (failed(err)) return;
    red[2 + slot + threadIdx.x] = 0ull;
}

// One rk3_step (solver.hpp:304-332) enqueued without a host round trip;
// post_prepare appends advance()'s prepare_stage(1) (solver.hpp:345).
void t_step(const Team& T, int a, double time, double dt, int step, bool post_prepare) {
    const int b = (a + 1) % 3, c = (a + 2) % 3;
    const int slot = (step & 1) * 3;
    for (ign_context* x : T.m) {
        k_clip_reset<<<1, 3, 0, x->stream>>>(x->err, x->red, slot);
        ++x->launches;
    }
    // Stage 1: U <- U0 + dt L(U0)   (ghosts/cache already fresh)
    t_fluxes(T, a, 1, step);
    t_assemble(T, 1, a, a, b, dt, 0.0, time, 1, step, slot + 0);
    t_prepare(T, b, 2, step);
    // Stage 2: U <- U0 + 1/4 [(U1 - U0) + dt L(U1)]
    t_fluxes(T, b, 2, step);
    t_assemble(T, 2, a, b, c, dt, 0.25, time + dt, 2, step, slot + 1);
    t_prepare(T, c, 3, step);
    // Stage 3: U <- U0 + 2/3 [(U2 - U0) + dt L(U2)]
    t_fluxes(T, c, 3, step);
    t_assemble(T, 2, a, c, b, dt, 2.0 / 3.0, time + 0.5 * dt, 3, step, slot + 2);
    if (post_prepare) t_prepare(T, b, 4, step);
}

// Clip slots of all slabs (MAX over slabs: the reference's clip is a max).
void read_clips(const Team& T, unsigned long long red[8]) {
    ign_context* L = T.lead();
    if (!T.local() && L->comm) {
        nccl_check(nccl().AllReduce(L->red + 2, L->red + 2, 6, ncclUint64, ncclMax, L->comm,
                                    L->stream),
                   "ncclAllReduce(clip)");
        cuda_check(cudaStreamSynchronize(L->stream), "clip reduce");
    }
    std::memset(red, 0, 8 * sizeof(unsigned long long));
    for (ign_context* c : T.m) {
        unsigned long long r[8];
        cuda_check(cudaMemcpy(r, c->red, sizeof(r), cudaMemcpyDeviceToHost), "reductions");
        for (int k = 2; k < 8; ++k) red[k] = std::max(red[k], r[k]);
    }
}

double clip_of(const unsigned long long* red, int slot) {
    double d;
    std::memcpy(&d, &red[2 + slot], sizeof(d));
    return d;
}

void for_all(const Team& T, const std::function<void(ign_context*)>& f) {
    for (ign_context* c : T.m) f(c);
}

// Launch steps [done, done+chunk) of a run that started at buffer a0 and time
// t (advanced in place); no host synchronisation.
void t_enqueue_chunk(const Team& T, int a0, double& t, double dt, int64_t done, int64_t chunk,
                     bool post_prepare) {
    for (int64_t k = 0; k < chunk; ++k) {
        const int64_t s = done + k;
        t_step(T, (int)((a0 + s) % 3), t, dt, (int)(s - done), post_prepare);
        t += dt;
    }
    cuda_check(cudaGetLastError(), "kernel launch");
}

// Synchronise on a launched chunk and account it: time/iter/buffer/last_clip
// advance; on a device failure reproduce the reference's state, time/iter and
// last_clip at the point it would have thrown, then throw.
void t_finish_chunk(const Team& T, int a0, double dt, int64_t done, int64_t chunk) {
    const DevFail f = sync_and_read(T);
    unsigned long long red[8];
    read_clips(T, red);
    if (!f.any) {
        const int last = (int)(chunk - 1);
        const int slot = (last & 1) * 3;
        const double lc = std::max(std::max(clip_of(red, slot), clip_of(red, slot + 1)),
                                   clip_of(red, slot + 2));
        for_all(T, [&](ign_context* c) {
            for (int64_t k = 0; k < chunk; ++k) {
                c->time += dt;
                ++c->iter;
            }
            c->last_clip = lc;
            c->cur = (int)((a0 + done + chunk) % 3);
        });
        return;
    }
    const int64_t kk = f.step;  // failing step within this chunk
    const int64_t k = done + kk;
    double clip_prev = T.lead()->last_clip;
    if (kk > 0) {
        const int slot = ((int)(kk - 1) & 1) * 3;
        clip_prev = std::max(std::max(clip_of(red, slot), clip_of(red, slot + 1)),
                             clip_of(red, slot + 2));
    }
    const int ak = (int)((a0 + k) % 3);
    const int slot = ((int)kk & 1) * 3;
    const Error e = to_error(T.lead(), f);
    if (f.stage == 4) {  // advance's prepare_stage(1) after a completed step
        const double lc = std::max(std::max(clip_of(red, slot), clip_of(red, slot + 1)),
                                   clip_of(red, slot + 2));
        for_all(T, [&](ign_context* c) {
            for (int64_t q = done; q <= k; ++q) {
                c->time += dt;
                ++c->iter;
            }
            c->cur = (ak + 1) % 3;
            c->last_clip = lc;
        });
        throw e;
    }
    // inside rk3_step: last_clip covers the stages that completed post_stage
    double lc = clip_prev;
    for (unsigned s = 1; s < f.stage; ++s)
        lc = s == 1 ? clip_of(red, slot) : std::max(lc, clip_of(red, slot + s - 1));
    const int cur = e.status == IGN_STEP_FAILURE ? ak  // restore U0
                    : f.stage <= 1               ? ak
                    : f.stage == 2               ? (ak + 1) % 3
                                                 : (ak + 2) % 3;
    for_all(T, [&](ign_context* c) {
        for (int64_t q = done; q < k; ++q) {
            c->time += dt;
            ++c->iter;
        }
        c->last_clip = lc;
        c->cur = cur;
    });
    throw e;
}

constexpr int64_t kChunk = 256;  // steps between host synchronisations

// n consecutive steps (the advance() loop body with a pinned dt)
void t_run_steps(const Team& T, double dt, int64_t n, bool post_prepare) {
    if (n <= 0) return;
    const int a0 = T.lead()->cur;
    double t = T.lead()->time;
    for (int64_t done = 0; done < n;) {
        const int64_t chunk = std::min<int64_t>(n - done, kChunk);
        t_enqueue_chunk(T, a0, t, dt, done, chunk, post_prepare);
        t_finish_chunk(T, a0, dt, done, chunk);
        done += chunk;
    }
}

// Ensemble (BASELINE configs[4]): independent members on one GPU, each on its
// own stream, launched step-interleaved so small members share the SMs; every
// member keeps rk3_steps' semantics and its own failure (status per member,
// text via ign_last_error) without stopping the others.
void t_run_ensemble(const std::vector<ign_context*>& mem, const double* dt, int64_t n,
                    int* status) {
    const size_t M = mem.size();
    std::vector<int> a0(M);
    std::vector<double> t(M);
    std::vector<char> live(M, 1);
    for (size_t q = 0; q < M; ++q) {
        a0[q] = mem[q]->cur;
        t[q] = mem[q]->time;
        status[q] = IGN_OK;
    }
    for (int64_t done = 0; done < n;) {
        const int64_t chunk = std::min<int64_t>(n - done, kChunk);
        for (int64_t k = 0; k < chunk; ++k)
            for (size_t q = 0; q < M; ++q) {
                if (!live[q]) continue;
                try {
                    t_step(solo(mem[q]), (int)((a0[q] + done + k) % 3), t[q], dt[q], (int)k, true);
                    t[q] += dt[q];
                } catch (const Error& e) {
                    live[q] = 0;
                    status[q] = e.status;
                    set_error(&mem[q]->lasterr, e);
                }
            }
        for (size_t q = 0; q < M; ++q) {
            if (!live[q]) continue;
            try {
                t_finish_chunk(solo(mem[q]), a0[q], dt[q], done, chunk);
            } catch (const Error& e) {
                live[q] = 0;
                status[q] = e.status;
                set_error(&mem[q]->lasterr, e);
            }
        }
        done += chunk;
    }
}

double t_stable_dt(const Team& T) {
    unsigned long long init[2] = {0ull, 0x7ff0000000000000ull};
    for (ign_context* c : T.m) {
        cuda_check(cudaMemcpyAsync(c->red, init, sizeof(init), cudaMemcpyHostToDevice, c->stream),
                   "dt reset");
        c->launches += timed(c, IGN_PROF_DT, [&] { return c->ks.dt(c->kp, c->stream); });
    }
    ign_context* L = T.lead();
    if (!T.local() && L->comm) {  // max/min are exact in any order
        nccl_check(nccl().AllReduce(L->red, L->red, 1, ncclUint64, ncclMax, L->comm, L->stream),
                   "ncclAllReduce(lam)");
        nccl_check(nccl().AllReduce(L->red + 1, L->red + 1, 1, ncclUint64, ncclMin, L->comm,
                                    L->stream),
                   "ncclAllReduce(dt_chem)");
    }
    check(T);
    unsigned long long lam_bits = 0ull, chem_bits = 0x7ff0000000000000ull;
    for (ign_context* c : T.m) {
        unsigned long long r[2];
        cuda_check(cudaMemcpy(r, c->red, sizeof(r), cudaMemcpyDeviceToHost), "dt readback");
        lam_bits = std::max(lam_bits, r[0]);
        chem_bits = std::min(chem_bits, r[1]);
    }
    double lam_max, dt_chem;
    std::memcpy(&lam_max, &lam_bits, sizeof(double));
    std::memcpy(&dt_chem, &chem_bits, sizeof(double));
    double dt = L->cfg.scheme.cfl / lam_max;
    dt = smin(dt, dt_chem);
    const ign_laser& las = L->cfg.laser;
    if (las.present && las.energy != 0.0 && L->time - las.t0 < 6.0 * las.sigma_t &&
        L->time + dt > las.t0 - 6.0 * las.sigma_t)
        dt = smin(dt, las.sigma_t / 5.0);
    return dt;
}

void t_prepare_sync(const Team& T, int stage) {
    t_prepare(T, T.lead()->cur, stage, 0);
    check(T);
}

// Serial left folds in the reference's order (solver.hpp:387-418) across
// slabs: each slab continues the running accumulators of the slab below, so
// the decomposed result is bit-identical to the single-domain one.
void fold_ranks(const Team& T, std::vector<double>& acc,
                const std::function<void(ign_context*, std::vector<double>&)>& fold) {
    if (T.local()) {
        for (ign_context* c : T.m) fold(c, acc);
        return;
    }
    ign_context* c = T.lead();
    if (!c->comm || c->nranks == 1) {
        fold(c, acc);
        return;
    }
    NcclApi& n = nccl();
    double* d = dalloc(acc.size());
    try {
        if (c->rank > 0) {
            nccl_check(n.Recv(d, acc.size(), ncclFloat64, c->rank - 1, c->comm, c->stream),
                       "ncclRecv(fold)");
            cuda_check(cudaMemcpyAsync(acc.data(), d, acc.size() * 8, cudaMemcpyDeviceToHost,
                                       c->stream), "fold");
            cuda_check(cudaStreamSynchronize(c->stream), "fold");
        }
        fold(c, acc);
        cuda_check(cudaMemcpyAsync(d, acc.data(), acc.size() * 8, cudaMemcpyHostToDevice,
                                   c->stream), "fold");
        if (c->rank + 1 < c->nranks)
            nccl_check(n.Send(d, acc.size(), ncclFloat64, c->rank + 1, c->comm, c->stream),
                       "ncclSend(fold)");
        nccl_check(n.Broadcast(d, d, acc.size(), ncclFloat64, c->nranks - 1, c->comm, c->stream),
                   "ncclBroadcast(fold)");
        cuda_check(cudaMemcpyAsync(acc.data(), d, acc.size() * 8, cudaMemcpyDeviceToHost,
                                   c->stream), "fold");
        cuda_check(cudaStreamSynchronize(c->stream), "fold");
    } catch (...) {
        cudaFree(d);
        throw;
    }
    cudaFree(d);
}

// conserved_totals (solver.hpp:411-418)
void t_conserved_totals(const Team& T, double* tot) {
    const int nc = T.lead()->nc;
    std::vector<double> acc(nc, 0.0);
    // component-major in the reference: fold per component across slabs
    for (int comp = 0; comp < nc; ++comp) {
        std::vector<double> a1(1, 0.0);
        fold_ranks(T, a1, [&](ign_context* c, std::vector<double>& a) {
            const size_t P = c->plane;
            std::vector<double> U(P);
            cuda_check(cudaMemcpy(U.data(), c->S[c->cur] + comp * P, P * 8, cudaMemcpyDeviceToHost),
                       "totals");
            const int sx = c->nx + 2 * c->g, g = c->g;
            const size_t sxy = size_t(sx) * (c->ny + 2 * g);
            double s = a[0];
            for (int k = 0; k < (c->nz > 0 ? c->nz : 1); ++k)  // 3D: z-planes outermost
                for (int j = 0; j < c->ny; ++j)
                    for (int i = 0; i < c->nx; ++i)
                        s += U[(c->nz > 0 ? (k + g) * sxy : 0) + (size_t)(j + g) * sx + (i + g)];
            a[0] = s;
        });
        tot[comp] = a1[0];
    }
}

// product_mole_fraction (solver.hpp:387-407)
double t_product_fraction(const Team& T) {
    ign_context* L = T.lead();
    int ico2 = -1, ih2o = -1;
    for (int s = 0; s < L->ns; ++s) {
        const char* nm = L->cfg.mix.species[s].name;
        if (std::strncmp(nm, "CO2", IGN_NAME_LEN) == 0) ico2 = s;
        if (std::strncmp(nm, "H2O", IGN_NAME_LEN) == 0) ih2o = s;
    }
    if (ico2 < 0 && ih2o < 0) return 0.0;
    std::vector<double> acc(2, 0.0);
    fold_ranks(T, acc, [&](ign_context* c, std::vector<double>& a) {
        const size_t P = c->plane;
        std::vector<double> Y(c->ns * P);
        cuda_check(cudaMemcpy(Y.data(), c->prim + (c->nz > 0 ? 7 : 6) * P, Y.size() * 8,
                              cudaMemcpyDeviceToHost),
                   "Y readback");
        const DMix& m = c->kp.mix;
        const int sx = c->nx + 2 * c->g, g = c->g;
        const size_t sxy = size_t(sx) * (c->ny + 2 * g);
        double num = a[0], den = a[1];
        for (int kz = 0; kz < (c->nz > 0 ? c->nz : 1); ++kz)
        for (int j = 0; j < c->ny; ++j)
            for (int i = 0; i < c->nx; ++i) {
                const size_t id =
                    (c->nz > 0 ? (kz + g) * sxy : 0) + (size_t)(j + g) * sx + (i + g);
                double y[kMaxSpecies], x[kMaxSpecies];
                for (int s = 0; s < c->ns; ++s) y[s] = Y[s * P + id];
                double inv = 0.0;
                for (int s = 0; s < c->ns; ++s) inv += divW(m.sp[s], y[s]);
                const double wbar = 1.0 / inv;
                for (int s = 0; s < c->ns; ++s) x[s] = divW(m.sp[s], y[s] * wbar);
                const double w = 1.0 / c->met.jac(i, j);
                num += w * ((ico2 >= 0 ? x[ico2] : 0.0) + (ih2o >= 0 ? x[ih2o] : 0.0));
                den += w;
            }
        a[0] = num;
        a[1] = den;
    });
    return acc[0] / acc[1];
}

// ---------------------------------------------------------------- setup
// detail::inflow_profile (boundary.hpp:94-124) — host side, glibc tanh.
void inflow_profile(const ign_edge& es, double yc, int ns, double& u, double& v, double& T,
                    double* Y) {
    const double w = es.smooth_width > 0.0 ? es.smooth_width : 1e-30;
    double wsum = 0.0;
    u = v = T = 0.0;
    for (int s = 0; s < kMaxSpecies; ++s) Y[s] = 0.0;
    for (int k = 0; k < es.nseg; ++k) {
        const ign_inflow_segment& seg = es.seg[k];
        const double a = 0.5 * (std::tanh((yc - seg.lo) / w) - std::tanh((yc - seg.hi) / w));
        wsum += a;
        u += a * seg.u;
        v += a * seg.v;
        T += a * seg.T;
        for (int s = 0; s < ns; ++s) Y[s] += a * seg.Y[s];
    }
    if (wsum <= 1e-300) {
        const ign_inflow_segment& seg = es.seg[0];
        u = seg.u;
        v = seg.v;
        T = seg.T;
        for (int s = 0; s < kMaxSpecies; ++s) Y[s] = seg.Y[s];
        return;
    }
    u /= wsum;
    v /= wsum;
    T /= wsum;
    double ysum = 0.0;
    for (int s = 0; s < ns; ++s) ysum += Y[s];
    for (int s = 0; s < ns; ++s) Y[s] /= ysum;
}

// conservative_from_primitives for one node, runtime species count.
template <int NS>
void cons_from_prim_t(const DMix& m, double rho, double u, double v, double T, const double* Y,
                      double* U) {
    Prim<NS> pt;
    pt.rho = rho;
    pt.u = u;
    pt.v = v;
    pt.T = T;
    pt.p = 0.0;
    for (int s = 0; s < NS; ++s) pt.Y[s] = Y[s];
    conservative_from_primitives<NS>(pt, m, U);
}

void cons_from_prim(const DMix& m, double rho, double u, double v, double T, const double* Y,
                    double* U) {
    switch (m.ns) {
    case 1: return cons_from_prim_t<1>(m, rho, u, v, T, Y, U);
    case 2: return cons_from_prim_t<2>(m, rho, u, v, T, Y, U);
    case 3: return cons_from_prim_t<3>(m, rho, u, v, T, Y, U);
    case 4: return cons_from_prim_t<4>(m, rho, u, v, T, Y, U);
    case 5: return cons_from_prim_t<5>(m, rho, u, v, T, Y, U);
    case 6: return cons_from_prim_t<6>(m, rho, u, v, T, Y, U);
    case 7: return cons_from_prim_t<7>(m, rho, u, v, T, Y, U);
    default: return cons_from_prim_t<8>(m, rho, u, v, T, Y, U);
    }
}

template <int NS>
void cons_from_prim3_t(const DMix& m, const Prim3<kMaxSpecies>& in, const double* Y, double* U) {
    Prim3<NS> pt;
    pt.rho = in.rho;
    pt.u = in.u;
    pt.v = in.v;
    pt.w = in.w;
    pt.T = in.T;
    pt.p = 0.0;
    for (int s = 0; s < NS; ++s) pt.Y[s] = Y[s];
    conservative_from_primitives3<NS>(pt, m, U);
}

void cons_from_prim3(const DMix& m, const Prim3<kMaxSpecies>& pt, const double* Y, double* U) {
    switch (m.ns) {
    case 1: return cons_from_prim3_t<1>(m, pt, Y, U);
    case 2: return cons_from_prim3_t<2>(m, pt, Y, U);
    case 3: return cons_from_prim3_t<3>(m, pt, Y, U);
    case 4: return cons_from_prim3_t<4>(m, pt, Y, U);
    case 5: return cons_from_prim3_t<5>(m, pt, Y, U);
    case 6: return cons_from_prim3_t<6>(m, pt, Y, U);
    case 7: return cons_from_prim3_t<7>(m, pt, Y, U);
    default: return cons_from_prim3_t<8>(m, pt, Y, U);
    }
}

void upload_state(ign_context* ctx, const std::vector<double>& Ut) {
    cuda_check(cudaMemcpy(ctx->S[ctx->cur], Ut.data(), Ut.size() * sizeof(double),
                          cudaMemcpyHostToDevice),
               "state upload");
}

void destroy_impl(ign_context* ctx) {
    if (!ctx) return;
    for (double* p : ctx->S) cudaFree(p);
    cudaFree(ctx->prim);
    cudaFree(ctx->geom);
    cudaFree(ctx->Fx);
    cudaFree(ctx->Gy);
    cudaFree(ctx->Fv);
    cudaFree(ctx->Gv);
    cudaFree(ctx->Hz);
    cudaFree(ctx->Hv);
    cudaFree(ctx->rhs);
    for (double* p : ctx->inflow) cudaFree(p);
    for (double* p : ctx->wrap) cudaFree(p);
    cudaFree(ctx->own_err);
    cudaFree(ctx->red);
    for (auto& r : ctx->prof_pending) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (cudaEvent_t e : ctx->prof_pool) cudaEventDestroy(e);
    if (ctx->comm && nccl().ok) nccl().CommDestroy(ctx->comm);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    delete ctx;
}

void create_impl(const ign_config* cfg, ign_context* ctx) {
    if (!cfg || cfg->abi_version != IGN_ABI_VERSION)
        throw usage_error("ign_create: ABI version mismatch");
    ctx->cfg = *cfg;
    ctx->device = cfg->device;
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    ctx->nranks = cfg->slab_count > 1 ? cfg->slab_count : 1;
    ctx->rank = ctx->nranks > 1 ? cfg->slab_rank : 0;
    if (ctx->rank < 0 || ctx->rank >= ctx->nranks) throw usage_error("slab_rank out of range");
    // Simulation::init (solver.hpp:82-101), on this slab's rows
    // 2D: y-slabs of the mesh; 3D: z-slabs over the whole (x, y) mesh
    const bool three_d = cfg->nz > 0;
    ctx->mesh = three_d ? build_mesh(*cfg, 1, 0) : build_mesh(*cfg, ctx->nranks, ctx->rank);
    validate_config(*cfg, ctx->mesh);
    const int imode = inviscid_metric_mode(*cfg);
    ctx->met = compute_metrics(ctx->mesh, imode, cfg->skew_beta);
    ctx->metv = compute_metrics(ctx->mesh, MM_CENTRAL2, 0.0);
    ctx->integ = cfg->integ;
    int nz = 0;
    std::vector<double> mzz, vmzz;
    if (three_d) {
        // 3D extension: the (x, y) mesh extruded over lz (flux3.cuh)
        if (!(cfg->lz > 0.0)) throw config_error("3D: lz must be positive");
        // x / y edges take the reference's 2D rules on every z plane; z is periodic
        if (!cfg->periodic_z) throw usage_error("3D: z must be periodic");
        int k0 = 0;
        slab_rows(cfg->nz, ctx->nranks, ctx->rank, k0, nz);
        if (nz < cfg->g) throw config_error("3D: every z-slab needs >= g planes");
        if (ctx->nranks == 1 && nz < 2 * cfg->g + 1) throw config_error("3D: nz must be >= 2g+1");
        ctx->k0 = k0;
        ctx->nz_glob = cfg->nz;
        const double dz = cfg->lz / cfg->nz;
        // cofactor metrics of (x(i,j), y(i,j), z(k)): xi/eta rows scale by z_zeta
        // = dz, zeta row is the 2D area, J = 1/(area dz) — for dz = 1 every value
        // is the 2D one bit for bit (the z-extrusion cross-check)
        auto extrude = [&](HMetrics& m, std::vector<double>& zz) {
            zz.resize(m.jac.d.size());
            for (size_t q = 0; q < zz.size(); ++q) {
                const double area =
                    m.m_eta_y.d[q] * m.m_xi_x.d[q] - (-m.m_xi_y.d[q]) * (-m.m_eta_x.d[q]);
                zz[q] = area;
                m.jac.d[q] = 1.0 / (area * dz);
                m.m_xi_x.d[q] *= dz;
                m.m_xi_y.d[q] *= dz;
                m.m_eta_x.d[q] *= dz;
                m.m_eta_y.d[q] *= dz;
            }
        };
        extrude(ctx->met, mzz);
        extrude(ctx->metv, vmzz);
    }
    const int nx = cfg->nx, ny = ctx->mesh.ny, g = cfg->g, ns = cfg->mix.ns,
              nc = ns + (nz > 0 ? 4 : 3);
    ctx->nz = nz;
    const int N = ctx->nranks, r = ctx->rank;
    const bool py = (three_d ? cfg->periodic_z : cfg->periodic_y) != 0;
    if (N > 1) {
        ctx->lo_peer = r > 0 ? r - 1 : (py ? N - 1 : -1);
        ctx->hi_peer = r < N - 1 ? r + 1 : (py ? 0 : -1);
    }
    ctx->nx = nx;
    ctx->ny = ny;
    ctx->g = g;
    ctx->ns = ns;
    ctx->nc = nc;
    const size_t P2 = static_cast<size_t>(nx + 2 * g) * (ny + 2 * g);  // one (x, y) plane
    const size_t P = P2 * (nz > 0 ? nz + 2 * g : 1);
    if (P >= (1ull << 31)) throw config_error("padded box too large for one context (>= 2^31 nodes)");
    ctx->plane = P;
    cuda_check(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking), "stream");
    ctx->stream = ctx->own_stream;
    for (auto& s : ctx->S) {
        s = dalloc(nc * P);
        cuda_check(cudaMemset(s, 0, nc * P * sizeof(double)), "memset");
    }
    // primitive cache: rho,u,v,(w),p = 0, T = c = 1 (solver.hpp:94-100), Y, X
    const size_t head = nz > 0 ? 7 : 6;
    const size_t nprim = head + 2 * static_cast<size_t>(ns);
    ctx->prim = dalloc(nprim * P);
    {
        std::vector<double> init(nprim * P, 0.0);
        std::fill(init.begin() + (head - 2) * P, init.begin() + head * P, 1.0);
        cuda_check(cudaMemcpy(ctx->prim, init.data(), init.size() * sizeof(double),
                              cudaMemcpyHostToDevice),
                   "cache init");
    }
    ctx->geom = dalloc((nz > 0 ? 14 : 12) * P2);
    {
        // 2D: mesh x, y in slots 10, 11 (laser); 3D: the zeta metrics there
        const std::vector<double>* f[12] = {
            &ctx->met.jac.d,    &ctx->met.m_xi_x.d,  &ctx->met.m_xi_y.d,  &ctx->met.m_eta_x.d,
            &ctx->met.m_eta_y.d, &ctx->metv.jac.d,   &ctx->metv.m_xi_x.d, &ctx->metv.m_xi_y.d,
            &ctx->metv.m_eta_x.d, &ctx->metv.m_eta_y.d, nz > 0 ? &mzz : &ctx->mesh.x.d,
            nz > 0 ? &vmzz : &ctx->mesh.y.d};
        for (int k = 0; k < 12; ++k)
            cuda_check(cudaMemcpy(ctx->geom + k * P2, f[k]->data(), P2 * sizeof(double),
                                  cudaMemcpyHostToDevice),
                       "geometry upload");
        if (nz > 0) {  // 3D: mesh x, y in slots 12, 13 (laser)
            cuda_check(cudaMemcpy(ctx->geom + 12 * P2, ctx->mesh.x.d.data(), P2 * sizeof(double),
                                  cudaMemcpyHostToDevice),
                       "geometry upload");
            cuda_check(cudaMemcpy(ctx->geom + 13 * P2, ctx->mesh.y.d.data(), P2 * sizeof(double),
                                  cudaMemcpyHostToDevice),
                       "geometry upload");
        }
    }
    const size_t nzc = nz > 0 ? nz : 1;
    ctx->Fx = dalloc(static_cast<size_t>(nc) * (nx + 1) * ny * nzc);
    ctx->Gy = dalloc(static_cast<size_t>(nc) * nx * (ny + 1) * nzc);
    if (nz > 0) ctx->Hz = dalloc(static_cast<size_t>(nc) * nx * ny * (nz + 1));
    if (cfg->viscous) {
        ctx->Fv = dalloc(nc * P);
        ctx->Gv = dalloc(nc * P);
        if (nz > 0) ctx->Hv = dalloc(nc * P);
    }
    // inflow profile tables (boundary.hpp:227-241 ghost targets)
    const ign_edge* edges[4] = {&cfg->bc.left, &cfg->bc.right, &cfg->bc.bottom, &cfg->bc.top};
    int bc_type[4] = {edges[0]->type, edges[1]->type, edges[2]->type, edges[3]->type};
    if (!three_d && ctx->lo_peer >= 0) bc_type[2] = (r == 0) ? BC_HALO_WRAP : BC_HALO;
    if (!three_d && ctx->hi_peer >= 0) bc_type[3] = (r == N - 1) ? BC_HALO_WRAP : BC_HALO;
    for (int e = 0; e < 4; ++e) {
        if (bc_type[e] != 3) continue;
        const bool xedge = e < 2;
        const int tlo = xedge ? 0 : -g, ntr = xedge ? ny : nx + 2 * g;
        std::vector<double> tab(static_cast<size_t>(ntr) * g * (3 + ns));
        for (int t = tlo; t < tlo + ntr; ++t)
            for (int k = 1; k <= g; ++k) {
                int id, jd;
                switch (e) {
                case 0: id = -k; jd = t; break;
                case 1: id = nx - 1 + k; jd = t; break;
                case 2: id = t; jd = -k; break;
                default: id = t; jd = ny - 1 + k; break;
                }
                const double yc = xedge ? ctx->mesh.eta(jd) : ctx->mesh.xi(id);
                double u, v, T, Y[kMaxSpecies];
                inflow_profile(*edges[e], yc, ns, u, v, T, Y);
                double* q = &tab[(static_cast<size_t>(t - tlo) * g + (k - 1)) * (3 + ns)];
                q[0] = u;
                q[1] = v;
                q[2] = T;
                for (int s = 0; s < ns; ++s) q[3 + s] = Y[s];
            }
        ctx->inflow[e] = dalloc(tab.size());
        cuda_check(cudaMemcpy(ctx->inflow[e], tab.data(), tab.size() * sizeof(double),
                              cudaMemcpyHostToDevice),
                   "inflow upload");
    }
    // periodic wrap across slabs: ratio J(src)/J(dst) of the reference's
    // periodic copy (boundary.hpp:146-149); src rows belong to the far slab
    const int sx = nx + 2 * g;
    for (int side = 0; side < 2; ++side) {
        if (bc_type[2 + side] != BC_HALO_WRAP) continue;
        const int NG = ctx->mesh.ny_glob;
        // dst global rows: bottom -g..-1, top NG..NG+g-1; src: NG-g..NG-1 / 0..g-1
        const int dlo = side == 0 ? -g : NG, slo = side == 0 ? NG - g : 0;
        const std::vector<double> Jd = jac_rows(ctx->mesh, imode, cfg->skew_beta, dlo, dlo + g);
        const std::vector<double> Js = jac_rows(ctx->mesh, imode, cfg->skew_beta, slo, slo + g);
        std::vector<double> tab(size_t(g) * sx);
        for (int k = 1; k <= g; ++k) {
            // ghost layer k: dst row (bottom) -k / (top) NG-1+k; src row NG-k / k-1
            const int drow = side == 0 ? -k - dlo : NG - 1 + k - dlo;
            const int srow = side == 0 ? NG - k - slo : k - 1 - slo;
            for (int t = -g; t < nx + g; ++t)
                tab[size_t(k - 1) * sx + (t + g)] =
                    Js[size_t(srow) * sx + (t + g)] / Jd[size_t(drow) * sx + (t + g)];
        }
        ctx->wrap[side] = dalloc(tab.size());
        cuda_check(cudaMemcpy(ctx->wrap[side], tab.data(), tab.size() * sizeof(double),
                              cudaMemcpyHostToDevice),
                   "wrap upload");
    }
    void* p = nullptr;
    cuda_check(cudaMalloc(&p, sizeof(ErrRec)), "cudaMalloc");
    ctx->own_err = static_cast<ErrRec*>(p);
    ctx->err = ctx->own_err;
    cuda_check(cudaMemset(ctx->err, 0xff, sizeof(ErrRec)), "memset");
    cuda_check(cudaMalloc(&p, 8 * sizeof(unsigned long long)), "cudaMalloc");
    ctx->red = static_cast<unsigned long long*>(p);
    cuda_check(cudaMemset(ctx->red, 0, 8 * sizeof(unsigned long long)), "memset");

    KParams& k = ctx->kp;
    std::memset(&k, 0, sizeof(k));
    k.nx = nx;
    k.ny = ny;
    k.g = g;
    k.sx = sx;
    k.plane = static_cast<long long>(P);
    k.j0 = ctx->mesh.j0;
    k.ny_glob = ctx->mesh.ny_glob;
    k.ns = ns;
    k.viscous = cfg->viscous;
    for (int e = 0; e < 4; ++e) {
        k.bc_type[e] = bc_type[e];
        k.T_wall[e] = edges[e]->T_wall;
        k.inflow[e] = ctx->inflow[e];
    }
    k.wrap[0] = ctx->wrap[0];
    k.wrap[1] = ctx->wrap[1];
    k.sigma_out_right = cfg->bc.right.sigma_out;
    k.p_target_right = cfg->bc.right.p_target;
    k.lodi = cfg->bc.right.type == 4;
    k.lx = cfg->lx;
    k.ly = cfg->ly;
    k.cx = cfg->center_x;
    k.cy = cfg->center_y;
    k.rp = make_recon_params(cfg->scheme.teno_ct, cfg->scheme.eps);
    k.chem_dt_limit = cfg->integ.chem_dt_limit;
    k.chem_dt_factor = cfg->integ.chem_dt_factor;
    k.prim = ctx->prim;
    k.jac = ctx->geom;
    k.mxx = ctx->geom + P2;
    k.mxy = ctx->geom + 2 * P2;
    k.mex = ctx->geom + 3 * P2;
    k.mey = ctx->geom + 4 * P2;
    k.vjac = ctx->geom + 5 * P2;
    k.vmxx = ctx->geom + 6 * P2;
    k.vmxy = ctx->geom + 7 * P2;
    k.vmex = ctx->geom + 8 * P2;
    k.vmey = ctx->geom + 9 * P2;
    if (nz > 0) {
        k.mzz = ctx->geom + 10 * P2;
        k.vmzz = ctx->geom + 11 * P2;
        k.xc = ctx->geom + 12 * P2;
        k.yc = ctx->geom + 13 * P2;
    } else {
        k.xc = ctx->geom + 10 * P2;
        k.yc = ctx->geom + 11 * P2;
    }
    k.nz = nz;
    k.nz_glob = three_d ? ctx->nz_glob : 0;
    if (three_d) {
        k.j0 = ctx->k0;  // 3D: global z offset of the slab (error keys)
        k.zhalo = ctx->lo_peer >= 0 || ctx->hi_peer >= 0;
    }
    k.sxy = static_cast<long long>(P2);
    k.Fx = ctx->Fx;
    k.Gy = ctx->Gy;
    k.Hz = ctx->Hz;
    k.Fv = ctx->Fv;
    k.Gv = ctx->Gv;
    k.Hv = ctx->Hv;
    k.err = ctx->err;
    k.red = ctx->red;
    k.mix = build_mix(cfg->mix);
    k.mech = build_mech(cfg->mech);
    k.laser = build_laser(cfg->laser);
    ctx->ks = nz > 0 ? kernel_set3(ns) : kernel_set(ns);
}

void copy_hfield(const HField& f, double* out) { std::memcpy(out, f.d.data(), f.d.size() * 8); }

void metrics_out(const HMetrics& m, double* out, size_t P) {
    const HField* f[5] = {&m.jac, &m.m_xi_x, &m.m_xi_y, &m.m_eta_x, &m.m_eta_y};
    for (int k = 0; k < 5; ++k) copy_hfield(*f[k], out + k * P);
}

// ---------------------------------------------------------------- outputs
// sample_outputs (solver.hpp:353-385): box-averaged primitives per probe (on
// the device, serial sums in the reference's j-major order, continued slab to
// slab), and the product-fraction trace.  Results live on the lead context.
void t_sample(const Team& T) {
    ign_context* L = T.lead();
    const bool want_probe = L->probe_interval > 0 && (L->iter % L->probe_interval == 0);
    const bool want_trace = L->trace_interval > 0 && (L->iter % L->trace_interval == 0);
    if (want_probe) {
        const int nq = 5 + L->ns;
        double* d = dalloc(2 * static_cast<size_t>(nq));
        try {
            for (auto& pr : L->probes) {
                std::vector<double> row(nq, 0.0);
                fold_ranks(T, row, [&](ign_context* c, std::vector<double>& a) {
                    const int jlo = std::max(pr.j0, c->mesh.j0);
                    const int jhi = std::min(pr.j1, c->mesh.j0 + c->ny - 1);
                    if (jlo > jhi) return;
                    cuda_check(cudaMemcpyAsync(d, a.data(), nq * 8, cudaMemcpyHostToDevice,
                                               c->stream), "probe");
                    launch_probe(c->prim, (long long)c->plane, c->kp.sx, c->g, c->ns, pr.i0,
                                 jlo - c->mesh.j0, pr.i1, jhi - c->mesh.j0, d, d + nq, c->stream);
                    c->launches += 1;
                    cuda_check(cudaMemcpyAsync(a.data(), d + nq, nq * 8, cudaMemcpyDeviceToHost,
                                               c->stream), "probe");
                    cuda_check(cudaStreamSynchronize(c->stream), "probe");
                });
                const int n = (pr.i1 - pr.i0 + 1) * (pr.j1 - pr.j0 + 1);
                for (auto& x : row) x /= n;
                pr.times.push_back(L->time);
                pr.rows.insert(pr.rows.end(), row.begin(), row.end());
            }
        } catch (...) {
            cudaFree(d);
            throw;
        }
        cudaFree(d);
    }
    if (want_trace) {
        L->trace_t.push_back(L->time);
        L->trace_v.push_back(t_product_fraction(T));
    }
}

// Global padded layers (2D rows / 3D planes) of the current state, gathered
// on the lead (rank 0): each slab contributes its interior layers, the first
// and last also the global edge ghosts — exactly the undecomposed planes.
// `field` selects the source: the state components (nc planes) or the T cache.
void t_gather(const Team& T, bool tcache, std::vector<double>& out) {
    ign_context* L = T.lead();
    const int N = T.local() ? (int)T.m.size() : L->nranks, g = L->g;
    const bool three_d = L->nz > 0;
    const size_t st = halo_stride(L);
    const int NG = three_d ? L->nz_glob : L->mesh.ny_glob;
    const int nf = tcache ? 1 : L->nc;
    const size_t gplane = static_cast<size_t>(NG + 2 * g) * st;
    if (!T.local() && L->rank != 0 && L->comm) {
        // non-lead rank: send its layers to rank 0
        NcclApi& n = nccl();
        const int nl = (int)halo_count(L);
        const int p0 = g, p1 = (L->rank == N - 1) ? nl + 2 * g : nl + g;
        nccl_check(n.GroupStart(), "ncclGroupStart");
        for (int c = 0; c < nf; ++c) {
            const double* src = (tcache ? L->prim + (three_d ? 5 : 4) * L->plane
                                        : L->S[L->cur] + c * L->plane) + p0 * st;
            nccl_check(n.Send(src, (p1 - p0) * st, ncclFloat64, 0, L->comm, L->stream),
                       "ncclSend(gather)");
        }
        nccl_check(n.GroupEnd(), "ncclGroupEnd");
        cuda_check(cudaStreamSynchronize(L->stream), "gather");
        return;
    }
    out.assign(static_cast<size_t>(nf) * gplane, 0.0);
    double* stage = nullptr;
    for (int r = 0; r < N; ++r) {
        int lo, nl;
        slab_rows(NG, N, r, lo, nl);
        const int p0 = r == 0 ? 0 : g, p1 = r == N - 1 ? nl + 2 * g : nl + g;
        const size_t cnt = (p1 - p0) * st;
        for (int c = 0; c < nf; ++c) {
            double* dst = out.data() + c * gplane + (lo + p0) * st;
            const ign_context* m = T.local() ? T.m[r] : L;
            if (T.local() || r == 0) {
                const double* src = (tcache ? m->prim + (three_d ? 5 : 4) * m->plane
                                            : m->S[m->cur] + c * m->plane) + p0 * st;
                cuda_check(cudaMemcpy(dst, src, cnt * 8, cudaMemcpyDeviceToHost), "gather");
            } else {
                if (!stage) stage = dalloc(static_cast<size_t>(NG / N + 2 + 2 * g) * st);
                NcclApi& n = nccl();
                nccl_check(n.Recv(stage, cnt, ncclFloat64, r, L->comm, L->stream),
                           "ncclRecv(gather)");
                cuda_check(cudaMemcpyAsync(dst, stage, cnt * 8, cudaMemcpyDeviceToHost, L->stream),
                           "gather");
                cuda_check(cudaStreamSynchronize(L->stream), "gather");
            }
        }
    }
    if (stage) cudaFree(stage);
}

// write_snapshot (snapshot.hpp:52-76): version 1 = the reference's format
// (2D); version 2 adds nz (3D) and, with `with_t`, the T cache
void t_write_snapshot(const Team& T, const std::string& path, int version, bool with_t) {
    ign_context* L = T.lead();
    const bool three_d = L->nz > 0;
    if (three_d && version < 2) throw usage_error("snapshot: 3D state needs IGNS version 2");
    if (version != 1 && version != 2) throw usage_error("snapshot: version must be 1 or 2");
    Snapshot s;
    t_gather(T, false, s.state);
    if (with_t) t_gather(T, true, s.tcache);
    if (!T.local() && L->rank != 0 && L->comm) return;  // rank 0 writes
    s.version = (uint32_t)version;
    s.nx = L->nx;
    s.ny = three_d ? L->ny : L->mesh.ny_glob;
    s.g = L->g;
    s.ns = L->ns;
    s.nz = three_d ? L->nz_glob : 0;
    for (int k = 0; k < L->ns; ++k)
        s.species.emplace_back(L->cfg.mix.species[k].name,
                               strnlen(L->cfg.mix.species[k].name, IGN_NAME_LEN));
    s.time = L->time;
    s.iteration = L->iter;
    s.config_hash = L->config_hash;
    s.flags = with_t ? 1u : 0u;
    // J over the global padded rows (2D: the reference's met.jac; 3D: the
    // extruded J of every z plane)
    const int g = L->g, NG = s.ny;
    if (three_d || L->nranks == 1)
        s.jac = L->met.jac.d;  // the whole (x, y) plane already
    else                       // 2D slabs: the global rows, global stencils
        s.jac = jac_rows(L->mesh, inviscid_metric_mode(L->cfg), L->cfg.skew_beta, -g, NG + g);
    snapshot_write(s, path);
}

// read_snapshot + apply_snapshot (snapshot.hpp:78-145): every slab reads the
// file and takes its own layers; time, iteration and hash are restored, the
// T cache too when the file carries it (v2)
void t_read_snapshot(const Team& T, const std::string& path) {
    ign_context* L = T.lead();
    const Snapshot s = snapshot_read(path);
    const bool three_d = L->nz > 0;
    const int NG = three_d ? L->nz_glob : L->mesh.ny_glob;
    const int sny = three_d ? L->ny : L->mesh.ny_glob;
    if (s.nx != L->nx || s.ny != sny || s.g != L->g || s.nz != (three_d ? L->nz_glob : 0))
        throw Error(IGN_FORMAT_ERROR,
                    "snapshot: shape mismatch, file " + std::to_string(s.nx) + "x" +
                        std::to_string(s.ny) + " (g=" + std::to_string(s.g) +
                        ") vs simulation " + std::to_string(L->nx) + "x" + std::to_string(sny) +
                        " (g=" + std::to_string(L->g) + ")");
    if (s.ns != L->ns) throw Error(IGN_FORMAT_ERROR, "snapshot: species count mismatch");
    for (int k = 0; k < s.ns; ++k)
        if (s.species[k] != std::string(L->cfg.mix.species[k].name,
                                        strnlen(L->cfg.mix.species[k].name, IGN_NAME_LEN)))
            throw Error(IGN_FORMAT_ERROR,
                        "snapshot: species name mismatch at slot " + std::to_string(k));
    const size_t st = halo_stride(L);
    const size_t gplane = static_cast<size_t>(NG + 2 * L->g) * st;
    for (ign_context* c : T.m) {
        const int lo = three_d ? c->k0 : c->mesh.j0;  // global interior start
        const size_t cnt = (halo_count(c) + 2 * c->g) * st;
        for (int comp = 0; comp < c->nc; ++comp)
            cuda_check(cudaMemcpy(c->S[c->cur] + comp * c->plane,
                                  s.state.data() + comp * gplane + lo * st, cnt * 8,
                                  cudaMemcpyHostToDevice),
                       "snapshot upload");
        if (s.flags & 1u)
            cuda_check(cudaMemcpy(c->prim + (three_d ? 5 : 4) * c->plane,
                                  s.tcache.data() + lo * st, cnt * 8, cudaMemcpyHostToDevice),
                       "snapshot upload");
        c->time = s.time;
        c->iter = s.iteration;
        c->config_hash = s.config_hash;
    }
}

// advance (solver.hpp:336-349) over a team, sampling probes and the trace
void t_advance(const Team& T, ign_step_hook hook, void* user) {
    ign_context* L = T.lead();
    t_prepare_sync(T, 1);
    t_sample(T);
    const ign_integrator& in = L->integ;
    const double t_eps = 1e-12 * std::max(1.0, std::abs(in.t_end));
    const bool sampling = (L->probe_interval > 0 && !L->probes.empty()) || L->trace_interval > 0;
    if (in.fixed_dt > 0.0 && !hook) {
        // pinned step, no hook: the step count is known up front; runs are cut
        // at the sampling iterations
        int64_t n = 0;
        double t = L->time;
        int64_t it = L->iter;
        while (it < in.max_iter && t < in.t_end - t_eps) {
            t += in.fixed_dt;
            ++it;
            ++n;
        }
        while (n > 0) {
            int64_t k = n;
            if (sampling) {
                for (int iv : {L->probe_interval, L->trace_interval}) {
                    if (iv <= 0) continue;
                    const int64_t to_next = iv - (L->iter % iv);
                    k = std::min(k, to_next);
                }
            }
            t_run_steps(T, in.fixed_dt, k, true);
            n -= k;
            if (sampling) t_sample(T);
        }
        return;
    }
    while (L->iter < in.max_iter && L->time < in.t_end - t_eps) {
        double dt = in.fixed_dt > 0.0 ? in.fixed_dt : t_stable_dt(T);
        if (in.fixed_dt <= 0.0) dt = smin(dt, in.t_end - L->time);
        t_run_steps(T, dt, 1, false);
        t_prepare_sync(T, 1);
        t_sample(T);
        if (hook) hook(L, user);
    }
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

uint64_t ign_config_size(void) { return sizeof(ign_config); }

int ign_create(const ign_config* cfg, ign_context** out) {
    if (!out) return IGN_USAGE_ERROR;
    *out = nullptr;
    ign_context* ctx = new ign_context();
    const int st = guarded_err(nullptr, -1, [&] { create_impl(cfg, ctx); });
    if (st != IGN_OK) {
        destroy_impl(ctx);
        return st;
    }
    *out = ctx;
    return IGN_OK;
}

void ign_destroy(ign_context* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->group) return;  // owned by its group until ign_group_destroy
    destroy_impl(ctx);
}

int ign_last_error(const ign_context* ctx, ign_error* err) {
    if (!ctx || !err) return IGN_USAGE_ERROR;
    *err = ctx->lasterr;
    return IGN_OK;
}

int ign_dims(const ign_context* ctx, int32_t* nx, int32_t* ny, int32_t* g, int32_t* ns) {
    *nx = ctx->nx;
    *ny = ctx->ny;
    *g = ctx->g;
    *ns = ctx->ns;
    return IGN_OK;
}

int ign_get_mesh(const ign_context* ctx, double* x, double* y) {
    copy_hfield(ctx->mesh.x, x);
    copy_hfield(ctx->mesh.y, y);
    return IGN_OK;
}

int ign_dims3(const ign_context* ctx, int32_t* nz, int32_t* k0, int32_t* nz_glob) {
    if (nz) *nz = ctx->nz;
    if (k0) *k0 = ctx->k0;
    if (nz_glob) *nz_glob = ctx->nz_glob;
    return IGN_OK;
}

int ign_get_metrics(const ign_context* ctx, int which, double* out) {
    const HMetrics& m = which == 0 ? ctx->met : ctx->metv;
    metrics_out(m, out, m.jac.d.size());
    return IGN_OK;
}

int ign_set_initial_condition(ign_context* ctx, ign_ic_fn fn, void* user) {
    return guarded_err(&ctx->lasterr, ctx->device, [&] {
        if (ctx->nz > 0) throw usage_error("3D: use ign_set_initial_primitives");
        const int g = ctx->g, nc = ctx->nc;
        const size_t P = ctx->plane;
        std::vector<double> Ut(nc * P);
        size_t k = 0;
        for (int j = -g; j < ctx->ny + g; ++j)
            for (int i = -g; i < ctx->nx + g; ++i, ++k) {
                ign_prim_point q{};
                fn(ctx->mesh.x(i, j), ctx->mesh.y(i, j), user, &q);
                double U[kMaxComp];
                cons_from_prim(ctx->kp.mix, q.rho, q.u, q.v, q.T, q.Y, U);
                const double invJ = 1.0 / ctx->met.jac(i, j);
                for (int c = 0; c < nc; ++c) Ut[c * P + k] = U[c] * invJ;
            }
        upload_state(ctx, Ut);
    });
}

int ign_set_initial_primitives(ign_context* ctx, const double* prim) {
    return guarded_err(&ctx->lasterr, ctx->device, [&] {
        const int ns = ctx->ns, nc = ctx->nc;
        const size_t P = ctx->plane, P2 = ctx->met.jac.d.size();
        std::vector<double> Ut(nc * P);
        for (size_t k = 0; k < P; ++k) {
            double U[kMaxComp + 1];
            if (ctx->nz > 0) {  // rho, u, v, w, T, Y_s
                Prim3<kMaxSpecies> pt{};
                pt.rho = prim[k];
                pt.u = prim[P + k];
                pt.v = prim[2 * P + k];
                pt.w = prim[3 * P + k];
                pt.T = prim[4 * P + k];
                double Y[kMaxSpecies];
                for (int s = 0; s < ns; ++s) Y[s] = prim[(5 + s) * P + k];
                cons_from_prim3(ctx->kp.mix, pt, Y, U);
            } else {
                double Y[kMaxSpecies];
                for (int s = 0; s < ns; ++s) Y[s] = prim[(4 + s) * P + k];
                cons_from_prim(ctx->kp.mix, prim[k], prim[P + k], prim[2 * P + k],
                               prim[3 * P + k], Y, U);
            }
            const double invJ = 1.0 / ctx->met.jac.d[k % P2];
            for (int c = 0; c < nc; ++c) Ut[c * P + k] = U[c] * invJ;
        }
        upload_state(ctx, Ut);
    });
}

int ign_set_state(ign_context* ctx, const double* Ut, const double* Tc) {
    return guarded_err(&ctx->lasterr, ctx->device, [&] {
        cuda_check(cudaMemcpy(ctx->S[ctx->cur], Ut, ctx->nc * ctx->plane * sizeof(double),
                              cudaMemcpyHostToDevice),
                   "set_state");
        if (Tc)
            cuda_check(cudaMemcpy(ctx->prim + (ctx->nz > 0 ? 5 : 4) * ctx->plane, Tc,
                                  ctx->plane * sizeof(double),
                                  cudaMemcpyHostToDevice),
                       "set_state T");
    });
}

int ign_get_state(ign_context* ctx, double* Ut) {
    return guarded_err(&ctx->lasterr, ctx->device, [&] {
        cuda_check(cudaMemcpy(Ut, ctx->S[ctx->cur], ctx->nc * ctx->plane * sizeof(double),
                              cudaMemcpyDeviceToHost),
                   "get_state");
    });
}

int ign_get_cache(ign_context* ctx, double* prim) {
    return guarded_err(&ctx->lasterr, ctx->device, [&] {
        cuda_check(cudaMemcpy(prim, ctx->prim,
                              ((ctx->nz > 0 ? 7 : 6) + ctx->ns) * ctx->plane * sizeof(double),
                              cudaMemcpyDeviceToHost),
                   "get_cache");
    });
}

int ign_get_time(const ign_context* ctx, double* t, int64_t* it) {
    *t = ctx->time;
    *it = ctx->iter;
    return IGN_OK;
}

int ign_set_time(ign_context* ctx, double t, int64_t it) {
    ctx->time = t;
    ctx->iter = it;
    return IGN_OK;
}

int ign_set_integrator(ign_context* ctx, const ign_integrator* in) {
    ctx->integ = *in;
    ctx->kp.chem_dt_limit = in->chem_dt_limit;
    ctx->kp.chem_dt_factor = in->chem_dt_factor;
    return IGN_OK;
}

int ign_refill_ghosts(ign_context* ctx) {
    return guarded(ctx, [&] {
        const Team T = solo(ctx);
        ctx->launches += ctx->ks.bc(ctx->kp, ctx->S[ctx->cur], 0, 0, 0, ctx->stream);
        t_exchange(T, ctx->cur);
        ctx->launches += ctx->ks.bc(ctx->kp, ctx->S[ctx->cur], 1, 0, 0, ctx->stream);
        t_errsync(T);
        check(T);
    });
}

int ign_refresh_primitives(ign_context* ctx, int stage) {
    return guarded(ctx, [&] {
        ctx->launches += ctx->ks.prim(ctx->kp, ctx->S[ctx->cur], stage, 0, ctx->stream);
        t_errsync(solo(ctx));
        check(solo(ctx));
    });
}

int ign_prepare_stage(ign_context* ctx, int stage) {
    return guarded(ctx, [&] { t_prepare_sync(solo(ctx), stage); });
}

int ign_compute_rhs(ign_context* ctx, double t_stage, int stage, double* rhs) {
    return guarded(ctx, [&] {
        const Team T = solo(ctx);
        const size_t n = ctx->nc * ctx->plane;
        if (!ctx->rhs) ctx->rhs = dalloc(n);
        cuda_check(cudaMemsetAsync(ctx->rhs, 0, n * sizeof(double), ctx->stream), "memset");
        const double* U = ctx->S[ctx->cur];
        t_fluxes(T, ctx->cur, stage, 0);
        ctx->launches += timed(ctx, IGN_PROF_ASSEMBLE, [&] {
            return ctx->ks.assemble(ctx->kp, 0, U, U, ctx->rhs, 0.0, 0.0, t_stage, stage, 0, 0,
                                    ctx->stream);
        });
        t_errsync(T);
        check(T);
        if (rhs)
            cuda_check(cudaMemcpy(rhs, ctx->rhs, n * sizeof(double), cudaMemcpyDeviceToHost),
                       "rhs readback");
    });
}

int ign_stable_dt(ign_context* ctx, double* dt) {
    return guarded(ctx, [&] { *dt = t_stable_dt(solo(ctx)); });
}

int ign_rk3_step(ign_context* ctx, double dt) {
    return guarded(ctx, [&] { t_run_steps(solo(ctx), dt, 1, false); });
}

int ign_rk3_steps(ign_context* ctx, double dt, int64_t n) {
    return guarded(ctx, [&] { t_run_steps(solo(ctx), dt, n, true); });
}

int ign_ensemble_rk3_steps(ign_context** members, int n, const double* dt, int64_t nsteps,
                           int* status) {
    if (!members || n <= 0 || !dt || !status) return IGN_USAGE_ERROR;
    for (int q = 0; q < n; ++q)
        if (!members[q] || members[q]->nranks > 1 || members[q]->device != members[0]->device)
            return IGN_USAGE_ERROR;
    try {
        cuda_check(cudaSetDevice(members[0]->device), "cudaSetDevice");
        t_run_ensemble(std::vector<ign_context*>(members, members + n), dt, nsteps, status);
    } catch (const Error& e) {
        return e.status;
    } catch (const std::exception& e) {
        return IGN_INTERNAL_ERROR;
    }
    int worst = IGN_OK;
    for (int q = 0; q < n; ++q)
        if (status[q] != IGN_OK) worst = status[q];
    return worst;
}

int ign_advance(ign_context* ctx, ign_step_hook hook, void* user) {
    return guarded(ctx, [&] { t_advance(solo(ctx), hook, user); });
}

// ---- outputs: probes, trace, snapshots (solver.hpp:68-74, 130-135, 351-385;
// snapshot.hpp)
int ign_add_probe(ign_context* ctx, int32_t i0, int32_t j0, int32_t i1, int32_t j1) {
    return guarded_err(&ctx->lasterr, ctx->device, [&] {
        if (ctx->nz > 0) throw usage_error("probes: the 3D extension has no probe boxes");
        const int nyg = ctx->mesh.ny_glob;
        if (i0 < 0 || j0 < 0 || i1 >= ctx->nx || j1 >= nyg || i0 > i1 || j0 > j1)
            throw config_error("probe box out of range");
        ctx->probes.push_back(ign_context::Probe{i0, j0, i1, j1, {}, {}});
    });
}

int ign_set_sampling(ign_context* ctx, int32_t probe_interval, int32_t trace_interval) {
    ctx->probe_interval = probe_interval;
    ctx->trace_interval = trace_interval;
    return IGN_OK;
}

int ign_probe_samples(const ign_context* ctx, int32_t probe, int64_t* n, double* times,
                      double* rows) {
    if (probe < 0 || probe >= (int)ctx->probes.size()) return IGN_USAGE_ERROR;
    const auto& pr = ctx->probes[probe];
    if (n) *n = (int64_t)pr.times.size();
    if (times) std::memcpy(times, pr.times.data(), pr.times.size() * 8);
    if (rows) std::memcpy(rows, pr.rows.data(), pr.rows.size() * 8);
    return IGN_OK;
}

int ign_trace_samples(const ign_context* ctx, int64_t* n, double* times, double* values) {
    if (n) *n = (int64_t)ctx->trace_t.size();
    if (times) std::memcpy(times, ctx->trace_t.data(), ctx->trace_t.size() * 8);
    if (values) std::memcpy(values, ctx->trace_v.data(), ctx->trace_v.size() * 8);
    return IGN_OK;
}

int ign_set_config_hash(ign_context* ctx, uint64_t hash) {
    ctx->config_hash = hash;
    return IGN_OK;
}

int ign_get_config_hash(const ign_context* ctx, uint64_t* hash) {
    *hash = ctx->config_hash;
    return IGN_OK;
}

int ign_write_snapshot(ign_context* ctx, const char* path) {
    return guarded(ctx, [&] {
        t_write_snapshot(solo(ctx), path ? path : "", ctx->nz > 0 ? 2 : 1, false);
    });
}

int ign_write_snapshot_v2(ign_context* ctx, const char* path, int with_t) {
    return guarded(ctx, [&] { t_write_snapshot(solo(ctx), path ? path : "", 2, with_t != 0); });
}

int ign_read_snapshot(ign_context* ctx, const char* path) {
    return guarded(ctx, [&] { t_read_snapshot(solo(ctx), path ? path : ""); });
}

int ign_conserved_totals(ign_context* ctx, double* tot) {
    return guarded(ctx, [&] { t_conserved_totals(solo(ctx), tot); });
}

int ign_product_mole_fraction(ign_context* ctx, double* out) {
    return guarded(ctx, [&] { *out = t_product_fraction(solo(ctx)); });
}

int ign_last_clip(const ign_context* ctx, double* clip) {
    *clip = ctx->last_clip;
    return IGN_OK;
}

int ign_host_metrics(const ign_config* cfg, int which, double* out, ign_error* err) {
    return guarded_err(err, -1, [&] {
        const int nr = cfg->slab_count > 1 ? cfg->slab_count : 1;
        const HMesh m = build_mesh(*cfg, nr, nr > 1 ? cfg->slab_rank : 0);
        const HMetrics mf = which == 0 ? compute_metrics(m, inviscid_metric_mode(*cfg), cfg->skew_beta)
                                       : compute_metrics(m, MM_CENTRAL2, 0.0);
        metrics_out(mf, out, mf.jac.d.size());
    });
}

int ign_host_mesh(const ign_config* cfg, double* x, double* y, ign_error* err) {
    return guarded_err(err, -1, [&] {
        const int nr = cfg->slab_count > 1 ? cfg->slab_count : 1;
        const HMesh m = build_mesh(*cfg, nr, nr > 1 ? cfg->slab_rank : 0);
        copy_hfield(m.x, x);
        copy_hfield(m.y, y);
    });
}

int64_t ign_kernel_launches(const ign_context* ctx) { return ctx ? ctx->launches : 0; }

int ign_profile_enable(ign_context* ctx, int on) {
    return guarded_err(&ctx->lasterr, ctx->device, [&] {
        cuda_check(cudaStreamSynchronize(ctx->stream), "sync");
        prof_harvest(ctx);
        ctx->prof_on = on != 0;
        for (int k = 0; k < IGN_PROF_CLASSES; ++k) {
            ctx->prof_ms[k] = 0.0;
            ctx->prof_n[k] = 0;
        }
    });
}

int ign_profile_read(ign_context* ctx, double* ms, int64_t* counts) {
    return guarded_err(&ctx->lasterr, ctx->device, [&] {
        cuda_check(cudaStreamSynchronize(ctx->stream), "sync");
        prof_harvest(ctx);
        for (int k = 0; k < IGN_PROF_CLASSES; ++k) {
            ms[k] = ctx->prof_ms[k];
            counts[k] = ctx->prof_n[k];
        }
    });
}

void* ign_stream_handle(const ign_context* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

// ---------------------------------------------------------------- slabs over NCCL
int ign_nccl_unique_id(uint8_t* id) {
    ign_error e{};
    return guarded_err(&e, -1, [&] {
        if (!nccl().ok) throw Error(IGN_CUDA_ERROR, nccl().why);
        ncclUniqueId u;
        nccl_check(nccl().GetUniqueId(&u), "ncclGetUniqueId");
        std::memcpy(id, u.internal, IGN_NCCL_ID_BYTES);
    });
}

int ign_attach_nccl(ign_context* ctx, const uint8_t* id, int nranks, int rank) {
    return guarded(ctx, [&] {
        if (!nccl().ok) throw Error(IGN_CUDA_ERROR, nccl().why);
        if (nranks != ctx->nranks || rank != ctx->rank)
            throw usage_error("ign_attach_nccl: rank/size differ from the slab config");
        ncclUniqueId u;
        std::memcpy(u.internal, id, IGN_NCCL_ID_BYTES);
        nccl_check(nccl().CommInitRank(&ctx->comm, nranks, u, rank), "ncclCommInitRank");
    });
}

// ---------------------------------------------------------------- single-process groups
int ign_group_create(ign_context** members, int n, ign_group** out) {
    ign_error e{};
    *out = nullptr;
    auto* grp = new ign_group();
    const int st = guarded_err(&e, members && n > 0 ? members[0]->device : -1, [&] {
        if (n < 1) throw usage_error("ign_group_create: empty group");
        for (int r = 0; r < n; ++r) {
            ign_context* c = members[r];
            if (!c || c->nranks != n || c->rank != r || c->device != members[0]->device ||
                c->group || c->comm)
                throw usage_error("ign_group_create: members must be slabs 0..n-1 of one config");
        }
        for (int r = 0; r < n; ++r) {
            ign_context* c = members[r];
            c->group = grp;
            c->stream = members[0]->own_stream;  // lockstep on one stream
            c->err = members[0]->own_err;        // one error word for the group
            c->kp.err = c->err;
            grp->m.push_back(c);
        }
    });
    if (st != IGN_OK) {
        delete grp;
        return st;
    }
    *out = grp;
    return IGN_OK;
}

void ign_group_destroy(ign_group* grp) {
    if (!grp) return;
    for (ign_context* c : grp->m) {
        cudaSetDevice(c->device);
        c->group = nullptr;
        destroy_impl(c);
    }
    delete grp;
}

int ign_group_last_error(const ign_group* grp, ign_error* err) {
    *err = grp->lasterr;
    return IGN_OK;
}

static int group_guarded(ign_group* grp, const std::function<void(const Team&)>& f) {
    return guarded_err(&grp->lasterr, grp->m[0]->device, [&] { f(Team{grp->m}); });
}

int ign_group_prepare_stage(ign_group* grp, int stage) {
    return group_guarded(grp, [&](const Team& T) { t_prepare_sync(T, stage); });
}

int ign_group_rk3_steps(ign_group* grp, double dt, int64_t n) {
    return group_guarded(grp, [&](const Team& T) { t_run_steps(T, dt, n, true); });
}

int ign_group_stable_dt(ign_group* grp, double* dt) {
    return group_guarded(grp, [&](const Team& T) { *dt = t_stable_dt(T); });
}

int ign_group_conserved_totals(ign_group* grp, double* tot) {
    return group_guarded(grp, [&](const Team& T) { t_conserved_totals(T, tot); });
}

int ign_group_advance(ign_group* grp) {
    return group_guarded(grp, [&](const Team& T) { t_advance(T, nullptr, nullptr); });
}

int ign_group_write_snapshot(ign_group* grp, const char* path, int version, int with_t) {
    return group_guarded(grp, [&](const Team& T) {
        t_write_snapshot(T, path ? path : "", version, with_t != 0);
    });
}

int ign_group_read_snapshot(ign_group* grp, const char* path) {
    return group_guarded(grp, [&](const Team& T) { t_read_snapshot(T, path ? path : ""); });
}

}  // extern "C"
