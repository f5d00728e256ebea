// runtime.cu — NCCL binding, device-error decoding and the stage
// orchestration of a team (one context, an NCCL slab of a decomposed domain,
// or a single-process group of slabs): ghost fill, halo exchange, primitives,
// faces, viscous fluxes, update; RK3 steps in chunks between host syncs;
// stable_dt; advance; the ensemble runner.
#include "context_internal.hpp"

#include <cstdlib>
#include <mutex>
#include <unordered_map>

namespace ign {
namespace rt {

// ---------------------------------------------------------------- NCCL (dlopen)
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
    out->k = e.k;
    std::snprintf(out->msg, sizeof(out->msg), "%s", e.what());
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

// ---------------------------------------------------------------- allocation
// Red-zone guard mode (IGN_GUARD=1 in the environment when a buffer is
// allocated).  compute-sanitizer is closed on the GPU pool, so out-of-bounds
// accesses are caught by the allocator instead: every device buffer of a
// context gets kGuardWords words of canary on each side — a signalling-NaN bit
// pattern, so a kernel that READS past a buffer and uses the value turns the
// step non-finite (the error word / the oracle parity catch it), and a kernel
// that WRITES past one changes a canary, which dfree() and ign_guard_status()
// count.  The buffer itself starts filled with the same NaN, so a read of a
// word nothing wrote shows up the same way.  Off by default (the product
// allocates exactly what it uses).
namespace {
constexpr size_t kGuardWords = 4096;  // 32 KB per side: the user pointer keeps 32 KB alignment
constexpr unsigned long long kCanary = 0x7ff4dead0badf00dull;
struct GuardRec {
    char* base;
    size_t words;  // user words (bytes rounded up to 8)
};
std::mutex g_guard_mu;
std::unordered_map<void*, GuardRec> g_guard_live;
unsigned long long g_guard_checked = 0, g_guard_bad = 0;

bool guard_on() {
    const char* e = std::getenv("IGN_GUARD");
    return e && *e && *e != '0';
}

// canary words changed in the two zones of one buffer
unsigned long long guard_scan(const GuardRec& r) {
    std::vector<unsigned long long> h(kGuardWords);
    unsigned long long bad = 0;
    for (int side = 0; side < 2; ++side) {
        const char* z = r.base + (side ? (kGuardWords + r.words) * 8 : 0);
        cuda_check(cudaMemcpy(h.data(), z, kGuardWords * 8, cudaMemcpyDeviceToHost),
                   "guard scan");
        for (unsigned long long w : h) bad += w != kCanary;
    }
    return bad;
}
}  // namespace

// guard mode: the user region starts poisoned too (the same signalling NaN),
// so a kernel that reads a word nothing wrote turns the step non-finite
__global__ void k_poison(unsigned long long* p, size_t n) {
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n;
         q += (size_t)gridDim.x * blockDim.x)
        p[q] = kCanary;
}

void* dmalloc(size_t bytes) {
    bytes = std::max<size_t>(bytes, 1);
    if (!guard_on()) {
        void* p = nullptr;
        cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
        return p;
    }
    GuardRec r{nullptr, (bytes + 7) / 8};
    void* b = nullptr;
    cuda_check(cudaMalloc(&b, (2 * kGuardWords + r.words) * 8), "cudaMalloc");
    r.base = static_cast<char*>(b);
    const std::vector<unsigned long long> can(kGuardWords, kCanary);
    cuda_check(cudaMemcpy(r.base, can.data(), kGuardWords * 8, cudaMemcpyHostToDevice), "guard");
    cuda_check(cudaMemcpy(r.base + (kGuardWords + r.words) * 8, can.data(), kGuardWords * 8,
                          cudaMemcpyHostToDevice),
               "guard");
    k_poison<<<1184, 256>>>(reinterpret_cast<unsigned long long*>(r.base + kGuardWords * 8),
                            r.words);
    cuda_check(cudaGetLastError(), "guard poison");
    cuda_check(cudaDeviceSynchronize(), "guard");  // canaries in place before any kernel
    void* user = r.base + kGuardWords * 8;
    std::lock_guard<std::mutex> lk(g_guard_mu);
    g_guard_live[user] = r;
    return user;
}

double* dalloc(size_t n) { return static_cast<double*>(dmalloc(n * sizeof(double))); }

// Host -> device upload ordered on the context's stream.  The context's
// stream is non-blocking, so it is NOT ordered after the legacy default
// stream: a plain cudaMemcpy from pageable memory may return before its DMA
// lands, and the next kernel on the stream could read the old contents.
// The stream sync also makes the host buffer reusable on return.
void h2d(ign_context* c, void* dst, const void* src, size_t bytes, const char* what) {
    cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream), what);
    cuda_check(cudaStreamSynchronize(c->stream), what);
}

// Device -> host read after the context's stream has drained (the legacy
// stream a plain cudaMemcpy runs on does not wait for the non-blocking one).
void d2h(const ign_context* c, void* dst, const void* src, size_t bytes, const char* what) {
    cuda_check(cudaStreamSynchronize(c->stream), what);
    cuda_check(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost), what);
}

// Frees a dmalloc() buffer (nullptr is a no-op); a guarded one has its canaries
// checked first (the device is synchronised so pending kernels have written).
void dfree(void* p) {
    if (!p) return;
    GuardRec r{nullptr, 0};
    {
        std::lock_guard<std::mutex> lk(g_guard_mu);
        auto it = g_guard_live.find(p);
        if (it != g_guard_live.end()) {
            r = it->second;
            g_guard_live.erase(it);
        }
    }
    if (!r.base) {
        cudaFree(p);
        return;
    }
    unsigned long long bad = 0;
    if (cudaDeviceSynchronize() == cudaSuccess) {
        try {
            bad = guard_scan(r);
        } catch (const Error&) {
        }
    }
    {
        std::lock_guard<std::mutex> lk(g_guard_mu);
        ++g_guard_checked;
        g_guard_bad += bad;
        if (bad) std::fprintf(stderr, "ignis_b200 guard: %llu canary words overwritten around a "
                                      "%zu-byte buffer\n", bad, r.words * 8);
    }
    cudaFree(r.base);
}

// Scans every live guarded buffer (of the current device) and reports the
// totals including freed buffers.
void guard_status(int* enabled, unsigned long long* checked, unsigned long long* bad) {
    std::vector<GuardRec> live;
    {
        std::lock_guard<std::mutex> lk(g_guard_mu);
        for (auto& kv : g_guard_live) live.push_back(kv.second);
    }
    cuda_check(cudaDeviceSynchronize(), "guard sync");
    unsigned long long b = 0, n = 0;
    for (const GuardRec& r : live) {
        cudaPointerAttributes a{};
        int dev = -1;
        cudaGetDevice(&dev);
        if (cudaPointerGetAttributes(&a, r.base) != cudaSuccess || a.device != dev) continue;
        b += guard_scan(r);
        ++n;
    }
    std::lock_guard<std::mutex> lk(g_guard_mu);
    if (enabled) *enabled = guard_on() ? 1 : 0;
    if (checked) *checked = g_guard_checked + n;
    if (bad) *bad = g_guard_bad + b;
}

// Self-test of the detector: one guarded buffer, one word written past its end
// and one before its start; returns the canary words the scan saw changed (2).
unsigned long long guard_selftest() {
    GuardRec r{nullptr, 3};
    void* b = nullptr;
    cuda_check(cudaMalloc(&b, (2 * kGuardWords + r.words) * 8), "cudaMalloc");
    r.base = static_cast<char*>(b);
    const std::vector<unsigned long long> can(2 * kGuardWords + r.words, kCanary);
    cuda_check(cudaMemcpy(r.base, can.data(), can.size() * 8, cudaMemcpyHostToDevice), "guard");
    double* user = reinterpret_cast<double*>(r.base + kGuardWords * 8);
    cuda_check(cudaMemset(user + r.words, 0, 8), "guard");  // one past the end
    cuda_check(cudaMemset(user - 1, 0, 8), "guard");        // one before the start
    const unsigned long long bad = guard_scan(r);
    cudaFree(b);
    return bad;
}

// ---------------------------------------------------------------- teams

// Decoded device failure (key layout: kernels_common.cuh report()).

// Every rank reads the same (MIN-reduced) error word: a failure in the last
// kernels before this point (e.g. a step's final update) is seen everywhere.
DevFail sync_and_read(const Team& T) {
    t_join(T);
    t_errsync(T);
    cuda_check(cudaStreamSynchronize(T.stream()), "kernel execution");
    cuda_check(cudaGetLastError(), "kernel launch");
    for (ign_context* c : T.m) prof_harvest(c);
    ErrRec h{kNoError};
    for (ign_context* c : T.m) {  // NCCL: one (all-reduced) word; group: MIN over slabs
        ErrRec w;
        cuda_check(cudaMemcpy(&w, c->err, sizeof(w), cudaMemcpyDeviceToHost), "error word");
        h.key = std::min(h.key, w.key);
    }
    DevFail f;
    if (h.key == kNoError) return f;
    f.any = true;
    f.step = (int)(h.key >> 44);
    f.stage = (unsigned)((h.key >> 41) & 7);
    f.phase = (unsigned)((h.key >> 38) & 7);
    f.idx = (h.key >> 3) & ((1ull << 35) - 1);
    f.sub = (unsigned)(h.key & 7);
    for (ign_context* c : T.m)
        cuda_check(cudaMemsetAsync(c->own_err, 0xff, sizeof(ErrRec), c->stream), "error reset");
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
                                rep_stage, i, j, k);
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
        const int k = ctx->nz > 0 ? (int)(cell / ((unsigned long long)ctx->nx * ctx->ny)) : 0;
        return step_failure("non-finite RHS", rep_stage, i, j, k);
    }
    default: {
        const unsigned long long cell = f.idx / 2;
        const int i = (int)(cell % ctx->nx);
        const int j = (int)(ctx->nz > 0 ? (cell / ctx->nx) % ctx->ny : cell / ctx->nx);
        const int k = ctx->nz > 0 ? (int)(cell / ((unsigned long long)ctx->nx * ctx->ny)) : 0;
        return step_failure(f.idx % 2 ? "non-finite state" : "non-positive density", rep_stage,
                            i, j, k);
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
void t_exchange(const Team& T, int buf, cudaStream_t stream) {
    if (T.local()) {
        for (ign_context* c : T.m) {
            const size_t st = halo_stride(c), chunk = size_t(c->g) * st;
            for (int comp = 0; comp < c->nc; ++comp) {
                if (c->lo_peer >= 0) {
                    const ign_context* s = T.m[c->lo_peer];
                    cuda_check(cudaMemcpyAsync(c->S[buf] + comp * c->plane,
                                               s->S[buf] + comp * s->plane + halo_count(s) * st,
                                               chunk * sizeof(double), cudaMemcpyDeviceToDevice,
                                               stream),
                               "halo copy");
                }
                if (c->hi_peer >= 0) {
                    const ign_context* s = T.m[c->hi_peer];
                    cuda_check(cudaMemcpyAsync(c->S[buf] + comp * c->plane +
                                                   (halo_count(c) + c->g) * st,
                                               s->S[buf] + comp * s->plane + chunk,
                                               chunk * sizeof(double), cudaMemcpyDeviceToDevice,
                                               stream),
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
                              c->comm, stream), "ncclSend");
        if (c->lo_peer >= 0)
            nccl_check(n.Send(base + chunk, chunk, ncclFloat64, c->lo_peer, c->comm, stream),
                       "ncclSend");
        if (c->lo_peer >= 0)
            nccl_check(n.Recv(base, chunk, ncclFloat64, c->lo_peer, c->comm, stream),
                       "ncclRecv");
        if (c->hi_peer >= 0)
            nccl_check(n.Recv(base + (nl + c->g) * st, chunk, ncclFloat64,
                              c->hi_peer, c->comm, stream), "ncclRecv");
    }
    nccl_check(n.GroupEnd(), "ncclGroupEnd");
}

bool t_has_halo(const Team& T) {
    for (const ign_context* c : T.m)
        if (c->lo_peer >= 0 || c->hi_peer >= 0) return true;
    return false;
}

// The halo overlap can be switched off (IGN_HALO_OVERLAP=0) to compare the
// two schedules; results are bitwise identical either way.
static bool overlap_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("IGN_HALO_OVERLAP");
        return !(e && e[0] == '0');
    }();
    return on;
}

static void ensure_halo_stream(ign_context* L) {
    if (L->halo_stream) return;
    cuda_check(cudaStreamCreateWithFlags(&L->halo_stream, cudaStreamNonBlocking), "halo stream");
    cuda_check(cudaEventCreateWithFlags(&L->ev_ready, cudaEventDisableTiming), "event");
    cuda_check(cudaEventCreateWithFlags(&L->ev_halo, cudaEventDisableTiming), "event");
}

// Orders the team's stream after a pending halo leg.
void t_join(const Team& T) {
    ign_context* L = T.lead();
    if (!L->halo_pending) return;
    cuda_check(cudaStreamWaitEvent(T.stream(), L->ev_halo, 0), "halo join");
    L->halo_pending = false;
}

// prepare_stage (solver.hpp:422-425): fill_ghosts (x edges, halo, y edges)
// then refresh_primitives.  A slab overlaps its halo: once the
// x (3D: x, y) edge ghosts of its own rows exist, the halo leg — NCCL
// send/recv of the g boundary rows (planes), the remaining edge ghosts and the
// ghost-row primitives — runs on the halo stream while the team's stream
// computes the primitives of the slab's own rows and, in t_fluxes, every face
// whose stencil lies in those rows; only the halo faces, the viscous fluxes
// and the update wait for it.  Every kernel writes disjoint data in both
// orders, so the results are bitwise those of the serial schedule.
void t_prepare(const Team& T, int buf, int stage, int step) {
    t_join(T);  // the previous halo leg (a re-prepare without fluxes) is done
    for (ign_context* c : T.m)
        c->launches += timed(c, IGN_PROF_BC, [&] {
            return c->ks.bc(c->kp, c->S[buf], 0, stage, step, c->stream);
        });
    if (!t_has_halo(T) || !overlap_enabled()) {
        t_exchange(T, buf, T.stream());
        for (ign_context* c : T.m)
            c->launches += timed(c, IGN_PROF_BC, [&] {
                return c->ks.bc(c->kp, c->S[buf], 1, stage, step, c->stream);
            });
        for (ign_context* c : T.m)
            c->launches += timed(c, IGN_PROF_PRIM, [&] {
                return c->ks.prim(c->kp, c->S[buf], stage, step, c->stream, 0);
            });
        return;
    }
    ign_context* L = T.lead();
    ensure_halo_stream(L);
    cudaStream_t hs = L->halo_stream;
    NvtxRange nv("halo leg");
    cuda_check(cudaEventRecord(L->ev_ready, T.stream()), "event");
    cuda_check(cudaStreamWaitEvent(hs, L->ev_ready, 0), "halo wait");
    t_exchange(T, buf, hs);
    for (ign_context* c : T.m) c->launches += c->ks.bc(c->kp, c->S[buf], 1, stage, step, hs);
    for (ign_context* c : T.m) c->launches += c->ks.prim(c->kp, c->S[buf], stage, step, hs, 2);
    cuda_check(cudaEventRecord(L->ev_halo, hs), "event");
    L->halo_pending = true;
    for (ign_context* c : T.m)
        c->launches += timed(c, IGN_PROF_PRIM, [&] {
            return c->ks.prim(c->kp, c->S[buf], stage, step, c->stream, 1);
        });
}

void t_fluxes(const Team& T, int buf, int stage, int step) {
    const bool split = T.lead()->halo_pending;
    for (ign_context* c : T.m)
        c->launches += timed(c, IGN_PROF_FACES, [&] {
            return c->ks.faces(c->kp, c->cfg.scheme.scheme, c->cfg.scheme.split, c->S[buf], stage,
                               step, c->stream, split ? 1 : 0);
        });
    if (split) {
        t_join(T);
        for (ign_context* c : T.m)
            c->launches += timed(c, IGN_PROF_FACES, [&] {
                return c->ks.faces(c->kp, c->cfg.scheme.scheme, c->cfg.scheme.split, c->S[buf],
                                   stage, step, c->stream, 2);
            });
    }
    for (ign_context* c : T.m)
        if (c->cfg.viscous)
            c->launches += timed(c, IGN_PROF_VISC,
                                 [&] { return c->ks.visc(c->kp, stage, step, c->stream); });
}

// No error-word reduction here: each slab's kernels stop on their own word,
// and the words are MIN-reduced once per chunk (sync_and_read) — the first
// failure of any slab carries the smallest key, because a slab fed stale halo
// rows by a failed peer can only fail at a later (step, stage, phase).
void t_assemble(const Team& T, int mode, int a, int cur, int out, double dt, double w, double t,
                int stage, int step, int slot) {
    for (ign_context* c : T.m)
        c->launches += timed(c, IGN_PROF_ASSEMBLE, [&] {
            return c->ks.assemble(c->kp, mode, c->S[a], c->S[cur], c->S[out], dt, w, t, stage,
                                  step, slot, c->stream);
        });
}

// Zeroes one step's clip slots (slot = 3 step) unless a failure is pending.
__global__ void k_clip_reset(const ErrRec* err, unsigned long long* red, int slot) {
    if (failed(err)) return;
    red[2 + slot + threadIdx.x] = 0ull;
}

// One rk3_step (solver.hpp:304-332) enqueued without a host round trip;
// post_prepare appends advance()'s prepare_stage(1) (solver.hpp:345).
void t_step(const Team& T, int a, double time, double dt, int step, bool post_prepare) {
    const int b = (a + 1) % 3, c = (a + 2) % 3;
    const int slot = step * 3;  // step < kChunk: its own three clip slots
    for (ign_context* x : T.m) {
        k_clip_reset<<<1, 3, 0, x->stream>>>(x->err, x->red, slot);
        ++x->launches;
    }
    NvtxRange nv("rk3_step");
    {  // Stage 1: U <- U0 + dt L(U0)   (ghosts/cache already fresh)
        NvtxRange s("stage 1");
        t_fluxes(T, a, 1, step);
        t_assemble(T, 1, a, a, b, dt, 0.0, time, 1, step, slot + 0);
        t_prepare(T, b, 2, step);
    }
    {  // Stage 2: U <- U0 + 1/4 [(U1 - U0) + dt L(U1)]
        NvtxRange s("stage 2");
        t_fluxes(T, b, 2, step);
        t_assemble(T, 2, a, b, c, dt, 0.25, time + dt, 2, step, slot + 1);
        t_prepare(T, c, 3, step);
    }
    {  // Stage 3: U <- U0 + 2/3 [(U2 - U0) + dt L(U2)]
        NvtxRange s("stage 3");
        t_fluxes(T, c, 3, step);
        t_assemble(T, 2, a, c, b, dt, 2.0 / 3.0, time + 0.5 * dt, 3, step, slot + 2);
        if (post_prepare) t_prepare(T, b, 4, step);
    }
}

// Clip slots of a chunk's steps over all slabs (MAX: the reference's clip is a max).
void read_clips(const Team& T, int64_t chunk, std::vector<unsigned long long>& red) {
    const size_t n = size_t(2 + 3 * chunk);
    ign_context* L = T.lead();
    if (!T.local() && L->comm) {
        nccl_check(nccl().AllReduce(L->red + 2, L->red + 2, n - 2, ncclUint64, ncclMax, L->comm,
                                    L->stream),
                   "ncclAllReduce(clip)");
        cuda_check(cudaStreamSynchronize(L->stream), "clip reduce");
    }
    red.assign(n, 0ull);
    std::vector<unsigned long long> r(n);
    for (ign_context* c : T.m) {
        cuda_check(cudaMemcpy(r.data(), c->red, n * sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost),
                   "reductions");
        for (size_t k = 2; k < n; ++k) red[k] = std::max(red[k], r[k]);
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
    std::vector<unsigned long long> redv;
    read_clips(T, chunk, redv);
    const unsigned long long* red = redv.data();
    if (!f.any) {
        const int last = (int)(chunk - 1);
        const int slot = last * 3;
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
        const int slot = (int)(kk - 1) * 3;
        clip_prev = std::max(std::max(clip_of(red, slot), clip_of(red, slot + 1)),
                             clip_of(red, slot + 2));
    }
    const int ak = (int)((a0 + k) % 3);
    const int slot = (int)kk * 3;
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
        std::memset(&mem[q]->lasterr, 0, sizeof(ign_error));  // a healthy member reads no error
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
    t_join(T);
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
        // the hook returns nonzero to stop (ignis_b200.h); the reference's
        // void step_hook (solver.hpp:347) corresponds to always returning 0
        if (hook && hook(L, user) != 0) break;
    }
}

}  // namespace rt
}  // namespace ign
