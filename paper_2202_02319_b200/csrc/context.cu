// context.cu — the C-ABI (include/ignis_b200.h) over the sm_100a kernels.
//
// One ign_context = one ignis::Simulation (solver.hpp:53-853) on one GPU.
// The conservative state lives in three rotating device buffers S[0..2]; an
// RK3 step reads U0 from S[a], writes U1 to S[b], U2 to S[c] and U3 back into
// S[b], so no copy_interior (solver.hpp:310) is ever needed and U0 stays intact
// for the StepFailure restore (solver.hpp:326-329).  Errors raised on the
// device are collected in one error word and decoded here into the
// reference's exception kinds after the stream synchronises.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "host_core.hpp"
#include "ignis_b200.h"
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

struct ign_context {
    ign_config cfg;
    HMesh mesh;
    HMetrics met, metv;
    KParams kp;
    KernelSet ks;
    int nx = 0, ny = 0, g = 0, ns = 0, nc = 0;
    size_t plane = 0;
    int device = 0;
    cudaStream_t stream = nullptr;
    double* S[3] = {nullptr, nullptr, nullptr};
    int cur = 0;
    double* prim = nullptr;
    double* geom = nullptr;  // met(5), met_v(5), mesh x, y
    double *Fx = nullptr, *Gy = nullptr, *Fv = nullptr, *Gv = nullptr, *rhs = nullptr;
    double* inflow[4] = {nullptr, nullptr, nullptr, nullptr};
    ErrRec* err = nullptr;
    unsigned long long* red = nullptr;
    double time = 0.0;
    int64_t iter = 0;
    double last_clip = 0.0;
    ign_integrator integ{};
    ign_error lasterr{};
    int64_t launches = 0;
    // live per-kernel-class timing (CUDA events on this context's stream)
    bool prof_on = false;
    struct Rec { int cat; cudaEvent_t a, b; };
    std::vector<Rec> prof_pending;
    std::vector<cudaEvent_t> prof_pool;
    double prof_ms[IGN_PROF_CLASSES] = {};
    int64_t prof_n[IGN_PROF_CLASSES] = {};
};

namespace {

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw Error(IGN_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

void set_error(ign_error* out, const Error& e) {
    if (!out) return;
    out->status = e.status;
    out->stage = e.stage;
    out->i = e.i;
    out->j = e.j;
    std::snprintf(out->msg, sizeof(out->msg), "%s", e.what());
}

template <class F> int guarded(ign_context* ctx, F&& f) {
    try {
        if (ctx) cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
        f();
        if (ctx) std::memset(&ctx->lasterr, 0, sizeof(ctx->lasterr));
        return IGN_OK;
    } catch (const Error& e) {
        if (ctx) set_error(&ctx->lasterr, e);
        return e.status;
    } catch (const std::exception& e) {
        if (ctx) set_error(&ctx->lasterr, Error(IGN_INTERNAL_ERROR, e.what()));
        return IGN_INTERNAL_ERROR;
    }
}

const char* pstatus_msg(unsigned sub) {
    switch (sub) {
    case P_NONPOS_RHO: return "primitives: non-positive density";
    case P_BELOW_VACUUM: return "temperature_from_energy: energy below vacuum energy";
    default: return "temperature_from_energy: no convergence";
    }
}

// Decoded device failure.
struct DevFail {
    bool any = false;
    unsigned stage = 0, phase = 0, sub = 0;
    unsigned long long idx = 0;
    int step = 0;
};

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

DevFail sync_and_read(ign_context* ctx) {
    cuda_check(cudaStreamSynchronize(ctx->stream), "kernel execution");
    cuda_check(cudaGetLastError(), "kernel launch");
    prof_harvest(ctx);
    ErrRec h;
    cuda_check(cudaMemcpy(&h, ctx->err, sizeof(h), cudaMemcpyDeviceToHost), "error word");
    DevFail f;
    if (h.key == kNoError) return f;
    f.any = true;
    f.stage = (unsigned)(h.key >> 60);
    f.phase = (unsigned)((h.key >> 52) & 0xff);
    f.idx = (h.key >> 4) & ((1ull << 48) - 1);
    f.sub = (unsigned)(h.key & 0xf);
    f.step = h.step;
    cuda_check(cudaMemset(ctx->err, 0xff, sizeof(ErrRec)), "error reset");
    return f;
}

// Maps a device failure onto the exception the reference throws there.
Error to_error(const ign_context* ctx, const DevFail& f) {
    const int rep_stage = f.stage == 4 ? 1 : (int)f.stage;
    switch (f.phase) {
    case PH_BC: return state_error(pstatus_msg(f.sub));
    case PH_PRIM: {
        const int sx = ctx->nx + 2 * ctx->g;
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
        const int i = (int)(f.idx % ctx->nx), j = (int)(f.idx / ctx->nx);
        return step_failure("non-finite RHS", rep_stage, i, j);
    }
    default: {
        const unsigned long long cell = f.idx / 2;
        const int i = (int)(cell % ctx->nx), j = (int)(cell / ctx->nx);
        return step_failure(f.idx % 2 ? "non-finite state" : "non-positive density", rep_stage,
                            i, j);
    }
    }
}

void check(ign_context* ctx) {
    const DevFail f = sync_and_read(ctx);
    if (f.any) throw to_error(ctx, f);
}

double* dalloc(size_t n) {
    void* p = nullptr;
    cuda_check(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(double)), "cudaMalloc");
    return static_cast<double*>(p);
}

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

void upload_state(ign_context* ctx, const std::vector<double>& Ut) {
    cuda_check(cudaMemcpy(ctx->S[ctx->cur], Ut.data(), Ut.size() * sizeof(double),
                          cudaMemcpyHostToDevice),
               "state upload");
}

// ---------------------------------------------------------------- stage plumbing
// Zeroes one step's clip slots unless a failure is pending (a pending failure
// must keep the previous step's clips for last_clip, solver.hpp:847).
__global__ void k_clip_reset(const ErrRec* err, unsigned long long* red, int slot) {
    if (failed(err)) return;
    red[2 + slot + threadIdx.x] = 0ull;
}

void launch_prepare(ign_context* ctx, double* U, int stage, int step) {
    ctx->launches += timed(ctx, IGN_PROF_BC,
                           [&] { return ctx->ks.bc(ctx->kp, U, stage, step, ctx->stream); });
    ctx->launches += timed(ctx, IGN_PROF_PRIM,
                           [&] { return ctx->ks.prim(ctx->kp, U, stage, step, ctx->stream); });
}

void launch_fluxes(ign_context* ctx, const double* U, int stage, int step) {
    ctx->launches += timed(ctx, IGN_PROF_FACES, [&] {
        return ctx->ks.faces(ctx->kp, ctx->cfg.scheme.scheme, ctx->cfg.scheme.split, U, stage,
                             step, ctx->stream);
    });
    if (ctx->cfg.viscous)
        ctx->launches += timed(ctx, IGN_PROF_VISC,
                               [&] { return ctx->ks.visc(ctx->kp, stage, step, ctx->stream); });
}

int launch_assemble(ign_context* ctx, int mode, const double* U0, const double* Ucur,
                    double* Uout, double dt, double w, double t, int stage, int step, int slot) {
    return timed(ctx, IGN_PROF_ASSEMBLE, [&] {
        return ctx->ks.assemble(ctx->kp, mode, U0, Ucur, Uout, dt, w, t, stage, step, slot,
                                ctx->stream);
    });
}

// One rk3_step (solver.hpp:304-332) enqueued without a host round trip;
// post_prepare appends advance()'s prepare_stage(1) (solver.hpp:345).
void launch_step(ign_context* ctx, int a, double time, double dt, int step, bool post_prepare) {
    const int b = (a + 1) % 3, c = (a + 2) % 3;
    const int slot = (step & 1) * 3;
    k_clip_reset<<<1, 3, 0, ctx->stream>>>(ctx->err, ctx->red, slot);
    ++ctx->launches;
    double** S = ctx->S;
    // Stage 1: U <- U0 + dt L(U0)   (ghosts/cache already fresh)
    launch_fluxes(ctx, S[a], 1, step);
    ctx->launches += launch_assemble(ctx, 1, S[a], S[a], S[b], dt, 0.0, time, 1, step, slot + 0);
    launch_prepare(ctx, S[b], 2, step);
    // Stage 2: U <- U0 + 1/4 [(U1 - U0) + dt L(U1)]
    launch_fluxes(ctx, S[b], 2, step);
    ctx->launches += launch_assemble(ctx, 2, S[a], S[b], S[c], dt, 0.25, time + dt, 2, step,
                                     slot + 1);
    launch_prepare(ctx, S[c], 3, step);
    // Stage 3: U <- U0 + 2/3 [(U2 - U0) + dt L(U2)]
    launch_fluxes(ctx, S[c], 3, step);
    ctx->launches += launch_assemble(ctx, 2, S[a], S[c], S[b], dt, 2.0 / 3.0, time + 0.5 * dt,
                                     3, step, slot + 2);
    if (post_prepare) launch_prepare(ctx, S[b], 4, step);
}

double clip_of(const unsigned long long* red, int slot) {
    double d;
    std::memcpy(&d, &red[2 + slot], sizeof(d));
    return d;
}

// n consecutive steps; on a device failure reproduces the reference's state,
// time/iter and last_clip at the point it would have thrown.
void run_steps(ign_context* ctx, double dt, int64_t n, bool post_prepare) {
    if (n <= 0) return;
    const int a0 = ctx->cur;
    double t = ctx->time;
    int64_t done = 0;
    while (done < n) {
        const int64_t chunk = std::min<int64_t>(n - done, 256);
        for (int64_t k = 0; k < chunk; ++k) {
            const int64_t s = done + k;
            launch_step(ctx, (int)((a0 + s) % 3), t, dt, (int)s, post_prepare);
            t += dt;
        }
        cuda_check(cudaGetLastError(), "kernel launch");
        const DevFail f = sync_and_read(ctx);
        unsigned long long red[8];
        cuda_check(cudaMemcpy(red, ctx->red, sizeof(red), cudaMemcpyDeviceToHost), "reductions");
        if (!f.any) {
            // bookkeeping for the whole chunk
            for (int64_t k = 0; k < chunk; ++k) {
                ctx->time += dt;
                ++ctx->iter;
            }
            const int last = (int)(done + chunk - 1);
            const int slot = (last & 1) * 3;
            ctx->last_clip = std::max(std::max(clip_of(red, slot), clip_of(red, slot + 1)),
                                      clip_of(red, slot + 2));
            ctx->cur = (int)((a0 + done + chunk) % 3);
            done += chunk;
            continue;
        }
        const int64_t k = f.step;
        // completed steps before the failing one
        double clip_prev = ctx->last_clip;
        if (k > done) {
            const int slot = ((int)(k - 1) & 1) * 3;
            clip_prev = std::max(std::max(clip_of(red, slot), clip_of(red, slot + 1)),
                                 clip_of(red, slot + 2));
        }
        for (int64_t q = done; q < k; ++q) {
            ctx->time += dt;
            ++ctx->iter;
        }
        const int ak = (int)((a0 + k) % 3);
        const int slot = ((int)k & 1) * 3;
        const Error e = to_error(ctx, f);
        if (f.stage == 4) {  // advance's prepare_stage(1) after a completed step
            ctx->time += dt;
            ++ctx->iter;
            ctx->cur = (ak + 1) % 3;
            ctx->last_clip = std::max(std::max(clip_of(red, slot), clip_of(red, slot + 1)),
                                      clip_of(red, slot + 2));
            throw e;
        }
        // inside rk3_step: last_clip covers the stages that completed post_stage
        double lc = clip_prev;
        for (unsigned s = 1; s < f.stage; ++s)
            lc = s == 1 ? clip_of(red, slot) : std::max(lc, clip_of(red, slot + s - 1));
        ctx->last_clip = lc;
        if (e.status == IGN_STEP_FAILURE) ctx->cur = ak;  // restore U0
        else ctx->cur = f.stage <= 1 ? ak : f.stage == 2 ? (ak + 1) % 3 : (ak + 2) % 3;
        throw e;
    }
}

double stable_dt_impl(ign_context* ctx) {
    unsigned long long init[2] = {0ull, 0x7ff0000000000000ull};
    cuda_check(cudaMemcpyAsync(ctx->red, init, sizeof(init), cudaMemcpyHostToDevice, ctx->stream),
               "dt reset");
    ctx->launches += timed(ctx, IGN_PROF_DT, [&] { return ctx->ks.dt(ctx->kp, ctx->stream); });
    check(ctx);
    unsigned long long red[2];
    cuda_check(cudaMemcpy(red, ctx->red, sizeof(red), cudaMemcpyDeviceToHost), "dt readback");
    double lam_max, dt_chem;
    std::memcpy(&lam_max, &red[0], sizeof(double));
    std::memcpy(&dt_chem, &red[1], sizeof(double));
    double dt = ctx->cfg.scheme.cfl / lam_max;
    dt = smin(dt, dt_chem);
    const ign_laser& L = ctx->cfg.laser;
    if (L.present && L.energy != 0.0 && ctx->time - L.t0 < 6.0 * L.sigma_t &&
        ctx->time + dt > L.t0 - 6.0 * L.sigma_t)
        dt = smin(dt, L.sigma_t / 5.0);
    return dt;
}

void prepare_impl(ign_context* ctx, int stage) {
    launch_prepare(ctx, ctx->S[ctx->cur], stage, 0);
    check(ctx);
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
    cudaFree(ctx->rhs);
    for (double* p : ctx->inflow) cudaFree(p);
    cudaFree(ctx->err);
    cudaFree(ctx->red);
    for (auto& r : ctx->prof_pending) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (cudaEvent_t e : ctx->prof_pool) cudaEventDestroy(e);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

void create_impl(const ign_config* cfg, ign_context* ctx) {
    if (!cfg || cfg->abi_version != IGN_ABI_VERSION)
        throw usage_error("ign_create: ABI version mismatch");
    ctx->cfg = *cfg;
    ctx->device = cfg->device;
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    // Simulation::init (solver.hpp:82-101)
    ctx->mesh = build_mesh(*cfg);
    validate_config(*cfg, ctx->mesh);
    ctx->met = compute_metrics(ctx->mesh, inviscid_metric_mode(*cfg), cfg->skew_beta);
    ctx->metv = compute_metrics(ctx->mesh, MM_CENTRAL2, 0.0);
    ctx->integ = cfg->integ;
    const int nx = cfg->nx, ny = cfg->ny, g = cfg->g, ns = cfg->mix.ns, nc = ns + 3;
    ctx->nx = nx;
    ctx->ny = ny;
    ctx->g = g;
    ctx->ns = ns;
    ctx->nc = nc;
    const size_t P = static_cast<size_t>(nx + 2 * g) * (ny + 2 * g);
    ctx->plane = P;
    cuda_check(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking), "stream");
    for (auto& s : ctx->S) {
        s = dalloc(nc * P);
        cuda_check(cudaMemset(s, 0, nc * P * sizeof(double)), "memset");
    }
    // primitive cache: rho,u,v,p = 0, T = c = 1 (solver.hpp:94-100), Y, X
    const size_t nprim = 6 + 2 * static_cast<size_t>(ns);
    ctx->prim = dalloc(nprim * P);
    {
        std::vector<double> init(nprim * P, 0.0);
        std::fill(init.begin() + 4 * P, init.begin() + 6 * P, 1.0);
        cuda_check(cudaMemcpy(ctx->prim, init.data(), init.size() * sizeof(double),
                              cudaMemcpyHostToDevice),
                   "cache init");
    }
    ctx->geom = dalloc(12 * P);
    {
        const HField* f[12] = {&ctx->met.jac,  &ctx->met.m_xi_x,  &ctx->met.m_xi_y,
                               &ctx->met.m_eta_x, &ctx->met.m_eta_y, &ctx->metv.jac,
                               &ctx->metv.m_xi_x, &ctx->metv.m_xi_y, &ctx->metv.m_eta_x,
                               &ctx->metv.m_eta_y, &ctx->mesh.x,   &ctx->mesh.y};
        for (int k = 0; k < 12; ++k)
            cuda_check(cudaMemcpy(ctx->geom + k * P, f[k]->d.data(), P * sizeof(double),
                                  cudaMemcpyHostToDevice),
                       "geometry upload");
    }
    ctx->Fx = dalloc(static_cast<size_t>(nc) * (nx + 1) * ny);
    ctx->Gy = dalloc(static_cast<size_t>(nc) * nx * (ny + 1));
    if (cfg->viscous) {
        ctx->Fv = dalloc(nc * P);
        ctx->Gv = dalloc(nc * P);
    }
    // inflow profile tables (boundary.hpp:227-241 ghost targets)
    const ign_edge* edges[4] = {&cfg->bc.left, &cfg->bc.right, &cfg->bc.bottom, &cfg->bc.top};
    for (int e = 0; e < 4; ++e) {
        if (edges[e]->type != 3) continue;
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
    void* p = nullptr;
    cuda_check(cudaMalloc(&p, sizeof(ErrRec)), "cudaMalloc");
    ctx->err = static_cast<ErrRec*>(p);
    cuda_check(cudaMemset(ctx->err, 0xff, sizeof(ErrRec)), "memset");
    cuda_check(cudaMalloc(&p, 8 * sizeof(unsigned long long)), "cudaMalloc");
    ctx->red = static_cast<unsigned long long*>(p);
    cuda_check(cudaMemset(ctx->red, 0, 8 * sizeof(unsigned long long)), "memset");

    KParams& k = ctx->kp;
    std::memset(&k, 0, sizeof(k));
    k.nx = nx;
    k.ny = ny;
    k.g = g;
    k.sx = nx + 2 * g;
    k.plane = static_cast<long long>(P);
    k.ns = ns;
    k.viscous = cfg->viscous;
    for (int e = 0; e < 4; ++e) {
        k.bc_type[e] = edges[e]->type;
        k.T_wall[e] = edges[e]->T_wall;
        k.inflow[e] = ctx->inflow[e];
    }
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
    k.mxx = ctx->geom + P;
    k.mxy = ctx->geom + 2 * P;
    k.mex = ctx->geom + 3 * P;
    k.mey = ctx->geom + 4 * P;
    k.vjac = ctx->geom + 5 * P;
    k.vmxx = ctx->geom + 6 * P;
    k.vmxy = ctx->geom + 7 * P;
    k.vmex = ctx->geom + 8 * P;
    k.vmey = ctx->geom + 9 * P;
    k.xc = ctx->geom + 10 * P;
    k.yc = ctx->geom + 11 * P;
    k.Fx = ctx->Fx;
    k.Gy = ctx->Gy;
    k.Fv = ctx->Fv;
    k.Gv = ctx->Gv;
    k.err = ctx->err;
    k.red = ctx->red;
    k.mix = build_mix(cfg->mix);
    k.mech = build_mech(cfg->mech);
    k.laser = build_laser(cfg->laser);
    ctx->ks = kernel_set(ns);
}

void copy_hfield(const HField& f, double* out) { std::memcpy(out, f.d.data(), f.d.size() * 8); }

void metrics_out(const HMetrics& m, double* out, size_t P) {
    const HField* f[5] = {&m.jac, &m.m_xi_x, &m.m_xi_y, &m.m_eta_x, &m.m_eta_y};
    for (int k = 0; k < 5; ++k) copy_hfield(*f[k], out + k * P);
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

uint64_t ign_config_size(void) { return sizeof(ign_config); }

int ign_create(const ign_config* cfg, ign_context** out) {
    if (!out) return IGN_USAGE_ERROR;
    *out = nullptr;
    ign_context* ctx = new ign_context();
    const int st = guarded(nullptr, [&] { create_impl(cfg, ctx); });
    if (st != IGN_OK) {
        destroy_impl(ctx);
        return st;
    }
    *out = ctx;
    return IGN_OK;
}

void ign_destroy(ign_context* ctx) {
    if (ctx) cudaSetDevice(ctx->device);
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

int ign_get_metrics(const ign_context* ctx, int which, double* out) {
    metrics_out(which == 0 ? ctx->met : ctx->metv, out, ctx->plane);
    return IGN_OK;
}

int ign_set_initial_condition(ign_context* ctx, ign_ic_fn fn, void* user) {
    return guarded(ctx, [&] {
        const int g = ctx->g, ns = ctx->ns, nc = ctx->nc;
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
        (void)ns;
        upload_state(ctx, Ut);
    });
}

int ign_set_initial_primitives(ign_context* ctx, const double* prim) {
    return guarded(ctx, [&] {
        const int ns = ctx->ns, nc = ctx->nc;
        const size_t P = ctx->plane;
        std::vector<double> Ut(nc * P);
        for (size_t k = 0; k < P; ++k) {
            double Y[kMaxSpecies];
            for (int s = 0; s < ns; ++s) Y[s] = prim[(4 + s) * P + k];
            double U[kMaxComp];
            cons_from_prim(ctx->kp.mix, prim[k], prim[P + k], prim[2 * P + k], prim[3 * P + k], Y,
                           U);
            const double invJ = 1.0 / ctx->met.jac.d[k];
            for (int c = 0; c < nc; ++c) Ut[c * P + k] = U[c] * invJ;
        }
        upload_state(ctx, Ut);
    });
}

int ign_set_state(ign_context* ctx, const double* Ut, const double* Tc) {
    return guarded(ctx, [&] {
        cuda_check(cudaMemcpy(ctx->S[ctx->cur], Ut, ctx->nc * ctx->plane * sizeof(double),
                              cudaMemcpyHostToDevice),
                   "set_state");
        if (Tc)
            cuda_check(cudaMemcpy(ctx->prim + 4 * ctx->plane, Tc, ctx->plane * sizeof(double),
                                  cudaMemcpyHostToDevice),
                       "set_state T");
    });
}

int ign_get_state(ign_context* ctx, double* Ut) {
    return guarded(ctx, [&] {
        cuda_check(cudaMemcpy(Ut, ctx->S[ctx->cur], ctx->nc * ctx->plane * sizeof(double),
                              cudaMemcpyDeviceToHost),
                   "get_state");
    });
}

int ign_get_cache(ign_context* ctx, double* prim) {
    return guarded(ctx, [&] {
        cuda_check(cudaMemcpy(prim, ctx->prim, (6 + ctx->ns) * ctx->plane * sizeof(double),
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
        ctx->launches += ctx->ks.bc(ctx->kp, ctx->S[ctx->cur], 0, 0, ctx->stream);
        check(ctx);
    });
}

int ign_refresh_primitives(ign_context* ctx, int stage) {
    return guarded(ctx, [&] {
        ctx->launches += ctx->ks.prim(ctx->kp, ctx->S[ctx->cur], stage, 0, ctx->stream);
        check(ctx);
    });
}

int ign_prepare_stage(ign_context* ctx, int stage) {
    return guarded(ctx, [&] { prepare_impl(ctx, stage); });
}

int ign_compute_rhs(ign_context* ctx, double t_stage, int stage, double* rhs) {
    return guarded(ctx, [&] {
        const size_t n = ctx->nc * ctx->plane;
        if (!ctx->rhs) ctx->rhs = dalloc(n);
        cuda_check(cudaMemsetAsync(ctx->rhs, 0, n * sizeof(double), ctx->stream), "memset");
        const double* U = ctx->S[ctx->cur];
        launch_fluxes(ctx, U, stage, 0);
        ctx->launches += launch_assemble(ctx, 0, U, U, ctx->rhs, 0.0, 0.0, t_stage, stage, 0, 0);
        check(ctx);
        if (rhs)
            cuda_check(cudaMemcpy(rhs, ctx->rhs, n * sizeof(double), cudaMemcpyDeviceToHost),
                       "rhs readback");
    });
}

int ign_stable_dt(ign_context* ctx, double* dt) {
    return guarded(ctx, [&] { *dt = stable_dt_impl(ctx); });
}

int ign_rk3_step(ign_context* ctx, double dt) {
    return guarded(ctx, [&] { run_steps(ctx, dt, 1, false); });
}

int ign_rk3_steps(ign_context* ctx, double dt, int64_t n) {
    return guarded(ctx, [&] { run_steps(ctx, dt, n, true); });
}

// Simulation::advance (solver.hpp:336-349).  With a pinned step and no hook the
// step count is known up front, so the steps are enqueued back to back.
int ign_advance(ign_context* ctx, ign_step_hook hook, void* user) {
    return guarded(ctx, [&] {
        prepare_impl(ctx, 1);
        const ign_integrator& in = ctx->integ;
        const double t_eps = 1e-12 * std::max(1.0, std::abs(in.t_end));
        if (in.fixed_dt > 0.0 && !hook) {
            int64_t n = 0;
            double t = ctx->time;
            int64_t it = ctx->iter;
            while (it < in.max_iter && t < in.t_end - t_eps) {
                t += in.fixed_dt;
                ++it;
                ++n;
            }
            run_steps(ctx, in.fixed_dt, n, true);
            return;
        }
        while (ctx->iter < in.max_iter && ctx->time < in.t_end - t_eps) {
            double dt = in.fixed_dt > 0.0 ? in.fixed_dt : stable_dt_impl(ctx);
            if (in.fixed_dt <= 0.0) dt = smin(dt, in.t_end - ctx->time);
            run_steps(ctx, dt, 1, false);
            prepare_impl(ctx, 1);
            if (hook) hook(ctx, user);
        }
    });
}

// conserved_totals (solver.hpp:411-418): serial host sum in the reference order
int ign_conserved_totals(ign_context* ctx, double* tot) {
    return guarded(ctx, [&] {
        const size_t P = ctx->plane;
        std::vector<double> Ut(ctx->nc * P);
        cuda_check(cudaMemcpy(Ut.data(), ctx->S[ctx->cur], Ut.size() * 8, cudaMemcpyDeviceToHost),
                   "totals");
        const int sx = ctx->nx + 2 * ctx->g, g = ctx->g;
        for (int c = 0; c < ctx->nc; ++c) {
            double s = 0.0;
            for (int j = 0; j < ctx->ny; ++j)
                for (int i = 0; i < ctx->nx; ++i) s += Ut[c * P + (size_t)(j + g) * sx + (i + g)];
            tot[c] = s;
        }
    });
}

// product_mole_fraction (solver.hpp:387-407), serial host sum
int ign_product_mole_fraction(ign_context* ctx, double* out) {
    return guarded(ctx, [&] {
        int ico2 = -1, ih2o = -1;
        for (int s = 0; s < ctx->ns; ++s) {
            const char* nm = ctx->cfg.mix.species[s].name;
            if (std::strncmp(nm, "CO2", IGN_NAME_LEN) == 0) ico2 = s;
            if (std::strncmp(nm, "H2O", IGN_NAME_LEN) == 0) ih2o = s;
        }
        if (ico2 < 0 && ih2o < 0) {
            *out = 0.0;
            return;
        }
        const size_t P = ctx->plane;
        std::vector<double> Y(ctx->ns * P);
        cuda_check(cudaMemcpy(Y.data(), ctx->prim + 6 * P, Y.size() * 8, cudaMemcpyDeviceToHost),
                   "Y readback");
        const DMix& m = ctx->kp.mix;
        const int sx = ctx->nx + 2 * ctx->g, g = ctx->g;
        double num = 0.0, den = 0.0;
        for (int j = 0; j < ctx->ny; ++j)
            for (int i = 0; i < ctx->nx; ++i) {
                const size_t id = (size_t)(j + g) * sx + (i + g);
                double y[kMaxSpecies], x[kMaxSpecies];
                for (int s = 0; s < ctx->ns; ++s) y[s] = Y[s * P + id];
                double inv = 0.0;
                for (int s = 0; s < ctx->ns; ++s) inv += divW(m.sp[s], y[s]);
                const double wbar = 1.0 / inv;
                for (int s = 0; s < ctx->ns; ++s) x[s] = divW(m.sp[s], y[s] * wbar);
                const double w = 1.0 / ctx->met.jac(i, j);
                num += w * ((ico2 >= 0 ? x[ico2] : 0.0) + (ih2o >= 0 ? x[ih2o] : 0.0));
                den += w;
            }
        *out = num / den;
    });
}

int ign_last_clip(const ign_context* ctx, double* clip) {
    *clip = ctx->last_clip;
    return IGN_OK;
}

int ign_host_metrics(const ign_config* cfg, int which, double* out, ign_error* err) {
    try {
        const HMesh m = build_mesh(*cfg);
        const HMetrics mf = which == 0 ? compute_metrics(m, inviscid_metric_mode(*cfg), cfg->skew_beta)
                                       : compute_metrics(m, MM_CENTRAL2, 0.0);
        metrics_out(mf, out, mf.jac.d.size());
        return IGN_OK;
    } catch (const Error& e) {
        set_error(err, e);
        return e.status;
    }
}

int ign_host_mesh(const ign_config* cfg, double* x, double* y, ign_error* err) {
    try {
        const HMesh m = build_mesh(*cfg);
        copy_hfield(m.x, x);
        copy_hfield(m.y, y);
        return IGN_OK;
    } catch (const Error& e) {
        set_error(err, e);
        return e.status;
    }
}

int64_t ign_kernel_launches(const ign_context* ctx) { return ctx ? ctx->launches : 0; }

int ign_profile_enable(ign_context* ctx, int on) {
    return guarded(ctx, [&] {
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
    return guarded(ctx, [&] {
        cuda_check(cudaStreamSynchronize(ctx->stream), "sync");
        prof_harvest(ctx);
        for (int k = 0; k < IGN_PROF_CLASSES; ++k) {
            ms[k] = ctx->prof_ms[k];
            counts[k] = ctx->prof_n[k];
        }
    });
}

void* ign_stream_handle(const ign_context* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

}  // extern "C"
