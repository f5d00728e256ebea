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
#include "context_internal.hpp"

using namespace ign::rt;

// ====================================================================== C ABI
extern "C" {

uint64_t ign_config_size(void) { return sizeof(ign_config); }

int ign_guard_status(int* enabled, unsigned long long* checked, unsigned long long* corrupted) {
    return guarded_err(nullptr, -1, [&] { guard_status(enabled, checked, corrupted); });
}

int ign_guard_selftest(int device, unsigned long long* detected) {
    if (!detected) return IGN_USAGE_ERROR;
    return guarded_err(nullptr, device, [&] { *detected = guard_selftest(); });
}

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
    if (!ctx) return IGN_USAGE_ERROR;
    if (nx) *nx = ctx->nx;
    if (ny) *ny = ctx->ny;
    if (g) *g = ctx->g;
    if (ns) *ns = ctx->ns;
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
        h2d(ctx, ctx->S[ctx->cur], Ut, ctx->nc * ctx->plane * sizeof(double), "set_state");
        if (Tc)
            h2d(ctx, ctx->prim + (ctx->nz > 0 ? 5 : 4) * ctx->plane, Tc,
                ctx->plane * sizeof(double), "set_state T");
    });
}

int ign_get_state(ign_context* ctx, double* Ut) {
    return guarded_err(&ctx->lasterr, ctx->device, [&] {
        d2h(ctx, Ut, ctx->S[ctx->cur], ctx->nc * ctx->plane * sizeof(double), "get_state");
    });
}

int ign_get_cache(ign_context* ctx, double* prim) {
    return guarded_err(&ctx->lasterr, ctx->device, [&] {
        d2h(ctx, prim, ctx->prim, ((ctx->nz > 0 ? 7 : 6) + ctx->ns) * ctx->plane * sizeof(double),
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
        t_exchange(T, ctx->cur, ctx->stream);
        ctx->launches += ctx->ks.bc(ctx->kp, ctx->S[ctx->cur], 1, 0, 0, ctx->stream);
        t_errsync(T);
        check(T);
    });
}

int ign_refresh_primitives(ign_context* ctx, int stage) {
    return guarded(ctx, [&] {
        ctx->launches += ctx->ks.prim(ctx->kp, ctx->S[ctx->cur], stage, 0, ctx->stream, 0);
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
            d2h(ctx, rhs, ctx->rhs, n * sizeof(double), "rhs readback");
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
    // a usage error is every member's outcome: no member steps
    auto fail_all = [&](int st, const Error& e) {
        for (int q = 0; q < n; ++q) {
            status[q] = st;
            if (members[q]) set_error(&members[q]->lasterr, e);
        }
        return st;
    };
    for (int q = 0; q < n; ++q)
        if (!members[q] || members[q]->nranks > 1 || members[q]->group ||
            members[q]->device != members[0]->device)
            return fail_all(IGN_USAGE_ERROR,
                            usage_error("ensemble: members must be whole-domain contexts on one "
                                        "device"));
    try {
        cuda_check(cudaSetDevice(members[0]->device), "cudaSetDevice");
        t_run_ensemble(std::vector<ign_context*>(members, members + n), dt, nsteps, status);
    } catch (const Error& e) {
        return fail_all(e.status, e);
    } catch (const std::exception& e) {
        return fail_all(IGN_INTERNAL_ERROR, Error(IGN_INTERNAL_ERROR, e.what()));
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

int ign_add_probe3(ign_context* ctx, int32_t i0, int32_t j0, int32_t k0, int32_t i1, int32_t j1,
                   int32_t k1) {
    return guarded_err(&ctx->lasterr, ctx->device, [&] {
        if (ctx->nz == 0) throw usage_error("probes: ign_add_probe3 is for 3D contexts");
        if (i0 < 0 || j0 < 0 || k0 < 0 || i1 >= ctx->nx || j1 >= ctx->ny || k1 >= ctx->nz_glob ||
            i0 > i1 || j0 > j1 || k0 > k1)
            throw config_error("probe box out of range");
        ign_context::Probe p{i0, j0, i1, j1, {}, {}};
        p.k0 = k0;
        p.k1 = k1;
        ctx->probes.push_back(p);
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

int ign_set_diagnostics(ign_context* ctx, int mode) {
    if (!ctx || (mode != IGN_DIAG_DEVICE && mode != IGN_DIAG_REFERENCE)) return IGN_USAGE_ERROR;
    ctx->diag_mode = mode;
    return IGN_OK;
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
            // each slab keeps its OWN error word, exactly as NCCL ranks do: a
            // slab runs on past a peer's failure and the words are MIN-folded
            // once per chunk (sync_and_read), so the group validates the
            // multi-rank failure semantics on one GPU
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
