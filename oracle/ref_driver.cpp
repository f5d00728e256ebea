// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the
// product).  Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may
// load the library this file builds.
//
// A C-ABI shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/ignis/*.hpp, compiled in place by
// oracle/build_ref.sh into oracle/_ref/libignis_ref.so).  It exports the same
// entry points as include/ignis_b200.h with the prefix `ignref_`, each one a
// direct call of the reference member it names, so parity tests can drive the
// reference and the B200 path with one config and compare outputs.
// No reference source is copied here: the headers are #included from where
// they lie.
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "ignis/snapshot.hpp"
#include "ignis/solver.hpp"
#include "ignis_b200.h"

#include "ref3d_faces.hpp"
#include "ref3d_viscous.hpp"
#include "ref3d_step.hpp"

using namespace ignis;

struct ref_ctx {
    Simulation sim;
    ign_error err{};
    int ns = 0;
    std::size_t plane = 0;
};

namespace {

void set_err(ign_error* e, int status, const char* msg, int stage = 0,
             int i = 0, int j = 0) {
    if (!e) return;
    e->status = status;
    e->stage = stage;
    e->i = i;
    e->j = j;
    e->k = 0;
    std::snprintf(e->msg, sizeof(e->msg), "%s", msg);
}

// Maps the reference's exception hierarchy (errors.hpp:10-47) onto statuses.
template <class F> int guarded(ign_error* e, F&& f) {
    try {
        f();
        if (e) set_err(e, IGN_OK, "");
        return IGN_OK;
    } catch (const StepFailure& x) {
        set_err(e, IGN_STEP_FAILURE, x.what(), x.stage, x.i, x.j);
        return IGN_STEP_FAILURE;
    } catch (const NumericsError& x) {
        set_err(e, IGN_NUMERICS_ERROR, x.what());
        return IGN_NUMERICS_ERROR;
    } catch (const ConfigError& x) {
        set_err(e, IGN_CONFIG_ERROR, x.what());
        return IGN_CONFIG_ERROR;
    } catch (const StateError& x) {
        set_err(e, IGN_STATE_ERROR, x.what());
        return IGN_STATE_ERROR;
    } catch (const FormatError& x) {
        set_err(e, IGN_FORMAT_ERROR, x.what());
        return IGN_FORMAT_ERROR;
    } catch (const UsageError& x) {
        set_err(e, IGN_USAGE_ERROR, x.what());
        return IGN_USAGE_ERROR;
    } catch (const std::exception& x) {
        set_err(e, IGN_INTERNAL_ERROR, x.what());
        return IGN_INTERNAL_ERROR;
    }
}

MixtureModel to_mix(const ign_mixture& m) {
    MixtureModel mix;
    mix.mode = m.mode == 0 ? MixtureModel::Mode::CaloricallyPerfect
                           : MixtureModel::Mode::MultiSpecies;
    mix.R = m.R;
    mix.Le = m.Le;
    mix.Pr = m.Pr;
    for (int s = 0; s < m.ns; ++s) {
        const ign_species& a = m.species[s];
        SpeciesData sp;
        sp.name = std::string(a.name, strnlen(a.name, IGN_NAME_LEN));
        sp.W = a.W;
        sp.mu_ref = a.mu_ref;
        sp.t_ref = a.t_ref;
        sp.n_exp = a.n_exp;
        for (int k = 0; k < a.npieces; ++k) {
            const ign_thermo_piece& q = a.pieces[k];
            ThermoPiece p;
            p.t_lo = q.t_lo;
            p.t_hi = q.t_hi;
            p.cm2 = q.cm2;
            p.cm1 = q.cm1;
            p.c0 = q.c0;
            p.c1 = q.c1;
            p.c2 = q.c2;
            p.c3 = q.c3;
            p.c4 = q.c4;
            p.b = q.b;
            sp.pieces.push_back(p);
        }
        mix.species.push_back(sp);
    }
    return mix;
}

EdgeSpec to_edge(const ign_edge& e) {
    EdgeSpec s;
    s.type = static_cast<BCType>(e.type);
    s.T_wall = e.T_wall;
    for (int k = 0; k < e.nseg; ++k) {
        InflowSegment g;
        g.lo = e.seg[k].lo;
        g.hi = e.seg[k].hi;
        g.u = e.seg[k].u;
        g.v = e.seg[k].v;
        g.T = e.seg[k].T;
        for (int q = 0; q < IGN_MAX_SPECIES; ++q) g.Y[q] = e.seg[k].Y[q];
        s.segments.push_back(g);
    }
    s.smooth_width = e.smooth_width;
    s.p_target = e.p_target;
    s.sigma_out = e.sigma_out;
    return s;
}

Mesh make_mesh(const ign_config& c) {
    Mesh m = build_uniform(c.nx, c.ny, c.lx, c.ly, {c.center_x, c.center_y},
                           c.periodic_x != 0, c.periodic_y != 0, c.g);
    if (c.mesh_x && c.mesh_y) {  // a hand-built Mesh: the caller's coordinates
        std::memcpy(m.x.raw().data(), c.mesh_x, m.x.raw().size() * sizeof(double));
        std::memcpy(m.y.raw().data(), c.mesh_y, m.y.raw().size() * sizeof(double));
        return m;
    }
    if (c.apply_skew) m = apply_skew(m, c.skew_beta);
    return m;
}

SchemeConfig to_scheme(const ign_scheme& s) {
    SchemeConfig sc;
    sc.scheme = static_cast<InviscidScheme>(s.scheme);
    sc.split = static_cast<FluxSplit>(s.split);
    sc.teno_ct = s.teno_ct;
    sc.eps = s.eps;
    sc.cfl = s.cfl;
    sc.metrics = static_cast<InviscidMetrics>(s.metrics);
    return sc;
}

MetricMode inviscid_mode(const ign_config& c, const SchemeConfig& sc) {
    if (c.metric_mode < 0) return Simulation::metric_mode_for(sc);
    return static_cast<MetricMode>(c.metric_mode);
}

void copy_out(const FieldSet& fs, int n, double* out, std::size_t plane) {
    for (int c = 0; c < n; ++c)
        std::memcpy(out + c * plane, fs[c].raw().data(), plane * sizeof(double));
}

void copy_field(const Field& f, double* out, std::size_t plane) {
    std::memcpy(out, f.raw().data(), plane * sizeof(double));
}

} // namespace

void init_sim(Simulation& sim, const ign_config* cfg) {
    const SchemeConfig sc = to_scheme(cfg->scheme);
    BoundarySpec bs;
    bs.left = to_edge(cfg->bc.left);
    bs.right = to_edge(cfg->bc.right);
    bs.bottom = to_edge(cfg->bc.bottom);
    bs.top = to_edge(cfg->bc.top);
    sim.init(make_mesh(*cfg), inviscid_mode(*cfg, sc), cfg->skew_beta,
             to_mix(cfg->mix), sc, bs);
    sim.viscous = cfg->viscous != 0;
    if (cfg->mech.present) {
        ReactionMechanism m;
        m.A = cfg->mech.A;
        m.Ta = cfg->mech.Ta;
        m.a = cfg->mech.a;
        m.b = cfg->mech.b;
        m.T_cutoff = cfg->mech.T_cutoff;
        m.i_fuel = cfg->mech.i_fuel;
        m.i_ox = cfg->mech.i_ox;
        m.i_co2 = cfg->mech.i_co2;
        m.i_h2o = cfg->mech.i_h2o;
        for (int s = 0; s < IGN_MAX_SPECIES; ++s) m.nu[s] = cfg->mech.nu[s];
        sim.mech = m;
    }
    if (cfg->laser.present) {
        LaserParams p;
        p.energy = cfg->laser.energy;
        p.sigma_r = cfg->laser.sigma_r;
        p.sigma_t = cfg->laser.sigma_t;
        p.x0 = cfg->laser.x0;
        p.y0 = cfg->laser.y0;
        p.t0 = cfg->laser.t0;
        p.kernel = static_cast<LaserKernel>(cfg->laser.kernel);
        p.edot_rate = cfg->laser.edot_rate;
        p.profile.lobe_sep = cfg->laser.lobe_sep;
        p.profile.width_up = cfg->laser.width_up;
        p.profile.width_down = cfg->laser.width_down;
        p.profile.amp_down = cfg->laser.amp_down;
        p.profile.width_radial = cfg->laser.width_radial;
        sim.laser = p;
    }
    sim.integ.fixed_dt = cfg->integ.fixed_dt;
    sim.integ.t_end = cfg->integ.t_end;
    sim.integ.max_iter = cfg->integ.max_iter;
    sim.integ.chem_dt_limit = cfg->integ.chem_dt_limit != 0;
    sim.integ.chem_dt_factor = cfg->integ.chem_dt_factor;
    sim.partitions = cfg->partitions > 0 ? cfg->partitions : 1;
}

extern "C" {

uint64_t ignref_config_size(void) { return sizeof(ign_config); }

int ignref_create(const ign_config* cfg, ref_ctx** out) {
    ign_error e{};
    *out = nullptr;
    if (!cfg || cfg->abi_version != IGN_ABI_VERSION) return IGN_USAGE_ERROR;
    auto ctx = std::make_unique<ref_ctx>();
    const int st = guarded(&e, [&] {
        Simulation& sim = ctx->sim;
        init_sim(sim, cfg);
        ctx->ns = sim.ns();
        ctx->plane = sim.Ut[0].raw().size();
    });
    if (st != IGN_OK) return st;
    *out = ctx.release();
    return IGN_OK;
}

void ignref_destroy(ref_ctx* ctx) { delete ctx; }

int ignref_last_error(const ref_ctx* ctx, ign_error* err) {
    *err = ctx->err;
    return IGN_OK;
}

int ignref_dims(const ref_ctx* ctx, int32_t* nx, int32_t* ny, int32_t* g,
                int32_t* ns) {
    *nx = ctx->sim.mesh.nx;
    *ny = ctx->sim.mesh.ny;
    *g = ctx->sim.mesh.g;
    *ns = ctx->ns;
    return IGN_OK;
}

int ignref_get_mesh(const ref_ctx* ctx, double* x, double* y) {
    copy_field(ctx->sim.mesh.x, x, ctx->plane);
    copy_field(ctx->sim.mesh.y, y, ctx->plane);
    return IGN_OK;
}

int ignref_get_metrics(const ref_ctx* ctx, int which, double* out) {
    const MetricField& m = which == 0 ? ctx->sim.met : ctx->sim.met_v;
    const Field* f[5] = {&m.jac, &m.m_xi_x, &m.m_xi_y, &m.m_eta_x, &m.m_eta_y};
    for (int k = 0; k < 5; ++k) copy_field(*f[k], out + k * ctx->plane, ctx->plane);
    return IGN_OK;
}

int ignref_set_initial_condition(ref_ctx* ctx, ign_ic_fn fn, void* user) {
    return guarded(&ctx->err, [&] {
        ctx->sim.set_initial_condition([&](double x, double y) {
            ign_prim_point q{};
            fn(x, y, user, &q);
            PrimPoint pt;
            pt.rho = q.rho;
            pt.u = q.u;
            pt.v = q.v;
            pt.p = q.p;
            pt.T = q.T;
            for (int s = 0; s < IGN_MAX_SPECIES; ++s) pt.Y[s] = q.Y[s];
            return pt;
        });
    });
}

// Calls the reference's own set_initial_condition; its loop visits the padded
// nodes in storage order (solver.hpp:118-119), so a running index addresses
// the caller's arrays.
int ignref_set_initial_primitives(ref_ctx* ctx, const double* prim) {
    const std::size_t P = ctx->plane;
    std::size_t k = 0;
    return guarded(&ctx->err, [&] {
        ctx->sim.set_initial_condition([&](double, double) {
            PrimPoint pt;
            pt.rho = prim[0 * P + k];
            pt.u = prim[1 * P + k];
            pt.v = prim[2 * P + k];
            pt.T = prim[3 * P + k];
            for (int s = 0; s < ctx->ns; ++s) pt.Y[s] = prim[(4 + s) * P + k];
            ++k;
            return pt;
        });
    });
}

int ignref_set_state(ref_ctx* ctx, const double* Ut, const double* Tc) {
    const std::size_t P = ctx->plane;
    for (int c = 0; c < ctx->ns + 3; ++c)
        std::memcpy(ctx->sim.Ut[c].raw().data(), Ut + c * P, P * sizeof(double));
    if (Tc) std::memcpy(ctx->sim.T.raw().data(), Tc, P * sizeof(double));
    return IGN_OK;
}

int ignref_get_state(ref_ctx* ctx, double* Ut) {
    copy_out(ctx->sim.Ut, ctx->ns + 3, Ut, ctx->plane);
    return IGN_OK;
}

int ignref_get_cache(ref_ctx* ctx, double* prim) {
    const std::size_t P = ctx->plane;
    const Simulation& s = ctx->sim;
    const Field* f[6] = {&s.rho, &s.u, &s.v, &s.p, &s.T, &s.c};
    for (int k = 0; k < 6; ++k) copy_field(*f[k], prim + k * P, P);
    for (int q = 0; q < ctx->ns; ++q) copy_field(s.Ys[q], prim + (6 + q) * P, P);
    return IGN_OK;
}

int ignref_get_time(const ref_ctx* ctx, double* t, int64_t* it) {
    *t = ctx->sim.time;
    *it = ctx->sim.iter;
    return IGN_OK;
}

int ignref_set_time(ref_ctx* ctx, double t, int64_t it) {
    ctx->sim.time = t;
    ctx->sim.iter = it;
    return IGN_OK;
}

int ignref_set_integrator(ref_ctx* ctx, const ign_integrator* in) {
    ctx->sim.integ.fixed_dt = in->fixed_dt;
    ctx->sim.integ.t_end = in->t_end;
    ctx->sim.integ.max_iter = in->max_iter;
    ctx->sim.integ.chem_dt_limit = in->chem_dt_limit != 0;
    ctx->sim.integ.chem_dt_factor = in->chem_dt_factor;
    return IGN_OK;
}

int ignref_set_partitions(ref_ctx* ctx, int n) {
    ctx->sim.partitions = n > 0 ? n : 1;
    return IGN_OK;
}

int ignref_refill_ghosts(ref_ctx* ctx) {
    return guarded(&ctx->err, [&] { ctx->sim.refill_ghosts(); });
}

int ignref_refresh_primitives(ref_ctx* ctx, int stage) {
    return guarded(&ctx->err, [&] { ctx->sim.refresh_primitives(stage); });
}

int ignref_prepare_stage(ref_ctx* ctx, int stage) {
    return guarded(&ctx->err, [&] { ctx->sim.prepare_stage(stage); });
}

int ignref_compute_rhs(ref_ctx* ctx, double t_stage, int stage, double* rhs) {
    return guarded(&ctx->err, [&] {
        FieldSet r;
        ctx->sim.compute_rhs(r, t_stage, stage);
        if (rhs) copy_out(r, ctx->ns + 3, rhs, ctx->plane);
    });
}

int ignref_stable_dt(ref_ctx* ctx, double* dt) {
    return guarded(&ctx->err, [&] { *dt = ctx->sim.stable_dt(); });
}

int ignref_rk3_step(ref_ctx* ctx, double dt) {
    return guarded(&ctx->err, [&] { ctx->sim.rk3_step(dt); });
}

// advance()'s loop body with a pinned step: rk3_step then prepare_stage(1)
// (solver.hpp:344-345), n times.
int ignref_rk3_steps(ref_ctx* ctx, double dt, int64_t n) {
    return guarded(&ctx->err, [&] {
        for (int64_t k = 0; k < n; ++k) {
            ctx->sim.rk3_step(dt);
            ctx->sim.prepare_stage(1);
        }
    });
}

int ignref_advance(ref_ctx* ctx, ign_step_hook hook, void* user) {
    return guarded(&ctx->err, [&] {
        if (hook) {
            // the ABI hook returns nonzero to stop; the reference's void hook
            // (solver.hpp:336-348) is stopped through its public loop bound
            const auto max_iter = ctx->sim.integ.max_iter;
            ctx->sim.advance([&](Simulation& s) {
                if (hook(ctx, user) != 0) s.integ.max_iter = s.iter;
            });
            ctx->sim.integ.max_iter = max_iter;
        } else
            ctx->sim.advance();
    });
}

int ignref_conserved_totals(ref_ctx* ctx, double* tot) {
    const auto v = ctx->sim.conserved_totals();
    for (std::size_t c = 0; c < v.size(); ++c) tot[c] = v[c];
    return IGN_OK;
}

int ignref_product_mole_fraction(ref_ctx* ctx, double* out) {
    *out = ctx->sim.product_mole_fraction();
    return IGN_OK;
}

int ignref_last_clip(const ref_ctx* ctx, double* clip) {
    *clip = ctx->sim.last_clip;
    return IGN_OK;
}

// The reference always reduces serially (solver.hpp:387-418): any mode reads
// the same values.
int ignref_set_diagnostics(ref_ctx* ctx, int mode) {
    (void)ctx;
    return mode == IGN_DIAG_DEVICE || mode == IGN_DIAG_REFERENCE ? IGN_OK : IGN_USAGE_ERROR;
}

// 3D extension checker (ref3d_faces.hpp): the inviscid RHS of a padded 3D
// state Ut given the product's primitive cache (rho, u, v, w, p, T, c, Y_s);
// rhs = nc padded planes, interior written.  Returns IGN_OK or the error.
int ignref3d_inviscid_rhs(const ign_config* cfg, const double* Ut, const double* prim,
                          double* rhs, ign_error* err) {
    return guarded(err, [&] {
        if (cfg->nz <= 0) throw UsageError("ref3d: nz must be > 0");
        const Mesh mesh = make_mesh(*cfg);
        const SchemeConfig sc = to_scheme(cfg->scheme);
        const MetricField met = compute_metrics(mesh, inviscid_mode(*cfg, sc), cfg->skew_beta);
        const ref3d::Met3 M = ref3d::extrude(met, cfg->lz / cfg->nz);
        const MixtureModel mix = to_mix(cfg->mix);
        ref3d::Grid G{cfg->nx, cfg->ny, cfg->nz, cfg->g, mix.ns(), 0, 0, 0};
        G.sx = cfg->nx + 2 * cfg->g;
        G.sxy = G.sx * (cfg->ny + 2 * cfg->g);
        G.plane = G.sxy * (cfg->nz + 2 * cfg->g);
        ref3d::inviscid_rhs(G, M, mix, sc, Ut, prim, rhs);
    });
}

// The 3D extension's viscous divergence (oracle/ref3d_viscous.hpp) from the
// product's primitive cache; interior of the returned planes written.
int ignref3d_viscous_rhs(const ign_config* cfg, const double* prim, double* dv,
                         ign_error* err) {
    return guarded(err, [&] {
        if (cfg->nz <= 0) throw UsageError("ref3d: nz must be > 0");
        const Mesh mesh = make_mesh(*cfg);
        const MetricField metv = compute_metrics(mesh, MetricMode::Central2);
        const ref3d::Met3 Mv = ref3d::extrude(metv, cfg->lz / cfg->nz);
        const MixtureModel mix = to_mix(cfg->mix);
        ref3d::Grid G{cfg->nx, cfg->ny, cfg->nz, cfg->g, mix.ns(), 0, 0, 0};
        G.sx = cfg->nx + 2 * cfg->g;
        G.sxy = G.sx * (cfg->ny + 2 * cfg->g);
        G.plane = G.sxy * (cfg->nz + 2 * cfg->g);
        ref3d::viscous_rhs(G, Mv, mix, prim, dv);
    });
}

// n advance() steps of the 3D extension (every edge rule, LODI, chemistry, laser)
// (oracle/ref3d_step.hpp) from the product's state and primitive cache
// (Ut: nc planes, prim: rho, u, v, w, p, T, c, Y_s planes; both in/out).
int ignref3d_steps(const ign_config* cfg, double* Ut, double* prim, double t0, double dt, int n,
                   ign_error* err) {
    return guarded(err, [&] {
        if (cfg->nz <= 0) throw UsageError("ref3d: nz must be > 0");
        const ign_edge* e[4] = {&cfg->bc.left, &cfg->bc.right, &cfg->bc.bottom, &cfg->bc.top};
        Simulation sim;  // the reference's mesh, bc, mech, laser for this config
        init_sim(sim, cfg);
        const Mesh& mesh = sim.mesh;
        const SchemeConfig sc = to_scheme(cfg->scheme);
        const double dz = cfg->lz / cfg->nz;
        ref3d::Run3 R;
        R.M = ref3d::extrude(compute_metrics(mesh, inviscid_mode(*cfg, sc), cfg->skew_beta), dz);
        R.Mv = ref3d::extrude(compute_metrics(mesh, MetricMode::Central2), dz);
        R.mix = to_mix(cfg->mix);
        R.sc = sc;
        R.viscous = cfg->viscous != 0;
        R.S = &sim;
        R.laser_zmode = cfg->laser.zmode;
        R.laser_z0 = cfg->laser.z0;
        R.zc0 = cfg->center_z - 0.5 * cfg->lz;
        R.dz = dz;
        R.time = t0;
        for (int q = 0; q < 4; ++q) {
            R.etype[q] = e[q]->type;
            R.Twall[q] = e[q]->T_wall;
        }
        if (!cfg->periodic_z) {
            R.ztype[0] = cfg->zlo.type;
            R.ztype[1] = cfg->zhi.type;
            R.Tzwall[0] = cfg->zlo.T_wall;
            R.Tzwall[1] = cfg->zhi.T_wall;
            if (R.ztype[0] == 0 || R.ztype[1] == 0 || R.ztype[0] == 3 || R.ztype[1] == 3)
                throw UsageError("ref3d_steps: z edges periodic_z or walls / outflow");
        }
        ref3d::Grid& G = R.G;
        G = ref3d::Grid{cfg->nx, cfg->ny, cfg->nz, cfg->g, R.mix.ns(), 0, 0, 0};
        G.sx = cfg->nx + 2 * cfg->g;
        G.sxy = G.sx * (cfg->ny + 2 * cfg->g);
        G.plane = G.sxy * (cfg->nz + 2 * cfg->g);
        const size_t nU = size_t(G.ns + 4) * G.plane, nP = size_t(G.ns + 7) * G.plane;
        R.Ut.assign(Ut, Ut + nU);
        R.prim.assign(prim, prim + nP);
        R.steps(dt, n);
        std::copy(R.Ut.begin(), R.Ut.end(), Ut);
        std::copy(R.prim.begin(), R.prim.end(), prim);
    });
}

int ignref_host_metrics(const ign_config* cfg, int which, double* out,
                        ign_error* err) {
    return guarded(err, [&] {
        const Mesh m = make_mesh(*cfg);
        const SchemeConfig sc = to_scheme(cfg->scheme);
        const MetricField mf =
            which == 0 ? compute_metrics(m, inviscid_mode(*cfg, sc), cfg->skew_beta)
                       : compute_metrics(m, MetricMode::Central2);
        const std::size_t P = mf.jac.raw().size();
        const Field* f[5] = {&mf.jac, &mf.m_xi_x, &mf.m_xi_y, &mf.m_eta_x,
                             &mf.m_eta_y};
        for (int k = 0; k < 5; ++k) copy_field(*f[k], out + k * P, P);
    });
}

int ignref_host_mesh(const ign_config* cfg, double* x, double* y,
                     ign_error* err) {
    return guarded(err, [&] {
        const Mesh m = make_mesh(*cfg);
        const std::size_t P = m.x.raw().size();
        copy_field(m.x, x, P);
        copy_field(m.y, y, P);
    });
}

// IGNS v1 snapshot round trip through the reference's own IO
// (snapshot.hpp:52-145).
int ignref_write_snapshot(ref_ctx* ctx, const char* path) {
    return guarded(&ctx->err, [&] { write_snapshot(ctx->sim, path); });
}

int ignref_read_snapshot(ref_ctx* ctx, const char* path) {
    return guarded(&ctx->err, [&] {
        const SnapshotData sd = read_snapshot(path);
        apply_snapshot(sd, ctx->sim);
    });
}

// probes and the product-fraction trace (solver.hpp:68-74, 130-135, 351-385)
int ignref_add_probe(ref_ctx* ctx, int32_t i0, int32_t j0, int32_t i1, int32_t j1) {
    return guarded(&ctx->err, [&] { ctx->sim.add_probe(ProbeSpec{i0, j0, i1, j1}); });
}

int ignref_set_sampling(ref_ctx* ctx, int32_t probe_interval, int32_t trace_interval) {
    ctx->sim.probe_interval = probe_interval;
    ctx->sim.trace_interval = trace_interval;
    return IGN_OK;
}

int ignref_probe_samples(const ref_ctx* ctx, int32_t probe, int64_t* n, double* times,
                         double* rows) {
    if (probe < 0 || probe >= (int)ctx->sim.probes.size()) return IGN_USAGE_ERROR;
    const auto& pr = ctx->sim.probes[probe];
    if (n) *n = (int64_t)pr.times.size();
    for (std::size_t k = 0; k < pr.times.size(); ++k) {
        if (times) times[k] = pr.times[k];
        if (rows)
            for (std::size_t q = 0; q < pr.rows[k].size(); ++q)
                rows[k * pr.rows[k].size() + q] = pr.rows[k][q];
    }
    return IGN_OK;
}

int ignref_trace_samples(const ref_ctx* ctx, int64_t* n, double* times, double* values) {
    const auto& tr = ctx->sim.product_fraction;
    if (n) *n = (int64_t)tr.times.size();
    for (std::size_t k = 0; k < tr.times.size(); ++k) {
        if (times) times[k] = tr.times[k];
        if (values) values[k] = tr.values[k];
    }
    return IGN_OK;
}

int ignref_set_config_hash(ref_ctx* ctx, uint64_t hash) {
    ctx->sim.config_hash = hash;
    return IGN_OK;
}

int ignref_get_config_hash(const ref_ctx* ctx, uint64_t* hash) {
    *hash = ctx->sim.config_hash;
    return IGN_OK;
}

int64_t ignref_kernel_launches(const ref_ctx*) { return 0; }

} // extern "C"
