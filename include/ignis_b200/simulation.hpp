// ignis_b200/simulation.hpp — header-only C++ facade over the C ABI
// (include/ignis_b200.h) with the reference's class name, method names and
// exception types (solver.hpp:53-853, errors.hpp:10-47), so a caller of
// ignis::Simulation switches by changing the include and the namespace.
//
//   ignis_b200::Simulation sim(cfg);              // Simulation::init
//   sim.set_initial_condition([](double x, double y) { ...; return pt; });
//   sim.prepare_stage(1);
//   sim.compute_rhs(rhs, t, 1);                   // host buffer, padded layout
//   sim.rk3_step(dt);
//   sim.advance();
//
// Field access is by copy (get_state / set_state): the state lives on the GPU.
#pragma once

#include <cstdint>
#include <cstdio>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "ignis_b200.h"

namespace ignis_b200 {

struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct StateError : std::runtime_error { using std::runtime_error::runtime_error; };
struct NumericsError : std::runtime_error { using std::runtime_error::runtime_error; };
struct StepFailure : NumericsError {
    StepFailure(const std::string& w, int s, int i_, int j_, int k_ = 0)
        : NumericsError(w), stage(s), i(i_), j(j_), k(k_) {}
    int stage, i, j, k;  // k: z plane (3D extension), 0 in 2D
};
struct FormatError : std::runtime_error { using std::runtime_error::runtime_error; };
struct UsageError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DeviceError : std::runtime_error { using std::runtime_error::runtime_error; };

inline void throw_status(int st, const ign_error& e) {
    const std::string m = e.msg;
    switch (st) {
    case IGN_OK: return;
    case IGN_CONFIG_ERROR: throw ConfigError(m);
    case IGN_STATE_ERROR: throw StateError(m);
    case IGN_NUMERICS_ERROR: throw NumericsError(m);
    case IGN_STEP_FAILURE: throw StepFailure(m, e.stage, e.i, e.j, e.k);
    case IGN_FORMAT_ERROR: throw FormatError(m);
    case IGN_USAGE_ERROR: throw UsageError(m);
    default: throw DeviceError(m);
    }
}

class Simulation {
public:
    explicit Simulation(const ign_config& cfg) {
        const int st = ign_create(&cfg, &h_);
        if (st != IGN_OK) {
            ign_error e{};
            std::snprintf(e.msg, sizeof e.msg, "ign_create failed");
            throw_status(st, e);
        }
        ign_dims(h_, &nx_, &ny_, &g_, &ns_);
        ign_dims3(h_, &nz_, nullptr, nullptr);
    }
    ~Simulation() { ign_destroy(h_); }
    Simulation(const Simulation&) = delete;
    Simulation& operator=(const Simulation&) = delete;

    int ns() const { return ns_; }
    int ncomp() const { return ns_ + (nz_ > 0 ? 4 : 3); }
    size_t plane() const {
        return size_t(nx_ + 2 * g_) * (ny_ + 2 * g_) * (nz_ > 0 ? size_t(nz_ + 2 * g_) : 1);
    }

    // solver.hpp:115-128
    void set_initial_condition(const std::function<ign_prim_point(double, double)>& ic) {
        auto tramp = [](double x, double y, void* u, ign_prim_point* out) {
            *out = (*static_cast<const std::function<ign_prim_point(double, double)>*>(u))(x, y);
        };
        check(ign_set_initial_condition(h_, tramp, const_cast<void*>(static_cast<const void*>(&ic))));
    }
    void refill_ghosts() { check(ign_refill_ghosts(h_)); }               // solver.hpp:144
    void refresh_primitives(int stage) { check(ign_refresh_primitives(h_, stage)); }
    void prepare_stage(int stage) { check(ign_prepare_stage(h_, stage)); }  // :422
    // solver.hpp:185; rhs resized to ncomp()*plane() doubles (padded layout)
    void compute_rhs(std::vector<double>& rhs, double t_stage, int stage = 0) {
        rhs.resize(ncomp() * plane());
        check(ign_compute_rhs(h_, t_stage, stage, rhs.data()));
    }
    double stable_dt() { double dt; check(ign_stable_dt(h_, &dt)); return dt; }  // :240
    void rk3_step(double dt) { check(ign_rk3_step(h_, dt)); }                 // :304
    void advance() { check(ign_advance(h_, nullptr, nullptr)); }             // :336
    std::vector<double> conserved_totals() {                                 // :411
        std::vector<double> t(ncomp());
        check(ign_conserved_totals(h_, t.data()));
        return t;
    }
    double product_mole_fraction() { double v; check(ign_product_mole_fraction(h_, &v)); return v; }
    std::vector<double> get_state() {
        std::vector<double> u(ncomp() * plane());
        check(ign_get_state(h_, u.data()));
        return u;
    }
    void set_state(const std::vector<double>& u, const double* Tcache = nullptr) {
        check(ign_set_state(h_, u.data(), Tcache));
    }
    double time() const { double t; int64_t it; ign_get_time(h_, &t, &it); return t; }
    long iter() const { double t; int64_t it; ign_get_time(h_, &t, &it); return (long)it; }
    void set_integrator(const ign_integrator& in) { check(ign_set_integrator(h_, &in)); }

    // outputs (solver.hpp:68-74, 130-135, 351-385)
    struct ProbeSpec { int i0 = 0, j0 = 0, i1 = 0, j1 = 0; };
    struct ProbeSeries { std::vector<double> times; std::vector<std::vector<double>> rows; };
    void add_probe(const ProbeSpec& p) { check(ign_add_probe(h_, p.i0, p.j0, p.i1, p.j1)); }
    void set_sampling(int probe_interval, int trace_interval) {
        check(ign_set_sampling(h_, probe_interval, trace_interval));
    }
    ProbeSeries probe(int k) {
        int64_t n = 0;
        check(ign_probe_samples(h_, k, &n, nullptr, nullptr));
        std::vector<double> t(n), r(n * (5 + ns_));
        check(ign_probe_samples(h_, k, &n, t.data(), r.data()));
        ProbeSeries ps{t, {}};
        for (int64_t i = 0; i < n; ++i)
            ps.rows.emplace_back(r.begin() + i * (5 + ns_), r.begin() + (i + 1) * (5 + ns_));
        return ps;
    }
    std::uint64_t config_hash() const { std::uint64_t h; ign_get_config_hash(h_, &h); return h; }
    void set_config_hash(std::uint64_t h) { check(ign_set_config_hash(h_, h)); }
    ign_context* handle() { return h_; }

private:
    void check(int st) {
        if (st == IGN_OK) return;
        ign_error e{};
        ign_last_error(h_, &e);
        throw_status(st, e);
    }
    ign_context* h_ = nullptr;
    int32_t nx_ = 0, ny_ = 0, g_ = 0, ns_ = 0, nz_ = 0;
};

// snapshot.hpp:52-145: write_snapshot(sim, path); read_snapshot + apply_snapshot
inline void write_snapshot(Simulation& sim, const std::string& path) {
    const int st = ign_write_snapshot(sim.handle(), path.c_str());
    if (st != IGN_OK) {
        ign_error e{};
        ign_last_error(sim.handle(), &e);
        throw_status(st, e);
    }
}
inline void read_and_apply_snapshot(Simulation& sim, const std::string& path) {
    const int st = ign_read_snapshot(sim.handle(), path.c_str());
    if (st != IGN_OK) {
        ign_error e{};
        ign_last_error(sim.handle(), &e);
        throw_status(st, e);
    }
}

}  // namespace ignis_b200
