// TEST INFRASTRUCTURE: the reference-typed drop-in (include/ignis_b200/drop_in.hpp)
// against the unmodified reference class, both driven by the SAME caller code
// (a template over the simulation type) — the migration a reference user makes.
// Built against the reference headers and libignis_b200.so; run on a GPU box.
// Exit 0 and "drop_in parity OK" when every check holds.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iterator>
#include <string>

#include "ignis/snapshot.hpp"
#include "ignis/solver.hpp"
#include "ignis_b200/drop_in.hpp"

using namespace ignis;
using B200 = ignis_b200::drop_in::Simulation;

static int g_fail = 0;
#define CHECK(cond, what)                                 \
    do {                                                  \
        if (!(cond)) {                                    \
            std::printf("FAIL %s (line %d)\n", what, __LINE__); \
            ++g_fail;                                     \
        }                                                 \
    } while (0)

static double field_err(const FieldSet& a, const FieldSet& b, bool interior_only) {
    double m = 0.0;
    for (int c = 0; c < a.ncomp(); ++c) {
        double scale = 0.0, d = 0.0;
        for (int j = interior_only ? 0 : -a.ghosts(); j < a.ny() + (interior_only ? 0 : a.ghosts()); ++j)
            for (int i = interior_only ? 0 : -a.ghosts(); i < a.nx() + (interior_only ? 0 : a.ghosts()); ++i) {
                scale = std::max(scale, std::abs(b[c](i, j)));
                d = std::max(d, std::abs(a[c](i, j) - b[c](i, j)));
            }
        m = std::max(m, scale > 0 ? d / scale : d);
    }
    return m;
}
static bool bitwise(const FieldSet& a, const FieldSet& b) {
    for (int c = 0; c < a.ncomp(); ++c)
        if (std::memcmp(a[c].raw().data(), b[c].raw().data(), a[c].raw().size() * 8) != 0)
            return false;
    return true;
}
static std::string slurp(const std::string& p) {
    std::ifstream f(p, std::ios::binary);
    return std::string(std::istreambuf_iterator<char>(f), {});
}

// the caller code, identical for both types
template <class Sim> void setup_tgv(Sim& sim, int n, const Mesh* custom = nullptr) {
    const double L = 2.0 * M_PI;
    MixtureModel mix = MixtureModel::calorically_perfect(1.4, 1.0, 6.25e-4);
    mix.species[0].pieces[0].t_hi = 1e6;
    SchemeConfig sc;
    BoundarySpec bs;
    sim.init(custom ? *custom : build_uniform(n, n, L, L), Sim::metric_mode_for(sc), 0.0, mix,
             sc, bs);
    sim.viscous = true;
    const double p0 = 1.0 / (1.4 * 0.01);
    sim.set_initial_condition([&](double x, double y) {
        PrimPoint q;
        q.rho = 1.0;
        q.u = std::sin(x) * std::cos(y);
        q.v = -std::cos(x) * std::sin(y);
        q.p = p0 + 0.25 * (std::cos(2.0 * x) + std::cos(2.0 * y));
        q.T = q.p / q.rho;
        q.Y[0] = 1.0;
        return q;
    });
}

// the repo's one-step H2/O2 table (data/h2_o2.mix; the mechanism filled by
// hand as SURVEY §8c prescribes: make_one_step_mechanism hard-codes CH4)
template <class Sim> void setup_h2o2(Sim& sim, int n) {
    const double L = 0.01;
    MixtureModel mix = load_mixture_file(REPO_DATA_DIR "/h2_o2.mix");
    SchemeConfig sc;
    BoundarySpec bs;
    sim.init(build_uniform(n, n, L, L), Sim::metric_mode_for(sc), 0.0, mix, sc, bs);
    sim.viscous = true;
    ReactionMechanism mk;
    mk.A = 1e9;
    mk.Ta = 15000.0;
    mk.a = mk.b = 1.0;
    mk.T_cutoff = 300.0;
    mk.i_fuel = 0;
    mk.i_ox = 1;
    mk.i_co2 = -1;
    mk.i_h2o = 2;
    const double nu[4] = {-2.0, -1.0, 2.0, 0.0};
    for (int s = 0; s < 4; ++s) mk.nu[s] = nu[s];
    sim.mech = mk;
    LaserParams lp;
    lp.energy = 2.0;
    lp.sigma_r = 8e-4;
    lp.sigma_t = 2e-6;
    lp.x0 = 1e-3;
    lp.y0 = -5e-4;
    lp.t0 = 1e-6;
    sim.laser = lp;
    sim.set_initial_condition([&](double x, double y) {
        const double r2 = (x - 1e-3) * (x - 1e-3) + (y + 1e-3) * (y + 1e-3);
        const double f = std::exp(-r2 / (2.0 * 1.5e-3 * 1.5e-3));
        PrimPoint q;
        const double Y0[4] = {0.03, 0.22, 0.0, 0.75}, Yb[4] = {0.005, 0.1, 0.2, 0.695};
        double tot = 0.0;
        for (int s = 0; s < 4; ++s) tot += (q.Y[s] = Y0[s] * (1 - f) + Yb[s] * f);
        for (int s = 0; s < 4; ++s) q.Y[s] /= tot;
        q.T = 300.0 + 1700.0 * f;
        q.rho = 101325.0 / (thermo::r_specific(q.Y, mix) * q.T);
        q.u = 3.0 * std::sin(2 * M_PI * y / L);
        q.v = -2.0 * std::cos(2 * M_PI * x / L);
        return q;
    });
    sim.add_probe(ProbeSpec{2, 3, 10, 12});
    sim.probe_interval = 2;
    sim.trace_interval = 1;
}

int main() {
    try {
        {  // 2D TGV, gamma-gas: everything bitwise
            ignis::Simulation ref;
            B200 gpu;
            setup_tgv(ref, 48);
            setup_tgv(gpu, 48);
            CHECK(bitwise(gpu.Ut, ref.Ut), "tgv initial condition");
            ref.prepare_stage(1);
            gpu.prepare_stage(1);
            CHECK(std::memcmp(gpu.T.raw().data(), ref.T.raw().data(), ref.T.raw().size() * 8) == 0,
                  "tgv primitive cache T");
            FieldSet ra(ref.comp().ncomp(), 48, 48, 3), rb(ref.comp().ncomp(), 48, 48, 3);
            ref.compute_rhs(ra, 0.0, 1);
            gpu.compute_rhs(rb, 0.0, 1);
            CHECK(bitwise(ra, rb), "tgv compute_rhs");
            CHECK(gpu.stable_dt() == ref.stable_dt(), "tgv stable_dt");
            const double dt = 0.4 * (2 * M_PI / 48) / (2.0 * (std::sqrt(1.4 / (1.4 * 0.01)) + 1.0));
            for (int k = 0; k < 5; ++k) {
                ref.rk3_step(dt);
                ref.prepare_stage(1);
                gpu.rk3_step(dt);
                gpu.prepare_stage(1);
            }
            CHECK(bitwise(gpu.Ut, ref.Ut), "tgv 5 rk3 steps");
            int ha = 0, hb = 0;
            ref.integ.fixed_dt = gpu.integ.fixed_dt = dt;
            ref.integ.t_end = gpu.integ.t_end = ref.time + 4.5 * dt;
            ref.advance([&](ignis::Simulation& s) { ha += (int)(s.iter % 7); });
            gpu.advance([&](B200& s) { hb += (int)(s.iter % 7); });
            CHECK(ha == hb && gpu.iter == ref.iter && gpu.time == ref.time, "tgv advance + hook");
            CHECK(bitwise(gpu.Ut, ref.Ut), "tgv advance state");
            CHECK(gpu.conserved_totals() == ref.conserved_totals(), "tgv conserved_totals");
            ignis::write_snapshot(ref, "/tmp/dropin_ref.igns");
            ignis_b200::drop_in::write_snapshot(gpu, "/tmp/dropin_b200.igns");
            CHECK(slurp("/tmp/dropin_ref.igns") == slurp("/tmp/dropin_b200.igns"),
                  "snapshot bytes");
            // restart from the reference's file, step both again
            const SnapshotData sd = read_snapshot("/tmp/dropin_ref.igns");
            apply_snapshot(sd, ref);
            ignis_b200::drop_in::apply_snapshot(sd, gpu);
            ref.prepare_stage(1);
            gpu.prepare_stage(1);
            ref.rk3_step(dt);
            gpu.rk3_step(dt);
            CHECK(bitwise(gpu.Ut, ref.Ut) && gpu.iter == ref.iter, "restart step");
            // StepFailure: U0 restored, same stage and location
            ref.prepare_stage(1);
            gpu.prepare_stage(1);
            int sa = -1, sb = -2, ia = 0, ib = 1, ja = 0, jb = 1;
            std::string wa, wb;
            try { ref.rk3_step(50.0); } catch (const StepFailure& e) { sa = e.stage; ia = e.i; ja = e.j; wa = e.what(); }
            catch (const std::exception& e) { wa = std::string("other: ") + e.what(); }
            try { gpu.rk3_step(50.0); } catch (const StepFailure& e) { sb = e.stage; ib = e.i; jb = e.j; wb = e.what(); }
            catch (const std::exception& e) { wb = std::string("other: ") + e.what(); }
            if (!(sa == sb && ia == ib && ja == jb && sa > 0))
                std::printf("reference: %d (%d,%d) %s\nb200: %d (%d,%d) %s\n", sa, ia, ja, wa.c_str(),
                            sb, ib, jb, wb.c_str());
            CHECK(sa == sb && ia == ib && ja == jb && sa > 0, "StepFailure payload");
            CHECK(bitwise(gpu.Ut, ref.Ut), "StepFailure restores U0");
        }
        {  // a hand-built (stretched, sheared) Mesh
            Mesh m = build_uniform(40, 40, 2 * M_PI, 2 * M_PI);
            for (int j = -m.g; j < m.ny + m.g; ++j)
                for (int i = -m.g; i < m.nx + m.g; ++i) {
                    const double x = m.x(i, j), y = m.y(i, j);
                    m.x(i, j) = x + 0.08 * std::sin(x) + 0.03 * std::sin(y);
                    m.y(i, j) = y + 0.05 * std::sin(x + 0.5);
                }
            ignis::Simulation ref;
            B200 gpu;
            setup_tgv(ref, 40, &m);
            setup_tgv(gpu, 40, &m);
            ref.prepare_stage(1);
            gpu.prepare_stage(1);
            for (int k = 0; k < 3; ++k) {
                ref.rk3_step(1e-3);
                ref.prepare_stage(1);
                gpu.rk3_step(1e-3);
                gpu.prepare_stage(1);
            }
            CHECK(bitwise(gpu.Ut, ref.Ut), "hand-built mesh 3 steps");
        }
        {  // H2/O2 reacting with laser, probes, trace: tolerance (device libm)
            ignis::Simulation ref;
            B200 gpu;
            setup_h2o2(ref, 24);
            setup_h2o2(gpu, 24);
            const double dt = 0.2 * (0.01 / 24) / 900.0;
            ref.integ.fixed_dt = gpu.integ.fixed_dt = dt;
            ref.integ.t_end = gpu.integ.t_end = 10.5 * dt;
            ref.advance();
            gpu.advance();
            CHECK(gpu.iter == ref.iter && gpu.iter == 11, "h2o2 advance iterations");
            CHECK(field_err(gpu.Ut, ref.Ut, true) <= 1e-10, "h2o2 11 steps within 1e-10");
            CHECK(gpu.probes[0].rows.size() == ref.probes[0].rows.size(), "h2o2 probe samples");
            CHECK(gpu.product_fraction.values.size() == ref.product_fraction.values.size(),
                  "h2o2 trace samples");
            double dtr = 0.0;
            for (size_t k = 0; k < ref.product_fraction.values.size(); ++k)
                dtr = std::max(dtr, std::abs(gpu.product_fraction.values[k] -
                                             ref.product_fraction.values[k]) /
                                        std::abs(ref.product_fraction.values[k]));
            CHECK(dtr <= 1e-10, "h2o2 trace within 1e-10");
            CHECK(std::abs(gpu.last_clip - ref.last_clip) <= 1e-10 * (1.0 + ref.last_clip),
                  "h2o2 last_clip");
        }
    } catch (const std::exception& e) {
        std::printf("exception: %s\n", e.what());
        return 3;
    }
    if (g_fail) {
        std::printf("drop_in parity: %d failures\n", g_fail);
        return 1;
    }
    std::printf("drop_in parity OK\n");
    return 0;
}
