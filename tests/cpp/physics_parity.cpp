// tests/cpp/physics_parity.cpp — TEST INFRASTRUCTURE (CPU, this container only).
//
// Compiles the product's point physics (paper_2202_02319_b200/csrc/physics.cuh,
// flux.cuh: the exact source the sm_100a kernels are built from) for the host
// and checks it BITWISE against the unmodified reference functions
// (/root/reference/proj/include/ignis/*.hpp) on seeded random inputs.  This pins
// the operation-order transcription independently of the GPU; the device
// build adds only nvcc's libm (exp/log/pow/hypot), covered by the GPU tests.
#include <cstdio>
#include <cstring>
#include <random>
#include <string>

#include "ignis/solver.hpp"
#include "flux.cuh"
#include "host_core.hpp"
#include "physics.cuh"

static int g_fail = 0, g_checks = 0;

static bool same(double a, double b) {
    return std::memcmp(&a, &b, sizeof(double)) == 0 || (std::isnan(a) && std::isnan(b));
}

#define EXPECT_BITWISE(what, a, b)                                                       \
    do {                                                                                 \
        ++g_checks;                                                                      \
        const double _a = (a), _b = (b);                                                 \
        if (!same(_a, _b)) {                                                             \
            if (g_fail < 30)                                                             \
                std::printf("MISMATCH %s: product %.17g reference %.17g\n", what, _a, _b); \
            ++g_fail;                                                                    \
        }                                                                                \
    } while (0)

static ign_mixture to_abi(const ignis::MixtureModel& m) {
    ign_mixture o;
    std::memset(&o, 0, sizeof(o));
    o.mode = m.mode == ignis::MixtureModel::Mode::CaloricallyPerfect ? 0 : 1;
    o.ns = m.ns();
    o.R = m.R;
    o.Le = m.Le;
    o.Pr = m.Pr;
    for (int s = 0; s < m.ns(); ++s) {
        const auto& sp = m.species[s];
        std::snprintf(o.species[s].name, IGN_NAME_LEN, "%s", sp.name.c_str());
        o.species[s].W = sp.W;
        o.species[s].mu_ref = sp.mu_ref;
        o.species[s].t_ref = sp.t_ref;
        o.species[s].n_exp = sp.n_exp;
        o.species[s].npieces = (int)sp.pieces.size();
        for (size_t k = 0; k < sp.pieces.size(); ++k) {
            const auto& p = sp.pieces[k];
            ign_thermo_piece& q = o.species[s].pieces[k];
            q.t_lo = p.t_lo; q.t_hi = p.t_hi; q.cm2 = p.cm2; q.cm1 = p.cm1; q.c0 = p.c0;
            q.c1 = p.c1; q.c2 = p.c2; q.c3 = p.c3; q.c4 = p.c4; q.b = p.b;
        }
    }
    return o;
}

template <int NS>
static void check_mixture(const ignis::MixtureModel& mix, const char* name, unsigned seed) {
    const ign::DMix dm = ign::build_mix(to_abi(mix));
    std::mt19937 rng(seed);
    std::uniform_real_distribution<double> uT(250.0, 3200.0), uy(0.0, 1.0), ur(0.05, 5.0),
        uu(-400.0, 400.0);
    const double Tscale = mix.mode == ignis::MixtureModel::Mode::CaloricallyPerfect ? 0.05 : 1.0;
    char lbl[128];
    for (int trial = 0; trial < 2000; ++trial) {
        ignis::SpeciesArray Y{}, X{};
        double Yp[NS], Xp[NS];
        double sum = 0.0;
        for (int s = 0; s < NS; ++s) sum += (Y[s] = uy(rng) + 1e-3);
        for (int s = 0; s < NS; ++s) Yp[s] = (Y[s] /= sum);
        const double T = uT(rng) * Tscale;
        std::snprintf(lbl, sizeof lbl, "%s cp_mass", name);
        EXPECT_BITWISE(lbl, ign::cp_mass<NS>(T, Yp, dm), ignis::thermo::cp_mass(T, Y, mix));
        std::snprintf(lbl, sizeof lbl, "%s h_mass", name);
        EXPECT_BITWISE(lbl, ign::h_mass<NS>(T, Yp, dm), ignis::thermo::h_mass(T, Y, mix));
        // the branch-free (full Horner) forms of the primitive kernels
        std::snprintf(lbl, sizeof lbl, "%s cp_mass bf", name);
        EXPECT_BITWISE(lbl, (ign::cp_mass<NS, true>(T, Yp, dm)), ignis::thermo::cp_mass(T, Y, mix));
        std::snprintf(lbl, sizeof lbl, "%s h_mass bf", name);
        EXPECT_BITWISE(lbl, (ign::h_mass<NS, true>(T, Yp, dm)), ignis::thermo::h_mass(T, Y, mix));
        const double rs = ign::r_specific<NS>(Yp, dm);
        EXPECT_BITWISE("r_specific", rs, ignis::thermo::r_specific(Y, mix));
        EXPECT_BITWISE("e_mass", ign::e_mass_rs<NS>(T, Yp, rs, dm), ignis::thermo::e_mass(T, Y, mix));
        EXPECT_BITWISE("sound_speed", ign::sound_speed_rs<NS>(T, Yp, rs, dm),
                       ignis::thermo::sound_speed(T, Y, mix));
        EXPECT_BITWISE("sound_speed bf", (ign::sound_speed_rs<NS, true>(T, Yp, rs, dm)),
                       ignis::thermo::sound_speed(T, Y, mix));
        EXPECT_BITWISE("mean_molar_mass", ign::mean_molar_mass<NS>(Yp, dm),
                       ignis::thermo::mean_molar_mass(Y, mix));
        ign::mole_fractions<NS>(Yp, dm, Xp);
        ignis::thermo::mole_fractions(Y, mix, X);
        for (int s = 0; s < NS; ++s) EXPECT_BITWISE("mole_fractions", Xp[s], X[s]);
        for (int s = 0; s < NS; ++s)
            EXPECT_BITWISE("h_species", ign::h_species(T, dm.sp[s], dm.R),
                           ignis::thermo::h_species(T, s, mix));
        // transport (thermo.hpp:231-262)
        ignis::ThermoState st;
        st.rho = ur(rng);
        st.T = T;
        st.Y = Y;
        st.X = X;
        ignis::transport(st, mix);
        double mu, lam, D, cp;
        ign::transport<NS>(st.rho, T, Yp, Xp, dm, mu, lam, D, cp);
        EXPECT_BITWISE("transport mu", mu, st.mu);
        EXPECT_BITWISE("transport lambda", lam, st.lambda);
        EXPECT_BITWISE("transport D", D, st.D[0]);
        // conservative <-> primitive with a perturbed guess (state.hpp:26-57)
        ignis::PrimPoint pt;
        pt.rho = ur(rng);
        pt.u = uu(rng) * Tscale;
        pt.v = uu(rng) * Tscale;
        pt.T = T;
        pt.Y = Y;
        const ignis::ConsVec U = ignis::conservative_from_primitives(pt, mix);
        ign::Prim<NS> pp;
        pp.rho = pt.rho; pp.u = pt.u; pp.v = pt.v; pp.T = pt.T; pp.p = 0.0;
        for (int s = 0; s < NS; ++s) pp.Y[s] = Yp[s];
        double Up[NS + 3];
        ign::conservative_from_primitives<NS>(pp, dm, Up);
        for (int c = 0; c < NS + 3; ++c) EXPECT_BITWISE("conservative_from_primitives", Up[c], U[c]);
        const double guess = T * (0.5 + uy(rng));
        const ignis::PrimPoint back = ignis::primitives_from_conservative(U.data(), mix, guess);
        ign::Prim<NS> bp;
        double rsb;
        const int pst = ign::primitives_from_conservative<NS>(U.data(), dm, guess, bp, &rsb);
        ++g_checks;
        if (pst != 0) { ++g_fail; std::printf("primitives status %d\n", pst); continue; }
        EXPECT_BITWISE("prim T", bp.T, back.T);
        EXPECT_BITWISE("prim p", bp.p, back.p);
        EXPECT_BITWISE("prim u", bp.u, back.u);
        ign::Prim<NS> bq;
        double rsq;
        if (ign::primitives_from_conservative<NS, true>(U.data(), dm, guess, bq, &rsq) == 0) {
            EXPECT_BITWISE("prim T bf", bq.T, back.T);
            EXPECT_BITWISE("prim p bf", bq.p, back.p);
        } else {
            ++g_fail;
        }
        // Roe average + eigensystem (flux.hpp:55-186) between two random states
        ignis::SpeciesArray Y2{};
        double Y2p[NS], s2 = 0.0;
        for (int s = 0; s < NS; ++s) s2 += (Y2[s] = uy(rng) + 1e-3);
        for (int s = 0; s < NS; ++s) Y2p[s] = (Y2[s] /= s2);
        const double T2 = uT(rng) * Tscale, r1 = ur(rng), r2 = ur(rng);
        const double u1 = uu(rng) * Tscale, v1 = uu(rng) * Tscale, u2 = uu(rng) * Tscale,
                     v2 = uu(rng) * Tscale;
        const ignis::RoeAverage ra = ignis::roe_average(r1, Y, T, u1, v1, r2, Y2, T2, u2, v2, mix);
        double Ya[NS], Ta, ua, va;
        ign::roe_average<NS>(r1, Yp, T, u1, v1, r2, Y2p, T2, u2, v2, dm, Ya, Ta, ua, va);
        EXPECT_BITWISE("roe T", Ta, ra.T);
        EXPECT_BITWISE("roe u", ua, ra.u);
        const double m1 = uu(rng) / 400.0, m2 = uu(rng) / 400.0;
        const ignis::EigenSystem es = ignis::EigenSystem::at_state(ra.Y, ra.T, ra.u, ra.v, m1, m2, mix);
        ign::Eigen<NS> ep;
        ign::eigen_at_state<NS>(Ya, Ta, ua, va, m1, m2, dm, ep);
        EXPECT_BITWISE("eigen c", ep.c, es.c);
        EXPECT_BITWISE("eigen kappa", ep.kappa, es.kappa);
        double q[NS + 3], w1[NS + 3], w2[ignis::kMaxComp], a1[NS + 3], a2[ignis::kMaxComp];
        for (int c = 0; c < NS + 3; ++c) q[c] = uu(rng);
        ign::eigen_project<NS>(ep, q, w1);
        es.project(q, w2);
        for (int c = 0; c < NS + 3; ++c) EXPECT_BITWISE("eigen project", w1[c], w2[c]);
        ign::eigen_assemble<NS>(ep, w1, a1);
        es.assemble(w2, a2);
        for (int c = 0; c < NS + 3; ++c) EXPECT_BITWISE("eigen assemble", a1[c], a2[c]);
        double F1[NS + 3], F2[ignis::kMaxComp];
        ign::mapped_flux<NS>(q, back.p, m1, m2, F1);
        ignis::mapped_flux(q, back.p, m1, m2, ignis::CompIndex{NS}, F2);
        for (int c = 0; c < NS + 3; ++c) EXPECT_BITWISE("mapped_flux", F1[c], F2[c]);
        // the face kernels' form: velocities from the primitive path's quotients
        double rq = 0.0;
        for (int s = 0; s < NS; ++s) rq += q[s];
        const double yq = 1.0 / rq;
        double F3[NS + 3];
        ign::mapped_flux_uv<NS>(q, back.p, ign::fdiv(q[NS], rq, yq), ign::fdiv(q[NS + 1], rq, yq),
                                m1, m2, F3);
        for (int c = 0; c < NS + 3; ++c) EXPECT_BITWISE("mapped_flux_uv", F3[c], F2[c]);
    }
}

// TENO6's cutoff filter (physics.cuh teno_cutoff_filter) at the decision
// boundary: for random stencils, ct is placed ON one candidate's exact ratio
// g_k/gsum (times 1 + O(1e-7 .. 1e-3) jitter, inside and outside the filter
// band), so
// every branch of the filter and its exact fallback is exercised.
static void check_teno_cutoff_boundary() {
    std::mt19937 rng(4242);
    std::uniform_real_distribution<double> u(-2.0, 2.0), jit(-3e-7, 3e-7), wide(-1.5e-3, 1.5e-3);
    std::uniform_int_distribution<int> pick(0, 3);
    std::uniform_real_distribution<double> lg(-12.0, 0.0);
    int filtered = 0, exact = 0;
    for (int trial = 0; trial < 300000; ++trial) {
        double w[6];
        const double amp = std::pow(10.0, lg(rng));  // discontinuity strength
        for (int q = 0; q < 6; ++q) w[q] = (q < 3 ? 1.0 : 0.0) + amp * u(rng);
        // exact ratios Q_k of the reference's sequence (reconstruction.hpp:65-115)
        const double v0 = w[0] - w[2], v1 = w[1] - w[2], v3 = w[3] - w[2], v4 = w[4] - w[2],
                     v5 = w[5] - w[2];
        const double b[4] = {
            (13.0 / 12.0) * (v0 - 2.0 * v1) * (v0 - 2.0 * v1) +
                0.25 * (v0 - 4.0 * v1) * (v0 - 4.0 * v1),
            (13.0 / 12.0) * (v1 + v3) * (v1 + v3) + 0.25 * (v1 - v3) * (v1 - v3),
            (13.0 / 12.0) * (v4 - 2.0 * v3) * (v4 - 2.0 * v3) +
                0.25 * (v4 - 4.0 * v3) * (v4 - 4.0 * v3),
            (1.0 / 240.0) * (v3 * (11003.0 * v3 - 17246.0 * v4 + 4642.0 * v5) +
                             v4 * (7043.0 * v4 - 3882.0 * v5) + 547.0 * v5 * v5)};
        const double b6 =
            (1.0 / 120960.0) *
            (v0 * (271779.0 * v0 - 2380800.0 * v1 - 3462252.0 * v3 + 1458762.0 * v4 -
                   245620.0 * v5) +
             v1 * (5653317.0 * v1 + 17905032.0 * v3 - 7727988.0 * v4 + 1325006.0 * v5) +
             v3 * (17195652.0 * v3 - 15880404.0 * v4 + 2863984.0 * v5) +
             v4 * (3824847.0 * v4 - 1429976.0 * v5) + 139633.0 * v5 * v5);
        const double tau = std::abs(b6 - (b[0] + 4.0 * b[1] + b[2]) / 6.0);
        double g[4], gsum = 0.0;
        for (int k = 0; k < 4; ++k) {
            double t = 1.0 + tau / (b[k] + 1e-40);
            const double t2 = t * t;
            g[k] = t2 * t2 * t2;
        }
        gsum = g[0] + g[1] + g[2] + g[3];
        const double Q = g[pick(rng)] / gsum;
        // ct on the exact ratio, 1 + O(1e-7 .. 1e-6) away from it, or up to
        // 1.5e-3 away — across the filter's 2e-4 band edges on both sides
        const int mode = trial % 5;
        double ct = mode == 0 ? Q
                    : mode == 4 ? Q * (1.0 + wide(rng))
                                : Q * (1.0 + (mode == 1 ? 1.0 : 10.0) * jit(rng));
        if (!(ct > 0.0 && ct < 1.0)) continue;
        const ign::ReconParams rp = ign::make_recon_params(ct, 1e-40);
        const double B[4] = {b[0] + 1e-40, b[1] + 1e-40, b[2] + 1e-40, b[3] + 1e-40};
        (ign::teno_cutoff_filter(tau, B[0], B[1], B[2], B[3], rp) < 0 ? exact : filtered) += 1;
        EXPECT_BITWISE("teno6 cutoff boundary",
                       ign::teno6_plus(w[0], w[1], w[2], w[3], w[4], w[5], rp),
                       ignis::recon::teno6_plus(w + 2, ct, 1e-40));
    }
    std::printf("teno cutoff boundary: %d decided by the filter, %d exact fallbacks\n", filtered,
                exact);
}

// TENO6's keep-all shortcut (ReconParams::keep_r): for cutoffs across the
// whole range, random smooth / kinked / flat / step stencils, bitwise
static void check_teno_keep_all() {
    std::mt19937 rng(7);
    std::uniform_real_distribution<double> u(-1.0, 1.0), lg(-15.0, 3.0);
    const double cts[] = {1e-300, 1e-12, 1e-5, 1e-3, 0.02, 0.1, 0.2, 0.6};
    for (const double ct : cts) {
        const ign::ReconParams rp = ign::make_recon_params(ct, 1e-40);
        for (int trial = 0; trial < 40000; ++trial) {
            double w[6];
            const double a = std::pow(10.0, lg(rng)), c = u(rng);
            for (int q = 0; q < 6; ++q) {
                switch (trial % 4) {
                case 0: w[q] = c + a * std::sin(0.4 * q + u(rng) * 0.01); break;  // smooth
                case 1: w[q] = c + a * std::abs(q - 2.5 + 0.3 * u(rng)); break;    // kink
                case 2: w[q] = c; break;                                          // flat
                default: w[q] = c + (q < 3 ? 0.0 : a) + 1e-3 * a * u(rng); break; // step
                }
            }
            EXPECT_BITWISE("teno6_plus keep-all", 
                           ign::teno6_plus(w[0], w[1], w[2], w[3], w[4], w[5], rp),
                           ignis::recon::teno6_plus(w + 2, ct, 1e-40));
        }
    }
}

static void check_recon() {
    const ign::ReconParams rp = ign::make_recon_params(1e-5, 1e-40);
    std::mt19937 rng(42);
    std::uniform_real_distribution<double> u(-2.0, 2.0);
    std::uniform_int_distribution<int> kind(0, 3);
    for (int trial = 0; trial < 200000; ++trial) {
        double w[6];
        const int k = kind(rng);
        for (int q = 0; q < 6; ++q) {
            w[q] = u(rng);
            if (k == 1) w[q] = q < 3 ? 1.0 : 0.125;            // step
            if (k == 2) w[q] = 3.0 + 1e-9 * u(rng);             // near-constant
            if (k == 3) w[q] = std::sin(0.3 * q + u(rng));      // smooth
        }
        EXPECT_BITWISE("teno6_plus", ign::teno6_plus(w[0], w[1], w[2], w[3], w[4], w[5], rp),
                       ignis::recon::teno6_plus(w + 2, 1e-5, 1e-40));
        EXPECT_BITWISE("weno3z_plus", ign::weno3z_plus(w[0], w[1], w[2], 1e-40),
                       ignis::recon::weno3z_plus(w + 1, 1e-40));
        double wm[6];
        for (int q = 0; q < 6; ++q) wm[q] = u(rng);
        EXPECT_BITWISE("face teno6",
                       ign::face_pm<true>(w, wm, rp),
                       ignis::recon::face_plus(ignis::InviscidScheme::TENO6, w + 2, 1e-5, 1e-40) +
                           ignis::recon::face_minus(ignis::InviscidScheme::TENO6, wm + 2, 1e-5, 1e-40));
        EXPECT_BITWISE("face weno3z",
                       ign::face_pm<false>(w, wm, rp),
                       ignis::recon::face_plus(ignis::InviscidScheme::WENO3Z, w + 1, 1e-5, 1e-40) +
                           ignis::recon::face_minus(ignis::InviscidScheme::WENO3Z, wm + 1, 1e-5, 1e-40));
    }
}

static void check_sources(const ignis::MixtureModel& mix) {
    const ign::DMix dm = ign::build_mix(to_abi(mix));
    const ignis::ReactionMechanism rm = ignis::make_one_step_mechanism(mix, 2e5, 12000.0, 1.0, 1.0, 300.0);
    ign_mechanism am{};
    am.present = 1; am.i_fuel = rm.i_fuel; am.i_ox = rm.i_ox;
    am.A = rm.A; am.Ta = rm.Ta; am.a = rm.a; am.b = rm.b; am.T_cutoff = rm.T_cutoff;
    for (int s = 0; s < 8; ++s) am.nu[s] = rm.nu[s];
    const ign::DMech dk = ign::build_mech(am);
    std::mt19937 rng(5);
    std::uniform_real_distribution<double> uy(0.0, 1.0), uT(250.0, 3500.0), ur(0.05, 4.0);
    for (int trial = 0; trial < 20000; ++trial) {
        ignis::SpeciesArray Y{}, w{};
        double Yp[4], wp[4], sum = 0.0;
        for (int s = 0; s < 4; ++s) sum += (Y[s] = uy(rng) + 1e-6);
        for (int s = 0; s < 4; ++s) Yp[s] = (Y[s] /= sum);
        const double rho = ur(rng), T = uT(rng);
        ignis::source_terms(rho, T, Y, mix, rm, w);
        ign::source_terms<4>(rho, T, Yp, dm, dk, wp);
        for (int s = 0; s < 4; ++s) EXPECT_BITWISE("source_terms", wp[s], w[s]);
    }
    // laser (laser.hpp:53-91)
    ignis::LaserParams lp;
    lp.energy = 2.5; lp.sigma_r = 0.3; lp.sigma_t = 0.4; lp.x0 = 1.0; lp.y0 = -1.0; lp.t0 = 9.6;
    ign_laser al{};
    al.present = 1; al.kernel = 0; al.energy = lp.energy; al.sigma_r = lp.sigma_r;
    al.sigma_t = lp.sigma_t; al.x0 = lp.x0; al.y0 = lp.y0; al.t0 = lp.t0;
    const ign::DLaser dl = ign::build_laser(al);
    std::uniform_real_distribution<double> ux(-1.0, 3.0), ut(8.0, 11.0);
    for (int trial = 0; trial < 20000; ++trial) {
        const double x = ux(rng), y = ux(rng) - 2.0, t = ut(rng);
        EXPECT_BITWISE("q_gaussian", ign::laser_power(x, y, t, dl), ignis::laser_power(x, y, t, lp));
    }
    // shaped two-lobe kernel (laser.hpp:64-85): the product squares with z*z
    // where the reference calls pow(z, 2) (tests/cpp/pow2_check.c)
    ignis::LaserParams sp = lp;
    sp.kernel = ignis::LaserKernel::Shaped;
    sp.edot_rate = 3.7e10;
    sp.profile.lobe_sep = 0.35; sp.profile.width_up = 0.5; sp.profile.width_down = 0.2;
    sp.profile.amp_down = 0.8; sp.profile.width_radial = 0.25;
    ign_laser as = al;
    as.kernel = 1; as.edot_rate = sp.edot_rate; as.lobe_sep = sp.profile.lobe_sep;
    as.width_up = sp.profile.width_up; as.width_down = sp.profile.width_down;
    as.amp_down = sp.profile.amp_down; as.width_radial = sp.profile.width_radial;
    const ign::DLaser ds = ign::build_laser(as);
    for (int trial = 0; trial < 200000; ++trial) {
        const double x = ux(rng), y = ux(rng) - 2.0, t = ut(rng);
        EXPECT_BITWISE("shaped_profile", ign::shaped_profile(x, y, ds),
                       ignis::shaped_profile(x, y, sp));
        EXPECT_BITWISE("q_shaped", ign::laser_power(x, y, t, ds), ignis::laser_power(x, y, t, sp));
    }
}

int main() {
    const std::string data = IGNIS_DATA_DIR;
    const ignis::MixtureModel ch4 = ignis::load_mixture_file(data + "/ch4_o2.mix");
    ignis::MixtureModel gas = ignis::MixtureModel::calorically_perfect(1.4, 1.0, 6.25e-4);
    gas.species[0].pieces[0].t_hi = 1e6;
    check_recon();
    check_teno_keep_all();
    check_teno_cutoff_boundary();
    check_mixture<4>(ch4, "ch4_o2", 1234);  // two linear-cp ranges: DSpecies::lin2 path
    // the repo's H2/O2 table (one linear range and two), and a quartic variant
    // of the CH4 table that keeps the general branch-free piece path covered
    const ignis::MixtureModel h2 = ignis::load_mixture_file(REPO_DATA_DIR "/h2_o2.mix");
    check_mixture<4>(h2, "h2_o2", 4321);
    ignis::MixtureModel quartic = ch4;
    for (auto& sp : quartic.species)
        for (auto& pc : sp.pieces) {
            pc.c2 = 1e-7;
            pc.c4 = -2e-15;
        }
    check_mixture<4>(quartic, "ch4_o2 quartic", 99);
    ignis::MixtureModel one = ch4;  // single linear range per species
    for (auto& sp : one.species) sp.pieces.resize(1), sp.pieces[0].t_hi = 6000.0;
    check_mixture<4>(one, "ch4_o2 one range", 7);
    check_mixture<1>(gas, "gamma_gas", 77);
    check_sources(ch4);
    std::printf("physics parity: %d checks, %d mismatches\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
