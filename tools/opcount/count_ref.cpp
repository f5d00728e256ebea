// count_ref.cpp — TOOL: algorithmic FP64 op counts of the reference's OWN code
// (SURVEY §8d method).  The unmodified reference headers are compiled with
// `double` redefined to the counting type of counted.hpp; each case is set up
// as paper_2202_02319_b200/configs.py sets it up and every public hot-path
// call is counted separately, per interior cell.  Prints one JSON object.
//   g++ -std=c++20 -O1 -I/root/reference/proj/include count_ref.cpp -o count_ref
#include "counted.hpp"
#define double CD
#define private public  // counting only: reach inviscid_direction / compute_viscous
#include "ignis/solver.hpp"
#undef private
#undef double

using namespace ignis;

static opc::Counts measure(const std::function<void()>& f) {
    opc::counts() = opc::Counts{};
    opc::enabled() = true;
    f();
    opc::enabled() = false;
    return opc::counts();
}

static void emit(const char* name, const opc::Counts& c, double cells, bool last = false) {
    std::printf("    \"%s\": {\"ops\": %.1f, \"add\": %.1f, \"mul\": %.1f, \"div\": %.1f, "
                "\"sqrt\": %.2f, \"log\": %.2f, \"exp\": %.2f, \"pow\": %.2f, \"hypot\": %.2f, "
                "\"cmp\": %.1f}%s\n",
                name, c.ops() / cells, c.add / cells, c.mul / cells, c.div / cells,
                c.sqrt / cells, c.log / cells, c.exp / cells, c.pow / cells, c.hypot / cells,
                c.cmp / cells, last ? "" : ",");
}

struct Setup {
    std::string name;
    std::function<void(Simulation&)> make;
    int n;
};

static void tgv(Simulation& sim, int n, InviscidScheme sch, FluxSplit sp, bool visc) {
    const double L = 2.0 * M_PI;
    MixtureModel mix = MixtureModel::calorically_perfect(1.4, 1.0, visc ? 6.25e-4 : 0.0);
    mix.species[0].pieces[0].t_hi = 1e6;  // SURVEY §8c harness fix
    SchemeConfig sc;
    sc.scheme = sch;
    sc.split = sp;
    BoundarySpec bs;
    sim.init(build_uniform(n, n, L, L), Simulation::metric_mode_for(sc), 0.0, mix, sc, bs);
    sim.viscous = visc;
    const double p0 = 1.0 / (1.4 * 0.01);
    sim.set_initial_condition([&](CD x, CD y) {
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

// configs.h2o2_counterflow (BASELINE configs[2]) at n x n
static void h2o2(Simulation& sim, int n, InviscidScheme sch, FluxSplit sp) {
    const double L = 0.02;
    MixtureModel mix = load_mixture_file(REPO_DATA_DIR "/h2_o2.mix");
    SchemeConfig sc;
    sc.scheme = sch;
    sc.split = sp;
    BoundarySpec bs;
    const double Yf[4] = {0.1, 0.0, 0.0, 0.9}, Yo[4] = {0.0, 0.23, 0.0, 0.77};
    for (int e = 0; e < 2; ++e) {
        EdgeSpec& es = e == 0 ? bs.left : bs.right;
        es.type = BCType::Inflow;
        InflowSegment s;
        s.lo = -0.5 * L;
        s.hi = 0.5 * L;
        s.u = e == 0 ? 1.0 : -1.0;
        s.T = 300.0;
        for (int k = 0; k < 4; ++k) s.Y[k] = e == 0 ? Yf[k] : Yo[k];
        es.segments = {s};
    }
    bs.bottom.type = bs.top.type = BCType::Outflow;
    sim.init(build_uniform(n, n, L, L, {0.0, 0.0}, false, false), Simulation::metric_mode_for(sc),
             0.0, mix, sc, bs);
    sim.viscous = true;
    ReactionMechanism m;
    m.A = 1e9;
    m.Ta = 15000.0;
    m.a = m.b = 1.0;
    m.T_cutoff = 300.0;
    m.i_fuel = 0;
    m.i_ox = 1;
    m.i_co2 = -1;
    m.i_h2o = 2;
    const double nu[4] = {-2.0, -1.0, 2.0, 0.0};
    for (int s = 0; s < 4; ++s) m.nu[s] = nu[s];
    sim.mech = m;
    LaserParams lp;
    lp.energy = 5.0;
    lp.sigma_r = 5e-4;
    lp.sigma_t = 1e-6;
    lp.t0 = 3e-6;
    sim.laser = lp;
    const double W[4] = {0.002, 0.032, 0.018, 0.028};
    sim.set_initial_condition([&](CD x, CD) {
        const CD w = 0.5 * (1.0 - std::tanh(x / 1e-3));
        PrimPoint q;
        CD rbar = 0.0;
        for (int k = 0; k < 4; ++k) {
            q.Y[k] = Yf[k] * w + Yo[k] * (1.0 - w);
            rbar = rbar + q.Y[k] / W[k];
        }
        q.T = 300.0;
        q.rho = 101325.0 / (8.31446261815324 * rbar * q.T);
        q.u = -std::tanh(x / 4e-3);
        q.v = 0.0;
        return q;
    });
}

int main(int argc, char** argv) {
    // grid sizes: 2D TGV (the 3D workload's 2D analogue) and H2/O2 at the
    // bench size of BASELINE configs[2]
    const int nt = argc > 1 ? std::atoi(argv[1]) : 256;
    const int nh = argc > 2 ? std::atoi(argv[2]) : 512;
    std::vector<Setup> cases = {
        {"tgv2d_char_teno6_visc", [&](Simulation& s) { tgv(s, nt, InviscidScheme::TENO6, FluxSplit::Characteristic, true); }, nt},
        {"tgv2d_comp_teno6_visc", [&](Simulation& s) { tgv(s, nt, InviscidScheme::TENO6, FluxSplit::Componentwise, true); }, nt},
        {"tgv2d_comp_weno3z_visc", [&](Simulation& s) { tgv(s, nt, InviscidScheme::WENO3Z, FluxSplit::Componentwise, true); }, nt},
        {"h2o2_char_teno6", [&](Simulation& s) { h2o2(s, nh, InviscidScheme::TENO6, FluxSplit::Characteristic); }, nh},
        {"h2o2_comp_weno3z", [&](Simulation& s) { h2o2(s, nh, InviscidScheme::WENO3Z, FluxSplit::Componentwise); }, nh},
    };
    std::printf("{\n");
    for (size_t k = 0; k < cases.size(); ++k) {
        const Setup& c = cases[k];
        const double cells = double(c.n) * c.n;
        Simulation sim;
        c.make(sim);
        sim.prepare_stage(1);
        FieldSet rhs(sim.comp().ncomp(), sim.mesh.nx, sim.mesh.ny, sim.mesh.g);
        const bool visc = sim.viscous;
        auto mech = sim.mech;
        auto laser = sim.laser;
        const opc::Counts prep = measure([&] { sim.prepare_stage(1); });
        const opc::Counts full = measure([&] { sim.compute_rhs(rhs, 0.0, 1); });
        // inviscid part: the same RHS with the viscous and source terms off
        sim.viscous = false;
        sim.mech.reset();
        sim.laser.reset();
        const opc::Counts inv = measure([&] { sim.compute_rhs(rhs, 0.0, 1); });
        sim.viscous = visc;
        sim.mech = mech;
        sim.laser = laser;
        const opc::Counts fx = measure([&] { sim.inviscid_direction(true); });
        const opc::Counts fy = measure([&] { sim.inviscid_direction(false); });
        opc::Counts faces = fx;
        faces.add += fy.add; faces.mul += fy.mul; faces.div += fy.div; faces.sqrt += fy.sqrt;
        faces.log += fy.log; faces.exp += fy.exp; faces.pow += fy.pow; faces.hypot += fy.hypot;
        faces.cmp += fy.cmp;
        opc::Counts vis{};
        if (visc) vis = measure([&] { sim.compute_viscous(); });
        const opc::Counts dt = measure([&] { (void)sim.stable_dt(); });
        const CD dtv = sim.stable_dt();
        const opc::Counts step = measure([&] {
            sim.rk3_step(0.5 * dtv);
            sim.prepare_stage(1);
        });
        std::printf("  \"%s\": {\n    \"grid\": \"%dx%d\",\n", c.name.c_str(), c.n, c.n);
        emit("prepare_stage_per_cell", prep, cells);
        emit("compute_rhs_per_cell_stage", full, cells);
        emit("inviscid_rhs_per_cell_stage", inv, cells);
        emit("inviscid_faces_x_per_cell_stage", fx, cells);
        emit("inviscid_faces_y_per_cell_stage", fy, cells);
        emit("inviscid_faces_per_cell_stage", faces, cells);
        emit("viscous_per_cell_stage", vis, cells);
        emit("stable_dt_per_cell", dt, cells);
        emit("rk3_step_plus_prepare_per_cell_step", step, cells, true);
        std::printf("  }%s\n", k + 1 < cases.size() ? "," : "");
    }
    std::printf("}\n");
    return 0;
}
