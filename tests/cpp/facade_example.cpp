// Example C++ caller of the drop-in facade: 2D TGV through
// ignis_b200::Simulation.  Compiled and linked by the CPU suite; run on a GPU
// box it performs one step and prints the conserved totals.
#include <cmath>
#include <cstdio>
#include <cstring>

#include "ignis_b200/simulation.hpp"

int main() {
    ign_config cfg;
    std::memset(&cfg, 0, sizeof cfg);
    cfg.abi_version = IGN_ABI_VERSION;
    cfg.nx = cfg.ny = 32;
    cfg.g = 3;
    cfg.lx = cfg.ly = 2.0 * M_PI;
    cfg.periodic_x = cfg.periodic_y = 1;
    cfg.metric_mode = -1;
    // MixtureModel::calorically_perfect(1.4, 1.0, 6.25e-4) with the t_hi cap
    cfg.mix.mode = 0;
    cfg.mix.ns = 1;
    cfg.mix.R = 1.0;
    cfg.mix.Le = 1.0;
    cfg.mix.Pr = 0.7;
    std::snprintf(cfg.mix.species[0].name, IGN_NAME_LEN, "gas");
    cfg.mix.species[0].W = 1.0;
    cfg.mix.species[0].mu_ref = 6.25e-4;
    cfg.mix.species[0].t_ref = 1.0;
    cfg.mix.species[0].npieces = 1;
    cfg.mix.species[0].pieces[0].t_hi = 1e6;
    cfg.mix.species[0].pieces[0].c0 = 1.4 / 0.4;
    cfg.scheme.scheme = 1;
    cfg.scheme.split = 1;
    cfg.scheme.teno_ct = 1e-5;
    cfg.scheme.eps = 1e-40;
    cfg.scheme.cfl = 0.5;
    cfg.viscous = 1;
    cfg.integ.max_iter = 1;
    cfg.integ.t_end = 1.0;
    cfg.integ.fixed_dt = 1e-3;
    for (ign_edge* e : {&cfg.bc.left, &cfg.bc.right, &cfg.bc.bottom, &cfg.bc.top}) e->sigma_out = 0.25;
    try {
        ignis_b200::Simulation sim(cfg);
        const double p0 = 1.0 / (1.4 * 0.01);
        sim.set_initial_condition([&](double x, double y) {
            ign_prim_point p{};
            p.rho = 1.0;
            p.u = std::sin(x) * std::cos(y);
            p.v = -std::cos(x) * std::sin(y);
            p.T = p0 + 0.25 * (std::cos(2 * x) + std::cos(2 * y));
            p.Y[0] = 1.0;
            return p;
        });
        sim.advance();
        const auto tot = sim.conserved_totals();
        std::printf("iter %ld time %g mass %.15g energy %.15g\n", sim.iter(), sim.time(), tot[0], tot[3]);
    } catch (const ignis_b200::DeviceError& e) {
        std::printf("no device: %s\n", e.what());
        return 2;
    }
    return 0;
}
