// count_3d.cpp — TOOL: algorithmic FP64 op count of the 3D inviscid faces,
// counted on oracle/ref3d_faces.hpp (the reference's per-face algorithm with
// the z terms, calling the reference's own recon/thermo functions) compiled
// with the counting double — independent of the product's kernels
// (the r1 3D count was the 2D count x the product's own FP64
// instruction ratio).  Workload: the bench's TGV 3D (gamma-gas, Ma 0.1) at
// n^3, TENO6/WENO3Z x char/comp.  Prints one JSON object.
#include "counted.hpp"
#define double CD
#define private public
#include "ignis/solver.hpp"
#include "../../oracle/ref3d_faces.hpp"
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

int main(int argc, char** argv) {
    const int n = argc > 1 ? std::atoi(argv[1]) : 32;
    const int g = 3;
    const CD L = 2.0 * M_PI;
    MixtureModel mix = MixtureModel::calorically_perfect(1.4, 1.0, 0.0);
    mix.species[0].pieces[0].t_hi = 1e6;
    const Mesh mesh = build_uniform(n, n, L, L);
    const CD gamma = 1.4, p0 = 1.0 / (1.4 * 0.01);
    ref3d::Grid G{n, n, n, g, 1, 0, 0, 0};
    G.sx = n + 2 * g;
    G.sxy = G.sx * (n + 2 * g);
    G.plane = G.sxy * (n + 2 * g);
    const int nc = 5;
    std::vector<CD> Ut(size_t(nc) * G.plane), prim(size_t(8) * G.plane), rhs(size_t(nc) * G.plane);
    struct Case { const char* name; InviscidScheme s; FluxSplit f; };
    const Case cases[] = {{"tgv3d_char_teno6", InviscidScheme::TENO6, FluxSplit::Characteristic},
                          {"tgv3d_comp_teno6", InviscidScheme::TENO6, FluxSplit::Componentwise},
                          {"tgv3d_char_weno3z", InviscidScheme::WENO3Z, FluxSplit::Characteristic},
                          {"tgv3d_comp_weno3z", InviscidScheme::WENO3Z, FluxSplit::Componentwise}};
    std::printf("{\n  \"grid\": \"%d^3\",\n", n);
    for (size_t q = 0; q < 4; ++q) {
        SchemeConfig sc;
        sc.scheme = cases[q].s;
        sc.split = cases[q].f;
        const MetricField met = compute_metrics(mesh, Simulation::metric_mode_for(sc));
        const ref3d::Met3 M = ref3d::extrude(met, L / n);
        // the analytic TGV 3D state (configs.tgv3d) and its primitive cache
        for (int k = -g; k < n + g; ++k)
            for (int j = -g; j < n + g; ++j)
                for (int i = -g; i < n + g; ++i) {
                    const CD x = mesh.x(i, j), y = mesh.y(i, j);
                    const CD z = -0.5 * L + (k + 0.5) * (L / n);
                    const CD u = std::sin(x) * std::cos(y) * std::cos(z);
                    const CD v = -std::cos(x) * std::sin(y) * std::cos(z);
                    const CD w = 0.0;
                    const CD p = p0 + (1.0 / 16.0) * (std::cos(2.0 * x) + std::cos(2.0 * y)) *
                                          (std::cos(2.0 * z) + 2.0);
                    const long id = G.at(i, j, k);
                    const CD rho = 1.0, T = p / rho;
                    const CD J = M.jac[G.at2(i, j)];
                    const CD e = p / (rho * (gamma - 1.0));
                    const CD U[5] = {rho, rho * u, rho * v, rho * w,
                                     rho * (e + 0.5 * ((u * u + v * v) + w * w))};
                    for (int cc = 0; cc < 5; ++cc) Ut[size_t(cc) * G.plane + id] = U[cc] / J;
                    const CD pr[8] = {rho, u, v, w, p, T, std::sqrt(gamma * T), 1.0};
                    for (int f = 0; f < 8; ++f) prim[size_t(f) * G.plane + id] = pr[f];
                }
        const opc::Counts c = measure([&] {
            ref3d::inviscid_rhs(G, M, mix, sc, Ut.data(), prim.data(), rhs.data());
        });
        const double cells = double(n) * n * n;
        std::printf("  \"%s\": {\"inviscid_faces_per_cell_stage\": {\"ops\": %.1f, \"add\": %.1f, "
                    "\"mul\": %.1f, \"div\": %.1f, \"sqrt\": %.2f, \"log\": %.2f, \"hypot\": %.2f, "
                    "\"cmp\": %.1f}}%s\n",
                    cases[q].name, c.ops() / cells, c.add / cells, c.mul / cells, c.div / cells,
                    c.sqrt / cells, c.log / cells, c.hypot / cells, c.cmp / cells,
                    q + 1 < 4 ? "," : "");
    }
    std::printf("}\n");
    return 0;
}
