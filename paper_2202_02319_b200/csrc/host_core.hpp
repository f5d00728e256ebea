// host_core.hpp — host-side setup of the B200 path: mesh, metrics, config
// validation and the device parameter tables.  Setup runs once per context;
// its arithmetic restates the reference's (mesh.hpp, metrics.hpp,
// boundary.hpp) operation for operation so the metric arrays the kernels read
// are bit-identical to the ones the reference computes.
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

#include "ignis_b200.h"
#include "physics.cuh"

namespace ign {

// Exception types mirroring errors.hpp:10-47; mapped to ign_status at the ABI.
struct Error : std::runtime_error {
    int status;
    int stage = 0, i = 0, j = 0;
    Error(int st, const std::string& w) : std::runtime_error(w), status(st) {}
};
inline Error config_error(const std::string& w) { return Error(IGN_CONFIG_ERROR, w); }
inline Error numerics_error(const std::string& w) { return Error(IGN_NUMERICS_ERROR, w); }
inline Error usage_error(const std::string& w) { return Error(IGN_USAGE_ERROR, w); }
inline Error state_error(const std::string& w) { return Error(IGN_STATE_ERROR, w); }
inline Error step_failure(const std::string& w, int stage, int i, int j) {
    Error e(IGN_STEP_FAILURE, w);
    e.stage = stage;
    e.i = i;
    e.j = j;
    return e;
}

// Padded 2D host field (field.hpp:15-56 layout).
struct HField {
    int nx = 0, ny = 0, g = 0, sx = 0;
    std::vector<double> d;
    HField() = default;
    HField(int nx_, int ny_, int g_, double init = 0.0)
        : nx(nx_), ny(ny_), g(g_), sx(nx_ + 2 * g_),
          d(static_cast<size_t>(nx_ + 2 * g_) * (ny_ + 2 * g_), init) {}
    double& operator()(int i, int j) { return d[static_cast<size_t>(j + g) * sx + (i + g)]; }
    double operator()(int i, int j) const { return d[static_cast<size_t>(j + g) * sx + (i + g)]; }
};

// Mesh (mesh.hpp:23-54)
struct HMesh {
    int nx = 0, ny = 0, g = 3;
    double lx = 0, ly = 0, cx = 0, cy = 0;
    bool periodic_x = false, periodic_y = false;
    HField x, y;
    double dxi() const { return lx / nx; }
    double deta() const { return ly / ny; }
    double xi(int i) const { return cx - 0.5 * lx + (i + 0.5) * dxi(); }
    double eta(int j) const { return cy - 0.5 * ly + (j + 0.5) * deta(); }
};

// MetricField (metrics.hpp:28-35)
struct HMetrics {
    HField jac, m_xi_x, m_xi_y, m_eta_x, m_eta_y;
};

enum MetricMode { MM_CENTRAL2 = 0, MM_ORDER4 = 1, MM_ORDER6 = 2, MM_ANALYTIC_SKEW = 3 };

HMesh build_mesh(const ign_config& c);                       // mesh.hpp:48-117
HMetrics compute_metrics(const HMesh& m, int mode, double beta);  // metrics.hpp:73-118
int inviscid_metric_mode(const ign_config& c);               // solver.hpp:104-112
void validate_config(const ign_config& c, const HMesh& m);   // scheme/bc/laser validate
DMix build_mix(const ign_mixture& mx);
DMech build_mech(const ign_mechanism& mk);
DLaser build_laser(const ign_laser& l);

}  // namespace ign
