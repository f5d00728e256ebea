// host_core.hpp — host-side setup of the B200 path: mesh, metrics, config
// validation and the device parameter tables.  Setup runs once per context;
// its arithmetic restates the reference's (mesh.hpp, metrics.hpp,
// boundary.hpp) operation for operation so the metric arrays the kernels read
// are bit-identical to the ones the reference computes.
#pragma once

#include <stdexcept>
#include <string>
#include <memory>
#include <vector>

#include "ignis_b200.h"
#include "physics.cuh"

namespace ign {

// Exception types mirroring errors.hpp:10-47; mapped to ign_status at the ABI.
struct Error : std::runtime_error {
    int status;
    int stage = 0, i = 0, j = 0, k = 0;  // k: z plane of a 3D failure
    Error(int st, const std::string& w) : std::runtime_error(w), status(st) {}
};
inline Error config_error(const std::string& w) { return Error(IGN_CONFIG_ERROR, w); }
inline Error numerics_error(const std::string& w) { return Error(IGN_NUMERICS_ERROR, w); }
inline Error usage_error(const std::string& w) { return Error(IGN_USAGE_ERROR, w); }
inline Error state_error(const std::string& w) { return Error(IGN_STATE_ERROR, w); }
inline Error step_failure(const std::string& w, int stage, int i, int j, int k = 0) {
    Error e(IGN_STEP_FAILURE, w);
    e.stage = stage;
    e.i = i;
    e.j = j;
    e.k = k;
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

// Mesh (mesh.hpp:23-54) as seen by one slab: the global mesh is
// nx x ny_glob; this object holds the padded local rows ny (global rows
// j0 .. j0+ny-1 plus g ghost rows each side).  Without slabs j0 = 0 and
// ny = ny_glob, and every coordinate is the reference's expression.
struct HMesh {
    int nx = 0, ny = 0, g = 3;
    int ny_glob = 0, j0 = 0;
    double lx = 0, ly = 0, cx = 0, cy = 0;
    bool periodic_x = false, periodic_y = false;
    bool skew = false;
    double beta = 0.0;
    HField x, y;  // local padded box
    // a hand-built mesh (ign_config.mesh_x/mesh_y): the GLOBAL padded
    // coordinate arrays, which coords() then reads instead of the formulas
    std::shared_ptr<const std::vector<double>> gx, gy;
    double dxi() const { return lx / nx; }
    double deta() const { return ly / ny_glob; }
    double xi(int i) const { return cx - 0.5 * lx + (i + 0.5) * dxi(); }
    // computational coordinate of GLOBAL row jg (mesh.hpp:41-42)
    double eta_glob(int jg) const { return cy - 0.5 * ly + (jg + 0.5) * deta(); }
    // of LOCAL row j
    double eta(int j) const { return eta_glob(j0 + j); }
    // physical coordinates of global node (i, jg): build_uniform + apply_skew
    // (mesh.hpp:48-77, 92-117)
    void coords(int i, int jg, double& X, double& Y) const;
};

// MetricField (metrics.hpp:28-35)
struct HMetrics {
    HField jac, m_xi_x, m_xi_y, m_eta_x, m_eta_y;
};

enum MetricMode { MM_CENTRAL2 = 0, MM_ORDER4 = 1, MM_ORDER6 = 2, MM_ANALYTIC_SKEW = 3 };

// Rows of the slab decomposition: rank r of n owns global rows
// [lo, lo+count) with the ThreadTeam block split (thread_team.hpp:63-69).
void slab_rows(int ny_glob, int nranks, int rank, int& lo, int& count);

// mesh.hpp:48-117 for the rows of one slab (nranks = 1: the whole mesh)
HMesh build_mesh(const ign_config& c, int nranks = 1, int rank = 0);
// metrics.hpp:73-118 over the slab's padded rows, evaluated with the GLOBAL
// stencils and rim fallbacks, so each slab holds exact slices of the global
// metric arrays.
HMetrics compute_metrics(const HMesh& m, int mode, double beta);
// the same for arbitrary global rows [jlo, jhi): out[5] = jac, m_xi_x, m_xi_y,
// m_eta_x, m_eta_y, each (nx+2g) x (jhi-jlo) row-major
void metric_rows(const HMesh& m, int mode, double beta, int jlo, int jhi, double* const* out);
std::vector<double> jac_rows(const HMesh& m, int mode, double beta, int jlo, int jhi);
int inviscid_metric_mode(const ign_config& c);               // solver.hpp:104-112
void validate_config(const ign_config& c, const HMesh& m);   // scheme/bc/laser validate
DMix build_mix(const ign_mixture& mx);
DMech build_mech(const ign_mechanism& mk);
DLaser build_laser(const ign_laser& l);

}  // namespace ign
