// host_core.cpp — see host_core.hpp.  Compiled with g++ -O2 -ffp-contract=off
// (the reference's flags) so setup arithmetic is bit-identical to the oracle.
#include "host_core.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>

namespace ign {

namespace {

// skew_jacobian (mesh.hpp:81-87)
void skew_jacobian(double xc, double yc, double beta, double L, double d[4]) {
    const double k = 2.0 * M_PI / L;
    d[0] = 1.0 + beta * std::sin(k * yc);
    d[1] = xc * beta * k * std::cos(k * yc);
    d[2] = yc * beta * k * std::cos(k * xc);
    d[3] = 1.0 + beta * std::sin(k * xc);
}

// Coordinates of the global padded rows [wlo, whi) of the mesh (all columns).
struct CoordWindow {
    int nx, g, wlo, whi;
    std::vector<double> x, y;
    double X(int i, int jg) const { return x[size_t(jg - wlo) * (nx + 2 * g) + (i + g)]; }
    double Y(int i, int jg) const { return y[size_t(jg - wlo) * (nx + 2 * g) + (i + g)]; }
};

CoordWindow coord_window(const HMesh& m, int wlo, int whi) {
    CoordWindow w{m.nx, m.g, wlo, whi, {}, {}};
    const size_t n = size_t(m.nx + 2 * m.g) * (whi - wlo);
    w.x.resize(n);
    w.y.resize(n);
    for (int jg = wlo; jg < whi; ++jg)
        for (int i = -m.g; i < m.nx + m.g; ++i) {
            const size_t k = size_t(jg - wlo) * (m.nx + 2 * m.g) + (i + m.g);
            m.coords(i, jg, w.x[k], w.y[k]);
        }
    return w;
}

// detail::index_deriv (metrics.hpp:45-67) on a coordinate window; n and g are
// the GLOBAL extents so rim fallbacks match the single-domain mesh.
template <class F>
double index_deriv(const F& f, int nx, int ny_glob, int g, int i, int j, bool xdir, int pref) {
    const int n = xdir ? nx : ny_glob;
    const int c = xdir ? i : j;
    auto at = [&](int off) { return xdir ? f(i + off, j) : f(i, j + off); };
    int w = pref;
    if (c - w < -g || c + w >= n + g) w = 2;
    if (c - w < -g || c + w >= n + g) w = 1;
    if (c - w < -g || c + w >= n + g) {
        if (c + 2 < n + g) return 0.5 * (-3.0 * at(0) + 4.0 * at(1) - at(2));
        return 0.5 * (3.0 * at(0) - 4.0 * at(-1) + at(-2));
    }
    switch (w) {
    case 3:
        return (-at(-3) + 9.0 * at(-2) - 45.0 * at(-1) + 45.0 * at(1) - 9.0 * at(2) + at(3)) /
               60.0;
    case 2: return (at(-2) - 8.0 * at(-1) + 8.0 * at(1) - at(2)) / 12.0;
    default: return 0.5 * (at(1) - at(-1));
    }
}

}  // namespace

void slab_rows(int ny_glob, int nranks, int rank, int& lo, int& count) {
    const int base = ny_glob / nranks, rem = ny_glob % nranks;
    lo = rank * base + (rank < rem ? rank : rem);
    count = base + (rank < rem ? 1 : 0);
}

void HMesh::coords(int i, int jg, double& X, double& Y) const {
    if (gx) {  // the caller's Mesh (mesh.hpp:33-34)
        const size_t k = size_t(jg + g) * (nx + 2 * g) + (i + g);
        X = (*gx)[k];
        Y = (*gy)[k];
        return;
    }
    const double xc = xi(i), yc = eta_glob(jg);  // build_uniform (mesh.hpp:70-75)
    if (!skew) {
        X = xc;
        Y = yc;
        return;
    }
    const double L = lx;  // apply_skew (mesh.hpp:108-115)
    X = xc * (1.0 + beta * std::sin(2.0 * M_PI * yc / L));
    Y = yc * (1.0 + beta * std::sin(2.0 * M_PI * xc / L));
}

HMesh build_mesh(const ign_config& c, int nranks, int rank) {
    // build_uniform (mesh.hpp:48-77)
    if (c.lx <= 0.0 || c.ly <= 0.0)
        throw config_error("build_uniform: domain extents must be positive");
    if (c.g < 1) throw config_error("build_uniform: ghost width must be >= 1");
    if (c.nx < 2 * c.g + 1 || c.ny < 2 * c.g + 1)
        throw config_error("build_uniform: node counts must be >= 2g+1, got " +
                           std::to_string(c.nx) + "x" + std::to_string(c.ny));
    HMesh m;
    m.nx = c.nx;
    m.ny_glob = c.ny;
    slab_rows(c.ny, nranks, rank, m.j0, m.ny);
    if (m.ny < c.g)
        throw config_error("slab decomposition: each slab needs at least g rows");
    m.g = c.g;
    m.lx = c.lx;
    m.ly = c.ly;
    m.cx = c.center_x;
    m.cy = c.center_y;
    m.periodic_x = c.periodic_x != 0;
    m.periodic_y = c.periodic_y != 0;
    m.skew = c.apply_skew != 0;
    m.beta = c.skew_beta;
    if (c.mesh_x && c.mesh_y) {  // hand-built Mesh: its coordinates, no apply_skew
        const size_t n = size_t(m.nx + 2 * m.g) * (m.ny_glob + 2 * m.g);
        m.gx = std::make_shared<const std::vector<double>>(c.mesh_x, c.mesh_x + n);
        m.gy = std::make_shared<const std::vector<double>>(c.mesh_y, c.mesh_y + n);
        m.skew = false;
    }
    if (m.skew) {
        // apply_skew (mesh.hpp:92-105) validation, over this slab's interior rows
        if (std::abs(m.lx - m.ly) > 1e-14 * m.lx || m.cx != 0.0 || m.cy != 0.0)
            throw config_error("apply_skew: mesh must be square and origin-centered");
        const double L = m.lx;
        for (int j = m.j0; j < m.j0 + m.ny; ++j)
            for (int i = 0; i < m.nx; ++i) {
                double d[4];
                skew_jacobian(m.xi(i), m.eta_glob(j), m.beta, L, d);
                if (d[0] * d[3] - d[1] * d[2] <= 0.0)
                    throw numerics_error("apply_skew: grid folding (J <= 0) at node (" +
                                         std::to_string(i) + "," + std::to_string(j) +
                                         ") for beta=" + std::to_string(m.beta));
            }
    }
    m.x = HField(m.nx, m.ny, m.g);
    m.y = HField(m.nx, m.ny, m.g);
    for (int j = -m.g; j < m.ny + m.g; ++j)
        for (int i = -m.g; i < m.nx + m.g; ++i) m.coords(i, m.j0 + j, m.x(i, j), m.y(i, j));
    return m;
}

HMetrics compute_metrics(const HMesh& mesh, int mode, double beta) {
    HMetrics mf;
    const int g = mesh.g;
    mf.jac = HField(mesh.nx, mesh.ny, g);
    mf.m_xi_x = HField(mesh.nx, mesh.ny, g);
    mf.m_xi_y = HField(mesh.nx, mesh.ny, g);
    mf.m_eta_x = HField(mesh.nx, mesh.ny, g);
    mf.m_eta_y = HField(mesh.nx, mesh.ny, g);
    double* out[5] = {mf.jac.d.data(), mf.m_xi_x.d.data(), mf.m_xi_y.d.data(),
                      mf.m_eta_x.d.data(), mf.m_eta_y.d.data()};
    metric_rows(mesh, mode, beta, mesh.j0 - g, mesh.j0 + mesh.ny + g, out);
    return mf;
}

std::vector<double> jac_rows(const HMesh& mesh, int mode, double beta, int jlo, int jhi) {
    const size_t n = size_t(mesh.nx + 2 * mesh.g) * (jhi - jlo);
    std::vector<double> buf(5 * n);
    double* out[5] = {buf.data(), buf.data() + n, buf.data() + 2 * n, buf.data() + 3 * n,
                      buf.data() + 4 * n};
    metric_rows(mesh, mode, beta, jlo, jhi, out);
    buf.resize(n);
    return buf;
}

void metric_rows(const HMesh& mesh, int mode, double beta, int jlo, int jhi, double* const* out) {
    const int g = mesh.g;
    const int sx = mesh.nx + 2 * g;
    const int pref = (mode == MM_ORDER6) ? 3 : (mode == MM_ORDER4) ? 2 : 1;
    // coordinates of the rows plus the 3-row stencil reach, clipped to the
    // global padded box
    const int wlo = std::max(jlo - g, -g);
    const int whi = std::min(jhi + g, mesh.ny_glob + g);
    const CoordWindow w =
        mode == MM_ANALYTIC_SKEW ? CoordWindow{mesh.nx, g, 0, 0, {}, {}}
                                 : coord_window(mesh, wlo, whi);
    auto fx = [&](int i, int j) { return w.X(i, j); };
    auto fy = [&](int i, int j) { return w.Y(i, j); };
    for (int j = jlo; j < jhi; ++j) {  // global row
        const size_t row = size_t(j - jlo) * sx;
        for (int i = -g; i < mesh.nx + g; ++i) {
            double x_xi, x_eta, y_xi, y_eta;
            if (mode == MM_ANALYTIC_SKEW) {
                double d[4];
                skew_jacobian(mesh.xi(i), mesh.eta_glob(j), beta, mesh.lx, d);
                x_xi = d[0] * mesh.dxi();
                x_eta = d[1] * mesh.deta();
                y_xi = d[2] * mesh.dxi();
                y_eta = d[3] * mesh.deta();
            } else {
                x_xi = index_deriv(fx, mesh.nx, mesh.ny_glob, g, i, j, true, pref);
                x_eta = index_deriv(fx, mesh.nx, mesh.ny_glob, g, i, j, false, pref);
                y_xi = index_deriv(fy, mesh.nx, mesh.ny_glob, g, i, j, true, pref);
                y_eta = index_deriv(fy, mesh.nx, mesh.ny_glob, g, i, j, false, pref);
            }
            const double area = x_xi * y_eta - x_eta * y_xi;
            if (!(area > 0.0) && i >= 0 && i < mesh.nx && j >= 0 && j < mesh.ny_glob)
                throw numerics_error("grid folding: J <= 0 at node (" + std::to_string(i) +
                                     "," + std::to_string(j) + ")");
            const size_t k = row + (i + g);
            out[0][k] = 1.0 / area;
            out[1][k] = y_eta;
            out[2][k] = -x_eta;
            out[3][k] = -y_xi;
            out[4][k] = x_xi;
        }
    }
}

int inviscid_metric_mode(const ign_config& c) {
    if (c.metric_mode >= 0) return c.metric_mode;
    switch (c.scheme.metrics) {
    case 1: return MM_ANALYTIC_SKEW;
    case 2: return MM_CENTRAL2;
    default: return c.scheme.scheme == 1 ? MM_ORDER6 : MM_ORDER4;
    }
}

void validate_config(const ign_config& c, const HMesh& mesh) {
    if (c.mix.ns < 1 || c.mix.ns > kMaxSpecies) throw usage_error("mixture: ns must be 1..8");
    for (int s = 0; s < c.mix.ns; ++s)
        if (c.mix.species[s].npieces < 1 || c.mix.species[s].npieces > kMaxPieces)
            throw usage_error("mixture: species needs 1..4 polynomial pieces");
    // SchemeConfig::validate (reconstruction.hpp:28-34)
    const ign_scheme& sc = c.scheme;
    if (!(sc.eps > 0.0)) throw config_error("scheme: eps must be positive");
    if (!(sc.teno_ct > 0.0 && sc.teno_ct < 1.0))
        throw config_error("scheme: teno_ct must lie in (0,1)");
    if (!(sc.cfl > 0.0 && sc.cfl <= 1.0)) throw config_error("scheme: cfl must lie in (0,1]");
    // BoundarySpec::validate (boundary.hpp:57-88)
    const bool px = c.bc.left.type == 0;
    if (px != (c.bc.right.type == 0) || px != mesh.periodic_x)
        throw config_error("boundary: periodic x edges must be paired and match the mesh");
    const bool py = c.bc.bottom.type == 0;
    if (py != (c.bc.top.type == 0) || py != mesh.periodic_y)
        throw config_error("boundary: periodic y edges must be paired and match the mesh");
    if (c.nz > 0) {
        // 3D extension: z edges are periodic (paired) or walls / outflow
        const bool pz = c.periodic_z != 0;
        if (pz && (c.zlo.type != 0 || c.zhi.type != 0))
            throw config_error("boundary: periodic z needs periodic zlo / zhi edges");
        for (const ign_edge* e : {&c.zlo, &c.zhi}) {
            if (pz) continue;
            if (e->type == 0)
                throw config_error("boundary: periodic z edges must be paired and match periodic_z");
            if (e->type == 3) throw usage_error("boundary: inflow is not supported on z edges");
            if (e->type < 0 || e->type > 4) throw usage_error("boundary: unknown BC type");
        }
    }
    auto check_inflow = [&](const ign_edge& s, bool xedge) {
        if (s.type != 3) return;
        if (s.nseg <= 0) throw config_error("boundary: inflow edge needs segments");
        if (s.nseg > kMaxSeg) throw usage_error("boundary: at most 4 inflow segments");
        const double lo = xedge ? mesh.cy - 0.5 * mesh.ly : mesh.cx - 0.5 * mesh.lx;
        const double hi = xedge ? mesh.cy + 0.5 * mesh.ly : mesh.cx + 0.5 * mesh.lx;
        for (int k = 0; k < s.nseg; ++k) {
            const ign_inflow_segment& seg = s.seg[k];
            if (seg.lo >= seg.hi || seg.lo < lo - 1e-12 * (hi - lo) ||
                seg.hi > hi + 1e-12 * (hi - lo))
                throw config_error("boundary: inflow segment [" + std::to_string(seg.lo) +
                                   "," + std::to_string(seg.hi) + "] outside edge extent [" +
                                   std::to_string(lo) + "," + std::to_string(hi) + "]");
        }
    };
    check_inflow(c.bc.left, true);
    check_inflow(c.bc.right, true);
    check_inflow(c.bc.bottom, false);
    check_inflow(c.bc.top, false);
    for (const ign_edge* e : {&c.bc.left, &c.bc.right, &c.bc.bottom, &c.bc.top})
        if (e->type < 0 || e->type > 4) throw usage_error("boundary: unknown BC type");
    if (c.mech.present) {
        const ign_mechanism& k = c.mech;
        if (k.i_fuel < 0 || k.i_fuel >= c.mix.ns || k.i_ox < 0 || k.i_ox >= c.mix.ns)
            throw usage_error("mechanism: fuel/oxidizer index out of range");
    }
}

DMix build_mix(const ign_mixture& mx) {
    DMix m;
    std::memset(&m, 0, sizeof(m));
    m.ns = mx.ns;
    m.R = mx.R;
    m.Le = mx.Le;
    m.Pr = mx.Pr;
    // temperature_from_energy bracket (thermo.hpp:187-192)
    double t_lo = 1e300, t_hi = 0.0;
    for (int s = 0; s < mx.ns; ++s) {
        const ign_species& a = mx.species[s];
        t_lo = std::min(t_lo, a.pieces[0].t_lo);
        t_hi = std::max(t_hi, a.pieces[a.npieces - 1].t_hi);
    }
    m.t_lo = std::max(t_lo, 1e-12);
    m.t_hi = t_hi;
    for (int s = 0; s < mx.ns; ++s) {
        const ign_species& a = mx.species[s];
        DSpecies& d = m.sp[s];
        d.W = a.W;
        d.mu_ref = a.mu_ref;
        d.t_ref = a.t_ref;
        d.n_exp = a.n_exp;
        d.npieces = a.npieces;
        d.unit_W = a.W == 1.0;
        d.yW = 1.0 / a.W;
        for (int k = 0; k < a.npieces; ++k) {
            const ign_thermo_piece& q = a.pieces[k];
            DPiece& p = d.pc[k];
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
            p.h1 = q.c1 / 2;
            p.h2 = q.c2 / 3;
            p.h3 = q.c3 / 4;
            p.cp_deg = q.c4 != 0.0 ? 4 : q.c3 != 0.0 ? 3 : q.c2 != 0.0 ? 2 : q.c1 != 0.0 ? 1 : 0;
            p.inv_terms = (q.cm2 != 0.0 || q.cm1 != 0.0) ? 1 : 0;
        }
        d.simple = (a.npieces == 1 && d.pc[0].cp_deg == 0 && d.pc[0].inv_terms == 0 &&
                    !std::signbit(d.pc[0].c0))
                       ? 1
                       : 0;
        d.lin2 = a.npieces >= 1 && a.npieces <= 2;
        for (int k = 0; k < a.npieces; ++k) {
            const DPiece& p = d.pc[k];
            if (p.inv_terms || p.cp_deg > 1 || (p.cp_deg == 0 && std::signbit(p.c0))) d.lin2 = 0;
        }
        if (d.lin2 && a.npieces == 1) d.pc[1] = d.pc[0];
    }
    m.all_simple = 1;
    m.all_lin2 = 1;
    m.w_pos_ok = 1;
    for (int s = 0; s < mx.ns; ++s) {
        m.all_simple &= m.sp[s].simple;
        m.all_lin2 &= m.sp[s].lin2;
        m.w_pos_ok &= (m.sp[s].unit_W || fdiv_pos_divisor_ok(m.sp[s].W)) ? 1 : 0;
    }
    if (m.all_simple) m.all_lin2 = 0;
    // W-only factors of Wilke's rule (thermo.hpp:249-251), same glibc calls
    for (int i = 0; i < mx.ns; ++i)
        for (int j = 0; j < mx.ns; ++j) {
            const double wi = mx.species[i].W, wj = mx.species[j].W;
            m.wilke_pw[i][j] = std::pow(wj / wi, 0.25);
            m.wilke_sq[i][j] = std::sqrt(8.0 * (1.0 + wi / wj));
        }
    return m;
}

DMech build_mech(const ign_mechanism& k) {
    DMech d;
    std::memset(&d, 0, sizeof(d));
    d.present = k.present;
    d.i_fuel = k.i_fuel;
    d.i_ox = k.i_ox;
    d.A = k.A;
    d.Ta = k.Ta;
    d.a = k.a;
    d.b = k.b;
    d.T_cutoff = k.T_cutoff;
    for (int s = 0; s < kMaxSpecies; ++s) d.nu[s] = k.nu[s];
    return d;
}

DLaser build_laser(const ign_laser& l) {
    DLaser d;
    std::memset(&d, 0, sizeof(d));
    d.on = (l.present && l.energy != 0.0) ? 1 : 0;
    d.kernel = l.kernel;
    d.energy = l.energy;
    d.sigma_r = l.sigma_r;
    d.sigma_t = l.sigma_t;
    d.x0 = l.x0;
    d.y0 = l.y0;
    d.t0 = l.t0;
    d.edot_rate = l.edot_rate;
    d.lobe_sep = l.lobe_sep;
    d.width_up = l.width_up;
    d.width_down = l.width_down;
    d.amp_down = l.amp_down;
    d.width_radial = l.width_radial;
    d.pow2pi15 = std::pow(2.0 * M_PI, 1.5);
    d.zmode = l.zmode;
    d.z0 = l.z0;
    d.pow2pi2 = (2.0 * M_PI) * (2.0 * M_PI);
    return d;
}

}  // namespace ign
