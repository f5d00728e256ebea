// setup.cu — Simulation::init on the device: mesh, metrics (and their 3D
// extrusion), slab geometry, buffers, inflow tables, kernel parameters; the
// per-species-count kernel sets.
#include "context_internal.hpp"

namespace ign {
KernelSet kernel_set3(int ns) {
    switch (ns) {
    case 1: return kernel_set3_1();
    case 2: return kernel_set3_2();
    case 3: return kernel_set3_3();
    case 4: return kernel_set3_4();
    case 5: return kernel_set3_5();
    case 6: return kernel_set3_6();
    case 7: return kernel_set3_7();
    default: return kernel_set3_8();
    }
}

KernelSet kernel_set(int ns) {
    switch (ns) {
    case 1: return kernel_set_1();
    case 2: return kernel_set_2();
    case 3: return kernel_set_3();
    case 4: return kernel_set_4();
    case 5: return kernel_set_5();
    case 6: return kernel_set_6();
    case 7: return kernel_set_7();
    default: return kernel_set_8();
    }
}
}  // namespace ign
namespace ign {
namespace rt {

// ---------------------------------------------------------------- setup
// detail::inflow_profile (boundary.hpp:94-124) — host side, glibc tanh.
void inflow_profile(const ign_edge& es, double yc, int ns, double& u, double& v, double& T,
                    double* Y) {
    const double w = es.smooth_width > 0.0 ? es.smooth_width : 1e-30;
    double wsum = 0.0;
    u = v = T = 0.0;
    for (int s = 0; s < kMaxSpecies; ++s) Y[s] = 0.0;
    for (int k = 0; k < es.nseg; ++k) {
        const ign_inflow_segment& seg = es.seg[k];
        const double a = 0.5 * (std::tanh((yc - seg.lo) / w) - std::tanh((yc - seg.hi) / w));
        wsum += a;
        u += a * seg.u;
        v += a * seg.v;
        T += a * seg.T;
        for (int s = 0; s < ns; ++s) Y[s] += a * seg.Y[s];
    }
    if (wsum <= 1e-300) {
        const ign_inflow_segment& seg = es.seg[0];
        u = seg.u;
        v = seg.v;
        T = seg.T;
        for (int s = 0; s < kMaxSpecies; ++s) Y[s] = seg.Y[s];
        return;
    }
    u /= wsum;
    v /= wsum;
    T /= wsum;
    double ysum = 0.0;
    for (int s = 0; s < ns; ++s) ysum += Y[s];
    for (int s = 0; s < ns; ++s) Y[s] /= ysum;
}

// conservative_from_primitives for one node, runtime species count.
template <int NS>
void cons_from_prim_t(const DMix& m, double rho, double u, double v, double T, const double* Y,
                      double* U) {
    Prim<NS> pt;
    pt.rho = rho;
    pt.u = u;
    pt.v = v;
    pt.T = T;
    pt.p = 0.0;
    for (int s = 0; s < NS; ++s) pt.Y[s] = Y[s];
    conservative_from_primitives<NS>(pt, m, U);
}

void cons_from_prim(const DMix& m, double rho, double u, double v, double T, const double* Y,
                    double* U) {
    switch (m.ns) {
    case 1: return cons_from_prim_t<1>(m, rho, u, v, T, Y, U);
    case 2: return cons_from_prim_t<2>(m, rho, u, v, T, Y, U);
    case 3: return cons_from_prim_t<3>(m, rho, u, v, T, Y, U);
    case 4: return cons_from_prim_t<4>(m, rho, u, v, T, Y, U);
    case 5: return cons_from_prim_t<5>(m, rho, u, v, T, Y, U);
    case 6: return cons_from_prim_t<6>(m, rho, u, v, T, Y, U);
    case 7: return cons_from_prim_t<7>(m, rho, u, v, T, Y, U);
    default: return cons_from_prim_t<8>(m, rho, u, v, T, Y, U);
    }
}

template <int NS>
void cons_from_prim3_t(const DMix& m, const Prim3<kMaxSpecies>& in, const double* Y, double* U) {
    Prim3<NS> pt;
    pt.rho = in.rho;
    pt.u = in.u;
    pt.v = in.v;
    pt.w = in.w;
    pt.T = in.T;
    pt.p = 0.0;
    for (int s = 0; s < NS; ++s) pt.Y[s] = Y[s];
    conservative_from_primitives3<NS>(pt, m, U);
}

void cons_from_prim3(const DMix& m, const Prim3<kMaxSpecies>& pt, const double* Y, double* U) {
    switch (m.ns) {
    case 1: return cons_from_prim3_t<1>(m, pt, Y, U);
    case 2: return cons_from_prim3_t<2>(m, pt, Y, U);
    case 3: return cons_from_prim3_t<3>(m, pt, Y, U);
    case 4: return cons_from_prim3_t<4>(m, pt, Y, U);
    case 5: return cons_from_prim3_t<5>(m, pt, Y, U);
    case 6: return cons_from_prim3_t<6>(m, pt, Y, U);
    case 7: return cons_from_prim3_t<7>(m, pt, Y, U);
    default: return cons_from_prim3_t<8>(m, pt, Y, U);
    }
}

void upload_state(ign_context* ctx, const std::vector<double>& Ut) {
    h2d(ctx, ctx->S[ctx->cur], Ut.data(), Ut.size() * sizeof(double), "state upload");
}

void destroy_impl(ign_context* ctx) {
    if (!ctx) return;
    for (double* p : ctx->S) dfree(p);
    dfree(ctx->prim);
    dfree(ctx->geom);
    dfree(ctx->Fx);
    dfree(ctx->Gy);
    dfree(ctx->Fv);
    dfree(ctx->Gv);
    dfree(ctx->Hz);
    dfree(ctx->Hv);
    dfree(ctx->rhs);
    for (double* p : ctx->inflow) dfree(p);
    for (double* p : ctx->wrap) dfree(p);
    dfree(ctx->own_err);
    dfree(ctx->red);
    for (auto& r : ctx->prof_pending) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (cudaEvent_t e : ctx->prof_pool) cudaEventDestroy(e);
    if (ctx->comm && nccl().ok) nccl().CommDestroy(ctx->comm);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    if (ctx->halo_stream) cudaStreamDestroy(ctx->halo_stream);
    if (ctx->diag_buf) dfree(ctx->diag_buf);
    if (ctx->ev_ready) cudaEventDestroy(ctx->ev_ready);
    if (ctx->ev_halo) cudaEventDestroy(ctx->ev_halo);
    delete ctx;
}

void create_impl(const ign_config* cfg, ign_context* ctx) {
    if (!cfg || cfg->abi_version != IGN_ABI_VERSION)
        throw usage_error("ign_create: ABI version mismatch");
    ctx->cfg = *cfg;
    ctx->device = cfg->device;
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    ctx->nranks = cfg->slab_count > 1 ? cfg->slab_count : 1;
    ctx->rank = ctx->nranks > 1 ? cfg->slab_rank : 0;
    if (ctx->rank < 0 || ctx->rank >= ctx->nranks) throw usage_error("slab_rank out of range");
    // Simulation::init (solver.hpp:82-101), on this slab's rows
    // 2D: y-slabs of the mesh; 3D: z-slabs over the whole (x, y) mesh
    const bool three_d = cfg->nz > 0;
    ctx->mesh = three_d ? build_mesh(*cfg, 1, 0) : build_mesh(*cfg, ctx->nranks, ctx->rank);
    validate_config(*cfg, ctx->mesh);
    const int imode = inviscid_metric_mode(*cfg);
    ctx->met = compute_metrics(ctx->mesh, imode, cfg->skew_beta);
    ctx->metv = compute_metrics(ctx->mesh, MM_CENTRAL2, 0.0);
    ctx->integ = cfg->integ;
    int nz = 0;
    std::vector<double> mzz, vmzz;
    if (three_d) {
        // 3D extension: the (x, y) mesh extruded over lz (flux3.cuh)
        if (!(cfg->lz > 0.0)) throw config_error("3D: lz must be positive");
        // x / y edges take the reference's 2D rules on every z plane; z is
        // periodic or bounded by walls / outflow (cfg->zlo / zhi)
        int k0 = 0;
        slab_rows(cfg->nz, ctx->nranks, ctx->rank, k0, nz);
        if (nz < cfg->g) throw config_error("3D: every z-slab needs >= g planes");
        if (ctx->nranks == 1 && nz < 2 * cfg->g + 1) throw config_error("3D: nz must be >= 2g+1");
        ctx->k0 = k0;
        ctx->nz_glob = cfg->nz;
        const double dz = cfg->lz / cfg->nz;
        // cofactor metrics of (x(i,j), y(i,j), z(k)): xi/eta rows scale by z_zeta
        // = dz, zeta row is the 2D area, J = 1/(area dz) — for dz = 1 every value
        // is the 2D one bit for bit (the z-extrusion cross-check)
        auto extrude = [&](HMetrics& m, std::vector<double>& zz) {
            zz.resize(m.jac.d.size());
            for (size_t q = 0; q < zz.size(); ++q) {
                const double area =
                    m.m_eta_y.d[q] * m.m_xi_x.d[q] - (-m.m_xi_y.d[q]) * (-m.m_eta_x.d[q]);
                zz[q] = area;
                m.jac.d[q] = 1.0 / (area * dz);
                m.m_xi_x.d[q] *= dz;
                m.m_xi_y.d[q] *= dz;
                m.m_eta_x.d[q] *= dz;
                m.m_eta_y.d[q] *= dz;
            }
        };
        extrude(ctx->met, mzz);
        extrude(ctx->metv, vmzz);
    }
    const int nx = cfg->nx, ny = ctx->mesh.ny, g = cfg->g, ns = cfg->mix.ns,
              nc = ns + (nz > 0 ? 4 : 3);
    ctx->nz = nz;
    const int N = ctx->nranks, r = ctx->rank;
    const bool py = (three_d ? cfg->periodic_z : cfg->periodic_y) != 0;
    if (N > 1) {
        ctx->lo_peer = r > 0 ? r - 1 : (py ? N - 1 : -1);
        ctx->hi_peer = r < N - 1 ? r + 1 : (py ? 0 : -1);
    }
    ctx->nx = nx;
    ctx->ny = ny;
    ctx->g = g;
    ctx->ns = ns;
    ctx->nc = nc;
    const size_t P2 = static_cast<size_t>(nx + 2 * g) * (ny + 2 * g);  // one (x, y) plane
    const size_t P = P2 * (nz > 0 ? nz + 2 * g : 1);
    if (P >= (1ull << 31)) throw config_error("padded box too large for one context (>= 2^31 nodes)");
    ctx->plane = P;
    cuda_check(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking), "stream");
    ctx->stream = ctx->own_stream;
    for (auto& s : ctx->S) {
        s = dalloc(nc * P);
        cuda_check(cudaMemset(s, 0, nc * P * sizeof(double)), "memset");
    }
    // primitive cache: rho,u,v,(w),p = 0, T = c = 1 (solver.hpp:94-100), Y, X
    const size_t head = nz > 0 ? 7 : 6;
    const size_t nprim = head + 2 * static_cast<size_t>(ns);
    ctx->prim = dalloc(nprim * P);
    {
        std::vector<double> init(nprim * P, 0.0);
        std::fill(init.begin() + (head - 2) * P, init.begin() + head * P, 1.0);
        cuda_check(cudaMemcpy(ctx->prim, init.data(), init.size() * sizeof(double),
                              cudaMemcpyHostToDevice),
                   "cache init");
    }
    ctx->geom = dalloc((nz > 0 ? 14 : 12) * P2);
    {
        // 2D: mesh x, y in slots 10, 11 (laser); 3D: the zeta metrics there
        const std::vector<double>* f[12] = {
            &ctx->met.jac.d,    &ctx->met.m_xi_x.d,  &ctx->met.m_xi_y.d,  &ctx->met.m_eta_x.d,
            &ctx->met.m_eta_y.d, &ctx->metv.jac.d,   &ctx->metv.m_xi_x.d, &ctx->metv.m_xi_y.d,
            &ctx->metv.m_eta_x.d, &ctx->metv.m_eta_y.d, nz > 0 ? &mzz : &ctx->mesh.x.d,
            nz > 0 ? &vmzz : &ctx->mesh.y.d};
        for (int k = 0; k < 12; ++k)
            cuda_check(cudaMemcpy(ctx->geom + k * P2, f[k]->data(), P2 * sizeof(double),
                                  cudaMemcpyHostToDevice),
                       "geometry upload");
        if (nz > 0) {  // 3D: mesh x, y in slots 12, 13 (laser)
            cuda_check(cudaMemcpy(ctx->geom + 12 * P2, ctx->mesh.x.d.data(), P2 * sizeof(double),
                                  cudaMemcpyHostToDevice),
                       "geometry upload");
            cuda_check(cudaMemcpy(ctx->geom + 13 * P2, ctx->mesh.y.d.data(), P2 * sizeof(double),
                                  cudaMemcpyHostToDevice),
                       "geometry upload");
        }
    }
    const size_t nzc = nz > 0 ? nz : 1;
    ctx->Fx = dalloc(static_cast<size_t>(nc) * (nx + 1) * ny * nzc);
    ctx->Gy = dalloc(static_cast<size_t>(nc) * nx * (ny + 1) * nzc);
    if (nz > 0) ctx->Hz = dalloc(static_cast<size_t>(nc) * nx * ny * (nz + 1));
    if (cfg->viscous) {
        ctx->Fv = dalloc(nc * P);
        ctx->Gv = dalloc(nc * P);
        if (nz > 0) ctx->Hv = dalloc(nc * P);
    }
    // inflow profile tables (boundary.hpp:227-241 ghost targets)
    const ign_edge* edges[4] = {&cfg->bc.left, &cfg->bc.right, &cfg->bc.bottom, &cfg->bc.top};
    int bc_type[4] = {edges[0]->type, edges[1]->type, edges[2]->type, edges[3]->type};
    if (!three_d && ctx->lo_peer >= 0) bc_type[2] = (r == 0) ? BC_HALO_WRAP : BC_HALO;
    if (!three_d && ctx->hi_peer >= 0) bc_type[3] = (r == N - 1) ? BC_HALO_WRAP : BC_HALO;
    for (int e = 0; e < 4; ++e) {
        if (bc_type[e] != 3) continue;
        const bool xedge = e < 2;
        const int tlo = xedge ? 0 : -g, ntr = xedge ? ny : nx + 2 * g;
        std::vector<double> tab(static_cast<size_t>(ntr) * g * (3 + ns));
        for (int t = tlo; t < tlo + ntr; ++t)
            for (int k = 1; k <= g; ++k) {
                int id, jd;
                switch (e) {
                case 0: id = -k; jd = t; break;
                case 1: id = nx - 1 + k; jd = t; break;
                case 2: id = t; jd = -k; break;
                default: id = t; jd = ny - 1 + k; break;
                }
                const double yc = xedge ? ctx->mesh.eta(jd) : ctx->mesh.xi(id);
                double u, v, T, Y[kMaxSpecies];
                inflow_profile(*edges[e], yc, ns, u, v, T, Y);
                double* q = &tab[(static_cast<size_t>(t - tlo) * g + (k - 1)) * (3 + ns)];
                q[0] = u;
                q[1] = v;
                q[2] = T;
                for (int s = 0; s < ns; ++s) q[3 + s] = Y[s];
            }
        ctx->inflow[e] = dalloc(tab.size());
        cuda_check(cudaMemcpy(ctx->inflow[e], tab.data(), tab.size() * sizeof(double),
                              cudaMemcpyHostToDevice),
                   "inflow upload");
    }
    // periodic wrap across slabs: ratio J(src)/J(dst) of the reference's
    // periodic copy (boundary.hpp:146-149); src rows belong to the far slab
    const int sx = nx + 2 * g;
    for (int side = 0; side < 2; ++side) {
        if (bc_type[2 + side] != BC_HALO_WRAP) continue;
        const int NG = ctx->mesh.ny_glob;
        // dst global rows: bottom -g..-1, top NG..NG+g-1; src: NG-g..NG-1 / 0..g-1
        const int dlo = side == 0 ? -g : NG, slo = side == 0 ? NG - g : 0;
        const std::vector<double> Jd = jac_rows(ctx->mesh, imode, cfg->skew_beta, dlo, dlo + g);
        const std::vector<double> Js = jac_rows(ctx->mesh, imode, cfg->skew_beta, slo, slo + g);
        std::vector<double> tab(size_t(g) * sx);
        for (int k = 1; k <= g; ++k) {
            // ghost layer k: dst row (bottom) -k / (top) NG-1+k; src row NG-k / k-1
            const int drow = side == 0 ? -k - dlo : NG - 1 + k - dlo;
            const int srow = side == 0 ? NG - k - slo : k - 1 - slo;
            for (int t = -g; t < nx + g; ++t)
                tab[size_t(k - 1) * sx + (t + g)] =
                    Js[size_t(srow) * sx + (t + g)] / Jd[size_t(drow) * sx + (t + g)];
        }
        ctx->wrap[side] = dalloc(tab.size());
        cuda_check(cudaMemcpy(ctx->wrap[side], tab.data(), tab.size() * sizeof(double),
                              cudaMemcpyHostToDevice),
                   "wrap upload");
    }
    void* p = dmalloc(sizeof(ErrRec));
    ctx->own_err = static_cast<ErrRec*>(p);
    ctx->err = ctx->own_err;
    cuda_check(cudaMemset(ctx->err, 0xff, sizeof(ErrRec)), "memset");
    p = dmalloc(kRedSlots * sizeof(unsigned long long));
    ctx->red = static_cast<unsigned long long*>(p);
    cuda_check(cudaMemset(ctx->red, 0, kRedSlots * sizeof(unsigned long long)), "memset");

    KParams& k = ctx->kp;
    std::memset(&k, 0, sizeof(k));
    k.nx = nx;
    k.ny = ny;
    k.g = g;
    k.sx = sx;
    k.plane = static_cast<long long>(P);
    k.j0 = ctx->mesh.j0;
    k.ny_glob = ctx->mesh.ny_glob;
    k.ns = ns;
    k.viscous = cfg->viscous;
    for (int e = 0; e < 4; ++e) {
        k.bc_type[e] = bc_type[e];
        k.T_wall[e] = edges[e]->T_wall;
        k.inflow[e] = ctx->inflow[e];
    }
    k.wrap[0] = ctx->wrap[0];
    k.wrap[1] = ctx->wrap[1];
    k.sigma_out_right = cfg->bc.right.sigma_out;
    k.p_target_right = cfg->bc.right.p_target;
    k.lodi = cfg->bc.right.type == 4;
    k.lx = cfg->lx;
    k.ly = cfg->ly;
    k.cx = cfg->center_x;
    k.cy = cfg->center_y;
    if (cfg->nz > 0) {
        k.zc0 = cfg->center_z - 0.5 * cfg->lz;
        k.dz = cfg->lz / cfg->nz;  // nz is the GLOBAL plane count in the config
    }
    k.rp = make_recon_params(cfg->scheme.teno_ct, cfg->scheme.eps);
    k.chem_dt_limit = cfg->integ.chem_dt_limit;
    k.chem_dt_factor = cfg->integ.chem_dt_factor;
    k.prim = ctx->prim;
    k.jac = ctx->geom;
    k.mxx = ctx->geom + P2;
    k.mxy = ctx->geom + 2 * P2;
    k.mex = ctx->geom + 3 * P2;
    k.mey = ctx->geom + 4 * P2;
    k.vjac = ctx->geom + 5 * P2;
    k.vmxx = ctx->geom + 6 * P2;
    k.vmxy = ctx->geom + 7 * P2;
    k.vmex = ctx->geom + 8 * P2;
    k.vmey = ctx->geom + 9 * P2;
    if (nz > 0) {
        k.mzz = ctx->geom + 10 * P2;
        k.vmzz = ctx->geom + 11 * P2;
        k.xc = ctx->geom + 12 * P2;
        k.yc = ctx->geom + 13 * P2;
    } else {
        k.xc = ctx->geom + 10 * P2;
        k.yc = ctx->geom + 11 * P2;
    }
    k.nz = nz;
    k.nz_glob = three_d ? ctx->nz_glob : 0;
    if (three_d) {
        k.j0 = ctx->k0;  // 3D: global z offset of the slab (error keys)
        k.zhalo = ctx->lo_peer >= 0 || ctx->hi_peer >= 0;
        const ign_edge* ze[2] = {&cfg->zlo, &cfg->zhi};
        const bool peer[2] = {ctx->lo_peer >= 0, ctx->hi_peer >= 0};
        for (int side = 0; side < 2; ++side) {
            k.bc_z[side] = peer[side] ? BC_HALO : cfg->periodic_z ? 0 : ze[side]->type;
            k.T_wall_z[side] = ze[side]->T_wall;
        }
    }
    k.sxy = static_cast<long long>(P2);
    k.Fx = ctx->Fx;
    k.Gy = ctx->Gy;
    k.Hz = ctx->Hz;
    k.Fv = ctx->Fv;
    k.Gv = ctx->Gv;
    k.Hv = ctx->Hv;
    k.err = ctx->err;
    k.red = ctx->red;
    k.mix = build_mix(cfg->mix);
    k.mech = build_mech(cfg->mech);
    k.laser = build_laser(cfg->laser);
    ctx->ks = nz > 0 ? kernel_set3(ns) : kernel_set(ns);
    // the uploads and memsets above ran on the legacy stream, which the
    // context's non-blocking stream does not wait for: finish them here
    cuda_check(cudaDeviceSynchronize(), "setup");
}

void copy_hfield(const HField& f, double* out) { std::memcpy(out, f.d.data(), f.d.size() * 8); }

void metrics_out(const HMetrics& m, double* out, size_t P) {
    const HField* f[5] = {&m.jac, &m.m_xi_x, &m.m_xi_y, &m.m_eta_x, &m.m_eta_y};
    for (int k = 0; k < 5; ++k) copy_hfield(*f[k], out + k * P);
}

}  // namespace rt
}  // namespace ign
