// outputs.cu — diagnostics and field output over a team: exact rank-ordered
// folds (conserved totals, product fraction), probes and the trace sampled
// by advance(), the gather / scatter of IGNS snapshots.
#include "context_internal.hpp"

namespace ign {
namespace rt {

// Serial left folds in the reference's order (solver.hpp:387-418) across
// slabs: each slab continues the running accumulators of the slab below, so
// the decomposed result is bit-identical to the single-domain one.
void fold_ranks(const Team& T, std::vector<double>& acc,
                const std::function<void(ign_context*, std::vector<double>&)>& fold) {
    if (T.local()) {
        for (ign_context* c : T.m) fold(c, acc);
        return;
    }
    ign_context* c = T.lead();
    if (!c->comm || c->nranks == 1) {
        fold(c, acc);
        return;
    }
    NcclApi& n = nccl();
    double* d = dalloc(acc.size());
    try {
        if (c->rank > 0) {
            nccl_check(n.Recv(d, acc.size(), ncclFloat64, c->rank - 1, c->comm, c->stream),
                       "ncclRecv(fold)");
            cuda_check(cudaMemcpyAsync(acc.data(), d, acc.size() * 8, cudaMemcpyDeviceToHost,
                                       c->stream), "fold");
            cuda_check(cudaStreamSynchronize(c->stream), "fold");
        }
        fold(c, acc);
        cuda_check(cudaMemcpyAsync(d, acc.data(), acc.size() * 8, cudaMemcpyHostToDevice,
                                   c->stream), "fold");
        if (c->rank + 1 < c->nranks)
            nccl_check(n.Send(d, acc.size(), ncclFloat64, c->rank + 1, c->comm, c->stream),
                       "ncclSend(fold)");
        nccl_check(n.Broadcast(d, d, acc.size(), ncclFloat64, c->nranks - 1, c->comm, c->stream),
                   "ncclBroadcast(fold)");
        cuda_check(cudaMemcpyAsync(acc.data(), d, acc.size() * 8, cudaMemcpyDeviceToHost,
                                   c->stream), "fold");
        cuda_check(cudaStreamSynchronize(c->stream), "fold");
    } catch (...) {
        dfree(d);
        throw;
    }
    dfree(d);
}

// ---------------------------------------------------------------- device tree sums
// The default diagnostics: conserved_totals and the product
// mole fraction reduced ON THE DEVICE by a fixed-shape tree — kTreeBlocks
// blocks of kTreeThreads threads; thread t of block b adds cells b T + t,
// (b + B) T + t, ... in increasing order, each block then adds pairwise with
// halving strides, and one thread per value adds the B block sums in block
// order.  Deterministic (same bits every call for a given decomposition) and
// free of any full-field D2H copy; it differs from the reference's serial
// left fold (solver.hpp:387-418) only by summation order: |tree - serial| <=
// ~(n + log2 n) eps sum|x| (tests use 1e-12 sum|x|; typically 1e-15).  The
// reference's serial order stays available, bitwise, as IGN_DIAG_REFERENCE.
namespace {
constexpr int kTreeBlocks = 296;  // 2 x 148 SMs
constexpr int kTreeThreads = 256;
constexpr int kTreeMaxValues = IGN_MAX_COMP + 1;

struct Interior {
    int nx, ny, nz, g, sx;
    long long sxy, n;
    __device__ long long padded(long long c) const {
        const long long i = c % nx, r = c / nx;
        const long long j = nz > 0 ? r % ny : r, k = nz > 0 ? r / ny : 0;
        return (nz > 0 ? (k + g) * sxy : 0) + (j + g) * sx + (i + g);
    }
    __device__ int plane2(long long c) const {  // (x, y) metric-plane index
        const long long i = c % nx, r = c / nx;
        const long long j = nz > 0 ? r % ny : r;
        return (int)((j + g) * sx + (i + g));
    }
};

Interior interior_of(const ign_context* c) {
    Interior d;
    d.nx = c->nx;
    d.ny = c->ny;
    d.nz = c->nz;
    d.g = c->g;
    d.sx = c->nx + 2 * c->g;
    d.sxy = (long long)d.sx * (c->ny + 2 * c->g);
    d.n = (long long)c->nx * c->ny * (c->nz > 0 ? c->nz : 1);
    return d;
}

template <class F>
__device__ void tree_block(const Interior& d, int nv, F&& cell, double* part) {
    __shared__ double sh[kTreeMaxValues][kTreeThreads];
    double a[kTreeMaxValues];
    for (int q = 0; q < nv; ++q) a[q] = 0.0;
    for (long long c = (long long)blockIdx.x * kTreeThreads + threadIdx.x; c < d.n;
         c += (long long)kTreeBlocks * kTreeThreads)
        cell(c, a);
    for (int q = 0; q < nv; ++q) sh[q][threadIdx.x] = a[q];
    __syncthreads();
    for (int s = kTreeThreads / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s)
            for (int q = 0; q < nv; ++q) sh[q][threadIdx.x] += sh[q][threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0)
        for (int q = 0; q < nv; ++q) part[q * kTreeBlocks + blockIdx.x] = sh[q][0];
}

__global__ void __launch_bounds__(kTreeThreads) k_tree_totals(Interior d, const double* __restrict__ U,
                                                          long long plane, int nc, double* part) {
    tree_block(d, nc, [&](long long c, double* a) {
        const long long id = d.padded(c);
        for (int q = 0; q < nc; ++q) a[q] += U[q * plane + id];
    }, part);
}

// per cell: w (X_CO2 + X_H2O) and w = 1/J, mole fractions as
// thermo::mole_fractions (solver.hpp:393-402, thermo.hpp)
__global__ void __launch_bounds__(kTreeThreads) k_tree_product(const __grid_constant__ KParams P,
                                                           Interior d, int ico2, int ih2o,
                                                           double* part) {
    const double* Y = P.nz > 0 ? PY3(P, 0) : PY(P, 0);
    tree_block(d, 2, [&](long long c, double* a) {
        const long long id = d.padded(c);
        double y[kMaxSpecies], x[kMaxSpecies];
        for (int s = 0; s < P.ns; ++s) y[s] = Y[s * P.plane + id];
        double inv = 0.0;
        for (int s = 0; s < P.ns; ++s) inv += divW(P.mix.sp[s], y[s]);
        const double wbar = 1.0 / inv;
        for (int s = 0; s < P.ns; ++s) x[s] = divW(P.mix.sp[s], y[s] * wbar);
        const double w = 1.0 / P.jac[d.plane2(c)];
        a[0] += w * ((ico2 >= 0 ? x[ico2] : 0.0) + (ih2o >= 0 ? x[ih2o] : 0.0));
        a[1] += w;
    }, part);
}

__global__ void k_tree_final(const double* __restrict__ part, int nv, double* out) {
    const int q = threadIdx.x;
    if (q >= nv) return;
    double s = 0.0;
    for (int b = 0; b < kTreeBlocks; ++b) s += part[q * kTreeBlocks + b];
    out[q] = s;
}

double* diag_scratch(ign_context* c) {
    if (!c->diag_buf) c->diag_buf = dalloc(size_t(kTreeMaxValues) * (kTreeBlocks + 1));
    return c->diag_buf;
}

// one slab's tree sums (nv values) -> host
void tree_read(ign_context* c, int nv, double* out) {
    double* part = diag_scratch(c);
    double* res = part + size_t(kTreeMaxValues) * kTreeBlocks;
    k_tree_final<<<1, 32, 0, c->stream>>>(part, nv, res);
    c->launches += 1;
    cuda_check(cudaGetLastError(), "tree reduction");
    cuda_check(cudaMemcpyAsync(out, res, nv * sizeof(double), cudaMemcpyDeviceToHost, c->stream),
               "tree readback");
    cuda_check(cudaStreamSynchronize(c->stream), "tree reduction");
}
}  // namespace

// conserved_totals (solver.hpp:411-418)
void t_conserved_totals(const Team& T, double* tot) {
    t_join(T);
    const int nc = T.lead()->nc;
    if (T.lead()->diag_mode == IGN_DIAG_DEVICE) {
        std::vector<double> acc(nc, 0.0);
        fold_ranks(T, acc, [&](ign_context* c, std::vector<double>& a) {
            k_tree_totals<<<kTreeBlocks, kTreeThreads, 0, c->stream>>>(
                interior_of(c), c->S[c->cur], (long long)c->plane, c->nc, diag_scratch(c));
            c->launches += 1;
            std::vector<double> v(nc);
            tree_read(c, nc, v.data());
            for (int q = 0; q < nc; ++q) a[q] += v[q];
        });
        for (int q = 0; q < nc; ++q) tot[q] = acc[q];
        return;
    }
    std::vector<double> acc(nc, 0.0);
    // component-major in the reference: fold per component across slabs
    for (int comp = 0; comp < nc; ++comp) {
        std::vector<double> a1(1, 0.0);
        fold_ranks(T, a1, [&](ign_context* c, std::vector<double>& a) {
            const size_t P = c->plane;
            std::vector<double> U(P);
            d2h(c, U.data(), c->S[c->cur] + comp * P, P * 8, "totals");
            const int sx = c->nx + 2 * c->g, g = c->g;
            const size_t sxy = size_t(sx) * (c->ny + 2 * g);
            double s = a[0];
            for (int k = 0; k < (c->nz > 0 ? c->nz : 1); ++k)  // 3D: z-planes outermost
                for (int j = 0; j < c->ny; ++j)
                    for (int i = 0; i < c->nx; ++i)
                        s += U[(c->nz > 0 ? (k + g) * sxy : 0) + (size_t)(j + g) * sx + (i + g)];
            a[0] = s;
        });
        tot[comp] = a1[0];
    }
}

// product_mole_fraction (solver.hpp:387-407)
double t_product_fraction(const Team& T) {
    ign_context* L = T.lead();
    int ico2 = -1, ih2o = -1;
    for (int s = 0; s < L->ns; ++s) {
        const char* nm = L->cfg.mix.species[s].name;
        if (std::strncmp(nm, "CO2", IGN_NAME_LEN) == 0) ico2 = s;
        if (std::strncmp(nm, "H2O", IGN_NAME_LEN) == 0) ih2o = s;
    }
    if (ico2 < 0 && ih2o < 0) return 0.0;
    t_join(T);
    std::vector<double> acc(2, 0.0);
    if (L->diag_mode == IGN_DIAG_DEVICE) {
        fold_ranks(T, acc, [&](ign_context* c, std::vector<double>& a) {
            k_tree_product<<<kTreeBlocks, kTreeThreads, 0, c->stream>>>(c->kp, interior_of(c),
                                                                        ico2, ih2o,
                                                                        diag_scratch(c));
            c->launches += 1;
            double v[2];
            tree_read(c, 2, v);
            a[0] += v[0];
            a[1] += v[1];
        });
        return acc[0] / acc[1];
    }
    fold_ranks(T, acc, [&](ign_context* c, std::vector<double>& a) {
        const size_t P = c->plane;
        std::vector<double> Y(c->ns * P);
        d2h(c, Y.data(), c->prim + (c->nz > 0 ? 7 : 6) * P, Y.size() * 8, "Y readback");
        const DMix& m = c->kp.mix;
        const int sx = c->nx + 2 * c->g, g = c->g;
        const size_t sxy = size_t(sx) * (c->ny + 2 * g);
        double num = a[0], den = a[1];
        for (int kz = 0; kz < (c->nz > 0 ? c->nz : 1); ++kz)
        for (int j = 0; j < c->ny; ++j)
            for (int i = 0; i < c->nx; ++i) {
                const size_t id =
                    (c->nz > 0 ? (kz + g) * sxy : 0) + (size_t)(j + g) * sx + (i + g);
                double y[kMaxSpecies], x[kMaxSpecies];
                for (int s = 0; s < c->ns; ++s) y[s] = Y[s * P + id];
                double inv = 0.0;
                for (int s = 0; s < c->ns; ++s) inv += divW(m.sp[s], y[s]);
                const double wbar = 1.0 / inv;
                for (int s = 0; s < c->ns; ++s) x[s] = divW(m.sp[s], y[s] * wbar);
                const double w = 1.0 / c->met.jac(i, j);
                num += w * ((ico2 >= 0 ? x[ico2] : 0.0) + (ih2o >= 0 ? x[ih2o] : 0.0));
                den += w;
            }
        a[0] = num;
        a[1] = den;
    });
    return acc[0] / acc[1];
}

// ---------------------------------------------------------------- outputs
// sample_outputs (solver.hpp:353-385): box-averaged primitives per probe (on
// the device, serial sums in the reference's j-major order, continued slab to
// slab), and the product-fraction trace.  Results live on the lead context.
void t_sample(const Team& T) {
    ign_context* L = T.lead();
    const bool want_probe = L->probe_interval > 0 && (L->iter % L->probe_interval == 0);
    const bool want_trace = L->trace_interval > 0 && (L->iter % L->trace_interval == 0);
    if (want_probe) {
        const bool three_d = L->nz > 0;
        const int nq = (three_d ? 6 : 5) + L->ns;
        double* d = dalloc(2 * static_cast<size_t>(nq));
        try {
            for (auto& pr : L->probes) {
                std::vector<double> row(nq, 0.0);
                fold_ranks(T, row, [&](ign_context* c, std::vector<double>& a) {
                    // this slab's share of the box: 2D y rows, 3D z planes
                    const int off = three_d ? c->k0 : c->mesh.j0;
                    const int cnt = three_d ? c->nz : c->ny;
                    const int lo = std::max(three_d ? pr.k0 : pr.j0, off);
                    const int hi = std::min(three_d ? pr.k1 : pr.j1, off + cnt - 1);
                    if (lo > hi) return;
                    cuda_check(cudaMemcpyAsync(d, a.data(), nq * 8, cudaMemcpyHostToDevice,
                                               c->stream), "probe");
                    if (three_d)
                        launch_probe3(c->prim, (long long)c->plane, c->kp.sx, c->kp.sxy, c->g,
                                      c->ns, pr.i0, pr.j0, lo - off, pr.i1, pr.j1, hi - off, d,
                                      d + nq, c->stream);
                    else
                        launch_probe(c->prim, (long long)c->plane, c->kp.sx, c->g, c->ns, pr.i0,
                                     lo - off, pr.i1, hi - off, d, d + nq, c->stream);
                    c->launches += 1;
                    cuda_check(cudaMemcpyAsync(a.data(), d + nq, nq * 8, cudaMemcpyDeviceToHost,
                                               c->stream), "probe");
                    cuda_check(cudaStreamSynchronize(c->stream), "probe");
                });
                const int n = (pr.i1 - pr.i0 + 1) * (pr.j1 - pr.j0 + 1) * (pr.k1 - pr.k0 + 1);
                for (auto& x : row) x /= n;
                pr.times.push_back(L->time);
                pr.rows.insert(pr.rows.end(), row.begin(), row.end());
            }
        } catch (...) {
            dfree(d);
            throw;
        }
        dfree(d);
    }
    if (want_trace) {
        L->trace_t.push_back(L->time);
        L->trace_v.push_back(t_product_fraction(T));
    }
}

// Global padded layers (2D rows / 3D planes) of the current state, gathered
// on the lead (rank 0): each slab contributes its interior layers, the first
// and last also the global edge ghosts — exactly the undecomposed planes.
// `field` selects the source: the state components (nc planes) or the T cache.
void t_gather(const Team& T, bool tcache, std::vector<double>& out) {
    ign_context* L = T.lead();
    const int N = T.local() ? (int)T.m.size() : L->nranks, g = L->g;
    const bool three_d = L->nz > 0;
    const size_t st = halo_stride(L);
    const int NG = three_d ? L->nz_glob : L->mesh.ny_glob;
    const int nf = tcache ? 1 : L->nc;
    const size_t gplane = static_cast<size_t>(NG + 2 * g) * st;
    if (!T.local() && L->rank != 0 && L->comm) {
        // non-lead rank: send its layers to rank 0
        NcclApi& n = nccl();
        const int nl = (int)halo_count(L);
        const int p0 = g, p1 = (L->rank == N - 1) ? nl + 2 * g : nl + g;
        nccl_check(n.GroupStart(), "ncclGroupStart");
        for (int c = 0; c < nf; ++c) {
            const double* src = (tcache ? L->prim + (three_d ? 5 : 4) * L->plane
                                        : L->S[L->cur] + c * L->plane) + p0 * st;
            nccl_check(n.Send(src, (p1 - p0) * st, ncclFloat64, 0, L->comm, L->stream),
                       "ncclSend(gather)");
        }
        nccl_check(n.GroupEnd(), "ncclGroupEnd");
        cuda_check(cudaStreamSynchronize(L->stream), "gather");
        return;
    }
    out.assign(static_cast<size_t>(nf) * gplane, 0.0);
    double* stage = nullptr;
    for (int r = 0; r < N; ++r) {
        int lo, nl;
        slab_rows(NG, N, r, lo, nl);
        const int p0 = r == 0 ? 0 : g, p1 = r == N - 1 ? nl + 2 * g : nl + g;
        const size_t cnt = (p1 - p0) * st;
        for (int c = 0; c < nf; ++c) {
            double* dst = out.data() + c * gplane + (lo + p0) * st;
            const ign_context* m = T.local() ? T.m[r] : L;
            if (T.local() || r == 0) {
                const double* src = (tcache ? m->prim + (three_d ? 5 : 4) * m->plane
                                            : m->S[m->cur] + c * m->plane) + p0 * st;
                d2h(m, dst, src, cnt * 8, "gather");
            } else {
                if (!stage) stage = dalloc(static_cast<size_t>(NG / N + 2 + 2 * g) * st);
                NcclApi& n = nccl();
                nccl_check(n.Recv(stage, cnt, ncclFloat64, r, L->comm, L->stream),
                           "ncclRecv(gather)");
                cuda_check(cudaMemcpyAsync(dst, stage, cnt * 8, cudaMemcpyDeviceToHost, L->stream),
                           "gather");
                cuda_check(cudaStreamSynchronize(L->stream), "gather");
            }
        }
    }
    if (stage) dfree(stage);
}

// write_snapshot (snapshot.hpp:52-76): version 1 = the reference's format
// (2D); version 2 adds nz (3D) and, with `with_t`, the T cache
void t_write_snapshot(const Team& T, const std::string& path, int version, bool with_t) {
    ign_context* L = T.lead();
    const bool three_d = L->nz > 0;
    if (three_d && version < 2) throw usage_error("snapshot: 3D state needs IGNS version 2");
    if (version != 1 && version != 2) throw usage_error("snapshot: version must be 1 or 2");
    Snapshot s;
    t_gather(T, false, s.state);
    if (with_t) t_gather(T, true, s.tcache);
    if (!T.local() && L->rank != 0 && L->comm) return;  // rank 0 writes
    s.version = (uint32_t)version;
    s.nx = L->nx;
    s.ny = three_d ? L->ny : L->mesh.ny_glob;
    s.g = L->g;
    s.ns = L->ns;
    s.nz = three_d ? L->nz_glob : 0;
    for (int k = 0; k < L->ns; ++k)
        s.species.emplace_back(L->cfg.mix.species[k].name,
                               strnlen(L->cfg.mix.species[k].name, IGN_NAME_LEN));
    s.time = L->time;
    s.iteration = L->iter;
    s.config_hash = L->config_hash;
    s.flags = with_t ? 1u : 0u;
    // J over the global padded rows (2D: the reference's met.jac; 3D: the
    // extruded J of every z plane)
    const int g = L->g, NG = s.ny;
    if (three_d || L->nranks == 1)
        s.jac = L->met.jac.d;  // the whole (x, y) plane already
    else                       // 2D slabs: the global rows, global stencils
        s.jac = jac_rows(L->mesh, inviscid_metric_mode(L->cfg), L->cfg.skew_beta, -g, NG + g);
    snapshot_write(s, path);
}

// read_snapshot + apply_snapshot (snapshot.hpp:78-145): every slab reads the
// file and takes its own layers; time, iteration and hash are restored, the
// T cache too when the file carries it (v2)
void t_read_snapshot(const Team& T, const std::string& path) {
    ign_context* L = T.lead();
    const Snapshot s = snapshot_read(path);
    const bool three_d = L->nz > 0;
    const int NG = three_d ? L->nz_glob : L->mesh.ny_glob;
    const int sny = three_d ? L->ny : L->mesh.ny_glob;
    if (s.nx != L->nx || s.ny != sny || s.g != L->g || s.nz != (three_d ? L->nz_glob : 0))
        throw Error(IGN_FORMAT_ERROR,
                    "snapshot: shape mismatch, file " + std::to_string(s.nx) + "x" +
                        std::to_string(s.ny) + " (g=" + std::to_string(s.g) +
                        ") vs simulation " + std::to_string(L->nx) + "x" + std::to_string(sny) +
                        " (g=" + std::to_string(L->g) + ")");
    if (s.ns != L->ns) throw Error(IGN_FORMAT_ERROR, "snapshot: species count mismatch");
    for (int k = 0; k < s.ns; ++k)
        if (s.species[k] != std::string(L->cfg.mix.species[k].name,
                                        strnlen(L->cfg.mix.species[k].name, IGN_NAME_LEN)))
            throw Error(IGN_FORMAT_ERROR,
                        "snapshot: species name mismatch at slot " + std::to_string(k));
    const size_t st = halo_stride(L);
    const size_t gplane = static_cast<size_t>(NG + 2 * L->g) * st;
    for (ign_context* c : T.m) {
        const int lo = three_d ? c->k0 : c->mesh.j0;  // global interior start
        const size_t cnt = (halo_count(c) + 2 * c->g) * st;
        for (int comp = 0; comp < c->nc; ++comp)
            h2d(c, c->S[c->cur] + comp * c->plane, s.state.data() + comp * gplane + lo * st,
                cnt * 8, "snapshot upload");
        if (s.flags & 1u)
            h2d(c, c->prim + (three_d ? 5 : 4) * c->plane, s.tcache.data() + lo * st, cnt * 8,
                "snapshot upload");
        c->time = s.time;
        c->iter = s.iteration;
        c->config_hash = s.config_hash;
    }
}

}  // namespace rt
}  // namespace ign
