// io.cu — IGNS snapshot codec (snapshot.hpp:16-145 restated) and the probe
// box-average kernel (solver.hpp:358-378).
#include "io.hpp"

#include <cstdio>
#include <cstring>
#include <memory>

#include "host_core.hpp"

namespace ign {

namespace {

inline Error format_error(const std::string& w) { return Error(IGN_FORMAT_ERROR, w); }

static const char kMagic[4] = {'I', 'G', 'N', 'S'};

struct File {
    std::FILE* f = nullptr;
    ~File() {
        if (f) std::fclose(f);
    }
};

template <class T> void put(std::FILE* f, T v, const std::string& path) {
    if (std::fwrite(&v, sizeof(T), 1, f) != 1)
        throw format_error("snapshot: write failed: " + path);
}

template <class T> T get(std::FILE* f) {
    T v{};
    if (std::fread(&v, sizeof(T), 1, f) != 1) throw format_error("snapshot: truncated file");
    return v;
}

void put_doubles(std::FILE* f, const double* p, size_t n, const std::string& path) {
    if (n && std::fwrite(p, sizeof(double), n, f) != n)
        throw format_error("snapshot: write failed: " + path);
}

void get_doubles(std::FILE* f, double* p, size_t n, const std::string& path) {
    if (n && std::fread(p, sizeof(double), n, f) != n)
        throw format_error("snapshot: truncated field data in " + path);
}

}  // namespace

// write_snapshot (snapshot.hpp:52-76): magic | u32 version | i32 nx, ny, g, ns
// | [v2: i32 nz] | names (u32 len + bytes) | f64 time | i64 iter | u64 hash |
// [v2: u32 flags] | nc state planes | J | [v2 flags&1: T plane]
void snapshot_write(const Snapshot& s, const std::string& path) {
    File fh;
    fh.f = std::fopen(path.c_str(), "wb");
    if (!fh.f) throw format_error("snapshot: cannot open for write: " + path);
    std::FILE* f = fh.f;
    if (std::fwrite(kMagic, 1, 4, f) != 4) throw format_error("snapshot: write failed: " + path);
    put<uint32_t>(f, s.version, path);
    put<int32_t>(f, s.nx, path);
    put<int32_t>(f, s.ny, path);
    put<int32_t>(f, s.g, path);
    put<int32_t>(f, s.ns, path);
    if (s.version >= 2) put<int32_t>(f, s.nz, path);
    for (int k = 0; k < s.ns; ++k) {
        const std::string& n = s.species[k];
        put<uint32_t>(f, static_cast<uint32_t>(n.size()), path);
        if (!n.empty() && std::fwrite(n.data(), 1, n.size(), f) != n.size())
            throw format_error("snapshot: write failed: " + path);
    }
    put<double>(f, s.time, path);
    put<int64_t>(f, s.iteration, path);
    put<uint64_t>(f, s.config_hash, path);
    if (s.version >= 2) put<uint32_t>(f, s.flags, path);
    put_doubles(f, s.state.data(), s.state.size(), path);
    put_doubles(f, s.jac.data(), s.jac.size(), path);
    if (s.version >= 2 && (s.flags & 1u)) put_doubles(f, s.tcache.data(), s.tcache.size(), path);
    if (std::fflush(f) != 0) throw format_error("snapshot: write failed: " + path);
}

// read_snapshot (snapshot.hpp:78-115) with the same checks and messages
Snapshot snapshot_read(const std::string& path) {
    File fh;
    fh.f = std::fopen(path.c_str(), "rb");
    if (!fh.f) throw format_error("snapshot: cannot open: " + path);
    std::FILE* f = fh.f;
    char magic[4];
    if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, kMagic, 4) != 0)
        throw format_error("snapshot: bad magic in " + path);
    Snapshot s;
    s.version = get<uint32_t>(f);
    if (s.version != 1 && s.version != 2)
        throw format_error("snapshot: unsupported version " + std::to_string(s.version));
    s.nx = get<int32_t>(f);
    s.ny = get<int32_t>(f);
    s.g = get<int32_t>(f);
    s.ns = get<int32_t>(f);
    if (s.version >= 2) s.nz = get<int32_t>(f);
    if (s.nx <= 0 || s.ny <= 0 || s.g < 0 || s.ns <= 0 || s.ns > kMaxSpecies || s.nz < 0)
        throw format_error("snapshot: implausible header in " + path);
    for (int k = 0; k < s.ns; ++k) {
        const uint32_t len = get<uint32_t>(f);
        if (len > 64) throw format_error("snapshot: species name too long");
        std::string name(len, '\0');
        if (len && std::fread(&name[0], 1, len, f) != len)
            throw format_error("snapshot: truncated file");
        s.species.push_back(name);
    }
    s.time = get<double>(f);
    s.iteration = get<int64_t>(f);
    s.config_hash = get<uint64_t>(f);
    if (s.version >= 2) s.flags = get<uint32_t>(f);
    const size_t p2 = static_cast<size_t>(s.nx + 2 * s.g) * (s.ny + 2 * s.g);
    s.plane = p2 * (s.nz > 0 ? static_cast<size_t>(s.nz + 2 * s.g) : 1);
    s.jplane = p2;
    const int nc = s.ns + (s.nz > 0 ? 4 : 3);
    s.state.resize(static_cast<size_t>(nc) * s.plane);
    get_doubles(f, s.state.data(), s.state.size(), path);
    s.jac.resize(s.jplane);
    get_doubles(f, s.jac.data(), s.jac.size(), path);
    if (s.flags & 1u) {
        s.tcache.resize(s.plane);
        get_doubles(f, s.tcache.data(), s.tcache.size(), path);
    }
    return s;
}

// ---------------------------------------------------------------- probes
__global__ void k_probe(const double* __restrict__ prim, long long plane, int sx, int g, int ns,
                        int i0, int j0, int i1, int j1, const double* __restrict__ init,
                        double* __restrict__ out) {
    const int q = threadIdx.x;
    if (q >= 5 + ns) return;
    // rho, u, v, p, T, then Y_s (cache slots 0..4, 6 + s; slot 5 is c)
    const double* f = prim + (q < 5 ? q : q + 1) * plane;
    double acc = init[q];
    for (int j = j0; j <= j1; ++j) {
        const double* row = f + (long long)(j + g) * sx + g;
        for (int i = i0; i <= i1; ++i) acc += row[i];
    }
    out[q] = acc;
}

__global__ void k_probe3(const double* __restrict__ prim, long long plane, int sx, long long sxy,
                         int g, int ns, int i0, int j0, int k0, int i1, int j1, int k1,
                         const double* __restrict__ init, double* __restrict__ out) {
    const int q = threadIdx.x;
    if (q >= 6 + ns) return;
    // rho, u, v, w, p, T, then Y_s (3D cache slots 0..5, 7 + s; slot 6 is c)
    const double* f = prim + (q < 6 ? q : q + 1) * plane;
    double acc = init[q];
    for (int k = k0; k <= k1; ++k)
        for (int j = j0; j <= j1; ++j) {
            const double* row = f + (long long)(k + g) * sxy + (long long)(j + g) * sx + g;
            for (int i = i0; i <= i1; ++i) acc += row[i];
        }
    out[q] = acc;
}

void launch_probe3(const double* prim, long long plane, int sx, long long sxy, int g, int ns,
                   int i0, int j0, int k0, int i1, int j1, int k1, const double* init,
                   double* out, cudaStream_t s) {
    k_probe3<<<1, 32, 0, s>>>(prim, plane, sx, sxy, g, ns, i0, j0, k0, i1, j1, k1, init, out);
}

void launch_probe(const double* prim, long long plane, int sx, int g, int ns, int i0, int j0,
                  int i1, int j1, const double* init, double* out, cudaStream_t s) {
    k_probe<<<1, 32, 0, s>>>(prim, plane, sx, g, ns, i0, j0, i1, j1, init, out);
}

}  // namespace ign
