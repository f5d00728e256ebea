// io.hpp — field output and diagnostics of the B200 path: the IGNS snapshot
// format (snapshot.hpp:16-145) and the probe box average (solver.hpp:351-378).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

namespace ign {

// snapshot.hpp:16-30.  Version 1 is the reference's format (2D, state + J).
// Version 2 (this library only) adds nz (3D extension) after ns and an
// optional T-cache plane set after J (flags bit 0), so a restart can be bit
// exact — the T cache is the Newton guess and therefore part of the state.
struct Snapshot {
    uint32_t version = 1;
    int32_t nx = 0, ny = 0, g = 0, ns = 0, nz = 0;
    std::vector<std::string> species;
    double time = 0.0;
    int64_t iteration = 0;
    uint64_t config_hash = 0;
    uint32_t flags = 0;             // v2: bit 0 = T cache present
    size_t plane = 0;               // doubles per state field
    size_t jplane = 0;              // doubles of the J field
    std::vector<double> state;      // nc fields, each `plane`
    std::vector<double> jac;        // `jplane`
    std::vector<double> tcache;     // `plane` when flags & 1
};

// write_snapshot / read_snapshot (snapshot.hpp:52-115); throw ign::Error with
// the reference's FormatError messages
void snapshot_write(const Snapshot& s, const std::string& path);
Snapshot snapshot_read(const std::string& path);

// Box average of the primitive cache (solver.hpp:358-378) for one probe,
// continuing the running sums `init` (5 + ns values: rho, u, v, p, T, Y_s) over
// the local rows [j0, j1] x [i0, i1] in the reference's j-major order; one
// thread per quantity, so every sum is the serial one.  Writes `out`.
void launch_probe(const double* prim, long long plane, int sx, int g, int ns, int i0, int j0,
                  int i1, int j1, const double* init, double* out, cudaStream_t s);
// 3D extension: k-outermost box over local planes [k0, k1], 6 + ns values
// (rho, u, v, w, p, T, Y_s); sxy = padded (x, y) plane size
void launch_probe3(const double* prim, long long plane, int sx, long long sxy, int g, int ns,
                   int i0, int j0, int k0, int i1, int j1, int k1, const double* init,
                   double* out, cudaStream_t s);

}  // namespace ign
