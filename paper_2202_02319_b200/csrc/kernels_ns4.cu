// Explicit instantiation of the stage kernels for ns = 4 species
// (one translation unit per species count keeps builds parallel).
#include "kernels.cuh"

namespace ign {
KernelSet kernel_set_4() { return Launch<4>::make(); }
}  // namespace ign
