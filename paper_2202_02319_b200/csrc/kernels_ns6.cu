// Explicit instantiation of the stage kernels for ns = 6 species
// (one translation unit per species count keeps builds parallel).
#include "kernels.cuh"

namespace ign {
KernelSet kernel_set_6() { return Launch<6>::make(); }
}  // namespace ign
