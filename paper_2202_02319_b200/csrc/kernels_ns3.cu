// Explicit instantiation of the stage kernels for ns = 3 species
// (one translation unit per species count keeps builds parallel).
#include "kernels.cuh"

namespace ign {
KernelSet kernel_set_3() { return Launch<3>::make(); }
}  // namespace ign
