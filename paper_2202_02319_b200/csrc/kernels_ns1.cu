// Explicit instantiation of the stage kernels for ns = 1 species
// (one translation unit per species count keeps builds parallel).
#include "kernels.cuh"

namespace ign {
KernelSet kernel_set_1() { return Launch<1>::make(); }
}  // namespace ign
