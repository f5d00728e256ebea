// Explicit instantiation of the stage kernels for ns = 2 species
// (one translation unit per species count keeps builds parallel).
#include "kernels.cuh"

namespace ign {
KernelSet kernel_set_2() { return Launch<2>::make(); }
}  // namespace ign
