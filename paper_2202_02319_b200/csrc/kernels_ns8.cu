// Explicit instantiation of the stage kernels for ns = 8 species
// (one translation unit per species count keeps builds parallel).
#include "kernels.cuh"

namespace ign {
KernelSet kernel_set_8() { return Launch<8>::make(); }
}  // namespace ign
