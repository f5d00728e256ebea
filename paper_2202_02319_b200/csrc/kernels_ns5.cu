// Explicit instantiation of the stage kernels for ns = 5 species
// (one translation unit per species count keeps builds parallel).
#include "kernels.cuh"

namespace ign {
KernelSet kernel_set_5() { return Launch<5>::make(); }
}  // namespace ign
