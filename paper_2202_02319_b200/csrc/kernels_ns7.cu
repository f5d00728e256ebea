// Explicit instantiation of the stage kernels for ns = 7 species
// (one translation unit per species count keeps builds parallel).
#include "kernels.cuh"

namespace ign {
KernelSet kernel_set_7() { return Launch<7>::make(); }
}  // namespace ign
