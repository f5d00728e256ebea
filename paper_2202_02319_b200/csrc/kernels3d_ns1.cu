// Explicit instantiation of the 3D stage kernels for ns = 1 species.
#include "kernels.cuh"
#include "kernels3d.cuh"

namespace ign {
KernelSet kernel_set3_1() { return Launch3<1>::make(); }
}  // namespace ign
