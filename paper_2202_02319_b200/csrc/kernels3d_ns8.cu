// Explicit instantiation of the 3D stage kernels for ns = 8 species.
#include "kernels.cuh"
#include "kernels3d.cuh"

namespace ign {
KernelSet kernel_set3_8() { return Launch3<8>::make(); }
}  // namespace ign
