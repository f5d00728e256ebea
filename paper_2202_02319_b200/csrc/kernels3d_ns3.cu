// Explicit instantiation of the 3D stage kernels for ns = 3 species.
#include "kernels.cuh"
#include "kernels3d.cuh"

namespace ign {
KernelSet kernel_set3_3() { return Launch3<3>::make(); }
}  // namespace ign
