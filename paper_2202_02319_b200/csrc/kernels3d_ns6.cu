// Explicit instantiation of the 3D stage kernels for ns = 6 species.
#include "kernels.cuh"
#include "kernels3d.cuh"

namespace ign {
KernelSet kernel_set3_6() { return Launch3<6>::make(); }
}  // namespace ign
