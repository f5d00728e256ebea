// Explicit instantiation of the 3D stage kernels for ns = 2 species.
#include "kernels.cuh"
#include "kernels3d.cuh"

namespace ign {
KernelSet kernel_set3_2() { return Launch3<2>::make(); }
}  // namespace ign
