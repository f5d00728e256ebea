// Explicit instantiation of the 3D stage kernels for ns = 7 species.
#include "kernels.cuh"
#include "kernels3d.cuh"

namespace ign {
KernelSet kernel_set3_7() { return Launch3<7>::make(); }
}  // namespace ign
