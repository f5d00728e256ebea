// Explicit instantiation of the 3D stage kernels for ns = 4 species.
#include "kernels.cuh"
#include "kernels3d.cuh"

namespace ign {
KernelSet kernel_set3_4() { return Launch3<4>::make(); }
}  // namespace ign
