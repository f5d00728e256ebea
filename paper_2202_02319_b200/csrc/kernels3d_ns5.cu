// Explicit instantiation of the 3D stage kernels for ns = 5 species.
#include "kernels.cuh"
#include "kernels3d.cuh"

namespace ign {
KernelSet kernel_set3_5() { return Launch3<5>::make(); }
}  // namespace ign
