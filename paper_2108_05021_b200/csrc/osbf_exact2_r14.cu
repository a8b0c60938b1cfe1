// Exact-mode fused strip kernel for radius 14 (explicit instantiation; see osbf_exact2_kernel.cuh).
#include "osbf_exact2_kernel.cuh"

namespace osbf_gpu {
template cudaError_t exact2_launch_radius<14>(const PlaneView&, const Geometry&, double*, int,
                                              double*, size_t, size_t, int, double*,
                                              cudaStream_t);
}  // namespace osbf_gpu
