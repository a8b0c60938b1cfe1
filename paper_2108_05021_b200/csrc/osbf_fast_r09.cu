// Fast-mode kernels for radius 9 (explicit instantiation; see osbf_fast_kernel.cuh).
#include "osbf_fast_kernel.cuh"

namespace osbf_gpu {
template cudaError_t fast_launch_radius<9>(const PlaneView&, const Geometry&, double*, size_t,
                                             size_t, double*, uint8_t*, cudaStream_t);
}  // namespace osbf_gpu
namespace osbf_gpu {
template cudaError_t fast_launch_radiusk<9>(const PlaneView&, const Geometry&, int, double*,
                                              size_t, size_t, cudaStream_t);
}  // namespace osbf_gpu
