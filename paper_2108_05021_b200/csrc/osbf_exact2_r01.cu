// Exact-mode kernels for radius 1 (explicit instantiations): the fused strip
// kernel (osbf_exact2_kernel.cuh) and the table-path stencil walk
// (osbf_exact_twalk.cuh).
#include "osbf_exact2_kernel.cuh"
#include "osbf_exact_twalk.cuh"

namespace osbf_gpu {
template cudaError_t exact2_launch_radius<1>(const PlaneView&, const Geometry&, double*, int,
                                              double*, size_t, size_t, int, double*,
                                              cudaStream_t);
template cudaError_t exact_twalk_launch<1>(const PlaneView&, const Geometry&, const double*,
                                           size_t, double*, size_t, size_t, const unsigned*,
                                           cudaStream_t);
}  // namespace osbf_gpu
