// Fast mode dispatch: radius -> compiled kernel (osbf_fast_rNN.cu).
// Design notes and the kernel itself: osbf_fast_kernel.cuh.
#include "osbf_internal.cuh"

namespace osbf_gpu {

template <int R>
cudaError_t fast_launch_radius(const PlaneView& in, const Geometry& g, double* out,
                               size_t out_pitch, size_t out_plane, double* means, uint8_t* sel,
                               cudaStream_t s);

namespace {
using LaunchFn = cudaError_t (*)(const PlaneView&, const Geometry&, double*, size_t, size_t,
                                 double*, uint8_t*, cudaStream_t);
constexpr LaunchFn kByRadius[kFastMaxRadius + 1] = {
    nullptr,
    fast_launch_radius<1>,  fast_launch_radius<2>,  fast_launch_radius<3>,
    fast_launch_radius<4>,  fast_launch_radius<5>,  fast_launch_radius<6>,
    fast_launch_radius<7>,  fast_launch_radius<8>,  fast_launch_radius<9>,
    fast_launch_radius<10>, fast_launch_radius<11>, fast_launch_radius<12>,
    fast_launch_radius<13>, fast_launch_radius<14>, fast_launch_radius<15>,
    fast_launch_radius<16>,
};
static_assert(kFastMaxRadius == 16, "update kByRadius");
}  // namespace

cudaError_t fast_step(const PlaneView& in, const Geometry& g, int radius, double* out,
                      size_t out_pitch, size_t out_plane, double* means, uint8_t* sel,
                      cudaStream_t s, LaunchCounter& lc) {
    if (radius < 1 || radius > kFastMaxRadius) return cudaErrorInvalidValue;
    ++lc.launches;
    return kByRadius[radius](in, g, out, out_pitch, out_plane, means, sel, s);
}

}  // namespace osbf_gpu
