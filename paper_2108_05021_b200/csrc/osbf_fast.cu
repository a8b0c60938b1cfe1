// Fast mode dispatch: radius -> compiled kernel (osbf_fast_rNN.cu).
// Design notes and the kernel itself: osbf_fast_kernel.cuh.
#include <cudaTypedefs.h>

#include <mutex>

#include "osbf_internal.cuh"
#include "osbf_tma.cuh"

namespace osbf_gpu {

namespace tma {
namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}
}  // namespace

bool encode_3d(CUtensorMap* map, CUtensorMapDataType dtype, const void* base, uint64_t width,
               uint64_t height, uint64_t planes, uint64_t pitch_bytes, uint64_t plane_bytes,
               uint32_t box_w, uint32_t box_h) {
    auto fn = encode_fn();
    if (!fn) return false;
    if ((reinterpret_cast<uintptr_t>(base) & 15u) != 0) return false;
    if (pitch_bytes % 16 != 0 || plane_bytes % 16 != 0) return false;
    if (box_w > 256 || box_h > 256) return false;
    const cuuint64_t dims[3] = {width, height, planes};
    const cuuint64_t strides[2] = {pitch_bytes, plane_bytes};
    const cuuint32_t box[3] = {box_w, box_h, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    return fn(map, dtype, 3, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
bool encode_rows_4d(CUtensorMap* map, CUtensorMapDataType dtype, size_t elem_bytes,
                    const void* base, uint64_t width, uint64_t height, uint64_t planes,
                    uint64_t pitch_bytes, uint64_t plane_bytes, uint32_t vec, uint32_t box_groups,
                    uint32_t box_h) {
    auto fn = encode_fn();
    if (!fn || vec == 0 || width % vec != 0) return false;
    if ((reinterpret_cast<uintptr_t>(base) & 15u) != 0) return false;
    if ((vec * elem_bytes) % 16 != 0) return false;
    if (pitch_bytes % 16 != 0 || plane_bytes % 16 != 0) return false;
    if (box_groups > 256 || box_h > 256 || vec > 256) return false;
    const cuuint64_t dims[4] = {vec, width / vec, height, planes};
    const cuuint64_t strides[3] = {vec * elem_bytes, pitch_bytes, plane_bytes};
    const cuuint32_t box[4] = {vec, box_groups, box_h, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    return fn(map, dtype, 4, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace tma

template <int R>
cudaError_t fast_launch_radius(const PlaneView& in, const Geometry& g, double* out,
                               size_t out_pitch, size_t out_plane, double* means, uint8_t* sel,
                               cudaStream_t s);

template <int R>
cudaError_t fast_launch_radiusk(const PlaneView& in, const Geometry& g, int k, double* out,
                                size_t out_pitch, size_t out_plane, cudaStream_t s);

namespace {
using LaunchKFn = cudaError_t (*)(const PlaneView&, const Geometry&, int, double*, size_t,
                                  size_t, cudaStream_t);
constexpr LaunchKFn kByRadiusK[kFastMaxRadius + 1] = {
    nullptr,
    fast_launch_radiusk<1>,  fast_launch_radiusk<2>,  fast_launch_radiusk<3>,
    fast_launch_radiusk<4>,  fast_launch_radiusk<5>,  fast_launch_radiusk<6>,
    fast_launch_radiusk<7>,  fast_launch_radiusk<8>,  fast_launch_radiusk<9>,
    fast_launch_radiusk<10>, fast_launch_radiusk<11>, fast_launch_radiusk<12>,
    fast_launch_radiusk<13>, fast_launch_radiusk<14>, fast_launch_radiusk<15>,
    fast_launch_radiusk<16>,
};
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

cudaError_t fast_stepk(const PlaneView& in, const Geometry& g, int radius, int k, double* out,
                       size_t out_pitch, size_t out_plane, cudaStream_t s, LaunchCounter& lc) {
    if (radius < 1 || radius > kFastMaxRadius) return cudaErrorNotSupported;
    const cudaError_t e = kByRadiusK[radius](in, g, k, out, out_pitch, out_plane, s);
    if (e == cudaSuccess) ++lc.launches;
    return e;
}

}  // namespace osbf_gpu
