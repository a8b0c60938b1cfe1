// Standalone TMA probe: load one 68x68 f32 box at (-2,-2) and copy it out.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_2108_05021_b200/csrc/osbf_tma.cuh"
#include <cudaTypedefs.h>
using namespace osbf_gpu;
namespace osbf_gpu { namespace tma {
bool encode_3d(CUtensorMap* map, CUtensorMapDataType dtype, const void* base, uint64_t width,
               uint64_t height, uint64_t planes, uint64_t pitch_bytes, uint64_t plane_bytes,
               uint32_t box_w, uint32_t box_h) {
    void* p = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    const cuuint64_t dims[3] = {width, height, planes};
    const cuuint64_t strides[2] = {pitch_bytes, plane_bytes};
    const cuuint32_t box[3] = {box_w, box_h, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(map, dtype, 3, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode -> %d\n", (int)r);
    return r == CUDA_SUCCESS;
}}}
__device__ __forceinline__ void init_v(uint64_t* bar, int v) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(tma::smem_u32(bar)), "r"(1));
    if (v & 1) asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    if (v & 2) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void load_v(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar, int v) {
    if (v & 4)
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(tma::smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(tma::smem_u32(bar)) : "memory");
    else
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(tma::smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(tma::smem_u32(bar)) : "memory");
}
template <int MODE>
__global__ void k(const __grid_constant__ CUtensorMap tmap, float* out, int v, int c) {
    extern __shared__ unsigned char smem_raw[];
    __shared__ uint64_t bar;
    const uint32_t base = tma::smem_u32(smem_raw);
    float* Us = reinterpret_cast<float*>(smem_raw + ((128u - (base & 127u)) & 127u));
    if (threadIdx.x == 0) init_v(&bar, v);
    __syncthreads();
    if (threadIdx.x == 0) {
        tma::mbar_arrive_expect_tx(&bar, 68 * 68 * 4);
        load_v(Us, &tmap, c, c, 0, &bar, v);
    }
    tma::mbar_wait(&bar, 0);
    for (int i = threadIdx.x; i < 68 * 68; i += blockDim.x) out[i] = Us[i];
}
int main(int argc, char** argv) {
    std::vector<float> h(128 * 128);
    for (int i = 0; i < 128 * 128; ++i) h[i] = (float)i;
    float *d, *o;
    cudaMalloc(&d, h.size() * 4); cudaMalloc(&o, 68 * 68 * 4);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    CUtensorMap map;
    tma::encode_3d(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, d, 128, 128, 1, 512, 65536, 68, 68);
    int v = argc > 1 ? atoi(argv[1]) : 0, c = argc > 2 ? atoi(argv[2]) : -2;
    k<0><<<1, 256, 68 * 68 * 4 + 128>>>(map, o, v, c);
    cudaError_t e = cudaDeviceSynchronize();
    printf("v=%d c=%d kernel -> %s\n", v, c, cudaGetErrorString(e));
    std::vector<float> r(68 * 68);
    cudaMemcpy(r.data(), o, r.size() * 4, cudaMemcpyDeviceToHost);
    printf("r[0]=%g r[2*68+2]=%g (expect 0 and 0) r[3*68+3]=%g (expect %g)\n", r[0], r[2 * 68 + 2], r[3 * 68 + 3], (float)(1 * 128 + 1));
    return 0;
}
