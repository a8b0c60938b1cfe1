// The `osbf smooth` edge (tools/osbf_main.cpp:63-83):
// read_image promotes decoded PGM/PPM samples to fp64 planes
// (io.hpp:122-178), filter_multichannel filters each channel, write_image
// quantises every sample (io.hpp:187-215, quantize io.hpp:108-115: round
// half up, negatives and NaN to 0, clamp to maxval) and interleaves them.
// On the GPU the raster crosses PCIe as 1-2 B per sample: raster_promote
// de-interleaves it on the device (8-bit planes stay uint8 and are promoted
// inside the first filter pass, OSBF_U8 — which is also what keeps fast
// mode's first pass bit-exact; 16-bit samples are widened to fp64 here),
// raster_quantize rounds, clamps and re-interleaves the filtered planes.  Both are streaming HBM kernels
// (grid-stride, a multiple of the SM count).
#include "osbf_internal.cuh"

namespace osbf_gpu {
namespace {

// De-interleave into channel planes of type P (uint8 planes stay uint8: the
// first filter pass promotes them; uint16 samples are widened to fp64 here).
template <typename T, typename P>
__global__ void __launch_bounds__(256)
    raster_promote(const T* __restrict__ raster, P* __restrict__ planes, int channels,
                   size_t pixels) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < pixels;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        for (int c = 0; c < channels; ++c)
            planes[c * pixels + i] = static_cast<P>(raster[i * channels + c]);
}

// io.hpp:108-115
__device__ __forceinline__ int quantize(double v, int maxval) {
    const double q = floor(__dadd_rn(v, 0.5));  // round half up
    if (!(q > 0.0)) return 0;                   // negatives and NaN clamp to 0
    if (q > maxval) return maxval;
    return static_cast<int>(q);
}

template <typename T>
__global__ void __launch_bounds__(256)
    raster_quantize(const double* __restrict__ planes, T* __restrict__ raster, int channels,
                    size_t pixels, int maxval) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < pixels;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        for (int c = 0; c < channels; ++c)
            raster[i * channels + c] = static_cast<T>(quantize(planes[c * pixels + i], maxval));
}

unsigned stream_grid(size_t pixels) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t want = (pixels + 255) / 256;
    return static_cast<unsigned>(std::max<size_t>(1, std::min<size_t>(want, 8ull * sms)));
}

}  // namespace

cudaError_t raster_to_planes(const void* raster, int sample_bytes, int channels, size_t pixels,
                             void* planes, cudaStream_t s, LaunchCounter& lc) {
    if (sample_bytes == 1)
        raster_promote<uint8_t, uint8_t><<<stream_grid(pixels), 256, 0, s>>>(
            static_cast<const uint8_t*>(raster), static_cast<uint8_t*>(planes), channels, pixels);
    else
        raster_promote<uint16_t, double><<<stream_grid(pixels), 256, 0, s>>>(
            static_cast<const uint16_t*>(raster), static_cast<double*>(planes), channels, pixels);
    lc.launches += 1;
    return cudaGetLastError();
}

cudaError_t planes_to_raster(const double* planes, int channels, size_t pixels, void* raster,
                             int sample_bytes, cudaStream_t s, LaunchCounter& lc) {
    if (sample_bytes == 1)
        raster_quantize<uint8_t><<<stream_grid(pixels), 256, 0, s>>>(
            planes, static_cast<uint8_t*>(raster), channels, pixels, 255);
    else
        raster_quantize<uint16_t><<<stream_grid(pixels), 256, 0, s>>>(
            planes, static_cast<uint16_t*>(raster), channels, pixels, 65535);
    lc.launches += 1;
    return cudaGetLastError();
}

}  // namespace osbf_gpu
