// Internal declarations shared by the OSBF kernels and the C ABI layer.
// Not installed; the public surface is include/osbf_gpu.h.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <stddef.h>
#include <stdint.h>

#include "osbf_gpu.h"

namespace osbf_gpu {

// A batch of planes in device memory: sample(b,x,y) = base[b*plane + y*pitch + x].
struct PlaneView {
    const void* base;
    osbf_dtype dtype;
    size_t pitch;  // elements
    size_t plane;  // elements
};

struct Geometry {
    int width;
    int height;  // output rows (the image height unless this is a row band)
    int batch;
    // Row-band mode (one band of a taller image, fast mode only): the input
    // buffer holds global rows [in_row0, in_row0 + in_rows), the output
    // buffer global rows [out_row0, out_row0 + height); windows are clipped
    // at the global image height img_height.  Defaults: the whole image.
    int img_height = -1;
    int in_row0 = 0;
    int out_row0 = 0;
    int in_rows = -1;
    // Fused halo push (row bands, fast mode): output rows [out_row0,
    // out_row0 + push_rows) are also stored to push_up (the upper
    // neighbour's bottom halo rows, pitch push_pitch) and rows
    // [out_row0 + height - push_rows, out_row0 + height) to push_dn (the
    // lower neighbour's top halo).  The pointers may be peer (NVLink) memory.
    double* push_up = nullptr;
    double* push_dn = nullptr;
    int push_rows = 0;
    size_t push_pitch = 0;
    int img_h() const { return img_height < 0 ? height : img_height; }
    int in_h() const { return in_rows < 0 ? height : in_rows; }
};

// cudaFuncSetAttribute is per device: `done` remembers, per call site, on
// which devices (bit = ordinal) a kernel's dynamic shared-memory limit has
// been raised, so contexts on several GPUs of one process all get it.
template <typename F>
inline cudaError_t ensure_smem(F* fn, size_t bytes, std::atomic<unsigned long long>& done) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const unsigned long long bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(bytes));
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
    return e;
}

// Name of the kernel family the last pass of this host thread launched
// (instrumentation: osbf_gpu_last_kernel, bench labels).  Set by each
// launcher just before its launch; a static string.
void note_kernel(const char* name);

// Process-wide override of the fast-pass kernel family (osbf_gpu_set_fast_kernel,
// diagnostics / A-B tests); null = none.
const char* fast_kernel_override();

// Process-wide override of the exact-pass kernel family
// (osbf_gpu_set_exact_kernel / OSBF_GPU_EXACT: "strip", "twalk", "gwalk",
// "stencil"); null = none.  Every family is bit-identical.
const char* exact_kernel_override();

// Launch statistics (kernels issued) for instrumentation.
struct LaunchCounter {
    uint64_t launches = 0;
};

// ---- exact mode (osbf_exact.cu) ------------------------------------------
// Whole-image summed-area table in the reference's serial order.
//   rowpfx: fp64 [batch][height][width] workspace (row running sums)
//   sat   : fp64 [batch][height+1][width+1]
//   tpitch: table row pitch in doubles (0 = width+1; the osbf pass path uses
//           an even pitch so the stencil walk can stage table rows with TMA)
//   table_flag: the caller's "table leaves the exact division's range" word
//           (device memory, cleared and set by the build, read by
//           exact_select); null = a sticky per-device word shared by all callers
cudaError_t exact_build_sat(const PlaneView& in, const Geometry& g, double* rowpfx, double* sat,
                            cudaStream_t s, LaunchCounter& lc, size_t tpitch = 0,
                            unsigned* table_flag = nullptr);
// One exact OSBF pass reading `in` and the SAT built from it.
//   out   : fp64 (nullable), out_pitch / out_plane in elements
//   means : fp64 [batch][height][width][8] (nullable)
//   sel   : uint8 [batch][height][width] (nullable)
cudaError_t exact_select(const PlaneView& in, const Geometry& g, int radius, const double* sat,
                         double* out, size_t out_pitch, size_t out_plane, double* means,
                         uint8_t* sel, cudaStream_t s, LaunchCounter& lc, size_t tpitch = 0,
                         const unsigned* table_flag = nullptr);

// Table-path stencil as a TMA-staged column walk (osbf_exact_twalk.cuh,
// instantiated per radius in osbf_exact2_rNN.cu); cudaErrorNotSupported
// (nothing launched) when the table / input layout is not TMA-able.
template <int R>
cudaError_t exact_twalk_launch(const PlaneView& in, const Geometry& g, const double* sat,
                               size_t tpitch, double* out, size_t op, size_t opl,
                               const unsigned* unsafe_flag, cudaStream_t s);

// Fused exact path (osbf_exact2_kernel.cuh): row carries + strip kernel.
// Bit-identical to exact_build_sat + exact_select; radius <= kExactFusedMaxRadius.
constexpr int kExactFusedMaxRadius = 16;
size_t exact_fused_carry_elems(const Geometry& g);
cudaError_t exact_fused_step(const PlaneView& in, const Geometry& g, int radius, double* carries,
                             double* out, size_t out_pitch, size_t out_plane, cudaStream_t s,
                             LaunchCounter& lc);

// ---- paper Algorithm 3 (osbf_fastosbf.cu) ----------------------------------
// One fast_osbf iteration (filters2d.hpp:105-154), bit-identical: exact SAT
// into rowpfx/sat (rowpfx: [batch][height][width], reused for the quarter
// field), then quarter means and the candidate selection into out.
cudaError_t fastosbf_pass(const PlaneView& in, const Geometry& g, int radius, double* rowpfx,
                          double* sat, double* out, size_t out_pitch, size_t out_plane,
                          cudaStream_t s, LaunchCounter& lc);

// One box_filter iteration (filters2d.hpp:38-56), bit-identical: exact SAT,
// then the valid-count mean of the clipped (2r+1)^2 window into out.
cudaError_t boxfilter_pass(const PlaneView& in, const Geometry& g, int radius, double* rowpfx,
                           double* sat, double* out, size_t out_pitch, size_t out_plane,
                           cudaStream_t s, LaunchCounter& lc);

// ---- 3-D extension (osbf_3d.cu) -------------------------------------------
// One osbf_3d / box_filter_3d iteration on an fp64 volume [D][H][W]:
// rowp W*H*D and table svt_elems(W, H, D) doubles of workspace.
size_t svt_elems(int W, int H, int D);
cudaError_t svt_build(const double* in, int W, int H, int D, double* rowp, double* table,
                      cudaStream_t s, LaunchCounter& lc);
cudaError_t filter3d_pass(const double* in, int W, int H, int D, int r, bool osbf,
                          double* rowp, double* table, double* out, cudaStream_t s,
                          LaunchCounter& lc);

// ---- smooth edge (osbf_edge.cu) --------------------------------------------
// Interleaved uint8/uint16 raster (sample_bytes 1/2) -> channel planes
// [channels][pixels] (uint8 planes for 8-bit samples, fp64 for 16-bit);
// fp64 planes -> raster, quantised like io.hpp:108-115 with maxval 255 / 65535.
cudaError_t raster_to_planes(const void* raster, int sample_bytes, int channels, size_t pixels,
                             void* planes, cudaStream_t s, LaunchCounter& lc);
cudaError_t planes_to_raster(const double* planes, int channels, size_t pixels, void* raster,
                             int sample_bytes, cudaStream_t s, LaunchCounter& lc);

// ---- fast mode (osbf_fast.cu) --------------------------------------------
// Largest radius with a compiled fast-mode kernel (64x64 tile + halo in smem).
constexpr int kFastMaxRadius = 16;
// One OSBF pass with tile-local fp64 summed-area tables.
cudaError_t fast_step(const PlaneView& in, const Geometry& g, int radius, double* out,
                      size_t out_pitch, size_t out_plane, double* means, uint8_t* sel,
                      cudaStream_t s, LaunchCounter& lc);

// One fast pass for kFastMaxRadius < radius <= fast_generic_max_radius():
// the vertical-first column walk (osbf_fast_vwalk.cu), O(1) state per thread
// in r.  cudaErrorNotSupported (nothing launched) when the layout or radius
// has no kernel.
cudaError_t fast_generic_step(const PlaneView& in, const Geometry& g, int radius, double* out,
                              size_t out_pitch, size_t out_plane, cudaStream_t s,
                              LaunchCounter& lc);
int fast_generic_max_radius();
// k = 2..4 fast passes in one launch (temporal blocking, radius <= 4).
// Returns cudaErrorNotSupported (nothing launched) when the radius / layout /
// k has no multi-pass kernel; the caller then runs fewer passes per launch.
cudaError_t fast_stepk(const PlaneView& in, const Geometry& g, int radius, int k, double* out,
                       size_t out_pitch, size_t out_plane, cudaStream_t s, LaunchCounter& lc);

// ---- utilities (osbf_capi.cu) ----------------------------------------------
cudaError_t convert_to_f64(const PlaneView& in, const Geometry& g, double* out, size_t out_pitch,
                           size_t out_plane, cudaStream_t s, LaunchCounter& lc);

}  // namespace osbf_gpu

// Device helpers -----------------------------------------------------------
#ifdef __CUDACC__
namespace osbf_gpu {

template <typename T>
__device__ __forceinline__ double to_f64(T v) {
    return static_cast<double>(v);  // exact for u8, f32, f64
}

// Reference window table (core.hpp:212-225) in selection order.
// u = column offset, v = row offset; +v is the next row in memory.
struct Win {
    int u0, u1, v0, v1;
};
__device__ __forceinline__ Win window(int i, int r) {
    switch (i) {
        case 0: return {-r, 0, 0, r};
        case 1: return {0, r, 0, r};
        case 2: return {0, r, -r, 0};
        case 3: return {-r, 0, -r, 0};
        case 4: return {-r, 0, -r, r};
        case 5: return {0, r, -r, r};
        case 6: return {-r, r, 0, r};
        default: return {-r, r, -r, 0};
    }
}

}  // namespace osbf_gpu
#endif
