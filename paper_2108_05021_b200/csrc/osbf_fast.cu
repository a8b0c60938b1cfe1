// Fast mode: one OSBF pass with tile-local fp64 summed-area tables.
//
// Each CTA owns a TW x TH output tile.  It stages the tile plus an r-pixel
// halo in shared memory (zero outside the image, so clipped window sums are
// plain 4-corner differences), builds a tile-local inclusive SAT in fp64, and
// evaluates the eight one-sided windows of the reference (core.hpp:212-225)
// with valid-count means (integral.hpp:53-69) and the strict-< first-minimum
// selection (filters2d.hpp:72-82), writing the selected mean a_m
// (filters2d.hpp:80-83).  Window sums never touch a whole-image prefix, so
// magnitudes stay tile-sized on arbitrarily large images.
#include "osbf_internal.cuh"

namespace osbf_gpu {
namespace {

constexpr int TW = 32;   // output tile width
constexpr int TH = 32;   // output tile height
constexpr int NT = 256;  // threads per CTA

template <typename T>
__global__ void __launch_bounds__(NT)
    fast_tile_step(const T* __restrict__ in, size_t in_pitch, size_t in_plane,
                   double* __restrict__ out, size_t out_pitch, size_t out_plane,
                   double* __restrict__ means, uint8_t* __restrict__ sel, int W, int H, int r) {
    extern __shared__ double S[];
    const int LW = TW + 2 * r, LH = TH + 2 * r;
    const int SP = LW + 1;  // SAT pitch (odd -> conflict-free column walks)
    const int X0 = blockIdx.x * TW, Y0 = blockIdx.y * TH, b = blockIdx.z;
    const int gx0 = X0 - r, gy0 = Y0 - r;
    const T* src = in + static_cast<size_t>(b) * in_plane;
    const int tid = threadIdx.x;

    for (int i = tid; i < SP; i += NT) S[i] = 0.0;
    for (int j = tid; j < LH; j += NT) S[(j + 1) * SP] = 0.0;
    for (int idx = tid; idx < LW * LH; idx += NT) {
        const int j = idx / LW, i = idx - j * LW;
        const int gx = gx0 + i, gy = gy0 + j;
        double v = 0.0;
        if (gx >= 0 && gx < W && gy >= 0 && gy < H)
            v = to_f64(src[static_cast<size_t>(gy) * in_pitch + gx]);
        S[(j + 1) * SP + i + 1] = v;
    }
    __syncthreads();
    for (int j = tid; j < LH; j += NT) {
        double* row = S + (j + 1) * SP + 1;
        double acc = 0.0;
        for (int i = 0; i < LW; ++i) {
            acc += row[i];
            row[i] = acc;
        }
    }
    __syncthreads();
    for (int i = tid; i < LW; i += NT) {
        double acc = 0.0;
        for (int j = 1; j <= LH; ++j) {
            acc += S[j * SP + i + 1];
            S[j * SP + i + 1] = acc;
        }
    }
    __syncthreads();

    const int tx = tid & 31;
    for (int ty = tid >> 5; ty < TH; ty += NT / 32) {
        const int x = X0 + tx, y = Y0 + ty;
        if (x >= W || y >= H) continue;
        // The centre sample comes from global memory (exact); the SAT only
        // holds sums.
        const double uc = to_f64(src[static_cast<size_t>(y) * in_pitch + x]);
        double best = 0.0;
        double best_abs = __longlong_as_double(0x7ff0000000000000LL);
        int best_id = 0;
        const size_t pix = (static_cast<size_t>(b) * H + y) * W + x;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const Win w = window(i, r);
            const int cx0 = max(x + w.u0, 0), cx1 = min(x + w.u1, W - 1);
            const int cy0 = max(y + w.v0, 0), cy1 = min(y + w.v1, H - 1);
            const int n = (cx1 - cx0 + 1) * (cy1 - cy0 + 1);
            const int i0 = cx0 - gx0, i1 = cx1 - gx0 + 1;
            const int j0 = cy0 - gy0, j1 = cy1 - gy0 + 1;
            const double s = S[j1 * SP + i1] - S[j1 * SP + i0] - S[j0 * SP + i1] + S[j0 * SP + i0];
            const double a = __ddiv_rn(s, static_cast<double>(n));
            if (means) means[pix * 8 + i] = a;
            const double d = fabs(a - uc);
            if (d < best_abs) {
                best_abs = d;
                best = a;
                best_id = i + 1;
            }
        }
        if (out) out[static_cast<size_t>(b) * out_plane + static_cast<size_t>(y) * out_pitch + x] = best;
        if (sel) sel[pix] = static_cast<uint8_t>(best_id);
    }
}

template <typename T>
cudaError_t launch(const PlaneView& in, const Geometry& g, int r, double* out, size_t op,
                   size_t opl, double* means, uint8_t* sel, cudaStream_t s) {
    const size_t smem = sizeof(double) * static_cast<size_t>(TW + 2 * r + 1) * (TH + 2 * r + 1);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(fast_tile_step<T>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    dim3 grid((g.width + TW - 1) / TW, (g.height + TH - 1) / TH, g.batch);
    fast_tile_step<T><<<grid, NT, smem, s>>>(static_cast<const T*>(in.base), in.pitch, in.plane,
                                             out, op, opl, means, sel, g.width, g.height, r);
    return cudaGetLastError();
}

}  // namespace

cudaError_t fast_step(const PlaneView& in, const Geometry& g, int radius, double* out,
                      size_t out_pitch, size_t out_plane, double* means, uint8_t* sel,
                      cudaStream_t s, LaunchCounter& lc) {
    ++lc.launches;
    switch (in.dtype) {
        case OSBF_U8:
            return launch<uint8_t>(in, g, radius, out, out_pitch, out_plane, means, sel, s);
        case OSBF_F32:
            return launch<float>(in, g, radius, out, out_pitch, out_plane, means, sel, s);
        default:
            return launch<double>(in, g, radius, out, out_pitch, out_plane, means, sel, s);
    }
}

}  // namespace osbf_gpu
