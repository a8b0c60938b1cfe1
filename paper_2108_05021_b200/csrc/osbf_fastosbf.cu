// Paper Algorithm 3, the reference's fast_osbf (filters2d.hpp:105-154), and
// the classical box filter (filters2d.hpp:38-56), both bit-identical.  Per iteration:
//   1. the whole-image summed-area table in the reference's serial order
//      (exact_build_sat, the same kernels the exact OSBF diagnostics use);
//   2. rect_mean_field: Q(x,y) = rect_mean(x-r, y-r, x, y) (filters2d.hpp:116-
//      119): clipped ((A-B)-C)+D, one IEEE division by the clipped count
//      (integral.hpp:41-69), written over the row-prefix workspace (free once
//      the table exists);
//   3. fosbf_select: the four clamped shifted quarters, the four pairwise
//      averages 0.5*(a+b) in the reference's order, strict-< first minimum of
//      |c - u|, write the candidate (filters2d.hpp:121-147).
// For r <= 64, 2 and 3 run as one kernel (fosbf_fused: the field stays in
// shared memory), so an iteration is the table build plus one pass.
// Every fp64 operation is an _rn intrinsic, so nothing is contracted.
#include <atomic>

#include "osbf_exact2_kernel.cuh"
#include "osbf_internal.cuh"

namespace osbf_gpu {
namespace {

// out(x,y) = rect_mean(x+dx0, y+dy0, x+dx1, y+dy1) on the table (clipped
// ((A-B)-C)+D, one IEEE division by the clipped count, integral.hpp:41-69);
// dx0, dy0 <= 0 <= dx1, dy1, so the clipped rectangle is never empty.
// fast_osbf's quarter field (-r, -r, 0, 0) and box_filter's window
// (-r, -r, r, r, filters2d.hpp:38-56).
__global__ void __launch_bounds__(256)
    rect_mean_field(const double* __restrict__ sat, double* __restrict__ q, size_t q_pitch,
                    size_t q_plane, int W, int H, int dx0, int dy0, int dx1, int dy1) {
    const int x = blockIdx.x * 32 + (threadIdx.x & 31);
    const int y = blockIdx.y * 8 + (threadIdx.x >> 5);
    const int b = blockIdx.z;
    if (x >= W || y >= H) return;
    const long long cols = static_cast<long long>(W) + 1;
    const double* C = sat + static_cast<long long>(b) * cols * (H + 1);
    const int x0 = max(x + dx0, 0), y0 = max(y + dy0, 0);
    const int x1 = min(x + dx1, W - 1), y1 = min(y + dy1, H - 1);
    const long long n = static_cast<long long>(x1 - x0 + 1) * (y1 - y0 + 1);
    const double A = C[(y1 + 1) * cols + (x1 + 1)];
    const double Bv = C[(y1 + 1) * cols + x0];
    const double Cv = C[y0 * cols + (x1 + 1)];
    const double D = C[y0 * cols + x0];
    const double s = __dadd_rn(__dsub_rn(__dsub_rn(A, Bv), Cv), D);
    q[b * q_plane + static_cast<size_t>(y) * q_pitch + x] = __ddiv_rn(s, static_cast<double>(n));
}

template <typename T>
__global__ void __launch_bounds__(256)
    fosbf_select(const T* __restrict__ in, size_t in_pitch, size_t in_plane,
                 const double* __restrict__ q, double* __restrict__ out, size_t out_pitch,
                 size_t out_plane, int W, int H, int r) {
    const int x = blockIdx.x * 32 + (threadIdx.x & 31);
    const int y = blockIdx.y * 8 + (threadIdx.x >> 5);
    const int b = blockIdx.z;
    if (x >= W || y >= H) return;
    const double* Q = q + static_cast<size_t>(b) * H * W;
    const int yr = min(y + r, H - 1), xr = min(x + r, W - 1);
    const double q00 = Q[static_cast<size_t>(y) * W + x];
    const double q10 = Q[static_cast<size_t>(y) * W + xr];
    const double q01 = Q[static_cast<size_t>(yr) * W + x];
    const double q11 = Q[static_cast<size_t>(yr) * W + xr];
    const double cand[8] = {q00,
                            q10,
                            q01,
                            q11,
                            __dmul_rn(0.5, __dadd_rn(q00, q01)),   // left half
                            __dmul_rn(0.5, __dadd_rn(q10, q11)),   // right half
                            __dmul_rn(0.5, __dadd_rn(q00, q10)),   // upper half
                            __dmul_rn(0.5, __dadd_rn(q01, q11))};  // lower half
    const double u = to_f64(in[b * in_plane + static_cast<size_t>(y) * in_pitch + x]);
    double best = cand[0];
    double best_abs = fabs(__dsub_rn(cand[0], u));
#pragma unroll
    for (int i = 1; i < 8; ++i) {
        const double d = fabs(__dsub_rn(cand[i], u));
        if (d < best_abs) {
            best_abs = d;
            best = cand[i];
        }
    }
    out[b * out_plane + static_cast<size_t>(y) * out_pitch + x] = best;
}

// Fused quarter field + selection: one CTA computes the quarter means of its
// 32 x 32 output tile plus the r-column / r-row margin the shifted lookups
// reach (x + r, y + r, clamped) into shared memory -- the same clipped
// ((A-B)-C)+D and IEEE division as rect_mean_field -- then selects from
// there: the field never goes through HBM (two plane passes fewer per
// iteration; bit-identical to the two kernels above).
constexpr int kFosbfMaxRadius = 64;

template <typename T>
__global__ void __launch_bounds__(256)
    fosbf_fused(const T* __restrict__ in, size_t in_pitch, size_t in_plane,
                const double* __restrict__ sat, double* __restrict__ out, size_t out_pitch,
                size_t out_plane, int W, int H, int r, double nq, double yq) {
    extern __shared__ double qs[];
    const int X0 = blockIdx.x * 32, Y0 = blockIdx.y * 32, b = blockIdx.z;
    const int n = 32 + r, pitch = n | 1;
    const long long cols = static_cast<long long>(W) + 1;
    const double* C = sat + static_cast<long long>(b) * cols * (H + 1);
    // quarter means Q(x, y) = rect_mean(x - r, y - r, x, y) (filters2d.hpp:116-119)
    for (int i = threadIdx.x; i < n * n; i += 256) {
        const int ty = i / n, tx = i - ty * n;
        const int x = X0 + tx, y = Y0 + ty;
        if (x >= W || y >= H) continue;
        const int x0 = max(x - r, 0), y0 = max(y - r, 0);
        const long long cnt = static_cast<long long>(x - x0 + 1) * (y - y0 + 1);
        const double A = C[(y + 1) * cols + (x + 1)];
        const double Bv = C[(y + 1) * cols + x0];
        const double Cv = C[y0 * cols + (x + 1)];
        const double D = C[y0 * cols + x0];
        const double sm = __dadd_rn(__dsub_rn(__dsub_rn(A, Bv), Cv), D);
        // interior: the full (r+1)^2 count, divided with the exact 3-op form
        // (div_by_count: the IEEE quotient, guarded for non-normal ranges)
        qs[ty * pitch + tx] = (x0 == x - r && y0 == y - r) ? div_by_count(sm, nq, yq)
                                                             : __ddiv_rn(sm, static_cast<double>(cnt));
    }
    __syncthreads();
    const int x = X0 + (threadIdx.x & 31);
    if (x >= W) return;
    const int xr = min(x + r, W - 1);
#pragma unroll 1
    for (int k = 0; k < 4; ++k) {
        const int y = Y0 + (threadIdx.x >> 5) + 8 * k;
        if (y >= H) return;
        const int yr = min(y + r, H - 1);
        const double q00 = qs[(y - Y0) * pitch + (x - X0)];
        const double q10 = qs[(y - Y0) * pitch + (xr - X0)];
        const double q01 = qs[(yr - Y0) * pitch + (x - X0)];
        const double q11 = qs[(yr - Y0) * pitch + (xr - X0)];
        const double cand[8] = {q00,
                                q10,
                                q01,
                                q11,
                                __dmul_rn(0.5, __dadd_rn(q00, q01)),   // left half
                                __dmul_rn(0.5, __dadd_rn(q10, q11)),   // right half
                                __dmul_rn(0.5, __dadd_rn(q00, q10)),   // upper half
                                __dmul_rn(0.5, __dadd_rn(q01, q11))};  // lower half
        const double u = to_f64(in[b * in_plane + static_cast<size_t>(y) * in_pitch + x]);
        double best = cand[0];
        double best_abs = fabs(__dsub_rn(cand[0], u));
#pragma unroll
        for (int i = 1; i < 8; ++i) {
            const double d = fabs(__dsub_rn(cand[i], u));
            if (d < best_abs) {
                best_abs = d;
                best = cand[i];
            }
        }
        out[b * out_plane + static_cast<size_t>(y) * out_pitch + x] = best;
    }
}

template <typename T>
cudaError_t launch_fosbf_fused(const PlaneView& in, const Geometry& g, int r, const double* sat,
                               double* out, size_t op, size_t opl, cudaStream_t s) {
    static std::atomic<unsigned long long> done{0};
    const int nmax = 32 + kFosbfMaxRadius;
    if (cudaError_t e = ensure_smem(fosbf_fused<T>, sizeof(double) * nmax * (nmax | 1), done))
        return e;
    const int n = 32 + r;
    const dim3 grid((g.width + 31) / 32, (g.height + 31) / 32, g.batch);
    const double nq = static_cast<double>((r + 1) * (r + 1));
    fosbf_fused<T><<<grid, 256, sizeof(double) * n * (n | 1), s>>>(
        static_cast<const T*>(in.base), in.pitch, in.plane, sat, out, op, opl, g.width, g.height,
        r, nq, 1.0 / nq);
    return cudaGetLastError();
}

}  // namespace

cudaError_t fastosbf_pass(const PlaneView& in, const Geometry& g, int radius, double* rowpfx,
                          double* sat, double* out, size_t out_pitch, size_t out_plane,
                          cudaStream_t s, LaunchCounter& lc) {
    cudaError_t e = exact_build_sat(in, g, rowpfx, sat, s, lc);
    if (e != cudaSuccess) return e;
    if (radius <= kFosbfMaxRadius) {
        ++lc.launches;
        switch (in.dtype) {
            case OSBF_U8:
                return launch_fosbf_fused<uint8_t>(in, g, radius, sat, out, out_pitch, out_plane, s);
            case OSBF_F32:
                return launch_fosbf_fused<float>(in, g, radius, sat, out, out_pitch, out_plane, s);
            default:
                return launch_fosbf_fused<double>(in, g, radius, sat, out, out_pitch, out_plane, s);
        }
    }
    const dim3 grid((g.width + 31) / 32, (g.height + 7) / 8, g.batch);
    rect_mean_field<<<grid, 256, 0, s>>>(sat, rowpfx, g.width,
                                         static_cast<size_t>(g.width) * g.height, g.width,
                                         g.height, -radius, -radius, 0, 0);
    ++lc.launches;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    ++lc.launches;
    switch (in.dtype) {
        case OSBF_U8:
            fosbf_select<<<grid, 256, 0, s>>>(static_cast<const uint8_t*>(in.base), in.pitch,
                                              in.plane, rowpfx, out, out_pitch, out_plane,
                                              g.width, g.height, radius);
            break;
        case OSBF_F32:
            fosbf_select<<<grid, 256, 0, s>>>(static_cast<const float*>(in.base), in.pitch,
                                              in.plane, rowpfx, out, out_pitch, out_plane,
                                              g.width, g.height, radius);
            break;
        default:
            fosbf_select<<<grid, 256, 0, s>>>(static_cast<const double*>(in.base), in.pitch,
                                              in.plane, rowpfx, out, out_pitch, out_plane,
                                              g.width, g.height, radius);
            break;
    }
    return cudaGetLastError();
}

cudaError_t boxfilter_pass(const PlaneView& in, const Geometry& g, int radius, double* rowpfx,
                           double* sat, double* out, size_t out_pitch, size_t out_plane,
                           cudaStream_t s, LaunchCounter& lc) {
    cudaError_t e = exact_build_sat(in, g, rowpfx, sat, s, lc);
    if (e != cudaSuccess) return e;
    const dim3 grid((g.width + 31) / 32, (g.height + 7) / 8, g.batch);
    rect_mean_field<<<grid, 256, 0, s>>>(sat, out, out_pitch, out_plane, g.width, g.height,
                                         -radius, -radius, radius, radius);
    ++lc.launches;
    return cudaGetLastError();
}

}  // namespace osbf_gpu
