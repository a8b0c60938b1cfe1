// 3-D extension: osbf_3d and box_filter_3d
// (filters3d.hpp:55-114) on a single fp64 volume, bit-identical.
//
// The summed-volume table (integral.hpp:98-113) is replayed in the
// reference's order: a running row sum over x per (y, z) row, and
//   T(x+1,y+1,z+1) = ((row + T(x+1,y,z+1)) + T(x+1,y+1,z)) - T(x+1,y,z)
// which, for a fixed column x, depends only on earlier (z, y) of the same
// column: one thread per column walks z then y (columns in parallel, loads
// coalesced across a warp).  The filter kernel evaluates per voxel the 8
// (box: 1) clipped box sums with the reference's inclusion-exclusion order,
// IEEE division by the clipped count, |a - u| and the strict-< first minimum
// over the 14 regions in filters3d.hpp:29-51 order.
#include "osbf_internal.cuh"

namespace osbf_gpu {
namespace {

__global__ void __launch_bounds__(128)
    svt_rows(const double* __restrict__ in, double* __restrict__ rowp, int W, long long rows) {
    const long long row = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (row >= rows) return;
    const double* src = in + row * W;
    double* dst = rowp + row * W;
    double acc = 0.0;
    for (int x = 0; x < W; ++x) {
        acc = __dadd_rn(acc, src[x]);  // row += vol(x, y, z)
        dst[x] = acc;
    }
}

__global__ void __launch_bounds__(128)
    svt_columns(const double* __restrict__ rowp, double* __restrict__ T, int W, int H, int D) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= W) return;
    const size_t W1 = static_cast<size_t>(W) + 1, H1 = static_cast<size_t>(H) + 1;
    auto at = [&](int xx, int yy, int zz) -> double& {
        return T[(static_cast<size_t>(zz) * H1 + yy) * W1 + xx];
    };
    for (int z = 0; z < D; ++z)
        for (int y = 0; y < H; ++y) {
            const double row = rowp[(static_cast<size_t>(z) * H + y) * W + x];
            at(x + 1, y + 1, z + 1) = __dsub_rn(
                __dadd_rn(__dadd_rn(row, at(x + 1, y, z + 1)), at(x + 1, y + 1, z)),
                at(x + 1, y, z));
        }
}

// integral.hpp:121-160: clipped box mean; regions here always contain the
// centre voxel, so the clipped box is never empty.
__device__ __forceinline__ double box_mean3(const double* __restrict__ T, int W, int H, int D,
                                            int x0, int y0, int z0, int x1, int y1, int z1) {
    const size_t W1 = static_cast<size_t>(W) + 1, H1 = static_cast<size_t>(H) + 1;
    x0 = max(x0, 0); y0 = max(y0, 0); z0 = max(z0, 0);
    x1 = min(x1, W - 1); y1 = min(y1, H - 1); z1 = min(z1, D - 1);
    const int ax = x0, bx = x1 + 1, ay = y0, by = y1 + 1, az = z0, bz = z1 + 1;
    auto c = [&](int xx, int yy, int zz) {
        return T[(static_cast<size_t>(zz) * H1 + yy) * W1 + xx];
    };
    double s = __dsub_rn(c(bx, by, bz), c(ax, by, bz));
    s = __dsub_rn(s, c(bx, ay, bz));
    s = __dsub_rn(s, c(bx, by, az));
    s = __dadd_rn(s, c(ax, ay, bz));
    s = __dadd_rn(s, c(ax, by, az));
    s = __dadd_rn(s, c(bx, ay, az));
    s = __dsub_rn(s, c(ax, ay, az));
    const long long n = static_cast<long long>(x1 - x0 + 1) * (y1 - y0 + 1) * (z1 - z0 + 1);
    return __ddiv_rn(s, static_cast<double>(n));
}

template <bool OSBF>
__global__ void __launch_bounds__(256)
    filter3d(const double* __restrict__ in, const double* __restrict__ T, double* __restrict__ out,
             int W, int H, int D, int r) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<long long>(W) * H * D) return;
    const int x = static_cast<int>(i % W);
    const int y = static_cast<int>((i / W) % H);
    const int z = static_cast<int>(i / (static_cast<long long>(W) * H));
    if (!OSBF) {
        out[i] = box_mean3(T, W, H, D, x - r, y - r, z - r, x + r, y + r, z + r);
        return;
    }
    const double u = in[i];
    double best = 0.0, best_abs = __longlong_as_double(0x7ff0000000000000LL);  // +inf
#pragma unroll
    for (int k = 0; k < 14; ++k) {
        int u0, u1, v0, v1, w0, w1;
        if (k < 8) {  // octants by sign pattern (x fastest), filters3d.hpp:36-45
            const int sx = k & 1, sy = (k >> 1) & 1, sz = k >> 2;
            u0 = sx ? 0 : -r; u1 = sx ? r : 0;
            v0 = sy ? 0 : -r; v1 = sy ? r : 0;
            w0 = sz ? 0 : -r; w1 = sz ? r : 0;
        } else {  // half windows -x, +x, -y, +y, -z, +z, filters3d.hpp:46-51
            const int h = k - 8, axis = h >> 1, pos = h & 1;
            u0 = -r; u1 = r; v0 = -r; v1 = r; w0 = -r; w1 = r;
            if (axis == 0) { u0 = pos ? 0 : -r; u1 = pos ? r : 0; }
            if (axis == 1) { v0 = pos ? 0 : -r; v1 = pos ? r : 0; }
            if (axis == 2) { w0 = pos ? 0 : -r; w1 = pos ? r : 0; }
        }
        const double a = box_mean3(T, W, H, D, x + u0, y + v0, z + w0, x + u1, y + v1, z + w1);
        const double dist = fabs(__dsub_rn(a, u));
        if (dist < best_abs) {
            best_abs = dist;
            best = a;
        }
    }
    out[i] = best;
}

}  // namespace

size_t svt_elems(int W, int H, int D) {
    return (static_cast<size_t>(W) + 1) * (static_cast<size_t>(H) + 1) * (static_cast<size_t>(D) + 1);
}

cudaError_t svt_build(const double* in, int W, int H, int D, double* rowp, double* table,
                      cudaStream_t s, LaunchCounter& lc) {
    const long long rows = static_cast<long long>(H) * D;
    cudaError_t e = cudaMemsetAsync(table, 0, sizeof(double) * svt_elems(W, H, D), s);
    if (e != cudaSuccess) return e;
    svt_rows<<<static_cast<unsigned>((rows + 127) / 128), 128, 0, s>>>(in, rowp, W, rows);
    svt_columns<<<(W + 127) / 128, 128, 0, s>>>(rowp, table, W, H, D);
    lc.launches += 2;
    return cudaGetLastError();
}

cudaError_t filter3d_pass(const double* in, int W, int H, int D, int r, bool osbf,
                          double* rowp, double* table, double* out, cudaStream_t s,
                          LaunchCounter& lc) {
    cudaError_t e = svt_build(in, W, H, D, rowp, table, s, lc);
    if (e != cudaSuccess) return e;
    const long long n = static_cast<long long>(W) * H * D;
    const unsigned blocks = static_cast<unsigned>((n + 255) / 256);
    if (osbf)
        filter3d<true><<<blocks, 256, 0, s>>>(in, table, out, W, H, D, r);
    else
        filter3d<false><<<blocks, 256, 0, s>>>(in, table, out, W, H, D, r);
    lc.launches += 1;
    return cudaGetLastError();
}

}  // namespace osbf_gpu
