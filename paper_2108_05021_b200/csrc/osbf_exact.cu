// Exact mode: bit-identical replay of the reference OSBF pass.
//
// The reference (integral.hpp:16-30) builds ONE whole-image fp64 summed-area
// table with a serial left-to-right running row sum, adding the table row
// above:  C(x+1,y+1) = C(x+1,y) + R(x,y),  R(x,y) = R(x-1,y) + U(x,y).
// Every later rounding depends on that order, and the selection's strict-<
// tie-break (filters2d.hpp:72-82) decides exact ties through that rounding
// noise, so this mode reproduces the order exactly:
//   K1 exact_row_prefix : R, one serial fp64 chain per row (H*B chains),
//                         coalesced through a per-warp shared-memory transpose;
//   K2 exact_col_chain  : C, one serial fp64 chain per table column;
//   K3 exact_stencil    : per pixel, 8 clipped ((A-B)-C)+D sums
//                         (integral.hpp:48-49), IEEE division by the valid
//                         count (integral.hpp:68), |a-u|, strict < in window
//                         order, write a_m itself (filters2d.hpp:80-83).
// All fp64 arithmetic uses the _rn intrinsics so nothing is contracted.
#include "osbf_exact2_kernel.cuh"
#include "osbf_internal.cuh"

namespace osbf_gpu {
namespace {

constexpr int kRowWarps = 4;   // warps per CTA in K1
constexpr int kChunk = 32;     // columns per transpose chunk

template <typename T>
__global__ void __launch_bounds__(kRowWarps * 32)
    exact_row_prefix(const T* __restrict__ in, size_t in_pitch, size_t in_plane,
                     double* __restrict__ rowpfx, int W, int H, long long total_rows) {
    __shared__ double tile[kRowWarps][kChunk][kChunk + 1];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const long long row0 = (static_cast<long long>(blockIdx.x) * kRowWarps + warp) * 32;
    if (row0 >= total_rows) return;
    double (*t)[kChunk + 1] = tile[warp];

    // Element offset of row (row0 + lane); broadcast per row inside the loads.
    long long my_base = -1;
    {
        const long long g = row0 + lane;
        if (g < total_rows) {
            const long long b = g / H, y = g - b * H;
            my_base = b * static_cast<long long>(in_plane) + y * static_cast<long long>(in_pitch);
        }
    }
    double acc = 0.0;
    for (int x0 = 0; x0 < W; x0 += kChunk) {
        const int x = x0 + lane;
#pragma unroll 8
        for (int rr = 0; rr < 32; ++rr) {
            const long long base = __shfl_sync(0xffffffffu, my_base, rr);
            double v = 0.0;
            if (base >= 0 && x < W) v = to_f64(in[base + x]);
            t[rr][lane] = v;
        }
        __syncwarp();
        const int n = min(kChunk, W - x0);
        for (int c = 0; c < n; ++c) {
            acc = __dadd_rn(acc, t[lane][c]);  // row += src[x]  (integral.hpp:25)
            t[lane][c] = acc;
        }
        __syncwarp();
#pragma unroll 8
        for (int rr = 0; rr < 32; ++rr) {
            const long long g = row0 + rr;
            if (g < total_rows && x < W) rowpfx[g * W + x] = t[rr][lane];
        }
        __syncwarp();
    }
}

// One thread per table column cx in [0, W] of each plane.
__global__ void exact_col_chain(const double* __restrict__ rowpfx, double* __restrict__ sat,
                                int W, int H, int B) {
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long cols = static_cast<long long>(W) + 1;
    if (t >= cols * B) return;
    const long long b = t / cols;
    const int cx = static_cast<int>(t - b * cols);
    double* C = sat + b * cols * (H + 1);
    C[cx] = 0.0;  // zero border row
    if (cx == 0) {
        for (int cy = 1; cy <= H; ++cy) C[static_cast<long long>(cy) * cols] = 0.0;
        return;
    }
    const double* R = rowpfx + b * static_cast<long long>(W) * H + (cx - 1);
    double acc = 0.0;
#pragma unroll 8
    for (int y = 0; y < H; ++y) {
        acc = __dadd_rn(acc, R[static_cast<long long>(y) * W]);  // above[x+1] + row (integral.hpp:26)
        C[static_cast<long long>(y + 1) * cols + cx] = acc;
    }
}

template <typename T>
__global__ void __launch_bounds__(256)
    exact_stencil(const T* __restrict__ in, size_t in_pitch, size_t in_plane,
                  const double* __restrict__ sat, double* __restrict__ out, size_t out_pitch,
                  size_t out_plane, double* __restrict__ means, uint8_t* __restrict__ sel, int W,
                  int H, int r) {
    const int x = blockIdx.x * 32 + (threadIdx.x & 31);
    const int y = blockIdx.y * 8 + (threadIdx.x >> 5);
    const int b = blockIdx.z;
    if (x >= W || y >= H) return;
    const long long cols = static_cast<long long>(W) + 1;
    const double* C = sat + static_cast<long long>(b) * cols * (H + 1);
    const double u = to_f64(in[b * in_plane + static_cast<size_t>(y) * in_pitch + x]);
    const bool diag = means != nullptr || sel != nullptr;
    if (!diag && x >= r && x + r < W && y >= r && y + r < H) {
        // interior pixel: the 8 windows share a 4x4 grid of table corners,
        // rows {y-r, y, y+1, y+r+1} x columns {x-r, x, x+1, x+r+1}; every sum
        // keeps the reference's ((A-B)-C)+D (integral.hpp:48-49) and the
        // division by the count is IEEE-exact (div_by_count)
        const double* rp[4] = {C + static_cast<long long>(y - r) * cols,
                               C + static_cast<long long>(y) * cols,
                               C + static_cast<long long>(y + 1) * cols,
                               C + static_cast<long long>(y + r + 1) * cols};
        const int co[4] = {x - r, x, x + 1, x + r + 1};
        double g[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int c = 0; c < 4; ++c) g[a][c] = __ldg(rp[a] + co[c]);
        // (ca, cb, ra, rb) per window in reference order (core.hpp:212-225)
        constexpr int W8[8][4] = {{0, 2, 1, 3}, {1, 3, 1, 3}, {1, 3, 0, 2}, {0, 2, 0, 2},
                                  {0, 2, 0, 3}, {1, 3, 0, 3}, {0, 3, 1, 3}, {0, 3, 0, 2}};
        const double nq = static_cast<double>((r + 1) * (r + 1));
        const double nh = static_cast<double>((r + 1) * (2 * r + 1));
        const double yq = __ddiv_rn(1.0, nq), yh = __ddiv_rn(1.0, nh);
        double av[8], dv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int ca = W8[i][0], cb = W8[i][1], ra = W8[i][2], rb = W8[i][3];
            const double sm =
                __dadd_rn(__dsub_rn(__dsub_rn(g[rb][cb], g[rb][ca]), g[ra][cb]), g[ra][ca]);
            av[i] = div_by_count(sm, i < 4 ? nq : nh, i < 4 ? yq : yh);
            dv[i] = fabs(__dsub_rn(av[i], u));
        }
        double best = 0.0;
        const double dsum = ((dv[0] + dv[1]) + (dv[2] + dv[3])) + ((dv[4] + dv[5]) + (dv[6] + dv[7]));
        if (fabs(dsum) < __longlong_as_double(0x7ff0000000000000LL)) {
            // all |a_i - u| finite: a stable depth-3 tournament returns the
            // first minimum, the reference's strict < (filters2d.hpp:78)
            auto pick = [](double& d0, double& a0, double d1, double a1) {
                const bool t = d1 < d0;
                d0 = t ? d1 : d0;
                a0 = t ? a1 : a0;
            };
            pick(dv[0], av[0], dv[1], av[1]);
            pick(dv[2], av[2], dv[3], av[3]);
            pick(dv[4], av[4], dv[5], av[5]);
            pick(dv[6], av[6], dv[7], av[7]);
            pick(dv[0], av[0], dv[2], av[2]);
            pick(dv[4], av[4], dv[6], av[6]);
            pick(dv[0], av[0], dv[4], av[4]);
            best = av[0];
        } else {  // non-finite samples: the sequential rule never selects them
            double best_abs = __longlong_as_double(0x7ff0000000000000LL);
#pragma unroll
            for (int i = 0; i < 8; ++i)
                if (dv[i] < best_abs) {
                    best_abs = dv[i];
                    best = av[i];
                }
        }
        out[b * out_plane + static_cast<size_t>(y) * out_pitch + x] = best;
        return;
    }
    double best = 0.0;
    double best_abs = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    int best_id = 0;
    const size_t pix = (static_cast<size_t>(b) * H + y) * W + x;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const Win w = window(i, r);
        const int x0 = max(x + w.u0, 0), x1 = min(x + w.u1, W - 1);
        const int y0 = max(y + w.v0, 0), y1 = min(y + w.v1, H - 1);
        const long long n = static_cast<long long>(x1 - x0 + 1) * (y1 - y0 + 1);
        const double A = C[(y1 + 1) * cols + (x1 + 1)];
        const double Bv = C[(y1 + 1) * cols + x0];
        const double Cv = C[y0 * cols + (x1 + 1)];
        const double D = C[y0 * cols + x0];
        const double s = __dadd_rn(__dsub_rn(__dsub_rn(A, Bv), Cv), D);
        const double a = __ddiv_rn(s, static_cast<double>(n));
        if (means) means[pix * 8 + i] = a;
        const double d = fabs(__dsub_rn(a, u));
        if (d < best_abs) {
            best_abs = d;
            best = a;
            best_id = i + 1;
        }
    }
    if (out) out[b * out_plane + static_cast<size_t>(y) * out_pitch + x] = best;
    if (sel) sel[pix] = static_cast<uint8_t>(best_id);
}

template <typename T>
cudaError_t launch_row_prefix(const PlaneView& in, const Geometry& g, double* rowpfx,
                              cudaStream_t s) {
    const long long rows = static_cast<long long>(g.batch) * g.height;
    const long long warps = (rows + 31) / 32;
    const unsigned blocks = static_cast<unsigned>((warps + kRowWarps - 1) / kRowWarps);
    exact_row_prefix<T><<<blocks, kRowWarps * 32, 0, s>>>(
        static_cast<const T*>(in.base), in.pitch, in.plane, rowpfx, g.width, g.height, rows);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_stencil(const PlaneView& in, const Geometry& g, int r, const double* sat,
                           double* out, size_t op, size_t opl, double* means, uint8_t* sel,
                           cudaStream_t s) {
    dim3 grid((g.width + 31) / 32, (g.height + 7) / 8, g.batch);
    exact_stencil<T><<<grid, 256, 0, s>>>(static_cast<const T*>(in.base), in.pitch, in.plane, sat,
                                          out, op, opl, means, sel, g.width, g.height, r);
    return cudaGetLastError();
}

}  // namespace

cudaError_t exact_build_sat(const PlaneView& in, const Geometry& g, double* rowpfx, double* sat,
                            cudaStream_t s, LaunchCounter& lc) {
    cudaError_t e;
    switch (in.dtype) {
        case OSBF_U8: e = launch_row_prefix<uint8_t>(in, g, rowpfx, s); break;
        case OSBF_F32: e = launch_row_prefix<float>(in, g, rowpfx, s); break;
        default: e = launch_row_prefix<double>(in, g, rowpfx, s); break;
    }
    ++lc.launches;
    if (e != cudaSuccess) return e;
    const long long threads = (static_cast<long long>(g.width) + 1) * g.batch;
    exact_col_chain<<<static_cast<unsigned>((threads + 127) / 128), 128, 0, s>>>(
        rowpfx, sat, g.width, g.height, g.batch);
    ++lc.launches;
    return cudaGetLastError();
}

cudaError_t exact_select(const PlaneView& in, const Geometry& g, int radius, const double* sat,
                         double* out, size_t out_pitch, size_t out_plane, double* means,
                         uint8_t* sel, cudaStream_t s, LaunchCounter& lc) {
    ++lc.launches;
    note_kernel("exact_row_prefix+exact_col_chain+exact_select");
    switch (in.dtype) {
        case OSBF_U8:
            return launch_stencil<uint8_t>(in, g, radius, sat, out, out_pitch, out_plane, means,
                                           sel, s);
        case OSBF_F32:
            return launch_stencil<float>(in, g, radius, sat, out, out_pitch, out_plane, means, sel,
                                         s);
        default:
            return launch_stencil<double>(in, g, radius, sat, out, out_pitch, out_plane, means,
                                          sel, s);
    }
}

// ---- fused exact path (osbf_exact2_kernel.cuh) ------------------------------

namespace {
using Exact2Fn = cudaError_t (*)(const PlaneView&, const Geometry&, double*, int, double*, size_t,
                                 size_t, int, double*, cudaStream_t);
constexpr Exact2Fn kExact2[kExactFusedMaxRadius + 1] = {
    nullptr,
    exact2_launch_radius<1>,  exact2_launch_radius<2>,  exact2_launch_radius<3>,
    exact2_launch_radius<4>,  exact2_launch_radius<5>,  exact2_launch_radius<6>,
    exact2_launch_radius<7>,  exact2_launch_radius<8>,  exact2_launch_radius<9>,
    exact2_launch_radius<10>, exact2_launch_radius<11>, exact2_launch_radius<12>,
    exact2_launch_radius<13>, exact2_launch_radius<14>, exact2_launch_radius<15>,
    exact2_launch_radius<16>,
};
static_assert(kExactFusedMaxRadius == 16, "update kExact2");

template <typename T>
cudaError_t launch_carries(const PlaneView& in, const Geometry& g, double* carries, int nsc,
                           cudaStream_t s) {
    static std::atomic<unsigned long long> done_k1{0}, done_k1d{0};
    cudaError_t e = ensure_smem(ex2::exact_row_carries<T>, ex2::K1_SMEM, done_k1);
    if (e == cudaSuccess)
        e = ensure_smem(ex2::exact_row_carries<T, 1, ex2::K1D_STAGES>, ex2::K1D_SMEM, done_k1d);
    if (e != cudaSuccess) return e;
    const long long rows = static_cast<long long>(g.batch) * g.height;
    const long long warps = (rows + 31) / 32;
    if (warps <= 2 * 148) {  // about one warp per SM: deep single-warp CTAs
        ex2::exact_row_carries<T, 1, ex2::K1D_STAGES>
            <<<static_cast<unsigned>(warps), 32, ex2::K1D_SMEM, s>>>(
                static_cast<const T*>(in.base), in.pitch, in.plane, carries, g.width, g.height,
                rows, nsc);
        return cudaGetLastError();
    }
    const long long ctas = (rows + ex2::NTK1 - 1) / ex2::NTK1;
    ex2::exact_row_carries<T><<<static_cast<unsigned>(ctas), ex2::NTK1, ex2::K1_SMEM, s>>>(
        static_cast<const T*>(in.base), in.pitch, in.plane, carries, g.width, g.height, rows, nsc);
    return cudaGetLastError();
}
}  // namespace

// Band height for under-occupied launches (few strips x planes): enough
// bands for ~4 CTAs per SM, each at least 128 rows (it re-walks 2 blocks).
int exact_band_height(const Geometry& g) {
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    const long long ctas = static_cast<long long>((g.width + ex2::TW - 1) / ex2::TW) * g.batch;
    const long long want = 4LL * sms;
    if (ctas >= want / 2 || g.height < 4 * 128) return 0;
    long long nb = (want + ctas - 1) / ctas;
    int bh = static_cast<int>((g.height + nb - 1) / nb);
    bh = (bh + ex2::BR - 1) / ex2::BR * ex2::BR;
    return bh < 128 ? 128 : bh;
}

size_t exact_fused_carry_elems(const Geometry& g) {
    const size_t rowc = static_cast<size_t>(g.batch) * g.height * (g.width / ex2::SW + 1);
    const int bh = exact_band_height(g);
    const size_t colc =
        bh > 0 ? static_cast<size_t>(g.batch) * ((g.height + bh - 1) / bh) * (g.width + 1) : 0;
    return rowc + colc;
}

cudaError_t exact_fused_step(const PlaneView& in, const Geometry& g, int radius, double* carries,
                             double* out, size_t out_pitch, size_t out_plane, cudaStream_t s,
                             LaunchCounter& lc) {
    if (radius < 1 || radius > kExactFusedMaxRadius) return cudaErrorInvalidValue;
    note_kernel("exact_row_carries+exact_strip");
    const int nsc = g.width / ex2::SW + 1;
    cudaError_t e;
    switch (in.dtype) {
        case OSBF_U8: e = launch_carries<uint8_t>(in, g, carries, nsc, s); break;
        case OSBF_F32: e = launch_carries<float>(in, g, carries, nsc, s); break;
        default: e = launch_carries<double>(in, g, carries, nsc, s); break;
    }
    ++lc.launches;
    if (e != cudaSuccess) return e;
    const int bh = exact_band_height(g);
    double* ccar = carries + static_cast<size_t>(g.batch) * g.height * nsc;
    lc.launches += bh > 0 ? 2 : 1;
    return kExact2[radius](in, g, carries, nsc, out, out_pitch, out_plane, bh, ccar, s);
}

}  // namespace osbf_gpu
