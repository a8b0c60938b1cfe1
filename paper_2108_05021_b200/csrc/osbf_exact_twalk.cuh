// Exact mode, whole-table path: the stencil as a column walk over TMA-staged
// table rows (exact_twalk).  Replaces the per-thread global corner loads of
// exact_stencil (osbf_exact.cu) for r <= 16 when the layouts are TMA-able.
//
// Input: the summed-area table of the pass, built in the reference's serial
// order by exact_build_sat (integral.hpp:16-30), row pitch `tpitch` (even, so
// TMA can describe it), and the pass input U.  Output: a_m per pixel,
// bit-identical to exact_stencil (same corner values, same ((A-B)-C)+D
// association, integral.hpp:48-49; the same IEEE-exact division by the count,
// integral.hpp:68; the same first-minimum selection, filters2d.hpp:72-82).
//
// One CTA of 128 threads owns 128 output columns and a block of BH output
// rows and walks down it:
//   * thread 0 streams chunks of CH table rows (columns [X0-R, X0+128+R], from
//     the 16-byte boundary at or left of X0-R: a TMA box must start on one) and
//     the matching CH rows of U (the centre samples of the rows the step
//     outputs) with cp.async.bulk.tensor into a ring of NCR chunk slots, one
//     mbarrier per slot (out-of-image rows / columns are zero-filled and only
//     ever feed skipped or clipped windows);
//   * step c (chunk c landed) outputs the rows whose last table row
//     (y + R + 1) lies in chunk c.  Their corner rows {y-R, y, y+1, y+R+1}
//     sit in chunks c-D..c; each of those chunk's slot base is computed once
//     per step, so every one of the 16 corner loads per pixel is a shared
//     load at a compile-time offset from one of D+1 per-step pointers;
//   * one CTA barrier per step frees chunk c-D's slot for chunk c+1+P.
#pragma once

#include <type_traits>
#include <utility>

#include "osbf_exact2_kernel.cuh"
#include "osbf_internal.cuh"
#include "osbf_tma.cuh"

namespace osbf_gpu {
namespace twk {

template <int R, typename T>
struct TWLay {
    static constexpr int NT = 128;  // threads = output columns per CTA
    static constexpr int SW = 128;
    static constexpr int CH = 8;                          // table rows per chunk
    static constexpr int D = (2 * R + 1 + CH - 1) / CH;   // chunks back a step reads
    static constexpr int P = 1;                           // chunks in flight ahead
    static constexpr int NCR = D + 1 + P;                 // table chunk slots
    static constexpr int NUS = P + 1;                     // U chunk slots
    // the box's first column must sit on a 16-byte boundary: start at X0 - RA
    static constexpr int RA = R + (R & 1);
    static constexpr int XOFF = RA - R;
    static constexpr int BWT = (RA + SW + R + 1 + 1) & ~1;  // table columns per row (even)
    static_assert(BWT <= 256, "TMA box width");
    static constexpr uint32_t T_CHUNK_BYTES = CH * BWT * 8;            // multiple of 128
    static constexpr uint32_t U_CHUNK_BYTES = CH * SW * sizeof(T);     // multiple of 128
    static_assert(T_CHUNK_BYTES % 128 == 0 && U_CHUNK_BYTES % 128 == 0, "slot alignment");
    static constexpr size_t SMEM = 128 + static_cast<size_t>(NCR) * T_CHUNK_BYTES +
                                   static_cast<size_t>(NUS) * U_CHUNK_BYTES;
    // 4 CTAs per SM while the ring fits (r <= 4), then 3 / 2
    static constexpr int MINB = SMEM <= 56 * 1024 ? 4 : (SMEM <= 74 * 1024 ? 3 : 2);
};

// f(integral_constant<int, K>) for K in Ks..., in order (compile-time row index).
template <int... Ks, typename F>
__device__ __forceinline__ void for_each_k(std::integer_sequence<int, Ks...>, F&& f) {
    (f(std::integral_constant<int, Ks>{}), ...);
}

// Clipped / guarded / non-finite pixel: the reference's per-window rule
// (clipped counts, guarded division, sequential strict <), corners looked up
// through the ring.  Out of line: only border pixels and unsafe tables.
template <int R, int RA, int CH, int NCR, int BWT>
__device__ __noinline__ double twalk_general_px(const double* ring, int X0, int ty0, int x, int y,
                                                int W, int H, double u, const double* rcp_tab) {
    double best = 0.0, best_abs = __longlong_as_double(0x7ff0000000000000LL);
    auto row = [&](int cy) {
        const int t = cy - ty0;  // >= 0: windows never reach above the block's first table row
        const int q = (t / CH) % NCR;
        return ring + (static_cast<ptrdiff_t>(q) * CH + (t % CH)) * BWT - (X0 - RA);
    };
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const Win w = window(i, R);
        const int x0 = max(x + w.u0, 0), x1 = min(x + w.u1, W - 1);
        const int y0 = max(y + w.v0, 0), y1 = min(y + w.v1, H - 1);
        const double* ra = row(y0);
        const double* rb = row(y1 + 1);
        const double A = rb[x1 + 1], Bv = rb[x0], Cv = ra[x1 + 1], Dv = ra[x0];
        const double s = __dadd_rn(__dsub_rn(__dsub_rn(A, Bv), Cv), Dv);
        const int ni = (x1 - x0 + 1) * (y1 - y0 + 1);
        const double a = div_by_count(s, static_cast<double>(ni), rcp_tab[ni]);
        const double d = fabs(__dsub_rn(a, u));
        if (d < best_abs) {  // NaN never wins, like the reference's loop
            best_abs = d;
            best = a;
        }
    }
    return best;
}

template <int R, typename T>
__global__ void __launch_bounds__(TWLay<R, T>::NT, TWLay<R, T>::MINB)
    exact_twalk(const __grid_constant__ CUtensorMap tmap_t, const __grid_constant__ CUtensorMap tmap_u,
                double* __restrict__ out, size_t out_pitch, size_t out_plane, int W, int H, int BH,
                const unsigned* __restrict__ unsafe_flag, double yq, double yh) {
    using Ly = TWLay<R, T>;
    constexpr int CH = Ly::CH, D = Ly::D, P = Ly::P, NCR = Ly::NCR, NUS = Ly::NUS, BWT = Ly::BWT;
    extern __shared__ unsigned char smem_raw[];
    __shared__ uint64_t full[NCR];
    __shared__ double rcp_tab[(2 * R + 1) * (R + 1) + 1];
    const uint32_t base = tma::smem_u32(smem_raw);
    unsigned char* sm = smem_raw + ((128u - (base & 127u)) & 127u);
    double* ring = reinterpret_cast<double*>(sm);
    T* uring = reinterpret_cast<T*>(sm + static_cast<size_t>(NCR) * Ly::T_CHUNK_BYTES);
    const int tid = threadIdx.x;
    const int X0 = blockIdx.x * Ly::SW;
    const int Y0 = blockIdx.y * BH;
    const int nout = min(BH, H - Y0);
    const int b = blockIdx.z;
    const int ty0 = Y0 - R;  // table row of ring row 0 of chunk 0
    const int nchunks = (nout + 2 * R + 1 + CH - 1) / CH;

    for (int n = tid; n <= (2 * R + 1) * (R + 1); n += Ly::NT)
        rcp_tab[n] = n ? __ddiv_rn(1.0, static_cast<double>(n)) : 0.0;
    if (tid == 0)
        for (int q = 0; q < NCR; ++q) tma::mbar_init(&full[q], 1);
    __syncthreads();
    auto issue = [&](int c) {  // thread 0: chunk c into slot c % NCR (+ its U rows)
        const int q = c % NCR;
        tma::mbar_arrive_expect_tx(&full[q], Ly::T_CHUNK_BYTES + Ly::U_CHUNK_BYTES);
        tma::load_3d(ring + static_cast<size_t>(q) * CH * BWT, &tmap_t, X0 - Ly::RA, ty0 + c * CH, b,
                     &full[q]);
        tma::load_3d(uring + static_cast<size_t>(c % NUS) * CH * Ly::SW, &tmap_u, X0,
                     Y0 + c * CH - 2 * R - 1, b, &full[q]);
    };
    if (tid == 0)
        for (int c = 0; c <= P && c < nchunks; ++c) issue(c);

    const bool safe = *unsafe_flag == 0u;
    const int x = X0 + tid;
    const bool warp_interior = __all_sync(0xffffffffu, x >= R && x + R < W);
    double* ocol = out + static_cast<size_t>(b) * out_plane + x;
    constexpr int co[4] = {0, R, R + 1, 2 * R + 1};
    constexpr double kNq = (R + 1) * (R + 1), kNh = (R + 1) * (2 * R + 1);

    for (int c = 0; c < nchunks; ++c) {
        const int q = c % NCR;
        tma::mbar_wait(&full[q], (c / NCR) & 1);
        // slot bases of chunks c-D .. c (+ this thread's column)
        const double* cb[D + 1];
#pragma unroll
        for (int j = 0; j <= D; ++j) {
            const int qq = ((c - D + j) % NCR + NCR) % NCR;
            cb[j] = ring + static_cast<size_t>(qq) * CH * BWT + tid + Ly::XOFF;
        }
        const T* uc = uring + static_cast<size_t>(c % NUS) * CH * Ly::SW + tid;
        const int i0 = c * CH - 2 * R - 1;  // output row index of the step's row 0
        const int gy0 = Y0 + i0;
        const bool rows_full = i0 >= 0 && i0 + CH <= nout && gy0 >= R && gy0 + CH + R <= H;
        auto rows = [&](auto kind_tag) {
            constexpr bool FAST = decltype(kind_tag)::value;
            for_each_k(std::make_integer_sequence<int, CH>{}, [&](auto k_tag) {
                constexpr int k = decltype(k_tag)::value;
                const int i = i0 + k;
                const int y = Y0 + i;
                if (!FAST && (i < 0 || i >= nout || x >= W)) return;
                const double u = to_f64(uc[k * Ly::SW]);
                double best;
                if (FAST || (safe && x >= R && x + R < W && y >= R && y + R < H)) {
                    // 4x4 corner grid: table rows {y-R, y, y+1, y+R+1} x
                    // columns {x-R, x, x+1, x+R+1}
                    const double* rp[4];
                    auto rowp = [&](auto o_tag) {
                        constexpr int rel = k + decltype(o_tag)::value + D * CH - 2 * R - 1;
                        return cb[rel / CH] + (rel % CH) * BWT;
                    };
                    rp[0] = rowp(std::integral_constant<int, 0>{});
                    rp[1] = rowp(std::integral_constant<int, R>{});
                    rp[2] = rowp(std::integral_constant<int, R + 1>{});
                    rp[3] = rowp(std::integral_constant<int, 2 * R + 1>{});
                    double g[4][4];
#pragma unroll
                    for (int a = 0; a < 4; ++a)
#pragma unroll
                        for (int cc = 0; cc < 4; ++cc) g[a][cc] = rp[a][co[cc]];
                    constexpr int W8[8][4] = {{0, 2, 1, 3}, {1, 3, 1, 3}, {1, 3, 0, 2},
                                              {0, 2, 0, 2}, {0, 2, 0, 3}, {1, 3, 0, 3},
                                              {0, 3, 1, 3}, {0, 3, 0, 2}};
                    double av[8], dv[8];
#pragma unroll
                    for (int w = 0; w < 8; ++w) {
                        const int ca = W8[w][0], cbb = W8[w][1], ra = W8[w][2], rb = W8[w][3];
                        const double s = __dadd_rn(
                            __dsub_rn(__dsub_rn(g[rb][cbb], g[rb][ca]), g[ra][cbb]), g[ra][ca]);
                        av[w] = div_by_count_unguarded(s, w < 4 ? kNq : kNh, w < 4 ? yq : yh);
                        dv[w] = fabs(__dsub_rn(av[w], u));
                    }
                    // safe table: every |a_i - u| finite; the stable depth-3
                    // tournament returns the first minimum (strict <)
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
                } else {
                    best = twalk_general_px<R, Ly::RA, CH, NCR, BWT>(ring, X0, ty0, x, y, W, H, u,
                                                             rcp_tab);
                }
                ocol[static_cast<size_t>(y) * out_pitch] = best;
            });
        };
        if (safe && rows_full && warp_interior)
            rows(std::true_type{});
        else
            rows(std::false_type{});
        __syncthreads();  // every thread is past step c: chunk c-D's slot is free
        if (tid == 0 && c + 1 + P < nchunks) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            issue(c + 1 + P);
        }
    }
}

}  // namespace twk

// Launch one table-path stencil pass with the walk; cudaErrorNotSupported
// (nothing launched) when the table or input layout is not TMA-able.
template <int R>
cudaError_t exact_twalk_launch(const PlaneView& in, const Geometry& g, const double* sat,
                               size_t tpitch, double* out, size_t op, size_t opl,
                               const unsigned* unsafe_flag, cudaStream_t s) {
    auto go = [&](auto tag) -> cudaError_t {
        using T = decltype(tag);
        using Ly = twk::TWLay<R, T>;
        CUtensorMap mt, mu;
        const uint64_t tplane = static_cast<uint64_t>(tpitch) * (g.height + 1) * sizeof(double);
        if (!tma::encode_3d(&mt, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, sat, g.width + 1, g.height + 1,
                            g.batch, tpitch * sizeof(double), tplane, Ly::BWT, Ly::CH))
            return cudaErrorNotSupported;
        const uint64_t uplane = (g.batch > 1 ? in.plane : in.pitch * g.height) * sizeof(T);
        constexpr CUtensorMapDataType dt =
            sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64
                           : (sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                             : CU_TENSOR_MAP_DATA_TYPE_UINT8);
        if (!tma::encode_3d(&mu, dt, in.base, g.width, g.height, g.batch, in.pitch * sizeof(T),
                            uplane, Ly::SW, Ly::CH))
            return cudaErrorNotSupported;
        static std::atomic<unsigned long long> done{0};
        if (cudaError_t e = ensure_smem(twk::exact_twalk<R, T>, Ly::SMEM, done)) return e;
        const int strips = (g.width + Ly::SW - 1) / Ly::SW;
        // row blocks: 256 rows, fewer when that leaves the device under two
        // waves of 4 CTAs per SM (a single 4096^2 plane: 32 x 32 CTAs)
        int bh = 256;
        while (bh > 64 && static_cast<long long>(strips) * ((g.height + bh - 1) / bh) * g.batch <
                              2LL * 148 * 4)
            bh /= 2;
        const double yq = 1.0 / static_cast<double>((R + 1) * (R + 1));
        const double yh = 1.0 / static_cast<double>((R + 1) * (2 * R + 1));
        dim3 grid(strips, (g.height + bh - 1) / bh, g.batch);
        twk::exact_twalk<R, T><<<grid, Ly::NT, Ly::SMEM, s>>>(mt, mu, out, op, opl, g.width,
                                                             g.height, bh, unsafe_flag, yq, yh);
        return cudaGetLastError();
    };
    switch (in.dtype) {
        case OSBF_U8: return go(uint8_t{});
        case OSBF_F32: return go(float{});
        default: return go(double{});
    }
}

}  // namespace osbf_gpu
