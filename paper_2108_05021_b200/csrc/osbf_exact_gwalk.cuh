// Exact mode, whole-table path, any radius 1..62: the stencil as a column walk
// over three TMA-staged streams of table rows (exact_gwalk).  Replaces the
// per-thread global corner loads of exact_stencil for radii above the
// templated walk (osbf_exact_twalk.cuh, r <= 16), whose shared-memory ring
// holds all 2r+2 table rows a pixel spans and therefore grows with r.
//
// An output row y reads only four table rows: y-r, y, y+1 and y+r+1
// (integral.hpp:41-49: the corners of the eight one-sided windows,
// core.hpp:212-225).  A CTA of 128 threads owns 128 output columns and a block
// of BH output rows and walks down it in chunks of CH rows; for chunk c thread
// 0 issues four cp.async.bulk.tensor loads into one stage of an NS-deep ring:
//   A: table rows y0-r   .. y0-r+CH-1      (CH rows)
//   B: table rows y0     .. y0+CH          (CH+1 rows: y and y+1)
//   C: table rows y0+r+1 .. y0+r+CH        (CH rows)
//   U: the CH input rows (centre samples)
// each table box covering columns [X0-r, X0+128+r] (from the 16-byte boundary
// at or left of X0-r).  Shared memory per CTA is (3 CH + 1)(130 + 2r) doubles
// per stage whatever r is, the work per pixel is 16 shared loads at four
// per-thread column offsets, and every table row is fetched three times from
// L2 (the streams of one CTA are r rows apart: ~(2r+1)(130+2r) doubles of
// live L2 footprint per CTA), once from HBM.
//
// Same arithmetic as exact_stencil / exact_twalk: ((A-B)-C)+D
// (integral.hpp:48-49), the IEEE-exact division by the count
// (integral.hpp:68), first strict minimum of |a-u| in window order
// (filters2d.hpp:72-82).  Pixels whose windows are clipped by the image border,
// and every pixel of a table flagged unsafe (non-finite / out-of-range values),
// take the reference's per-window rule on the table in global memory.
#pragma once

#include "osbf_exact2_kernel.cuh"
#include "osbf_internal.cuh"
#include "osbf_tma.cuh"

namespace osbf_gpu {
namespace gwk {

#ifndef OSBF_GWALK_MINB
#define OSBF_GWALK_MINB 4
#endif
constexpr int NT = 128;  // threads = output columns per CTA
constexpr int SW = 128;
constexpr int CH = 4;    // output rows per chunk
constexpr int MAXNS = 4;
constexpr int kMaxRadius = 62;  // box width RA + 128 + r + 2 <= 256 (TMA box limit)

__host__ __device__ constexpr unsigned align128(unsigned v) { return (v + 127u) & ~127u; }

// Byte offsets of the four boxes inside a stage (each 128-byte aligned).
struct Stage {
    unsigned offB, offC, offU, bytes, tx;
};
template <typename T>
__host__ __device__ constexpr Stage stage_of(int bwt) {
    Stage st{};
    const unsigned row = static_cast<unsigned>(bwt) * 8u;
    st.offB = align128(CH * row);
    st.offC = st.offB + align128((CH + 1) * row);
    st.offU = st.offC + align128(CH * row);
    st.bytes = st.offU + align128(CH * SW * static_cast<unsigned>(sizeof(T)));
    st.tx = (3 * CH + 1) * row + CH * SW * static_cast<unsigned>(sizeof(T));
    return st;
}

// Unsafe table (non-finite / out-of-range values, rare): the reference's
// rule on the table in global memory (clipped corners, IEEE division,
// sequential strict <, so NaN never wins).
static __device__ __noinline__ double gwalk_guarded_px(const double* __restrict__ C, long long tp,
                                                       int x, int y, int W, int H, int r,
                                                       double u) {
    double best = 0.0, best_abs = __longlong_as_double(0x7ff0000000000000LL);
#pragma unroll 1
    for (int i = 0; i < 8; ++i) {
        const Win w = window(i, r);
        const int x0 = max(x + w.u0, 0), x1 = min(x + w.u1, W - 1);
        const int y0 = max(y + w.v0, 0), y1 = min(y + w.v1, H - 1);
        const double* ra = C + y0 * tp;
        const double* rb = C + (y1 + 1) * tp;
        const double s = __dadd_rn(__dsub_rn(__dsub_rn(rb[x1 + 1], rb[x0]), ra[x1 + 1]), ra[x0]);
        const double n = static_cast<double>((x1 - x0 + 1) * (y1 - y0 + 1));
        const double a = __ddiv_rn(s, n);
        const double d = fabs(__dsub_rn(a, u));
        if (d < best_abs) {
            best_abs = d;
            best = a;
        }
    }
    return best;
}

// (ca, cb, ra, rb) of each window's corners in the 4x4 grid
// rows {y0, y, y+1, y1+1} x columns {x0, x, x+1, x1+1}, reference order
// (core.hpp:212-225); clipping only moves the outer rows / columns.
__device__ constexpr int kW8[8][4] = {{0, 2, 1, 3}, {1, 3, 1, 3}, {1, 3, 0, 2}, {0, 2, 0, 2},
                                      {0, 2, 0, 3}, {1, 3, 0, 3}, {0, 3, 1, 3}, {0, 3, 0, 2}};

// First strict minimum of dv (all finite) and its mean: stable depth-3 tournament.
__device__ __forceinline__ double first_min(double (&dv)[8], double (&av)[8]) {
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
    return av[0];
}

// BWT: staged table columns per row (a radius class: the smallest of 144 /
// 160 / 192 / 224 / 256 that holds RA + 128 + r + 2), compile-time so every
// shared load is [per-thread column pointer + immediate row offset].
template <typename T, int BWT>
__global__ void __launch_bounds__(NT, OSBF_GWALK_MINB)
    exact_gwalk(const __grid_constant__ CUtensorMap map_t, const __grid_constant__ CUtensorMap map_t1,
                const __grid_constant__ CUtensorMap map_u, const double* __restrict__ sat,
                long long tp, double* __restrict__ out, size_t out_pitch, size_t out_plane, int W,
                int H, int BH, int r, int ns, const unsigned* __restrict__ unsafe_flag) {
    constexpr int bwt = BWT;
    extern __shared__ unsigned char smem_raw[];
    __shared__ uint64_t full[MAXNS];
    const uint32_t base = tma::smem_u32(smem_raw);
    unsigned char* sm = smem_raw + ((128u - (base & 127u)) & 127u);
    constexpr Stage st = stage_of<T>(BWT);
    const int tid = threadIdx.x;
    const int X0 = blockIdx.x * SW;
    const int Y0 = blockIdx.y * BH;
    const int nout = min(BH, H - Y0);
    const int b = blockIdx.z;
    const int nchunks = (nout + CH - 1) / CH;
    const int RA = r + (r & 1);  // the boxes start at X0 - RA (a 16-byte boundary)

    if (tid == 0)
        for (int q = 0; q < ns; ++q) tma::mbar_init(&full[q], 1);
    __syncthreads();
    auto issue = [&](int c, int q) {  // thread 0: chunk c into stage q = c % ns
        unsigned char* s0 = sm + static_cast<size_t>(q) * st.bytes;
        const int y0 = Y0 + c * CH;
        tma::mbar_arrive_expect_tx(&full[q], st.tx);
        tma::load_3d(s0, &map_t, X0 - RA, y0 - r, b, &full[q]);
        tma::load_3d(s0 + st.offB, &map_t1, X0 - RA, y0, b, &full[q]);
        tma::load_3d(s0 + st.offC, &map_t, X0 - RA, y0 + r + 1, b, &full[q]);
        tma::load_3d(s0 + st.offU, &map_u, X0, y0, b, &full[q]);
    };
    if (tid == 0)
        for (int c = 0; c < ns && c < nchunks; ++c) issue(c, c);

    const bool safe = *unsafe_flag == 0u;
    const int x = min(X0 + tid, W - 1);  // lanes past the image compute column W-1, never store
    const bool live = X0 + tid < W;
    const double* Cg = sat + static_cast<long long>(b) * tp * (H + 1);
    double* ocol = out + static_cast<size_t>(b) * out_plane + x;
    // Table columns of the corner grid, clipped like integral.hpp:53-56:
    // x0 = max(x-r, 0), x, x+1, x1+1 = min(x+r, W-1)+1.  Clipping is per
    // thread, so border columns run the same code as interior ones.
    const int tx0 = max(x - r, 0), tx3 = min(x + r, W - 1) + 1;
    const int c0 = tx0 - (X0 - RA), c1 = x - (X0 - RA), c2 = c1 + 1, c3 = tx3 - (X0 - RA);
    const int nxl = x - tx0 + 1, nxr = tx3 - x, nxf = tx3 - tx0;
    // rows y-r .. y+r all inside the image: the five window counts and their
    // reciprocals RN(1/n) are per-thread constants
    const double n_ql = static_cast<double>(nxl * (r + 1)), n_qr = static_cast<double>(nxr * (r + 1));
    const double n_hl = static_cast<double>(nxl * (2 * r + 1)),
                 n_hr = static_cast<double>(nxr * (2 * r + 1));
    const double n_v = static_cast<double>(nxf * (r + 1));
    const double y_ql = __ddiv_rn(1.0, n_ql), y_qr = __ddiv_rn(1.0, n_qr);
    const double y_hl = __ddiv_rn(1.0, n_hl), y_hr = __ddiv_rn(1.0, n_hr);
    const double y_v = __ddiv_rn(1.0, n_v);

    int q = 0;             // stage of chunk c (c % ns, without the division)
    unsigned phase = 0;    // (c / ns) & 1
    for (int c = 0; c < nchunks; ++c) {
        tma::mbar_wait(&full[q], phase);
        const unsigned char* s0 = sm + static_cast<size_t>(q) * st.bytes;
        // the thread's four corner columns of the stage's first table row;
        // rows of the A / B / C boxes are immediate offsets from them
        const double* S = reinterpret_cast<const double*>(s0);
        const double* pc[4] = {S + c0, S + c1, S + c2, S + c3};
        constexpr int oB = static_cast<int>(st.offB / 8), oC = static_cast<int>(st.offC / 8);
        const T* U = reinterpret_cast<const T*>(s0 + st.offU) + min(tid, W - 1 - X0);
#pragma unroll
        for (int k = 0; k < CH; ++k) {
            const int i = c * CH + k;
            const int y = Y0 + i;
            if (i >= nout) break;  // uniform
            const double u = to_f64(U[k * SW]);
            double best;
            if (!safe) {
                best = gwalk_guarded_px(Cg, tp, x, y, W, H, r, u);
            } else if (y >= r && y + r < H) {
                // rows unclipped: the staged streams hold the four table rows
                const int ro[4] = {k * bwt, oB + k * bwt, oB + (k + 1) * bwt, oC + k * bwt};
                double g[4][4];
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int cc = 0; cc < 4; ++cc) g[a][cc] = pc[cc][ro[a]];
                const double nn[8] = {n_ql, n_qr, n_qr, n_ql, n_hl, n_hr, n_v, n_v};
                const double yy[8] = {y_ql, y_qr, y_qr, y_ql, y_hl, y_hr, y_v, y_v};
                double av[8], dv[8];
#pragma unroll
                for (int w = 0; w < 8; ++w) {
                    const int ca = kW8[w][0], cbb = kW8[w][1], ra = kW8[w][2], rb = kW8[w][3];
                    const double s = __dadd_rn(
                        __dsub_rn(__dsub_rn(g[rb][cbb], g[rb][ca]), g[ra][cbb]), g[ra][ca]);
                    av[w] = div_by_count_unguarded(s, nn[w], yy[w]);
                    dv[w] = fabs(__dsub_rn(av[w], u));
                }
                best = first_min(dv, av);
            } else {
                // rows clipped by the image top / bottom (whole rows, so the
                // branch is uniform): the same grid with clipped rows, from
                // the table in global memory; IEEE division by each count
                const int ty0 = max(y - r, 0), ty3 = min(y + r, H - 1) + 1;
                const double* rp[4] = {Cg + ty0 * tp, Cg + y * tp, Cg + (y + 1) * tp, Cg + ty3 * tp};
                double g[4][4];
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    g[a][0] = rp[a][tx0];
                    g[a][1] = rp[a][x];
                    g[a][2] = rp[a][x + 1];
                    g[a][3] = rp[a][tx3];
                }
                const int nyu = y - ty0 + 1, nyd = ty3 - y, nyf = ty3 - ty0;
                const int nn[8] = {nxl * nyd, nxr * nyd, nxr * nyu, nxl * nyu,
                                   nxl * nyf, nxr * nyf, nxf * nyd, nxf * nyu};
                double av[8], dv[8];
#pragma unroll
                for (int w = 0; w < 8; ++w) {
                    const int ca = kW8[w][0], cbb = kW8[w][1], ra = kW8[w][2], rb = kW8[w][3];
                    const double s = __dadd_rn(
                        __dsub_rn(__dsub_rn(g[rb][cbb], g[rb][ca]), g[ra][cbb]), g[ra][ca]);
                    av[w] = __ddiv_rn(s, static_cast<double>(nn[w]));
                    dv[w] = fabs(__dsub_rn(av[w], u));
                }
                best = first_min(dv, av);
            }
            if (live) ocol[static_cast<size_t>(y) * out_pitch] = best;
        }
        __syncthreads();  // every thread is past chunk c: its stage is free
        if (tid == 0 && c + ns < nchunks) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            issue(c + ns, q);
        }
        if (++q == ns) {
            q = 0;
            phase ^= 1u;
        }
    }
}

}  // namespace gwk

// One table-path stencil pass with the generic walk; cudaErrorNotSupported
// (nothing launched) when the radius, table or input layout is not covered.
template <typename T, int BWT>
cudaError_t exact_gwalk_launch_class(const PlaneView& in, const Geometry& g, int r,
                                     const double* sat, size_t tpitch, double* out, size_t op,
                                     size_t opl, const unsigned* unsafe_flag, cudaStream_t s) {
    using namespace gwk;
    CUtensorMap mt, mt1, mu;
    const uint64_t tplane = static_cast<uint64_t>(tpitch) * (g.height + 1) * sizeof(double);
    if (!tma::encode_3d(&mt, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, sat, g.width + 1, g.height + 1,
                        g.batch, tpitch * sizeof(double), tplane, BWT, CH) ||
        !tma::encode_3d(&mt1, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, sat, g.width + 1, g.height + 1,
                        g.batch, tpitch * sizeof(double), tplane, BWT, CH + 1))
        return cudaErrorNotSupported;
    const uint64_t uplane = (g.batch > 1 ? in.plane : in.pitch * g.height) * sizeof(T);
    constexpr CUtensorMapDataType dt =
        sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64
                       : (sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                         : CU_TENSOR_MAP_DATA_TYPE_UINT8);
    if (!tma::encode_3d(&mu, dt, in.base, g.width, g.height, g.batch, in.pitch * sizeof(T), uplane,
                        SW, CH))
        return cudaErrorNotSupported;
    constexpr Stage st = stage_of<T>(BWT);
    static const int kNs = [] {
        const char* e = std::getenv("OSBF_GPU_GWALK_STAGES");  // diagnostic override
        const int v = e ? atoi(e) : 0;
        return v >= 2 && v <= MAXNS ? v : 2;
    }();
    const size_t smem = 128 + static_cast<size_t>(kNs) * st.bytes;
    static std::atomic<unsigned long long> done{0};
    if (cudaError_t e = ensure_smem(exact_gwalk<T, BWT>, 128 + MAXNS * st.bytes, done)) return e;
    const int strips = (g.width + SW - 1) / SW;
    // row blocks: 256 rows, fewer when that leaves the device under two
    // waves of 4 CTAs per SM
    static const int kBh = [] {
        const char* e = std::getenv("OSBF_GPU_GWALK_BH");  // diagnostic override
        const int v = e ? atoi(e) : 0;
        return v >= 16 ? v : 0;
    }();
    int bh = 256;
    while (bh > 64 && static_cast<long long>(strips) * ((g.height + bh - 1) / bh) * g.batch <
                          2LL * 148 * 4)
        bh /= 2;
    if (kBh) bh = kBh;
    dim3 grid(strips, (g.height + bh - 1) / bh, g.batch);
    exact_gwalk<T, BWT><<<grid, NT, smem, s>>>(mt, mt1, mu, sat, static_cast<long long>(tpitch),
                                               out, op, opl, g.width, g.height, bh, r, kNs,
                                               unsafe_flag);
    return cudaGetLastError();
}

inline cudaError_t exact_gwalk_launch(const PlaneView& in, const Geometry& g, int r,
                                      const double* sat, size_t tpitch, double* out, size_t op,
                                      size_t opl, const unsigned* unsafe_flag, cudaStream_t s) {
    if (r < 1 || r > gwk::kMaxRadius) return cudaErrorNotSupported;
    const int need = r + (r & 1) + gwk::SW + r + 2;  // columns X0-RA .. X0+127+r+1
    auto go = [&](auto tag) -> cudaError_t {
        using T = decltype(tag);
#define OSBF_GWALK_CLASS(BW) \
    if (need <= BW)          \
        return exact_gwalk_launch_class<T, BW>(in, g, r, sat, tpitch, out, op, opl, unsafe_flag, s);
        OSBF_GWALK_CLASS(144)
        OSBF_GWALK_CLASS(160)
        OSBF_GWALK_CLASS(192)
        OSBF_GWALK_CLASS(224)
        OSBF_GWALK_CLASS(256)
#undef OSBF_GWALK_CLASS
        return cudaErrorNotSupported;
    };
    switch (in.dtype) {
        case OSBF_U8: return go(uint8_t{});
        case OSBF_F32: return go(float{});
        default: return go(double{});
    }
}

}  // namespace osbf_gpu
