// Fast mode, mid radii: streaming column strips with register rings.
//
// Included by osbf_fast_kernel.cuh (uses Band, select_store, ColFactors,
// tma_dtype).  One CTA owns a strip of TWS = 128 output columns (NWB = 4
// column warps) and a band of output rows, and walks down it once:
//
//   * Thread 0 streams the strip (plus an R-column halo each side) with TMA
//     in chunks of CH = 2R+2 (R+1 above r=10) rows through a 3-8 slot ring
//     (one mbarrier per slot; after each chunk one CTA barrier frees the
//     previous chunk's slot; hardware zero fill outside the image, so
//     clipped windows need no special casing; the valid counts are the
//     reference's clipped ones, integral.hpp:53-61).
//   * Four column warps, one thread per output column.  Per chunk each warp
//     first forms the horizontal left arms H(x) = sum U[x-R..x] of its own
//     32 + R columns (lanes = 16 rows x 2 odd-length segments: conflict-free,
//     fully unrolled so every sample is loaded once) into a private slice,
//     then walks the chunk's rows keeping vertical running sums Up/Dn of
//     F1 = H(x), F2 = H(x+R), F3 = U(x) (the decomposition of
//     osbf_fast_kernel.cuh) with the last 2R+2 values of each field in
//     REGISTERS (a ring indexed by the row within the chunk, so every index
//     is static).  Per pixel: 3 shared-memory loads for the walk, O(1) work
//     independent of R, and each input row is read once per strip (no tile
//     halo rows).
//
// Running sums start at zero over a zeroed ring at the first input row (the
// window rows above the strip's first output are the R rows of the halo), so
// the first output already has the complete sums.  Integer inputs keep exact
// integer sums (bit-exact first pass on uint8, as the tile kernels).
#include <stdlib.h>

#include <type_traits>

namespace osbf_gpu {
namespace fastk {

constexpr int kStreamMinRadius = 5;
constexpr int kStreamMaxRadius = 16;

template <int R, typename T>
struct SLay {
    static constexpr int NWB = 4;               // column warps (one per SM sub-partition)
    static constexpr int TWS = 32 * NWB;        // output columns per strip
    static constexpr int NTS = 32 * NWB;        // thread 0 also issues the TMA loads
    static constexpr int L = 2 * R + 2;         // register ring length
    // rows per chunk: the ring length, or half of it above r=10 (halves the
    // shared-memory slots so two CTAs still fit; chunks then alternate
    // between the two halves of the ring, a compile-time parity)
    static constexpr int NPAR = R > 10 ? 2 : 1;
    static constexpr int CH = L / NPAR;
    static constexpr int ALIGN = 16 / static_cast<int>(sizeof(T));
    static constexpr int RA = (R + ALIGN - 1) / ALIGN * ALIGN;  // TMA x start: X0 - RA
    static constexpr int XOFF = RA - R;
    static constexpr int BW0 = (TWS + RA + R + ALIGN - 1) / ALIGN * ALIGN;
    // fp64 rows: BW = 2 mod 4 doubles, so 16 rows x 2 odd-offset segments of
    // the arm pass hit all 16 bank pairs twice (conflict-free)
    static constexpr int BW = sizeof(T) == 8 ? (BW0 % 4 == 2 ? BW0 : BW0 + (BW0 % 4 == 0 ? 2 : 1))
                                             : BW0;
    static_assert(BW <= 256, "TMA box width");
    // per-warp arm slice: H(X0 + 32w + m), m < 32 + R, in 2 odd segments
    static constexpr int SEGA = ((32 + R + 1) / 2) | 1;
    static constexpr int HWP = (2 * SEGA) % 4 == 2 ? 2 * SEGA : 2 * SEGA + 2;
    static constexpr uint32_t CHUNK_BYTES = static_cast<uint32_t>(BW) * CH * sizeof(T);
    static constexpr size_t U_BYTES = (CHUNK_BYTES + 127) / 128 * 128;
    static constexpr size_t U_ELEMS = U_BYTES / sizeof(T);
    static constexpr size_t H_WARP = static_cast<size_t>(HWP) * CH;  // doubles
    static constexpr size_t H_BYTES = NWB * H_WARP * sizeof(double);
    static constexpr size_t PAD = 512;  // equal-length arm segments may read past the last row
    static constexpr size_t kSmemMax = 227 * 1024;
    // U ring depth: as deep as MINB CTAs per SM allow (3..8 slots)
    // CTAs per SM in the launch bound: 4-warp CTAs put MINB warps on each SM
    // sub-partition, whose 64K-register file then caps a thread at 128 / 168
    // / 255 registers (the prefix rings need 6R+6 doubles)
    static constexpr int MINB = R <= 5 ? 4 : (R <= 7 ? 3 : 2);
    static constexpr size_t kCtaSmem = (MINB == 4 ? 56 : MINB == 3 ? 74 : 112) * 1024;
    static constexpr int NU_FIT = static_cast<int>((kCtaSmem - 128 - PAD - H_BYTES) / U_BYTES);
    static constexpr int NU = NU_FIT > 8 ? 8 : (NU_FIT < 3 ? 3 : NU_FIT);
    static constexpr size_t SMEM = 128 + NU * U_BYTES + PAD + H_BYTES;
    static_assert(SMEM <= kSmemMax, "stream kernel shared memory");
};

template <int R, typename T, int N>
__device__ __forceinline__ void arm_segment(const T* __restrict__ u, double* __restrict__ h) {
    double v[N + R];
#pragma unroll
    for (int i = 0; i < N + R; ++i) v[i] = to_f64(u[i]);
    double acc = v[0];
#pragma unroll
    for (int i = 1; i <= R; ++i) acc += v[i];
    h[0] = acc;
#pragma unroll
    for (int m = 1; m < N; ++m) {
        acc += v[m + R] - v[m - 1];
        h[m] = acc;
    }
}

template <int R, typename T, bool EXACT_DIV>
__global__ void __launch_bounds__(SLay<R, T>::NTS, SLay<R, T>::MINB)
    fast_stream_step(const __grid_constant__ CUtensorMap tmap, double* __restrict__ out,
                     size_t out_pitch, size_t out_plane, int W, Band band, int band_rows) {
    using Ly = SLay<R, T>;
    constexpr int L = Ly::L, CH = Ly::CH;
    extern __shared__ unsigned char smem_raw[];
    // ufull: TMA landed (1 arrive + tx).  Each column warp computes the arms
    // of its own 32 + R columns (private slice, no cross-warp dependency) and
    // then its rows; one barrier per chunk frees the previous chunk's slot,
    // which thread 0 refills with TMA.
    __shared__ uint64_t ufull[Ly::NU];
    __shared__ double rtab[2 * R + 2];
    const uint32_t base = tma::smem_u32(smem_raw);
    unsigned char* sm = smem_raw + ((128u - (base & 127u)) & 127u);
    T* Ub = reinterpret_cast<T*>(sm);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    double* Hw = reinterpret_cast<double*>(sm + Ly::NU * Ly::U_BYTES + Ly::PAD) +
                 warp * Ly::H_WARP;

    const int X0 = blockIdx.x * Ly::TWS;
    const int Y0 = band.y_out0 + tile_row(band) * band_rows;
    const int nout = min(band_rows, band.y_end - Y0);
    const int nchunks = (nout + 2 * R + CH - 1) / CH;
    const int b = blockIdx.z;
    const int ytma0 = Y0 - R - band.y_in0;  // input-buffer row of strip input row 0

    if (tid < 2 * R + 2) rtab[tid] = tid ? 1.0 / tid : 0.0;
    if (tid == 0) {
        for (int q = 0; q < Ly::NU; ++q) tma::mbar_init(&ufull[q], 1);
    }
    __syncthreads();
    auto issue = [&](int c) {  // chunk c into slot c % NU (thread 0)
        const int q = c % Ly::NU;
        tma::mbar_arrive_expect_tx(&ufull[q], Ly::CHUNK_BYTES);
        tma::load_3d(Ub + q * Ly::U_ELEMS, &tmap, X0 - Ly::RA, ytma0 + c * CH, b, &ufull[q]);
    };
    if (tid == 0)
        for (int c = 0; c < Ly::NU && c < nchunks; ++c) issue(c);

    // Arms of this warp's slice for the chunk in U: lanes = 16 rows x 2 segments.
    auto arms = [&](const T* U) {
        const int rl = lane & 15, sl = lane >> 4;
        for (int k = rl; k < CH; k += 16)
            arm_segment<R, T, Ly::SEGA>(U + k * Ly::BW + 32 * warp + sl * Ly::SEGA + Ly::XOFF,
                                        Hw + k * Ly::HWP + sl * Ly::SEGA);
        __syncwarp();
    };

    // Column warps: one output column per thread.
    const int gx = X0 + tid;
    const int Himg = band.h_img;
    // Rings of column PREFIX sums (slot = row within the chunk):
    //   P1 = sum F1, P2 = sum F2, PG = sum G with G = F1 + F2 - F3 (the full
    //   2R+1 row arm).  Each window is one difference of two prefixes:
    //   Up = P(y) - P(y-R-1), Dn = P(y+R) - P(y-1), Full = P(y+R) - P(y-R-1).
    double q1[L], q2[L], qg[L];
#pragma unroll
    for (int i = 0; i < L; ++i) q1[i] = q2[i] = qg[i] = 0.0;
    double P1 = 0.0, P2 = 0.0, PG = 0.0;
    const bool col_border = gx < R || gx >= W - R;
    double* ocol = out + static_cast<size_t>(b) * out_plane + gx;
    ColFactors cf{0.0, 0.0, 0.0};
    if (gx < W) {  // border rows of interior columns need them too
        const int ncl = min(gx, R) + 1, ncr = min(W - 1 - gx, R) + 1;
        cf = ColFactors{rtab[ncl], rtab[ncr], rtab[ncl + ncr - 1]};
    }
    const bool warp_interior = __all_sync(0xffffffffu, gx < W && !col_border);
    const bool warp_border = !warp_interior;
    // Chunk kinds (all warp-uniform, so no lane of a warp runs a different
    // select than its neighbours):
    //   0  every row an output row away from the image top/bottom, no border
    //      column in the warp: interior reciprocals, no per-row branch;
    //   1  same rows, but the warp holds border (or out-of-image) columns:
    //      the clipped-count select for all its lanes (for a full window it
    //      forms exactly the interior reciprocal, select_store);
    //   2  otherwise: per-row output / border checks.
    // u / uprev: this column's samples in the chunk's / previous chunk's slot
    // (the centre sample of row k sits R rows up).
    auto chunk_rows = [&](auto kind_tag, auto parity_tag, const double* h, const T* u,
                          const T* uprev, int iy0, const ColFactors& cf) {
        constexpr int KIND = decltype(kind_tag)::value;
        constexpr int RB = decltype(parity_tag)::value * CH;  // ring slot of row 0
#pragma unroll
        for (int k = 0; k < CH; ++k) {
            const double a = h[k * Ly::HWP], c = h[k * Ly::HWP + R];
            const double e = to_f64(u[k * Ly::BW]);
            P1 += a;
            P2 += c;
            PG += (a + c) - e;
            const int iY = (RB + k + R + 2) % L, iYm1 = (RB + k + R + 1) % L,
                      iOld = (RB + k + 1) % L;
            const double p1y = q1[iY], p1m = q1[iYm1], p1o = q1[iOld];
            const double p2y = q2[iY], p2m = q2[iYm1], p2o = q2[iOld];
            const double pgy = qg[iY], pgm = qg[iYm1], pgo = qg[iOld];
            q1[RB + k] = P1;
            q2[RB + k] = P2;
            qg[RB + k] = PG;
            const int iy = iy0 + k;  // output row Y0 + iy - R when iy in [R, R + nout)
            if (KIND < 2 || (iy >= R && iy < R + nout)) {
                const int gy = Y0 + iy - R;
                const double uc = to_f64(k >= R ? u[(k - R) * Ly::BW] : uprev[(k - R + CH) * Ly::BW]);
                const double S[8] = {P1 - p1m, P2 - p2m, p2y - p2o, p1y - p1o,
                                     P1 - p1o, P2 - p2o, PG - pgm,  pgy - pgo};
                double* o = ocol + static_cast<size_t>(gy - band.y_out0) * out_pitch;
                const bool clipped = KIND == 1 || (KIND == 2 && (warp_border || gy < R ||
                                                                 gy >= Himg - R));
                if (KIND == 0 || (KIND == 2 && !clipped)) {
                    if (KIND == 0 || gx < W)
                        select_store<R, EXACT_DIV, false, false>(S, uc, gx, gy, W, Himg, b, o,
                                                                 nullptr, nullptr, cf, rtab);
                } else if (gx < W) {
                    select_store<R, EXACT_DIV, true, false>(S, uc, gx, gy, W, Himg, b, o, nullptr,
                                                            nullptr, cf, rtab);
                }
            }
        }
    };
    for (int c = 0; c < nchunks; ++c) {
        const int q = c % Ly::NU, qp = (c + Ly::NU - 1) % Ly::NU;
        tma::mbar_wait(&ufull[q], (c / Ly::NU) & 1);
        arms(Ub + q * Ly::U_ELEMS);
        const T* u = Ub + q * Ly::U_ELEMS + tid + Ly::RA;
        const T* uprev = Ub + qp * Ly::U_ELEMS + tid + Ly::RA;
        const double* h = Hw + lane;
        const int iy0 = c * CH - R;  // strip row index (input coords) of the k = 0 output
        const int gy0 = Y0 + iy0 - R;
        const bool rows_full =
            iy0 >= R && iy0 + CH <= R + nout && gy0 >= R && gy0 + CH <= Himg - R;
        auto run = [&](auto parity) {
            if (rows_full && warp_interior)
                chunk_rows(std::integral_constant<int, 0>{}, parity, h, u, uprev, iy0, cf);
            else if (rows_full)
                chunk_rows(std::integral_constant<int, 1>{}, parity, h, u, uprev, iy0, cf);
            else
                chunk_rows(std::integral_constant<int, 2>{}, parity, h, u, uprev, iy0, cf);
        };
        if (Ly::NPAR == 2 && (c & 1))
            run(std::integral_constant<int, Ly::NPAR - 1>{});
        else
            run(std::integral_constant<int, 0>{});
        __syncwarp();  // slice reads done before the next chunk's arms
        // every warp is done with chunk c, so the previous chunk's slot (its
        // centre samples were the last readers) takes chunk c - 1 + NU
        __syncthreads();
        if (tid == 0 && c > 0 && c - 1 + Ly::NU < nchunks) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            issue(c - 1 + Ly::NU);
        }
    }
    if (gx < W)
        push_tail(band, out + static_cast<size_t>(b) * out_plane, out_pitch, gx, Y0, Y0 + nout);
}

inline bool stream_enabled() {
    static int on = -1;
    if (on < 0) {
        const char* e = getenv("OSBF_GPU_STREAM");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on == 1;
}

// Returns cudaErrorNotSupported (no launch) when the layout is not TMA-able.
template <int R, typename T, bool EXACT_DIV>
cudaError_t launch_stream(const PlaneView& in, const Geometry& g, double* out, size_t op,
                          size_t opl, cudaStream_t s) {
    using Ly = SLay<R, T>;
    CUtensorMap map;
    const uint64_t plane_bytes = (g.batch > 1 ? in.plane : in.pitch * g.in_h()) * sizeof(T);
    if (!tma::encode_3d(&map, tma_dtype<T>(), in.base, g.width, g.in_h(), g.batch,
                        in.pitch * sizeof(T), plane_bytes, Ly::BW, Ly::CH))
        return cudaErrorNotSupported;
    static std::atomic<unsigned long long> done{0};
    if (cudaError_t e = ensure_smem(fast_stream_step<R, T, EXACT_DIV>, Ly::SMEM, done)) return e;
    // Strips walk in 512-row bands (each band re-reads a 2R-row halo): a
    // single plane still fills the SMs and a batch ends in a short last wave
    // (measured best of 128..2048 rows on 256 x 1024^2 and 32768^2).  The
    // split depends on the image height only, never on the batch size, so
    // results do not depend on how a batch is chunked.
    const int strips = (g.width + Ly::TWS - 1) / Ly::TWS;
    // (r >= 10 runs two CTAs per SM, so whole 1024-row planes still leave
    // a full last wave and save the second band's preamble)
    const int band_rows = (R >= 10 && g.height <= 1024) ? g.height
                                                        : (g.height < 512 ? g.height : 512);
    dim3 grid(strips, (g.height + band_rows - 1) / band_rows, g.batch);
    note_kernel("fast_stream_step");
    fast_stream_step<R, T, EXACT_DIV><<<grid, Ly::NTS, Ly::SMEM, s>>>(map, out, op, opl, g.width,
                                                                      band_of(g), band_rows);
    return cudaGetLastError();
}

}  // namespace fastk
}  // namespace osbf_gpu
