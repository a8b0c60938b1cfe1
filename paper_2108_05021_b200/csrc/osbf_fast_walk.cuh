// Fast mode: the column walk (one kernel for every radius 1..16).
//
// Included by osbf_fast_kernel.cuh (uses Band, select_store, ColFactors,
// tile_row, push_tail, tma_dtype).  One CTA of 128 threads owns a strip of
// 128 output columns and a band of output rows and walks down it once.
//
//   * Thread 0 streams the strip plus an R-column halo each side with TMA in
//     chunks of CH rows through a ring of NU slots (one mbarrier per slot,
//     hardware zero fill outside the image: clipped windows need no special
//     casing, only their valid counts do, integral.hpp:53-61).
//   * Arm pass (all 128 threads): the left arms H(c) = U(c-R) + ... + U(c)
//     of the chunk's rows are formed by sliding sums over 8 segments of LS
//     (odd) columns per row, so a half-warp is 2 rows x 8 segments and, with
//     row pitches of 8 mod 16 doubles, every load and store is conflict-free.
//     H is double-buffered, so one CTA barrier per chunk orders everything.
//   * Walk (one thread per output column): per row, F1 = H(x), F2 = H(x+R)
//     and the centre sample U(x) (3 shared loads); column prefix sums
//     P1 += F1, P2 += F2, PG += F1 + F2 - U keep the last L = 2R+2 values in
//     registers (ring slot = row mod L, a compile-time index because a chunk
//     is a multiple or an exact divisor of L), and the eight windows of the
//     output row R rows up are single differences:
//       Up = P(y) - P(y-R-1), Dn = P(y+R) - P(y-1), Full = P(y+R) - P(y-R-1)
//     (the decomposition of osbf_fast_kernel.cuh).  Then select_store.
//
// Work per pixel is O(1) in R (3 + 2.5 shared accesses, ~29 fp64 ops); the
// only R-dependent cost is the register ring (3L doubles per thread), which
// sets the occupancy.  Each input row is read from HBM once per band (no tile
// halo rows); the strip's R halo columns come from L2.
#include <type_traits>

namespace osbf_gpu {
namespace fastk {

constexpr int kWalkMaxRadius = 16;

template <int R, typename T>
struct WLay {
    static constexpr int NT = 128;   // threads = output columns per strip
    static constexpr int SW = 128;
    static constexpr int NSEG = 8;   // arm segments per row
    static constexpr int L = 2 * R + 2;  // register ring length
    // rows per chunk: a multiple of L (R <= 5) or L / 2 (NP = 2 ring phases;
    // keeps 4 CTAs per SM in shared memory at r = 6)
    static constexpr int CH = R == 1 ? 8 : (R <= 5 ? L : L / 2);
    static constexpr int NP = (CH % L == 0) ? 1 : L / CH;
    static_assert(CH % L == 0 || L % CH == 0, "chunk / ring");
    static_assert(CH > R, "centre row of a chunk's first row lies in the previous chunk");
    static constexpr int ALIGN = 16 / static_cast<int>(sizeof(T));
    static constexpr int RA = (R + ALIGN - 1) / ALIGN * ALIGN;  // TMA x start: X0 - RA
    static constexpr int XOFF = RA - R;
    static constexpr int BW0 = (RA + SW + R + ALIGN - 1) / ALIGN * ALIGN;
    // fp64 rows: pitch = 8 mod 16 doubles, so 2 rows x 8 odd-length segments
    // cover all 16 bank pairs
    static constexpr int BW = sizeof(T) == 8 ? BW0 + ((8 - BW0 % 16) + 16) % 16 : BW0;
    static_assert(BW <= 256, "TMA box width");
    static constexpr int LS = (((SW + R + NSEG - 1) / NSEG) | 1);
    static constexpr int HP = NSEG * LS;  // = 8 mod 16
    static constexpr uint32_t CHUNK_BYTES = static_cast<uint32_t>(BW) * CH * sizeof(T);
    static constexpr size_t U_BYTES = (CHUNK_BYTES + 127) / 128 * 128;
    static constexpr size_t U_ELEMS = U_BYTES / sizeof(T);
    static constexpr size_t H_ELEMS = static_cast<size_t>(CH) * HP;
    // the last segment of a row may read up to LS + R + XOFF elements past
    // the row's useful part (feeding unused arms only)
    static constexpr size_t PAD = ((LS + R + XOFF) * sizeof(T) + 127) / 128 * 128;
    // register budget: 4 CTAs per SM up to r = 4 and at r = 6 (128 registers,
    // no spills; r = 5 keeps its 12-row chunks at 3 CTAs: measured faster),
    // 3 to r = 8, then 2
    static constexpr int MINB = (R <= 4 || R == 6) ? 4 : (R <= 8 ? 3 : 2);
    static constexpr size_t kCtaSmem = (MINB == 4 ? 56 : MINB == 3 ? 74 : 112) * 1024;
    static constexpr size_t H_BYTES = 2 * H_ELEMS * sizeof(double);
    static constexpr int NU_FIT =
        static_cast<int>((kCtaSmem - 128 - PAD - H_BYTES) / U_BYTES);
    static constexpr int NU = NU_FIT > 4 ? 4 : (NU_FIT < 3 ? 3 : NU_FIT);
    static constexpr size_t SMEM = 128 + NU * U_BYTES + PAD + H_BYTES;
    static_assert(SMEM <= 227 * 1024, "walk kernel shared memory");
};

// Sliding left arms of one row segment: h[m] = u[m] + ... + u[m + R], m < N.
template <int R, typename T, int N>
__device__ __forceinline__ void walk_arm_segment(const T* __restrict__ u, double* __restrict__ h) {
    double acc = to_f64(u[0]);
#pragma unroll
    for (int i = 1; i <= R; ++i) acc += to_f64(u[i]);
    h[0] = acc;
#pragma unroll
    for (int m = 1; m < N; ++m) {
        acc += to_f64(u[m + R]) - to_f64(u[m - 1]);
        h[m] = acc;
    }
}

template <int R, typename T, bool EXACT_DIV>
__global__ void __launch_bounds__(WLay<R, T>::NT, WLay<R, T>::MINB)
    fast_walk_step(const __grid_constant__ CUtensorMap tmap, double* __restrict__ out,
                   size_t out_pitch, size_t out_plane, int W, Band band, int band_rows) {
    using Ly = WLay<R, T>;
    constexpr int L = Ly::L, CH = Ly::CH, NP = Ly::NP, NU = Ly::NU;
    extern __shared__ unsigned char smem_raw[];
    __shared__ uint64_t ufull[NU];
    __shared__ double rtab[2 * R + 2];
    const uint32_t base = tma::smem_u32(smem_raw);
    unsigned char* sm = smem_raw + ((128u - (base & 127u)) & 127u);
    T* Ub = reinterpret_cast<T*>(sm);
    double* Hb = reinterpret_cast<double*>(sm + NU * Ly::U_BYTES + Ly::PAD);
    const int tid = threadIdx.x;

    const int X0 = blockIdx.x * Ly::SW;
    // row blocks are aligned to multiples of band_rows in GLOBAL image rows,
    // so a row band that starts on a block boundary walks exactly the blocks
    // the whole image does (bit-identical results; dist.band_rows aligns)
    const int blk = band.y_out0 / band_rows + tile_row(band);
    const int Y0 = max(band.y_out0, blk * band_rows);
    const int nout = min(band.y_end, (blk + 1) * band_rows) - Y0;
    const int nchunks = (nout + 2 * R + CH - 1) / CH;
    const int b = blockIdx.z;
    const int ytma0 = Y0 - R - band.y_in0;  // buffer row of strip input row 0

    if (tid < 2 * R + 2) rtab[tid] = tid ? 1.0 / tid : 0.0;
    if (tid == 0)
        for (int q = 0; q < NU; ++q) tma::mbar_init(&ufull[q], 1);
    __syncthreads();
    auto issue = [&](int c) {  // chunk c into slot c % NU (thread 0)
        const int q = c % NU;
        tma::mbar_arrive_expect_tx(&ufull[q], Ly::CHUNK_BYTES);
        tma::load_3d(Ub + q * Ly::U_ELEMS, &tmap, X0 - Ly::RA, ytma0 + c * CH, b, &ufull[q]);
    };
    if (tid == 0)
        for (int c = 0; c < NU && c < nchunks; ++c) issue(c);

    const int gx = X0 + tid;
    const int Himg = band.h_img;
    double q1[L], q2[L], qg[L];
#pragma unroll
    for (int i = 0; i < L; ++i) q1[i] = q2[i] = qg[i] = 0.0;
    double P1 = 0.0, P2 = 0.0, PG = 0.0;
    ColFactors cf{0.0, 0.0, 0.0};
    if (gx < W) {
        const int ncl = min(gx, R) + 1, ncr = min(W - 1 - gx, R) + 1;
        cf = ColFactors{rtab[ncl], rtab[ncr], rtab[ncl + ncr - 1]};
    }
    const bool warp_interior = __all_sync(0xffffffffu, gx >= R && gx < W - R);
    double* ocol = out + static_cast<size_t>(b) * out_plane + gx;
    // chunk-relative row offsets fit 32 bits: one IMAD.WIDE per output row
    const unsigned obytes = static_cast<unsigned>(out_pitch * sizeof(double));

    // KIND 0: every row of the chunk is an output row away from the image
    // top/bottom and the warp has no border column (interior reciprocals, no
    // per-row test); 1: same rows, border columns in the warp; 2: per-row tests.
    auto chunk_rows = [&](auto kind_tag, auto phase_tag, const double* __restrict__ h,
                          const T* __restrict__ u, const T* __restrict__ uprev, int i0) {
        constexpr int KIND = decltype(kind_tag)::value;
        constexpr int RB = decltype(phase_tag)::value * CH;  // ring slot of row 0
        double* o0 = ocol + static_cast<ptrdiff_t>(Y0 + i0 - band.y_out0) *
                                    static_cast<ptrdiff_t>(out_pitch);
#pragma unroll
        for (int k = 0; k < CH; ++k) {
            const double a = h[k * Ly::HP], c = h[k * Ly::HP + R];
            const double e = to_f64(u[k * Ly::BW]);
            P1 += a;
            P2 += c;
            PG += (a + c) - e;
            const int sk = (RB + k) % L;
            const int sY = (sk + L - R) % L, sYm1 = (sk + L - R - 1) % L, sOld = (sk + 1) % L;
            const double p1y = q1[sY], p1m = q1[sYm1], p1o = q1[sOld];
            const double p2y = q2[sY], p2m = q2[sYm1], p2o = q2[sOld];
            const double pgy = qg[sY], pgm = qg[sYm1], pgo = qg[sOld];
            q1[sk] = P1;
            q2[sk] = P2;
            qg[sk] = PG;
            const int i = i0 + k;  // output row index (Y0 + i) of this step
            if (KIND < 2 || (i >= 0 && i < nout)) {
                const int gy = Y0 + i;
                const double uc =
                    to_f64(k >= R ? u[(k - R) * Ly::BW] : uprev[(k - R + CH) * Ly::BW]);
                const double S[8] = {P1 - p1m, P2 - p2m, p2y - p2o, p1y - p1o,
                                     P1 - p1o, P2 - p2o, PG - pgm,  pgy - pgo};
                double* o = reinterpret_cast<double*>(reinterpret_cast<char*>(o0) +
                                                      static_cast<size_t>(obytes) * k);
                if constexpr (KIND == 0) {
                    select_store<R, EXACT_DIV, false, false>(S, uc, gx, gy, W, Himg, b, o, nullptr,
                                                             nullptr, cf, rtab);
                } else {
                    const bool clipped = KIND == 1 || !warp_interior || gy < R || gy >= Himg - R;
                    if (gx < W) {
                        if (clipped)
                            select_store<R, EXACT_DIV, true, false>(S, uc, gx, gy, W, Himg, b, o,
                                                                    nullptr, nullptr, cf, rtab);
                        else
                            select_store<R, EXACT_DIV, false, false>(S, uc, gx, gy, W, Himg, b, o,
                                                                     nullptr, nullptr, cf, rtab);
                    }
                }
            }
        }
    };

    for (int c = 0; c < nchunks; ++c) {
        const int q = c % NU, qp = (c + NU - 1) % NU;
        tma::mbar_wait(&ufull[q], (c / NU) & 1);
        const T* U = Ub + q * Ly::U_ELEMS;
        double* H = Hb + (c & 1) * Ly::H_ELEMS;
        // arm pass: task t = (row t / 8, segment t % 8)
#pragma unroll 1
        for (int t = tid; t < CH * Ly::NSEG; t += Ly::NT) {
            const int k = t >> 3, s = t & 7;
            walk_arm_segment<R, T, Ly::LS>(U + k * Ly::BW + s * Ly::LS + Ly::XOFF,
                                           H + k * Ly::HP + s * Ly::LS);
        }
        // H of chunk c complete; every thread is past chunk c - 1's walk, so
        // chunk c - 2's slot (last read as chunk c - 1's previous slot) is free
        __syncthreads();
        if (tid == 0 && c >= 2 && c - 2 + NU < nchunks) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            issue(c - 2 + NU);
        }
        const T* u = U + tid + Ly::RA;
        const T* uprev = Ub + qp * Ly::U_ELEMS + tid + Ly::RA;
        const double* h = H + tid;
        const int i0 = c * CH - 2 * R;  // output row index of the chunk's row 0
        const int gy0 = Y0 + i0;
        const bool rows_full = i0 >= 0 && i0 + CH <= nout && gy0 >= R && gy0 + CH <= Himg - R;
        auto run = [&](auto phase) {
            if (rows_full && warp_interior)
                chunk_rows(std::integral_constant<int, 0>{}, phase, h, u, uprev, i0);
            else if (rows_full)
                chunk_rows(std::integral_constant<int, 1>{}, phase, h, u, uprev, i0);
            else
                chunk_rows(std::integral_constant<int, 2>{}, phase, h, u, uprev, i0);
        };
        if constexpr (NP == 2) {
            if (c & 1)
                run(std::integral_constant<int, 1>{});
            else
                run(std::integral_constant<int, 0>{});
        } else {
            run(std::integral_constant<int, 0>{});
        }
    }
    if (gx < W)
        push_tail(band, out + static_cast<size_t>(b) * out_plane, out_pitch, gx, Y0, Y0 + nout);
}

// Row-block height of a launch (see launch_walk): 512 rows, halved down to
// 128 for a tall plane that would not give one wave of CTAs on its own.
inline int walk_block_rows(const Geometry& g, int strips) {
    static const int kBand = [] {
        const char* e = getenv("OSBF_GPU_WALK_BAND");  // diagnostic override
        const int v = e ? atoi(e) : 0;
        return v >= 64 ? v : 0;
    }();
    if (kBand) return kBand;
    int band_rows = 512;
    const int himg = g.img_h();
    while (himg >= 2048 && band_rows > 128 &&
           strips * ((himg + band_rows - 1) / band_rows) < 148 * 4)
        band_rows /= 2;
    return band_rows;
}

// The walk pays a serial block walk per CTA: under one wave of CTAs
// (148 SMs x 4) the tile kernels finish first (measured: 3 x 1920x1080 at
// r = 3 0.035 vs 0.105 ms, one 1024^2 plane at r = 8 0.016 vs 0.111 ms).
inline bool walk_fills(const Geometry& g) {
    const int strips = (g.width + 127) / 128;
    const int br = walk_block_rows(g, strips);
    const long long blocks = (g.out_row0 + g.height - 1) / br - g.out_row0 / br + 1;
    return static_cast<long long>(strips) * blocks * g.batch >= 148 * 4;
}

// Returns cudaErrorNotSupported (no launch) when the layout is not TMA-able.
template <int R, typename T, bool EXACT_DIV>
cudaError_t launch_walk(const PlaneView& in, const Geometry& g, double* out, size_t op,
                        size_t opl, cudaStream_t s) {
    using Ly = WLay<R, T>;
    if (op * sizeof(double) * Ly::CH > UINT32_MAX) return cudaErrorNotSupported;
    CUtensorMap map;
    const uint64_t plane_bytes = (g.batch > 1 ? in.plane : in.pitch * g.in_h()) * sizeof(T);
    if (!tma::encode_3d(&map, tma_dtype<T>(), in.base, g.width, g.in_h(), g.batch,
                        in.pitch * sizeof(T), plane_bytes, Ly::BW, Ly::CH))
        return cudaErrorNotSupported;
    static std::atomic<unsigned long long> done{0};
    if (cudaError_t e = ensure_smem(fast_walk_step<R, T, EXACT_DIV>, Ly::SMEM, done)) return e;
    // Row blocks (each re-reads a 2R-row halo) sit at fixed global rows,
    // never depending on the batch or on a row-band split aligned to them.
    const int strips = (g.width + Ly::SW - 1) / Ly::SW;
    // Block height: 512 rows; a tall single plane too small to give one wave
    // of CTAs (148 SMs x 4) halves it down to 128 (a 4096^2 plane: 1024
    // CTAs).  A function of the image's own size only (not the batch, not a
    // row band's extent), so batching and aligned row bands never change it.
    const int band_rows = walk_block_rows(g, strips);
    const int y0 = g.out_row0, y1 = g.out_row0 + g.height;
    dim3 grid(strips, (y1 - 1) / band_rows - y0 / band_rows + 1, g.batch);
    note_kernel("fast_walk_step");
    fast_walk_step<R, T, EXACT_DIV><<<grid, Ly::NT, Ly::SMEM, s>>>(map, out, op, opl, g.width,
                                                                   band_of(g), band_rows);
    return cudaGetLastError();
}

}  // namespace fastk
}  // namespace osbf_gpu
