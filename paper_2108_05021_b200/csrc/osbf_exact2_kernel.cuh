// Exact mode, fused path: bit-identical to the reference, O(1) HBM passes.
//
// The reference's table (integral.hpp:16-30) is the serial fp64 recurrence
//     R(x,y) = R(x-1,y) + U(x,y)          (row running sum, left to right)
//     C(x+1,y+1) = C(x+1,y) + R(x,y)      (table column, top to bottom)
// and every window sum is ((A-B)-C)+D over it (integral.hpp:48-49).  Any
// re-association changes roundings that decide exact ties, so this path
// replays the recurrence in the same order, split across two kernels:
//
//  K1 exact_row_carries : one serial chain per row (H*B chains); stores only
//                         the carries R(16s-1, y) (every SW=16 columns).
//  K2 exact_strip       : one CTA per TW=32-column strip of one plane walks
//                         the plane top to bottom in blocks of BR=32 rows:
//      L  stage U rows of the block (columns from the carry boundary left of
//         the halo to the right halo), cp.async for fp64 input
//      RR thread-per-row: continue R from the stored carry across the strip
//         (same serial adds as the reference)
//      CC thread-per-table-column: continue C down the block, into a ring
//      S  stencil of the PREVIOUS block's rows (their windows need table rows
//         up to y+R+1): 8 clipped ((A-B)-C)+D sums, division by the valid
//         count, |a-u|, strict < in window order, write a_m
//         (filters2d.hpp:69-84).
//
// Division: s/n for a positive integer n is computed as
//     q0 = s*y, r = fma(-q0, n, s) (exact), q = fma(r, y, q0), y = RN(1/n)
// which is the IEEE quotient: the exact s/n is never a rounding midpoint for
// an integer divisor, and q0 + r*y is within 1.5*2^-53 ulp of it, far closer
// than any midpoint (>= ulp/(4n) away).  tools/probes/divcheck.c and
// tests/test_division.py check it (exhaustively over the uint8 domain).
// Non-normal magnitudes take __ddiv_rn.
#pragma once

#include "osbf_internal.cuh"

namespace osbf_gpu {

// Out of line so the compiler cannot if-convert (speculate) it into the fast path.
static __device__ __noinline__ double div_slow(double s, double n) { return __ddiv_rn(s, n); }

// IEEE-exact s / n for a positive integer n with precomputed y = RN(1/n),
// valid when s == 0 or |s| in [2^-900, 2^900] (normal, finite quotient).
__device__ __forceinline__ double div_by_count_unguarded(double s, double n, double y) {
    const double q0 = __dmul_rn(s, y);
    const double r = __fma_rn(-q0, n, s);
    return __fma_rn(r, y, q0);
}

// Same, for any s (subnormal quotients and non-finite sums take __ddiv_rn).
__device__ __forceinline__ double div_by_count(double s, double n, double y) {
    const double q = div_by_count_unguarded(s, n, y);
    const unsigned hi = static_cast<unsigned>(__double2hiint(s)) & 0x7ff00000u;
    if (s != 0.0 && (hi - (123u << 20)) > ((1923u - 123u) << 20)) return div_slow(s, n);
    return q;
}

// A table value is "safe" when it is 0 or |v| in [2^-800, 2^900]: then every
// window sum ((A-B)-C)+D of safe values is 0 or a multiple of 2^-852 below
// 2^902, so div_by_count_unguarded is exact for it.
__device__ __forceinline__ bool table_value_safe(double v) {
    // integer-only: |v| == 0 or its exponent in [223, 1923] (no fp64 compare)
    const unsigned hi = static_cast<unsigned>(__double2hiint(v)) & 0x7fffffffu;
    const unsigned lo = static_cast<unsigned>(__double2loint(v));
    const unsigned e = hi & 0x7ff00000u;
    return ((hi | lo) == 0u) | ((e - (223u << 20)) <= ((1923u - 223u) << 20));
}

namespace ex2 {

#ifndef EXACT_BR32_MAX
#define EXACT_BR32_MAX 6  // largest radius walking 32-row blocks (measured: r = 7, 8 faster at 16)
#endif

constexpr int TW = 32;   // output columns per strip
constexpr int SW = 16;   // spacing of the stored row carries (columns)
constexpr int BR = 32;   // rows per block (radii <= 8; larger radii use 16, see XLay)
constexpr int NT = 256;  // threads per strip CTA
constexpr int NTK1 = 64; // threads per carry CTA (2 warps, 32 rows each)

template <int R, int NUBV = 3, bool SP = false>
struct XLay {
    static constexpr int RAD = R;
    // rows per block: 16 above r=8 halves the U / row-sum / ring footprint
    // (r=16: 149 KB -> 74 KB, one CTA per SM -> three); the single-phase
    // schedule (SP) always uses 16
    static constexpr int BR = (SP || R > EXACT_BR32_MAX) ? 16 : ex2::BR;
    // staged U columns: [xs, xs + NU) with xs = floor((X0-R)/SW)*SW >= X0-R-SW+1,
    // covering up to X0 + TW + R - 1
    static constexpr int NU = TW + 2 * R + SW;
    // pitch = 2 (mod 4) doubles: 16-byte aligned rows for 16-byte cp.async,
    // at most 2-way conflicts on the lanes = rows walk
    static constexpr int PUB = (NU % 4 == 2) ? NU : NU + 2;
    static constexpr int NCC = TW + 2 * R + 1;  // table columns cx in [X0-R, X0+TW+R]
    static constexpr int PR = NCC | 1;
    // table rows kept: [y0-BR-R, y0+BR] (2BR+R+1 rows; SP: one more block),
    // as a power of two
    static constexpr int SPAN = (SP ? 3 : 2) * BR + R + 2;
    static constexpr int NRING = SPAN <= 64 ? 64 : (SPAN <= 128 ? 128 : 256);
    static constexpr int U_ELEMS = BR * PUB;
    // row segments of SW columns between stored carries (RR parallelism)
    static constexpr int NSEGR = (NU + SW - 1) / SW;
    static_assert(NSEGR * BR <= NT, "row segments exceed the CTA");
    // U (+ carry) buffers: S(k-1), block k, RR(k+1) and NUB-3 more blocks in
    // flight; block k+NUB-1 is staged into S(k-1)'s buffer after iteration
    // k's last barrier.  The stencil strips use 3; the carries pass (no
    // stencil, short iterations) stages deeper to cover DRAM latency.
    static constexpr int NUB = NUBV;
    // staged-carry buffers: blocks k+1 .. k+NUB-1 can be in flight, i.e.
    // NUB-1 of them (2 for the stencil strips, which keeps r=8 at two CTAs
    // per SM)
    static constexpr int NCS = SP ? 3 : NUB - 1;
    static constexpr int NRB = SP ? 2 : 1;  // row-sum buffers (SP: double-buffered)
    static constexpr size_t SMEM = sizeof(double) * (NUB * static_cast<size_t>(U_ELEMS) +
                                                     NRB * BR * PR + NRING * NCC +
                                                     NCS * BR * NSEGR);
    // warps: column chains on [0, CCW), the early stencil rows on the rest;
    // row prefixes on [0, RRW), the late stencil rows on the rest
    static constexpr int CCW = (NCC + 31) / 32;
    static constexpr int RRW = (NSEGR * BR + 31) / 32;
    static_assert(CCW < NT / 32 && RRW < NT / 32, "no warps left for the stencil");
    static_assert(SPAN <= NRING, "table ring too small");
};

}  // namespace ex2
}  // namespace osbf_gpu

namespace osbf_gpu {
namespace ex2 {

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src),
                 "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// ---------------------------------------------------------------------------
// K1: row carries.  carries[g*nsc + s] = R(s*SW - 1, y) for s >= 1, 0 for s = 0
// (g = b*H + y).  One warp walks 32 rows; 32-column chunks are transposed
// through shared memory (lane = column on the load, lane = row on the scan)
// with a 3-stage cp.async ring for fp64 input.
constexpr int K1_STAGES = 3;
constexpr size_t K1_SMEM = sizeof(double) * (NTK1 / 32) * K1_STAGES * 32 * 33;

// Few rows (one plane): one warp per CTA with a deep ring, so each SM's
// single warp keeps ~8 chunks of loads in flight across the DRAM latency.
constexpr int K1D_STAGES = 8;
constexpr size_t K1D_SMEM = sizeof(double) * K1D_STAGES * 32 * 33;

template <typename T, int WARPS = NTK1 / 32, int K1_STAGES = ex2::K1_STAGES>
__global__ void __launch_bounds__(WARPS * 32)
    exact_row_carries(const T* __restrict__ in, size_t pitch, size_t plane,
                      double* __restrict__ carries, int W, int H, long long rows, int nsc) {
    extern __shared__ double k1s[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long row0 = (static_cast<long long>(blockIdx.x) * WARPS + warp) * 32;
    if (row0 >= rows) return;
    double* ring = k1s + static_cast<size_t>(warp) * K1_STAGES * 32 * 33;
    long long my_base = -1;
    {
        const long long g = row0 + lane;
        if (g < rows) {
            const long long b = g / H, y = g - b * H;
            my_base = b * static_cast<long long>(plane) + y * static_cast<long long>(pitch);
        }
    }
    const int nchunks = (W + 31) / 32;
    auto issue = [&](int c) {
        double* t = ring + (c % K1_STAGES) * 32 * 33;
        const int x = 32 * c + lane;
#pragma unroll 8
        for (int rr = 0; rr < 32; ++rr) {
            const long long base = __shfl_sync(0xffffffffu, my_base, rr);
            const bool ok = base >= 0 && x < W;
            if constexpr (sizeof(T) == 8) {
                cp_async8(t + lane * 33 + rr, reinterpret_cast<const double*>(in) + (ok ? base + x : 0),
                          ok);
            } else {
                t[lane * 33 + rr] = ok ? to_f64(in[base + x]) : 0.0;
            }
        }
        cp_commit();
    };
    for (int c = 0; c < K1_STAGES - 1; ++c) {
        if (c < nchunks) issue(c);
        else cp_commit();
    }
    double acc = 0.0;
    const long long g = row0 + lane;
    double* crow = carries + (g < rows ? g : 0) * nsc;
    if (g < rows) crow[0] = 0.0;
    for (int c = 0; c < nchunks; ++c) {
        if (c + K1_STAGES - 1 < nchunks) issue(c + K1_STAGES - 1);
        else cp_commit();
        cp_wait<K1_STAGES - 1>();
        __syncwarp();
        const double* t = ring + (c % K1_STAGES) * 32 * 33;
        const int n = min(32, W - 32 * c);
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            if (k < n) {
                acc = __dadd_rn(acc, t[k * 33 + lane]);  // row += src[x]  (integral.hpp:25)
                if ((k + 1) % SW == 0 && g < rows) crow[(32 * c + k + 1) / SW] = acc;
            }
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// K2: fused strip kernel (see the header comment).
template <typename L, typename T>
__device__ __forceinline__ void stage_block(const T* __restrict__ src, size_t pitch,
                                            const double* __restrict__ carries, int nsc, int s0,
                                            long long gbase, int xs, int y0, int W, int H,
                                            double* __restrict__ U, double* __restrict__ cs,
                                            bool aligned16) {
    constexpr int BR = L::BR;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if constexpr (sizeof(T) == 8) {
        // warp per row, 16-byte copies (xs is a multiple of SW = 16 columns)
        const bool vec = aligned16;
        for (int rr = warp; rr < BR; rr += NT / 32) {
            const int y = y0 + rr;
            const double* row = reinterpret_cast<const double*>(src) +
                                static_cast<size_t>(y < H ? y : 0) * pitch;
            double* d = U + rr * L::PUB;
            if (vec) {
                for (int p = lane; p < L::NU / 2; p += 32) {
                    const int x = xs + 2 * p;
                    const int nbytes = (y < H && x < W) ? (x + 1 < W ? 16 : 8) : 0;
                    const unsigned da = static_cast<unsigned>(__cvta_generic_to_shared(d + 2 * p));
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(da),
                                 "l"(row + (nbytes ? x : 0)), "r"(nbytes));
                }
            } else {
                for (int i = lane; i < L::NU; i += 32) {
                    const int x = xs + i;
                    const bool ok = y < H && x < W;
                    cp_async8(d + i, row + (ok ? x : 0), ok);
                }
            }
        }
    } else {
        for (int rr = warp; rr < BR; rr += NT / 32) {
            const int y = y0 + rr;
            for (int i = lane; i < L::NU; i += 32) {
                const int x = xs + i;
                U[rr * L::PUB + i] =
                    (y < H && x < W) ? to_f64(src[static_cast<size_t>(y) * pitch + x]) : 0.0;
            }
        }
    }
    // carries R(xs + 16*seg - 1, y) for the row segments (cs[seg*BR + row]),
    // asynchronously like the samples (a plain load here would hold the
    // issuing warps for a full DRAM latency before the next barrier)
    if (threadIdx.x < BR * L::NSEGR) {
        const int rr = threadIdx.x % BR, seg = threadIdx.x / BR;
        const int y = y0 + rr;
        const bool ok = y < H && s0 + seg < nsc;
        cp_async8(cs + threadIdx.x, carries + (ok ? (gbase + y) * nsc + s0 + seg : 0), ok);
    }
    cp_commit();
}

template <typename L>
__device__ __forceinline__ int ring_row(int cy) {
    return cy & (L::NRING - 1);
}

// Stencil of rows [yb, yb + nrows) for output column x (lane-owned).  SAFE:
// every table value of the strip so far passed table_value_safe.
template <typename L, bool SAFE>
__device__ __forceinline__ void stencil_rows(const double* __restrict__ Cr,
                                             const double* __restrict__ U, int xs, int X0, int yb,
                                             int r_lo, int r_hi, int w_first, int n_w, int W,
                                             int H, double* __restrict__ outp, size_t opitch,
                                             const double* __restrict__ rcp) {
    constexpr int R = L::RAD;
    const int lx = threadIdx.x & 31, grp = (threadIdx.x >> 5) - w_first;
    const int x = X0 + lx;
    if (x >= W || grp < 0 || grp >= n_w) return;
    const int cbase = X0 - R;  // table column of Cr index 0
    constexpr double kYq = 1.0 / ((R + 1) * (R + 1));
    constexpr double kYh = 1.0 / ((R + 1) * (2 * R + 1));
    constexpr double kNq = (R + 1) * (R + 1), kNh = (R + 1) * (2 * R + 1);
    const bool col_int = x >= R && x + R < W;
    double* op = outp + static_cast<size_t>(yb + r_lo + grp) * opitch + x;
    const size_t ostep = static_cast<size_t>(n_w) * opitch;
    for (int rr = r_lo + grp; rr < r_hi; rr += n_w, op += ostep) {
        const int y = yb + rr;
        const double u = U[rr * L::PUB + (x - xs)];
        double best = 0.0, best_abs = __longlong_as_double(0x7ff0000000000000LL);
        if (col_int && y >= R && y + R < H) {
            // 4x4 corner grid: rows {y-R, y, y+1, y+R+1}, cols {x-R, x, x+1, x+R+1}
            const double* rp[4] = {Cr + ring_row<L>(y - R) * L::NCC + lx,
                                   Cr + ring_row<L>(y) * L::NCC + lx,
                                   Cr + ring_row<L>(y + 1) * L::NCC + lx,
                                   Cr + ring_row<L>(y + R + 1) * L::NCC + lx};
            constexpr int co[4] = {0, R, R + 1, 2 * R + 1};
            double g[4][4];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int c = 0; c < 4; ++c) g[a][c] = rp[a][co[c]];
            // (ca, cb, ra, rb) per window in reference order (core.hpp:212-225)
            constexpr int W8[8][4] = {{0, 2, 1, 3}, {1, 3, 1, 3}, {1, 3, 0, 2}, {0, 2, 0, 2},
                                      {0, 2, 0, 3}, {1, 3, 0, 3}, {0, 3, 1, 3}, {0, 3, 0, 2}};
            double av[8], dv[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int ca = W8[i][0], cb = W8[i][1], ra = W8[i][2], rb = W8[i][3];
                const double s =
                    __dadd_rn(__dsub_rn(__dsub_rn(g[rb][cb], g[rb][ca]), g[ra][cb]), g[ra][ca]);
                av[i] = SAFE ? div_by_count_unguarded(s, i < 4 ? kNq : kNh, i < 4 ? kYq : kYh)
                             : div_by_count(s, i < 4 ? kNq : kNh, i < 4 ? kYq : kYh);
                dv[i] = fabs(__dsub_rn(av[i], u));
            }
            // With every |a_i - u| finite, "first i with the smallest d_i"
            // (strict <, filters2d.hpp:78) is what a stable depth-3 tournament
            // returns; non-finite pixels (NaN/inf input) keep the sequential
            // rule, under which such windows are never selected.  SAFE strips
            // have only finite, in-range table values (a non-finite sample u
            // would have made its table column non-finite), so every d_i is
            // finite there without checking.
            bool finite = SAFE;
            if (!SAFE) {
                const double dsum =
                    ((dv[0] + dv[1]) + (dv[2] + dv[3])) + ((dv[4] + dv[5]) + (dv[6] + dv[7]));
                finite = fabs(dsum) < __longlong_as_double(0x7ff0000000000000LL);
            }
            if (finite) {
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
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    if (dv[i] < best_abs) {
                        best_abs = dv[i];
                        best = av[i];
                    }
                }
            }
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const Win w = window(i, R);
                const int x0 = max(x + w.u0, 0), x1 = min(x + w.u1, W - 1);
                const int y0 = max(y + w.v0, 0), y1 = min(y + w.v1, H - 1);
                const double* ra = Cr + ring_row<L>(y0) * L::NCC;
                const double* rb = Cr + ring_row<L>(y1 + 1) * L::NCC;
                const double A = rb[x1 + 1 - cbase], Bv = rb[x0 - cbase];
                const double Cv = ra[x1 + 1 - cbase], D = ra[x0 - cbase];
                const double s = __dadd_rn(__dsub_rn(__dsub_rn(A, Bv), Cv), D);
                const int ni = (x1 - x0 + 1) * (y1 - y0 + 1);
                const double n = static_cast<double>(ni);
                const double a = div_by_count(s, n, rcp[ni]);
                const double d = fabs(__dsub_rn(a, u));
                if (d < best_abs) {
                    best_abs = d;
                    best = a;
                }
            }
        }
        *op = best;
    }
}

// CARRIES: walk the whole plane without the stencil and store the table
// values C(cx, band*band_h - BR) of the strip's own columns for every band
// >= 1 (ccar[(b*nbands + band)*(W+1) + cx]).  Otherwise, with band_h > 0,
// the CTA (blockIdx.z = band) outputs rows [band*band_h, +band_h): it starts
// one block above the band from those stored table values and walks one
// block past it (the band's last rows need table rows up to +R).
template <int R, typename T, bool CARRIES>
__global__ void __launch_bounds__(NT, 2)
    exact_strip(const T* __restrict__ in, size_t pitch, size_t plane,
                const double* __restrict__ carries, int nsc, double* __restrict__ out,
                size_t opitch, size_t oplane, int W, int H, int band_h,
                double* __restrict__ ccar) {
    using L = XLay<R, CARRIES ? 6 : 3>;
    constexpr int BR = L::BR;
    constexpr int AHEAD = L::NUB - 2;  // blocks staged ahead of the row prefixes
    extern __shared__ double sm[];
    double* Ubuf = sm;                          // NUB x [BR][PUB]
    double* Rb = sm + L::NUB * L::U_ELEMS;      // [BR][PR]:  Rb[rr][j] = R(X0-R-1+j, y0+rr)
    double* Cr = Rb + BR * L::PR;               // [NRING][NCC]: table rows, column cx = X0-R+t
    double* cs = Cr + L::NRING * L::NCC;        // NCS x [NSEGR][BR] staged carries
    const int b = blockIdx.y;
    const int X0 = blockIdx.x * TW;
    const int xs_raw = X0 - R;
    const int xs = xs_raw <= 0 ? 0 : (xs_raw / SW) * SW;
    const int s0 = xs / SW;
    const T* src = in + static_cast<size_t>(b) * plane;
    double* outp = out + static_cast<size_t>(b) * oplane;
    const long long gbase = static_cast<long long>(b) * H;
    const int tid = threadIdx.x;
    // RN(1/n) for every clipped window count (border pixels): one load
    // instead of an IEEE division per window
    __shared__ double rcp_tab[(2 * R + 1) * (R + 1) + 1];
    for (int n = threadIdx.x; n <= (2 * R + 1) * (R + 1); n += blockDim.x)
        rcp_tab[n] = n ? __ddiv_rn(1.0, static_cast<double>(n)) : 0.0;
    const int nbands = band_h > 0 ? (H + band_h - 1) / band_h : 1;
    const int band = CARRIES ? 0 : blockIdx.z;
    int y_out_lo = 0, y_out_hi = H, y_walk0 = 0, y_walk_end = H;
    if (!CARRIES && band_h > 0) {
        y_out_lo = band * band_h;
        y_out_hi = min(H, y_out_lo + band_h);
        y_walk0 = band == 0 ? 0 : y_out_lo - BR;
        y_walk_end = min(H, y_out_hi + BR);
    }
    if (CARRIES) y_walk_end = min(H, (nbands - 1) * band_h - BR);  // last band's start row
    const int nblocks = (y_walk_end - y_walk0 + BR - 1) / BR;
    const int xe = min(X0 + TW + R - 1, W - 1);  // last R column needed

    double creg = 0.0;    // running table column (threads < NCC)
    bool unsafe = false;  // some table value outside the unguarded-division range
    const int warp = tid >> 5;
    const bool aligned16 = sizeof(T) == 8 && (pitch % 2 == 0) &&
                           (reinterpret_cast<uintptr_t>(src) % 16 == 0);
    auto U_of = [&](int k) { return Ubuf + (k % L::NUB) * L::U_ELEMS; };
    auto cs_of = [&](int k) { return cs + (k % L::NCS) * BR * L::NSEGR; };
    auto stage = [&](int k) {  // block k, or an empty group past the end
        if (k < nblocks)
            stage_block<L, T>(src, pitch, carries, nsc, s0, gbase, xs, y_walk0 + k * BR, W, H,
                              U_of(k), cs_of(k), aligned16);
        else
            cp_commit();
    };

    // RR: continue the row running sums of block k from the stored carries,
    // one SW-column segment per thread (each segment starts from the exact
    // carry K1 stored, so the adds are the reference's serial chain).
    auto row_prefix = [&](int k) {
        if (tid >= BR * L::NSEGR) return;
        const int rr = tid % BR, seg = tid / BR;
        const double* u = U_of(k) + rr * L::PUB;
        const double* c = cs_of(k);
        double* rb = Rb + rr * L::PR;
        const int jbase = X0 - R - 1;  // x of Rb[0]
        if (seg == 0) {
            const int jfirst = xs - 1 - jbase;
            for (int j = 0; j < jfirst && j < L::NCC; ++j) rb[j] = 0.0;  // x < -1 (strip 0)
            if (jfirst >= 0 && jfirst < L::NCC) rb[jfirst] = c[rr];
        }
        const int xa = xs + seg * SW;
        double acc = c[seg * BR + rr];  // R(xa - 1)
        // operands first: the chain then waits on DADD latency only (the
        // shared loads cannot be hoisted past the rb stores by the compiler)
        double uv[SW];
#pragma unroll
        for (int i = 0; i < SW; ++i) uv[i] = xa + i <= xe ? u[seg * SW + i] : 0.0;
#pragma unroll
        for (int i = 0; i < SW; ++i) {
            const int x = xa + i;
            if (x <= xe) {
                acc = __dadd_rn(acc, uv[i]);  // row += src[x]
                const int j = x - jbase;
                if (j >= 0 && j < L::NCC) rb[j] = acc;
            }
        }
    };

    if (tid < L::NCC) {
        const int cx = X0 - R + tid;
        if (y_walk0 > 0 && cx >= 0 && cx <= W)
            creg = ccar[(static_cast<size_t>(b) * nbands + band) * (W + 1) + cx];
        unsafe = !table_value_safe(creg);
        Cr[ring_row<L>(y_walk0) * L::NCC + tid] = creg;  // table row y_walk0 (zero border at 0)
    }
    stage(0);
    cp_wait<0>();
    __syncthreads();
    for (int j = 1; j <= AHEAD; ++j) stage(j);  // land during the first iterations
    row_prefix(0);
    __syncthreads();
    const int early = BR - R - 1 > 0 ? BR - R - 1 : 0;  // rows of block k-1 not needing block k
    // stencil rows of block j = rows [yb, yb + BR) restricted to the band
    auto stencil_part = [&](int j, int r_from, int r_to, int w_first, int n_w, bool safe) {
        const int yb = y_walk0 + j * BR;
        const int lo = max(r_from, y_out_lo - yb), hi = min(min(r_to, H - yb), y_out_hi - yb);
        if (lo >= hi) return;
        if (safe)
            stencil_rows<L, true>(Cr, U_of(j), xs, X0, yb, lo, hi, w_first, n_w, W, H, outp,
                                  opitch, rcp_tab);
        else
            stencil_rows<L, false>(Cr, U_of(j), xs, X0, yb, lo, hi, w_first, n_w, W, H, outp,
                                   opitch, rcp_tab);
    };
    for (int k = 0; k < nblocks; ++k) {
        const int y0 = y_walk0 + k * BR;
        const int nrows = min(BR, H - y0);
        // Phase A: table columns of block k  ||  rows of block k-1 whose
        // windows end before block k's table rows (all but the last R+1)
        const bool safe_prev = !unsafe;
        if (warp < L::CCW) {
            bool unsafe_here = false;
            if (tid < L::NCC) {
                const int cx = X0 - R + tid;
                if (cx >= 0 && cx <= W) {
                    int rr = 0;
                    // full 8-row chunks with the row sums loaded ahead (see row_prefix)
                    for (; rr + 8 <= nrows; rr += 8) {
                        double rv[8];
#pragma unroll
                        for (int i = 0; i < 8; ++i) rv[i] = Rb[(rr + i) * L::PR + tid];
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            creg = __dadd_rn(creg, rv[i]);  // above[x+1] + row
                            unsafe_here |= !table_value_safe(creg);
                            Cr[ring_row<L>(y0 + rr + i + 1) * L::NCC + tid] = creg;
                        }
                    }
                    for (; rr < nrows; ++rr) {
                        creg = __dadd_rn(creg, Rb[rr * L::PR + tid]);
                        unsafe_here |= !table_value_safe(creg);
                        Cr[ring_row<L>(y0 + rr + 1) * L::NCC + tid] = creg;
                    }
                }
            }
            unsafe |= unsafe_here;
            if (CARRIES && tid >= R && tid < L::NCC) {
                // table row y0 + nrows is a band start row (band*band_h - BR)?
                const int cy = y0 + nrows, cx = X0 - R + tid;
                if ((cy + BR) % band_h == 0 && cx <= W && (tid < R + TW || cx == W)) {
                    const int bnd = (cy + BR) / band_h;
                    if (bnd >= 1 && bnd < nbands)
                        ccar[(static_cast<size_t>(b) * nbands + bnd) * (W + 1) + cx] = creg;
                }
            }
        } else if (!CARRIES && k > 0) {
            stencil_part(k - 1, 0, early, L::CCW, NT / 32 - L::CCW, safe_prev);
        }
        cp_wait<AHEAD - 1>();  // block k+1 staged
        unsafe = __syncthreads_or(unsafe);  // sticky for the strip
        // Phase B: row prefixes of block k+1  ||  the last R+1 rows of block k-1
        if (warp < L::RRW) {
            if (k + 1 < nblocks) row_prefix(k + 1);
        } else if (!CARRIES && k > 0) {
            stencil_part(k - 1, early, BR, L::RRW, NT / 32 - L::RRW, !unsafe);
        }
        __syncthreads();
        // block k+AHEAD+1 into the buffer S(k-1) just released
        stage(k + AHEAD + 1);
    }
    if (!CARRIES) stencil_part(nblocks - 1, 0, BR, 0, NT / 32, !unsafe);
}

// Single-phase schedule (radius <= kSpMaxRadius, 16-row blocks): iteration
// k runs, side by side with ONE barrier,
//   column chains of block k          (CC warps; row sums of block k)
//   row prefixes of block k+1         (RR warps; into the other row-sum buffer)
//   stencil of block k-2, all rows    (every table row it needs was written
//                                      by block k-1's chains; CC / RR warps
//                                      join it once their chains are done)
// Same adds, same table values, same stencil as exact_strip: bit-identical.
// Used for 9 <= r <= 12, where it measured 5-11% faster than exact_strip
// (5.25/5.65/5.53/5.50 -> 4.98/5.04/5.02/5.01 ms on C4); at r <= 8 it ties
// or loses (the two-phase kernel's 32-row blocks amortise better), and
// above 12 its table ring no longer fits two CTAs per SM.
constexpr int kSpMinRadius = 9, kSpMaxRadius = 12;

template <int R, typename T>
__global__ void __launch_bounds__(NT, 2)
    exact_strip_sp(const T* __restrict__ in, size_t pitch, size_t plane,
                   const double* __restrict__ carries, int nsc, double* __restrict__ out,
                   size_t opitch, size_t oplane, int W, int H, int band_h,
                   const double* __restrict__ ccar) {
    using L = XLay<R, 5, true>;
    constexpr int BR = L::BR;
    constexpr int CO = XLay<R, 6>::BR;  // the carries pass stores table rows band*band_h - CO
    extern __shared__ double sm[];
    double* Ubuf = sm;                              // NUB x [BR][PUB]
    double* Rb0 = sm + L::NUB * L::U_ELEMS;          // 2 x [BR][PR] row sums
    double* Cr = Rb0 + 2 * BR * L::PR;               // [NRING][NCC] table rows
    double* cs = Cr + L::NRING * L::NCC;             // NCS x [NSEGR][BR] staged carries
    const int b = blockIdx.y;
    const int X0 = blockIdx.x * TW;
    const int xs_raw = X0 - R;
    const int xs = xs_raw <= 0 ? 0 : (xs_raw / SW) * SW;
    const int s0 = xs / SW;
    const T* src = in + static_cast<size_t>(b) * plane;
    double* outp = out + static_cast<size_t>(b) * oplane;
    const long long gbase = static_cast<long long>(b) * H;
    const int tid = threadIdx.x, warp = tid >> 5;
    // RN(1/n) for every clipped window count (border pixels): one load
    // instead of an IEEE division per window
    __shared__ double rcp_tab[(2 * R + 1) * (R + 1) + 1];
    for (int n = threadIdx.x; n <= (2 * R + 1) * (R + 1); n += blockDim.x)
        rcp_tab[n] = n ? __ddiv_rn(1.0, static_cast<double>(n)) : 0.0;
    const int nbands = band_h > 0 ? (H + band_h - 1) / band_h : 1;
    const int band = blockIdx.z;
    int y_out_lo = 0, y_out_hi = H, y_walk0 = 0, y_walk_end = H;
    if (band_h > 0) {
        y_out_lo = band * band_h;
        y_out_hi = min(H, y_out_lo + band_h);
        y_walk0 = band == 0 ? 0 : y_out_lo - CO;
        y_walk_end = min(H, y_out_hi + BR);
    }
    const int nblocks = (y_walk_end - y_walk0 + BR - 1) / BR;
    const int xe = min(X0 + TW + R - 1, W - 1);
    const bool aligned16 = sizeof(T) == 8 && (pitch % 2 == 0) &&
                           (reinterpret_cast<uintptr_t>(src) % 16 == 0);
    auto U_of = [&](int k) { return Ubuf + (k % L::NUB) * L::U_ELEMS; };
    auto cs_of = [&](int k) { return cs + (k % L::NCS) * BR * L::NSEGR; };
    auto Rb_of = [&](int k) { return Rb0 + (k & 1) * BR * L::PR; };
    auto stage = [&](int k) {
        if (k < nblocks)
            stage_block<L, T>(src, pitch, carries, nsc, s0, gbase, xs, y_walk0 + k * BR, W, H,
                              U_of(k), cs_of(k), aligned16);
        else
            cp_commit();
    };
    auto row_prefix = [&](int k, int t) {  // t: thread index within the RR warps
        if (t >= BR * L::NSEGR) return;
        const int rr = t % BR, seg = t / BR;
        const double* u = U_of(k) + rr * L::PUB;
        const double* c = cs_of(k);
        double* rb = Rb_of(k) + rr * L::PR;
        const int jbase = X0 - R - 1;
        if (seg == 0) {
            const int jfirst = xs - 1 - jbase;
            for (int j = 0; j < jfirst && j < L::NCC; ++j) rb[j] = 0.0;
            if (jfirst >= 0 && jfirst < L::NCC) rb[jfirst] = c[rr];
        }
        const int xa = xs + seg * SW;
        double acc = c[seg * BR + rr];
#pragma unroll
        for (int i = 0; i < SW; ++i) {
            const int x = xa + i;
            if (x <= xe) {
                acc = __dadd_rn(acc, u[seg * SW + i]);  // row += src[x]
                const int j = x - jbase;
                if (j >= 0 && j < L::NCC) rb[j] = acc;
            }
        }
    };
    auto stencil_part = [&](int j, int r_from, int r_to, int w_first, int n_w, bool safe) {
        if (j < 0) return;
        const int yb = y_walk0 + j * BR;
        const int lo = max(r_from, y_out_lo - yb), hi = min(min(r_to, H - yb), y_out_hi - yb);
        if (lo >= hi) return;
        if (safe)
            stencil_rows<L, true>(Cr, U_of(j), xs, X0, yb, lo, hi, w_first, n_w, W, H, outp,
                                  opitch, rcp_tab);
        else
            stencil_rows<L, false>(Cr, U_of(j), xs, X0, yb, lo, hi, w_first, n_w, W, H, outp,
                                   opitch, rcp_tab);
    };

    double creg = 0.0;
    bool unsafe = false;
    if (tid < L::NCC) {
        const int cx = X0 - R + tid;
        if (y_walk0 > 0 && cx >= 0 && cx <= W)
            creg = ccar[(static_cast<size_t>(b) * nbands + band) * (W + 1) + cx];
        unsafe = !table_value_safe(creg);
        Cr[ring_row<L>(y_walk0) * L::NCC + tid] = creg;
    }
    stage(0);
    stage(1);
    stage(2);
    cp_wait<1>();  // blocks 0 and 1
    __syncthreads();
    row_prefix(0, tid);
    unsafe = __syncthreads_or(unsafe);
    // warps: [0, CCW) chains, [CCW, CCW+RRW) row prefixes, the rest stencil
    // rows [0, SPLIT) of block k-2; chain warps then take rows [SPLIT, BR)
    constexpr int CCW = L::CCW, RRW = L::RRW, NCH = CCW + RRW;
    constexpr int NST = NT / 32 - NCH;
    static_assert(NST >= 2, "no warps left for the stencil");
    constexpr int SPLIT = 12;  // measured best of 4..16 at r = 2, 8, 9..12
    for (int k = 0; k < nblocks; ++k) {
        const int y0 = y_walk0 + k * BR;
        const int nrows = min(BR, H - y0);
        const bool safe = !unsafe;  // covers every chain up to block k-1
        if (warp < CCW) {
            bool unsafe_here = false;
            if (tid < L::NCC) {
                const int cx = X0 - R + tid;
                const double* rb = Rb_of(k);
                if (cx >= 0 && cx <= W) {
                    for (int rr = 0; rr < nrows; ++rr) {
                        creg = __dadd_rn(creg, rb[rr * L::PR + tid]);  // above[x+1] + row
                        unsafe_here |= !table_value_safe(creg);
                        Cr[ring_row<L>(y0 + rr + 1) * L::NCC + tid] = creg;
                    }
                }
            }
            unsafe |= unsafe_here;
            stencil_part(k - 2, SPLIT, BR, 0, NCH, safe);
        } else if (warp < NCH) {
            if (k + 1 < nblocks) row_prefix(k + 1, tid - CCW * 32);
            stencil_part(k - 2, SPLIT, BR, 0, NCH, safe);
        } else {
            stencil_part(k - 2, 0, SPLIT, NCH, NST, safe);
        }
        cp_wait<0>();  // block k+2 staged (for the row prefixes of the next iteration)
        unsafe = __syncthreads_or(unsafe);
        stage(k + 3);  // into block k-2's buffer, whose stencil just finished
    }
    // the last two blocks' stencils (their table rows are all written)
    stencil_part(nblocks - 2, 0, BR, 0, NT / 32, !unsafe);
    stencil_part(nblocks - 1, 0, BR, 0, NT / 32, !unsafe);
}

}  // namespace ex2

// One radius (instantiated in osbf_exact2_rNN.cu).
template <int R>
cudaError_t exact2_launch_radius(const PlaneView& in, const Geometry& g, double* carries,
                                 int nsc, double* out, size_t opitch, size_t oplane, int band_h,
                                 double* ccar, cudaStream_t s) {
    using L = ex2::XLay<R>;      // stencil strips
    using LC = ex2::XLay<R, 6>;  // carries pass (deeper staging)
    const int strips = (g.width + ex2::TW - 1) / ex2::TW;
    const int nbands = band_h > 0 ? (g.height + band_h - 1) / band_h : 1;
    auto go = [&](auto tag) -> cudaError_t {
        using T = decltype(tag);
        static std::atomic<unsigned long long> done_s{0}, done_c{0};
        cudaError_t e0 = ensure_smem(ex2::exact_strip<R, T, false>, L::SMEM, done_s);
        if (e0 == cudaSuccess) e0 = ensure_smem(ex2::exact_strip<R, T, true>, LC::SMEM, done_c);
        if (e0 != cudaSuccess) return e0;
        const T* base = static_cast<const T*>(in.base);
        if (nbands > 1) {
            ex2::exact_strip<R, T, true><<<dim3(strips, g.batch, 1), ex2::NT, LC::SMEM, s>>>(
                base, in.pitch, in.plane, carries, nsc, out, opitch, oplane, g.width, g.height,
                band_h, ccar);
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) return e;
        }
        if constexpr (R >= ex2::kSpMinRadius && R <= ex2::kSpMaxRadius) {
            {
                using LS = ex2::XLay<R, 5, true>;
                static std::atomic<unsigned long long> done_sp{0};
                if (cudaError_t e = ensure_smem(ex2::exact_strip_sp<R, T>, LS::SMEM, done_sp))
                    return e;
                ex2::exact_strip_sp<R, T>
                    <<<dim3(strips, g.batch, nbands), ex2::NT, LS::SMEM, s>>>(
                        base, in.pitch, in.plane, carries, nsc, out, opitch, oplane, g.width,
                        g.height, nbands > 1 ? band_h : 0, ccar);
                return cudaGetLastError();
            }
        }
        ex2::exact_strip<R, T, false><<<dim3(strips, g.batch, nbands), ex2::NT, L::SMEM, s>>>(
            base, in.pitch, in.plane, carries, nsc, out, opitch, oplane, g.width, g.height,
            nbands > 1 ? band_h : 0, ccar);
        return cudaGetLastError();
    };
    switch (in.dtype) {
        case OSBF_U8: return go(uint8_t{});
        case OSBF_F32: return go(float{});
        default: return go(double{});
    }
}

}  // namespace osbf_gpu
