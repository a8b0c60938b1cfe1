// Fast-mode kernel templates.
#pragma once
// Fast mode: one OSBF pass with local fp64 box sums (no whole-image prefix).
// Which kernel runs (launch_dtype below):
//   r <= 4      fast_tma_step     one TMA-staged tile per CTA, each column
//                                 thread forms its arms from 2r+1 loads
//   5 <= r <= 16  fast_stream_step  column strips streamed through a TMA ring
//                                 with register prefix rings
//                                 (osbf_fast_stream.cuh)
//   otherwise   fast_sep_step     the two-phase tile kernel described here:
//                                 layouts TMA cannot describe, and the
//                                 per-pixel diagnostics (means / selection)
//
// fast_sep_step: each CTA owns a TW x TH output tile.  It stages the tile plus an R-pixel
// halo in shared memory (zero outside the image, so clipped window sums need
// no special casing; only the valid counts do, integral.hpp:53-61) and
// evaluates the eight one-sided windows of the reference (core.hpp:212-225)
// separably, in two phases:
//
//   Phase A (thread per tile row, walking x):  H(x,j) = sum_{u=-R..0} U(x+u, j)
//            the "left arm" of every row; H(x+R, j) is the right arm.
//   Phase B (thread per output column, walking y) combines vertical sums of
//            three fields, F1 = H(x,.), F2 = H(x+R,.), F3 = U(x,.):
//              Up(F) = sum over rows [y-R, y],  Dn(F) = sum over rows [y, y+R]
//            and forms the eight windows
//              w1 = Dn(F1)  w2 = Dn(F2)  w3 = Up(F2)  w4 = Up(F1)
//              w5 = Up(F1)+Dn(F1)-F1(y)   w6 = Up(F2)+Dn(F2)-F2(y)
//              w7 = Dn(F1)+Dn(F2)-Dn(F3)  w8 = Up(F1)+Up(F2)-Up(F3)
//            then the valid-count means (integral.hpp:64-69), |a - u| and the
//            strict-< first-minimum selection (filters2d.hpp:72-82).  Lanes
//            are consecutive columns, so the output stores are coalesced.
//
// The radius is a template parameter (1..kFastMaxRadius): every shared-memory
// offset is an immediate; for small radii the walks are fully unrolled, so
// values loaded once stay in registers for their whole window.
// Interior tiles (no clipping anywhere) run a body with constant window counts;
// border tiles run a body with per-pixel valid counts.  Work per pixel is O(1)
// in R; sums never touch a whole-image prefix.
//
// Numerics: fp64 throughout.  Float input: selection on d_i = S_i/n_i - u
// computed as fma(S_i, 1/n_i, -u), output u + d_m (a few ulps from the
// reference's a_m; the tolerance is checked in tests).  uint8 input
// (EXACT_DIV): sums are exact integers in any order, a_i = S_i/n_i is IEEE,
// d_i = |a_i - u| and the output is a_m -> bit-identical to the reference.
#include <string.h>

#include "osbf_internal.cuh"
#include "osbf_tma.cuh"

namespace osbf_gpu {
namespace fastk {

constexpr int TW = 64;   // output tile width  (Phase B: one thread column each)
constexpr int TH = 64;   // output tile height
constexpr int NT = 256;  // threads per CTA
constexpr int NSB = NT / TW;    // Phase B row segments per column
constexpr int SEGB = TH / NSB;  // rows per Phase B segment
constexpr int kUnrollRadius = 4;  // full unroll (register ring) up to this radius

// Rows of one launch in global image coordinates (see Geometry).
struct Band {
    int h_img;   // image height: windows clip at [0, h_img)
    int y_in0;   // global row of input buffer row 0
    int in_rows; // rows held by the input buffer: [y_in0, y_in0 + in_rows)
    int y_out0;  // global row of output buffer row 0 (first output row)
    int y_end;   // one past the last output row (global)
    double* push_up;  // fused halo push (see Geometry); null = none
    double* push_dn;
    int push_rows;
    long long push_pitch;
};
inline Band band_of(const Geometry& g) {
    return Band{g.img_h(),  g.in_row0,  g.in_h(),  g.out_row0,    g.out_row0 + g.height,
                g.push_up,  g.push_dn,  g.push_rows,   static_cast<long long>(g.push_pitch)};
}

// Tile-row order of a launch: in row-band mode with the fused halo push the
// band's first and last tile rows run first (rows 0, n-1, 1, n-2, ...), so
// the pushes into the neighbours' halos fly while the interior is computed.
__device__ __forceinline__ int tile_row(const Band& bd) {
    const int i = blockIdx.y, n = gridDim.y;
    if (bd.push_rows == 0) return i;
    return (i & 1) ? n - 1 - (i >> 1) : (i >> 1);
}

// Fused halo exchange: a band's first / last push_rows output rows are also
// written straight into the neighbours' halo rows (peer memory over NVLink
// when the ranks are GPUs), so no separate exchange step follows the pass.
// Each thread forwards the rows [ya, yb) of column gx it has just stored to
// outp (row gy at (gy - y_out0) * pitch + gx): a re-read of its own stores,
// outside the per-pixel loop.
__device__ __forceinline__ void push_tail(const Band& bd, const double* outp, size_t pitch, int gx,
                                          int ya, int yb) {
    if (bd.push_rows == 0) return;
    if (bd.push_up) {
        for (int gy = max(ya, bd.y_out0); gy < min(yb, bd.y_out0 + bd.push_rows); ++gy)
            bd.push_up[static_cast<long long>(gy - bd.y_out0) * bd.push_pitch + gx] =
                outp[static_cast<size_t>(gy - bd.y_out0) * pitch + gx];
    }
    if (bd.push_dn) {
        const int y0 = bd.y_end - bd.push_rows;
        for (int gy = max(ya, y0); gy < min(yb, bd.y_end); ++gy)
            bd.push_dn[static_cast<long long>(gy - y0) * bd.push_pitch + gx] =
                outp[static_cast<size_t>(gy - bd.y_out0) * pitch + gx];
    }
}

template <int R>
struct Lay {
    static constexpr int LH = TH + 2 * R;      // staged rows
    static constexpr int LWU = TW + 2 * R;     // staged columns of U
    static constexpr int PU = LWU | 1;         // odd pitch: conflict-free row walks
    static constexpr int LWH = TW + R;         // columns of H: H(X0 + k), k < LWH
    static constexpr int PH = LWH | 1;
    static constexpr int PER_ROW = (NT / LH) > 0 ? (NT / LH) : 1;  // Phase A threads per row
    static constexpr int SEGA = (LWH + PER_ROW - 1) / PER_ROW;     // Phase A walk length
    static constexpr int NRT = 2 * R + 2;      // reciprocal table 1/k, k < NRT
    static constexpr size_t SMEM = sizeof(double) * (static_cast<size_t>(LH) * (PU + PH) + NRT);
    // 3 CTAs/SM when shared memory (incl. the 1 KB driver reserve per CTA)
    // allows it; the register budget then caps at 80/thread.
    template <bool SLOW>
    static constexpr int min_ctas() {
        return (!SLOW && (SMEM + 1024) * 3 <= 228 * 1024) ? 3 : 2;
    }
};

__device__ __forceinline__ void cp_async_f64(double* dst, const double* src, bool valid) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    const int n = valid ? 8 : 0;  // src-size 0 -> zero fill
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(n));
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// Stage U rows [Y0-R, Y0+TH+R) x cols [X0-R, X0+TW+R), zero outside the image.
template <int R, typename T, bool BORDER>
__device__ __forceinline__ void stage_tile(const T* __restrict__ src, size_t pitch, int X0,
                                           int Y0, int W, const Band& band,
                                           double* __restrict__ Us) {
    using Ly = Lay<R>;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int CHUNKS = (Ly::LWU + 31) / 32;
    for (int j = warp; j < Ly::LH; j += NT / 32) {
        const int gy = Y0 - R + j;  // global row; buffer row gy - y_in0
        // rows outside the image read as zero; so do rows outside the caller's
        // band buffer (they are only ever outside the windows' image part)
        const bool row_in = !BORDER || (gy >= 0 && gy < band.h_img && gy >= band.y_in0 &&
                                        gy < band.y_in0 + band.in_rows);
        const T* rowp = src + static_cast<size_t>(row_in ? gy - band.y_in0 : 0) * pitch;
#pragma unroll
        for (int c = 0; c < CHUNKS; ++c) {
            const int i = lane + 32 * c;
            if (i < Ly::LWU) {
                const int gx = X0 - R + i;
                const bool ok = row_in && (!BORDER || (gx >= 0 && gx < W));
                if constexpr (sizeof(T) == 8) {
                    cp_async_f64(Us + j * Ly::PU + i,
                                 reinterpret_cast<const double*>(rowp) + (ok ? gx : 0), ok);
                } else {
                    Us[j * Ly::PU + i] = ok ? to_f64(rowp[gx]) : 0.0;
                }
            }
        }
    }
    if constexpr (sizeof(T) == 8) cp_async_wait_all();
}

// Phase A: Hs[j][k] = sum_{i=k}^{k+R} Us[j][i] for k < LWH (lanes = rows).
template <int R>
__device__ __forceinline__ void arm_sums(const double* __restrict__ Us, double* __restrict__ Hs) {
    using Ly = Lay<R>;
    const int tid = threadIdx.x;
    const int j = tid % Ly::LH, s = tid / Ly::LH;
    if (s >= Ly::PER_ROW) return;
    const int k0 = s * Ly::SEGA;
    const double* __restrict__ u = Us + j * Ly::PU + k0;
    double* __restrict__ h = Hs + j * Ly::PH + k0;
    if (k0 + Ly::SEGA <= Ly::LWH) {
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i <= R; ++i) acc += u[i];
        h[0] = acc;
#pragma unroll(R <= kUnrollRadius ? Ly::SEGA : 4)
        for (int k = 1; k < Ly::SEGA; ++k) {
            acc += u[k + R] - u[k - 1];
            h[k] = acc;
        }
    } else {  // last, shorter segment
        const int n = Ly::LWH - k0;
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i <= R; ++i) acc += u[i];
        h[0] = acc;
        for (int k = 1; k < n; ++k) {
            acc += u[k + R] - u[k - 1];
            h[k] = acc;
        }
    }
}

// Per-window valid counts at (gx, gy) (integral.hpp:53-61, clipped ranges).
struct Counts {
    int n[8];
};
template <int R>
__device__ __forceinline__ Counts border_counts(int gx, int gy, int W, int H) {
    const int ncl = min(gx, R) + 1, ncr = min(W - 1 - gx, R) + 1;
    const int nru = min(gy, R) + 1, nrd = min(H - 1 - gy, R) + 1;
    Counts c;
    c.n[0] = ncl * nrd;
    c.n[1] = ncr * nrd;
    c.n[2] = ncr * nru;
    c.n[3] = ncl * nru;
    c.n[4] = ncl * (nru + nrd - 1);
    c.n[5] = ncr * (nru + nrd - 1);
    c.n[6] = (ncl + ncr - 1) * nrd;
    c.n[7] = (ncl + ncr - 1) * nru;
    return c;
}

// Valid-count factors of one column (border tiles): 1/ncl, 1/ncr, 1/(ncl+ncr-1).
struct ColFactors {
    double cL, cR, cF;
};

// Means, |a-u| selection and the store for one pixel (S = the eight window
// sums in reference order, u = the centre sample).
template <int R, bool EXACT_DIV, bool BORDER, bool DIAG, bool FAST_SEQ = false,
          bool INT_SEL = false>
__device__ __forceinline__ double select_store(const double (&S)[8], double u, int gx, int gy,
                                             int W, int H, int b, double* __restrict__ o,
                                             double* __restrict__ means,
                                             uint8_t* __restrict__ sel, const ColFactors& cf,
                                             const double* __restrict__ rtab) {
    // Interior reciprocals formed exactly as the border path forms them
    // (product of the per-axis reciprocals), so a pixel gets the same factor
    // whichever tile kind it sits in: results do not depend on the tiling and
    // row bands equal the whole image bit for bit.
    constexpr double kR1 = 1.0 / (R + 1), kR2 = 1.0 / (2 * R + 1);
    constexpr double kRq = kR1 * kR1;
    constexpr double kRh = kR1 * kR2;
    constexpr int kNq = (R + 1) * (R + 1), kNh = (R + 1) * (2 * R + 1);
    if (EXACT_DIV || DIAG) {
        // Reference arithmetic: a_i = S_i / n_i (IEEE), d_i = |a_i - u|,
        // strict < in window order, output a_m (filters2d.hpp:74-83).
        Counts cn;
        if (BORDER) {
            cn = border_counts<R>(gx, gy, W, H);
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) cn.n[i] = i < 4 ? kNq : kNh;
        }
        double best = 0.0, best_abs = __longlong_as_double(0x7ff0000000000000LL);
        int best_id = 0;
        const size_t pix = (static_cast<size_t>(b) * H + gy) * W + gx;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const double a = EXACT_DIV ? __ddiv_rn(S[i], static_cast<double>(cn.n[i]))
                                       : S[i] * (BORDER ? 1.0 / cn.n[i] : (i < 4 ? kRq : kRh));
            if (DIAG && means) means[pix * 8 + i] = a;
            const double d = fabs(a - u);
            if (d < best_abs) {
                best_abs = d;
                best = a;
                best_id = i + 1;
            }
        }
        if (DIAG && sel) sel[pix] = static_cast<uint8_t>(best_id);
        if (!DIAG || o) *o = best;
        return best;
    }
    // 1/n_i: interior constants, or products of clipped row/column factors
    // 1/n_row * 1/n_col from the per-CTA table (border tiles).
    double rc[8];
    if (BORDER) {
        const int nru = min(gy, R) + 1, nrd = min(H - 1 - gy, R) + 1;
        const double rU = rtab[nru], rD = rtab[nrd], rF = rtab[nru + nrd - 1];
        rc[0] = cf.cL * rD; rc[1] = cf.cR * rD; rc[2] = cf.cR * rU; rc[3] = cf.cL * rU;
        rc[4] = cf.cL * rF; rc[5] = cf.cR * rF; rc[6] = cf.cF * rD; rc[7] = cf.cF * rU;
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) rc[i] = i < 4 ? kRq : kRh;
    }
    // d_i = S_i/n_i - u in one rounding; the first minimum of |d_i|
    // (filters2d.hpp:78 strict <), output u + d_m.  (Carrying S_m to output
    // S_m / n_m costs 14 selects per pixel, measured 11-14% of a pass on
    // these issue-bound kernels; the result is within 1 ulp of it and the
    // sums themselves already differ from the reference's whole-image table
    // by rounding.)  FAST_SEQ: a sequential strict-< scan (2 live values, for
    // register-capped kernels); else a stable depth-3 tournament.  Finite
    // input assumed (non-finite samples: use exact mode).
    double best;
    if constexpr (INT_SEL) {
        // |d| compared on the integer pipe: for finite doubles the sign-cleared
        // bit patterns order like the magnitudes (ties equal), so a stable
        // tournament on (key, d) picks the same first minimum
        double d[8];
        long long k[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            d[i] = fma(S[i], rc[i], -u);
            k[i] = __double_as_longlong(d[i]) & 0x7fffffffffffffffLL;
        }
        auto pk = [](long long& ka, double& da, long long kc, double dc) {
            const bool p = kc < ka;
            ka = p ? kc : ka;
            da = p ? dc : da;
        };
        pk(k[0], d[0], k[1], d[1]);
        pk(k[2], d[2], k[3], d[3]);
        pk(k[4], d[4], k[5], d[5]);
        pk(k[6], d[6], k[7], d[7]);
        pk(k[0], d[0], k[2], d[2]);
        pk(k[4], d[4], k[6], d[6]);
        pk(k[0], d[0], k[4], d[4]);
        best = d[0];
    } else if constexpr (FAST_SEQ) {
        best = fma(S[0], rc[0], -u);
#pragma unroll
        for (int i = 1; i < 8; ++i) {
            const double d = fma(S[i], rc[i], -u);
            best = fabs(d) < fabs(best) ? d : best;
        }
    } else {
        double d[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) d[i] = fma(S[i], rc[i], -u);
        auto pick = [](double a, double c) { return fabs(c) < fabs(a) ? c : a; };
        best = pick(pick(pick(d[0], d[1]), pick(d[2], d[3])),
                    pick(pick(d[4], d[5]), pick(d[6], d[7])));
    }
    const double v = u + best;
    *o = v;
    return v;
}

// Phase B for one thread: output column x, rows [y0, y0 + SEGB) of the tile.
//
// Small radii (R <= kUnrollRadius): fully unrolled over column prefix sums
//   P1(j) = sum_{j'<=j} F1, P2 likewise, Q(j) = sum (F1 + F2 - F3), so that
//   w4 = P1(y+R)-P1(y-1)   w1 = P1(y+2R)-P1(y+R-1)   w5 = P1(y+2R)-P1(y-1)
//   w3 = P2(y+R)-P2(y-1)   w2 = P2(y+2R)-P2(y+R-1)   w6 = P2(y+2R)-P2(y-1)
//   w8 = Q(y+R)-Q(y-1)     w7 = Q(y+2R)-Q(y+R-1)
//   (one subtraction per window; every value stays in registers).
// Larger radii: rolled loop with running Up/Dn sums (register pressure),
//   pointers advance one row per step, every offset is an immediate.
template <int R, bool EXACT_DIV, bool BORDER, bool DIAG>
__device__ __forceinline__ void column_walk(const double* __restrict__ Us,
                                            const double* __restrict__ Hs, int X0, int Y0,
                                            int W, const Band& band, int b,
                                            double* __restrict__ outp,
                                            size_t out_pitch, double* __restrict__ means,
                                            uint8_t* __restrict__ sel,
                                            const double* __restrict__ rtab) {
    using Ly = Lay<R>;
    const int x = threadIdx.x % TW, s = threadIdx.x / TW;
    const int gx = X0 + x;
    if (BORDER && gx >= W) return;
    ColFactors cf{0.0, 0.0, 0.0};
    if (BORDER) {
        const int ncl = min(gx, R) + 1, ncr = min(W - 1 - gx, R) + 1;
        cf = ColFactors{rtab[ncl], rtab[ncr], rtab[ncl + ncr - 1]};
    }
    const int y0 = s * SEGB;
    const double* f1 = Hs + y0 * Ly::PH + x;      // F1(j) = f1[j*PH]
    const double* f2 = Hs + y0 * Ly::PH + x + R;  // F2(j)
    const double* f3 = Us + y0 * Ly::PU + x + R;  // F3(j)
    const int H = band.h_img;
    double* o = outp ? outp + static_cast<size_t>(Y0 + y0 - band.y_out0) * out_pitch + gx : nullptr;
#define F1(j) f1[(j) * Ly::PH]
#define F2(j) f2[(j) * Ly::PH]
#define F3(j) f3[(j) * Ly::PU]
    if constexpr (R <= kUnrollRadius) {
        constexpr int NJ = SEGB + 2 * R;  // rows touched by this segment
        double P1[NJ + 1], P2[NJ + 1], Q[NJ + 1], Uc[NJ];
        P1[0] = P2[0] = Q[0] = 0.0;  // P(j) lives at index j + 1
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            const double a = F1(j), c = F2(j), e = F3(j);
            Uc[j] = e;
            P1[j + 1] = P1[j] + a;
            P2[j + 1] = P2[j] + c;
            Q[j + 1] = Q[j] + ((a + c) - e);
            const int y = j - 2 * R;  // output row whose windows complete at row j
            if (y >= 0) {
                const int gy = Y0 + y0 + y;
                if (BORDER && gy >= band.y_end) break;
                const double S[8] = {P1[y + 2 * R + 1] - P1[y + R], P2[y + 2 * R + 1] - P2[y + R],
                                     P2[y + R + 1] - P2[y],         P1[y + R + 1] - P1[y],
                                     P1[y + 2 * R + 1] - P1[y],     P2[y + 2 * R + 1] - P2[y],
                                     Q[y + 2 * R + 1] - Q[y + R],   Q[y + R + 1] - Q[y]};
                select_store<R, EXACT_DIV, BORDER, DIAG>(
                    S, Uc[y + R], gx, gy, W, H, b, o ? o + static_cast<size_t>(y) * out_pitch : o,
                    means, sel, cf, rtab);
            }
        }
    } else {
        // Up(y) = sum_{j=y}^{y+R} F(j), Dn(y) = sum_{j=y+R}^{y+2R} F(j) (rows relative to y0)
        double up1 = 0.0, up2 = 0.0, up3 = 0.0, dn1 = 0.0, dn2 = 0.0, dn3 = 0.0;
#pragma unroll
        for (int j = 0; j <= R; ++j) {
            up1 += F1(j);
            up2 += F2(j);
            up3 += F3(j);
            dn1 += F1(j + R);
            dn2 += F2(j + R);
            dn3 += F3(j + R);
        }
        double c1 = F1(R), c2 = F2(R), u = F3(R);
#pragma unroll 1
        for (int y = 0; y < SEGB; ++y) {
            if (y > 0) {
                const double n1 = F1(R), n2 = F2(R), n3 = F3(R);  // pointers already advanced
                up1 += n1 - F1(-1);
                up2 += n2 - F2(-1);
                up3 += n3 - F3(-1);
                dn1 += F1(2 * R) - c1;
                dn2 += F2(2 * R) - c2;
                dn3 += F3(2 * R) - u;
                c1 = n1;
                c2 = n2;
                u = n3;
            }
            const int gy = Y0 + y0 + y;
            if (BORDER && gy >= band.y_end) break;
            const double S[8] = {dn1, dn2, up2, up1, up1 + dn1 - c1, up2 + dn2 - c2,
                                 dn1 + dn2 - dn3, up1 + up2 - up3};
            select_store<R, EXACT_DIV, BORDER, DIAG>(
                S, u, gx, gy, W, H, b, o ? o + static_cast<size_t>(y) * out_pitch : o, means, sel,
                cf, rtab);
            f1 += Ly::PH;
            f2 += Ly::PH;
            f3 += Ly::PU;
        }
    }
#undef F1
#undef F2
#undef F3
}

template <int R, typename T, bool EXACT_DIV, bool DIAG>
__global__ void __launch_bounds__(NT, Lay<R>::template min_ctas<EXACT_DIV || DIAG>())
    fast_sep_step(const T* __restrict__ in, size_t in_pitch, size_t in_plane,
                  double* __restrict__ out, size_t out_pitch, size_t out_plane,
                  double* __restrict__ means, uint8_t* __restrict__ sel, int W, Band band) {
    extern __shared__ double smem[];
    using Ly = Lay<R>;
    double* Us = smem;                   // [LH][PU]: tile row j <-> image row Y0 - R + j
    double* Hs = smem + Ly::LH * Ly::PU;  // [LH][PH]: Hs[j][k] = H(X0 + k, row j)
    const int X0 = blockIdx.x * TW, Y0 = band.y_out0 + blockIdx.y * TH, b = blockIdx.z;
    const T* src = in + static_cast<size_t>(b) * in_plane;
    double* outp = out ? out + static_cast<size_t>(b) * out_plane : nullptr;
    double* rtab = Hs + Ly::LH * Ly::PH;  // [NRT]: rtab[k] = 1/k
    if (threadIdx.x < Ly::NRT) rtab[threadIdx.x] = threadIdx.x ? 1.0 / threadIdx.x : 0.0;
    const bool interior = X0 >= R && X0 + TW + R <= W && Y0 >= R &&
                          Y0 + TH + R <= band.h_img && Y0 + TH <= band.y_end;
    if (interior) {
        stage_tile<R, T, false>(src, in_pitch, X0, Y0, W, band, Us);
    } else {
        stage_tile<R, T, true>(src, in_pitch, X0, Y0, W, band, Us);
    }
    __syncthreads();
    arm_sums<R>(Us, Hs);
    __syncthreads();
    if (interior) {
        column_walk<R, EXACT_DIV, false, DIAG>(Us, Hs, X0, Y0, W, band, b, outp, out_pitch,
                                               means, sel, rtab);
    } else {
        column_walk<R, EXACT_DIV, true, DIAG>(Us, Hs, X0, Y0, W, band, b, outp, out_pitch,
                                              means, sel, rtab);
    }
    if (!DIAG && band.push_rows && outp) {  // row-band mode with the fused halo push
        const int gx = X0 + threadIdx.x % TW, ya = Y0 + (threadIdx.x / TW) * SEGB;
        if (gx < W) push_tail(band, outp, out_pitch, gx, ya, min(ya + SEGB, band.y_end));
    }
}

template <int R, typename T, bool EXACT_DIV, bool DIAG>
cudaError_t launch_r(const PlaneView& in, const Geometry& g, double* out, size_t op, size_t opl,
                     double* means, uint8_t* sel, cudaStream_t s) {
    constexpr size_t smem = Lay<R>::SMEM;
    static std::atomic<unsigned long long> done{0};
    if (cudaError_t e = ensure_smem(fast_sep_step<R, T, EXACT_DIV, DIAG>, smem, done))
        return e;
    dim3 grid((g.width + TW - 1) / TW, (g.height + TH - 1) / TH, g.batch);
    note_kernel(DIAG ? "fast_sep_step (diagnostics)" : "fast_sep_step");
    fast_sep_step<R, T, EXACT_DIV, DIAG><<<grid, NT, smem, s>>>(
        static_cast<const T*>(in.base), in.pitch, in.plane, out, op, opl, means, sel, g.width,
        band_of(g));
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Small radii (R <= kUnrollRadius): TMA-staged tile, no separate Phase A.
//
// One thread issues a single cp.async.bulk.tensor for the whole (TW+2R) x
// (TH+2R) tile (hardware zero-fill outside the image); the column threads
// then form F1 = sum Us[j][x..x+R], F2 = sum Us[j][x+R..x+2R] themselves
// (2R+1 conflict-free loads per row, consecutive lanes = consecutive x) and
// run the prefix-sum walk.  The input is read in its own dtype (u8 / f32 /
// f64) and promoted to fp64 in registers, so the first pass needs no
// conversion kernel.
// Radii with the TMA direct kernel, and with the two-pass (temporally
// blocked) kernel.
constexpr int kTmaRadius = 4;
constexpr int kTb2Radius = 2;

template <int R, typename T, int THT_ = 0>
struct TLay {
    // taller tiles for larger radii: (SEGT + 2R) / SEGT rows are touched per
    // output row of a column segment
    static constexpr int THT = THT_ ? THT_ : (R <= 2 ? 64 : 128);
    static constexpr int SEGT = THT / NSB;
    static constexpr int LH = THT + 2 * R;
    static constexpr int LWU = TW + 2 * R;
    // TMA needs 16-byte aligned box rows AND a 16-byte aligned innermost start
    // coordinate, so the box starts RA >= R columns left of the tile
    // (RA = R rounded up to 16 bytes) and column x of the tile sits at
    // smem column x + XOFF.
    static constexpr int ALIGN = 16 / static_cast<int>(sizeof(T));
    static constexpr int RA = (R + ALIGN - 1) / ALIGN * ALIGN;
    static constexpr int XOFF = RA - R;
    static constexpr int BW = (TW + RA + R + ALIGN - 1) / ALIGN * ALIGN;  // TMA box width
    static constexpr uint32_t TILE_BYTES = static_cast<uint32_t>(BW) * LH * sizeof(T);
    static constexpr int NRT = 2 * R + 2;
    static constexpr size_t SMEM = TILE_BYTES + 128;  // + alignment slack
};

template <int R, typename T, bool EXACT_DIV, bool BORDER, class Ly = TLay<R, T>, bool SEQ = false,
          bool ISEL = false>
__device__ __forceinline__ void direct_walk(const T* __restrict__ Us, int X0, int Y0, int W,
                                            const Band& band, int b, double* __restrict__ outp,
                                            size_t out_pitch, const double* __restrict__ rtab) {
    const int x = threadIdx.x % TW, s = threadIdx.x / TW;
    const int gx = X0 + x;
    if (BORDER && gx >= W) return;
    ColFactors cf{0.0, 0.0, 0.0};
    if (BORDER) {
        const int ncl = min(gx, R) + 1, ncr = min(W - 1 - gx, R) + 1;
        cf = ColFactors{rtab[ncl], rtab[ncr], rtab[ncl + ncr - 1]};
    }
    const int y0 = s * Ly::SEGT;
    // image (X0 + x + i - R, Y0 + y0 + j - R) = col[j*BW + i]
    const T* __restrict__ col = Us + y0 * Ly::BW + x + Ly::XOFF;
    const int H = band.h_img;
    double* o = outp + static_cast<size_t>(Y0 + y0 - band.y_out0) * out_pitch + gx;
    constexpr int NJ = Ly::SEGT + 2 * R;
    double P1[NJ + 1], P2[NJ + 1], Q[NJ + 1], Uc[NJ];
    P1[0] = P2[0] = Q[0] = 0.0;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        double v[2 * R + 1];
#pragma unroll
        for (int i = 0; i <= 2 * R; ++i) v[i] = to_f64(col[j * Ly::BW + i]);
        double a = v[0], c = v[R];
#pragma unroll
        for (int i = 1; i <= R; ++i) {
            a += v[i];
            c += v[R + i];
        }
        const double e = v[R];
        Uc[j] = e;
        P1[j + 1] = P1[j] + a;
        P2[j + 1] = P2[j] + c;
        Q[j + 1] = Q[j] + ((a + c) - e);
        const int y = j - 2 * R;
        if (y >= 0) {
            const int gy = Y0 + y0 + y;
            if (BORDER && gy >= band.y_end) break;
            const double S[8] = {P1[y + 2 * R + 1] - P1[y + R], P2[y + 2 * R + 1] - P2[y + R],
                                 P2[y + R + 1] - P2[y],         P1[y + R + 1] - P1[y],
                                 P1[y + 2 * R + 1] - P1[y],     P2[y + 2 * R + 1] - P2[y],
                                 Q[y + 2 * R + 1] - Q[y + R],   Q[y + R + 1] - Q[y]};
            select_store<R, EXACT_DIV, BORDER, false, SEQ, ISEL>(S, Uc[y + R], gx, gy, W, H, b,
                                                                 o, nullptr, nullptr, cf, rtab);
            o += out_pitch;
        }
    }
}

// Tile-kernel variants: VAR 0 = depth-3 tournament, 64-row tiles (128 above
// r = 2), register bound for 3 / 2 CTAs per SM; VAR 1 = sequential scan and
// 64-row tiles, register bound for 4 CTAs per SM (r <= 2) / 3 (r 3..4).
template <int R, typename T, int VAR>
struct TVar {
    static constexpr bool SEQ = VAR == 1;
    static constexpr bool ISEL = VAR == 2;
    using Ly = TLay<R, T, VAR == 1 ? 64 : 0>;
    static constexpr int MINB = VAR == 1 ? (R <= 2 ? 4 : 3) : (R <= 2 ? 3 : (R <= 4 ? 2 : 1));
};

template <int R, typename T, bool EXACT_DIV, int VAR = 0>
__global__ void __launch_bounds__(NT, EXACT_DIV ? (R <= 2 ? 2 : 1) : TVar<R, T, VAR>::MINB)
    fast_tma_step(const __grid_constant__ CUtensorMap tmap, double* __restrict__ out,
                  size_t out_pitch, size_t out_plane, int W, Band band) {
    using Ly = typename TVar<R, T, VAR>::Ly;
    constexpr bool SEQ = TVar<R, T, VAR>::SEQ;
    constexpr bool ISEL = TVar<R, T, VAR>::ISEL;
    extern __shared__ unsigned char smem_raw[];
    __shared__ uint64_t bar;
    __shared__ double rtab[Ly::NRT];
    const uint32_t base = tma::smem_u32(smem_raw);
    T* Us = reinterpret_cast<T*>(smem_raw + ((128u - (base & 127u)) & 127u));
    const int X0 = blockIdx.x * TW, Y0 = band.y_out0 + tile_row(band) * Ly::THT, b = blockIdx.z;
    if (threadIdx.x == 0) tma::mbar_init(&bar, 1);
    if (threadIdx.x < Ly::NRT) rtab[threadIdx.x] = threadIdx.x ? 1.0 / threadIdx.x : 0.0;
    __syncthreads();
    if (threadIdx.x == 0) {
        tma::mbar_arrive_expect_tx(&bar, Ly::TILE_BYTES);
        tma::load_3d(Us, &tmap, X0 - Ly::RA, Y0 - R - band.y_in0, b, &bar);
    }
    tma::mbar_wait(&bar, 0);
    double* outp = out + static_cast<size_t>(b) * out_plane;
    if (X0 >= R && X0 + TW + R <= W && Y0 >= R && Y0 + Ly::THT + R <= band.h_img &&
        Y0 + Ly::THT <= band.y_end)
        direct_walk<R, T, EXACT_DIV, false, Ly, SEQ, ISEL>(Us, X0, Y0, W, band, b, outp, out_pitch,
                                                           rtab);
    else
        direct_walk<R, T, EXACT_DIV, true, Ly, SEQ, ISEL>(Us, X0, Y0, W, band, b, outp, out_pitch,
                                                          rtab);
    if (band.push_rows) {  // row-band mode with the fused halo push
        const int gx = X0 + threadIdx.x % TW, ya = Y0 + (threadIdx.x / TW) * Ly::SEGT;
        if (gx < W) push_tail(band, outp, out_pitch, gx, ya, min(ya + Ly::SEGT, band.y_end));
    }
}

template <typename T>
constexpr CUtensorMapDataType tma_dtype() {
    return sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64
                          : (sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                            : CU_TENSOR_MAP_DATA_TYPE_UINT8);
}

// Returns cudaErrorNotSupported (no launch) when the layout is not TMA-able.
template <int R, typename T, bool EXACT_DIV, int VAR = 0>
cudaError_t launch_tma(const PlaneView& in, const Geometry& g, double* out, size_t op,
                       size_t opl, cudaStream_t s) {
    using Ly = typename TVar<R, T, VAR>::Ly;
    CUtensorMap map;
    const uint64_t plane_bytes = (g.batch > 1 ? in.plane : in.pitch * g.in_h()) * sizeof(T);
    if (!tma::encode_3d(&map, tma_dtype<T>(), in.base, g.width, g.in_h(), g.batch,
                        in.pitch * sizeof(T), plane_bytes, Ly::BW, Ly::LH))
        return cudaErrorNotSupported;
    static std::atomic<unsigned long long> done{0};
    if (cudaError_t e = ensure_smem(fast_tma_step<R, T, EXACT_DIV, VAR>, Ly::SMEM, done)) return e;
    dim3 grid((g.width + TW - 1) / TW, (g.height + Ly::THT - 1) / Ly::THT, g.batch);
    note_kernel(VAR == 1 ? "fast_tma_step (seq)" : (VAR == 2 ? "fast_tma_step (intsel)" : "fast_tma_step"));
    fast_tma_step<R, T, EXACT_DIV, VAR><<<grid, NT, Ly::SMEM, s>>>(map, out, op, opl, g.width,
                                                                   band_of(g));
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// TMA tile with a shared arm pass (r = 3, 4): the walk of fast_tma_step loads
// 2R+1 samples per row per thread (at r = 4 the shared-memory pipe ran at 70%
// of its peak on the 32768^2 plane); here the tile's horizontal left arms
// H(k) = U(k-R) + ... + U(k) are formed once per staged row by sliding sums
// (lanes = rows x segments) into a second shared array, and each column
// thread's walk reads F1 = H(x), F2 = H(x+R) and U(x): 3 loads per row.
constexpr int kArmsMinRadius = 3, kArmsMaxRadius = 4;

// Phase-A mapping idx -> (row idx % LH? ...) chosen at compile time: lane idx
// covers row (idx / NSA) and segment (idx % NSA) of SA columns; 8-byte
// accesses at row*pitch + seg*SA + k must hit distinct bank pairs per
// half-warp.
constexpr bool arms_rows_conflict_free(int nlane, int nseg, int seg, int pitch) {
    for (int h0 = 0; h0 < nlane; h0 += 16) {
        unsigned mask = 0;
        for (int i = 0; i < 16 && h0 + i < nlane; ++i) {
            const int idx = h0 + i, row = idx / nseg, sg = idx % nseg;
            const int bank = (row * pitch + sg * seg) % 16;
            if ((mask >> bank) & 1u) return false;
            mask |= 1u << bank;
        }
    }
    return true;
}
constexpr int arms_rows_pitch(int nlane, int nseg, int seg, int minp, int step) {
    for (int p = minp; p < minp + 32 * step; p += step)
        if (arms_rows_conflict_free(nlane, nseg, seg, p)) return p;
    return minp;
}

template <int R, typename T>
struct ALay {
    static constexpr int THT = 64;
    static constexpr int SEGT = THT / NSB;
    static constexpr int LH = THT + 2 * R;
    static constexpr int ALIGN = 16 / static_cast<int>(sizeof(T));
    static constexpr int RA = (R + ALIGN - 1) / ALIGN * ALIGN;
    static constexpr int XOFF = RA - R;
    static constexpr int NHC = TW + R;                     // arm columns H(k), k < NHC
    static constexpr int NSA = NT / LH;                    // segments per row (phase A)
    static constexpr int SA = ((NHC + NSA - 1) / NSA) | 1; // columns per segment (odd)
    // staged row pitch: TMA box width (multiple of 16 bytes) >= XOFF + NSA*SA + R,
    // conflict-free for the phase-A lanes when fp64
    static constexpr int BW0 = (XOFF + NSA * SA + R + ALIGN - 1) / ALIGN * ALIGN;
    static constexpr int BW =
        sizeof(T) == 8 ? arms_rows_pitch(LH * NSA, NSA, SA, BW0, ALIGN) : BW0;
    static constexpr int PH = arms_rows_pitch(LH * NSA, NSA, SA, NSA * SA, 1);
    static constexpr uint32_t TILE_BYTES = static_cast<uint32_t>(BW) * LH * sizeof(T);
    static constexpr size_t UBUF = (TILE_BYTES + 15) / 16 * 16;
    static constexpr size_t SMEM = 128 + UBUF + sizeof(double) * static_cast<size_t>(LH) * PH;
    static constexpr int NRT = 2 * R + 2;
    static_assert(BW <= 256, "TMA box");
};

template <int R, typename T, bool EXACT_DIV, bool BORDER>
__device__ __forceinline__ void arms_walk(const T* __restrict__ Us, const double* __restrict__ Hs,
                                          int X0, int Y0, int W, const Band& band,
                                          double* __restrict__ outp, size_t out_pitch,
                                          const double* __restrict__ rtab) {
    using Ly = ALay<R, T>;
    const int x = threadIdx.x % TW, s = threadIdx.x / TW;
    const int gx = X0 + x;
    if (BORDER && gx >= W) return;
    ColFactors cf{0.0, 0.0, 0.0};
    if (BORDER) {
        const int ncl = min(gx, R) + 1, ncr = min(W - 1 - gx, R) + 1;
        cf = ColFactors{rtab[ncl], rtab[ncr], rtab[ncl + ncr - 1]};
    }
    const int y0 = s * Ly::SEGT;
    const double* __restrict__ h = Hs + y0 * Ly::PH + x;
    const T* __restrict__ uc = Us + y0 * Ly::BW + x + Ly::RA;
    const int H = band.h_img;
    double* o = outp + static_cast<size_t>(Y0 + y0 - band.y_out0) * out_pitch + gx;
    constexpr int NJ = Ly::SEGT + 2 * R;
    double P1[NJ + 1], P2[NJ + 1], Q[NJ + 1], Uc[NJ];
    P1[0] = P2[0] = Q[0] = 0.0;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        const double a = h[j * Ly::PH], c = h[j * Ly::PH + R];
        const double e = to_f64(uc[j * Ly::BW]);
        Uc[j] = e;
        P1[j + 1] = P1[j] + a;
        P2[j + 1] = P2[j] + c;
        Q[j + 1] = Q[j] + ((a + c) - e);
        const int y = j - 2 * R;
        if (y >= 0) {
            const int gy = Y0 + y0 + y;
            if (BORDER && gy >= band.y_end) break;
            const double S[8] = {P1[y + 2 * R + 1] - P1[y + R], P2[y + 2 * R + 1] - P2[y + R],
                                 P2[y + R + 1] - P2[y],         P1[y + R + 1] - P1[y],
                                 P1[y + 2 * R + 1] - P1[y],     P2[y + 2 * R + 1] - P2[y],
                                 Q[y + 2 * R + 1] - Q[y + R],   Q[y + R + 1] - Q[y]};
            select_store<R, EXACT_DIV, BORDER, false>(S, Uc[y + R], gx, gy, W, H, 0, o, nullptr,
                                                      nullptr, cf, rtab);
            o += out_pitch;
        }
    }
}

template <int R, typename T, bool EXACT_DIV>
__global__ void __launch_bounds__(NT, 2)
    fast_tma_arms(const __grid_constant__ CUtensorMap tmap, double* __restrict__ out,
                  size_t out_pitch, size_t out_plane, int W, Band band) {
    using Ly = ALay<R, T>;
    extern __shared__ unsigned char smem_raw[];
    __shared__ uint64_t bar;
    __shared__ double rtab[Ly::NRT];
    const uint32_t base = tma::smem_u32(smem_raw);
    unsigned char* al = smem_raw + ((128u - (base & 127u)) & 127u);
    T* Us = reinterpret_cast<T*>(al);
    double* Hs = reinterpret_cast<double*>(al + Ly::UBUF);
    const int X0 = blockIdx.x * TW, Y0 = band.y_out0 + tile_row(band) * Ly::THT, b = blockIdx.z;
    if (threadIdx.x == 0) tma::mbar_init(&bar, 1);
    if (threadIdx.x < Ly::NRT) rtab[threadIdx.x] = threadIdx.x ? 1.0 / threadIdx.x : 0.0;
    __syncthreads();
    if (threadIdx.x == 0) {
        tma::mbar_arrive_expect_tx(&bar, Ly::TILE_BYTES);
        tma::load_3d(Us, &tmap, X0 - Ly::RA, Y0 - R - band.y_in0, b, &bar);
    }
    tma::mbar_wait(&bar, 0);
    // ---- arms: lane (row, segment) slides a (R+1)-sample sum along its segment
    if (threadIdx.x < Ly::LH * Ly::NSA) {
        const int row = threadIdx.x / Ly::NSA, sg = threadIdx.x % Ly::NSA;
        const T* __restrict__ u = Us + row * Ly::BW + Ly::XOFF + sg * Ly::SA;
        double* __restrict__ hp = Hs + row * Ly::PH + sg * Ly::SA;
        double v[Ly::SA + R];
#pragma unroll
        for (int i = 0; i < Ly::SA + R; ++i) v[i] = to_f64(u[i]);
        double acc = v[0];
#pragma unroll
        for (int i = 1; i <= R; ++i) acc += v[i];
        hp[0] = acc;
#pragma unroll
        for (int m = 1; m < Ly::SA; ++m) {
            acc += v[m + R] - v[m - 1];
            hp[m] = acc;
        }
    }
    __syncthreads();
    double* outp = out + static_cast<size_t>(b) * out_plane;
    if (X0 >= R && X0 + TW + R <= W && Y0 >= R && Y0 + Ly::THT + R <= band.h_img &&
        Y0 + Ly::THT <= band.y_end)
        arms_walk<R, T, EXACT_DIV, false>(Us, Hs, X0, Y0, W, band, outp, out_pitch, rtab);
    else
        arms_walk<R, T, EXACT_DIV, true>(Us, Hs, X0, Y0, W, band, outp, out_pitch, rtab);
    if (band.push_rows) {  // row-band mode with the fused halo push
        const int gx = X0 + threadIdx.x % TW, ya = Y0 + (threadIdx.x / TW) * Ly::SEGT;
        if (gx < W) push_tail(band, outp, out_pitch, gx, ya, min(ya + Ly::SEGT, band.y_end));
    }
}

template <int R, typename T, bool EXACT_DIV>
cudaError_t launch_arms(const PlaneView& in, const Geometry& g, double* out, size_t op,
                        size_t opl, cudaStream_t s) {
    using Ly = ALay<R, T>;
    CUtensorMap map;
    const uint64_t plane_bytes = (g.batch > 1 ? in.plane : in.pitch * g.in_h()) * sizeof(T);
    if (!tma::encode_3d(&map, tma_dtype<T>(), in.base, g.width, g.in_h(), g.batch,
                        in.pitch * sizeof(T), plane_bytes, Ly::BW, Ly::LH))
        return cudaErrorNotSupported;
    static std::atomic<unsigned long long> done{0};
    if (cudaError_t e = ensure_smem(fast_tma_arms<R, T, EXACT_DIV>, Ly::SMEM, done)) return e;
    dim3 grid((g.width + TW - 1) / TW, (g.height + Ly::THT - 1) / Ly::THT, g.batch);
    note_kernel("fast_tma_arms");
    fast_tma_arms<R, T, EXACT_DIV><<<grid, NT, Ly::SMEM, s>>>(map, out, op, opl, g.width,
                                                              band_of(g));
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Two columns per thread (r <= kTmaRadius): the TMA-staged tile of
// fast_tma_step, but each thread walks the adjacent columns x0, x0 + 1 of its
// segment.  Their windows share 2R of their 2R + 2 samples per row, loaded as
// R + 1 aligned pairs (one 16-byte shared load per pair for fp64): per pixel
// and row (R+1)/2 loads instead of 2R + 1, and the arms of x0 + 1 follow from
// those of x0 with two adds each.  Outputs leave as 16-byte pair stores.
template <int R, typename T>
struct T2Lay {
    static constexpr int TW2 = 64;             // columns per tile (32 lanes x 2)
    static constexpr int NSB2 = 4;             // row segments (warps) per tile
    static constexpr int NT2 = 32 * NSB2;
    static constexpr int THT = R <= 2 ? 64 : 128;
    static constexpr int SEGT = THT / NSB2;
    static constexpr int LH = THT + 2 * R;
    static constexpr int ALIGN = 16 / static_cast<int>(sizeof(T));
    static constexpr int RA = (R + ALIGN - 1) / ALIGN * ALIGN;
    static constexpr int XOFF = RA - R;        // smem column of image column X0 - R
    static constexpr bool ODD = (XOFF & 1) != 0;  // pairs start one sample later
    static constexpr int BW = (TW2 + RA + R + 1 + ALIGN - 1) / ALIGN * ALIGN;
    static constexpr uint32_t TILE_BYTES = static_cast<uint32_t>(BW) * LH * sizeof(T);
    static constexpr int NRT = 2 * R + 2;
    static constexpr size_t SMEM = TILE_BYTES + 128;
    static constexpr int MINB = 2;
};

template <typename T>
struct Pair;
template <>
struct Pair<double> {
    using V = double2;
};
template <>
struct Pair<float> {
    using V = float2;
};
template <>
struct Pair<uint8_t> {
    using V = uchar2;
};

template <int R, typename T, bool EXACT_DIV, bool BORDER, bool VEC_OUT>
__device__ __forceinline__ void pair_walk(const T* __restrict__ Us, int X0, int Y0, int W,
                                          const Band& band, double* __restrict__ outp,
                                          size_t out_pitch, const double* __restrict__ rtab) {
    using Ly = T2Lay<R, T>;
    using PV = typename Pair<T>::V;
    const int lane = threadIdx.x & 31, s = threadIdx.x >> 5;
    const int gx0 = X0 + 2 * lane;  // columns gx0, gx0 + 1
    if (BORDER && gx0 >= W) return;
    const bool has1 = !BORDER || gx0 + 1 < W;
    ColFactors cf0{0.0, 0.0, 0.0}, cf1{0.0, 0.0, 0.0};
    if (BORDER) {
        int ncl = min(gx0, R) + 1, ncr = min(W - 1 - gx0, R) + 1;
        cf0 = ColFactors{rtab[ncl], rtab[ncr], rtab[ncl + ncr - 1]};
        ncl = min(gx0 + 1, R) + 1;
        ncr = max(min(W - 2 - gx0, R), 0) + 1;
        cf1 = ColFactors{rtab[ncl], rtab[ncr], rtab[ncl + ncr - 1]};
    }
    const int y0 = s * Ly::SEGT;
    // image (gx0 - R + i, Y0 + y0 + j - R) = row[j * BW + i], i in [0, 2R + 2)
    const T* __restrict__ row = Us + y0 * Ly::BW + 2 * lane + Ly::XOFF;
    const int H = band.h_img;
    double* o = outp + static_cast<size_t>(Y0 + y0 - band.y_out0) * out_pitch + gx0;
    constexpr int NJ = Ly::SEGT + 2 * R;
    double P1a[NJ + 1], P2a[NJ + 1], Qa[NJ + 1], Ua[NJ];
    double P1b[NJ + 1], P2b[NJ + 1], Qb[NJ + 1], Ub[NJ];
    P1a[0] = P2a[0] = Qa[0] = P1b[0] = P2b[0] = Qb[0] = 0.0;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        double v[2 * R + 2];
        const T* rj = row + j * Ly::BW;
        if constexpr (Ly::ODD) {
            v[0] = to_f64(rj[0]);
#pragma unroll
            for (int i = 0; i < R; ++i) {
                const PV p = *reinterpret_cast<const PV*>(rj + 1 + 2 * i);
                v[1 + 2 * i] = to_f64(p.x);
                v[2 + 2 * i] = to_f64(p.y);
            }
            v[2 * R + 1] = to_f64(rj[2 * R + 1]);
        } else {
#pragma unroll
            for (int i = 0; i <= R; ++i) {
                const PV p = *reinterpret_cast<const PV*>(rj + 2 * i);
                v[2 * i] = to_f64(p.x);
                v[2 * i + 1] = to_f64(p.y);
            }
        }
        // column a = gx0: arms over v[0..R] and v[R..2R]; column b = gx0 + 1
        // slides them by one sample
        double a1 = v[0], a2 = v[R];
#pragma unroll
        for (int i = 1; i <= R; ++i) {
            a1 += v[i];
            a2 += v[R + i];
        }
        const double b1 = a1 + (v[R + 1] - v[0]);
        const double b2 = a2 + (v[2 * R + 1] - v[R]);
        const double ua = v[R], ub = v[R + 1];
        Ua[j] = ua;
        Ub[j] = ub;
        P1a[j + 1] = P1a[j] + a1;
        P2a[j + 1] = P2a[j] + a2;
        Qa[j + 1] = Qa[j] + ((a1 + a2) - ua);
        P1b[j + 1] = P1b[j] + b1;
        P2b[j + 1] = P2b[j] + b2;
        Qb[j + 1] = Qb[j] + ((b1 + b2) - ub);
        const int y = j - 2 * R;
        if (y >= 0) {
            const int gy = Y0 + y0 + y;
            if (BORDER && gy >= band.y_end) break;
            const double Sa[8] = {P1a[y + 2 * R + 1] - P1a[y + R], P2a[y + 2 * R + 1] - P2a[y + R],
                                  P2a[y + R + 1] - P2a[y],         P1a[y + R + 1] - P1a[y],
                                  P1a[y + 2 * R + 1] - P1a[y],     P2a[y + 2 * R + 1] - P2a[y],
                                  Qa[y + 2 * R + 1] - Qa[y + R],   Qa[y + R + 1] - Qa[y]};
            const double Sb[8] = {P1b[y + 2 * R + 1] - P1b[y + R], P2b[y + 2 * R + 1] - P2b[y + R],
                                  P2b[y + R + 1] - P2b[y],         P1b[y + R + 1] - P1b[y],
                                  P1b[y + 2 * R + 1] - P1b[y],     P2b[y + 2 * R + 1] - P2b[y],
                                  Qb[y + 2 * R + 1] - Qb[y + R],   Qb[y + R + 1] - Qb[y]};
            double va, vb = 0.0, tmp;
            va = select_store<R, EXACT_DIV, BORDER, false>(Sa, Ua[y + R], gx0, gy, W, H, 0, &tmp,
                                                           nullptr, nullptr, cf0, rtab);
            if (!BORDER || has1)
                vb = select_store<R, EXACT_DIV, BORDER, false>(Sb, Ub[y + R], gx0 + 1, gy, W, H, 0,
                                                               &tmp, nullptr, nullptr, cf1, rtab);
            if constexpr (VEC_OUT && !BORDER) {
                *reinterpret_cast<double2*>(o) = make_double2(va, vb);
            } else {
                o[0] = va;
                if (!BORDER || has1) o[1] = vb;
            }
            o += out_pitch;
        }
    }
}

template <int R, typename T, bool EXACT_DIV, bool VEC_OUT>
__global__ void __launch_bounds__(T2Lay<R, T>::NT2, T2Lay<R, T>::MINB)
    fast_tma_pair(const __grid_constant__ CUtensorMap tmap, double* __restrict__ out,
                  size_t out_pitch, size_t out_plane, int W, Band band) {
    using Ly = T2Lay<R, T>;
    extern __shared__ unsigned char smem_raw[];
    __shared__ uint64_t bar;
    __shared__ double rtab[Ly::NRT];
    const uint32_t base = tma::smem_u32(smem_raw);
    T* Us = reinterpret_cast<T*>(smem_raw + ((128u - (base & 127u)) & 127u));
    const int X0 = blockIdx.x * Ly::TW2, Y0 = band.y_out0 + blockIdx.y * Ly::THT, b = blockIdx.z;
    if (threadIdx.x == 0) tma::mbar_init(&bar, 1);
    if (threadIdx.x < Ly::NRT) rtab[threadIdx.x] = threadIdx.x ? 1.0 / threadIdx.x : 0.0;
    __syncthreads();
    if (threadIdx.x == 0) {
        tma::mbar_arrive_expect_tx(&bar, Ly::TILE_BYTES);
        tma::load_3d(Us, &tmap, X0 - Ly::RA, Y0 - R - band.y_in0, b, &bar);
    }
    tma::mbar_wait(&bar, 0);
    double* outp = out + static_cast<size_t>(b) * out_plane;
    if (X0 >= R && X0 + Ly::TW2 + R <= W && Y0 >= R && Y0 + Ly::THT + R <= band.h_img &&
        Y0 + Ly::THT <= band.y_end)
        pair_walk<R, T, EXACT_DIV, false, VEC_OUT>(Us, X0, Y0, W, band, outp, out_pitch, rtab);
    else
        pair_walk<R, T, EXACT_DIV, true, VEC_OUT>(Us, X0, Y0, W, band, outp, out_pitch, rtab);
    if (band.push_rows) {  // row-band mode with the fused halo push
        const int lane = threadIdx.x & 31, ya = Y0 + (threadIdx.x >> 5) * Ly::SEGT;
        for (int c = 0; c < 2; ++c) {
            const int gx = X0 + 2 * lane + c;
            if (gx < W) push_tail(band, outp, out_pitch, gx, ya, min(ya + Ly::SEGT, band.y_end));
        }
    }
}

template <int R, typename T, bool EXACT_DIV>
cudaError_t launch_pair(const PlaneView& in, const Geometry& g, double* out, size_t op,
                        size_t opl, cudaStream_t s) {
    using Ly = T2Lay<R, T>;
    CUtensorMap map;
    const uint64_t plane_bytes = (g.batch > 1 ? in.plane : in.pitch * g.in_h()) * sizeof(T);
    if (!tma::encode_3d(&map, tma_dtype<T>(), in.base, g.width, g.in_h(), g.batch,
                        in.pitch * sizeof(T), plane_bytes, Ly::BW, Ly::LH))
        return cudaErrorNotSupported;
    const bool vec = (reinterpret_cast<uintptr_t>(out) & 15u) == 0 && op % 2 == 0 &&
                     (g.batch == 1 || opl % 2 == 0);
    dim3 grid((g.width + Ly::TW2 - 1) / Ly::TW2, (g.height + Ly::THT - 1) / Ly::THT, g.batch);
    note_kernel("fast_tma_pair");
    if (vec) {
        static std::atomic<unsigned long long> done{0};
        if (cudaError_t e = ensure_smem(fast_tma_pair<R, T, EXACT_DIV, true>, Ly::SMEM, done))
            return e;
        fast_tma_pair<R, T, EXACT_DIV, true><<<grid, Ly::NT2, Ly::SMEM, s>>>(
            map, out, op, opl, g.width, band_of(g));
    } else {
        static std::atomic<unsigned long long> done{0};
        if (cudaError_t e = ensure_smem(fast_tma_pair<R, T, EXACT_DIV, false>, Ly::SMEM, done))
            return e;
        fast_tma_pair<R, T, EXACT_DIV, false><<<grid, Ly::NT2, Ly::SMEM, s>>>(
            map, out, op, opl, g.width, band_of(g));
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Persistent tile kernel (r <= kTmaRadius): the same per-tile computation as
// fast_tma_step (bit-identical outputs), but a grid of #SMs x occupancy CTAs
// walks the tiles round robin with two shared-memory tile buffers, so the TMA
// load of a CTA's next tile is in flight while it computes the current one
// (fast_tma_step waited for every tile's load: ~25% of its stall samples).
template <int R, typename T>
struct PLay {
    using Base = TLay<R, T>;
    static constexpr int THT = 64;
    static constexpr int SEGT = THT / NSB;
    static constexpr int LH = THT + 2 * R;
    static constexpr int RA = Base::RA, XOFF = Base::XOFF, BW = Base::BW;
    static constexpr uint32_t TILE_BYTES = static_cast<uint32_t>(BW) * LH * sizeof(T);
    static constexpr size_t BUF = (TILE_BYTES + 127) / 128 * 128;
    static constexpr int NRT = 2 * R + 2;
    static constexpr size_t SMEM = 128 + 2 * BUF;
    static constexpr int MINB = R <= 2 ? 3 : 2;
};

template <int R, typename T, bool EXACT_DIV, bool BORDER>
__device__ __forceinline__ void tile_walk(const T* __restrict__ Us, int X0, int Y0, int W,
                                          const Band& band, double* __restrict__ outp,
                                          size_t out_pitch, const double* __restrict__ rtab) {
    using Ly = PLay<R, T>;
    const int x = threadIdx.x % TW, s = threadIdx.x / TW;
    const int gx = X0 + x;
    if (BORDER && gx >= W) return;
    ColFactors cf{0.0, 0.0, 0.0};
    if (BORDER) {
        const int ncl = min(gx, R) + 1, ncr = min(W - 1 - gx, R) + 1;
        cf = ColFactors{rtab[ncl], rtab[ncr], rtab[ncl + ncr - 1]};
    }
    const int y0 = s * Ly::SEGT;
    const T* __restrict__ col = Us + y0 * Ly::BW + x + Ly::XOFF;
    const int H = band.h_img;
    double* o = outp + static_cast<size_t>(Y0 + y0 - band.y_out0) * out_pitch + gx;
    constexpr int NJ = Ly::SEGT + 2 * R;
    double P1[NJ + 1], P2[NJ + 1], Q[NJ + 1], Uc[NJ];
    P1[0] = P2[0] = Q[0] = 0.0;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        double v[2 * R + 1];
#pragma unroll
        for (int i = 0; i <= 2 * R; ++i) v[i] = to_f64(col[j * Ly::BW + i]);
        double a = v[0], c = v[R];
#pragma unroll
        for (int i = 1; i <= R; ++i) {
            a += v[i];
            c += v[R + i];
        }
        const double e = v[R];
        Uc[j] = e;
        P1[j + 1] = P1[j] + a;
        P2[j + 1] = P2[j] + c;
        Q[j + 1] = Q[j] + ((a + c) - e);
        const int y = j - 2 * R;
        if (y >= 0) {
            const int gy = Y0 + y0 + y;
            if (BORDER && gy >= band.y_end) break;
            const double S[8] = {P1[y + 2 * R + 1] - P1[y + R], P2[y + 2 * R + 1] - P2[y + R],
                                 P2[y + R + 1] - P2[y],         P1[y + R + 1] - P1[y],
                                 P1[y + 2 * R + 1] - P1[y],     P2[y + 2 * R + 1] - P2[y],
                                 Q[y + 2 * R + 1] - Q[y + R],   Q[y + R + 1] - Q[y]};
            select_store<R, EXACT_DIV, BORDER, false>(S, Uc[y + R], gx, gy, W, H, 0, o, nullptr,
                                                      nullptr, cf, rtab);
            o += out_pitch;
        }
    }
}

template <int R, typename T, bool EXACT_DIV>
__global__ void __launch_bounds__(NT, PLay<R, T>::MINB)
    fast_tile(const __grid_constant__ CUtensorMap tmap, double* __restrict__ out,
              size_t out_pitch, size_t out_plane, int W, Band band, int ntx, int nty,
              int ntiles) {
    using Ly = PLay<R, T>;
    extern __shared__ unsigned char smem_raw[];
    __shared__ uint64_t bar[2];
    __shared__ double rtab[Ly::NRT];
    const uint32_t base = tma::smem_u32(smem_raw);
    unsigned char* sm = smem_raw + ((128u - (base & 127u)) & 127u);
    T* bufs[2] = {reinterpret_cast<T*>(sm), reinterpret_cast<T*>(sm + Ly::BUF)};
    const int tid = threadIdx.x;
    auto tile_of = [&](int t, int& X0, int& Y0, int& b) {
        const int tx = t % ntx, rest = t / ntx;
        X0 = tx * TW;
        Y0 = band.y_out0 + (rest % nty) * Ly::THT;
        b = rest / nty;
    };
    auto issue = [&](int t, int sl) {
        int X0, Y0, b;
        tile_of(t, X0, Y0, b);
        tma::mbar_arrive_expect_tx(&bar[sl], Ly::TILE_BYTES);
        tma::load_3d(bufs[sl], &tmap, X0 - Ly::RA, Y0 - R - band.y_in0, b, &bar[sl]);
    };
    if (tid == 0) {
        tma::mbar_init(&bar[0], 1);
        tma::mbar_init(&bar[1], 1);
    }
    if (tid < Ly::NRT) rtab[tid] = tid ? 1.0 / tid : 0.0;
    __syncthreads();
    if (tid == 0 && static_cast<int>(blockIdx.x) < ntiles) issue(blockIdx.x, 0);
    int i = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
        const int sl = i & 1;
        tma::mbar_wait(&bar[sl], (i >> 1) & 1);
        // every thread is done with the previous tile: its buffer takes the next
        __syncthreads();
        if (tid == 0 && t + static_cast<int>(gridDim.x) < ntiles) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            issue(t + gridDim.x, sl ^ 1);
        }
        int X0, Y0, b;
        tile_of(t, X0, Y0, b);
        double* outp = out + static_cast<size_t>(b) * out_plane;
        if (X0 >= R && X0 + TW + R <= W && Y0 >= R && Y0 + Ly::THT + R <= band.h_img &&
            Y0 + Ly::THT <= band.y_end)
            tile_walk<R, T, EXACT_DIV, false>(bufs[sl], X0, Y0, W, band, outp, out_pitch, rtab);
        else
            tile_walk<R, T, EXACT_DIV, true>(bufs[sl], X0, Y0, W, band, outp, out_pitch, rtab);
        if (band.push_rows) {  // row-band mode with the fused halo push
            const int gx = X0 + tid % TW, ya = Y0 + (tid / TW) * Ly::SEGT;
            if (gx < W) push_tail(band, outp, out_pitch, gx, ya, min(ya + Ly::SEGT, band.y_end));
        }
    }
}

template <int R, typename T, bool EXACT_DIV>
cudaError_t launch_tile(const PlaneView& in, const Geometry& g, double* out, size_t op,
                        size_t opl, cudaStream_t s) {
    using Ly = PLay<R, T>;
    CUtensorMap map;
    const uint64_t plane_bytes = (g.batch > 1 ? in.plane : in.pitch * g.in_h()) * sizeof(T);
    if (!tma::encode_3d(&map, tma_dtype<T>(), in.base, g.width, g.in_h(), g.batch,
                        in.pitch * sizeof(T), plane_bytes, Ly::BW, Ly::LH))
        return cudaErrorNotSupported;
    auto* fn = fast_tile<R, T, EXACT_DIV>;
    static std::atomic<unsigned long long> done{0};
    if (cudaError_t e = ensure_smem(fn, Ly::SMEM, done)) return e;
    int dev = 0, nsm = 0, per_sm = 0;
    if (cudaError_t e = cudaGetDevice(&dev)) return e;
    if (cudaError_t e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev)) return e;
    if (cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, NT, Ly::SMEM))
        return e;
    if (per_sm < 1) return cudaErrorNotSupported;
    const int ntx = (g.width + TW - 1) / TW, nty = (g.height + Ly::THT - 1) / Ly::THT;
    const long long ntiles = static_cast<long long>(ntx) * nty * g.batch;
    if (ntiles > (1ll << 31) - 1) return cudaErrorNotSupported;
    const long long cap = static_cast<long long>(nsm) * per_sm;
    const int grid = static_cast<int>(ntiles < cap ? ntiles : cap);
    note_kernel("fast_tile");
    fn<<<grid, NT, Ly::SMEM, s>>>(map, out, op, opl, g.width, band_of(g), ntx, nty,
                                  static_cast<int>(ntiles));
    return cudaGetLastError();
}

}  // namespace fastk
}  // namespace osbf_gpu

#include "osbf_fast_stream.cuh"
#include "osbf_fast_walk.cuh"
#include "osbf_strip.cuh"

namespace osbf_gpu {
namespace fastk {

// Kernel family for the fast pass.  OSBF_GPU_FAST (read once per process)
// forces one for A/B measurements: "strip", "tile" (persistent TMA tiles),
// "tma" (one tile per CTA), "stream" or "sep"; unset = the per-radius
// default below.
inline const char* fast_forced() {
    const char* o = fast_kernel_override();
    if (o) return o;
    static const char* v = [] {
        const char* e = getenv("OSBF_GPU_FAST");
        return (e && e[0]) ? e : "";
    }();
    return v;
}
inline bool fast_allowed(const char* name, bool dflt) {
    const char* f = fast_forced();
    if (!f[0]) return dflt;
    return strcmp(f, name) == 0;
}

template <int R, bool DIAG>
cudaError_t launch_dtype(const PlaneView& in, const Geometry& g, double* out, size_t op,
                         size_t opl, double* means, uint8_t* sel, cudaStream_t s) {
    if constexpr (!DIAG) {
        if (fast_allowed("strip", false)) {
            const cudaError_t e = strip_launch_radius<R>(in, g, out, op, opl, s);
            if (e != cudaErrorNotSupported) return e;
        }
    }
    if constexpr (R >= kArmsMinRadius && R <= kArmsMaxRadius && !DIAG) {
        if (fast_allowed("arms", false)) {
            cudaError_t e = cudaErrorNotSupported;
            switch (in.dtype) {
                case OSBF_U8: e = launch_arms<R, uint8_t, true>(in, g, out, op, opl, s); break;
                case OSBF_F32: e = launch_arms<R, float, false>(in, g, out, op, opl, s); break;
                default: e = launch_arms<R, double, false>(in, g, out, op, opl, s); break;
            }
            if (e != cudaErrorNotSupported) return e;
        }
    }
    if constexpr (R <= kTmaRadius && !DIAG) {
        if (fast_allowed("pair", false)) {
            cudaError_t e = cudaErrorNotSupported;
            switch (in.dtype) {
                case OSBF_U8: e = launch_pair<R, uint8_t, true>(in, g, out, op, opl, s); break;
                case OSBF_F32: e = launch_pair<R, float, false>(in, g, out, op, opl, s); break;
                default: e = launch_pair<R, double, false>(in, g, out, op, opl, s); break;
            }
            if (e != cudaErrorNotSupported) return e;
        }
    }
    if constexpr (R <= kTmaRadius && !DIAG) {
        if (fast_allowed("tmaint", false)) {
            cudaError_t e = cudaErrorNotSupported;
            switch (in.dtype) {
                case OSBF_U8: e = launch_tma<R, uint8_t, true>(in, g, out, op, opl, s); break;
                case OSBF_F32: e = launch_tma<R, float, false, 2>(in, g, out, op, opl, s); break;
                default: e = launch_tma<R, double, false, 2>(in, g, out, op, opl, s); break;
            }
            if (e != cudaErrorNotSupported) return e;
        }
    }
    if constexpr (R <= kTmaRadius && !DIAG) {
        if (fast_allowed("tmaseq", false)) {
            cudaError_t e = cudaErrorNotSupported;
            switch (in.dtype) {
                case OSBF_U8: e = launch_tma<R, uint8_t, true>(in, g, out, op, opl, s); break;
                case OSBF_F32: e = launch_tma<R, float, false, 1>(in, g, out, op, opl, s); break;
                default: e = launch_tma<R, double, false, 1>(in, g, out, op, opl, s); break;
            }
            if (e != cudaErrorNotSupported) return e;
        }
    }
    if constexpr (R <= kTmaRadius && !DIAG) {
        if (fast_allowed("tile", false)) {
            cudaError_t e = cudaErrorNotSupported;
            switch (in.dtype) {
                case OSBF_U8: e = launch_tile<R, uint8_t, true>(in, g, out, op, opl, s); break;
                case OSBF_F32: e = launch_tile<R, float, false>(in, g, out, op, opl, s); break;
                default: e = launch_tile<R, double, false>(in, g, out, op, opl, s); break;
            }
            if (e != cudaErrorNotSupported) return e;
        }
    }
    if constexpr (R <= kWalkMaxRadius && !DIAG) {
        if (fast_allowed("walk", R >= 3 && walk_fills(g))) {
            cudaError_t e = cudaErrorNotSupported;
            switch (in.dtype) {
                case OSBF_U8: e = launch_walk<R, uint8_t, true>(in, g, out, op, opl, s); break;
                case OSBF_F32: e = launch_walk<R, float, false>(in, g, out, op, opl, s); break;
                default: e = launch_walk<R, double, false>(in, g, out, op, opl, s); break;
            }
            if (e != cudaErrorNotSupported) return e;
        }
    }
    if constexpr (R >= kStreamMinRadius && R <= kStreamMaxRadius && !DIAG) {
        // superseded by the walk (kept as a selectable family for A/B runs)
        if (stream_enabled() && fast_allowed("stream", false)) {
            cudaError_t e = cudaErrorNotSupported;
            switch (in.dtype) {
                case OSBF_U8: e = launch_stream<R, uint8_t, true>(in, g, out, op, opl, s); break;
                case OSBF_F32: e = launch_stream<R, float, false>(in, g, out, op, opl, s); break;
                default: e = launch_stream<R, double, false>(in, g, out, op, opl, s); break;
            }
            if (e != cudaErrorNotSupported) return e;
        }
    }
    if constexpr (R <= kTmaRadius && !DIAG) {
        if (fast_allowed("tma", true)) {
            cudaError_t e = cudaErrorNotSupported;
            switch (in.dtype) {
                case OSBF_U8: e = launch_tma<R, uint8_t, true>(in, g, out, op, opl, s); break;
                case OSBF_F32: e = launch_tma<R, float, false>(in, g, out, op, opl, s); break;
                default: e = launch_tma<R, double, false>(in, g, out, op, opl, s); break;
            }
            if (e != cudaErrorNotSupported) return e;
        }
    }
    switch (in.dtype) {
        case OSBF_U8:
            return launch_r<R, uint8_t, true, DIAG>(in, g, out, op, opl, means, sel, s);
        case OSBF_F32:
            return launch_r<R, float, false, DIAG>(in, g, out, op, opl, means, sel, s);
        default:
            return launch_r<R, double, false, DIAG>(in, g, out, op, opl, means, sel, s);
    }
}

}  // namespace fastk

// One radius: all dtypes and the diagnostic variant (explicitly instantiated
// in osbf_fast_rNN.cu so the radii compile in parallel).
template <int R>
cudaError_t fast_launch_radius(const PlaneView& in, const Geometry& g, double* out,
                               size_t out_pitch, size_t out_plane, double* means, uint8_t* sel,
                               cudaStream_t s) {
    if (means || sel)
        return fastk::launch_dtype<R, true>(in, g, out, out_pitch, out_plane, means, sel, s);
    return fastk::launch_dtype<R, false>(in, g, out, out_pitch, out_plane, means, sel, s);
}

}  // namespace osbf_gpu

// ===========================================================================
// Temporal blocking: K OSBF passes per HBM round trip (north-star K4),
// K = 2..4, radius <= kTbRadius.
//
// The output tile is staged with a K*R halo; pass p (1..K-1) computes the
// intermediate plane over the output tile plus a (K-p)*R halo into shared
// memory (exactly what a separate pass would write to HBM: clipped counts at
// the GLOBAL image border, zero outside the image so the next pass's sums see
// the same zero fill); pass K computes the output tile from pass K-1.  HBM
// traffic per iteration drops K-fold; the extra work is the shrinking halo
// rings of intermediate pixels: sum_p (T + 2(K-p)R)^2 / (K T^2).
namespace osbf_gpu {
namespace fastk {

constexpr int kTbRadius = 4;
constexpr int kTbMaxPasses = 4;

template <int R, typename T, int K>
struct TBKLay {
    static constexpr int TWK = 64, THK = 64;  // output tile
    static constexpr int HALO = K * R;
    static constexpr int ALIGN = 16 / static_cast<int>(sizeof(T));
    static constexpr int RAK = (HALO + ALIGN - 1) / ALIGN * ALIGN;  // aligned K*R halo
    static constexpr int XOFF = RAK - HALO;
    static constexpr int BW = (TWK + RAK + HALO + ALIGN - 1) / ALIGN * ALIGN;
    static constexpr int LH = THK + 2 * HALO;
    static constexpr uint32_t TILE_BYTES = static_cast<uint32_t>(BW) * LH * sizeof(T);
    static constexpr int NSEG = 4;  // row segments per column in every pass
    static constexpr int IW(int p) { return TWK + 2 * (K - p) * R; }  // pass p's width = height
    // A walk of SEG rows reads SEG + 2R source rows even when its last
    // segment is shorter: the intermediates carry PADR spare rows.
    static constexpr int PADR = NSEG + 2;
    static constexpr size_t IA = sizeof(double) * static_cast<size_t>(IW(1)) * (IW(1) + PADR);
    static constexpr size_t IB =
        K >= 3 ? sizeof(double) * static_cast<size_t>(IW(2)) * (IW(2) + PADR) : 0;
    static constexpr int NTT = (IW(1) * NSEG + 31) / 32 * 32;
    static constexpr int NRT = 2 * R + 2;
    static constexpr size_t SMEM = 128 + ((TILE_BYTES + 15) / 16) * 16 + IA + IB;
    static constexpr int MINB = (SMEM + 1024) * 2 <= 227 * 1024 ? 2 : 1;
};

// One column walk (prefix-sum formulation, see direct_walk): source rows
// src[j*pitch + i], j in [0, nrows + 2R), i in [0, 2R]; outputs for rows
// [0, nrows) at global (gx, gy0 + y).  TO_SMEM: write to dst[y*dst_pitch]
// with 0 for positions outside the image; else to global memory.
template <int R, typename S, bool EXACT_DIV, bool BORDER, bool TO_SMEM, int NSEG>
__device__ __forceinline__ void tb_walk(const S* __restrict__ col, int pitch, int nrows, int gx,
                                        int gy0, int W, const Band& band, double* __restrict__ o,
                                        size_t o_pitch, const double* __restrict__ rtab) {
    const int H = band.h_img;
    const bool col_in = gx >= 0 && gx < W;
    ColFactors cf{0.0, 0.0, 0.0};
    if (BORDER && col_in) {
        const int ncl = min(gx, R) + 1, ncr = min(W - 1 - gx, R) + 1;
        cf = ColFactors{rtab[ncl], rtab[ncr], rtab[ncl + ncr - 1]};
    }
    constexpr int NJ = NSEG + 2 * R;
    double P1[NJ + 1], P2[NJ + 1], Q[NJ + 1], Uc[NJ];
    P1[0] = P2[0] = Q[0] = 0.0;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        double v[2 * R + 1];
#pragma unroll
        for (int i = 0; i <= 2 * R; ++i) v[i] = to_f64(col[j * pitch + i]);
        double a = v[0], c = v[R];
#pragma unroll
        for (int i = 1; i <= R; ++i) {
            a += v[i];
            c += v[R + i];
        }
        const double e = v[R];
        Uc[j] = e;
        P1[j + 1] = P1[j] + a;
        P2[j + 1] = P2[j] + c;
        Q[j + 1] = Q[j] + ((a + c) - e);
        const int y = j - 2 * R;
        if (y >= 0 && y < nrows) {
            const int gy = gy0 + y;
            const double S8[8] = {P1[y + 2 * R + 1] - P1[y + R], P2[y + 2 * R + 1] - P2[y + R],
                                  P2[y + R + 1] - P2[y],         P1[y + R + 1] - P1[y],
                                  P1[y + 2 * R + 1] - P1[y],     P2[y + 2 * R + 1] - P2[y],
                                  Q[y + 2 * R + 1] - Q[y + R],   Q[y + R + 1] - Q[y]};
            if (TO_SMEM) {
                if (!BORDER || (col_in && gy >= 0 && gy < H))
                    select_store<R, EXACT_DIV, BORDER, false>(S8, Uc[y + R], gx, gy, W, H, 0, o,
                                                              nullptr, nullptr, cf, rtab);
                else
                    *o = 0.0;
            } else {
                if (BORDER && gy >= band.y_end) break;
                select_store<R, EXACT_DIV, BORDER, false>(S8, Uc[y + R], gx, gy, W, H, 0, o,
                                                          nullptr, nullptr, cf, rtab);
            }
            o += o_pitch;
        }
    }
}

// Pass P of K (P < K) into shared memory: columns / rows [X0, Y0) - (K-P)R,
// width = height = IW(P); the source is the staged tile (P = 1) or pass P-1.
template <int R, typename T, int K, int P, bool EXACT1>
__device__ __forceinline__ void tbk_smem_pass(const void* src, double* dst, int X0, int Y0,
                                              int W, const Band& band, bool interior,
                                              const double* rtab) {
    using Ly = TBKLay<R, T, K>;
    using S = std::conditional_t<P == 1, T, double>;
    constexpr int IWp = Ly::IW(P);
    constexpr int SPITCH = P == 1 ? Ly::BW : Ly::IW(P - 1);
    constexpr int SOFF = P == 1 ? Ly::XOFF : 0;
    constexpr int SEGp = (IWp + Ly::NSEG - 1) / Ly::NSEG;
    constexpr bool EX = P == 1 && EXACT1;
    const int tid = threadIdx.x;
    if (tid >= IWp * Ly::NSEG) return;
    const int xi = tid % IWp, s = tid / IWp;
    const int yi0 = s * SEGp;
    const int nrows = min(SEGp, IWp - yi0);
    if (nrows <= 0) return;
    const S* col = static_cast<const S*>(src) + yi0 * SPITCH + xi + SOFF;
    double* o = dst + yi0 * IWp + xi;
    const int gx = X0 - (K - P) * R + xi, gy0 = Y0 - (K - P) * R + yi0;
    if (interior)
        tb_walk<R, S, EX, false, true, SEGp>(col, SPITCH, nrows, gx, gy0, W, band, o, IWp, rtab);
    else
        tb_walk<R, S, EX, true, true, SEGp>(col, SPITCH, nrows, gx, gy0, W, band, o, IWp, rtab);
}

template <int R, typename T, int K, bool EXACT1>
__global__ void __launch_bounds__(TBKLay<R, T, K>::NTT, TBKLay<R, T, K>::MINB)
    fast_tma_stepk(const __grid_constant__ CUtensorMap tmap, double* __restrict__ out,
                   size_t out_pitch, size_t out_plane, int W, Band band) {
    using Ly = TBKLay<R, T, K>;
    extern __shared__ unsigned char smem_raw[];
    __shared__ uint64_t bar;
    __shared__ double rtab[Ly::NRT];
    const uint32_t base = tma::smem_u32(smem_raw);
    unsigned char* aligned = smem_raw + ((128u - (base & 127u)) & 127u);
    T* Us = reinterpret_cast<T*>(aligned);
    double* IA = reinterpret_cast<double*>(aligned + ((Ly::TILE_BYTES + 15) / 16) * 16);
    double* IB = IA + Ly::IA / sizeof(double);
    const int X0 = blockIdx.x * Ly::TWK, Y0 = band.y_out0 + tile_row(band) * Ly::THK;
    const int b = blockIdx.z;
    const int tid = threadIdx.x;
    if (tid == 0) tma::mbar_init(&bar, 1);
    if (tid < Ly::NRT) rtab[tid] = tid ? 1.0 / tid : 0.0;
    __syncthreads();
    if (tid == 0) {
        tma::mbar_arrive_expect_tx(&bar, Ly::TILE_BYTES);
        tma::load_3d(Us, &tmap, X0 - Ly::RAK, Y0 - Ly::HALO - band.y_in0, b, &bar);
    }
    tma::mbar_wait(&bar, 0);
    // interior: every intermediate and output position inside the image
    const bool interior = X0 >= Ly::HALO && X0 + Ly::TWK + Ly::HALO <= W && Y0 >= Ly::HALO &&
                          Y0 + Ly::THK + Ly::HALO <= band.h_img && Y0 + Ly::THK <= band.y_end;
    tbk_smem_pass<R, T, K, 1, EXACT1>(Us, IA, X0, Y0, W, band, interior, rtab);
    __syncthreads();
    if constexpr (K >= 3) {
        tbk_smem_pass<R, T, K, 2, EXACT1>(IA, IB, X0, Y0, W, band, interior, rtab);
        __syncthreads();
    }
    if constexpr (K >= 4) {
        tbk_smem_pass<R, T, K, 3, EXACT1>(IB, IA, X0, Y0, W, band, interior, rtab);
        __syncthreads();
    }
    // ---- pass K: the output tile from pass K-1
    const double* last = (K % 2 == 0) ? IA : IB;  // pass K-1 wrote IA when K-1 is odd
    constexpr int IWl = Ly::IW(K - 1);
    constexpr int SEGK = Ly::THK / Ly::NSEG;
    if (tid < Ly::TWK * Ly::NSEG) {
        const int x = tid % Ly::TWK, s = tid / Ly::TWK;
        const int gx = X0 + x;
        if (interior || gx < W) {
            const int y0 = s * SEGK;
            const double* col = last + y0 * IWl + x;
            double* o = out + static_cast<size_t>(b) * out_plane +
                        static_cast<size_t>(Y0 + y0 - band.y_out0) * out_pitch + gx;
            if (interior)
                tb_walk<R, double, false, false, false, SEGK>(col, IWl, SEGK, gx, Y0 + y0, W,
                                                              band, o, out_pitch, rtab);
            else
                tb_walk<R, double, false, true, false, SEGK>(col, IWl, SEGK, gx, Y0 + y0, W,
                                                             band, o, out_pitch, rtab);
        }
    }
    if (band.push_rows) {  // row-band mode with the fused halo push
        __syncthreads();
        if (tid < Ly::TWK * Ly::NSEG) {
            const int gx = X0 + tid % Ly::TWK, ya = Y0 + (tid / Ly::TWK) * SEGK;
            if (gx < W) push_tail(band, out + static_cast<size_t>(b) * out_plane, out_pitch, gx, ya,
                                  min(ya + SEGK, band.y_end));
        }
    }
}

template <int R, typename T, int K, bool EXACT1>
cudaError_t launch_tmak(const PlaneView& in, const Geometry& g, double* out, size_t op,
                        size_t opl, cudaStream_t s) {
    using Ly = TBKLay<R, T, K>;
    if constexpr (Ly::SMEM > 227 * 1024) {
        return cudaErrorNotSupported;
    } else {
        CUtensorMap map;
        const uint64_t plane_bytes = (g.batch > 1 ? in.plane : in.pitch * g.in_h()) * sizeof(T);
        if (!tma::encode_3d(&map, tma_dtype<T>(), in.base, g.width, g.in_h(), g.batch,
                            in.pitch * sizeof(T), plane_bytes, Ly::BW, Ly::LH))
            return cudaErrorNotSupported;
        static std::atomic<unsigned long long> done{0};
        if (cudaError_t e = ensure_smem(fast_tma_stepk<R, T, K, EXACT1>, Ly::SMEM, done)) return e;
        dim3 grid((g.width + Ly::TWK - 1) / Ly::TWK, (g.height + Ly::THK - 1) / Ly::THK, g.batch);
        note_kernel("fast_tma_stepk");
        fast_tma_stepk<R, T, K, EXACT1><<<grid, Ly::NTT, Ly::SMEM, s>>>(map, out, op, opl, g.width,
                                                                        band_of(g));
        return cudaGetLastError();
    }
}

template <int R, typename T, bool EXACT1>
cudaError_t launch_tmak_passes(const PlaneView& in, const Geometry& g, int k, double* out,
                               size_t op, size_t opl, cudaStream_t s) {
    switch (k) {
        case 2: return launch_tmak<R, T, 2, EXACT1>(in, g, out, op, opl, s);
        case 3: return launch_tmak<R, T, 3, EXACT1>(in, g, out, op, opl, s);
        case 4: return launch_tmak<R, T, 4, EXACT1>(in, g, out, op, opl, s);
        default: return cudaErrorNotSupported;
    }
}

}  // namespace fastk

// k passes in one launch (2 <= k <= kTbMaxPasses, radius <= kTbRadius);
// cudaErrorNotSupported when not applicable (caller runs fewer passes).
template <int R>
cudaError_t fast_launch_radiusk(const PlaneView& in, const Geometry& g, int k, double* out,
                                size_t out_pitch, size_t out_plane, cudaStream_t s) {
    if constexpr (R <= fastk::kTbRadius) {
        switch (in.dtype) {
            case OSBF_U8:
                return fastk::launch_tmak_passes<R, uint8_t, true>(in, g, k, out, out_pitch,
                                                                   out_plane, s);
            case OSBF_F32:
                return fastk::launch_tmak_passes<R, float, false>(in, g, k, out, out_pitch,
                                                                  out_plane, s);
            default:
                return fastk::launch_tmak_passes<R, double, false>(in, g, k, out, out_pitch,
                                                                   out_plane, s);
        }
    }
    return cudaErrorNotSupported;
}

}  // namespace osbf_gpu
