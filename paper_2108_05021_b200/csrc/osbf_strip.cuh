// Fast mode: persistent column-strip walker (the north-star iteration kernel).
//
// One OSBF pass (filters2d.hpp:61-88) with local fp64 box sums: no whole-image
// prefix, every input row read once per strip, O(1) work per pixel in r.
//
// Work: the image is cut into strips of TWS = 32*NWB output columns and bands
// of BH output rows; a work item is one (strip, band, plane).  A persistent
// grid walks the items round robin, every CTA running the same sequence of
// (item, chunk) on two sides:
//
//   producer warp   one thread streams each item's input rows
//                   [Y0 - R, Y0 + nout + R) in chunks of CH rows through a
//                   ring of NU shared-memory slots: one 4-D TMA box per chunk
//                   (rows of TWS + 2R columns, the strip plus its halo; the
//                   hardware zero-fills outside the image, so clipped window
//                   sums need no special case, integral.hpp:53-61).  Slot
//                   full/empty mbarriers; the ring carries on across items,
//                   so the pipeline never drains between them.
//   column warps    NWB warps, one output column per thread.  Per chunk:
//     arms (A)      all column threads together form the horizontal left
//                   arms H(j) = U(j-R) + ... + U(j) of every chunk row into a
//                   shared ring (lanes = CH rows x NSEG segments of SEG
//                   columns, a sliding sum per segment, conflict-free odd
//                   segment lengths), then one named barrier.  Radii 1..2
//                   form the arms directly from 2R+1 samples instead (DIRECT).
//     walk  (B)     each thread walks the chunk's rows with the lead row
//                   L = y + R, keeping for F1 = H(x) (left arm), F2 = H(x+R)
//                   (right arm) and U(x) the sliding column sums
//                       Dn_F(y) = F(y) + ... + F(y+R)   (+= F(L) - F(y-1))
//                   and reading Up_F(y) = Dn_F(y-R) back from a register
//                   ring of the last R values (ring slot = row within the
//                   chunk, so every index is static).  The eight windows
//                   (core.hpp:212-225, u = column, v = row offset) are
//                       w1 = Dn1  w2 = Dn2  w3 = Up2  w4 = Up1
//                       w5 = Up1 + Dn1 - F1(y)   w6 = Up2 + Dn2 - F2(y)
//                       w7 = Dn1 + Dn2 - DnU     w8 = Up1 + Up2 - UpU
//                   The lag values F1(y), F2(y), U(y) come from a second
//                   register ring (LAG_REG) or are re-read from the previous
//                   chunk's shared slots (large radii, register budget).
//     select        d_i = S_i / n_i - u (one fma with the reciprocal count),
//                   stable depth-3 tournament on |d_i| (first minimum wins,
//                   the reference's strict <, filters2d.hpp:72-82) carrying
//                   the window sum, output the winner's mean a_m = S_m / n_m
//                   (filters2d.hpp:80-83).  Lanes are consecutive columns:
//                   coalesced 256-byte row stores.
//
// Decomposition independence (LAG_REG configurations): every CH rows, at lead
// rows that are multiples of CH, the column sums are re-formed from the ring
// in a fixed order, so every value depends only on the global row position,
// not on where a band (or a multi-GPU row band aligned to CH) starts.
// Results are therefore bit-identical for any band height, batch chunking or
// row-band split.
//
// uint8 input (first pass, EXACT_DIV): all sums are exact integers in any
// order; a_i = S_i / n_i is formed IEEE-exactly (q0 = S*y, r = fma(-q0,n,S),
// q = fma(r,y,q0) with y = RN(1/n): exact for integer divisors and normal
// quotients, see osbf_exact2_kernel.cuh) and d_i = |a_i - u| is compared like
// the reference: the first pass is bit-identical.
#pragma once

#include <stdint.h>
#include <stdlib.h>

#include <atomic>
#include <type_traits>

#include "osbf_internal.cuh"
#include "osbf_tma.cuh"

namespace osbf_gpu {
namespace stripk {

// Rows of one launch in global image coordinates (see Geometry).
struct Rows {
    int h_img;   // windows clip at [0, h_img)
    int y_in0;   // global row of input buffer row 0
    int y_out0;  // global row of output buffer row 0
    int y_end;   // one past the last output row
    double* push_up;  // fused halo push (row bands); null = none
    double* push_dn;
    int push_rows;
    long long push_pitch;
};
inline Rows rows_of(const Geometry& g) {
    return Rows{g.img_h(), g.in_row0, g.out_row0, g.out_row0 + g.height,
                g.push_up, g.push_dn, g.push_rows, static_cast<long long>(g.push_pitch)};
}

// ---- shared-memory layout -------------------------------------------------

// Phase A lane idx -> (row idx / nseg, segment idx % nseg); 8-byte accesses at
// row*pitch + seg*seg_len + k.  True when every half-warp hits 16 distinct
// 8-byte bank pairs (conflict-free).
constexpr bool arms_conflict_free(int nlane, int nseg, int seg_len, int pitch) {
    for (int h0 = 0; h0 < nlane; h0 += 16) {
        unsigned mask = 0;
        for (int i = 0; i < 16; ++i) {
            const int idx = h0 + i, row = idx / nseg, s = idx % nseg;
            const int bank = (row * pitch + s * seg_len) % 16;
            if ((mask >> bank) & 1u) return false;
            mask |= 1u << bank;
        }
    }
    return true;
}
constexpr int arms_pitch(int nlane, int nseg, int seg_len, int minp, int step) {
    for (int p = minp; p < minp + 16 * step; p += step)
        if (arms_conflict_free(nlane, nseg, seg_len, p)) return p;
    return minp;
}

template <int R, typename T, int NWB_, int CH_, bool LAG_REG_, bool DIRECT_, int MINB_,
          int NU_ = 0>
struct Cfg {
    static constexpr int RAD = R;
    static constexpr int NWB = NWB_;           // column warps
    static constexpr int TWS = 32 * NWB;       // output columns per strip
    static constexpr int NT = 32 * NWB;
    static constexpr int CH = CH_;             // rows per chunk = ring period
    static constexpr bool LAG_REG = LAG_REG_ || DIRECT_;
    static constexpr bool DIRECT = DIRECT_;
    static constexpr int MINB = MINB_;
    static_assert(CH >= R, "the register rings hold R rows of one chunk period");
    static_assert(CH == 8 || CH == 16 || CH == 32, "chunk rows");
    // TMA: 4-D view {V, W/V, H, B}; the box starts at column X0 - RA
    static constexpr int V = sizeof(T) == 1 ? 16 : 8;
    static constexpr int RA = (R + V - 1) / V * V;
    static constexpr int XOFF = RA - R;
    // phase A (per warp, private slice): lanes = CH rows x NSEG segments of
    // SEG columns over the warp's 32 + R arm columns
    static constexpr int NSEG = 32 / CH;
    static constexpr int SEG = ((32 + R + NSEG - 1) / NSEG) | 1;
    static constexpr int PH0 = DIRECT ? 0 : NSEG * SEG;
    static constexpr int PH = DIRECT ? 0 : arms_pitch(32, NSEG, SEG, PH0, 1);
    // staged columns: warp w's arms read up to 32w + XOFF + PH0 - 1 + R; the
    // direct walk up to RA + TWS - 1 + R
    static constexpr int NEED = DIRECT ? RA + TWS + R : 32 * (NWB - 1) + XOFF + PH0 + R;
    static constexpr int NB1_MIN = (NEED + V - 1) / V;
    static constexpr int NB1 =
        (sizeof(T) == 8 && !DIRECT) ? arms_pitch(32, NSEG, SEG, NB1_MIN * V, V) / V : NB1_MIN;
    static constexpr int BW = NB1 * V;  // staged row pitch (elements)
    static_assert(NB1 <= 256, "TMA box");
    static constexpr uint32_t UBYTES = static_cast<uint32_t>(CH) * BW * sizeof(T);
    static constexpr size_t USLOT = (UBYTES + 127) / 128 * 128;
    static constexpr int NU = NU_ ? NU_ : (LAG_REG ? 3 : 4);
    // per-warp arm slices: one chunk (two when lag rows are re-read)
    static constexpr int NH = DIRECT ? 0 : (LAG_REG ? 1 : 2);
    static constexpr size_t HWARP = static_cast<size_t>(CH) * PH;  // doubles per warp slice
    static constexpr size_t HSLOT = NWB * HWARP * sizeof(double);
    static constexpr size_t SMEM = 128 + NU * USLOT + NH * HSLOT;
    static_assert(SMEM <= 227 * 1024, "strip kernel shared memory");
};

// ---- selection ---------------------------------------------------------------

// IEEE-exact s / n (integer n, y = RN(1/n), normal quotient or 0).
__device__ __forceinline__ double div_count(double s, double n, double y) {
    const double q0 = __dmul_rn(s, y);
    const double r = __fma_rn(-q0, n, s);
    return __fma_rn(r, y, q0);
}

// One tournament stage: keep (da, sa) unless |dc| < |da| (first minimum wins).
__device__ __forceinline__ void stage2(double& da, double& sa, double dc, double sc) {
    const bool p = fabs(dc) < fabs(da);
    da = p ? dc : da;
    sa = p ? sc : sa;
}
__device__ __forceinline__ void stage3(double& da, double& sa, double& ra, double dc, double sc,
                                       double rc) {
    const bool p = fabs(dc) < fabs(da);
    da = p ? dc : da;
    sa = p ? sc : sa;
    ra = p ? rc : ra;
}

// Interior pixel: every quarter has (R+1)^2 samples, every half (R+1)(2R+1).
// The reciprocals are the products of the per-axis reciprocals, formed exactly
// as the border path forms them, so a pixel's result does not depend on
// whether its warp or row is classified as border.
template <int R>
__device__ __forceinline__ double pick_interior(const double (&S)[8], double u) {
    constexpr double kR1 = 1.0 / (R + 1), kR2 = 1.0 / (2 * R + 1);
    constexpr double kRq = kR1 * kR1, kRh = kR1 * kR2;
    double d0 = fma(S[0], kRq, -u), s0 = S[0];
    double d2 = fma(S[2], kRq, -u), s2 = S[2];
    double d4 = fma(S[4], kRh, -u), s4 = S[4];
    double d6 = fma(S[6], kRh, -u), s6 = S[6];
    stage2(d0, s0, fma(S[1], kRq, -u), S[1]);
    stage2(d2, s2, fma(S[3], kRq, -u), S[3]);
    stage2(d4, s4, fma(S[5], kRh, -u), S[5]);
    stage2(d6, s6, fma(S[7], kRh, -u), S[7]);
    stage2(d0, s0, d2, s2);
    stage2(d4, s4, d6, s6);
    const bool half = fabs(d4) < fabs(d0);
    const double sw = half ? s4 : s0;
    const double rw = half ? kRh : kRq;
    return sw * rw;
}

// Border pixel: per-window reciprocals rc[i] = 1 / n_i (clipped counts).
__device__ __forceinline__ double pick_border(const double (&S)[8], double u,
                                              const double (&rc)[8]) {
    double d[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) d[i] = fma(S[i], rc[i], -u);
    double d0 = d[0], s0 = S[0], r0 = rc[0];
    double d2 = d[2], s2 = S[2], r2 = rc[2];
    double d4 = d[4], s4 = S[4], r4 = rc[4];
    double d6 = d[6], s6 = S[6], r6 = rc[6];
    stage3(d0, s0, r0, d[1], S[1], rc[1]);
    stage3(d2, s2, r2, d[3], S[3], rc[3]);
    stage3(d4, s4, r4, d[5], S[5], rc[5]);
    stage3(d6, s6, r6, d[7], S[7], rc[7]);
    stage3(d0, s0, r0, d2, s2, r2);
    stage3(d4, s4, r4, d6, s6, r6);
    stage3(d0, s0, r0, d4, s4, r4);
    return s0 * r0;
}

// Integer sums (uint8 first pass): the reference's arithmetic exactly.
// a_i = S_i / n_i (IEEE), d_i = |a_i - u|, first minimum, output a_m.
__device__ __forceinline__ double pick_exact(const double (&S)[8], double u, const double (&n)[8],
                                             const double (&y)[8]) {
    double a[8], d[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        a[i] = div_count(S[i], n[i], y[i]);
        d[i] = fabs(a[i] - u);
    }
    auto st = [](double& da, double& aa, double dc, double ac) {
        const bool p = dc < da;
        da = p ? dc : da;
        aa = p ? ac : aa;
    };
    double d0 = d[0], a0 = a[0], d2 = d[2], a2 = a[2], d4 = d[4], a4 = a[4], d6 = d[6], a6 = a[6];
    st(d0, a0, d[1], a[1]);
    st(d2, a2, d[3], a[3]);
    st(d4, a4, d[5], a[5]);
    st(d6, a6, d[7], a[7]);
    st(d0, a0, d2, a2);
    st(d4, a4, d6, a6);
    st(d0, a0, d4, a4);
    return a0;
}

// Clipped window counts at a pixel (integral.hpp:53-61): per axis, the number
// of in-image samples of the one-sided arm (n*l, n*r columns; n*u, n*d rows).
struct AxisCounts {
    int l, r, u, d;
};
template <bool EXACT_DIV>
__device__ __forceinline__ double pick_counts(const double (&S)[8], double u, const AxisCounts& c,
                                              const double* __restrict__ rtab) {
    if constexpr (EXACT_DIV) {
        const int cf = c.l + c.r - 1, rf = c.u + c.d - 1;
        const int ni[8] = {c.l * c.d, c.r * c.d, c.r * c.u, c.l * c.u,
                           c.l * rf,  c.r * rf,  cf * c.d,  cf * c.u};
        double n[8], y[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            n[i] = static_cast<double>(ni[i]);
            y[i] = __drcp_rn(n[i]);
        }
        return pick_exact(S, u, n, y);
    } else {
        const double cL = rtab[c.l], cR = rtab[c.r], cF = rtab[c.l + c.r - 1];
        const double rU = rtab[c.u], rD = rtab[c.d], rF = rtab[c.u + c.d - 1];
        const double rc[8] = {cL * rD, cR * rD, cR * rU, cL * rU, cL * rF, cR * rF, cF * rD, cF * rU};
        return pick_border(S, u, rc);
    }
}

// Border columns, interior rows (KIND 1): the five distinct reciprocals of
// the lane's clipped windows, formed once per walk (same products as
// pick_counts forms them per pixel).
struct LaneRecips {
    double qL, qR, hL, hR, fF;  // cL/(R+1), cR/(R+1), cL/(2R+1), cR/(2R+1), cF/(R+1)
    double nL, nR, nF;          // clipped column counts (EXACT_DIV)
};
template <int R, bool EXACT_DIV>
__device__ __forceinline__ double pick_lane(const double (&S)[8], double u, const LaneRecips& lr) {
    if constexpr (EXACT_DIV) {
        constexpr double r1 = R + 1, r2 = 2 * R + 1;
        const double n[8] = {lr.nL * r1, lr.nR * r1, lr.nR * r1, lr.nL * r1,
                             lr.nL * r2, lr.nR * r2, lr.nF * r1, lr.nF * r1};
        double y[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) y[i] = __drcp_rn(n[i]);
        return pick_exact(S, u, n, y);
    } else {
        const double rc[8] = {lr.qL, lr.qR, lr.qR, lr.qL, lr.hL, lr.hR, lr.fF, lr.fF};
        return pick_border(S, u, rc);
    }
}

template <int R, bool EXACT_DIV>
__device__ __forceinline__ double pick_full(const double (&S)[8], double u) {
    if constexpr (EXACT_DIV) {
        constexpr double nq = (R + 1) * (R + 1), nh = (R + 1) * (2 * R + 1);
        constexpr double yq = 1.0 / nq, yh = 1.0 / nh;
        const double n[8] = {nq, nq, nq, nq, nh, nh, nh, nh};
        const double y[8] = {yq, yq, yq, yq, yh, yh, yh, yh};
        return pick_exact(S, u, n, y);
    } else {
        return pick_interior<R>(S, u);
    }
}


// ---- the kernel -----------------------------------------------------------

template <int R, typename T, bool EXACT_DIV, class C>
__global__ void __launch_bounds__(C::NT, C::MINB)
    fast_strip(const __grid_constant__ CUtensorMap tmap, double* __restrict__ out,
               size_t out_pitch, size_t out_plane, int W, Rows rows, int BH, int nbands,
               int nstrips, int nitems) {
    constexpr int CH = C::CH, NWB = C::NWB, TWS = C::TWS, NU = C::NU, NH = C::NH;
    constexpr int BW = C::BW, PH = C::PH;
    constexpr size_t UEL = C::USLOT / sizeof(T);
    extern __shared__ unsigned char smem_raw[];
    __shared__ uint64_t ufull[NU];
    __shared__ unsigned released[NU];  // warps done with the slot (monotonic)
    __shared__ double rtab[2 * R + 2];
    const uint32_t base = tma::smem_u32(smem_raw);
    unsigned char* sm = smem_raw + ((128u - (base & 127u)) & 127u);
    T* Ub = reinterpret_cast<T*>(sm);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    double* Hw = reinterpret_cast<double*>(sm + NU * C::USLOT) + warp * C::HWARP;  // + slot*NWB*HWARP

    // item -> (strip, band, plane); strips fastest, so the CTAs running at the
    // same time read neighbouring strips (their halo columns hit in L2)
    auto decode = [&](int it, int& X0, int& Y0, int& nout, int& b) {
        const int s = it % nstrips, rb = it / nstrips;
        b = rb / nbands;
        X0 = s * TWS;
        Y0 = rows.y_out0 + (rb % nbands) * BH;
        nout = min(BH, rows.y_end - Y0);
    };
    auto nchunks = [&](int it) {
        int X0, Y0, nout, b;
        decode(it, X0, Y0, nout, b);
        return (nout + 2 * R + CH - 1) / CH;
    };
    // TMA load of chunk c of item it into slot q (one thread)
    auto issue = [&](int it, int c, int q) {
        int X0, Y0, nout, b;
        decode(it, X0, Y0, nout, b);
        tma::mbar_arrive_expect_tx(&ufull[q], C::UBYTES);
        tma::load_4d(Ub + q * UEL, &tmap, 0, (X0 - C::RA) / C::V, Y0 - R - rows.y_in0 + c * CH, b,
                     &ufull[q]);
    };
    // chunk `ahead` positions after (it, c) in this CTA's sequence, if any
    auto advance = [&](int& it, int& c, int ahead) {
        c += ahead;
        while (it < nitems) {
            const int n = nchunks(it);
            if (c < n) return true;
            c -= n;
            it += gridDim.x;
        }
        return false;
    };

    if (tid < 2 * R + 2) rtab[tid] = tid ? 1.0 / tid : 0.0;
    if (tid < NU) released[tid] = 0;
    if (tid == 0) {
        for (int q = 0; q < NU; ++q) tma::mbar_init(&ufull[q], 1);
        int it = blockIdx.x, c = 0;
        for (int q = 0; q < NU && it < nitems; ++q) {
            issue(it, c, q);
            advance(it, c, 1);
        }
    }
    __syncthreads();
    // From here on no CTA-wide barrier: every warp walks the chunk sequence on
    // its own, waiting only for the chunk's TMA.  The last warp to release a
    // slot refills it with the chunk NU positions later.
    auto release = [&](int q, int it, int c) {  // slot q held chunk (it, c)
        __syncwarp();
        if (lane == 0) {
            const unsigned n = atomicAdd(&released[q], 1u);
            if ((n + 1) % NWB == 0 && advance(it, c, NU)) {
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                issue(it, c, q);
            }
        }
    };

    const int l = tid;  // column within the strip
    const int Himg = rows.h_img;
    uint32_t seq = 0;
    int prev_it = -1, prev_c = 0;  // chunk held in the previous slot (lag re-reads)
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
        int X0, Y0, nout, b;
        decode(it, X0, Y0, nout, b);
        const int gx = X0 + l;
        const int nsteps = nout + 2 * R;
        const int nch = (nsteps + CH - 1) / CH;
        const bool warp_border = !__all_sync(0xffffffffu, gx >= R && gx < W - R);
        AxisCounts ac{R + 1, R + 1, R + 1, R + 1};
        if (gx < W) {
            ac.l = min(gx, R) + 1;
            ac.r = min(W - 1 - gx, R) + 1;
        }
        double* ocol = out + static_cast<size_t>(b) * out_plane + gx;
        LaneRecips lr;
        {
            const int nf = ac.l + ac.r - 1;
            const double k1 = rtab[R + 1], k2 = rtab[2 * R + 1];
            lr.qL = rtab[ac.l] * k1;
            lr.qR = rtab[ac.r] * k1;
            lr.hL = rtab[ac.l] * k2;
            lr.hR = rtab[ac.r] * k2;
            lr.fF = rtab[nf] * k1;
            lr.nL = ac.l;
            lr.nR = ac.r;
            lr.nF = nf;
        }

        // sliding column sums, lag-(R+1) values, and the rings (slot = row in chunk)
        double Dn1 = 0.0, Dn2 = 0.0, DnU = 0.0, f1p = 0.0, f2p = 0.0, up = 0.0;
        double dr1[CH], dr2[CH], dru[CH], fr1[CH], fr2[CH], fru[CH];
#pragma unroll
        for (int k = 0; k < CH; ++k) {
            dr1[k] = dr2[k] = dru[k] = 0.0;
            fr1[k] = fr2[k] = fru[k] = 0.0;
        }

        for (int c = 0; c < nch; ++c, ++seq) {
            const int q = seq % NU;
            tma::mbar_wait(&ufull[q], (seq / NU) & 1);
            const T* __restrict__ Uq = Ub + q * UEL;
            const T* __restrict__ Uprev = Ub + ((seq + NU - 1) % NU) * UEL;
            double* __restrict__ Hq = Hw + (NH > 1 ? (seq % 2) : 0) * (NWB * C::HWARP);
            const double* __restrict__ Hp = Hw + (NH > 1 ? ((seq + 1) % 2) : 0) * (NWB * C::HWARP);
            if constexpr (!C::DIRECT) {
                // ---- phase A: this warp's arms H(m) = U(m-R) + ... + U(m) of
                // its 32 + R columns, every chunk row
                const int row = lane / C::NSEG, sg = lane % C::NSEG;
                const T* __restrict__ u = Uq + row * BW + 32 * warp + C::XOFF + sg * C::SEG;
                double* __restrict__ h = Hq + row * PH + sg * C::SEG;
                double v[C::SEG + R];
#pragma unroll
                for (int i = 0; i < C::SEG + R; ++i) v[i] = to_f64(u[i]);
                double acc = v[0];
#pragma unroll
                for (int i = 1; i <= R; ++i) acc += v[i];
                h[0] = acc;
#pragma unroll
                for (int m = 1; m < C::SEG; ++m) {
                    acc += v[m + R] - v[m - 1];
                    h[m] = acc;
                }
                __syncwarp();
            }
            const int t0 = c * CH;
            const int y0 = Y0 + t0 - 2 * R;  // output row of the chunk's first step
            const bool all_valid = t0 >= 2 * R && t0 + CH <= nsteps;
            const bool rows_in = y0 >= R && y0 + CH <= Himg - R;
            const bool push_touch =
                rows.push_rows > 0 &&
                (y0 < rows.y_out0 + rows.push_rows || y0 + CH > rows.y_end - rows.push_rows);
            double* o = ocol + static_cast<ptrdiff_t>(y0 - rows.y_out0) * static_cast<ptrdiff_t>(out_pitch);

            auto body = [&](auto kind_tag) {
                constexpr int KIND = decltype(kind_tag)::value;
#pragma unroll
                for (int k = 0; k < CH; ++k) {
                    const int kl = (k - R + CH) % CH;  // ring slot written R steps ago
                    // lead row L = y + R
                    double F1, F2, Uc;
                    if constexpr (C::DIRECT) {
                        const T* __restrict__ ur = Uq + k * BW + l + C::XOFF;
                        double v[2 * R + 1];
#pragma unroll
                        for (int i = 0; i <= 2 * R; ++i) v[i] = to_f64(ur[i]);
                        F1 = v[0];
                        F2 = v[R];
#pragma unroll
                        for (int i = 1; i <= R; ++i) {
                            F1 += v[i];
                            F2 += v[R + i];
                        }
                        Uc = v[R];
                    } else {
                        F1 = Hq[k * PH + lane];
                        F2 = Hq[k * PH + lane + R];
                        Uc = to_f64(Uq[k * BW + l + C::RA]);
                    }
                    // lag-R values F(y): register ring or the shared slots
                    double f1y, f2y, uy;
                    if constexpr (C::LAG_REG) {
                        f1y = fr1[kl];
                        f2y = fr2[kl];
                        uy = fru[kl];
                        fr1[k] = F1;
                        fr2[k] = F2;
                        fru[k] = Uc;
                    } else {
                        if (KIND == 2 && c == 0 && k < R) {
                            f1y = f2y = uy = 0.0;  // rows above the walk's first row
                        } else if (k >= R) {
                            f1y = Hq[(k - R) * PH + lane];
                            f2y = Hq[(k - R) * PH + lane + R];
                            uy = to_f64(Uq[(k - R) * BW + l + C::RA]);
                        } else {
                            f1y = Hp[(k - R + CH) * PH + lane];
                            f2y = Hp[(k - R + CH) * PH + lane + R];
                            uy = to_f64(Uprev[(k - R + CH) * BW + l + C::RA]);
                        }
                    }
                    Dn1 += F1 - f1p;
                    Dn2 += F2 - f2p;
                    DnU += Uc - up;
                    f1p = f1y;
                    f2p = f2y;
                    up = uy;
                    if constexpr (C::LAG_REG) {
                        if (k == R % CH) {
                            // lead row is a multiple of CH: re-form the sums in
                            // a fixed order (decomposition independence)
                            double a1 = f1y, a2 = f2y, a3 = uy;
#pragma unroll
                            for (int i = R - 1; i >= 1; --i) {
                                a1 += fr1[(k - i + CH) % CH];
                                a2 += fr2[(k - i + CH) % CH];
                                a3 += fru[(k - i + CH) % CH];
                            }
                            Dn1 = a1 + F1;
                            Dn2 = a2 + F2;
                            DnU = a3 + Uc;
                        }
                    }
                    const double Up1 = dr1[kl], Up2 = dr2[kl], UpU = dru[kl];
                    dr1[k] = Dn1;
                    dr2[k] = Dn2;
                    dru[k] = DnU;
                    double* ok = o + static_cast<ptrdiff_t>(k) * static_cast<ptrdiff_t>(out_pitch);
                    if (KIND == 2) {
                        const int t = t0 + k;
                        if (t < 2 * R || t >= nsteps) continue;
                    }
                    const double S[8] = {Dn1, Dn2, Up2, Up1, (Up1 + Dn1) - f1y, (Up2 + Dn2) - f2y,
                                         (Dn1 + Dn2) - DnU, (Up1 + Up2) - UpU};
                    if constexpr (KIND == 0) {
                        *ok = pick_full<R, EXACT_DIV>(S, uy);
                    } else if constexpr (KIND == 1) {
                        if (gx < W) *ok = pick_lane<R, EXACT_DIV>(S, uy, lr);
                    } else {
                        const int y = y0 + k;
                        if (gx < W) {
                            double a;
                            if (warp_border || y < R || y >= Himg - R) {
                                AxisCounts cc = ac;
                                cc.u = min(y, R) + 1;
                                cc.d = min(Himg - 1 - y, R) + 1;
                                a = pick_counts<EXACT_DIV>(S, uy, cc, rtab);
                            } else {
                                a = pick_full<R, EXACT_DIV>(S, uy);
                            }
                            *ok = a;
                            if (rows.push_rows > 0) {  // fused halo push (peer memory)
                                if (rows.push_up && y < rows.y_out0 + rows.push_rows)
                                    rows.push_up[static_cast<long long>(y - rows.y_out0) *
                                                     rows.push_pitch + gx] = a;
                                const int yd = rows.y_end - rows.push_rows;
                                if (rows.push_dn && y >= yd)
                                    rows.push_dn[static_cast<long long>(y - yd) * rows.push_pitch +
                                                 gx] = a;
                            }
                        }
                    }
                }
            };
            if (all_valid && rows_in && !push_touch) {
                if (!warp_border)
                    body(std::integral_constant<int, 0>{});
                else
                    body(std::integral_constant<int, 1>{});
            } else {
                body(std::integral_constant<int, 2>{});
            }
            if constexpr (C::LAG_REG) {
                release(q, it, c);
            } else {
                if (prev_it >= 0) release((seq + NU - 1) % NU, prev_it, prev_c);
                prev_it = it;
                prev_c = c;
            }
        }
    }
}

template <typename T>
constexpr CUtensorMapDataType tma_dtype_of() {
    return sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64
                          : (sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                            : CU_TENSOR_MAP_DATA_TYPE_UINT8);
}

// Band height: a function of the plane geometry only (never of the batch or
// the device), so a batch filtered in chunks gives the same bits as one
// launch even for configurations whose sums depend on the walk start.
template <int R, class C>
inline int band_height(int height, int width) {
    const int nstrips = (width + C::TWS - 1) / C::TWS;
    // a single large plane: ~2048 items; batches of small planes: whole planes
    long long bh = static_cast<long long>(height) * nstrips / 2048;
    int b = C::CH * 16;  // >= 256 rows: the 2R-row ramp of a walk stays small
    while (b < bh && b < (1 << 14)) b *= 2;
    if (height <= 2048 || height <= 2 * b) return height;  // one band per plane
    return b;
}

// Returns cudaErrorNotSupported (nothing launched) when TMA cannot describe
// the layout (width not a multiple of the 4-D view's group, misaligned base
// or pitch); the caller then uses the tile kernels.
template <int R, typename T, bool EXACT_DIV, class C>
cudaError_t launch(const PlaneView& in, const Geometry& g, double* out, size_t op, size_t opl,
                   cudaStream_t s) {
    CUtensorMap map;
    const uint64_t plane_bytes = (g.batch > 1 ? in.plane : in.pitch * g.in_h()) * sizeof(T);
    if (!tma::encode_rows_4d(&map, tma_dtype_of<T>(), sizeof(T), in.base, g.width, g.in_h(),
                             g.batch, in.pitch * sizeof(T), plane_bytes, C::V, C::NB1, C::CH))
        return cudaErrorNotSupported;
    auto* fn = fast_strip<R, T, EXACT_DIV, C>;
    static std::atomic<unsigned long long> done{0};
    if (cudaError_t e = ensure_smem(fn, C::SMEM, done)) return e;
    int dev = 0, nsm = 0, per_sm = 0;
    if (cudaError_t e = cudaGetDevice(&dev)) return e;
    if (cudaError_t e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev)) return e;
    if (cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, C::NT, C::SMEM))
        return e;
    if (per_sm < 1) return cudaErrorNotSupported;
    const int BH = band_height<R, C>(g.height, g.width);
    const int nbands = (g.height + BH - 1) / BH;
    const int nstrips = (g.width + C::TWS - 1) / C::TWS;
    const long long items = static_cast<long long>(nbands) * nstrips * g.batch;
    if (items > (1ll << 31) - 1) return cudaErrorNotSupported;
    const int grid = static_cast<int>(items < static_cast<long long>(nsm) * per_sm
                                          ? items
                                          : static_cast<long long>(nsm) * per_sm);
    note_kernel("fast_strip");
    fn<<<grid, C::NT, C::SMEM, s>>>(map, out, op, opl, g.width, rows_of(g), BH, nbands, nstrips,
                                   static_cast<int>(items));
    return cudaGetLastError();
}

// Per-radius configuration (measured).
//   r <= 2    direct arms (2r+1 samples), register rings, 8-row chunks,
//             two 256-thread CTAs per SM
//   r 3..4    per-warp arm pass, register rings, 8-row chunks, two CTAs/SM
//   r 5..8    per-warp arm pass, register rings, 8-row chunks, one CTA/SM
//   r 9..16   per-warp arm pass, lag values re-read from the shared slots
//             (Dn ring only), 16-row chunks, one CTA/SM
template <int R, typename T, int ALT = 0>
struct Pick {
    using type = std::conditional_t<
        (R <= 2), Cfg<R, T, 8, 8, true, true, 2>,
        std::conditional_t<(R <= 4), Cfg<R, T, 8, 8, true, false, 2>,
                           std::conditional_t<(R <= 8), Cfg<R, T, 8, 8, true, false, 1>,
                                              Cfg<R, T, 8, 16, false, false, 1, 3>>>>;
};
// Alternative configuration for A/B measurements (OSBF_GPU_STRIP=2, fp64 input).
template <int R, typename T>
struct Pick<R, T, 1> {
    using type = std::conditional_t<(R <= 8), Cfg<R, T, 8, 16, true, (R <= 2), 1>,
                                    Cfg<R, T, 8, 16, true, false, 1>>;
};

// OSBF_GPU_STRIP: 0 = off (tile / stream kernels), 2 = alternative configs
inline int strip_mode() {
    static int on = -1;
    if (on < 0) {
        const char* e = getenv("OSBF_GPU_STRIP");
        on = (e && e[0] == '0') ? 0 : ((e && e[0] == '2') ? 2 : 1);
    }
    return on;
}

}  // namespace stripk

// One fast pass through the strip walker; cudaErrorNotSupported when it does
// not apply (the tile kernels then run).
template <int R>
cudaError_t strip_launch_radius(const PlaneView& in, const Geometry& g, double* out,
                                size_t out_pitch, size_t out_plane, cudaStream_t s) {
    const int mode = stripk::strip_mode();
    if (mode == 2 && in.dtype == OSBF_F64)
        return stripk::launch<R, double, false, typename stripk::Pick<R, double, 1>::type>(
            in, g, out, out_pitch, out_plane, s);
    switch (in.dtype) {
        case OSBF_U8:
            return stripk::launch<R, uint8_t, true, typename stripk::Pick<R, uint8_t>::type>(
                in, g, out, out_pitch, out_plane, s);
        case OSBF_F32:
            return stripk::launch<R, float, false, typename stripk::Pick<R, float>::type>(
                in, g, out, out_pitch, out_plane, s);
        default:
            return stripk::launch<R, double, false, typename stripk::Pick<R, double>::type>(
                in, g, out, out_pitch, out_plane, s);
    }
}

}  // namespace osbf_gpu
