// Fast mode for any radius above the compiled ones (r > kFastMaxRadius): the
// vertical-first column walk, with O(1) state per thread whatever r is.
//
// The templated kernels keep 2r+2 column prefixes per field in registers,
// which stops scaling past r = 16.  Here the eight windows are rebuilt from
// quantities whose state does not grow with r (filters2d.hpp:61-88 windows,
// core.hpp:212-225 order):
//
//   Vup(c,y) = U(c,y-r) + ... + U(c,y)     Vdn(c,y) = U(c,y) + ... + U(c,y+r)
//   NW = sum_{c=x-r..x} Vup   NE = sum_{c=x..x+r} Vup
//   SW = sum_{c=x-r..x} Vdn   SE = sum_{c=x..x+r} Vdn
//   W  = NW + SW - rowL       E  = NE + SE - rowR      (rowL/R: arms of row y)
//   N  = NW + NE - Vup(x)     S  = SW + SE - Vdn(x)
//
// One CTA (128 threads) owns a strip of SW output columns and a block of rows
// and walks down it.  Per chunk of CH walk steps:
//   V  one thread per staged column c (SW + 2r of them): running sums
//        lead += U(j) - U(j-r-1)   (= Vdn of output row y = j - r)
//        lag  += U(j-r) - U(j-2r-1) (= Vup of row y)
//      the new row U(j) arrives by TMA (zero fill outside the image); the
//      rows r and 2r+1 steps back were staged earlier and are re-read from
//      L2 (plain loads), so nothing of size r is kept on chip;
//   A  sliding left arms over the staged columns of Vup, Vdn and U(y)
//      (row segments, one task per field x row x segment);
//   S  one thread per output column: the eight windows, valid-count means,
//      first minimum of |a - u| (fma form, output u + d_m; uint8 input:
//      exact division and a_m, bit-exact first pass), coalesced store.
// Work per pixel is O(1) in r; the only r-dependent costs are the strip's
// 2r halo columns (staged from L2) and the block's r warm-up rows.
#include <stdlib.h>
#include <string.h>

#include "osbf_internal.cuh"
#include "osbf_tma.cuh"

namespace osbf_gpu {
namespace vwalk {

constexpr int NT = 256;  // >= every staged column count (nv <= 256)
constexpr int CH = 8;      // walk steps per chunk
constexpr int NS = 2;      // TMA slots (new rows)
constexpr int BLOCK = 512; // output rows per CTA

// Strip width for radius r: the widest of 128 / 64 / 32 whose staged row
// (SW + 2r columns plus the 16-byte alignment pad) fits one TMA box (256).
inline int strip_width(int r, int align) {
    for (int sw : {128, 64, 32}) {
        const int ra = (r + align - 1) / align * align;
        const int bw = (ra + sw + r + align - 1) / align * align;
        if (bw <= 256) return sw;
    }
    return 0;
}

struct Lay {
    int r, sw, align, ra, xoff, bw, nv, vp, ap, nseg, lsa;
    size_t n_bytes, off_v, off_a, off_rt, total;
};

__host__ __device__ inline Lay make_lay(int r, int sw, int tbytes) {
    Lay l;
    l.r = r;
    l.sw = sw;
    l.align = 16 / tbytes;
    l.ra = (r + l.align - 1) / l.align * l.align;  // TMA x start X0 - ra (16-byte aligned)
    l.xoff = l.ra - r;                             // staged column of V-column 0
    l.bw = (l.ra + sw + r + l.align - 1) / l.align * l.align;
    l.nv = sw + 2 * r;          // V-columns: image columns X0 - r + v
    l.vp = l.nv | 1;            // pitch of the V / Uc rows
    l.ap = (sw + r) | 1;        // pitch of the arm rows
    // arm segments per row (3 fields x CH rows x nseg tasks <= 240): long
    // enough that the r+1-term start of each sliding segment amortises
    l.nseg = (sw + r) / (r + 1);
    l.nseg = l.nseg < 5 ? 5 : (l.nseg > 10 ? 10 : l.nseg);
    l.lsa = (((sw + r) + l.nseg - 1) / l.nseg) | 1;
    const size_t nb = static_cast<size_t>(l.bw) * CH * tbytes;
    l.n_bytes = (nb + 127) / 128 * 128;
    l.off_v = NS * l.n_bytes;                                          // Vu, Vd, Uc
    l.off_a = l.off_v + 3 * sizeof(double) * CH * static_cast<size_t>(l.vp);  // Au, Ad, AU
    // arm segments may read up to lsa + r past a row's last V-column
    l.off_rt = l.off_a + 3 * sizeof(double) * CH * static_cast<size_t>(l.ap) +
               sizeof(double) * (l.lsa + r + 8);
    l.total = l.off_rt + sizeof(double) * (2 * r + 2) + 128;  // + alignment slack
    return l;
}

struct Band {
    int h_img, y_in0, in_rows, y_out0, y_end;
    double* push_up;
    double* push_dn;
    int push_rows;
    long long push_pitch;
};

template <typename T, bool EXACT_DIV, bool TMA>
__global__ void __launch_bounds__(NT, 2)
    fast_vwalk_step(const __grid_constant__ CUtensorMap tmap, const T* __restrict__ in,
                    size_t in_pitch, size_t in_plane, double* __restrict__ out, size_t out_pitch,
                    size_t out_plane, int W, Band band, int R, int SWd) {
    extern __shared__ unsigned char smem_raw[];
    __shared__ uint64_t full[NS];
    const Lay ly = make_lay(R, SWd, sizeof(T));
    const uint32_t base = tma::smem_u32(smem_raw);
    unsigned char* sm = smem_raw + ((128u - (base & 127u)) & 127u);
    T* Nb = reinterpret_cast<T*>(sm);
    double* Vu = reinterpret_cast<double*>(sm + ly.off_v);
    double* Vd = Vu + CH * ly.vp;
    double* Uc = Vd + CH * ly.vp;
    double* Au = reinterpret_cast<double*>(sm + ly.off_a);
    double* Ad = Au + CH * ly.ap;
    double* AU = Ad + CH * ly.ap;
    double* rtab = reinterpret_cast<double*>(sm + ly.off_rt);
    const int tid = threadIdx.x;
    const int X0 = blockIdx.x * ly.sw;
    const int blk = band.y_out0 / BLOCK + static_cast<int>(blockIdx.y);
    const int Y0 = max(band.y_out0, blk * BLOCK);
    const int nout = min(band.y_end, (blk + 1) * BLOCK) - Y0;
    const int nsteps = nout + R;
    const int nchunks = (nsteps + CH - 1) / CH;
    const int b = blockIdx.z;
    const T* src = in + static_cast<size_t>(b) * in_plane;
    const int Himg = band.h_img;
    // rows [lo_ok, hi_ok) of the image are readable from the input buffer
    const int lo_ok = max(0, band.y_in0), hi_ok = min(Himg, band.y_in0 + band.in_rows);

    for (int i = tid; i < 2 * R + 2; i += NT) rtab[i] = i ? 1.0 / i : 0.0;
    if (TMA && tid == 0)
        for (int q = 0; q < NS; ++q) tma::mbar_init(&full[q], 1);
    __syncthreads();
    const size_t n_elems = ly.n_bytes / sizeof(T);
    auto issue = [&](int c) {  // new rows [Y0 + c*CH, +CH) into slot c % NS
        const int q = c % NS;
        tma::mbar_arrive_expect_tx(&full[q], static_cast<uint32_t>(ly.bw * CH * sizeof(T)));
        tma::load_3d(Nb + q * n_elems, &tmap, X0 - ly.ra, Y0 + c * CH - band.y_in0, b, &full[q]);
    };
    if (TMA && tid == 0)
        for (int c = 0; c < NS && c < nchunks; ++c) issue(c);

    // V: one staged column per thread (nv <= 256 = NT)
    const int v = tid;
    const int gc = X0 - R + v;
    const bool vcol = v < ly.nv && gc >= 0 && gc < W;  // column holds image samples
    const T* colp = src + (vcol ? gc : 0);
    double lead = 0.0, lag = 0.0, carry = 0.0;
    // S: output column x = tid % sw, rows k = grp (mod ngrp)
    const int x = tid % ly.sw, grp = tid / ly.sw, ngrp = NT / ly.sw;
    const int gx = X0 + x;
    const bool col_ok = gx < W;
    const bool col_int = gx >= R && gx < W - R;
    const double kR1 = 1.0 / (R + 1), kR2 = 1.0 / (2 * R + 1);
    const double kRq = kR1 * kR1, kRh = kR1 * kR2;
    double cL = 0.0, cR = 0.0, cF = 0.0;
    if (col_ok) {
        const int ncl = min(gx, R) + 1, ncr = min(W - 1 - gx, R) + 1;
        cL = 1.0 / ncl;
        cR = 1.0 / ncr;
        cF = 1.0 / (ncl + ncr - 1);
    }
    const long long pitch_b = static_cast<long long>(in_pitch * sizeof(T));
    auto row_ptr = [&](int gy) { return colp + static_cast<ptrdiff_t>(gy - band.y_in0) * static_cast<ptrdiff_t>(in_pitch); };

    for (int c = 0; c < nchunks; ++c) {
        const int q = c % NS;
        const int j0 = Y0 + c * CH;  // image row of step 0's new row
        // ---- V: running column sums.  U(j-r) and U(j-2r-1) are re-read from
        // L2 (issued before the wait); chunk-uniform row checks keep the
        // interior loads free of per-element tests.
        double ladd[CH], lold[CH], lnew[CH];
        const bool rows_in = j0 - 2 * R - 1 >= lo_ok && j0 + CH - 1 < hi_ok;
        if (vcol && rows_in) {
            const char* pa = reinterpret_cast<const char*>(row_ptr(j0 - R));
            const char* po = reinterpret_cast<const char*>(row_ptr(j0 - 2 * R - 1));
            const bool sub0 = j0 - R - 1 >= Y0;  // every old row subtracted (all but the warm-up)
#pragma unroll
            for (int k = 0; k < CH; ++k) {
                ladd[k] = to_f64(*reinterpret_cast<const T*>(pa + k * pitch_b));
                lold[k] = (sub0 || j0 + k - R - 1 >= Y0)
                              ? to_f64(*reinterpret_cast<const T*>(po + k * pitch_b))
                              : 0.0;
            }
            if constexpr (!TMA) {
                const char* pn = reinterpret_cast<const char*>(row_ptr(j0));
#pragma unroll
                for (int k = 0; k < CH; ++k)
                    lnew[k] = to_f64(*reinterpret_cast<const T*>(pn + k * pitch_b));
            }
        } else {
#pragma unroll
            for (int k = 0; k < CH; ++k) {
                const int j = j0 + k;
                const int ya = j - R, yo = j - 2 * R - 1;
                ladd[k] = (vcol && ya >= lo_ok && ya < hi_ok) ? to_f64(*row_ptr(ya)) : 0.0;
                lold[k] = (vcol && j - R - 1 >= Y0 && yo >= lo_ok && yo < hi_ok)
                              ? to_f64(*row_ptr(yo))
                              : 0.0;
                if constexpr (!TMA)
                    lnew[k] = (vcol && j >= lo_ok && j < hi_ok) ? to_f64(*row_ptr(j)) : 0.0;
            }
        }
        if constexpr (TMA) {
            tma::mbar_wait(&full[q], (c / NS) & 1);
            const T* nrow = Nb + q * n_elems + ly.xoff + v;
#pragma unroll
            for (int k = 0; k < CH; ++k) lnew[k] = to_f64(nrow[k * ly.bw]);
        }
        if (v < ly.nv) {
#pragma unroll
            for (int k = 0; k < CH; ++k) {
                const double lsub = j0 + k - R - 1 >= Y0 ? carry : 0.0;
                lead = (lead + lnew[k]) - lsub;
                lag = (lag + ladd[k]) - lold[k];
                carry = ladd[k];
                Vd[k * ly.vp + v] = lead;
                Vu[k * ly.vp + v] = lag;
                Uc[k * ly.vp + v] = ladd[k];
            }
        }
        __syncthreads();  // V rows of the chunk done; slot q free
        if (TMA && tid == 0 && c + NS < nchunks) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            issue(c + NS);
        }
        // ---- A: left arms over the V rows, a in [0, sw + r) ----------------
        const int narm = ly.sw + R;
        for (int t = tid; t < 3 * CH * ly.nseg; t += NT) {
            const int s = t % ly.nseg, fk = t / ly.nseg, k = fk % CH, f = fk / CH;
            const double* vsrc = (f == 0 ? Vu : f == 1 ? Vd : Uc) + k * ly.vp;
            double* adst = (f == 0 ? Au : f == 1 ? Ad : AU) + k * ly.ap;
            const int a0 = s * ly.lsa;
            if (a0 >= narm) continue;
            const int a1 = min(narm, a0 + ly.lsa);
            const double* vp0 = vsrc + a0;
            double acc = 0.0;
#pragma unroll 4
            for (int i = 0; i <= R; ++i) acc += vp0[i];
            double* ap0 = adst + a0;
            ap0[0] = acc;
            const double* vin = vp0 + R;  // entering column a + R
#pragma unroll 4
            for (int m = 1; m < a1 - a0; ++m) {
                acc += vin[m] - vp0[m - 1];
                ap0[m] = acc;
            }
        }
        __syncthreads();
        // ---- S: windows and selection for the chunk's output rows ---------
        if (col_ok) {
            const double* au = Au + grp * ly.ap + x;
            const double* vv = Vu + grp * ly.vp + x + R;
            const int astep = ngrp * ly.ap, vstep = ngrp * ly.vp;
            const int ad = static_cast<int>(Ad - Au), vd_off = static_cast<int>(Vd - Vu);
            const int uc_off = static_cast<int>(Uc - Vu);
            for (int k = grp; k < CH; k += ngrp, au += astep, vv += vstep) {
                const int y = j0 + k - R;
                if (y < Y0 || y >= Y0 + nout) continue;
                const double nw = au[0], ne = au[R];
                const double sw = au[ad], se = au[ad + R];
                const double hl = au[2 * ad], hr = au[2 * ad + R];
                const double vu = vv[0], vd = vv[vd_off];
                const double u = vv[uc_off];
                const double S[8] = {sw, se, ne, nw, (nw + sw) - hl, (ne + se) - hr,
                                     (sw + se) - vd, (nw + ne) - vu};
                double* o = out + static_cast<size_t>(b) * out_plane +
                            static_cast<size_t>(y - band.y_out0) * out_pitch + gx;
                const bool interior = col_int && y >= R && y < Himg - R;
                if constexpr (EXACT_DIV) {
                    // integer sums: reference arithmetic a_i = S_i / n_i, |a - u|,
                    // strict < in window order, output a_m (filters2d.hpp:74-83)
                    const int ncl = min(gx, R) + 1, ncr = min(W - 1 - gx, R) + 1;
                    const int nru = min(y, R) + 1, nrd = min(Himg - 1 - y, R) + 1;
                    const int n[8] = {ncl * nrd, ncr * nrd, ncr * nru, ncl * nru,
                                      ncl * (nru + nrd - 1), ncr * (nru + nrd - 1),
                                      (ncl + ncr - 1) * nrd, (ncl + ncr - 1) * nru};
                    double best = 0.0, best_abs = __longlong_as_double(0x7ff0000000000000LL);
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const double a = __ddiv_rn(S[i], static_cast<double>(n[i]));
                        const double d = fabs(a - u);
                        if (d < best_abs) {
                            best_abs = d;
                            best = a;
                        }
                    }
                    *o = best;
                } else {
                    // 1/n: interior constants, or products of the clipped
                    // per-axis reciprocals (as the templated kernels form them)
                    double rc[8];
                    if (interior) {
#pragma unroll
                        for (int i = 0; i < 8; ++i) rc[i] = i < 4 ? kRq : kRh;
                    } else {
                        const int nru = min(y, R) + 1, nrd = min(Himg - 1 - y, R) + 1;
                        const double rU = rtab[nru], rD = rtab[nrd], rF = rtab[nru + nrd - 1];
                        rc[0] = cL * rD; rc[1] = cR * rD; rc[2] = cR * rU; rc[3] = cL * rU;
                        rc[4] = cL * rF; rc[5] = cR * rF; rc[6] = cF * rD; rc[7] = cF * rU;
                    }
                    double d[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) d[i] = fma(S[i], rc[i], -u);
                    auto pick = [](double a, double cc) { return fabs(cc) < fabs(a) ? cc : a; };
                    const double best = pick(pick(pick(d[0], d[1]), pick(d[2], d[3])),
                                             pick(pick(d[4], d[5]), pick(d[6], d[7])));
                    *o = u + best;
                }
            }
        }
        __syncthreads();  // V / A rows free for the next chunk
    }
    // fused halo push (row-band mode): forward the band's first / last rows
    if (band.push_rows && col_ok && grp == 0) {
        const double* outp = out + static_cast<size_t>(b) * out_plane;
        for (int gy = Y0; gy < Y0 + nout; ++gy) {
            const double val = outp[static_cast<size_t>(gy - band.y_out0) * out_pitch + gx];
            if (band.push_up && gy < band.y_out0 + band.push_rows)
                band.push_up[static_cast<long long>(gy - band.y_out0) * band.push_pitch + gx] = val;
            if (band.push_dn && gy >= band.y_end - band.push_rows)
                band.push_dn[static_cast<long long>(gy - (band.y_end - band.push_rows)) *
                                 band.push_pitch + gx] = val;
        }
    }
}

template <typename T>
constexpr CUtensorMapDataType tma_dtype() {
    return sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64
                          : (sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                            : CU_TENSOR_MAP_DATA_TYPE_UINT8);
}

template <typename T, bool EXACT_DIV>
cudaError_t launch(const PlaneView& in, const Geometry& g, int r, double* out, size_t op,
                   size_t opl, cudaStream_t s) {
    const int sw = strip_width(r, 16 / static_cast<int>(sizeof(T)));
    if (!sw) return cudaErrorNotSupported;
    const Lay ly = make_lay(r, sw, sizeof(T));
    if (ly.total > 227 * 1024) return cudaErrorNotSupported;
    CUtensorMap map;
    memset(&map, 0, sizeof(map));
    const uint64_t plane_bytes = (g.batch > 1 ? in.plane : in.pitch * g.in_h()) * sizeof(T);
    // TMA for the new rows when the layout allows it; otherwise the new rows
    // are plain loads like the old ones (odd fp64 widths, unaligned views)
    const bool use_tma = tma::encode_3d(&map, tma_dtype<T>(), in.base, g.width, g.in_h(), g.batch,
                                        in.pitch * sizeof(T), plane_bytes, ly.bw, CH);
    auto kern = use_tma ? fast_vwalk_step<T, EXACT_DIV, true> : fast_vwalk_step<T, EXACT_DIV, false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(ly.total));
    if (e != cudaSuccess) return e;
    Band bd{g.img_h(), g.in_row0, g.in_h(), g.out_row0, g.out_row0 + g.height,
            g.push_up, g.push_dn, g.push_rows, static_cast<long long>(g.push_pitch)};
    const int y0 = g.out_row0, y1 = g.out_row0 + g.height;
    dim3 grid((g.width + sw - 1) / sw, (y1 - 1) / BLOCK - y0 / BLOCK + 1, g.batch);
    note_kernel("fast_vwalk_step");
    kern<<<grid, NT, ly.total, s>>>(map, static_cast<const T*>(in.base), in.pitch, in.plane, out,
                                    op, opl, g.width, bd, r, sw);
    return cudaGetLastError();
}

}  // namespace vwalk

cudaError_t fast_generic_step(const PlaneView& in, const Geometry& g, int radius, double* out,
                              size_t out_pitch, size_t out_plane, cudaStream_t s,
                              LaunchCounter& lc) {
    if (radius < 1) return cudaErrorInvalidValue;
    cudaError_t e = cudaErrorNotSupported;
    switch (in.dtype) {
        case OSBF_U8: e = vwalk::launch<uint8_t, true>(in, g, radius, out, out_pitch, out_plane, s); break;
        case OSBF_F32: e = vwalk::launch<float, false>(in, g, radius, out, out_pitch, out_plane, s); break;
        default: e = vwalk::launch<double, false>(in, g, radius, out, out_pitch, out_plane, s); break;
    }
    if (e == cudaSuccess) ++lc.launches;
    return e;
}

int fast_generic_max_radius() {
    // the largest radius every input dtype's staged row fits (one TMA box,
    // strip >= 32 columns, shared memory within the CTA limit)
    auto fits = [](int r) {
        for (int tb : {8, 4, 1}) {
            const int sw = vwalk::strip_width(r, 16 / tb);
            if (!sw || vwalk::make_lay(r, sw, tb).total > 227 * 1024) return false;
        }
        return true;
    };
    int r = kFastMaxRadius;
    while (fits(r + 1)) ++r;
    return r;
}

}  // namespace osbf_gpu
