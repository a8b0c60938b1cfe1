/*
 * TEST INFRASTRUCTURE ONLY — not part of the product.
 *
 * Plain-C restatement of the reference OSBF hot path (arXiv 2108.05021,
 * exact one-sided box filter, paper Algorithm 2) used as the parity checker
 * for the CUDA implementation.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it.
 *
 * Every function restates the reference's arithmetic in the same fp64
 * operation order, so results are bit-identical to the reference's
 * osbf::osbf (pinned against the compiled reference in oracle/_ref and the
 * golden fixtures in tests/golden/).
 */
#ifndef OSBF_ORACLE_H
#define OSBF_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes mirror include/osbf_gpu.h so tests can compare error behaviour. */
#define ORACLE_OK 0
#define ORACLE_ERR_INVALID_ARGUMENT 1
#define ORACLE_ERR_DOMAIN 2

/* Reference window table, core.hpp:212-225.  Fills 8 x {id,u0,u1,v0,v1}. */
int oracle_sub_windows(int r, int out[8][5]);

/* Whole-image summed-area table with zero border, integral.hpp:16-30.
 * cumsum has (w+1)*(h+1) entries, row-major with stride w+1. */
void oracle_sat_build(const double* plane, int w, int h, double* cumsum);

/* integral.hpp:41-50 (clip, ((A-B)-C)+D). */
double oracle_rect_sum(const double* cumsum, int w, int h, int x0, int y0, int x1, int y1);
/* integral.hpp:53-61. */
long long oracle_rect_count(int w, int h, int x0, int y0, int x1, int y1);
/* integral.hpp:64-69; returns ORACLE_ERR_DOMAIN for an empty clipped rect. */
int oracle_rect_mean(const double* cumsum, int w, int h, int x0, int y0, int x1, int y1,
                     double* mean);

/* filters2d.hpp:26-34: the eight window means at (x,y). */
int oracle_subwindow_means(const double* cumsum, int w, int h, int x, int y, int r,
                           double out[8]);

/* filters2d.hpp:61-88: one Jacobi pass.  sel (nullable) receives the
 * 1-based selected window id per pixel (0 if no window won, e.g. NaN). */
int oracle_osbf_step(const double* in, double* out, int w, int h, int r, uint8_t* sel);

/* filters2d.hpp:91-98: `iterations` passes; 0 copies without checking r. */
int oracle_osbf(const double* in, double* out, int w, int h, int r, int iterations);

/* Multi-threaded variant of oracle_osbf (row blocks, like parallel.hpp:33-53);
 * bit-identical to oracle_osbf for any thread count.  Used only as the
 * "port" CPU baseline when the compiled reference is unavailable. */
int oracle_osbf_mt(const double* in, double* out, int w, int h, int r, int iterations,
                   int threads);

/* filters2d.hpp:105-154 (paper Algorithm 3, "fast_osbf"): per iteration one
 * quarter-mean field Q(x,y) = rect_mean(x-r, y-r, x, y) on the whole-image
 * SAT, then 8 candidates from the clamped shifted lookups Q(x,y), Q(x+r,y),
 * Q(x,y+r), Q(x+r,y+r) and their pairwise averages; strict-< first minimum of
 * |c - u|, output the candidate.  r < 1 is rejected even for 0 iterations. */
int oracle_fast_osbf(const double* in, double* out, int w, int h, int r, int iterations);

/* filters2d.hpp:38-56: per iteration the valid-count mean of the clipped
 * (2r+1)^2 window on the whole-image SAT.  r < 1 is rejected even for 0
 * iterations. */
int oracle_box_filter(const double* in, double* out, int w, int h, int r, int iterations);

/* 3-D extension. Volumes are x-fastest, then y, then z.
 * integral.hpp:98-113: summed-volume table with zero border slabs,
 * cumsum[(z*(h+1)+y)*(w+1)+x], built with a running row sum per (y,z) row:
 *   T(x+1,y+1,z+1) = ((row + T(x+1,y,z+1)) + T(x+1,y+1,z)) - T(x+1,y,z). */
void oracle_svt_build(const double* vol, int w, int h, int d, double* cumsum);
/* filters3d.hpp:55-76 (box_filter_3d) and :78-114 (osbf_3d, 14 regions,
 * strict-< first minimum).  r < 1 / iterations < 0 are rejected. */
int oracle_box_filter_3d(const double* in, double* out, int w, int h, int d, int r, int iters);
int oracle_osbf_3d(const double* in, double* out, int w, int h, int d, int r, int iters);

/* The `osbf smooth` edge (tools/osbf_main.cpp:63-83):
 * io.hpp:108-115 quantize (floor(v + 0.5); negatives and NaN -> 0; clamp to
 * maxval), and promote (io.hpp:157-168) -> filter_multichannel
 * (filters2d.hpp:371-400; filter 0 osbf, 1 fast_osbf, 2 box) -> quantise +
 * interleave (io.hpp:202-212) on an interleaved raster of uint8
 * (sample_bytes 1) or uint16 (2) samples; out_sample_bytes 1 -> maxval 255,
 * 2 -> 65535.  Returns nonzero on invalid arguments. */
int oracle_quantize(double v, int maxval);
int oracle_smooth_raster(const void* raster, int sample_bytes, int channels, int w, int h,
                         int filter, int r, int iterations, void* out, int out_sample_bytes);

#ifdef __cplusplus
}
#endif

#endif /* OSBF_ORACLE_H */
