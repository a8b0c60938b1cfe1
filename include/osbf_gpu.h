/*
 * osbf_gpu.h — C ABI of the B200-native One-Sided Box Filter (OSBF) library
 * (libosbf_gpu.so, hand-written sm_100a CUDA).
 *
 * This is the drop-in boundary for the reference's exact-OSBF hot path.  The
 * reference is header-only C++ (namespace osbf, /root/reference/proj/include);
 * the C++ headers in include/osbf/ keep its declarations and forward to the
 * entry points below.  Each entry point names the reference interface it
 * replaces (paths relative to /root/reference/proj/include/osbf/).
 *
 * Conventions
 *  - Planes are row-major, x (column) fastest: sample(x,y) = base[y*pitch + x]
 *    (core.hpp:61-63).  `pitch` is in ELEMENTS of the plane's dtype.
 *  - A batch is `batch` planes of identical size, `plane_stride` elements apart
 *    (channels of a MultiChannelImage are batch entries).
 *  - Outputs are always fp64, like ImagePlane (core.hpp:73).
 *  - Every function returns an osbf_status; on failure osbf_gpu_last_error()
 *    returns a thread-local message.  Status codes map 1:1 onto the exception
 *    types the reference throws (std::invalid_argument, std::domain_error,
 *    std::out_of_range); CUDA failures are OSBF_ERR_CUDA.
 *  - There is no CPU fallback: without a usable sm_100 device every compute
 *    entry point fails with OSBF_ERR_NO_DEVICE.
 */
#ifndef OSBF_GPU_H
#define OSBF_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OSBF_GPU_ABI_VERSION 1

typedef enum osbf_status {
    OSBF_OK = 0,
    OSBF_ERR_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument */
    OSBF_ERR_DOMAIN = 2,           /* reference: std::domain_error     */
    OSBF_ERR_OUT_OF_RANGE = 3,     /* reference: std::out_of_range     */
    OSBF_ERR_CUDA = 4,             /* CUDA runtime / launch failure     */
    OSBF_ERR_NO_DEVICE = 5,        /* no usable sm_100 GPU              */
    OSBF_ERR_ALLOC = 6             /* device or pinned allocation failed */
} osbf_status;

typedef enum osbf_dtype {
    OSBF_U8 = 0,  /* 8-bit integer samples, promoted exactly to fp64 */
    OSBF_F32 = 1, /* float32 samples, promoted exactly to fp64       */
    OSBF_F64 = 2  /* fp64 samples (the reference's ImagePlane)        */
} osbf_dtype;

typedef enum osbf_mode {
    /* Bit-identical to the reference: replays the whole-image fp64
     * summed-area table in the reference's serial order (integral.hpp:16-30),
     * ((A-B)-C)+D window sums (integral.hpp:48-49), IEEE division by the
     * valid count (integral.hpp:68) and the strict-< first-minimum selection
     * (filters2d.hpp:72-82).  Default for the drop-in C++ API. */
    OSBF_MODE_EXACT = 0,
    /* Tile-local fp64 sums (no whole-image prefix, no drift on huge images),
     * same selection rule.  Bit-identical to the reference whenever the
     * window sums are exact (integer-valued input, e.g. uint8 first pass);
     * otherwise within a few fp64 ulps per pass.  Radii above 16 run the
     * exact kernels. */
    OSBF_MODE_FAST = 1
} osbf_mode;

typedef struct osbf_ctx osbf_ctx;

/* ---- library / context --------------------------------------------------- */

int osbf_gpu_abi_version(void);
/* Thread-local text of the last failure on this thread ("" if none). */
const char* osbf_gpu_last_error(void);

/* Name of the kernel family that ran the last pass issued by this host thread
 * (e.g. "fast_strip", "fast_tma_step", "exact_strip"); instrumentation for
 * tests and the benchmark, no reference counterpart. */
const char* osbf_gpu_last_kernel(void);

/* Diagnostics: force the kernel family of fast passes process-wide ("walk",
 * "tma", "stream", "strip", "tile", "sep", ...; NULL or "" = per-radius default).  A family
 * that does not apply to a pass (radius, layout) falls through to the
 * default order.  No reference counterpart; results stay within fast mode's
 * tolerance whichever family runs. */
osbf_status osbf_gpu_set_fast_kernel(const char* name);
/* Diagnostics: force the kernel family of exact passes process-wide: "strip"
 * (the fused strip walk, r <= 16), or the stencil of the whole-table path:
 * "gwalk" (generic-radius walk, the default), "twalk" (templated walk,
 * r <= 16), "stencil" (per-thread corner loads); NULL or "" = default.  A
 * family that does not apply falls through to the next.  Every family is
 * bit-identical to the reference.  No reference counterpart. */
osbf_status osbf_gpu_set_exact_kernel(const char* name);
/* Largest radius with a fast-mode kernel: radii up to 16 run the templated
 * kernels; above that whole planes run the exact table path in either mode
 * (bit-identical to the reference and faster there than the generic walk;
 * the reference accepts any r >= 1, filters2d.hpp:61-63), and row bands
 * (osbf_gpu_step_band*) run the generic vertical-first walk (O(1) state per
 * thread in r) for radii up to this value.  No reference counterpart;
 * host-only, no device needed. */
int osbf_gpu_fast_max_radius(void);
/* 1 if a CUDA device of compute capability 10.x is visible, else 0. */
int osbf_gpu_device_available(void);

/* A context owns device scratch (ping-pong planes, SAT workspace) and a
 * default stream on `device`.  Reentrant per context; use one per thread. */
osbf_status osbf_gpu_ctx_create(int device, osbf_ctx** out);
osbf_status osbf_gpu_ctx_destroy(osbf_ctx* ctx);
/* Release cached scratch (it is regrown on demand). */
osbf_status osbf_gpu_ctx_trim(osbf_ctx* ctx);
/* Number of kernels this context has launched so far (instrumentation). */
uint64_t osbf_gpu_ctx_launch_count(const osbf_ctx* ctx);
/* Fast mode temporal blocking (north-star K4): passes_per_launch = k in
 * 2..4 runs k passes per launch over tiles staged with a k*r halo (the k-1
 * intermediate planes live in shared memory, every pass clips its windows at
 * the global image border), for radius <= 4; the HBM traffic per iteration
 * drops k-fold.  1 = one pass per launch (default).  Results equal the
 * single-pass ones up to the fast mode's fp64 rounding. */
osbf_status osbf_gpu_ctx_set_temporal_blocking(osbf_ctx* ctx, int passes_per_launch);

/* ---- device-resident entry points (throughput path) ---------------------- */

/*
 * Replaces osbf::osbf (filters2d.hpp:91-98) and, for iterations == 1,
 * osbf::osbf_step (filters2d.hpp:61-88), batched over `batch` planes.
 *   d_in  : device pointer, dtype `in_dtype`, batch x height x in_pitch
 *   d_out : device pointer, fp64, batch x height x out_pitch (may alias d_in
 *           only when in_dtype == OSBF_F64 and the pitches/strides match)
 *   stream: cudaStream_t (NULL = the CUDA default stream, as everywhere in
 *           CUDA); the call is asynchronous with respect to the host.
 * Errors (reference behaviour): iterations < 0 -> INVALID_ARGUMENT
 * (filters2d.hpp:92-93); radius < 1 with iterations > 0 -> INVALID_ARGUMENT
 * (filters2d.hpp:62-63); iterations == 0 copies without checking radius
 * (filters2d.hpp:94-97); width or height < 1 -> INVALID_ARGUMENT (core.hpp:20-21).
 */
osbf_status osbf_gpu_iterate(osbf_ctx* ctx, osbf_dtype in_dtype, const void* d_in,
                             size_t in_pitch, size_t in_plane_stride, double* d_out,
                             size_t out_pitch, size_t out_plane_stride, int width, int height,
                             int batch, int radius, int iterations, osbf_mode mode,
                             void* stream);

/*
 * Per-pixel diagnostics for one pass over `batch` planes (exact SAT):
 *   d_means (nullable): fp64 [batch][height][width][8] — subwindow_means
 *                       (filters2d.hpp:26-34) at every pixel;
 *   d_sel   (nullable): uint8 [batch][height][width] — 1-based id of the
 *                       window osbf_step selects (filters2d.hpp:72-82).
 */
osbf_status osbf_gpu_subwindow_means(osbf_ctx* ctx, osbf_dtype in_dtype, const void* d_in,
                                     size_t in_pitch, size_t in_plane_stride, int width,
                                     int height, int batch, int radius, double* d_means,
                                     uint8_t* d_sel, osbf_mode mode, void* stream);

/*
 * Paper Algorithm 3 — the reference's fast_osbf (filters2d.hpp:105-154) —
 * bit-identical: per iteration the whole-image SAT in the reference's order,
 * the quarter field Q(x,y) = rect_mean(x-r, y-r, x, y), then the 8
 * candidates from the clamped shifted quarters and their pairwise averages,
 * strict-< first minimum of |c - u|.  Same buffer conventions as
 * osbf_gpu_iterate.  radius < 1 is INVALID_ARGUMENT even for 0 iterations
 * (filters2d.hpp:107-110).
 */
osbf_status osbf_gpu_fast_osbf(osbf_ctx* ctx, osbf_dtype in_dtype, const void* d_in,
                              size_t in_pitch, size_t in_plane_stride, double* d_out,
                              size_t out_pitch, size_t out_plane_stride, int width, int height,
                              int batch, int radius, int iterations, void* stream);

/*
 * The classical box filter (filters2d.hpp:38-56), bit-identical: per
 * iteration the whole-image SAT in the reference's order and the
 * valid-count mean of the clipped (2r+1)^2 window.  Same conventions and
 * error order as osbf_gpu_fast_osbf (radius checked first).
 */
osbf_status osbf_gpu_box_filter(osbf_ctx* ctx, osbf_dtype in_dtype, const void* d_in,
                               size_t in_pitch, size_t in_plane_stride, double* d_out,
                               size_t out_pitch, size_t out_plane_stride, int width, int height,
                               int batch, int radius, int iterations, void* stream);

/*
 * 3-D extension (filters3d.hpp:55-114): osbf_3d (14 one-sided regions) and
 * box_filter_3d on one fp64 volume, samples x-fastest then y then z (the
 * reference's Volume layout, core.hpp:148-150), bit-identical (the
 * summed-volume table of integral.hpp:98-113 in the reference's order).
 * radius < 1 is INVALID_ARGUMENT even for 0 iterations.
 */
osbf_status osbf_gpu_osbf_3d(osbf_ctx* ctx, const double* d_in, double* d_out, int width,
                            int height, int depth, int radius, int iterations, void* stream);
osbf_status osbf_gpu_box_filter_3d(osbf_ctx* ctx, const double* d_in, double* d_out, int width,
                                  int height, int depth, int radius, int iterations,
                                  void* stream);

/*
 * Whole-image summed-area table, bit-identical to SummedAreaTable
 * (integral.hpp:16-30): d_cumsum is fp64 [batch][height+1][width+1].
 */
osbf_status osbf_gpu_sat(osbf_ctx* ctx, osbf_dtype in_dtype, const void* d_in, size_t in_pitch,
                         size_t in_plane_stride, int width, int height, int batch,
                         double* d_cumsum, void* stream);

/*
 * One FAST-mode pass over a row band of a taller image (multi-GPU row-band
 * partitioning).  d_in holds global rows [in_row0, in_row0 + in_rows) — the
 * band plus `radius` halo rows on each side where the image has them;
 * d_out receives global rows [out_row0, out_row0 + out_rows).  Windows clip
 * at the global image [0, image_height), so the union of the bands equals a
 * pass over the whole image (bit-identical when every out_row0 is a multiple
 * of the 64-row tile).  Exact mode is rejected with INVALID_ARGUMENT: its
 * whole-image serial prefix (integral.hpp:20-29) cannot be split into bands.
 */
osbf_status osbf_gpu_step_band(osbf_ctx* ctx, osbf_dtype in_dtype, const void* d_in,
                               size_t in_pitch, int in_row0, int in_rows, double* d_out,
                               size_t out_pitch, int out_row0, int out_rows, int width,
                               int image_height, int radius, osbf_mode mode, void* stream);

/*
 * osbf_gpu_step_band with the halo exchange fused into the pass: output rows
 * [out_row0, out_row0 + push_rows) are also stored to d_push_up (the upper
 * neighbour's bottom halo rows, row pitch push_pitch elements) and rows
 * [out_row0 + out_rows - push_rows, out_row0 + out_rows) to d_push_down (the
 * lower neighbour's top halo rows).  The push pointers may be peer memory
 * (NVLink / symmetric memory) or NULL (no neighbour on that side); the
 * caller orders the next pass after every rank's push (e.g. a device-side
 * barrier).  Replaces the separate send/recv step the reference does not
 * have (it is single-node CPU).
 */
osbf_status osbf_gpu_step_band_push(osbf_ctx* ctx, osbf_dtype in_dtype, const void* d_in,
                                    size_t in_pitch, int in_row0, int in_rows, double* d_out,
                                    size_t out_pitch, int out_row0, int out_rows, int width,
                                    int image_height, int radius, osbf_mode mode,
                                    double* d_push_up, double* d_push_down, int push_rows,
                                    size_t push_pitch, void* stream);

/* ---- host-buffer entry points (what the drop-in C++ API calls) ------------ */

/* osbf::osbf on host memory: copies in, filters, copies out, synchronizes.
 * h_in has `batch` planes of width*height samples back to back (dtype
 * in_dtype); h_out receives batch*width*height doubles. */
osbf_status osbf_gpu_osbf_host(osbf_ctx* ctx, osbf_dtype in_dtype, const void* h_in,
                               double* h_out, int width, int height, int batch, int radius,
                               int iterations, osbf_mode mode);

/* osbf::osbf_step (filters2d.hpp:61-88) on one host plane: always validates r. */
osbf_status osbf_gpu_osbf_step_host(osbf_ctx* ctx, const double* h_in, double* h_out, int width,
                                    int height, int radius, osbf_mode mode);

/* osbf::filter_multichannel, OsbfExact branch (filters2d.hpp:371-400):
 * `channels` (1..4) separate host planes, each width*height doubles. */
osbf_status osbf_gpu_filter_multichannel_host(osbf_ctx* ctx, const double* const* h_in,
                                              double* const* h_out, int channels, int width,
                                              int height, int radius, int iterations,
                                              osbf_mode mode);

/* osbf::fast_osbf on host memory (batch planes back to back), like
 * osbf_gpu_osbf_host. */
osbf_status osbf_gpu_fast_osbf_host(osbf_ctx* ctx, osbf_dtype in_dtype, const void* h_in,
                                    double* h_out, int width, int height, int batch, int radius,
                                    int iterations);

/* osbf::osbf_3d / box_filter_3d on host memory (one volume). */
osbf_status osbf_gpu_osbf_3d_host(osbf_ctx* ctx, const double* h_in, double* h_out, int width,
                                 int height, int depth, int radius, int iterations);
osbf_status osbf_gpu_box_filter_3d_host(osbf_ctx* ctx, const double* h_in, double* h_out,
                                       int width, int height, int depth, int radius,
                                       int iterations);

/* SummedVolumeTable (integral.hpp:98-113) built on the GPU, bit-identical:
 * h_cumsum receives (width+1)*(height+1)*(depth+1) doubles, x fastest. */
osbf_status osbf_gpu_svt_host(osbf_ctx* ctx, const double* h_in, int width, int height, int depth,
                             double* h_cumsum);

/* osbf::box_filter on host memory (batch planes back to back). */
osbf_status osbf_gpu_box_filter_host(osbf_ctx* ctx, osbf_dtype in_dtype, const void* h_in,
                                     double* h_out, int width, int height, int batch, int radius,
                                     int iterations);

/* osbf::filter_multichannel with FilterVariant::Box (filters2d.hpp:379). */
osbf_status osbf_gpu_filter_multichannel_box_host(osbf_ctx* ctx, const double* const* h_in,
                                                  double* const* h_out, int channels, int width,
                                                  int height, int radius, int iterations);

/* osbf::filter_multichannel with FilterVariant::OsbfFast (filters2d.hpp:386):
 * fast_osbf on every channel (one batched launch per pass). */
osbf_status osbf_gpu_filter_multichannel_fast_host(osbf_ctx* ctx, const double* const* h_in,
                                                   double* const* h_out, int channels, int width,
                                                   int height, int radius, int iterations);

/* The `osbf smooth` edge (tools/osbf_main.cpp:63-83):
 * read_image's promotion (io.hpp:122-178), filter_multichannel with the
 * given filter and write_image's quantisation (io.hpp:187-215: round half
 * up, negatives/NaN to 0, clamp to 255 or 65535, quantize io.hpp:108-115)
 * in one call.  `h_raster` holds the decoded, host-endian samples of a
 * PGM/PPM payload, interleaved (channels 1 or 3, sample_bytes 1 = uint8,
 * 2 = uint16); `h_out` receives the quantised interleaved samples
 * (out_sample_bytes 1 -> maxval 255, 2 -> 65535).  Promotion and
 * quantisation run on the GPU, so the raster crosses PCIe as 1-2 B per
 * sample.  `mode` applies to OSBF_FILTER_OSBF only. */
typedef enum osbf_filter {
    OSBF_FILTER_OSBF = 0,      /* FilterVariant::OsbfExact, CLI "osbf"       */
    OSBF_FILTER_FAST_OSBF = 1, /* FilterVariant::OsbfFast,  CLI "fast-osbf"  */
    OSBF_FILTER_BOX = 2        /* FilterVariant::Box,       CLI "box"        */
} osbf_filter;

osbf_status osbf_gpu_smooth_raster_host(osbf_ctx* ctx, const void* h_raster, int sample_bytes,
                                        int channels, int width, int height, osbf_filter filter,
                                        int radius, int iterations, osbf_mode mode, void* h_out,
                                        int out_sample_bytes);

/* SummedAreaTable construction (integral.hpp:16-30) for host planes. */
osbf_status osbf_gpu_sat_host(osbf_ctx* ctx, const double* h_in, int width, int height,
                              double* h_cumsum);

#ifdef __cplusplus
}
#endif

#endif /* OSBF_GPU_H */
