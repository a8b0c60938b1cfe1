/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference OSBF path.
 * See osbf_oracle.h.  Reference citations are relative to
 * /root/reference/proj/include/osbf/.
 *
 * Build: oracle/Makefile (gcc -O2 -std=c11, no -ffast-math; x86-64 baseline
 * has no FMA so nothing can be contracted and the op order is the source
 * order, exactly like the reference built with its CMake Release flags).
 */
#include "osbf_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

int oracle_sub_windows(int r, int out[8][5]) {
    /* core.hpp:212-225 — order is the tie-break order (first minimum wins). */
    if (r < 1) return ORACLE_ERR_INVALID_ARGUMENT;
    const int t[8][5] = {
        {1, -r, 0, 0, r}, {2, 0, r, 0, r},  {3, 0, r, -r, 0}, {4, -r, 0, -r, 0},
        {5, -r, 0, -r, r}, {6, 0, r, -r, r}, {7, -r, r, 0, r}, {8, -r, r, -r, 0},
    };
    memcpy(out, t, sizeof(t));
    return ORACLE_OK;
}

void oracle_sat_build(const double* plane, int w, int h, double* cumsum) {
    /* integral.hpp:16-30: serial row running sum, then add the table row above. */
    const size_t stride = (size_t)w + 1;
    memset(cumsum, 0, sizeof(double) * stride * ((size_t)h + 1));
    for (int y = 0; y < h; ++y) {
        double row = 0.0;
        const double* src = plane + (size_t)y * w;
        const double* above = cumsum + (size_t)y * stride;
        double* out = cumsum + (size_t)(y + 1) * stride;
        for (int x = 0; x < w; ++x) {
            row += src[x];
            out[x + 1] = above[x + 1] + row;
        }
    }
}

static inline int imax(int a, int b) { return a > b ? a : b; }
static inline int imin(int a, int b) { return a < b ? a : b; }

double oracle_rect_sum(const double* c, int w, int h, int x0, int y0, int x1, int y1) {
    /* integral.hpp:41-50 */
    x0 = imax(x0, 0);
    y0 = imax(y0, 0);
    x1 = imin(x1, w - 1);
    y1 = imin(y1, h - 1);
    if (x0 > x1 || y0 > y1) return 0.0;
    const size_t s = (size_t)w + 1;
    return c[(size_t)(y1 + 1) * s + (x1 + 1)] - c[(size_t)(y1 + 1) * s + x0] -
           c[(size_t)y0 * s + (x1 + 1)] + c[(size_t)y0 * s + x0];
}

long long oracle_rect_count(int w, int h, int x0, int y0, int x1, int y1) {
    /* integral.hpp:53-61 */
    x0 = imax(x0, 0);
    y0 = imax(y0, 0);
    x1 = imin(x1, w - 1);
    y1 = imin(y1, h - 1);
    if (x0 > x1 || y0 > y1) return 0;
    return (long long)(x1 - x0 + 1) * (y1 - y0 + 1);
}

int oracle_rect_mean(const double* c, int w, int h, int x0, int y0, int x1, int y1,
                     double* mean) {
    /* integral.hpp:64-69 */
    const long long n = oracle_rect_count(w, h, x0, y0, x1, y1);
    if (n == 0) return ORACLE_ERR_DOMAIN;
    *mean = oracle_rect_sum(c, w, h, x0, y0, x1, y1) / (double)n;
    return ORACLE_OK;
}

int oracle_subwindow_means(const double* c, int w, int h, int x, int y, int r, double out[8]) {
    /* filters2d.hpp:26-34 */
    int wins[8][5];
    int st = oracle_sub_windows(r, wins);
    if (st) return st;
    for (int i = 0; i < 8; ++i) {
        st = oracle_rect_mean(c, w, h, x + wins[i][1], y + wins[i][3], x + wins[i][2],
                              y + wins[i][4], &out[i]);
        if (st) return st;
    }
    return ORACLE_OK;
}

/* Inner loop of filters2d.hpp:68-86 over rows [y0, y1). */
static void step_rows(const double* in, const double* c, double* out, uint8_t* sel, int w,
                      int h, int wins[8][5], int y0, int y1) {
    for (int y = y0; y < y1; ++y) {
        for (int x = 0; x < w; ++x) {
            const double u = in[(size_t)y * w + x];
            double best = 0.0;
            double best_abs = INFINITY;
            int best_id = 0;
            for (int i = 0; i < 8; ++i) {
                double a;
                /* every window contains (x,y) so the mean never throws */
                oracle_rect_mean(c, w, h, x + wins[i][1], y + wins[i][3], x + wins[i][2],
                                 y + wins[i][4], &a);
                const double d = fabs(a - u);
                if (d < best_abs) {
                    best_abs = d;
                    best = a;
                    best_id = i + 1;
                }
            }
            out[(size_t)y * w + x] = best;
            if (sel) sel[(size_t)y * w + x] = (uint8_t)best_id;
        }
    }
}

int oracle_osbf_step(const double* in, double* out, int w, int h, int r, uint8_t* sel) {
    /* filters2d.hpp:61-88 */
    int wins[8][5];
    if (oracle_sub_windows(r, wins)) return ORACLE_ERR_INVALID_ARGUMENT;
    if (w < 1 || h < 1) return ORACLE_ERR_INVALID_ARGUMENT;
    double* c = (double*)malloc(sizeof(double) * ((size_t)w + 1) * ((size_t)h + 1));
    if (!c) return ORACLE_ERR_INVALID_ARGUMENT;
    oracle_sat_build(in, w, h, c);
    step_rows(in, c, out, sel, w, h, wins, 0, h);
    free(c);
    return ORACLE_OK;
}

typedef struct {
    const double* in;
    const double* c;
    double* out;
    int w, h, y0, y1;
    int (*wins)[5];
} rows_job;

static void* rows_worker(void* p) {
    rows_job* j = (rows_job*)p;
    step_rows(j->in, j->c, j->out, NULL, j->w, j->h, j->wins, j->y0, j->y1);
    return NULL;
}

static int osbf_impl(const double* in, double* out, int w, int h, int r, int iterations,
                     int threads) {
    /* filters2d.hpp:91-98 — iterations==0 is a copy and does not validate r. */
    if (iterations < 0) return ORACLE_ERR_INVALID_ARGUMENT;
    if (w < 1 || h < 1) return ORACLE_ERR_INVALID_ARGUMENT;
    const size_t n = (size_t)w * h;
    if (iterations == 0) {
        memmove(out, in, sizeof(double) * n);
        return ORACLE_OK;
    }
    int wins[8][5];
    if (oracle_sub_windows(r, wins)) return ORACLE_ERR_INVALID_ARGUMENT;
    double* cur = (double*)malloc(sizeof(double) * n);
    double* nxt = (double*)malloc(sizeof(double) * n);
    double* c = (double*)malloc(sizeof(double) * ((size_t)w + 1) * ((size_t)h + 1));
    if (!cur || !nxt || !c) {
        free(cur); free(nxt); free(c);
        return ORACLE_ERR_INVALID_ARGUMENT;
    }
    memcpy(cur, in, sizeof(double) * n);
    if (threads < 1) threads = 1;
    if (threads > h) threads = h;
    pthread_t* tids = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    rows_job* jobs = (rows_job*)malloc(sizeof(rows_job) * (size_t)threads);
    for (int it = 0; it < iterations; ++it) {
        oracle_sat_build(cur, w, h, c);
        if (threads == 1) {
            step_rows(cur, c, nxt, NULL, w, h, wins, 0, h);
        } else {
            const int chunk = (h + threads - 1) / threads;
            int started = 0;
            for (int t = 0; t < threads; ++t) {
                const int y0 = t * chunk, y1 = imin(h, y0 + chunk);
                if (y0 >= y1) break;
                jobs[t] = (rows_job){cur, c, nxt, w, h, y0, y1, wins};
                pthread_create(&tids[t], NULL, rows_worker, &jobs[t]);
                ++started;
            }
            for (int t = 0; t < started; ++t) pthread_join(tids[t], NULL);
        }
        double* tmp = cur;
        cur = nxt;
        nxt = tmp;
    }
    memcpy(out, cur, sizeof(double) * n);
    free(tids); free(jobs);
    free(cur); free(nxt); free(c);
    return ORACLE_OK;
}

int oracle_osbf(const double* in, double* out, int w, int h, int r, int iterations) {
    return osbf_impl(in, out, w, h, r, iterations, 1);
}

int oracle_osbf_mt(const double* in, double* out, int w, int h, int r, int iterations,
                   int threads) {
    return osbf_impl(in, out, w, h, r, iterations, threads);
}

/* filters2d.hpp:105-154.  Same operation order as the reference: the
 * quarter mean is rect_mean (integral.hpp:64-69: ((A-B)-C)+D, then one IEEE
 * division by the clipped count); the half candidates are 0.5 * (a + b) in
 * the listed order; selection is the strict-< first minimum of |c - u|. */
int oracle_fast_osbf(const double* in, double* out, int w, int h, int r, int iterations) {
    if (r < 1) return ORACLE_ERR_INVALID_ARGUMENT;          /* :107-108 */
    if (iterations < 0) return ORACLE_ERR_INVALID_ARGUMENT; /* :109-110 */
    if (w < 1 || h < 1) return ORACLE_ERR_INVALID_ARGUMENT;
    const size_t n = (size_t)w * h;
    double* cur = (double*)malloc(sizeof(double) * n);
    double* nxt = (double*)malloc(sizeof(double) * n);
    double* q = (double*)malloc(sizeof(double) * n);
    double* c = (double*)malloc(sizeof(double) * ((size_t)w + 1) * ((size_t)h + 1));
    if (!cur || !nxt || !q || !c) {
        free(cur); free(nxt); free(q); free(c);
        return ORACLE_ERR_INVALID_ARGUMENT;
    }
    memcpy(cur, in, sizeof(double) * n);
    for (int it = 0; it < iterations; ++it) {
        oracle_sat_build(cur, w, h, c);
        for (int y = 0; y < h; ++y)          /* :116-119 */
            for (int x = 0; x < w; ++x)
                oracle_rect_mean(c, w, h, x - r, y - r, x, y, &q[(size_t)y * w + x]);
        for (int y = 0; y < h; ++y) {        /* :121-147 */
            const int yr = imin(y + r, h - 1);
            for (int x = 0; x < w; ++x) {
                const int xr = imin(x + r, w - 1);
                const double q00 = q[(size_t)y * w + x], q10 = q[(size_t)y * w + xr];
                const double q01 = q[(size_t)yr * w + x], q11 = q[(size_t)yr * w + xr];
                const double cand[8] = {q00, q10, q01, q11, 0.5 * (q00 + q01), 0.5 * (q10 + q11),
                                        0.5 * (q00 + q10), 0.5 * (q01 + q11)};
                const double u = cur[(size_t)y * w + x];
                double best = cand[0], best_abs = fabs(cand[0] - u);
                for (int i = 1; i < 8; ++i) {
                    const double d = fabs(cand[i] - u);
                    if (d < best_abs) {
                        best_abs = d;
                        best = cand[i];
                    }
                }
                nxt[(size_t)y * w + x] = best;
            }
        }
        double* t = cur;
        cur = nxt;
        nxt = t;
    }
    memcpy(out, cur, sizeof(double) * n);
    free(cur); free(nxt); free(q); free(c);
    return ORACLE_OK;
}

/* filters2d.hpp:38-56 (box_filter): rect_mean (integral.hpp:64-69) of the
 * clipped window [x-r, x+r] x [y-r, y+r], iterated. */
int oracle_box_filter(const double* in, double* out, int w, int h, int r, int iterations) {
    if (r < 1) return ORACLE_ERR_INVALID_ARGUMENT;          /* :39-40 */
    if (iterations < 0) return ORACLE_ERR_INVALID_ARGUMENT; /* :41-42 */
    if (w < 1 || h < 1) return ORACLE_ERR_INVALID_ARGUMENT;
    const size_t n = (size_t)w * h;
    double* cur = (double*)malloc(sizeof(double) * n);
    double* nxt = (double*)malloc(sizeof(double) * n);
    double* c = (double*)malloc(sizeof(double) * ((size_t)w + 1) * ((size_t)h + 1));
    if (!cur || !nxt || !c) {
        free(cur); free(nxt); free(c);
        return ORACLE_ERR_INVALID_ARGUMENT;
    }
    memcpy(cur, in, sizeof(double) * n);
    for (int it = 0; it < iterations; ++it) {
        oracle_sat_build(cur, w, h, c);
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x)
                oracle_rect_mean(c, w, h, x - r, y - r, x + r, y + r, &nxt[(size_t)y * w + x]);
        double* t = cur;
        cur = nxt;
        nxt = t;
    }
    memcpy(out, cur, sizeof(double) * n);
    free(cur); free(nxt); free(c);
    return ORACLE_OK;
}

/* ---- 3-D extension -------------------------------------------------------- */

void oracle_svt_build(const double* vol, int w, int h, int d, double* c) {
    const size_t W1 = (size_t)w + 1, H1 = (size_t)h + 1;
    memset(c, 0, sizeof(double) * W1 * H1 * ((size_t)d + 1));
#define T3(x, y, z) c[((size_t)(z) * H1 + (size_t)(y)) * W1 + (size_t)(x)]
    for (int z = 0; z < d; ++z)
        for (int y = 0; y < h; ++y) {
            double row = 0.0;
            for (int x = 0; x < w; ++x) {
                row += vol[((size_t)z * h + y) * w + x];
                /* integral.hpp:107-108, evaluated left to right */
                T3(x + 1, y + 1, z + 1) =
                    row + T3(x + 1, y, z + 1) + T3(x + 1, y + 1, z) - T3(x + 1, y, z);
            }
        }
}

/* integral.hpp:121-160 (box_sum / box_count / box_mean); 0 count -> 0.0 */
static double box_mean3(const double* c, int w, int h, int d, int x0, int y0, int z0, int x1,
                        int y1, int z1, int* empty) {
    const size_t W1 = (size_t)w + 1, H1 = (size_t)h + 1;
    x0 = imax(x0, 0); y0 = imax(y0, 0); z0 = imax(z0, 0);
    x1 = imin(x1, w - 1); y1 = imin(y1, h - 1); z1 = imin(z1, d - 1);
    if (x0 > x1 || y0 > y1 || z0 > z1) {
        *empty = 1;
        return 0.0;
    }
    const int ax = x0, bx = x1 + 1, ay = y0, by = y1 + 1, az = z0, bz = z1 + 1;
    const double s = T3(bx, by, bz) - T3(ax, by, bz) - T3(bx, ay, bz) - T3(bx, by, az) +
                     T3(ax, ay, bz) + T3(ax, by, az) + T3(bx, ay, az) - T3(ax, ay, az);
    const long long n = (long long)(x1 - x0 + 1) * (y1 - y0 + 1) * (z1 - z0 + 1);
    return s / (double)n;
}
#undef T3

static void regions3(int r, int reg[14][6]) {
    /* filters3d.hpp:29-51: octants by sign pattern, then -x,+x,-y,+y,-z,+z */
    int id = 0;
    for (int sz = 0; sz < 2; ++sz)
        for (int sy = 0; sy < 2; ++sy)
            for (int sx = 0; sx < 2; ++sx) {
                int* g = reg[id++];
                g[0] = sx ? 0 : -r; g[1] = sx ? r : 0;
                g[2] = sy ? 0 : -r; g[3] = sy ? r : 0;
                g[4] = sz ? 0 : -r; g[5] = sz ? r : 0;
            }
    const int half[6][6] = {{-r, 0, -r, r, -r, r}, {0, r, -r, r, -r, r}, {-r, r, -r, 0, -r, r},
                            {-r, r, 0, r, -r, r},  {-r, r, -r, r, -r, 0}, {-r, r, -r, r, 0, r}};
    for (int i = 0; i < 6; ++i)
        for (int k = 0; k < 6; ++k) reg[8 + i][k] = half[i][k];
}

static int filter3(const double* in, double* out, int w, int h, int d, int r, int iters,
                   int osbf) {
    if (r < 1 || iters < 0 || w < 1 || h < 1 || d < 1) return ORACLE_ERR_INVALID_ARGUMENT;
    const size_t n = (size_t)w * h * d;
    double* cur = (double*)malloc(sizeof(double) * n);
    double* nxt = (double*)malloc(sizeof(double) * n);
    double* c = (double*)malloc(sizeof(double) * ((size_t)w + 1) * ((size_t)h + 1) * ((size_t)d + 1));
    if (!cur || !nxt || !c) {
        free(cur); free(nxt); free(c);
        return ORACLE_ERR_INVALID_ARGUMENT;
    }
    int reg[14][6];
    regions3(r, reg);
    memcpy(cur, in, sizeof(double) * n);
    for (int it = 0; it < iters; ++it) {
        oracle_svt_build(cur, w, h, d, c);
        for (int z = 0; z < d; ++z)
            for (int y = 0; y < h; ++y)
                for (int x = 0; x < w; ++x) {
                    const size_t i = ((size_t)z * h + y) * w + x;
                    int empty = 0;
                    if (!osbf) {
                        nxt[i] = box_mean3(c, w, h, d, x - r, y - r, z - r, x + r, y + r, z + r,
                                           &empty);
                        continue;
                    }
                    const double u = cur[i];
                    double best = 0.0, best_abs = INFINITY;
                    for (int k = 0; k < 14; ++k) {
                        const double a = box_mean3(c, w, h, d, x + reg[k][0], y + reg[k][2],
                                                   z + reg[k][4], x + reg[k][1], y + reg[k][3],
                                                   z + reg[k][5], &empty);
                        const double dist = fabs(a - u);
                        if (dist < best_abs) {
                            best_abs = dist;
                            best = a;
                        }
                    }
                    nxt[i] = best;
                }
        double* t = cur;
        cur = nxt;
        nxt = t;
    }
    memcpy(out, cur, sizeof(double) * n);
    free(cur); free(nxt); free(c);
    return ORACLE_OK;
}

int oracle_box_filter_3d(const double* in, double* out, int w, int h, int d, int r, int iters) {
    return filter3(in, out, w, h, d, r, iters, 0);
}

int oracle_osbf_3d(const double* in, double* out, int w, int h, int d, int r, int iters) {
    return filter3(in, out, w, h, d, r, iters, 1);
}

/* io.hpp:108-115 */
int oracle_quantize(double v, int maxval) {
    const double q = floor(v + 0.5);
    if (!(q > 0.0)) return 0;
    if (q > maxval) return maxval;
    return (int)q;
}

/* tools/osbf_main.cpp:63-83 without the file I/O: read_image's promotion
 * (io.hpp:157-168), FilterConfig::validate, filter_multichannel per channel,
 * write_image's quantise + interleave (io.hpp:202-212). */
int oracle_smooth_raster(const void* raster, int sample_bytes, int channels, int w, int h,
                         int filter, int r, int iterations, void* out, int out_sample_bytes) {
    if (r < 1 || iterations < 0 || (channels != 1 && channels != 3) || w < 1 || h < 1) return 1;
    if ((sample_bytes != 1 && sample_bytes != 2) || (out_sample_bytes != 1 && out_sample_bytes != 2))
        return 1;
    if (filter < 0 || filter > 2) return 1;
    const size_t n = (size_t)w * h;
    double* plane = (double*)malloc(n * sizeof(double));
    double* res = (double*)malloc(n * sizeof(double));
    if (!plane || !res) {
        free(plane);
        free(res);
        return 2;
    }
    const int maxval = out_sample_bytes == 1 ? 255 : 65535;
    int st = 0;
    for (int c = 0; c < channels && !st; ++c) {
        for (size_t i = 0; i < n; ++i)
            plane[i] = sample_bytes == 1 ? (double)((const uint8_t*)raster)[i * channels + c]
                                         : (double)((const uint16_t*)raster)[i * channels + c];
        st = filter == 1   ? oracle_fast_osbf(plane, res, w, h, r, iterations)
             : filter == 2 ? oracle_box_filter(plane, res, w, h, r, iterations)
                           : oracle_osbf(plane, res, w, h, r, iterations);
        for (size_t i = 0; i < n && !st; ++i) {
            const int q = oracle_quantize(res[i], maxval);
            if (out_sample_bytes == 1)
                ((uint8_t*)out)[i * channels + c] = (uint8_t)q;
            else
                ((uint16_t*)out)[i * channels + c] = (uint16_t)q;
        }
    }
    free(plane);
    free(res);
    return st;
}
