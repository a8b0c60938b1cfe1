// Exact mode: bit-identical replay of the reference OSBF pass.
//
// The reference (integral.hpp:16-30) builds ONE whole-image fp64 summed-area
// table with a serial left-to-right running row sum, adding the table row
// above:  C(x+1,y+1) = C(x+1,y) + R(x,y),  R(x,y) = R(x-1,y) + U(x,y).
// Every later rounding depends on that order, and the selection's strict-<
// tie-break (filters2d.hpp:72-82) decides exact ties through that rounding
// noise, so this mode reproduces the order exactly:
//   K1 exact_row_prefix : R, one serial fp64 chain per row (H*B chains),
//                         coalesced through a per-warp shared-memory transpose;
//   K2 exact_col_chain  : C, one serial fp64 chain per table column;
//   K3 exact_stencil    : per pixel, 8 clipped ((A-B)-C)+D sums
//                         (integral.hpp:48-49), IEEE division by the valid
//                         count (integral.hpp:68), |a-u|, strict < in window
//                         order, write a_m itself (filters2d.hpp:80-83).
// All fp64 arithmetic uses the _rn intrinsics so nothing is contracted.
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <utility>

#include "osbf_exact2_kernel.cuh"
#include "osbf_exact_gwalk.cuh"
#include "osbf_internal.cuh"

namespace osbf_gpu {
namespace {

constexpr int kRowWarps = 4;   // warps per CTA in K1
constexpr int kChunk = 32;     // columns per transpose chunk

template <typename T>
__global__ void __launch_bounds__(kRowWarps * 32)
    exact_row_prefix(const T* __restrict__ in, size_t in_pitch, size_t in_plane,
                     double* __restrict__ rowpfx, int W, int H, long long total_rows,
                     unsigned* __restrict__ reset_flag) {
    __shared__ double tile[kRowWarps][kChunk][kChunk + 1];
    // the table flag of this pass starts clear (the column chains that may
    // raise it run after this kernel, in stream order)
    if (reset_flag && blockIdx.x == 0 && threadIdx.x == 0) *reset_flag = 0u;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const long long row0 = (static_cast<long long>(blockIdx.x) * kRowWarps + warp) * 32;
    if (row0 >= total_rows) return;
    double (*t)[kChunk + 1] = tile[warp];

    // Element offset of row (row0 + lane); broadcast per row inside the loads.
    long long my_base = -1;
    {
        const long long g = row0 + lane;
        if (g < total_rows) {
            const long long b = g / H, y = g - b * H;
            my_base = b * static_cast<long long>(in_plane) + y * static_cast<long long>(in_pitch);
        }
    }
    double acc = 0.0;
    for (int x0 = 0; x0 < W; x0 += kChunk) {
        const int x = x0 + lane;
#pragma unroll 8
        for (int rr = 0; rr < 32; ++rr) {
            const long long base = __shfl_sync(0xffffffffu, my_base, rr);
            double v = 0.0;
            if (base >= 0 && x < W) v = to_f64(in[base + x]);
            t[rr][lane] = v;
        }
        __syncwarp();
        const int n = min(kChunk, W - x0);
        for (int c = 0; c < n; ++c) {
            acc = __dadd_rn(acc, t[lane][c]);  // row += src[x]  (integral.hpp:25)
            t[lane][c] = acc;
        }
        __syncwarp();
#pragma unroll 8
        for (int rr = 0; rr < 32; ++rr) {
            const long long g = row0 + rr;
            if (g < total_rows && x < W) rowpfx[g * W + x] = t[rr][lane];
        }
        __syncwarp();
    }
}

// Table flag: raised by a column chain that produced a table value outside
// the range where the 3-operation division is exact (table_value_safe); the
// stencil then keeps the guarded division.  Set and read in stream order
// (chain kernel, then stencil kernel).  A caller that owns the table passes
// its own flag word (cleared by the row-prefix kernel of every pass, so one
// non-finite image does not slow later ones down); callers without one share
// this sticky per-device word, which is never cleared.
__device__ unsigned g_table_unsafe = 0u;

__device__ __forceinline__ void flag_unsafe(unsigned* flag, bool unsafe) {
    if (__any_sync(__activemask(), unsafe) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

// One thread per table column cx in [0, W] of each plane.
__global__ void exact_col_chain(const double* __restrict__ rowpfx, double* __restrict__ sat,
                                int W, int H, int B, long long tp, unsigned* __restrict__ flag) {
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long cols = static_cast<long long>(W) + 1;
    if (t >= cols * B) return;
    const long long b = t / cols;
    const int cx = static_cast<int>(t - b * cols);
    double* C = sat + b * tp * (H + 1);
    C[cx] = 0.0;  // zero border row
    if (cx == 0) {
        for (int cy = 1; cy <= H; ++cy) C[static_cast<long long>(cy) * tp] = 0.0;
        return;
    }
    const double* R = rowpfx + b * static_cast<long long>(W) * H + (cx - 1);
    double acc = 0.0;
    bool unsafe = false;
#pragma unroll 8
    for (int y = 0; y < H; ++y) {
        acc = __dadd_rn(acc, R[static_cast<long long>(y) * W]);  // above[x+1] + row (integral.hpp:26)
        unsafe |= !table_value_safe(acc);
        C[static_cast<long long>(y + 1) * tp + cx] = acc;
    }
    if (unsafe) atomicOr(flag, 1u);
}

// ---- deep-prefetch table builders (few planes) -------------------------------
// The two serial recurrences have only H (rows) and W+1 (columns) independent
// chains per plane, so a single 4096^2 plane gives ~130 warps: the kernels
// above then wait a full memory latency every few elements.  These keep
// ROW_STAGES / COL_STAGES chunks of loads in flight per warp (cp.async ring
// through shared memory); the adds are the same serial chains, in the same
// order, so the table is bit-identical.
constexpr int ROW_STAGES = 8;   // 32x32 chunks in flight per row warp
constexpr int COL_ROWS = 16;    // rows per column-chain stage
constexpr int COL_STAGES = 12;  // stages in flight per column warp
constexpr size_t ROW2_SMEM = sizeof(double) * ROW_STAGES * 32 * 33;
constexpr size_t COL2_SMEM = sizeof(double) * COL_STAGES * COL_ROWS * 32;

__device__ __forceinline__ void cpa8(double* dst, const double* src, bool valid) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src),
                 "r"(valid ? 8 : 0));
}

__device__ __forceinline__ void mb_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(static_cast<unsigned>(
                     __cvta_generic_to_shared(bar))), "r"(count));
}
__device__ __forceinline__ void mb_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(static_cast<unsigned>(
                     __cvta_generic_to_shared(bar))) : "memory");
}
// arrive once this thread's earlier cp.async copies have landed
__device__ __forceinline__ void mb_arrive_cpasync(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(static_cast<unsigned>(
                     __cvta_generic_to_shared(bar))) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra W_%=;\n}\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(bar))),
        "r"(parity)
        : "memory");
}

// R(x, y) for 32 rows per CTA, as a three-warp pipeline over 32x32 chunks
// (one padded 32x33 transpose tile per ring stage):
//   warp 0 loads chunk c (lanes = columns, cp.async, coalesced),
//   warp 1 runs the 32 serial row chains over it in place (lanes = rows;
//          row += src[x], integral.hpp:25),
//   warp 2 stores it back row-major (lanes = columns, coalesced).
// The chain warp issues only load / add / store per element, so the serial
// recurrence (4096 dependent adds per row on a 4096^2 plane) is no longer
// buried under the copy instructions of a single warp.
template <typename T>
__global__ void __launch_bounds__(96)
    exact_row_prefix_deep(const T* __restrict__ in, size_t in_pitch, size_t in_plane,
                          double* __restrict__ rowpfx, int W, int H, long long total_rows,
                          unsigned* __restrict__ reset_flag) {
    extern __shared__ double ring[];
    __shared__ uint64_t full[ROW_STAGES], done[ROW_STAGES], empty[ROW_STAGES];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long row0 = static_cast<long long>(blockIdx.x) * 32;
    if (reset_flag && blockIdx.x == 0 && threadIdx.x == 0) *reset_flag = 0u;
    if (threadIdx.x == 0)
        for (int q = 0; q < ROW_STAGES; ++q) {
            mb_init(&full[q], 32);
            mb_init(&done[q], 32);
            mb_init(&empty[q], 32);
        }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    __syncthreads();
    const int nchunks = (W + 31) / 32;
    if (warp == 0) {
        long long my_base = -1;
        const long long g = row0 + lane;
        if (g < total_rows) {
            const long long b = g / H, y = g - b * H;
            my_base = b * static_cast<long long>(in_plane) + y * static_cast<long long>(in_pitch);
        }
        for (int c = 0; c < nchunks; ++c) {
            const int q = c % ROW_STAGES;
            if (c >= ROW_STAGES) mb_wait(&empty[q], ((c / ROW_STAGES) - 1) & 1);
            double* t = ring + q * 32 * 33;
            const int x = 32 * c + lane;
#pragma unroll 8
            for (int rr = 0; rr < 32; ++rr) {
                const long long base = __shfl_sync(0xffffffffu, my_base, rr);
                const bool ok = base >= 0 && x < W;
                if constexpr (sizeof(T) == 8) {
                    cpa8(t + lane * 33 + rr,
                         reinterpret_cast<const double*>(in) + (ok ? base + x : 0), ok);
                } else {
                    t[lane * 33 + rr] = ok ? to_f64(in[base + x]) : 0.0;
                }
            }
            if constexpr (sizeof(T) == 8) mb_arrive_cpasync(&full[q]);
            else mb_arrive(&full[q]);
        }
    } else if (warp == 1) {
        double acc = 0.0;
        for (int c = 0; c < nchunks; ++c) {
            const int q = c % ROW_STAGES;
            mb_wait(&full[q], (c / ROW_STAGES) & 1);
            double* t = ring + q * 32 * 33;
            const int n = min(32, W - 32 * c);
            double v[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) v[k] = t[k * 33 + lane];
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                if (k < n) {
                    acc = __dadd_rn(acc, v[k]);
                    t[k * 33 + lane] = acc;
                }
            }
            mb_arrive(&done[q]);
        }
    } else {
        for (int c = 0; c < nchunks; ++c) {
            const int q = c % ROW_STAGES;
            mb_wait(&done[q], (c / ROW_STAGES) & 1);
            const double* t = ring + q * 32 * 33;
            const int x = 32 * c + lane;
#pragma unroll 8
            for (int rr = 0; rr < 32; ++rr) {
                const long long g = row0 + rr;
                if (g < total_rows && x < W) rowpfx[g * W + x] = t[lane * 33 + rr];
            }
            mb_arrive(&empty[q]);
        }
    }
}

// C(cx, y+1) = C(cx, y) + R(cx-1, y) for 32 table columns per CTA, as a
// three-warp pipeline over COL_ROWS-row stages: warp 0 streams the R rows in
// (cp.async), warp 1 runs the 32 serial column chains (above[x+1] + row,
// integral.hpp:26) in place, warp 2 stores the table rows (coalesced) and
// flags values outside the exact division's range.  The chain warp issues
// only load / add / store per element.
__global__ void __launch_bounds__(96)
    exact_col_chain_deep(const double* __restrict__ rowpfx, double* __restrict__ sat, int W,
                         int H, int B, long long tp, unsigned* __restrict__ flag) {
    extern __shared__ double cring[];
    __shared__ uint64_t full[COL_STAGES], done[COL_STAGES], empty[COL_STAGES];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long cols = static_cast<long long>(W) + 1;
    const int wpp = static_cast<int>((cols + 31) / 32);  // CTAs per plane
    const int b = blockIdx.x / wpp;
    const int cx = (blockIdx.x - b * wpp) * 32 + lane;
    if (threadIdx.x == 0)
        for (int q = 0; q < COL_STAGES; ++q) {
            mb_init(&full[q], 32);
            mb_init(&done[q], 32);
            mb_init(&empty[q], 32);
        }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    __syncthreads();
    const bool live = cx >= 1 && cx <= W;
    const int nst = (H + COL_ROWS - 1) / COL_ROWS;
    if (warp == 0) {
        const double* R = rowpfx + static_cast<long long>(b) * W * H + (live ? cx - 1 : 0);
        for (int st = 0; st < nst; ++st) {
            const int q = st % COL_STAGES;
            if (st >= COL_STAGES) mb_wait(&empty[q], ((st / COL_STAGES) - 1) & 1);
            double* t = cring + q * COL_ROWS * 32;
            const double* rs = R + static_cast<long long>(st) * COL_ROWS * W;
#pragma unroll
            for (int k = 0; k < COL_ROWS; ++k) {
                const bool ok = live && st * COL_ROWS + k < H;
                cpa8(t + k * 32 + lane, ok ? rs + static_cast<long long>(k) * W : R, ok);
            }
            mb_arrive_cpasync(&full[q]);
        }
    } else if (warp == 1) {
        double acc = 0.0;
        for (int st = 0; st < nst; ++st) {
            const int q = st % COL_STAGES;
            mb_wait(&full[q], (st / COL_STAGES) & 1);
            double* t = cring + q * COL_ROWS * 32;
            double v[COL_ROWS];
#pragma unroll
            for (int k = 0; k < COL_ROWS; ++k) v[k] = t[k * 32 + lane];
            // rows past H are zero-filled and never stored
#pragma unroll
            for (int k = 0; k < COL_ROWS; ++k) {
                acc = __dadd_rn(acc, v[k]);
                t[k * 32 + lane] = acc;
            }
            mb_arrive(&done[q]);
        }
    } else {
        double* C = sat + static_cast<long long>(b) * tp * (H + 1);
        if (cx <= W) C[cx] = 0.0;  // zero border row
        bool unsafe = false;
        double* cp = C + tp + cx;  // table row 1
        for (int st = 0; st < nst; ++st) {
            const int q = st % COL_STAGES;
            mb_wait(&done[q], (st / COL_STAGES) & 1);
            const double* t = cring + q * COL_ROWS * 32;
            double v[COL_ROWS];
#pragma unroll
            for (int k = 0; k < COL_ROWS; ++k) v[k] = t[k * 32 + lane];
            mb_arrive(&empty[q]);
            const int nk = min(COL_ROWS, H - st * COL_ROWS);
            if (cx <= W) {
                if (nk == COL_ROWS) {  // full stage: straight-line stores
#pragma unroll
                    for (int k = 0; k < COL_ROWS; ++k) {
                        unsafe |= !table_value_safe(v[k]);
                        *cp = v[k];
                        cp += tp;
                    }
                } else {
                    for (int k = 0; k < nk; ++k) {
                        unsafe |= !table_value_safe(v[k]);
                        *cp = v[k];
                        cp += tp;
                    }
                }
            }
        }
        flag_unsafe(flag, unsafe);
    }
}

// ---- strip table builder ------------------------------------------------------
// The table straight from the input, without the row-prefix plane: the row
// carries R(16s-1, y) come from exact_row_carries (osbf_exact2_kernel.cuh, K1
// of the fused path), then one CTA per 32-column strip of a plane walks down
// it in 32 x 32 tiles as a four-warp pipeline on mbarriers over a ring of
// padded 32 x 33 transpose tiles:
//   warp 0 loads tile t of U (lanes = columns, coalesced),
//   warp 1 continues the 32 row chains from their carries, in place
//          (lanes = rows; row += src[x], integral.hpp:25),
//   warp 2 continues the 32 column chains down the tile, in place
//          (lanes = columns; above[x+1] + row, integral.hpp:26),
//   warp 3 stores the table rows (coalesced) and flags unsafe values.
// Same serial adds in the same order as exact_row_prefix + exact_col_chain:
// the table is bit-identical, and the row-prefix plane's write and re-read
// (half the build's HBM traffic) is gone.
constexpr int TS_STAGES = 6;        // many CTAs per SM
constexpr int TS_STAGES_DEEP = 16;  // about one CTA per SM: hide the full HBM latency
constexpr int TS_LOADERS = 4;  // loader warps (8 tile rows each)
constexpr int TS_STORERS = 4;  // storer warps (8 tile rows each)
constexpr int TS_THREADS = 32 * (TS_LOADERS + 2 + TS_STORERS);
constexpr int TS_TILE = 32 * 33 + 32;  // padded transpose tile + the 32 row carries of the tile

// One arrival per warp: the lanes' shared-memory accesses are ordered before
// it by the warp barrier (32 per-lane arrivals on one mbarrier word serialise).
__device__ __forceinline__ void mb_arrive_warp(uint64_t* bar, int lane) {
    __syncwarp();
    if (lane == 0) mb_arrive(bar);
}

// Rows rr0 .. rr0 + 7 of a 32 x 32 tile into a padded transpose tile
// (element (column lane, row rr) at tile[lane * 33 + rr]); src points at this
// lane's column in tile row 0, rows_left = valid rows from there, col_ok =
// the lane's column exists.  fp64 input goes through cp.async (arrival on
// `bar` when the copies land), narrower types through registers.
template <typename T>
__device__ __forceinline__ void load_tile_rows(double* tile, const T* src, size_t pitch, int rr0,
                                               int rows_left, bool col_ok, int lane,
                                               uint64_t* bar) {
    if constexpr (sizeof(T) == 8) {
#pragma unroll
        for (int j = 0; j < 32 / TS_LOADERS; ++j) {
            const int rr = rr0 + j;
            const bool ok = col_ok && rr < rows_left;
            cpa8(tile + lane * 33 + rr,
                 reinterpret_cast<const double*>(src) + (ok ? static_cast<size_t>(rr) * pitch : 0),
                 ok);
        }
        mb_arrive_cpasync(bar);
    } else {
        T v[32 / TS_LOADERS];
#pragma unroll
        for (int j = 0; j < 32 / TS_LOADERS; ++j) {
            const int rr = rr0 + j;
            const bool ok = col_ok && rr < rows_left;
            v[j] = ok ? src[static_cast<size_t>(rr) * pitch] : T(0);
        }
#pragma unroll
        for (int j = 0; j < 32 / TS_LOADERS; ++j) tile[lane * 33 + rr0 + j] = to_f64(v[j]);
        mb_arrive(bar);
    }
}

constexpr size_t ts_smem(int stages) { return sizeof(double) * static_cast<size_t>(stages) * TS_TILE; }

// A strip is the 32 TABLE columns cx = 32 j .. 32 j + 31 (so a bulk store of
// its tiles starts on a 16-byte boundary); table column cx holds the running
// row sums R(cx - 1, y): the strip's first column is the stored carry
// R(32 j - 1, y) itself (0 for j = 0: the table's zero column), the others
// continue it with U(32 j .. 32 j + 30).
// (A variant whose column-chain warp wrote dense tiles and stored them with
// cp.async.bulk.tensor measured slower, 338 vs 216 us on 64 x 1024^2: the
// extra shared stores and the issue of the bulk store serialise on the one
// chain warp; two storer warps write the rows instead.)
template <typename T, int NST>
__global__ void __launch_bounds__(TS_THREADS)
    exact_table_strip(const T* __restrict__ in, size_t in_pitch, size_t in_plane,
                      const double* __restrict__ carries, int nsc, double* __restrict__ sat,
                      long long tp, int W, int H, unsigned* __restrict__ flag) {
    extern __shared__ double tring[];
    __shared__ uint64_t full[NST], rdone[NST], cdone[NST], empty[NST];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int b = blockIdx.y;
    const int x0 = blockIdx.x * 32;
    if (threadIdx.x == 0)
        for (int q = 0; q < NST; ++q) {
            mb_init(&full[q], 32 * TS_LOADERS);
            mb_init(&rdone[q], 1);
            mb_init(&cdone[q], 1);
            mb_init(&empty[q], TS_STORERS);
        }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    __syncthreads();
    const int ntiles = (H + 31) / 32;
    const int x = x0 + lane;  // table column of this lane (column chains, stores)
    const int ux = x - 1;     // input column feeding it (lane 0: the carry, no input)
    const bool u_ok = ux >= 0 && ux < W && lane > 0;
    double* C = sat + static_cast<long long>(b) * tp * (H + 1);
    if (warp < TS_LOADERS) {
        const T* src = in + static_cast<size_t>(b) * in_plane + (u_ok ? ux : 0);
        // loader 0 also brings the tile's row carries R(x0 - 1, y), lane = row
        const double* crow = carries + static_cast<size_t>(b) * H * nsc + x0 / 16;
        if constexpr (sizeof(T) == 8) {
            for (int t = 0; t < ntiles; ++t) {
                const int q = t % NST;
                if (t >= NST) mb_wait(&empty[q], ((t / NST) - 1) & 1);
                double* tile = tring + q * TS_TILE;
                if (warp == 0) {
                    const int y = t * 32 + lane;
                    const bool ok = y < H;
                    cpa8(tile + 32 * 33 + lane, crow + (ok ? static_cast<size_t>(y) * nsc : 0), ok);
                }
                load_tile_rows<T>(tile, src + static_cast<size_t>(t) * 32 * in_pitch, in_pitch,
                                  warp * (32 / TS_LOADERS), H - t * 32, u_ok, lane, &full[q]);
            }
        } else {
            // uint8 / float32 input goes through registers: keep the loads of
            // PF tiles in flight per warp (a register ring), convert and store
            // a tile once its stage is free
            constexpr int RPL = 32 / TS_LOADERS, PF = 3;
            const int rr0 = warp * RPL;
            T buf[PF][RPL];
            double cbuf[PF];
            auto fetch = [&](T (&v)[RPL], double& c, int t) {
                const T* rs = src + static_cast<size_t>(t) * 32 * in_pitch;
#pragma unroll
                for (int j = 0; j < RPL; ++j) {
                    const bool ok = u_ok && t * 32 + rr0 + j < H;
                    v[j] = ok ? rs[static_cast<size_t>(rr0 + j) * in_pitch] : T(0);
                }
                const int y = t * 32 + lane;
                c = (warp == 0 && y < H) ? crow[static_cast<size_t>(y) * nsc] : 0.0;
            };
            auto put = [&](const T (&v)[RPL], double c, int t) {
                const int q = t % NST;
                if (t >= NST) mb_wait(&empty[q], ((t / NST) - 1) & 1);
                double* tile = tring + q * TS_TILE;
                if (warp == 0) tile[32 * 33 + lane] = c;
#pragma unroll
                for (int j = 0; j < RPL; ++j) tile[lane * 33 + rr0 + j] = to_f64(v[j]);
                mb_arrive(&full[q]);
            };
#pragma unroll
            for (int i = 0; i < PF; ++i)
                if (i < ntiles) fetch(buf[i], cbuf[i], i);
            for (int t0 = 0; t0 < ntiles; t0 += PF) {
#pragma unroll
                for (int i = 0; i < PF; ++i) {
                    const int t = t0 + i;
                    if (t < ntiles) {
                        put(buf[i], cbuf[i], t);
                        if (t + PF < ntiles) fetch(buf[i], cbuf[i], t + PF);
                    }
                }
            }
        }
    } else if (warp == TS_LOADERS) {
        // lane = row of the tile: column 0 is the carry R(x0 - 1, y), then the chain
        const int n = min(32, W + 1 - x0);  // table columns of this strip
        for (int t = 0; t < ntiles; ++t) {
            const int q = t % NST;
            mb_wait(&full[q], (t / NST) & 1);
            double* tile = tring + q * TS_TILE;
            double acc = tile[32 * 33 + lane];
            double v[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) v[k] = tile[k * 33 + lane];
            tile[lane] = acc;
            if (n == 32) {  // nothing but the adds on the dependent chain
#pragma unroll
                for (int k = 1; k < 32; ++k) {
                    acc = __dadd_rn(acc, v[k]);
                    tile[k * 33 + lane] = acc;
                }
            } else {  // last, partial strip
#pragma unroll
                for (int k = 1; k < 32; ++k) {
                    if (k < n) {
                        acc = __dadd_rn(acc, v[k]);
                        tile[k * 33 + lane] = acc;
                    }
                }
            }
            mb_arrive_warp(&rdone[q], lane);
        }
    } else if (warp == TS_LOADERS + 1) {
        double acc = 0.0;  // lane = table column x: C(x, y) so far
        // zero border row 0 of the table over this strip's columns
        if (x <= W) C[x] = 0.0;
        // the range check of every table value rides in the shadow of the
        // dependent adds (integer ops only; rows past H repeat the last value)
        bool unsafe = false;
        for (int t = 0; t < ntiles; ++t) {
            const int q = t % NST;
            mb_wait(&rdone[q], (t / NST) & 1);
            double* tile = tring + q * TS_TILE;
            double v[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) v[k] = tile[lane * 33 + k];
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                acc = __dadd_rn(acc, v[k]);
                tile[lane * 33 + k] = acc;
                unsafe |= !table_value_safe(acc);
            }
            mb_arrive_warp(&cdone[q], lane);
        }
        flag_unsafe(flag, unsafe && x <= W);
    } else {
        constexpr int RPS = 32 / TS_STORERS;  // tile rows per storer warp
        const int k0 = (warp - TS_LOADERS - 2) * RPS;
        for (int t = 0; t < ntiles; ++t) {
            const int q = t % NST;
            mb_wait(&cdone[q], (t / NST) & 1);
            const double* tile = tring + q * TS_TILE;
            double v[RPS];
#pragma unroll
            for (int k = 0; k < RPS; ++k) v[k] = tile[lane * 33 + k0 + k];
            mb_arrive_warp(&empty[q], lane);
            const int nk = H - t * 32 - k0;  // rows of this warp's part inside the table
            double* cp = C + static_cast<long long>(t * 32 + k0 + 1) * tp + x;
            if (x <= W) {
                if (nk >= RPS) {  // straight-line stores
#pragma unroll
                    for (int k = 0; k < RPS; ++k) cp[static_cast<long long>(k) * tp] = v[k];
                } else {
#pragma unroll
                    for (int k = 0; k < RPS; ++k)
                        if (k < nk) cp[static_cast<long long>(k) * tp] = v[k];
                }
            }
        }
    }
}

// The row carries R(16 s - 1, y) for few rows (about one chain warp per SM
// or fewer): CTA per 32 rows as loader warps + one chain warp over a ring of
// 32 x 32 chunks, so the serial chain (row += src[x], integral.hpp:25) is not
// slowed by the copy instructions.  Same values as ex2::exact_row_carries.
constexpr int RC_STAGES_DEEP = 16;  // about one CTA per SM
constexpr int RC_STAGES_MANY = 4;   // several CTAs per SM
constexpr size_t rc_smem(int stages) { return sizeof(double) * stages * 32 * 33; }

template <typename T, int RC_STAGES>
__global__ void __launch_bounds__(32 * (TS_LOADERS + 1))
    exact_row_carries_pipe(const T* __restrict__ in, size_t pitch, size_t plane,
                           double* __restrict__ carries, int W, int H, long long rows, int nsc) {
    extern __shared__ double cring[];
    __shared__ uint64_t full[RC_STAGES], empty[RC_STAGES];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long row0 = static_cast<long long>(blockIdx.x) * 32;
    if (threadIdx.x == 0)
        for (int q = 0; q < RC_STAGES; ++q) {
            mb_init(&full[q], 32 * TS_LOADERS);
            mb_init(&empty[q], 1);
        }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    __syncthreads();
    const int nchunks = (W + 31) / 32;
    if (warp < TS_LOADERS) {
        // element offsets of this warp's 8 rows (rows may straddle planes)
        constexpr int RPL = 32 / TS_LOADERS;
        long long base[RPL];
#pragma unroll
        for (int j = 0; j < RPL; ++j) {
            const long long g = row0 + warp * RPL + j;
            base[j] = -1;
            if (g < rows) {
                const long long b = g / H, y = g - b * H;
                base[j] = b * static_cast<long long>(plane) + y * static_cast<long long>(pitch);
            }
        }
        if constexpr (sizeof(T) == 8) {
            for (int c = 0; c < nchunks; ++c) {
                const int q = c % RC_STAGES;
                if (c >= RC_STAGES) mb_wait(&empty[q], ((c / RC_STAGES) - 1) & 1);
                double* t = cring + q * 32 * 33;
                const int x = 32 * c + lane;
#pragma unroll
                for (int j = 0; j < RPL; ++j) {
                    const bool ok = base[j] >= 0 && x < W;
                    cpa8(t + lane * 33 + warp * RPL + j,
                         reinterpret_cast<const double*>(in) + (ok ? base[j] + x : 0), ok);
                }
                mb_arrive_cpasync(&full[q]);
            }
        } else {
            // through registers: the loads of PF chunks stay in flight per warp
            constexpr int PF = 3;
            T buf[PF][RPL];
            auto fetch = [&](T (&v)[RPL], int c) {
                const int x = 32 * c + lane;
#pragma unroll
                for (int j = 0; j < RPL; ++j)
                    v[j] = (base[j] >= 0 && x < W) ? in[base[j] + x] : T(0);
            };
            auto put = [&](const T (&v)[RPL], int c) {
                const int q = c % RC_STAGES;
                if (c >= RC_STAGES) mb_wait(&empty[q], ((c / RC_STAGES) - 1) & 1);
                double* t = cring + q * 32 * 33;
#pragma unroll
                for (int j = 0; j < RPL; ++j) t[lane * 33 + warp * RPL + j] = to_f64(v[j]);
                mb_arrive(&full[q]);
            };
#pragma unroll
            for (int i = 0; i < PF; ++i)
                if (i < nchunks) fetch(buf[i], i);
            for (int c0 = 0; c0 < nchunks; c0 += PF) {
#pragma unroll
                for (int i = 0; i < PF; ++i) {
                    const int c = c0 + i;
                    if (c < nchunks) {
                        put(buf[i], c);
                        if (c + PF < nchunks) fetch(buf[i], c + PF);
                    }
                }
            }
        }
    } else {
        const long long g = row0 + lane;
        double* crow = carries + (g < rows ? g : 0) * nsc;
        if (g < rows) crow[0] = 0.0;
        double acc = 0.0;
        for (int c = 0; c < nchunks; ++c) {
            const int q = c % RC_STAGES;
            mb_wait(&full[q], (c / RC_STAGES) & 1);
            const double* t = cring + q * 32 * 33;
            double v[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) v[k] = t[k * 33 + lane];
            mb_arrive_warp(&empty[q], lane);
            const int n = min(32, W - 32 * c);
            if (n == 32) {  // nothing but the adds on the dependent chain
#pragma unroll
                for (int k = 0; k < 32; ++k) {
                    acc = __dadd_rn(acc, v[k]);
                    if ((k + 1) % ex2::SW == 0 && g < rows) crow[(32 * c + k + 1) / ex2::SW] = acc;
                }
            } else {
#pragma unroll
                for (int k = 0; k < 32; ++k) {
                    if (k < n) {
                        acc = __dadd_rn(acc, v[k]);
                        if ((k + 1) % ex2::SW == 0 && g < rows)
                            crow[(32 * c + k + 1) / ex2::SW] = acc;
                    }
                }
            }
        }
    }
}

// C / cols: the table of plane b (or a shared-memory copy of the part this
// pixel reads: C then points at the copy's virtual origin, cols is its pitch).
// RT > 0: the radius as a compile-time constant (corner offsets become
// immediates); ro1..ro3 = r, r+1, 2r+1 table rows, precomputed per thread.
template <typename T, int RT>
__device__ __forceinline__ void stencil_px(const T* __restrict__ in, size_t in_pitch,
                                           size_t in_plane, const double* C, long long cols,
                                           double* __restrict__ out, size_t out_pitch,
                                           size_t out_plane, double* __restrict__ means,
                                           uint8_t* __restrict__ sel, int W, int H, int r_rt,
                                           int x, int y, int b, bool safe, double yq, double yh,
                                           int ro1, int ro2, int ro3) {
    const int r = RT > 0 ? RT : r_rt;
    if (x >= W || y >= H) return;
    const double u = to_f64(in[b * in_plane + static_cast<size_t>(y) * in_pitch + x]);
    const bool diag = means != nullptr || sel != nullptr;
    if (!diag && x >= r && x + r < W && y >= r && y + r < H) {
        // interior pixel: the 8 windows share a 4x4 grid of table corners,
        // rows {y-r, y, y+1, y+r+1} x columns {x-r, x, x+1, x+r+1}; every sum
        // keeps the reference's ((A-B)-C)+D (integral.hpp:48-49) and the
        // division by the count is IEEE-exact (div_by_count)
        // one 64-bit base, then 32-bit row / column offsets (a table row of
        // W+1 doubles; (2r+1) rows of it fit an int for any plane we accept)
        const double* p0 = C + static_cast<long long>(y - r) * cols + (x - r);
        const int ro[4] = {0, ro1, ro2, ro3};
        const int co[4] = {0, r, r + 1, 2 * r + 1};
        double g[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const double* rp = p0 + ro[a];
#pragma unroll
            for (int c = 0; c < 4; ++c) g[a][c] = rp[co[c]];
        }
        // (ca, cb, ra, rb) per window in reference order (core.hpp:212-225)
        constexpr int W8[8][4] = {{0, 2, 1, 3}, {1, 3, 1, 3}, {1, 3, 0, 2}, {0, 2, 0, 2},
                                  {0, 2, 0, 3}, {1, 3, 0, 3}, {0, 3, 1, 3}, {0, 3, 0, 2}};
        const double nq = static_cast<double>((r + 1) * (r + 1));
        const double nh = static_cast<double>((r + 1) * (2 * r + 1));
        double av[8], dv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int ca = W8[i][0], cb = W8[i][1], ra = W8[i][2], rb = W8[i][3];
            const double sm =
                __dadd_rn(__dsub_rn(__dsub_rn(g[rb][cb], g[rb][ca]), g[ra][cb]), g[ra][ca]);
            // every table value in the exact division's range (no chain set
            // the sticky flag): the unguarded 3-operation division is exact
            av[i] = safe ? div_by_count_unguarded(sm, i < 4 ? nq : nh, i < 4 ? yq : yh)
                         : div_by_count(sm, i < 4 ? nq : nh, i < 4 ? yq : yh);
            dv[i] = fabs(__dsub_rn(av[i], u));
        }
        double best = 0.0;
        // a safe table (finite, in range) gives finite d_i; otherwise check
        bool finite = safe;
        if (!safe) {
            const double dsum =
                ((dv[0] + dv[1]) + (dv[2] + dv[3])) + ((dv[4] + dv[5]) + (dv[6] + dv[7]));
            finite = fabs(dsum) < __longlong_as_double(0x7ff0000000000000LL);
        }
        if (finite) {
            // all |a_i - u| finite: a stable depth-3 tournament returns the
            // first minimum, the reference's strict < (filters2d.hpp:78)
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
        } else {  // non-finite samples: the sequential rule never selects them
            double best_abs = __longlong_as_double(0x7ff0000000000000LL);
#pragma unroll
            for (int i = 0; i < 8; ++i)
                if (dv[i] < best_abs) {
                    best_abs = dv[i];
                    best = av[i];
                }
        }
        out[b * out_plane + static_cast<size_t>(y) * out_pitch + x] = best;
        return;
    }
    double best = 0.0;
    double best_abs = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    int best_id = 0;
    const size_t pix = (static_cast<size_t>(b) * H + y) * W + x;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const Win w = window(i, r);
        const int x0 = max(x + w.u0, 0), x1 = min(x + w.u1, W - 1);
        const int y0 = max(y + w.v0, 0), y1 = min(y + w.v1, H - 1);
        const long long n = static_cast<long long>(x1 - x0 + 1) * (y1 - y0 + 1);
        const double A = C[(y1 + 1) * cols + (x1 + 1)];
        const double Bv = C[(y1 + 1) * cols + x0];
        const double Cv = C[y0 * cols + (x1 + 1)];
        const double D = C[y0 * cols + x0];
        const double s = __dadd_rn(__dsub_rn(__dsub_rn(A, Bv), Cv), D);
        const double a = __ddiv_rn(s, static_cast<double>(n));
        if (means) means[pix * 8 + i] = a;
        const double d = fabs(__dsub_rn(a, u));
        if (d < best_abs) {
            best_abs = d;
            best = a;
            best_id = i + 1;
        }
    }
    if (out) out[b * out_plane + static_cast<size_t>(y) * out_pitch + x] = best;
    if (sel) sel[pix] = static_cast<uint8_t>(best_id);
}

// The shared sticky flag word (callers that pass no flag of their own).
unsigned* table_flag_address() {
    // the symbol lives on every device: one address per device ordinal
    static std::atomic<unsigned*> cache[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    std::atomic<unsigned*>& slot = cache[dev & 63];
    if (unsigned* p = slot.load(std::memory_order_acquire)) return p;
    void* p = nullptr;
    if (cudaGetSymbolAddress(&p, g_table_unsafe) != cudaSuccess) return nullptr;
    slot.store(static_cast<unsigned*>(p), std::memory_order_release);
    return static_cast<unsigned*>(p);
}

constexpr int kStencilRows = 4;  // rows per thread (block: 32 x 8 threads, 32 x 32 pixels)

template <typename T, int RT>
__global__ void __launch_bounds__(256)
    exact_stencil(const T* __restrict__ in, size_t in_pitch, size_t in_plane,
                  const double* __restrict__ sat, double* __restrict__ out, size_t out_pitch,
                  size_t out_plane, double* __restrict__ means, uint8_t* __restrict__ sel, int W,
                  int H, int r_rt, double yq, double yh, long long cols,
                  const unsigned* __restrict__ flag) {
    const int r = RT > 0 ? RT : r_rt;
    const int x = blockIdx.x * 32 + (threadIdx.x & 31);
    const int b = blockIdx.z;
    const bool safe = *flag == 0u;
    const double* C = sat + static_cast<long long>(b) * cols * (H + 1);
    const int ic = static_cast<int>(cols);
    const int ro1 = r * ic, ro2 = (r + 1) * ic, ro3 = (2 * r + 1) * ic;
#pragma unroll 1
    for (int k = 0; k < kStencilRows; ++k) {
        const int y = blockIdx.y * (8 * kStencilRows) + (threadIdx.x >> 5) + 8 * k;
        stencil_px<T, RT>(in, in_pitch, in_plane, C, cols, out, out_pitch, out_plane, means, sel,
                          W, H, r, x, y, b, safe, yq, yh, ro1, ro2, ro3);
    }
}

template <typename T, int RT>
void launch_stencil_rt(dim3 grid, cudaStream_t s, const T* in, size_t ip, size_t ipl,
                       const double* sat, double* out, size_t op, size_t opl, int W, int H, int r,
                       double yq, double yh, long long tp, const unsigned* flag) {
    exact_stencil<T, RT><<<grid, 256, 0, s>>>(in, ip, ipl, sat, out, op, opl, nullptr, nullptr, W,
                                              H, r, yq, yh, tp, flag);
}
template <typename T, int... Rs>
bool launch_stencil_fixed(std::integer_sequence<int, Rs...>, dim3 grid, cudaStream_t s,
                          const T* in, size_t ip, size_t ipl, const double* sat, double* out,
                          size_t op, size_t opl, int W, int H, int r, double yq, double yh,
                          long long tp, const unsigned* flag) {
    bool hit = false;
    ((r == Rs + 1 ? (launch_stencil_rt<T, Rs + 1>(grid, s, in, ip, ipl, sat, out, op, opl, W, H,
                                                  r, yq, yh, tp, flag),
                     hit = true)
                  : false),
     ...);
    return hit;
}

template <typename T>
cudaError_t launch_row_prefix(const PlaneView& in, const Geometry& g, double* rowpfx,
                              cudaStream_t s, unsigned* reset_flag) {
    const long long rows = static_cast<long long>(g.batch) * g.height;
    const long long warps = (rows + 31) / 32;
    const unsigned blocks = static_cast<unsigned>((warps + kRowWarps - 1) / kRowWarps);
    exact_row_prefix<T><<<blocks, kRowWarps * 32, 0, s>>>(
        static_cast<const T*>(in.base), in.pitch, in.plane, rowpfx, g.width, g.height, rows,
        reset_flag);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_stencil(const PlaneView& in, const Geometry& g, int r, const double* sat,
                           double* out, size_t op, size_t opl, double* means, uint8_t* sel,
                           cudaStream_t s, long long tp, const unsigned* flag) {
    dim3 grid((g.width + 31) / 32, (g.height + 8 * kStencilRows - 1) / (8 * kStencilRows),
              g.batch);
    // interior reciprocals RN(1/n) (IEEE on the host, the same value)
    const double yq = 1.0 / static_cast<double>((r + 1) * (r + 1));
    const double yh = 1.0 / static_cast<double>((r + 1) * (2 * r + 1));
    // fp64 planes (every pass after the first), no diagnostics, r <= 16: the
    // radius as a template constant
    if constexpr (sizeof(T) == 8) {
        if (!means && !sel && out &&
            launch_stencil_fixed<T>(std::make_integer_sequence<int, 16>{}, grid, s,
                                    static_cast<const T*>(in.base), in.pitch, in.plane, sat, out,
                                    op, opl, g.width, g.height, r, yq, yh, tp, flag))
            return cudaGetLastError();
    }
    exact_stencil<T, 0><<<grid, 256, 0, s>>>(static_cast<const T*>(in.base), in.pitch, in.plane,
                                             sat, out, op, opl, means, sel, g.width, g.height, r,
                                             yq, yh, tp, flag);
    return cudaGetLastError();
}

}  // namespace

// Few-plane launches (about one chain warp per SM or fewer) take the deep
// prefetch builders; same chains, same table.
template <typename T>
cudaError_t launch_row_prefix_deep(const PlaneView& in, const Geometry& g, double* rowpfx,
                                   cudaStream_t s, unsigned* reset_flag) {
    static std::atomic<unsigned long long> done{0};
    if (cudaError_t e = ensure_smem(exact_row_prefix_deep<T>, ROW2_SMEM, done)) return e;
    const long long rows = static_cast<long long>(g.batch) * g.height;
    exact_row_prefix_deep<T><<<static_cast<unsigned>((rows + 31) / 32), 96, ROW2_SMEM, s>>>(
        static_cast<const T*>(in.base), in.pitch, in.plane, rowpfx, g.width, g.height, rows,
        reset_flag);
    return cudaGetLastError();
}

// Table build family: the strip builder (row carries + exact_table_strip) or
// the two chain kernels (OSBF_GPU_TABLE=chains: A/B runs, tests).
bool table_chains_forced() {
    static const bool on = [] {
        const char* e = std::getenv("OSBF_GPU_TABLE");
        return e && std::strcmp(e, "chains") == 0;
    }();
    return on;
}
cudaError_t build_sat_strips(const PlaneView& in, const Geometry& g, double* carries, double* sat,
                             long long tp, unsigned* flag, unsigned* reset, cudaStream_t s,
                             LaunchCounter& lc);

bool table_deep(const Geometry& g);
bool table_uses_strips(const PlaneView&, const Geometry&) { return !table_chains_forced(); }

bool table_deep(const Geometry& g) {
    static const int forced = [] {  // OSBF_GPU_TABLE_DEEP=0/1: A/B runs
        const char* e = std::getenv("OSBF_GPU_TABLE_DEEP");
        return e ? (e[0] == '0' ? 0 : 1) : -1;
    }();
    if (forced >= 0) return forced != 0;
    // measured (r02_exact_paths.jsonl): 2048 chain warps (64 x 1024^2) 1.12 vs
    // 1.38 ms per pass, 1024 warps (16 x 2048^2) 1.12 vs 1.95; 8192 warps
    // (256 x 1024^2) 4.33 vs 4.14
    const long long warps = (static_cast<long long>(g.batch) * g.height + 31) / 32;
    return warps <= 4096;
}

cudaError_t exact_build_sat(const PlaneView& in, const Geometry& g, double* rowpfx, double* sat,
                            cudaStream_t s, LaunchCounter& lc, size_t tpitch, unsigned* table_flag) {
    const long long tp = tpitch ? static_cast<long long>(tpitch) : g.width + 1LL;
    cudaError_t e;
    // the caller's own flag word is cleared by the row-prefix kernel; the
    // shared word stays sticky
    unsigned* const reset = table_flag;
    unsigned* const flag = table_flag ? table_flag : table_flag_address();
    if (!flag) return cudaErrorInvalidDevicePointer;
    // every dtype and shape builds by strips (float32 256 x 1024^2: 3.23 vs
    // 3.65 ms with the chain kernels, uint8 64 x 1024^2: 0.82 vs 1.65)
    if (table_uses_strips(in, g)) return build_sat_strips(in, g, rowpfx, sat, tp, flag, reset, s, lc);
    if (table_deep(g)) {
        switch (in.dtype) {
            case OSBF_U8: e = launch_row_prefix_deep<uint8_t>(in, g, rowpfx, s, reset); break;
            case OSBF_F32: e = launch_row_prefix_deep<float>(in, g, rowpfx, s, reset); break;
            default: e = launch_row_prefix_deep<double>(in, g, rowpfx, s, reset); break;
        }
        ++lc.launches;
        if (e != cudaSuccess) return e;
        static std::atomic<unsigned long long> done{0};
        if ((e = ensure_smem(exact_col_chain_deep, COL2_SMEM, done)) != cudaSuccess) return e;
        const long long wpp = (static_cast<long long>(g.width) + 1 + 31) / 32;
        exact_col_chain_deep<<<static_cast<unsigned>(wpp * g.batch), 96, COL2_SMEM, s>>>(
            rowpfx, sat, g.width, g.height, g.batch, tp, flag);
        ++lc.launches;
        return cudaGetLastError();
    }
    switch (in.dtype) {
        case OSBF_U8: e = launch_row_prefix<uint8_t>(in, g, rowpfx, s, reset); break;
        case OSBF_F32: e = launch_row_prefix<float>(in, g, rowpfx, s, reset); break;
        default: e = launch_row_prefix<double>(in, g, rowpfx, s, reset); break;
    }
    ++lc.launches;
    if (e != cudaSuccess) return e;
    const long long threads = (static_cast<long long>(g.width) + 1) * g.batch;
    exact_col_chain<<<static_cast<unsigned>((threads + 127) / 128), 128, 0, s>>>(
        rowpfx, sat, g.width, g.height, g.batch, tp, flag);
    ++lc.launches;
    return cudaGetLastError();
}

namespace {
using TwalkFn = cudaError_t (*)(const PlaneView&, const Geometry&, const double*, size_t, double*,
                                size_t, size_t, const unsigned*, cudaStream_t);
constexpr TwalkFn kTwalk[kExactFusedMaxRadius + 1] = {
    nullptr,
    exact_twalk_launch<1>,  exact_twalk_launch<2>,  exact_twalk_launch<3>,
    exact_twalk_launch<4>,  exact_twalk_launch<5>,  exact_twalk_launch<6>,
    exact_twalk_launch<7>,  exact_twalk_launch<8>,  exact_twalk_launch<9>,
    exact_twalk_launch<10>, exact_twalk_launch<11>, exact_twalk_launch<12>,
    exact_twalk_launch<13>, exact_twalk_launch<14>, exact_twalk_launch<15>,
    exact_twalk_launch<16>,
};

// Stencil family of a table-path pass: the generic walk (any r <= 62), then
// the templated walk (r <= 16), then the per-thread stencil; an override
// (exact_kernel_override) starts further down the list.
int stencil_family_start() {
    const char* o = exact_kernel_override();
    if (o && std::strcmp(o, "twalk") == 0) return 1;
    if (o && std::strcmp(o, "stencil") == 0) return 2;
    return 0;
}
}  // namespace

cudaError_t exact_select(const PlaneView& in, const Geometry& g, int radius, const double* sat,
                         double* out, size_t out_pitch, size_t out_plane, double* means,
                         uint8_t* sel, cudaStream_t s, LaunchCounter& lc, size_t tpitch,
                         const unsigned* table_flag) {
    ++lc.launches;
    const long long tp = tpitch ? static_cast<long long>(tpitch) : g.width + 1LL;
    const unsigned* const flag = table_flag ? table_flag : table_flag_address();
    if (!flag) return cudaErrorInvalidDevicePointer;
    // label: the table build of this pass + the stencil family
    const bool chains = !table_uses_strips(in, g);
    const int start = stencil_family_start();
    if (out && !means && !sel && start <= 0) {
        // any radius up to 62: three TMA streams of table rows per CTA
        const cudaError_t e = exact_gwalk_launch(in, g, radius, sat, static_cast<size_t>(tp), out,
                                                 out_pitch, out_plane, flag, s);
        if (e != cudaErrorNotSupported) {
            note_kernel(chains ? "exact_row_prefix+exact_col_chain+exact_gwalk"
                               : "exact_row_carries+exact_table_strip+exact_gwalk");
            return e;
        }
    }
    if (out && !means && !sel && radius <= kExactFusedMaxRadius && start <= 1) {
        const cudaError_t e = kTwalk[radius](in, g, sat, static_cast<size_t>(tp), out, out_pitch,
                                             out_plane, flag, s);
        if (e != cudaErrorNotSupported) {
            note_kernel(chains ? "exact_row_prefix+exact_col_chain+exact_twalk"
                               : "exact_row_carries+exact_table_strip+exact_twalk");
            return e;
        }
    }
    note_kernel(chains ? "exact_row_prefix+exact_col_chain+exact_select"
                       : "exact_row_carries+exact_table_strip+exact_select");
    switch (in.dtype) {
        case OSBF_U8:
            return launch_stencil<uint8_t>(in, g, radius, sat, out, out_pitch, out_plane, means,
                                           sel, s, tp, flag);
        case OSBF_F32:
            return launch_stencil<float>(in, g, radius, sat, out, out_pitch, out_plane, means, sel,
                                         s, tp, flag);
        default:
            return launch_stencil<double>(in, g, radius, sat, out, out_pitch, out_plane, means,
                                          sel, s, tp, flag);
    }
}

// ---- fused exact path (osbf_exact2_kernel.cuh) ------------------------------

namespace {
using Exact2Fn = cudaError_t (*)(const PlaneView&, const Geometry&, double*, int, double*, size_t,
                                 size_t, int, double*, cudaStream_t);
constexpr Exact2Fn kExact2[kExactFusedMaxRadius + 1] = {
    nullptr,
    exact2_launch_radius<1>,  exact2_launch_radius<2>,  exact2_launch_radius<3>,
    exact2_launch_radius<4>,  exact2_launch_radius<5>,  exact2_launch_radius<6>,
    exact2_launch_radius<7>,  exact2_launch_radius<8>,  exact2_launch_radius<9>,
    exact2_launch_radius<10>, exact2_launch_radius<11>, exact2_launch_radius<12>,
    exact2_launch_radius<13>, exact2_launch_radius<14>, exact2_launch_radius<15>,
    exact2_launch_radius<16>,
};
static_assert(kExactFusedMaxRadius == 16, "update kExact2");

// OSBF_GPU_CARRIES=warp: keep the single-warp carries kernel (A/B runs).
bool carries_single_warp() {
    static const bool on = [] {
        const char* e = std::getenv("OSBF_GPU_CARRIES");
        return e && std::strcmp(e, "warp") == 0;
    }();
    return on;
}

template <typename T>
cudaError_t launch_carries(const PlaneView& in, const Geometry& g, double* carries, int nsc,
                           cudaStream_t s) {
    static std::atomic<unsigned long long> done_k1{0}, done_k1d{0};
    cudaError_t e = ensure_smem(ex2::exact_row_carries<T>, ex2::K1_SMEM, done_k1);
    if (e == cudaSuccess)
        e = ensure_smem(ex2::exact_row_carries<T, 1, ex2::K1D_STAGES>, ex2::K1D_SMEM, done_k1d);
    if (e != cudaSuccess) return e;
    const long long rows = static_cast<long long>(g.batch) * g.height;
    const long long warps = (rows + 31) / 32;
    if (!carries_single_warp()) {
        // loader warps + a chain warp per 32 rows; a deep ring when there is
        // about one CTA per SM
        static std::atomic<unsigned long long> done_deep{0}, done_many{0};
        auto launch = [&](auto kern, int stages,
                          std::atomic<unsigned long long>& done) -> cudaError_t {
            if (cudaError_t e2 = ensure_smem(kern, rc_smem(stages), done)) return e2;
            kern<<<static_cast<unsigned>(warps), 32 * (TS_LOADERS + 1), rc_smem(stages), s>>>(
                static_cast<const T*>(in.base), in.pitch, in.plane, carries, g.width, g.height,
                rows, nsc);
            return cudaGetLastError();
        };
        static const bool many_ok = [] {  // OSBF_GPU_CARRIES=old: the 2-warp kernel for many rows
            const char* e2 = std::getenv("OSBF_GPU_CARRIES");
            return !(e2 && std::strcmp(e2, "old") == 0);
        }();
        if (warps <= 4 * 148)
            return launch(exact_row_carries_pipe<T, RC_STAGES_DEEP>, RC_STAGES_DEEP, done_deep);
        if (many_ok)
            return launch(exact_row_carries_pipe<T, RC_STAGES_MANY>, RC_STAGES_MANY, done_many);
    }
    if (warps <= 2 * 148) {  // about one warp per SM: deep single-warp CTAs
        ex2::exact_row_carries<T, 1, ex2::K1D_STAGES>
            <<<static_cast<unsigned>(warps), 32, ex2::K1D_SMEM, s>>>(
                static_cast<const T*>(in.base), in.pitch, in.plane, carries, g.width, g.height,
                rows, nsc);
        return cudaGetLastError();
    }
    const long long ctas = (rows + ex2::NTK1 - 1) / ex2::NTK1;
    ex2::exact_row_carries<T><<<static_cast<unsigned>(ctas), ex2::NTK1, ex2::K1_SMEM, s>>>(
        static_cast<const T*>(in.base), in.pitch, in.plane, carries, g.width, g.height, rows, nsc);
    return cudaGetLastError();
}
}  // namespace

// `carries` needs batch * height * (width / 16 + 1) doubles: it fits the
// row-prefix workspace (batch * height * width) of exact_build_sat's contract.
cudaError_t build_sat_strips(const PlaneView& in, const Geometry& g, double* carries, double* sat,
                             long long tp, unsigned* flag, unsigned* reset, cudaStream_t s,
                             LaunchCounter& lc) {
    const int nsc = g.width / ex2::SW + 1;
    if (reset) {  // this pass's flag starts clear (the strips may raise it)
        if (cudaError_t e = cudaMemsetAsync(reset, 0, sizeof(unsigned), s)) return e;
    }
    cudaError_t e;
    switch (in.dtype) {
        case OSBF_U8: e = launch_carries<uint8_t>(in, g, carries, nsc, s); break;
        case OSBF_F32: e = launch_carries<float>(in, g, carries, nsc, s); break;
        default: e = launch_carries<double>(in, g, carries, nsc, s); break;
    }
    ++lc.launches;
    if (e != cudaSuccess) return e;
    dim3 grid((g.width + 1 + 31) / 32, g.batch);  // strips of 32 table columns
    auto go = [&](auto tag) -> cudaError_t {
        using T = decltype(tag);
        static const int forced = [] {  // OSBF_GPU_TABLE_STAGES=6/16: A/B runs
            const char* e2 = std::getenv("OSBF_GPU_TABLE_STAGES");
            return e2 ? atoi(e2) : 0;
        }();
        const bool deep = forced ? forced > TS_STAGES
                                 : static_cast<long long>(grid.x) * grid.y <= 2 * 148;
        auto launch = [&](auto kern, size_t smem,
                          std::atomic<unsigned long long>& done) -> cudaError_t {
            if (cudaError_t e2 = ensure_smem(kern, smem, done)) return e2;
            kern<<<grid, TS_THREADS, smem, s>>>(static_cast<const T*>(in.base), in.pitch, in.plane,
                                                carries, nsc, sat, tp, g.width, g.height, flag);
            return cudaGetLastError();
        };
        static std::atomic<unsigned long long> d0{0}, d1{0};
        return deep ? launch(exact_table_strip<T, TS_STAGES_DEEP>, ts_smem(TS_STAGES_DEEP), d0)
                    : launch(exact_table_strip<T, TS_STAGES>, ts_smem(TS_STAGES), d1);
    };
    switch (in.dtype) {
        case OSBF_U8: e = go(uint8_t{}); break;
        case OSBF_F32: e = go(float{}); break;
        default: e = go(double{}); break;
    }
    ++lc.launches;
    return e;
}

// Band height for under-occupied launches (few strips x planes): enough
// bands for ~4 CTAs per SM, each at least 128 rows (it re-walks 2 blocks).
int exact_band_height(const Geometry& g) {
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    const long long ctas = static_cast<long long>((g.width + ex2::TW - 1) / ex2::TW) * g.batch;
    const long long want = 4LL * sms;
    if (ctas >= want / 2 || g.height < 4 * 128) return 0;
    long long nb = (want + ctas - 1) / ctas;
    int bh = static_cast<int>((g.height + nb - 1) / nb);
    bh = (bh + ex2::BR - 1) / ex2::BR * ex2::BR;
    return bh < 128 ? 128 : bh;
}

size_t exact_fused_carry_elems(const Geometry& g) {
    const size_t rowc = static_cast<size_t>(g.batch) * g.height * (g.width / ex2::SW + 1);
    const int bh = exact_band_height(g);
    const size_t colc =
        bh > 0 ? static_cast<size_t>(g.batch) * ((g.height + bh - 1) / bh) * (g.width + 1) : 0;
    return rowc + colc;
}

cudaError_t exact_fused_step(const PlaneView& in, const Geometry& g, int radius, double* carries,
                             double* out, size_t out_pitch, size_t out_plane, cudaStream_t s,
                             LaunchCounter& lc) {
    if (radius < 1 || radius > kExactFusedMaxRadius) return cudaErrorInvalidValue;
    note_kernel("exact_row_carries+exact_strip");
    const int nsc = g.width / ex2::SW + 1;
    cudaError_t e;
    switch (in.dtype) {
        case OSBF_U8: e = launch_carries<uint8_t>(in, g, carries, nsc, s); break;
        case OSBF_F32: e = launch_carries<float>(in, g, carries, nsc, s); break;
        default: e = launch_carries<double>(in, g, carries, nsc, s); break;
    }
    ++lc.launches;
    if (e != cudaSuccess) return e;
    const int bh = exact_band_height(g);
    double* ccar = carries + static_cast<size_t>(g.batch) * g.height * nsc;
    lc.launches += bh > 0 ? 2 : 1;
    return kExact2[radius](in, g, carries, nsc, out, out_pitch, out_plane, bh, ccar, s);
}

}  // namespace osbf_gpu
