// 3-D extension: osbf_3d and box_filter_3d
// (filters3d.hpp:55-114) on a single fp64 volume, bit-identical.
//
// The summed-volume table (integral.hpp:98-113) is replayed in the
// reference's order: a running row sum over x per (y, z) row, and
//   T(x+1,y+1,z+1) = ((row + T(x+1,y,z+1)) + T(x+1,y+1,z)) - T(x+1,y,z)
// which, for a fixed column x, depends only on earlier (z, y) of the same
// column: svt_yz runs it as a pipelined plane wavefront (see there).  The
// filter kernel evaluates per voxel the 14 (box: 1) clipped box sums with the
// reference's inclusion-exclusion order, IEEE division by the clipped count,
// |a - u| and the strict-< first minimum in filters3d.hpp:29-51 order.
//
// Per pass (256^3): svt_rows ~55 us (HBM-streaming), svt_yz ~180 us (one
// barrier per wavefront step; 2 columns x 128 plane slots per CTA measured
// best: 4 columns 214 us, 1 column 288 us), filter3d ~800 us — fp64-latency/L1 bound:
// 64 distinct table corners, 98 dependent-chain DADDs and 14 divisions per
// voxel, not an HBM roofline kernel.
#include "osbf_exact2_kernel.cuh"  // div_by_count
#include "osbf_internal.cuh"

namespace osbf_gpu {
namespace {

// Running row sums over x (integral.hpp:104-106), one thread per (y, z) row,
// 128 rows per CTA; columns go through a padded shared tile 32 at a time so
// global loads and stores are coalesced while each row is still summed
// serially from x = 0.
constexpr int kRowsCta = 128, kRowsTile = 32;

__global__ void __launch_bounds__(kRowsCta)
    svt_rows(const double* __restrict__ in, double* __restrict__ rowp, int W, long long rows) {
    __shared__ double tile[kRowsCta][kRowsTile + 1];
    const long long row0 = static_cast<long long>(blockIdx.x) * kRowsCta;
    const int nrows = static_cast<int>(min(static_cast<long long>(kRowsCta), rows - row0));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double acc = 0.0;
    for (int x0 = 0; x0 < W; x0 += kRowsTile) {
        const int nx = min(kRowsTile, W - x0);
        for (int rr = warp; rr < nrows; rr += kRowsCta / 32)
            if (lane < nx) tile[rr][lane] = in[(row0 + rr) * W + x0 + lane];
        __syncthreads();
        if (threadIdx.x < nrows)
            for (int k = 0; k < nx; ++k) {
                acc = __dadd_rn(acc, tile[threadIdx.x][k]);  // row += vol(x, y, z)
                tile[threadIdx.x][k] = acc;
            }
        __syncthreads();
        for (int rr = warp; rr < nrows; rr += kRowsCta / 32)
            if (lane < nx) rowp[(row0 + rr) * W + x0 + lane] = tile[rr][lane];
        __syncthreads();
    }
}

// The (y, z) recurrence of one x column is a 2-D wavefront: plane z may
// compute row y as soon as plane z-1 has produced row y.  A CTA owns XL
// adjacent columns (one 32 B sector per row) and NP = PL * NW plane slots
// (lane groups); slot g runs planes g, g+NP, g+2NP, ... one row per step,
// lagging slot g-1 by one step, so T(y, z-1) arrives through a shared-memory
// double buffer written the step before (one barrier per step).  A slot's
// planes start every Hp >= NP steps; when Hp > NP slot 0 reads T(y, z-1) of
// slot NP-1 back from the table instead (written Hp-NP+1 >= PF+1 steps
// earlier), prefetched PF steps ahead with cp.async together with the row
// prefixes.
// T(y-1, z) and T(y-1, z-1) stay in registers.
constexpr int kSvtXL = 2, kSvtPL = 16, kSvtNW = 8, kSvtPF = 8;
constexpr int kSvtNP = kSvtPL * kSvtNW;

struct SvtCursor {  // plane slot position: row y (negative while waiting), plane z
    int y, z;
    __device__ void advance(int Hp) {
        if (++y == Hp) {
            y = 0;
            z += kSvtNP;
        }
    }
    __device__ bool active(int H, int D) const { return y >= 0 && y < H && z < D; }
};

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}

__global__ void __launch_bounds__(32 * kSvtNW, 1)
    svt_yz(const double* __restrict__ rowp, double* T, int W, int H, int D, int Hp, int steps) {
    // PF + 1 slots: slot of step s is refilled at step s + 1, after the barrier
    // that ends step s.  Each thread reads only the slots it filled itself, so
    // cp.async.wait_group is the only wait (a plain global load in flight would
    // be drained by every barrier).
    __shared__ double rs[kSvtPF + 1][kSvtNP][kSvtXL];
    __shared__ double us[kSvtPF + 1][kSvtXL];  // slot 0's T(y, z-1) when Hp > NP
    __shared__ double xb[2][kSvtNP][kSvtXL];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int xi = lane % kSvtXL, g = warp * kSvtPL + lane / kSvtXL;
    const int x = blockIdx.x * kSvtXL + xi;
    const bool xok = x < W;
    const bool up_smem = g > 0 || Hp == kSvtNP;
    const int gp = g == 0 ? kSvtNP - 1 : g - 1;
    const size_t W1 = static_cast<size_t>(W) + 1, H1 = static_cast<size_t>(H) + 1;

    auto fetch = [&](const SvtCursor& c, int slot) {
        if (xok && c.active(H, D)) {
            cp_async8(&rs[slot][g][xi], rowp + (static_cast<size_t>(c.z) * H + c.y) * W + x);
            if (!up_smem && c.z > 0)
                cp_async8(&us[slot][xi], T + (static_cast<size_t>(c.z) * H1 + c.y + 1) * W1 + x + 1);
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };

    SvtCursor cur{-g, g}, pre{-g, g};
    for (int k = 0; k < kSvtPF; ++k) {
        fetch(pre, k);
        pre.advance(Hp);
    }
    double own = 0.0, diag = 0.0;  // T(y-1, z), T(y-1, z-1)
    int slot = 0, pslot = kSvtPF;
    for (int s = 0; s < steps; ++s) {
        fetch(pre, pslot);  // step s + PF (its T(y, z-1) was written >= 1 step ago)
        pre.advance(Hp);
        asm volatile("cp.async.wait_group %0;\n" ::"n"(kSvtPF) : "memory");
        if (cur.active(H, D)) {
            if (cur.y == 0) {
                own = 0.0;
                diag = 0.0;
            }
            double up = 0.0;
            if (cur.z > 0) up = up_smem ? xb[(s - 1) & 1][gp][xi] : us[slot][xi];
            // integral.hpp:108-109: row + T(x+1,y,z+1) + T(x+1,y+1,z) - T(x+1,y,z)
            const double v = __dsub_rn(__dadd_rn(__dadd_rn(rs[slot][g][xi], own), up), diag);
            if (xok) T[(static_cast<size_t>(cur.z + 1) * H1 + cur.y + 1) * W1 + x + 1] = v;
            own = v;
            diag = up;
            xb[s & 1][g][xi] = v;
        }
        cur.advance(Hp);
        slot = slot == kSvtPF ? 0 : slot + 1;
        pslot = pslot == kSvtPF ? 0 : pslot + 1;
        __syncthreads();
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// Per voxel and axis the clipped box bounds take four cumsum indices
// (integral.hpp:121-134 clipping): A0 = max(c-r, 0), A1 = c, B0 = c+1,
// B1 = min(c+r, n-1)+1; a region picks per axis L = [A0, B0) (offsets
// [-r, 0]), R = [A1, B1) ([0, r]) or F = [A0, B1) ([-r, r]).  Sums follow the
// reference's inclusion-exclusion order; the clipped count is the product of
// the per-axis extents.  Interior voxels divide with the precomputed
// reciprocal (div_by_count: the IEEE quotient), border voxels with __ddiv_rn.
enum : int { kSelL = 0, kSelR = 1, kSelF = 2 };

struct Axis3 {
    int idx[4];  // A0, A1, B0, B1
    __device__ Axis3(int c, int r, int n) {
        idx[0] = max(c - r, 0);
        idx[1] = c;
        idx[2] = c + 1;
        idx[3] = min(c + r, n - 1) + 1;
    }
    __device__ static constexpr int lo(int sel) { return sel == kSelR ? 1 : 0; }
    __device__ static constexpr int hi(int sel) { return sel == kSelL ? 2 : 3; }
    __device__ int count(int sel) const { return idx[hi(sel)] - idx[lo(sel)]; }
};

template <int SX, int SY, int SZ>
__device__ __forceinline__ double box_sum3(const double* __restrict__ T, const long long (&zo)[4],
                                           const long long (&yo)[4], const int (&xo)[4]) {
    constexpr int ax = Axis3::lo(SX), bx = Axis3::hi(SX), ay = Axis3::lo(SY), by = Axis3::hi(SY),
                  az = Axis3::lo(SZ), bz = Axis3::hi(SZ);
    auto c = [&](int xi, int yi, int zi) { return __ldg(T + (zo[zi] + yo[yi] + xo[xi])); };
    // integral.hpp:132-134
    double s = __dsub_rn(c(bx, by, bz), c(ax, by, bz));
    s = __dsub_rn(s, c(bx, ay, bz));
    s = __dsub_rn(s, c(bx, by, az));
    s = __dadd_rn(s, c(ax, ay, bz));
    s = __dadd_rn(s, c(ax, by, az));
    s = __dadd_rn(s, c(bx, ay, az));
    return __dsub_rn(s, c(ax, ay, az));
}

template <int SX, int SY, int SZ>
__device__ __forceinline__ double box_mean3(const double* __restrict__ T, const long long (&zo)[4],
                                            const long long (&yo)[4], const int (&xo)[4],
                                            const Axis3& ax, const Axis3& ay, const Axis3& az,
                                            bool interior, double n_in, double recip) {
    const double s = box_sum3<SX, SY, SZ>(T, zo, yo, xo);
    if (interior) return div_by_count(s, n_in, recip);
    const double n = static_cast<double>(static_cast<long long>(ax.count(SX)) * ay.count(SY) *
                                         az.count(SZ));
    return __ddiv_rn(s, n);
}

template <int SX, int SY, int SZ>
__device__ __forceinline__ void consider(double a, double u, double& best, double& best_abs) {
    const double dist = fabs(__dsub_rn(a, u));
    if (dist < best_abs) {  // strict <: ties keep the smaller region id
        best_abs = dist;
        best = a;
    }
}

struct Counts3 {  // interior region sizes and RN(1/n)
    double n_oct, r_oct, n_half, r_half, n_box, r_box;
};

constexpr int kF3X = 32, kF3Y = 8;

// One thread per voxel, CTA = 32 x 8 (x, y) tile of one z plane; grid
// (ceil(W/32), ceil(H/8), min(D, 65535)) with a z stride loop.
template <bool OSBF>
__global__ void __launch_bounds__(kF3X * kF3Y, 3)
    filter3d(const double* __restrict__ in, const double* __restrict__ T, double* __restrict__ out,
             int W, int H, int D, int r, Counts3 k) {
    const int x = blockIdx.x * kF3X + threadIdx.x;
    const int y = blockIdx.y * kF3Y + threadIdx.y;
    if (x >= W || y >= H) return;
    for (int z = blockIdx.z; z < D; z += gridDim.z) {
    const size_t i = (static_cast<size_t>(z) * H + y) * W + x;
    const Axis3 ax(x, r, W), ay(y, r, H), az(z, r, D);
    const long long W1 = static_cast<long long>(W) + 1, PS = W1 * (H + 1);
    int xo[4];
    long long yo[4], zo[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        xo[q] = ax.idx[q];
        yo[q] = ay.idx[q] * W1;
        zo[q] = az.idx[q] * PS;
    }
    const bool interior = x >= r && x < W - r && y >= r && y < H - r && z >= r && z < D - r;
    if (!OSBF) {
        out[i] = box_mean3<kSelF, kSelF, kSelF>(T, zo, yo, xo, ax, ay, az, interior, k.n_box,
                                                k.r_box);
        continue;
    }
    const double u = in[i];
    double best = 0.0, best_abs = __longlong_as_double(0x7ff0000000000000LL);  // +inf
#define OSBF3_REGION(SX, SY, SZ, N, RC)                                                            \
    consider<SX, SY, SZ>(box_mean3<SX, SY, SZ>(T, zo, yo, xo, ax, ay, az, interior, N, RC), u, best, \
                         best_abs)
    // filters3d.hpp:29-51 order: octants by sign pattern, x fastest ...
    OSBF3_REGION(kSelL, kSelL, kSelL, k.n_oct, k.r_oct);
    OSBF3_REGION(kSelR, kSelL, kSelL, k.n_oct, k.r_oct);
    OSBF3_REGION(kSelL, kSelR, kSelL, k.n_oct, k.r_oct);
    OSBF3_REGION(kSelR, kSelR, kSelL, k.n_oct, k.r_oct);
    OSBF3_REGION(kSelL, kSelL, kSelR, k.n_oct, k.r_oct);
    OSBF3_REGION(kSelR, kSelL, kSelR, k.n_oct, k.r_oct);
    OSBF3_REGION(kSelL, kSelR, kSelR, k.n_oct, k.r_oct);
    OSBF3_REGION(kSelR, kSelR, kSelR, k.n_oct, k.r_oct);
    // ... then the half windows -x, +x, -y, +y, -z, +z
    OSBF3_REGION(kSelL, kSelF, kSelF, k.n_half, k.r_half);
    OSBF3_REGION(kSelR, kSelF, kSelF, k.n_half, k.r_half);
    OSBF3_REGION(kSelF, kSelL, kSelF, k.n_half, k.r_half);
    OSBF3_REGION(kSelF, kSelR, kSelF, k.n_half, k.r_half);
    OSBF3_REGION(kSelF, kSelF, kSelL, k.n_half, k.r_half);
    OSBF3_REGION(kSelF, kSelF, kSelR, k.n_half, k.r_half);
#undef OSBF3_REGION
    out[i] = best;
    }
}

}  // namespace

size_t svt_elems(int W, int H, int D) {
    return (static_cast<size_t>(W) + 1) * (static_cast<size_t>(H) + 1) * (static_cast<size_t>(D) + 1);
}

cudaError_t svt_build(const double* in, int W, int H, int D, double* rowp, double* table,
                      cudaStream_t s, LaunchCounter& lc) {
    const long long rows = static_cast<long long>(H) * D;
    cudaError_t e = cudaMemsetAsync(table, 0, sizeof(double) * svt_elems(W, H, D), s);
    if (e != cudaSuccess) return e;
    svt_rows<<<static_cast<unsigned>((rows + kRowsCta - 1) / kRowsCta), kRowsCta, 0, s>>>(in, rowp, W,
                                                                                     rows);
    // plane slots restart every Hp steps; Hp > NP leaves PF steps of slack so
    // slot 0's prefetched T(y, z-1) is always written before it is read
    const int Hp = H <= kSvtNP ? kSvtNP : std::max(H, kSvtNP + kSvtPF);
    const long long last = static_cast<long long>((D - 1) / kSvtNP) * Hp + (D - 1) % kSvtNP + H;
    if (last > INT32_MAX) return cudaErrorInvalidValue;
    svt_yz<<<(W + kSvtXL - 1) / kSvtXL, 32 * kSvtNW, 0, s>>>(rowp, table, W, H, D, Hp,
                                                           static_cast<int>(last));
    lc.launches += 2;
    return cudaGetLastError();
}

cudaError_t filter3d_pass(const double* in, int W, int H, int D, int r, bool osbf,
                          double* rowp, double* table, double* out, cudaStream_t s,
                          LaunchCounter& lc) {
    cudaError_t e = svt_build(in, W, H, D, rowp, table, s, lc);
    if (e != cudaSuccess) return e;
    // interior counts: octant (r+1)^3, half window (r+1)(2r+1)^2, box (2r+1)^3
    const double r1 = r + 1.0, r2 = 2.0 * r + 1.0;
    Counts3 k;
    k.n_oct = r1 * r1 * r1;
    k.n_half = r1 * r2 * r2;
    k.n_box = r2 * r2 * r2;
    k.r_oct = 1.0 / k.n_oct;
    k.r_half = 1.0 / k.n_half;
    k.r_box = 1.0 / k.n_box;
    const dim3 grid((W + kF3X - 1) / kF3X, (H + kF3Y - 1) / kF3Y, std::min(D, 65535));
    const dim3 block(kF3X, kF3Y);
    if (osbf)
        filter3d<true><<<grid, block, 0, s>>>(in, table, out, W, H, D, r, k);
    else
        filter3d<false><<<grid, block, 0, s>>>(in, table, out, W, H, D, r, k);
    lc.launches += 1;
    return cudaGetLastError();
}

}  // namespace osbf_gpu
