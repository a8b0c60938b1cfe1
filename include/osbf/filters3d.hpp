// Drop-in 3-D filters (GPU build): the reference's proj/include/osbf/
// filters3d.hpp declarations, run on the GPU through libosbf_gpu.so:
//   SubRegion3D / sub_regions_3d   filters3d.hpp:15-51 (host table)
//   box_filter_3d                  filters3d.hpp:55-76
//   osbf_3d                        filters3d.hpp:78-114
// Bit-identical to the reference (the summed-volume table is replayed in its
// order); the same exceptions (radius checked before the iteration count).
#pragma once

#include <array>
#include <stdexcept>
#include <string>
#include <vector>

#include "osbf/core.hpp"
#include "osbf/gpu_runtime.hpp"
#include "osbf/integral.hpp"
#include "osbf/parallel.hpp"

namespace osbf {

/// Per-axis offset ranges of one one-sided 3-D region (relative to the
/// centre voxel), each [-r,0], [0,r] or [-r,r].
struct SubRegion3D {
    int id;  // 1..14
    int u0, u1;
    int v0, v1;
    int w0, w1;
};

/// The 14 regions in selection order: 8 octants by sign pattern (x fastest:
/// (-,-,-), (+,-,-), (-,+,-), ... (+,+,+)), then the half windows -x, +x,
/// -y, +y, -z, +z.
inline std::array<SubRegion3D, 14> sub_regions_3d(int r) {
    if (r < 1) throw std::invalid_argument("sub_regions_3d: radius must be >= 1");
    std::array<SubRegion3D, 14> out{};
    for (int k = 0; k < 8; ++k) {
        const bool px = k & 1, py = (k >> 1) & 1, pz = (k >> 2) & 1;
        out[static_cast<size_t>(k)] = {k + 1,          px ? 0 : -r, px ? r : 0, py ? 0 : -r,
                                       py ? r : 0,     pz ? 0 : -r, pz ? r : 0};
    }
    for (int h = 0; h < 6; ++h) {
        SubRegion3D g{9 + h, -r, r, -r, r, -r, r};
        const int axis = h / 2;
        const bool plus = h & 1;
        int& lo = axis == 0 ? g.u0 : (axis == 1 ? g.v0 : g.w0);
        int& hi = axis == 0 ? g.u1 : (axis == 1 ? g.v1 : g.w1);
        lo = plus ? 0 : -r;
        hi = plus ? r : 0;
        out[static_cast<size_t>(8 + h)] = g;
    }
    return out;
}

namespace detail {
template <typename Entry>
inline Volume run_filter3d(const Volume& vol, int r, int iterations, const char* name,
                           Entry entry) {
    if (r < 1) throw std::invalid_argument(std::string(name) + ": radius must be >= 1");
    if (iterations < 0)
        throw std::invalid_argument(std::string(name) + ": iterations must be >= 0");
    if (iterations == 0) return vol;
    std::vector<double> out(vol.size());
    gpu::detail::check(entry(gpu::detail::context(), vol.samples().data(), out.data(),
                             vol.width(), vol.height(), vol.depth(), r, iterations));
    return Volume(vol.width(), vol.height(), vol.depth(), std::move(out));
}
}  // namespace detail

/// Classical 3-D box filter: valid-count mean over the (2r+1)^3 box, iterated.
inline Volume box_filter_3d(const Volume& vol, int r, int iterations) {
    return detail::run_filter3d(vol, r, iterations, "box_filter_3d", osbf_gpu_box_filter_3d_host);
}

/// 3-D one-sided box filter: the closest of the 14 region means replaces the
/// voxel (ties to the smallest region id); Jacobi iterations.
inline Volume osbf_3d(const Volume& vol, int r, int iterations) {
    return detail::run_filter3d(vol, r, iterations, "osbf_3d", osbf_gpu_osbf_3d_host);
}

}  // namespace osbf
