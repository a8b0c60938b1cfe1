// Drop-in exact OSBF (GPU build) — the reference's hot path.
//
// Same declarations, argument meaning and exceptions as the reference's
// proj/include/osbf/filters2d.hpp for the exact one-sided box filter:
//   SubWindowMeans / subwindow_means   filters2d.hpp:19-34
//   osbf_step                          filters2d.hpp:61-88
//   osbf                               filters2d.hpp:91-98
//   box_filter                         filters2d.hpp:38-56
//   fast_osbf (paper Algorithm 3)      filters2d.hpp:105-154
//   filter_multichannel (OsbfExact, OsbfFast, Box)  filters2d.hpp:371-400
// Each call runs on the GPU through libosbf_gpu.so (include/osbf_gpu.h).
// The default arithmetic mode is gpu::Mode::Exact: results are bit-identical
// to the reference.  gpu::set_mode(gpu::Mode::Fast) selects the tile-local
// kernel (same selection rule, fp64 sums within a few ulps).  fast_osbf is
// always bit-identical to the reference.
//
// Out of scope for the GPU build: the generic one-sided / Gaussian filters
// and kernel_spectrum; filter_multichannel throws std::invalid_argument for
// those variants.
#pragma once

#include <array>
#include <stdexcept>
#include <vector>

#include "osbf/core.hpp"
#include "osbf/gpu_runtime.hpp"
#include "osbf/integral.hpp"
#include "osbf/parallel.hpp"

namespace osbf {

/// The eight one-sided window means a1..a8 at one pixel.
struct SubWindowMeans {
    std::array<double, 8> a;
};

/// Valid-count means of the eight windows centred at (x,y) (host lookups
/// into a GPU-built, bit-identical summed-area table).
inline SubWindowMeans subwindow_means(const SummedAreaTable& sat, int x, int y, int r) {
    const auto wins = sub_windows(r);
    SubWindowMeans m{};
    for (size_t i = 0; i < wins.size(); ++i)
        m.a[i] = sat.rect_mean(x + wins[i].u0, y + wins[i].v0, x + wins[i].u1, y + wins[i].v1);
    return m;
}

/// One Jacobi pass: every pixel becomes the window mean closest to it
/// (strict <, first minimum wins).  Throws std::invalid_argument if r < 1.
inline ImagePlane osbf_step(const ImagePlane& plane, int r) {
    std::vector<double> out(plane.size());
    gpu::detail::check(osbf_gpu_osbf_step_host(gpu::detail::context(), plane.samples().data(),
                                               out.data(), plane.width(), plane.height(), r,
                                               static_cast<osbf_mode>(gpu::mode())));
    return ImagePlane(plane.width(), plane.height(), std::move(out));
}

/// `iterations` Jacobi passes.  iterations < 0 throws; iterations == 0
/// returns a copy without checking r (as the reference does).
inline ImagePlane osbf(const ImagePlane& plane, int r, int iterations) {
    if (iterations < 0) throw std::invalid_argument("osbf: iterations must be >= 0");
    if (iterations == 0) return plane;
    std::vector<double> out(plane.size());
    gpu::detail::check(osbf_gpu_osbf_host(gpu::detail::context(), OSBF_F64,
                                          plane.samples().data(), out.data(), plane.width(),
                                          plane.height(), 1, r, iterations,
                                          static_cast<osbf_mode>(gpu::mode())));
    return ImagePlane(plane.width(), plane.height(), std::move(out));
}

/// Classical box filter: valid-count mean over the full (2r+1)^2 window,
/// iterated.  Throws std::invalid_argument if r < 1 (even for 0
/// iterations) or iterations < 0.  Bit-identical to the reference.
inline ImagePlane box_filter(const ImagePlane& plane, int r, int iterations) {
    if (r < 1) throw std::invalid_argument("box_filter: radius must be >= 1");
    if (iterations < 0) throw std::invalid_argument("box_filter: iterations must be >= 0");
    if (iterations == 0) return plane;
    std::vector<double> out(plane.size());
    gpu::detail::check(osbf_gpu_box_filter_host(gpu::detail::context(), OSBF_F64,
                                                plane.samples().data(), out.data(), plane.width(),
                                                plane.height(), 1, r, iterations));
    return ImagePlane(plane.width(), plane.height(), std::move(out));
}

/// Paper Algorithm 3: one quarter-mean field per iteration, the other
/// candidates are clamped shifted lookups and pairwise averages of it.
/// Throws std::invalid_argument if r < 1 (even for 0 iterations) or
/// iterations < 0.  Bit-identical to the reference.
inline ImagePlane fast_osbf(const ImagePlane& plane, int r, int iterations) {
    if (r < 1) throw std::invalid_argument("fast_osbf: radius must be >= 1");
    if (iterations < 0) throw std::invalid_argument("fast_osbf: iterations must be >= 0");
    if (iterations == 0) return plane;
    std::vector<double> out(plane.size());
    gpu::detail::check(osbf_gpu_fast_osbf_host(gpu::detail::context(), OSBF_F64,
                                               plane.samples().data(), out.data(), plane.width(),
                                               plane.height(), 1, r, iterations));
    return ImagePlane(plane.width(), plane.height(), std::move(out));
}

/// Channels filtered independently (one batched GPU launch per pass).
inline MultiChannelImage filter_multichannel(const MultiChannelImage& img,
                                             const FilterConfig& config) {
    config.validate();
    if (config.variant != FilterVariant::OsbfExact && config.variant != FilterVariant::OsbfFast &&
        config.variant != FilterVariant::Box)
        throw std::invalid_argument(
            "filter_multichannel: only FilterVariant::OsbfExact, OsbfFast and Box are provided by "
            "the GPU build");
    const int c = img.channel_count();
    std::vector<const double*> in(static_cast<size_t>(c));
    std::vector<std::vector<double>> res(static_cast<size_t>(c));
    std::vector<double*> out(static_cast<size_t>(c));
    for (int i = 0; i < c; ++i) {
        in[static_cast<size_t>(i)] = img.channel(i).samples().data();
        res[static_cast<size_t>(i)].resize(img.channel(i).size());
        out[static_cast<size_t>(i)] = res[static_cast<size_t>(i)].data();
    }
    if (config.variant == FilterVariant::Box)
        gpu::detail::check(osbf_gpu_filter_multichannel_box_host(
            gpu::detail::context(), in.data(), out.data(), c, img.width(), img.height(),
            config.radius, config.iterations));
    else if (config.variant == FilterVariant::OsbfFast)
        gpu::detail::check(osbf_gpu_filter_multichannel_fast_host(
            gpu::detail::context(), in.data(), out.data(), c, img.width(), img.height(),
            config.radius, config.iterations));
    else
        gpu::detail::check(osbf_gpu_filter_multichannel_host(
            gpu::detail::context(), in.data(), out.data(), c, img.width(), img.height(),
            config.radius, config.iterations, static_cast<osbf_mode>(gpu::mode())));
    std::vector<ImagePlane> planes;
    planes.reserve(static_cast<size_t>(c));
    for (int i = 0; i < c; ++i)
        planes.emplace_back(img.width(), img.height(), std::move(res[static_cast<size_t>(i)]));
    return MultiChannelImage(std::move(planes));
}

}  // namespace osbf
