// TEST INFRASTRUCTURE ONLY — a C-ABI shim around the UNMODIFIED reference
// headers (/root/reference/proj/include, header-only C++20).  Compiled by
// oracle/Makefile straight from the reference tree into oracle/_ref/; no
// reference source is copied into this repository.  Used to (1) pin the C
// restatement in osbf_oracle.c bit-for-bit, (2) generate tests/golden/, and
// (3) time the reference CPU path for bench.py's cpu_baseline / --impl
// reference legs.
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <vector>

#include "osbf/bench.hpp"
#include "osbf/filters2d.hpp"
#include "osbf/filters3d.hpp"
#include "osbf/io.hpp"
#include "osbf/metrics.hpp"
#include "osbf/parallel.hpp"
#include "osbf/synth.hpp"
#include "support/fixtures.hpp"

namespace {

int map_exception() {
    try {
        throw;
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (const std::domain_error&) {
        return 2;
    } catch (const std::out_of_range&) {
        return 3;
    } catch (...) {
        return 9;
    }
}

osbf::ImagePlane to_plane(const double* p, int w, int h) {
    return osbf::ImagePlane(w, h, std::vector<double>(p, p + static_cast<size_t>(w) * h));
}

osbf::Volume to_volume(const double* p, int w, int h, int d) {
    return osbf::Volume(w, h, d, std::vector<double>(p, p + static_cast<size_t>(w) * h * d));
}

}  // namespace

extern "C" {

void ref_set_max_threads(int n) { osbf::set_max_threads(n); }
int ref_max_threads(void) { return osbf::max_threads(); }
void ref_pin_allocator_for_timing(void) { osbf::pin_allocator_for_timing(); }

// osbf::osbf (filters2d.hpp:91-98)
int ref_osbf(const double* in, double* out, int w, int h, int r, int iterations) {
    try {
        const auto res = osbf::osbf(to_plane(in, w, h), r, iterations);
        std::memcpy(out, res.samples().data(), sizeof(double) * res.size());
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// osbf::osbf_3d / box_filter_3d (filters3d.hpp:55-114)
int ref_filter_3d(const double* in, double* out, int w, int h, int d, int r, int iterations,
                  int osbf3) {
    try {
        const auto v = to_volume(in, w, h, d);
        const auto res = osbf3 ? osbf::osbf_3d(v, r, iterations) : osbf::box_filter_3d(v, r, iterations);
        for (int z = 0; z < d; ++z)
            for (int y = 0; y < h; ++y)
                for (int x = 0; x < w; ++x)
                    out[(static_cast<size_t>(z) * h + y) * w + x] = res(x, y, z);
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// SummedVolumeTable (integral.hpp:98-113): cumsum((w+1)x(h+1)x(d+1))
int ref_svt(const double* in, int w, int h, int d, double* cumsum) {
    try {
        const osbf::SummedVolumeTable t(to_volume(in, w, h, d));
        for (int z = 0; z <= d; ++z)
            for (int y = 0; y <= h; ++y)
                for (int x = 0; x <= w; ++x)
                    cumsum[(static_cast<size_t>(z) * (h + 1) + y) * (w + 1) + x] = t.cumsum(x, y, z);
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// osbf::box_filter (filters2d.hpp:38-56)
int ref_box_filter(const double* in, double* out, int w, int h, int r, int iterations) {
    try {
        const auto res = osbf::box_filter(to_plane(in, w, h), r, iterations);
        std::memcpy(out, res.samples().data(), sizeof(double) * res.size());
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// osbf::fast_osbf (filters2d.hpp:105-154, paper Algorithm 3)
int ref_fast_osbf(const double* in, double* out, int w, int h, int r, int iterations) {
    try {
        const auto res = osbf::fast_osbf(to_plane(in, w, h), r, iterations);
        std::memcpy(out, res.samples().data(), sizeof(double) * res.size());
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// osbf::filter_multichannel with FilterVariant::OsbfFast (filters2d.hpp:371-400).
int ref_filter_multichannel_fast(const double* in, double* out, int channels, int w, int h, int r,
                                 int iterations) {
    try {
        std::vector<osbf::ImagePlane> planes;
        for (int c = 0; c < channels; ++c)
            planes.push_back(to_plane(in + static_cast<size_t>(c) * w * h, w, h));
        osbf::FilterConfig cfg;
        cfg.radius = r;
        cfg.iterations = iterations;
        cfg.variant = osbf::FilterVariant::OsbfFast;
        const auto res = osbf::filter_multichannel(osbf::MultiChannelImage(std::move(planes)), cfg);
        for (int c = 0; c < channels; ++c)
            std::memcpy(out + static_cast<size_t>(c) * w * h, res.channel(c).samples().data(),
                        sizeof(double) * static_cast<size_t>(w) * h);
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// osbf::osbf_step (filters2d.hpp:61-88)
int ref_osbf_step(const double* in, double* out, int w, int h, int r) {
    try {
        const auto res = osbf::osbf_step(to_plane(in, w, h), r);
        std::memcpy(out, res.samples().data(), sizeof(double) * res.size());
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// osbf::filter_multichannel with FilterVariant::OsbfExact (filters2d.hpp:371-400).
// in/out: `channels` planes of w*h doubles, back to back.
int ref_filter_multichannel(const double* in, double* out, int channels, int w, int h, int r,
                            int iterations) {
    try {
        std::vector<osbf::ImagePlane> planes;
        for (int c = 0; c < channels; ++c)
            planes.push_back(to_plane(in + static_cast<size_t>(c) * w * h, w, h));
        osbf::FilterConfig cfg;
        cfg.radius = r;
        cfg.iterations = iterations;
        cfg.variant = osbf::FilterVariant::OsbfExact;
        const auto res = osbf::filter_multichannel(osbf::MultiChannelImage(std::move(planes)), cfg);
        for (int c = 0; c < channels; ++c)
            std::memcpy(out + static_cast<size_t>(c) * w * h, res.channel(c).samples().data(),
                        sizeof(double) * static_cast<size_t>(w) * h);
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// SummedAreaTable cumsum (integral.hpp:16-30), (w+1)*(h+1) doubles.
int ref_sat(const double* in, int w, int h, double* cumsum) {
    try {
        const auto sat = osbf::build_sat(to_plane(in, w, h));
        for (int y = 0; y <= h; ++y)
            for (int x = 0; x <= w; ++x)
                cumsum[static_cast<size_t>(y) * (w + 1) + x] = sat.cumsum(x, y);
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// subwindow_means (filters2d.hpp:26-34) at every pixel: out[(y*w+x)*8 + i],
// plus the selected window id (strict <, filters2d.hpp:72-82) in sel.
int ref_subwindow_means(const double* in, int w, int h, int r, double* out, uint8_t* sel) {
    try {
        const auto plane = to_plane(in, w, h);
        const auto sat = osbf::build_sat(plane);
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x) {
                const auto m = osbf::subwindow_means(sat, x, y, r);
                const double u = plane(x, y);
                double best_abs = 1.0 / 0.0;
                int id = 0;
                for (int i = 0; i < 8; ++i) {
                    out[(static_cast<size_t>(y) * w + x) * 8 + i] = m.a[i];
                    const double d = std::abs(m.a[i] - u);
                    if (d < best_abs) {
                        best_abs = d;
                        id = i + 1;
                    }
                }
                if (sel) sel[static_cast<size_t>(y) * w + x] = static_cast<uint8_t>(id);
            }
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// rect_mean on the reference SAT (integral.hpp:64-69) — error behaviour probe.
int ref_rect_mean(const double* in, int w, int h, int x0, int y0, int x1, int y1, double* mean) {
    try {
        const auto sat = osbf::build_sat(to_plane(in, w, h));
        *mean = osbf::rect_mean(sat, x0, y0, x1, y1);
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// osbf::detail::quantize (io.hpp:108-115)
int ref_quantize(double v, int maxval) { return osbf::detail::quantize(v, maxval); }

// tools/osbf_main.cpp:63-83 (cmd_smooth) through the reference's own file
// I/O: read_image -> FilterConfig::validate -> filter_multichannel ->
// write_image(bit depth 8 if maxval <= 255 else 16).  filter: 0 osbf,
// 1 fast-osbf, 2 box.
int ref_smooth_file(const char* in_path, const char* out_path, int filter, int r, int iterations) {
    try {
        int maxval = 255;
        const osbf::MultiChannelImage img = osbf::read_image(in_path, &maxval);
        osbf::FilterConfig cfg;
        cfg.radius = r;
        cfg.iterations = iterations;
        cfg.variant = filter == 1   ? osbf::FilterVariant::OsbfFast
                      : filter == 2 ? osbf::FilterVariant::Box
                                    : osbf::FilterVariant::OsbfExact;
        cfg.validate();
        const osbf::MultiChannelImage out = osbf::filter_multichannel(img, cfg);
        osbf::write_image(out, out_path, maxval <= 255 ? 8 : 16);
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// ---- acceptance-criterion inputs and metrics (acceptance.cpp:82-102,
// :220-235, :293-319), generated by the reference's own synth / fixtures so
// the GPU runs see the exact bytes the reference's checks use.

// osbf::checkerboard (synth.hpp:52) + osbf::add_gaussian_noise (synth.hpp:94)
int ref_checkerboard(int w, int h, int cell, double lo, double hi, double sigma,
                     unsigned long long seed, double* clean, double* noisy) {
    try {
        const auto c = osbf::checkerboard(w, h, cell, lo, hi);
        const auto n = osbf::add_gaussian_noise(c, {sigma, seed});
        std::memcpy(clean, c.samples().data(), sizeof(double) * c.size());
        std::memcpy(noisy, n.samples().data(), sizeof(double) * n.size());
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// osbf::step_volume (synth.hpp:81) + add_gaussian_noise (synth.hpp:106)
int ref_step_volume(int w, int h, int d, int edge, double lo, double hi, double sigma,
                    unsigned long long seed, double* clean, double* noisy) {
    try {
        const auto c = osbf::step_volume(w, h, d, edge, lo, hi);
        const auto n = osbf::add_gaussian_noise(c, {sigma, seed});
        std::memcpy(clean, c.samples().data(), sizeof(double) * c.size());
        std::memcpy(noisy, n.samples().data(), sizeof(double) * n.size());
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// fixtures::phantom (tests/support/fixtures.hpp:36), the stand-in natural image
int ref_phantom(int w, int h, double* out) {
    try {
        const auto p = fixtures::phantom(w, h);
        std::memcpy(out, p.samples().data(), sizeof(double) * p.size());
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// osbf::psnr / osbf::rmse (metrics.hpp:37-53)
double ref_psnr(const double* a, const double* b, int w, int h, double peak) {
    return osbf::psnr(to_plane(a, w, h), to_plane(b, w, h), peak);
}
double ref_rmse(const double* a, const double* b, int w, int h) {
    return osbf::rmse(to_plane(a, w, h), to_plane(b, w, h));
}

}  // extern "C"
