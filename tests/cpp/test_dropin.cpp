// C++ drop-in test: the reference's hot-path test cases (proj/tests/
// test_core.cpp, test_integral.cpp, test_filters2d.cpp, test_filters3d.cpp,
// acceptance.cpp
// criteria 1, 2, 5) re-expressed against include/osbf/*.hpp, which run on the
// GPU through libosbf_gpu.so.  The CPU checker is the oracle restatement
// (oracle/osbf_oracle.c; test infrastructure only).  Prints one PASS/FAIL
// line per case; exit code = number of failures.
#include <array>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <functional>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "osbf/osbf.hpp"
#include "osbf_oracle.h"

using osbf::ImagePlane;

namespace {

int failures = 0;

void run(const char* name, const std::function<bool()>& fn) {
    bool ok = false;
    std::string why;
    try {
        ok = fn();
    } catch (const std::exception& e) {
        why = e.what();
    }
    std::printf("%s %s%s%s\n", ok ? "PASS" : "FAIL", name, why.empty() ? "" : ": ", why.c_str());
    if (!ok) ++failures;
}

template <typename E, typename F>
bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

// fixtures::random_plane equivalent (mt19937_64, 53-bit uniform on [lo,hi)).
ImagePlane random_plane(int w, int h, std::uint64_t seed, double lo = 0.0, double hi = 255.0) {
    ImagePlane p(w, h);
    std::mt19937_64 rng(seed);
    for (double& v : p.samples()) v = lo + (hi - lo) * (static_cast<double>(rng() >> 11) * 0x1.0p-53);
    return p;
}

ImagePlane step(int w, int h, int edge, double lo, double hi) {
    ImagePlane p(w, h);
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) p(x, y) = x < edge ? lo : hi;
    return p;
}

ImagePlane checkerboard(int w, int h, int cell, double lo, double hi) {
    ImagePlane p(w, h);
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) p(x, y) = ((x / cell + y / cell) % 2 == 0) ? lo : hi;
    return p;
}

double max_abs_diff(const ImagePlane& a, const ImagePlane& b) {
    double m = 0.0;
    for (size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a.samples()[i] - b.samples()[i]));
    return m;
}

bool bit_equal(const ImagePlane& a, const ImagePlane& b) {
    return a.same_size(b) &&
           std::memcmp(a.samples().data(), b.samples().data(), a.size() * sizeof(double)) == 0;
}

ImagePlane checker_osbf(const ImagePlane& p, int r, int it) {
    ImagePlane out(p.width(), p.height());
    if (oracle_osbf(p.samples().data(), out.samples().data(), p.width(), p.height(), r, it) != 0)
        throw std::runtime_error("oracle failed");
    return out;
}

osbf::Volume random_volume(int w, int h, int d, std::uint64_t seed, double lo = 0.0,
                           double hi = 255.0) {
    osbf::Volume v(w, h, d);
    std::mt19937_64 rng(seed);
    for (double& s : v.samples()) s = lo + (hi - lo) * (static_cast<double>(rng() >> 11) * 0x1.0p-53);
    return v;
}

bool bit_equal(const osbf::Volume& a, const std::vector<double>& b) {
    return a.size() == b.size() && std::memcmp(a.samples().data(), b.data(), b.size() * sizeof(double)) == 0;
}

double max_abs_diff(const osbf::Volume& a, const osbf::Volume& b) {
    double m = 0.0;
    for (size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a.samples()[i] - b.samples()[i]));
    return m;
}

}  // namespace

int main() {
    // ---- core.hpp (test_core.cpp:95-114)
    run("sub-window geometry", [] {
        const int r = 3;
        const auto w = osbf::sub_windows(r);
        for (int i = 0; i < 8; ++i) {
            const auto& s = w[static_cast<size_t>(i)];
            if (s.id != i + 1 || s.u0 > 0 || s.u1 < 0 || s.v0 > 0 || s.v1 < 0) return false;
            const long long px = static_cast<long long>(s.u1 - s.u0 + 1) * (s.v1 - s.v0 + 1);
            if (px != (i < 4 ? (r + 1) * (r + 1) : (r + 1) * (2 * r + 1))) return false;
        }
        return throws<std::invalid_argument>([] { osbf::sub_windows(0); });
    });
    run("ImagePlane errors", [] {
        return throws<std::invalid_argument>([] { ImagePlane(0, 3); }) &&
               throws<std::out_of_range>([] { ImagePlane(2, 2).get(2, 0); });
    });

    // ---- integral.hpp (test_integral.cpp:19-29, 42-47, 80-89)
    run("summed-area table prefix sums", [] {
        const auto sat = osbf::build_sat(ImagePlane(2, 2, std::vector<double>{1, 2, 3, 4}));
        return sat.cumsum(0, 0) == 0.0 && sat.cumsum(2, 0) == 0.0 && sat.cumsum(0, 2) == 0.0 &&
               sat.cumsum(1, 1) == 1.0 && sat.cumsum(2, 1) == 3.0 && sat.cumsum(1, 2) == 4.0 &&
               sat.cumsum(2, 2) == 10.0;
    });
    run("SAT bit-identical to the reference order", [] {
        const auto p = random_plane(37, 23, 11);
        const auto sat = osbf::build_sat(p);
        std::vector<double> want(38 * 24);
        oracle_sat_build(p.samples().data(), 37, 23, want.data());
        for (int y = 0; y <= 23; ++y)
            for (int x = 0; x <= 37; ++x)
                if (sat.cumsum(x, y) != want[static_cast<size_t>(y) * 38 + x]) return false;
        return true;
    });
    run("rect_sum / rect_mean basics", [] {
        const auto ones = osbf::build_sat(ImagePlane(5, 5, 1.0));
        const auto c = osbf::build_sat(ImagePlane(6, 4, 3.25));
        const auto tiny = osbf::build_sat(ImagePlane(2, 1, std::vector<double>{0, 100}));
        return osbf::rect_sum(ones, 1, 1, 3, 3) == 9.0 && osbf::rect_sum(ones, 10, 10, 20, 20) == 0.0 &&
               osbf::rect_mean(c, 0, 0, 5, 3) == 3.25 && osbf::rect_mean(c, -3, -3, 2, 2) == 3.25 &&
               osbf::rect_mean(tiny, 0, 0, 1, 0) == 50.0 &&
               throws<std::domain_error>([&] { osbf::rect_mean(c, 10, 10, 12, 12); });
    });

    // ---- filters2d.hpp (test_filters2d.cpp)
    run("subwindow means on a constant plane", [] {
        const auto sat = osbf::build_sat(ImagePlane(10, 10, 7.25));
        for (double a : osbf::subwindow_means(sat, 4, 5, 2).a)
            if (a != 7.25) return false;
        return true;
    });
    run("left half window stays on the low side of a step", [] {
        const auto sat = osbf::build_sat(step(16, 16, 8, 0.0, 100.0));
        for (int r : {1, 2, 3})
            if (osbf::subwindow_means(sat, 7, 8, r).a[4] != 0.0) return false;
        return true;
    });
    for (osbf::gpu::Mode mode : {osbf::gpu::Mode::Exact, osbf::gpu::Mode::Fast}) {
        const std::string tag = mode == osbf::gpu::Mode::Exact ? " [exact]" : " [fast]";
        osbf::gpu::ScopedMode scoped(mode);
        run(("osbf_step keeps constant planes" + tag).c_str(), [] {
            const ImagePlane p(9, 9, 3.5);
            return max_abs_diff(osbf::osbf_step(p, 2), p) == 0.0;
        });
        run(("osbf_step keeps ideal vertical steps" + tag).c_str(), [] {
            for (int r : {1, 2, 5, 8}) {
                const auto p = step(32, 16, 16, 0.0, 100.0);
                if (max_abs_diff(osbf::osbf_step(p, r), p) != 0.0) return false;
            }
            return true;
        });
        run(("checkerboards with cell >= 2r are fixed points" + tag).c_str(), [] {
            for (int r : {1, 2, 3}) {
                const auto p = checkerboard(8 * r, 8 * r, 2 * r, 0.0, 255.0);
                const auto q = checkerboard(64, 64, 2 * r + 3, 10.0, 200.0);
                if (max_abs_diff(osbf::osbf_step(p, r), p) != 0.0) return false;
                if (max_abs_diff(osbf::osbf_step(q, r), q) != 0.0) return false;
            }
            return max_abs_diff(osbf::osbf_step(checkerboard(32, 32, 4, 0.0, 255.0), 3),
                                checkerboard(32, 32, 4, 0.0, 255.0)) > 1.0;
        });
        run(("step stays fixed for 30 iterations" + tag).c_str(), [] {
            const auto p = step(64, 32, 32, 0.0, 100.0);
            return max_abs_diff(osbf::osbf(p, 2, 30), p) == 0.0;
        });
        run(("zero iterations is the identity; argument errors" + tag).c_str(), [] {
            const auto p = random_plane(10, 10, 3);
            return bit_equal(osbf::osbf(p, 2, 0), p) && bit_equal(osbf::osbf(p, 0, 0), p) &&
                   throws<std::invalid_argument>([&] { osbf::osbf(p, 2, -1); }) &&
                   throws<std::invalid_argument>([&] { osbf::osbf(p, 0, 1); }) &&
                   throws<std::invalid_argument>([&] { osbf::osbf_step(p, 0); });
        });
        run(("range preservation" + tag).c_str(), [] {
            const auto p = random_plane(20, 20, 17, 10.0, 90.0);
            double lo = 1e300, hi = -1e300;
            for (double v : p.samples()) lo = std::min(lo, v), hi = std::max(hi, v);
            const auto out = osbf::osbf(p, 2, 5);
            for (double v : out.samples())
                if (v < lo || v > hi) return false;
            return true;
        });
        run(("filter_multichannel applies per channel" + tag).c_str(), [] {
            osbf::FilterConfig cfg;
            cfg.radius = 2;
            cfg.iterations = 2;
            const osbf::MultiChannelImage rgb(
                {random_plane(12, 12, 1), random_plane(12, 12, 2), random_plane(12, 12, 3)});
            const auto out = osbf::filter_multichannel(rgb, cfg);
            for (int c = 0; c < 3; ++c)
                if (!bit_equal(out.channel(c), osbf::osbf(rgb.channel(c), 2, 2))) return false;
            osbf::FilterConfig bad = cfg;
            bad.radius = 0;
            osbf::FilterConfig generic = cfg;
            generic.variant = osbf::FilterVariant::OneSidedGeneric;
            osbf::FilterConfig box = cfg;
            box.variant = osbf::FilterVariant::Box;
            const auto boxed = osbf::filter_multichannel(rgb, box);
            for (int c = 0; c < 3; ++c)
                if (!bit_equal(boxed.channel(c), osbf::box_filter(rgb.channel(c), 2, 2)))
                    return false;
            return throws<std::invalid_argument>([&] { osbf::filter_multichannel(rgb, bad); }) &&
                   throws<std::invalid_argument>([&] { osbf::filter_multichannel(rgb, generic); });
        });
        run(("outputs identical for any thread cap" + tag).c_str(), [] {
            const auto p = random_plane(33, 29, 123);
            osbf::set_max_threads(1);
            const auto a = osbf::osbf(p, 2, 2);
            osbf::set_max_threads(4);
            const auto b = osbf::osbf(p, 2, 2);
            osbf::set_max_threads(0);
            return bit_equal(a, b);
        });
    }
    run("osbf bit-identical to the oracle (24x24, r in {1,2,3,5}, 3 it) [exact]", [] {
        for (int r : {1, 2, 3, 5}) {
            const auto p = random_plane(24, 24, 200 + r);
            if (!bit_equal(osbf::osbf(p, r, 3), checker_osbf(p, r, 3))) return false;
        }
        return true;
    });
    run("osbf within 1e-9 of the oracle [fast]", [] {
        osbf::gpu::ScopedMode fast(osbf::gpu::Mode::Fast);
        for (int r : {1, 2, 3, 5}) {
            const auto p = random_plane(24, 24, 200 + r);
            if (max_abs_diff(osbf::osbf(p, r, 3), checker_osbf(p, r, 3)) > 1e-9) return false;
        }
        return true;
    });

    // ---- box_filter: test_filters2d.cpp:44-69 (fixed points, oracle, errors)
    run("box_filter bit-identical to the oracle; constant planes fixed; errors", [] {
        const ImagePlane c(9, 7, 3.25);
        for (int r : {1, 2, 5})
            if (max_abs_diff(osbf::box_filter(c, r, 3), c) != 0.0) return false;
        for (int r : {1, 2, 4, 9}) {
            const auto p = random_plane(33, 21, 400 + r);
            std::vector<double> want(p.size());
            if (oracle_box_filter(p.samples().data(), want.data(), 33, 21, r, 3) != 0) return false;
            const auto got = osbf::box_filter(p, r, 3);
            if (std::memcmp(got.samples().data(), want.data(), sizeof(double) * want.size()) != 0)
                return false;
        }
        const auto p = random_plane(8, 8, 2);
        return bit_equal(osbf::box_filter(p, 2, 0), p) &&
               throws<std::invalid_argument>([&] { osbf::box_filter(p, 0, 0); }) &&
               throws<std::invalid_argument>([&] { osbf::box_filter(p, 2, -1); });
    });

    // ---- parallel.hpp: parallel_for_rows covers [0, count) in disjoint blocks
    run("parallel_for_rows covers every row once for any thread cap", [] {
        for (int cap : {0, 1, 3, 64}) {
            osbf::set_max_threads(cap);
            for (int count : {0, 1, 7, 100}) {
                std::vector<std::atomic<int>> hits(static_cast<size_t>(count));
                osbf::parallel_for_rows(count, [&](int b, int e) {
                    for (int i = b; i < e; ++i) hits[static_cast<size_t>(i)]++;
                });
                for (auto& h : hits)
                    if (h.load() != 1) return false;
            }
        }
        osbf::set_max_threads(0);
        return true;
    });

    // ---- fast_osbf (paper Algorithm 3): test_filters2d.cpp:169-186 + errors
    run("fast_osbf keeps constant planes and ideal steps", [] {
        const ImagePlane c(9, 9, 11.0);
        if (max_abs_diff(osbf::fast_osbf(c, 3, 2), c) != 0.0) return false;
        for (int r : {1, 2, 5}) {
            const auto p = step(32, 16, 16, 0.0, 100.0);
            if (max_abs_diff(osbf::fast_osbf(p, r, 1), p) != 0.0) return false;
        }
        return true;
    });
    run("fast_osbf bit-identical to the oracle; errors as the reference", [] {
        for (int r : {1, 2, 3, 7}) {
            const auto p = random_plane(41, 27, 300 + r);
            std::vector<double> want(p.size());
            if (oracle_fast_osbf(p.samples().data(), want.data(), 41, 27, r, 4) != 0) return false;
            const auto got = osbf::fast_osbf(p, r, 4);
            if (std::memcmp(got.samples().data(), want.data(), sizeof(double) * want.size()) != 0)
                return false;
        }
        const auto p = random_plane(8, 8, 1);
        osbf::FilterConfig cfg;
        cfg.radius = 2;
        cfg.iterations = 3;
        cfg.variant = osbf::FilterVariant::OsbfFast;
        const osbf::MultiChannelImage rgb({random_plane(12, 10, 4), random_plane(12, 10, 5)});
        const auto out = osbf::filter_multichannel(rgb, cfg);
        for (int c = 0; c < 2; ++c)
            if (!bit_equal(out.channel(c), osbf::fast_osbf(rgb.channel(c), 2, 3))) return false;
        return throws<std::invalid_argument>([&] { osbf::fast_osbf(p, 0, 0); }) &&
               throws<std::invalid_argument>([&] { osbf::fast_osbf(p, 2, -1); }) &&
               bit_equal(osbf::fast_osbf(p, 2, 0), p);
    });

    // ---- acceptance.cpp criteria 1, 2, 5
    run("acceptance 1: edge fixed point (256^2, r in {1,2,5,10}, 30 it)", [] {
        double worst = 0.0;
        for (int r : {1, 2, 5, 10}) {
            const auto p = step(256, 256, 128, 100.0, 200.0);
            worst = std::max(worst, max_abs_diff(osbf::osbf(p, r, 30), p));
        }
        return worst <= 1e-6;
    });
    run("acceptance 2: corner fixed point (cell 32, r 1..10)", [] {
        const auto board = checkerboard(256, 256, 32, 0.0, 255.0);
        double worst = 0.0;
        for (int r = 1; r <= 10; ++r) worst = std::max(worst, max_abs_diff(osbf::osbf(board, r, 1), board));
        return worst <= 1e-6;
    });
    run("acceptance 5: 50 planes 64x64, r in {1,2,3,5}, 3 it, bit-identical to the oracle", [] {
        for (int k = 0; k < 50; ++k) {
            const auto p = random_plane(64, 64, 1000 + k);
            for (int r : {1, 2, 3, 5})
                if (!bit_equal(osbf::osbf(p, r, 3), checker_osbf(p, r, 3))) return false;
        }
        return true;
    });

    // ---- 3-D extension: test_core.cpp:73-78, test_integral.cpp:101-129,
    //      test_filters3d.cpp:32-117
    run("Volume extents, accessors and errors", [] {
        osbf::Volume v(2, 3, 2, 0.0);
        v.set(1, 2, 1, 5.0);
        return v.size() == 12 && v(1, 2, 1) == 5.0 && v.get(1, 2, 1) == 5.0 &&
               v.samples()[(1 * 3 + 2) * 2 + 1] == 5.0 &&
               throws<std::out_of_range>([&] { v.get(2, 0, 0); }) &&
               throws<std::invalid_argument>([] { osbf::Volume(0, 1, 1); }) &&
               throws<std::invalid_argument>([] { osbf::Volume(2, 2, 2, std::vector<double>(7)); });
    });
    run("SummedVolumeTable (GPU-built) bit-identical to the oracle; box lookups", [] {
        const auto ones = osbf::build_svt(osbf::Volume(4, 4, 4, 1.0));
        if (osbf::box_sum_3d(ones, {0, 0, 0, 3, 3, 3}) != 64.0 ||
            osbf::box_sum_3d(ones, {-5, -5, -5, 10, 10, 10}) != 64.0)
            return false;
        osbf::Volume v(3, 3, 3, 0.0);
        v(1, 2, 1) = 42.0;
        const auto sv = osbf::build_svt(v);
        if (osbf::box_sum_3d(sv, {1, 2, 1, 1, 2, 1}) != 42.0 ||
            osbf::box_mean_3d(sv, {1, 2, 1, 1, 2, 1}) != 42.0)
            return false;
        if (!throws<std::domain_error>([&] { osbf::box_mean_3d(sv, {5, 5, 5, 9, 9, 9}); })) return false;
        const std::array<std::array<int, 3>, 3> shapes{{{8, 8, 8}, {13, 5, 9}, {1, 17, 3}}};
        for (const auto& [w, h, d] : shapes) {
            const auto rv = random_volume(w, h, d, 61 + w);
            std::vector<double> want(static_cast<size_t>(w + 1) * (h + 1) * (d + 1));
            oracle_svt_build(rv.samples().data(), w, h, d, want.data());
            const osbf::SummedVolumeTable svt(rv);
            for (int z = 0; z <= d; ++z)
                for (int y = 0; y <= h; ++y)
                    for (int x = 0; x <= w; ++x) {
                        const double g = svt.cumsum(x, y, z);
                        const double e = want[(static_cast<size_t>(z) * (h + 1) + y) * (w + 1) + x];
                        if (std::memcmp(&g, &e, sizeof(double)) != 0) return false;
                    }
        }
        return true;
    });
    run("sub_regions_3d: ids, one-sided extents, voxel counts", [] {
        const int r = 2;
        const auto regions = osbf::sub_regions_3d(r);
        for (int i = 0; i < 14; ++i) {
            const auto& g = regions[static_cast<size_t>(i)];
            if (g.id != i + 1 || g.u0 > 0 || g.u1 < 0 || g.v0 > 0 || g.v1 < 0 || g.w0 > 0 || g.w1 < 0)
                return false;
            const long long n = static_cast<long long>(g.u1 - g.u0 + 1) * (g.v1 - g.v0 + 1) * (g.w1 - g.w0 + 1);
            if (n != (i < 8 ? 27LL : 75LL)) return false;
        }
        return throws<std::invalid_argument>([] { osbf::sub_regions_3d(0); });
    });
    run("box_filter_3d / osbf_3d bit-identical to the oracle; fixed points; errors", [] {
        const osbf::Volume c(6, 6, 6, 4.0);
        if (max_abs_diff(osbf::box_filter_3d(c, 2, 3), c) != 0.0 ||
            max_abs_diff(osbf::osbf_3d(c, 2, 2), c) != 0.0)
            return false;
        for (int r : {1, 2, 3}) {
            const auto v = random_volume(11, 9, 7, 62 + r);
            std::vector<double> want(v.size());
            if (oracle_box_filter_3d(v.samples().data(), want.data(), 11, 9, 7, r, 2) != 0 ||
                !bit_equal(osbf::box_filter_3d(v, r, 2), want))
                return false;
            if (oracle_osbf_3d(v.samples().data(), want.data(), 11, 9, 7, r, 2) != 0 ||
                !bit_equal(osbf::osbf_3d(v, r, 2), want))
                return false;
        }
        // axis steps stay fixed (test_filters3d.cpp:80-100)
        osbf::Volume sx(16, 8, 8, 0.0), sy(8, 16, 8, 0.0), sz(8, 8, 16, 0.0);
        for (int z = 0; z < 8; ++z)
            for (int y = 0; y < 8; ++y)
                for (int x = 0; x < 16; ++x) {
                    sx(x, y, z) = x < 8 ? 0.0 : 100.0;
                    sy(y, x, z) = x < 8 ? 0.0 : 100.0;
                    sz(y, z, x) = x < 8 ? 0.0 : 100.0;
                }
        const std::array<const osbf::Volume*, 3> steps{&sx, &sy, &sz};
        for (const auto* s : steps)
            if (max_abs_diff(osbf::osbf_3d(*s, 2, 1), *s) != 0.0) return false;
        const auto v = random_volume(10, 10, 10, 63, 5.0, 50.0);
        const auto filtered = osbf::osbf_3d(v, 2, 3);
        for (double s : filtered.samples())
            if (s < 5.0 || s > 50.0) return false;
        return max_abs_diff(osbf::osbf_3d(v, 2, 0), v) == 0.0 &&
               throws<std::invalid_argument>([&] { osbf::osbf_3d(v, 0, 1); }) &&
               throws<std::invalid_argument>([&] { osbf::box_filter_3d(v, 1, -1); });
    });

    // ---- smooth edge: test_cli.cpp:97-114 through smooth_file, and the
    //      GPU raster path against the oracle restatement
    run("smooth_file keeps a step bit-identical; zero iterations copy; errors", [] {
        const std::string dir = std::filesystem::temp_directory_path().string();
        const std::string in = dir + "/osbf_dropin_step.pgm", out = dir + "/osbf_dropin_out.pgm";
        osbf::gpu::Raster step;
        step.width = step.height = 64;
        step.u8.resize(64 * 64);
        for (int y = 0; y < 64; ++y)
            for (int x = 0; x < 64; ++x) step.u8[static_cast<size_t>(y) * 64 + x] = x < 32 ? 0 : 100;
        osbf::gpu::write_raster(step, in);
        osbf::FilterConfig cfg;  // osbf, r=2, 10 iterations (the CLI defaults)
        osbf::gpu::smooth_file(in, out, cfg);
        if (osbf::gpu::read_raster(out).u8 != step.u8) return false;
        cfg.variant = osbf::FilterVariant::Box;
        cfg.iterations = 0;
        osbf::gpu::smooth_file(in, out, cfg);
        const auto back = osbf::gpu::read_raster(out);
        std::filesystem::remove(in);
        std::filesystem::remove(out);
        cfg.variant = osbf::FilterVariant::Gaussian;
        return back.u8 == step.u8 && back.maxval == 255 &&
               throws<std::invalid_argument>([&] { osbf::gpu::smooth(step, cfg); }) &&
               throws<osbf::gpu::ParseError>([&] { osbf::gpu::read_raster(in + ".missing.pgm"); }) ==
                   false;
    });
    run("smooth (GPU promote/filter/quantise) byte-identical to the oracle; u8 RGB and u16", [] {
        std::mt19937_64 rng(81);
        for (int wide = 0; wide < 2; ++wide)
            for (int f = 0; f < 3; ++f) {
                osbf::gpu::Raster r;
                r.width = 45;
                r.height = 31;
                r.channels = wide ? 1 : 3;
                r.maxval = wide ? 65535 : 255;
                const size_t n = r.sample_count();
                if (wide) {
                    r.u16.resize(n);
                    for (auto& v : r.u16) v = static_cast<uint16_t>(rng() >> 48);
                } else {
                    r.u8.resize(n);
                    for (auto& v : r.u8) v = static_cast<uint8_t>(rng() >> 56);
                }
                osbf::FilterConfig cfg;
                cfg.radius = 2 + f;
                cfg.iterations = 3;
                cfg.variant = f == 0 ? osbf::FilterVariant::OsbfExact
                              : f == 1 ? osbf::FilterVariant::OsbfFast
                                       : osbf::FilterVariant::Box;
                const auto got = osbf::gpu::smooth(r, cfg);
                std::vector<uint16_t> want16(n);
                std::vector<uint8_t> want8(n);
                const void* src = wide ? static_cast<const void*>(r.u16.data()) : r.u8.data();
                void* dst = wide ? static_cast<void*>(want16.data()) : want8.data();
                if (oracle_smooth_raster(src, wide ? 2 : 1, r.channels, r.width, r.height, f,
                                         cfg.radius, cfg.iterations, dst, wide ? 2 : 1) != 0)
                    return false;
                if (wide ? got.u16 != want16 : got.u8 != want8) return false;
            }
        return true;
    });
    run("read_raster: netpbm header rules and errors as read_image", [] {
        const std::string p = std::filesystem::temp_directory_path().string() + "/osbf_dropin.pnm";
        auto put = [&](const std::string& bytes) {
            std::ofstream(p, std::ios::binary) << bytes;
        };
        put("P2\n# comment\n3 1 # more\n9\n0 4 9\n");
        const auto a = osbf::gpu::read_raster(p);
        if (a.width != 3 || a.u8 != std::vector<uint8_t>{0, 4, 9}) return false;
        put(std::string("P5\n2 1\n65535\n") + std::string("\x01\x02\xff\xfe", 4));
        const auto b = osbf::gpu::read_raster(p);
        if (b.u16 != std::vector<uint16_t>{0x0102, 0xfffe}) return false;
        bool ok = true;
        for (const char* bad : {"P7\n1 1\n255\n", "P5\n0 1\n255\n", "P5\n1 1\n70000\n",
                                "P5\n2 2\n255\nab", "P2\n1 1\n5\n6\n", "P2\n1 1\n"})
            ok = ok && (put(bad), throws<osbf::gpu::ParseError>([&] { osbf::gpu::read_raster(p); }));
        std::filesystem::remove(p);
        return ok;
    });

    std::printf("%d failure(s)\n", failures);
    return failures;
}
