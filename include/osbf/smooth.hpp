// The `osbf smooth` edge on the GPU: the reference's
// cmd_smooth (tools/osbf_main.cpp:63-83) is
//     read_image (io.hpp:119-178)  -> samples promoted to fp64 on the host
//     filter_multichannel          -> filters2d.hpp:371-400
//     write_image (io.hpp:183-215) -> quantize (io.hpp:108-115), P5/P6 out
// Here the decoded samples stay uint8/uint16 until they reach the GPU, which
// promotes, filters and quantises them (osbf_gpu_smooth_raster_host), so a
// raster crosses PCIe as 1-2 B per sample instead of 8.  The netpbm parse
// follows read_image's rules (P2/P3/P5/P6, comments anywhere in the header,
// maxval in [1, 65535], big-endian 16-bit payloads, one whitespace byte
// before a binary payload, samples <= maxval) with its messages; the output
// is write_image's (P5/P6, 8 bits when maxval <= 255 else 16, written to
// path.tmp then renamed).  Everything lives in osbf::gpu so it can sit next to
// the reference's own io.hpp.
#pragma once

#include <cctype>
#include <climits>
#include <cstdint>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <stdexcept>
#include <string>
#include <vector>

#include "osbf/core.hpp"
#include "osbf/gpu_runtime.hpp"

namespace osbf::gpu {

/// Malformed netpbm input; `offset` is where parsing stopped (io.hpp ParseError).
class ParseError : public std::runtime_error {
public:
    ParseError(const std::string& message, size_t offset)
        : std::runtime_error(message + " (byte offset " + std::to_string(offset) + ")"),
          offset_(offset) {}
    size_t offset() const { return offset_; }

private:
    size_t offset_;
};

/// Decoded PGM/PPM samples, interleaved, not promoted: `u8` when maxval <= 255,
/// `u16` otherwise.
struct Raster {
    int width = 0, height = 0, channels = 1, maxval = 255;
    std::vector<uint8_t> u8;
    std::vector<uint16_t> u16;

    bool wide() const { return maxval > 255; }
    size_t sample_count() const { return static_cast<size_t>(width) * height * channels; }
};

namespace detail {

class NetpbmHeader {
public:
    NetpbmHeader(const std::string& d, size_t pos) : d_(d), pos_(pos) {}
    size_t pos() const { return pos_; }

    static bool space(char c) {
        return c == ' ' || c == '\t' || c == '\r' || c == '\n' || c == '\v' || c == '\f';
    }

    long number(const char* what) {
        for (;;) {  // whitespace and '#' comments may appear before any field
            if (pos_ < d_.size() && space(d_[pos_])) {
                ++pos_;
            } else if (pos_ < d_.size() && d_[pos_] == '#') {
                while (pos_ < d_.size() && d_[pos_] != '\n') ++pos_;
            } else {
                break;
            }
        }
        const size_t start = pos_;
        long v = 0;
        bool overflow = false;
        while (pos_ < d_.size() && std::isdigit(static_cast<unsigned char>(d_[pos_]))) {
            if (v > (LONG_MAX - 9) / 10) overflow = true;
            if (!overflow) v = v * 10 + (d_[pos_] - '0');
            ++pos_;
        }
        if (pos_ == start) throw ParseError(std::string("expected ") + what, start);
        if (overflow) throw ParseError(std::string("unparsable ") + what, start);
        return v;
    }

    void single_space(const char* what) {
        if (pos_ >= d_.size() || !space(d_[pos_]))
            throw ParseError(std::string("expected whitespace before ") + what, pos_);
        ++pos_;
    }

private:
    const std::string& d_;
    size_t pos_;
};

inline std::string slurp(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open file: " + path);
    std::string data((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    if (in.bad()) throw std::runtime_error("read failed: " + path);
    return data;
}

}  // namespace detail

/// read_image (io.hpp:119-178) without the promotion to fp64.
inline Raster read_raster(const std::string& path) {
    const std::string data = detail::slurp(path);
    const char kind = data.size() >= 2 && data[0] == 'P' ? data[1] : '\0';
    if (kind != '2' && kind != '3' && kind != '5' && kind != '6')
        throw ParseError("unknown magic, expected P2/P3/P5/P6", 0);
    Raster r;
    r.channels = (kind == '3' || kind == '6') ? 3 : 1;
    detail::NetpbmHeader hdr(data, 2);
    const long w = hdr.number("width");
    const long h = hdr.number("height");
    if (w < 1 || h < 1) throw ParseError("image dimensions must be >= 1", hdr.pos());
    const long maxval = hdr.number("maxval");
    if (maxval < 1 || maxval > 65535) throw ParseError("maxval out of range [1, 65535]", hdr.pos());
    r.width = static_cast<int>(w);
    r.height = static_cast<int>(h);
    r.maxval = static_cast<int>(maxval);
    const size_t n = r.sample_count();
    (r.wide() ? r.u16.resize(n) : r.u8.resize(n));
    auto put = [&](size_t i, unsigned v, size_t at) {
        if (v > static_cast<unsigned>(maxval)) throw ParseError("sample exceeds maxval", at);
        if (r.wide())
            r.u16[i] = static_cast<uint16_t>(v);
        else
            r.u8[i] = static_cast<uint8_t>(v);
    };
    if (kind == '5' || kind == '6') {
        hdr.single_space("payload");
        const size_t per = r.wide() ? 2 : 1, need = n * per, have = data.size() - hdr.pos();
        if (have < need)
            throw ParseError("truncated payload: expected " + std::to_string(need) +
                                 " bytes, got " + std::to_string(have),
                             hdr.pos());
        const auto* p = reinterpret_cast<const unsigned char*>(data.data()) + hdr.pos();
        for (size_t i = 0; i < n; ++i)
            put(i, per == 1 ? p[i] : (static_cast<unsigned>(p[2 * i]) << 8 | p[2 * i + 1]),
                hdr.pos());
    } else {
        for (size_t i = 0; i < n; ++i) {
            const size_t at = hdr.pos();
            const long v = hdr.number("sample");
            put(i, v > 65535 ? 65536u : static_cast<unsigned>(v), at);
        }
    }
    return r;
}

/// write_image (io.hpp:183-215) for an already quantised raster: P5/P6 with
/// maxval 255 (u8) or 65535 (u16), 16-bit big-endian, temp file + rename.
inline void write_raster(const Raster& r, const std::string& path) {
    if (r.channels != 1 && r.channels != 3)
        throw std::invalid_argument("write_image: only 1- or 3-channel images can be saved");
    const int maxval = r.wide() ? 65535 : 255;
    std::string out = (r.channels == 1 ? "P5\n" : "P6\n") + std::to_string(r.width) + " " +
                      std::to_string(r.height) + "\n" + std::to_string(maxval) + "\n";
    const size_t n = r.sample_count();
    if (r.wide()) {
        for (size_t i = 0; i < n; ++i) {
            out += static_cast<char>(r.u16[i] >> 8);
            out += static_cast<char>(r.u16[i] & 0xff);
        }
    } else {
        out.append(reinterpret_cast<const char*>(r.u8.data()), n);
    }
    const std::string tmp = path + ".tmp";
    {
        std::ofstream f(tmp, std::ios::binary | std::ios::trunc);
        if (!f) throw std::runtime_error("cannot open file for writing: " + tmp);
        f.write(out.data(), static_cast<std::streamsize>(out.size()));
        f.flush();
        if (!f) throw std::runtime_error("write failed: " + tmp);
    }
    std::filesystem::rename(tmp, path);
}

/// filter_multichannel + write_image's quantisation on the GPU; the result
/// has maxval 255 when in.maxval <= 255, else 65535 (cmd_smooth's bit depth).
/// Variants: OsbfExact (honours osbf::gpu::set_mode), OsbfFast, Box.
inline Raster smooth(const Raster& in, const FilterConfig& cfg) {
    cfg.validate();
    osbf_filter f;
    switch (cfg.variant) {
        case FilterVariant::OsbfExact: f = OSBF_FILTER_OSBF; break;
        case FilterVariant::OsbfFast: f = OSBF_FILTER_FAST_OSBF; break;
        case FilterVariant::Box: f = OSBF_FILTER_BOX; break;
        default:
            throw std::invalid_argument(
                "smooth: only the osbf, fast-osbf and box filters run on the GPU");
    }
    Raster out;
    out.width = in.width;
    out.height = in.height;
    out.channels = in.channels;
    out.maxval = in.wide() ? 65535 : 255;
    (out.wide() ? out.u16.resize(in.sample_count()) : out.u8.resize(in.sample_count()));
    const void* src = in.wide() ? static_cast<const void*>(in.u16.data()) : in.u8.data();
    void* dst = out.wide() ? static_cast<void*>(out.u16.data()) : out.u8.data();
    detail::check(osbf_gpu_smooth_raster_host(detail::context(), src, in.wide() ? 2 : 1,
                                              in.channels, in.width, in.height, f, cfg.radius,
                                              cfg.iterations, static_cast<osbf_mode>(mode()), dst,
                                              out.wide() ? 2 : 1));
    return out;
}

/// cmd_smooth (tools/osbf_main.cpp:63-83) minus the timing printout.
inline void smooth_file(const std::string& in_path, const std::string& out_path,
                        const FilterConfig& cfg) {
    write_raster(smooth(read_raster(in_path), cfg), out_path);
}

}  // namespace osbf::gpu
