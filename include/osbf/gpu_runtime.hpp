// Glue between the drop-in C++ API and libosbf_gpu.so (include/osbf_gpu.h):
// one context per thread, the path's arithmetic mode, and the mapping of
// osbf_status codes back onto the reference's exception types.
#pragma once

#include <stdexcept>
#include <string>

#include "osbf_gpu.h"

namespace osbf {
namespace gpu {

enum class Mode {
    Exact = OSBF_MODE_EXACT,  // bit-identical to the reference (default)
    Fast = OSBF_MODE_FAST,    // tile-local sums, within a few fp64 ulps per pass
};

namespace detail {

inline Mode& mode_ref() {
    thread_local Mode m = Mode::Exact;
    return m;
}

[[noreturn]] inline void raise(osbf_status st) {
    const std::string msg = osbf_gpu_last_error();
    switch (st) {
        case OSBF_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case OSBF_ERR_DOMAIN: throw std::domain_error(msg);
        case OSBF_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
        default: throw std::runtime_error("osbf GPU: " + msg);
    }
}

inline void check(osbf_status st) {
    if (st != OSBF_OK) raise(st);
}

class Context {
public:
    Context() { check(osbf_gpu_ctx_create(0, &ctx_)); }
    ~Context() { osbf_gpu_ctx_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    osbf_ctx* get() const { return ctx_; }

private:
    osbf_ctx* ctx_ = nullptr;
};

inline osbf_ctx* context() {
    thread_local Context ctx;
    return ctx.get();
}

}  // namespace detail

/// Arithmetic mode of this thread's osbf()/osbf_step()/filter_multichannel().
inline void set_mode(Mode m) { detail::mode_ref() = m; }
inline Mode mode() { return detail::mode_ref(); }

/// RAII mode switch.
class ScopedMode {
public:
    explicit ScopedMode(Mode m) : prev_(mode()) { set_mode(m); }
    ~ScopedMode() { set_mode(prev_); }

private:
    Mode prev_;
};

}  // namespace gpu
}  // namespace osbf
