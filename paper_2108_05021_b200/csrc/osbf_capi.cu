// C ABI of libosbf_gpu.so (include/osbf_gpu.h): contexts, argument validation
// with the reference's error behaviour, the Jacobi iteration driver and the
// host-buffer entry points used by the drop-in C++ headers.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "osbf_internal.cuh"

namespace {

thread_local std::string g_last_error;
thread_local const char* g_last_kernel = "";

osbf_status fail(osbf_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return st;
}

osbf_status cuda_fail(cudaError_t e, const char* where) {
    return fail(e == cudaErrorMemoryAllocation ? OSBF_ERR_ALLOC : OSBF_ERR_CUDA, "%s: %s (%s)",
                where, cudaGetErrorString(e), cudaGetErrorName(e));
}

#define OSBF_CUDA(call, where)                         \
    do {                                               \
        cudaError_t e_ = (call);                       \
        if (e_ != cudaSuccess) return cuda_fail(e_, where); \
    } while (0)

size_t dtype_size(osbf_dtype d) {
    switch (d) {
        case OSBF_U8: return 1;
        case OSBF_F32: return 4;
        default: return 8;
    }
}

// Grow-only device buffer.
struct DevBuf {
    void* ptr = nullptr;
    size_t bytes = 0;
    cudaError_t ensure(size_t need) {
        if (need <= bytes) return cudaSuccess;
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        bytes = 0;
        cudaError_t e = cudaMalloc(&ptr, need);
        if (e == cudaSuccess) bytes = need;
        return e;
    }
    void release() {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        bytes = 0;
    }
    template <typename T>
    T* as() const { return static_cast<T*>(ptr); }
};

}  // namespace

// One captured launch sequence (a whole multi-pass call) and what it was
// captured for: every argument and every scratch buffer it touches.
struct GraphEntry {
    std::vector<uintptr_t> key;
    cudaGraphExec_t exec = nullptr;
    uint64_t launches = 0;  // kernels inside the graph (for the launch counter)
    const char* kernel = "";  // kernel family of its last pass (osbf_gpu_last_kernel)
    int state = 0;          // 0 seen once (ran plain), 1 captured, -1 never capture
};

struct osbf_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    DevBuf ping, pong;         // fp64 Jacobi planes
    DevBuf rowpfx, sat;        // exact-mode workspace
    DevBuf host_in, host_out;  // staging for the host entry points
    osbf_gpu::LaunchCounter lc;
    int passes_per_launch = 1;  // fast mode temporal blocking: 1..4 passes per launch
    cudaStream_t copy_in = nullptr, copy_out = nullptr;  // host entry points: copy overlap
    cudaStream_t capture = nullptr;                      // CUDA-graph capture stream
    std::vector<GraphEntry> graphs;                      // small LRU of replayable calls
    // Scratch ordering across caller streams: the stream the last device call
    // ran on, and an event recorded on it when a call switches streams.
    cudaStream_t last_stream = nullptr;
    bool have_last = false;
    cudaEvent_t switch_ev = nullptr;
    void drop_graphs() {
        for (auto& gph : graphs)
            if (gph.exec) cudaGraphExecDestroy(gph.exec);
        graphs.clear();
    }
};

namespace {

int device_ok_cached = -1;
std::mutex device_mu;

bool device_ok() {
    std::lock_guard<std::mutex> lock(device_mu);
    if (device_ok_cached >= 0) return device_ok_cached == 1;
    int n = 0;
    device_ok_cached = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n < 1) {
        cudaGetLastError();
        return false;
    }
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, 0) == cudaSuccess && prop.major == 10) device_ok_cached = 1;
    return device_ok_cached == 1;
}

osbf_status check_geometry(int width, int height, int batch) {
    if (width < 1 || height < 1)
        return fail(OSBF_ERR_INVALID_ARGUMENT, "ImagePlane: dimensions must be >= 1");
    if (batch < 1) return fail(OSBF_ERR_INVALID_ARGUMENT, "batch must be >= 1");
    // the kernels put the plane index in gridDim.z
    if (batch > 65535)
        return fail(OSBF_ERR_INVALID_ARGUMENT, "batch must be <= 65535 planes per call (got %d)",
                    batch);
    return OSBF_OK;
}

osbf_status check_dtype(osbf_dtype d) {
    if (d != OSBF_U8 && d != OSBF_F32 && d != OSBF_F64)
        return fail(OSBF_ERR_INVALID_ARGUMENT, "unknown dtype %d", static_cast<int>(d));
    return OSBF_OK;
}

osbf_status check_mode(osbf_mode m) {
    if (m != OSBF_MODE_EXACT && m != OSBF_MODE_FAST)
        return fail(OSBF_ERR_INVALID_ARGUMENT, "unknown mode %d", static_cast<int>(m));
    return OSBF_OK;
}

// NULL is the CUDA default stream (standard cudaStream_t semantics), so work
// is ordered with e.g. PyTorch's default stream.  The context's own stream is
// used only by the host-buffer entry points.
//
// The context's scratch (ping/pong planes, exact-mode workspace, graphs) is
// shared by every call, so calls issued on different streams must not
// overlap: when a call arrives on a stream other than the previous call's,
// the new stream first waits for everything already enqueued on the old one.
cudaStream_t pick_stream(osbf_ctx* ctx, void* stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (ctx->have_last && ctx->last_stream != s) {
        if (!ctx->switch_ev) cudaEventCreateWithFlags(&ctx->switch_ev, cudaEventDisableTiming);
        if (ctx->switch_ev && cudaEventRecord(ctx->switch_ev, ctx->last_stream) == cudaSuccess)
            cudaStreamWaitEvent(s, ctx->switch_ev, 0);
        else
            cudaGetLastError();  // old stream gone: its work was synchronized by its owner
    }
    ctx->last_stream = s;
    ctx->have_last = true;
    return s;
}

// Temporal blocking (k fast passes per launch, k = 2..4) is opt-in per
// context (osbf_gpu_ctx_set_temporal_blocking) or process-wide with
// OSBF_GPU_TB=k (OSBF_GPU_TB2=1 = k 2).
int tb_env() {
    static const int k = [] {
        const char* v = std::getenv("OSBF_GPU_TB");
        if (v && v[0] >= '2' && v[0] <= '4' && v[1] == 0) return v[0] - '0';
        const char* v2 = std::getenv("OSBF_GPU_TB2");
        return (v2 && v2[0] == '1') ? 2 : 1;
    }();
    return k;
}

// The exact-pass family forced by osbf_gpu_set_exact_kernel or OSBF_GPU_EXACT
// ("strip": the fused strip walk whenever its radius allows; "twalk" /
// "gwalk" / "stencil": that stencil on the whole-table path) -- A/B runs and
// tests of the kernels a launch would not pick by default.
bool exact_strip_forced() {
    const char* o = osbf_gpu::exact_kernel_override();
    return o && std::strcmp(o, "strip") == 0;
}

// The fast-pass family forced by osbf_gpu_set_fast_kernel or OSBF_GPU_FAST.
bool fast_family_forced(const char* name) {
    const char* o = osbf_gpu::fast_kernel_override();
    if (!o) {
        static const char* env = [] {
            const char* e = std::getenv("OSBF_GPU_FAST");
            return e ? e : "";
        }();
        o = env;
    }
    return std::strcmp(o, name) == 0;
}

// One pass in the requested mode: src (typed view) -> dst (fp64).
osbf_status one_pass(osbf_ctx* ctx, const osbf_gpu::PlaneView& src, const osbf_gpu::Geometry& g,
                     int r, double* dst, size_t dp, size_t dpl, double* means, uint8_t* sel,
                     osbf_mode mode, cudaStream_t s) {
    // Fast mode: templated kernels up to kFastMaxRadius, the generic
    // vertical-first walk above it (up to fast_generic_max_radius()); beyond
    // that, or for the per-pixel diagnostics, the exact GPU kernels
    // (bit-identical to the reference, hence also within the fast mode's
    // tolerance), like the reference accepts any r.
    if (mode == OSBF_MODE_FAST && r > osbf_gpu::kFastMaxRadius) {
        // Whole planes above the templated radii run the exact table path: it
        // is bit-identical to the reference (so within fast mode's tolerance),
        // its cost does not grow with r, and since the strip table builder and
        // the generic stencil walk it is faster than the generic fast walk at
        // every r > 16 (32768^2: 14.1 vs 14.9 ms per pass at r = 17, 14.6 vs
        // 22.3 at r = 32; profiles/r02_exact_paths.jsonl).  The generic walk
        // (osbf_fast_vwalk.cu) serves row bands, which the table path cannot
        // split, a table workspace that cannot be allocated, and
        // OSBF_GPU_FAST / osbf_gpu_set_fast_kernel "vwalk".
        bool walk = fast_family_forced("vwalk");
        if (!walk && dst && !means && !sel && r <= osbf_gpu::fast_generic_max_radius()) {
            const size_t n = static_cast<size_t>(g.batch) * g.width * g.height;
            const size_t tp = (static_cast<size_t>(g.width) + 2) & ~static_cast<size_t>(1);
            const size_t ns = static_cast<size_t>(g.batch) * tp * (g.height + 1);
            if (ctx->rowpfx.ensure(n * sizeof(double)) != cudaSuccess ||
                ctx->sat.ensure((ns + 2) * sizeof(double)) != cudaSuccess) {
                (void)cudaGetLastError();
                walk = true;
            }
        }
        if (walk && dst && !means && !sel && r <= osbf_gpu::fast_generic_max_radius()) {
            const cudaError_t e =
                osbf_gpu::fast_generic_step(src, g, r, dst, dp, dpl, s, ctx->lc);
            if (e != cudaErrorNotSupported) {
                OSBF_CUDA(e, "fast generic step");
                return OSBF_OK;
            }
        }
        mode = OSBF_MODE_EXACT;
    }
    // Exact mode runs the whole-table path (serial-order table build + the
    // stencil walk: measured faster than the fused strip walk on every shape,
    // profiles/r02_exact_paths.jsonl).  The fused strip walk (same bits, r <=
    // 16) needs no table workspace: it serves when that workspace (two fp64
    // planes) cannot be allocated, or when forced.
    bool fused = false;
    if (mode == OSBF_MODE_EXACT && dst && !means && !sel && r <= osbf_gpu::kExactFusedMaxRadius) {
        fused = exact_strip_forced();
        if (!fused) {
            const size_t n = static_cast<size_t>(g.batch) * g.width * g.height;
            const size_t tp = (static_cast<size_t>(g.width) + 2) & ~static_cast<size_t>(1);
            const size_t ns = static_cast<size_t>(g.batch) * tp * (g.height + 1);
            if (ctx->rowpfx.ensure(n * sizeof(double)) != cudaSuccess ||
                ctx->sat.ensure((ns + 2) * sizeof(double)) != cudaSuccess) {
                (void)cudaGetLastError();  // out of memory for the table: not an error yet
                fused = true;
            }
        }
    }
    if (fused) {
        // fused exact path: row carries + strip kernel (same bits as below)
        OSBF_CUDA(ctx->rowpfx.ensure(osbf_gpu::exact_fused_carry_elems(g) * sizeof(double)),
                  "alloc carries");
        OSBF_CUDA(osbf_gpu::exact_fused_step(src, g, r, ctx->rowpfx.as<double>(), dst, dp, dpl, s,
                                             ctx->lc),
                  "exact fused step");
    } else if (mode == OSBF_MODE_EXACT) {
        const size_t n = static_cast<size_t>(g.batch) * g.width * g.height;
        // even table pitch: 16-byte rows, so the stencil walk can stage them with TMA
        const size_t tp = (static_cast<size_t>(g.width) + 2) & ~static_cast<size_t>(1);
        const size_t ns = static_cast<size_t>(g.batch) * tp * (g.height + 1);
        OSBF_CUDA(ctx->rowpfx.ensure(n * sizeof(double)), "alloc row prefix");
        // + the table's own flag word behind it (cleared / raised by the
        // build of every pass, read by the stencil)
        OSBF_CUDA(ctx->sat.ensure((ns + 2) * sizeof(double)), "alloc sat");
        unsigned* const tflag = reinterpret_cast<unsigned*>(ctx->sat.as<double>() + ns);
        OSBF_CUDA(osbf_gpu::exact_build_sat(src, g, ctx->rowpfx.as<double>(), ctx->sat.as<double>(),
                                            s, ctx->lc, tp, tflag),
                  "exact SAT");
        OSBF_CUDA(osbf_gpu::exact_select(src, g, r, ctx->sat.as<double>(), dst, dp, dpl, means, sel,
                                         s, ctx->lc, tp, tflag),
                  "exact select");
    } else {
        OSBF_CUDA(osbf_gpu::fast_step(src, g, r, dst, dp, dpl, means, sel, s, ctx->lc),
                  "fast step");
    }
    return OSBF_OK;
}

// Copy/convert kernel: typed batch -> fp64 batch.
template <typename T>
__global__ void convert_kernel(const T* __restrict__ in, size_t ip, size_t ipl,
                               double* __restrict__ out, size_t op, size_t opl, int W, int H,
                               int B) {
    // grid-stride over rows of all planes (no 65535 limit on rows or planes)
    const size_t rows = static_cast<size_t>(H) * B;
    for (size_t r = blockIdx.y; r < rows; r += gridDim.y) {
        const size_t b = r / H, y = r % H;
        for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < W; x += gridDim.x * blockDim.x)
            out[b * opl + y * op + x] = static_cast<double>(in[b * ipl + y * ip + x]);
    }
}

}  // namespace

namespace osbf_gpu {
void note_kernel(const char* name) { g_last_kernel = name; }

namespace {
std::atomic<const char*> g_fast_override{nullptr};
std::atomic<const char*> g_exact_override{nullptr};
constexpr const char* kExactFamilies[] = {"strip", "twalk", "gwalk", "stencil"};
}
const char* fast_kernel_override() { return g_fast_override.load(std::memory_order_acquire); }
const char* exact_kernel_override() {
    if (const char* o = g_exact_override.load(std::memory_order_acquire)) return o;
    static const char* env = []() -> const char* {
        const char* e = std::getenv("OSBF_GPU_EXACT");
        if (e)
            for (const char* k : kExactFamilies)
                if (std::strcmp(k, e) == 0) return k;
        return nullptr;
    }();
    return env;
}

cudaError_t convert_to_f64(const PlaneView& in, const Geometry& g, double* out, size_t op,
                           size_t opl, cudaStream_t s, LaunchCounter& lc) {
    const size_t rows = static_cast<size_t>(g.height) * g.batch;
    dim3 grid(static_cast<unsigned>(std::min((g.width + 255) / 256, 64)),
              static_cast<unsigned>(std::min<size_t>(rows, 65535)), 1);
    ++lc.launches;
    note_kernel("convert_to_f64");
    switch (in.dtype) {
        case OSBF_U8:
            convert_kernel<<<grid, 256, 0, s>>>(static_cast<const uint8_t*>(in.base), in.pitch,
                                                in.plane, out, op, opl, g.width, g.height,
                                                g.batch);
            break;
        case OSBF_F32:
            convert_kernel<<<grid, 256, 0, s>>>(static_cast<const float*>(in.base), in.pitch,
                                                in.plane, out, op, opl, g.width, g.height,
                                                g.batch);
            break;
        default:
            convert_kernel<<<grid, 256, 0, s>>>(static_cast<const double*>(in.base), in.pitch,
                                                in.plane, out, op, opl, g.width, g.height,
                                                g.batch);
            break;
    }
    return cudaGetLastError();
}
}  // namespace osbf_gpu

namespace {

// Jacobi ping-pong through context scratch (filters2d.hpp:94-97 / :112-152:
// every iteration reads the previous plane and writes a fresh one); the last
// launch writes d_out.  want(remaining) is the number of passes (1..4) the
// next launch should run; run(src, dst, dst_pitch, dst_plane, n, &retry)
// launches them, setting retry when n > 1 has no kernel (then one pass).
template <typename Want, typename Run>
osbf_status jacobi(osbf_ctx* ctx, const osbf_gpu::PlaneView& input, const osbf_gpu::Geometry& g,
                   int iterations, double* d_out, size_t out_pitch, size_t out_plane,
                   cudaStream_t s, Want&& want, Run&& run) {
    const size_t plane = static_cast<size_t>(g.width) * g.height;
    const bool alias = static_cast<const void*>(d_out) == input.base;
    const int scratch_needed = (iterations > 1 ? 2 : 0) + (alias ? 1 : 0);
    if (scratch_needed > 0) OSBF_CUDA(ctx->ping.ensure(plane * g.batch * sizeof(double)), "alloc ping");
    if (scratch_needed > 1) OSBF_CUDA(ctx->pong.ensure(plane * g.batch * sizeof(double)), "alloc pong");
    osbf_gpu::PlaneView src = input;
    int done = 0;
    for (int k = 0; done < iterations; ++k) {
        int n = want(iterations - done);
        for (;;) {
            const bool last = done + n == iterations;
            double* dst;
            size_t dp, dpl;
            if (last && !alias) {
                dst = d_out;
                dp = out_pitch;
                dpl = out_plane;
            } else {
                DevBuf& buf = (k % 2 == 0) ? ctx->ping : ctx->pong;
                dst = buf.as<double>();
                dp = g.width;
                dpl = plane;
            }
            bool retry = false;
            const osbf_status st = run(src, dst, dp, dpl, n, &retry);
            if (retry && n > 1) {
                n = 1;
                continue;
            }
            if (st != OSBF_OK) return st;
            src = osbf_gpu::PlaneView{dst, OSBF_F64, dp, dpl};
            break;
        }
        done += n;
    }
    if (alias) {
        OSBF_CUDA(cudaMemcpy2DAsync(d_out, out_pitch * sizeof(double), src.base,
                                    src.pitch * sizeof(double), g.width * sizeof(double),
                                    static_cast<size_t>(g.height) * g.batch,
                                    cudaMemcpyDeviceToDevice, s),
                  "copy back");
    }
    return OSBF_OK;
}

bool graphs_enabled() {
    static const bool on = [] {
        const char* v = std::getenv("OSBF_GPU_GRAPHS");
        return !(v && v[0] == '0');
    }();
    return on;
}

// A multi-pass call is a fixed sequence of launches, so a repeated call
// (same buffers, geometry, radius, passes) replays it as one CUDA graph:
// the first call runs plainly (allocations, kernel attributes), the second
// is captured on a private stream and instantiated, later ones are one
// cudaGraphLaunch on the caller's stream.  Any change of argument or of a
// scratch buffer is a different key.  OSBF_GPU_GRAPHS=0 disables it.
template <typename Body>
osbf_status run_graphed(osbf_ctx* ctx, std::vector<uintptr_t> key, cudaStream_t s, Body&& body) {
    if (!graphs_enabled()) return body(s);
    for (void* p : {ctx->ping.ptr, ctx->pong.ptr, ctx->rowpfx.ptr, ctx->sat.ptr})
        key.push_back(reinterpret_cast<uintptr_t>(p));
    for (size_t b : {ctx->ping.bytes, ctx->pong.bytes, ctx->rowpfx.bytes, ctx->sat.bytes})
        key.push_back(b);
    // a forced kernel family is part of what a call launches
    key.push_back(reinterpret_cast<uintptr_t>(osbf_gpu::fast_kernel_override()));
    key.push_back(reinterpret_cast<uintptr_t>(osbf_gpu::exact_kernel_override()));
    auto it = std::find_if(ctx->graphs.begin(), ctx->graphs.end(),
                           [&](const GraphEntry& e) { return e.key == key; });
    if (it == ctx->graphs.end()) {
        if (ctx->graphs.size() >= 8) {  // evict the oldest
            if (ctx->graphs.front().exec) cudaGraphExecDestroy(ctx->graphs.front().exec);
            ctx->graphs.erase(ctx->graphs.begin());
        }
        GraphEntry e;
        e.key = std::move(key);
        ctx->graphs.push_back(std::move(e));
        return body(s);  // first time: plain (may allocate; the key is re-taken next time)
    }
    if (it->state == -1) return body(s);
    if (it->state == 0) {
        if (!ctx->capture)
            OSBF_CUDA(cudaStreamCreateWithFlags(&ctx->capture, cudaStreamNonBlocking), "stream");
        const uint64_t before = ctx->lc.launches;
        cudaGraph_t graph = nullptr;
        cudaError_t e = cudaStreamBeginCapture(ctx->capture, cudaStreamCaptureModeThreadLocal);
        osbf_status st = OSBF_OK;
        if (e == cudaSuccess) {
            st = body(ctx->capture);
            e = cudaStreamEndCapture(ctx->capture, &graph);
        }
        const uint64_t captured = ctx->lc.launches - before;  // kernels inside the graph
        ctx->lc.launches = before;
        cudaGraphExec_t exec = nullptr;
        if (e == cudaSuccess && st == OSBF_OK && graph)
            e = cudaGraphInstantiate(&exec, graph, 0);
        if (graph) cudaGraphDestroy(graph);
        if (e != cudaSuccess || st != OSBF_OK || !exec) {
            cudaGetLastError();  // capture unsupported here: run plainly from now on
            it->state = -1;
            return body(s);
        }
        it->exec = exec;
        it->launches = captured;
        it->kernel = g_last_kernel;
        it->state = 1;
    }
    OSBF_CUDA(cudaGraphLaunch(it->exec, s), "graph launch");
    ctx->lc.launches += it->launches;
    g_last_kernel = it->kernel;
    return OSBF_OK;
}

}  // namespace

extern "C" {

int osbf_gpu_abi_version(void) { return OSBF_GPU_ABI_VERSION; }

const char* osbf_gpu_last_error(void) { return g_last_error.c_str(); }

const char* osbf_gpu_last_kernel(void) { return g_last_kernel; }

int osbf_gpu_fast_max_radius(void) { return osbf_gpu::fast_generic_max_radius(); }

osbf_status osbf_gpu_set_fast_kernel(const char* name) {
    static const char* const kNames[] = {"strip", "tile", "tma", "tmaseq", "tmaint", "pair", "arms", "stream", "walk", "vwalk", "sep"};
    if (!name || !name[0]) {
        osbf_gpu::g_fast_override.store(nullptr, std::memory_order_release);
        return OSBF_OK;
    }
    for (const char* k : kNames)
        if (std::strcmp(k, name) == 0) {
            osbf_gpu::g_fast_override.store(k, std::memory_order_release);
            return OSBF_OK;
        }
    return fail(OSBF_ERR_INVALID_ARGUMENT, "unknown fast kernel family '%s'", name);
}

osbf_status osbf_gpu_set_exact_kernel(const char* name) {
    if (!name || !name[0]) {
        osbf_gpu::g_exact_override.store(nullptr, std::memory_order_release);
        return OSBF_OK;
    }
    for (const char* k : osbf_gpu::kExactFamilies)
        if (std::strcmp(k, name) == 0) {
            osbf_gpu::g_exact_override.store(k, std::memory_order_release);
            return OSBF_OK;
        }
    return fail(OSBF_ERR_INVALID_ARGUMENT, "unknown exact kernel family '%s'", name);
}

int osbf_gpu_device_available(void) { return device_ok() ? 1 : 0; }

osbf_status osbf_gpu_ctx_create(int device, osbf_ctx** out) {
    if (!out) return fail(OSBF_ERR_INVALID_ARGUMENT, "ctx_create: null out pointer");
    *out = nullptr;
    if (!device_ok()) return fail(OSBF_ERR_NO_DEVICE, "no CUDA device of compute capability 10.x");
    OSBF_CUDA(cudaSetDevice(device), "cudaSetDevice");
    osbf_ctx* ctx = new (std::nothrow) osbf_ctx();
    if (!ctx) return fail(OSBF_ERR_ALLOC, "ctx_create: out of host memory");
    ctx->device = device;
    cudaError_t e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete ctx;
        return cuda_fail(e, "cudaStreamCreate");
    }
    *out = ctx;
    return OSBF_OK;
}

osbf_status osbf_gpu_ctx_destroy(osbf_ctx* ctx) {
    if (!ctx) return OSBF_OK;
    cudaSetDevice(ctx->device);
    if (ctx->switch_ev) cudaEventDestroy(ctx->switch_ev);
    cudaStreamSynchronize(ctx->stream);
    ctx->ping.release();
    ctx->pong.release();
    ctx->rowpfx.release();
    ctx->sat.release();
    ctx->host_in.release();
    ctx->host_out.release();
    ctx->drop_graphs();
    if (ctx->capture) cudaStreamDestroy(ctx->capture);
    if (ctx->copy_in) cudaStreamDestroy(ctx->copy_in);
    if (ctx->copy_out) cudaStreamDestroy(ctx->copy_out);
    cudaStreamDestroy(ctx->stream);
    delete ctx;
    return OSBF_OK;
}

osbf_status osbf_gpu_ctx_trim(osbf_ctx* ctx) {
    if (!ctx) return fail(OSBF_ERR_INVALID_ARGUMENT, "null context");
    cudaSetDevice(ctx->device);
    OSBF_CUDA(cudaStreamSynchronize(ctx->stream), "sync");
    OSBF_CUDA(cudaDeviceSynchronize(), "sync");  // graphs may run on caller streams
    ctx->drop_graphs();
    ctx->ping.release();
    ctx->pong.release();
    ctx->rowpfx.release();
    ctx->sat.release();
    ctx->host_in.release();
    ctx->host_out.release();
    return OSBF_OK;
}

uint64_t osbf_gpu_ctx_launch_count(const osbf_ctx* ctx) { return ctx ? ctx->lc.launches : 0; }

osbf_status osbf_gpu_ctx_set_temporal_blocking(osbf_ctx* ctx, int passes_per_launch) {
    if (!ctx) return fail(OSBF_ERR_INVALID_ARGUMENT, "null context");
    if (passes_per_launch < 1 || passes_per_launch > 4)
        return fail(OSBF_ERR_INVALID_ARGUMENT, "passes_per_launch must be in 1..4");
    ctx->passes_per_launch = passes_per_launch;
    return OSBF_OK;
}

osbf_status osbf_gpu_iterate(osbf_ctx* ctx, osbf_dtype in_dtype, const void* d_in,
                             size_t in_pitch, size_t in_plane_stride, double* d_out,
                             size_t out_pitch, size_t out_plane_stride, int width, int height,
                             int batch, int radius, int iterations, osbf_mode mode,
                             void* stream) {
    if (!ctx) return fail(OSBF_ERR_INVALID_ARGUMENT, "null context");
    osbf_status st;
    if ((st = check_geometry(width, height, batch)) != OSBF_OK) return st;
    if ((st = check_dtype(in_dtype)) != OSBF_OK) return st;
    if ((st = check_mode(mode)) != OSBF_OK) return st;
    if (iterations < 0) return fail(OSBF_ERR_INVALID_ARGUMENT, "osbf: iterations must be >= 0");
    if (iterations > 0 && radius < 1)
        return fail(OSBF_ERR_INVALID_ARGUMENT, "osbf_step: radius must be >= 1");
    if (!d_in || !d_out) return fail(OSBF_ERR_INVALID_ARGUMENT, "null plane pointer");
    if (in_pitch < static_cast<size_t>(width) || out_pitch < static_cast<size_t>(width))
        return fail(OSBF_ERR_INVALID_ARGUMENT, "pitch smaller than width");
    if (batch > 1 && (in_plane_stride < in_pitch * height || out_plane_stride < out_pitch * height))
        return fail(OSBF_ERR_INVALID_ARGUMENT, "plane stride smaller than pitch*height");
    OSBF_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
    cudaStream_t s = pick_stream(ctx, stream);

    const osbf_gpu::Geometry g{width, height, batch};
    const osbf_gpu::PlaneView input{d_in, in_dtype, in_pitch, in_plane_stride};
    if (iterations == 0) {
        // filters2d.hpp:94-97: a copy, radius unchecked.
        if (static_cast<const void*>(d_out) == d_in && in_dtype == OSBF_F64) return OSBF_OK;
        OSBF_CUDA(osbf_gpu::convert_to_f64(input, g, d_out, out_pitch, out_plane_stride, s, ctx->lc),
                  "copy");
        return OSBF_OK;
    }
    // Fast mode runs two passes per launch (temporal blocking) when enabled
    // and the radius has a two-pass kernel; otherwise one pass per launch.
    const int tbk = mode != OSBF_MODE_FAST ? 1
                    : (ctx->passes_per_launch > 1 ? ctx->passes_per_launch : tb_env());
    auto body = [&](cudaStream_t st_) {
        return jacobi(
            ctx, input, g, iterations, d_out, out_pitch, out_plane_stride, st_,
            [&](int remaining) { return remaining < tbk ? remaining : tbk; },
            [&](const osbf_gpu::PlaneView& src, double* dst, size_t dp, size_t dpl, int n,
                bool* retry) -> osbf_status {
                if (n > 1) {
                    const cudaError_t e =
                        osbf_gpu::fast_stepk(src, g, radius, n, dst, dp, dpl, st_, ctx->lc);
                    if (e == cudaErrorNotSupported) {
                        cudaGetLastError();
                        *retry = true;
                        return OSBF_OK;
                    }
                    OSBF_CUDA(e, "fast two-pass step");
                    return OSBF_OK;
                }
                return one_pass(ctx, src, g, radius, dst, dp, dpl, nullptr, nullptr, mode, st_);
            });
    };
    const std::vector<uintptr_t> key = {
        1, static_cast<uintptr_t>(in_dtype), reinterpret_cast<uintptr_t>(d_in), in_pitch,
        in_plane_stride, reinterpret_cast<uintptr_t>(d_out), out_pitch, out_plane_stride,
        static_cast<uintptr_t>(width), static_cast<uintptr_t>(height),
        static_cast<uintptr_t>(batch), static_cast<uintptr_t>(radius),
        static_cast<uintptr_t>(iterations), static_cast<uintptr_t>(mode),
        static_cast<uintptr_t>(tbk)};
    return run_graphed(ctx, key, s, body);
}

}  // extern "C"

namespace {
// The SAT-based companions of the OSBF path (fast_osbf, box_filter): the
// reference checks the radius before the iteration count, even for 0
// iterations (filters2d.hpp:39-42, :107-110), then iterates a pass that
// rebuilds the whole-image table (bit-identical order) every iteration.
enum class SatFilter { FastOsbf = 2, Box = 3 };

osbf_status sat_filter(osbf_ctx* ctx, SatFilter which, osbf_dtype in_dtype, const void* d_in,
                       size_t in_pitch, size_t in_plane_stride, double* d_out, size_t out_pitch,
                       size_t out_plane_stride, int width, int height, int batch, int radius,
                       int iterations, void* stream) {
    const char* name = which == SatFilter::Box ? "box_filter" : "fast_osbf";
    if (!ctx) return fail(OSBF_ERR_INVALID_ARGUMENT, "null context");
    if (radius < 1) return fail(OSBF_ERR_INVALID_ARGUMENT, "%s: radius must be >= 1", name);
    if (iterations < 0)
        return fail(OSBF_ERR_INVALID_ARGUMENT, "%s: iterations must be >= 0", name);
    osbf_status st;
    if ((st = check_geometry(width, height, batch)) != OSBF_OK) return st;
    if ((st = check_dtype(in_dtype)) != OSBF_OK) return st;
    if (!d_in || !d_out) return fail(OSBF_ERR_INVALID_ARGUMENT, "null plane pointer");
    if (in_pitch < static_cast<size_t>(width) || out_pitch < static_cast<size_t>(width))
        return fail(OSBF_ERR_INVALID_ARGUMENT, "pitch smaller than width");
    if (batch > 1 && (in_plane_stride < in_pitch * height || out_plane_stride < out_pitch * height))
        return fail(OSBF_ERR_INVALID_ARGUMENT, "plane stride smaller than pitch*height");
    OSBF_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
    cudaStream_t s = pick_stream(ctx, stream);
    const osbf_gpu::Geometry g{width, height, batch};
    const osbf_gpu::PlaneView input{d_in, in_dtype, in_pitch, in_plane_stride};
    if (iterations == 0) {
        if (static_cast<const void*>(d_out) == d_in && in_dtype == OSBF_F64) return OSBF_OK;
        OSBF_CUDA(osbf_gpu::convert_to_f64(input, g, d_out, out_pitch, out_plane_stride, s, ctx->lc),
                  "copy");
        return OSBF_OK;
    }
    const size_t n = static_cast<size_t>(batch) * width * height;
    const size_t ns = static_cast<size_t>(batch) * (width + 1) * (height + 1);
    OSBF_CUDA(ctx->rowpfx.ensure(n * sizeof(double)), "alloc row prefix");
    OSBF_CUDA(ctx->sat.ensure(ns * sizeof(double)), "alloc sat");
    auto body = [&](cudaStream_t st_) {
        return jacobi(
            ctx, input, g, iterations, d_out, out_pitch, out_plane_stride, st_,
            [](int) { return 1; },
            [&](const osbf_gpu::PlaneView& src, double* dst, size_t dp, size_t dpl, int,
                bool*) -> osbf_status {
                auto pass = which == SatFilter::Box ? osbf_gpu::boxfilter_pass
                                                    : osbf_gpu::fastosbf_pass;
                OSBF_CUDA(pass(src, g, radius, ctx->rowpfx.as<double>(), ctx->sat.as<double>(),
                               dst, dp, dpl, st_, ctx->lc),
                          name);
                return OSBF_OK;
            });
    };
    const std::vector<uintptr_t> key = {
        static_cast<uintptr_t>(which), static_cast<uintptr_t>(in_dtype),
        reinterpret_cast<uintptr_t>(d_in), in_pitch, in_plane_stride,
        reinterpret_cast<uintptr_t>(d_out), out_pitch, out_plane_stride,
        static_cast<uintptr_t>(width), static_cast<uintptr_t>(height),
        static_cast<uintptr_t>(batch), static_cast<uintptr_t>(radius),
        static_cast<uintptr_t>(iterations)};
    return run_graphed(ctx, key, s, body);
}
}  // namespace

extern "C" {

osbf_status osbf_gpu_fast_osbf(osbf_ctx* ctx, osbf_dtype in_dtype, const void* d_in,
                              size_t in_pitch, size_t in_plane_stride, double* d_out,
                              size_t out_pitch, size_t out_plane_stride, int width, int height,
                              int batch, int radius, int iterations, void* stream) {
    return sat_filter(ctx, SatFilter::FastOsbf, in_dtype, d_in, in_pitch, in_plane_stride, d_out,
                      out_pitch, out_plane_stride, width, height, batch, radius, iterations,
                      stream);
}

osbf_status osbf_gpu_box_filter(osbf_ctx* ctx, osbf_dtype in_dtype, const void* d_in,
                               size_t in_pitch, size_t in_plane_stride, double* d_out,
                               size_t out_pitch, size_t out_plane_stride, int width, int height,
                               int batch, int radius, int iterations, void* stream) {
    return sat_filter(ctx, SatFilter::Box, in_dtype, d_in, in_pitch, in_plane_stride, d_out,
                      out_pitch, out_plane_stride, width, height, batch, radius, iterations,
                      stream);
}

}  // extern "C"

namespace {
// osbf_3d / box_filter_3d (filters3d.hpp:55-114) on one fp64 volume [D][H][W].
osbf_status filter3d(osbf_ctx* ctx, bool osbf3, const double* d_in, double* d_out, int width,
                     int height, int depth, int radius, int iterations, void* stream) {
    const char* name = osbf3 ? "osbf_3d" : "box_filter_3d";
    if (!ctx) return fail(OSBF_ERR_INVALID_ARGUMENT, "null context");
    if (radius < 1) return fail(OSBF_ERR_INVALID_ARGUMENT, "%s: radius must be >= 1", name);
    if (iterations < 0)
        return fail(OSBF_ERR_INVALID_ARGUMENT, "%s: iterations must be >= 0", name);
    if (width < 1 || height < 1 || depth < 1)
        return fail(OSBF_ERR_INVALID_ARGUMENT, "Volume: extents must be >= 1");
    if (!d_in || !d_out) return fail(OSBF_ERR_INVALID_ARGUMENT, "null volume pointer");
    OSBF_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
    cudaStream_t s = pick_stream(ctx, stream);
    const size_t n = static_cast<size_t>(width) * height * depth;
    // the volume as a width x (height*depth) plane for the ping-pong logic
    const osbf_gpu::Geometry g{width, height * depth, 1};
    const osbf_gpu::PlaneView input{d_in, OSBF_F64, static_cast<size_t>(width), n};
    if (iterations == 0) {
        if (d_out != d_in)
            OSBF_CUDA(cudaMemcpyAsync(d_out, d_in, n * sizeof(double), cudaMemcpyDeviceToDevice, s),
                      "copy");
        return OSBF_OK;
    }
    OSBF_CUDA(ctx->rowpfx.ensure(n * sizeof(double)), "alloc rows");
    OSBF_CUDA(ctx->sat.ensure(osbf_gpu::svt_elems(width, height, depth) * sizeof(double)),
              "alloc table");
    auto body = [&](cudaStream_t st_) {
        return jacobi(
            ctx, input, g, iterations, d_out, static_cast<size_t>(width), n, st_,
            [](int) { return 1; },
            [&](const osbf_gpu::PlaneView& src, double* dst, size_t, size_t, int,
                bool*) -> osbf_status {
                OSBF_CUDA(osbf_gpu::filter3d_pass(static_cast<const double*>(src.base), width,
                                                  height, depth, radius, osbf3,
                                                  ctx->rowpfx.as<double>(), ctx->sat.as<double>(),
                                                  dst, st_, ctx->lc),
                          name);
                return OSBF_OK;
            });
    };
    const std::vector<uintptr_t> key = {
        osbf3 ? 5u : 4u, reinterpret_cast<uintptr_t>(d_in), reinterpret_cast<uintptr_t>(d_out),
        static_cast<uintptr_t>(width), static_cast<uintptr_t>(height),
        static_cast<uintptr_t>(depth), static_cast<uintptr_t>(radius),
        static_cast<uintptr_t>(iterations)};
    return run_graphed(ctx, key, s, body);
}

osbf_status filter3d_host(osbf_ctx* ctx, bool osbf3, const double* h_in, double* h_out, int width,
                          int height, int depth, int radius, int iterations) {
    if (!ctx) return fail(OSBF_ERR_INVALID_ARGUMENT, "null context");
    if (!h_in || !h_out) return fail(OSBF_ERR_INVALID_ARGUMENT, "null host pointer");
    if (width < 1 || height < 1 || depth < 1)
        return fail(OSBF_ERR_INVALID_ARGUMENT, "Volume: extents must be >= 1");
    OSBF_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
    const size_t n = static_cast<size_t>(width) * height * depth;
    OSBF_CUDA(ctx->host_in.ensure(n * sizeof(double)), "alloc input");
    OSBF_CUDA(ctx->host_out.ensure(n * sizeof(double)), "alloc output");
    cudaStream_t s = pick_stream(ctx, ctx->stream);
    OSBF_CUDA(cudaMemcpyAsync(ctx->host_in.ptr, h_in, n * sizeof(double), cudaMemcpyHostToDevice, s),
              "H2D");
    osbf_status st = filter3d(ctx, osbf3, ctx->host_in.as<double>(), ctx->host_out.as<double>(),
                              width, height, depth, radius, iterations, s);
    if (st != OSBF_OK) return st;
    OSBF_CUDA(cudaMemcpyAsync(h_out, ctx->host_out.ptr, n * sizeof(double), cudaMemcpyDeviceToHost,
                              s),
              "D2H");
    OSBF_CUDA(cudaStreamSynchronize(s), "sync");
    return OSBF_OK;
}
}  // namespace

extern "C" {

osbf_status osbf_gpu_osbf_3d(osbf_ctx* ctx, const double* d_in, double* d_out, int width,
                            int height, int depth, int radius, int iterations, void* stream) {
    return filter3d(ctx, true, d_in, d_out, width, height, depth, radius, iterations, stream);
}

osbf_status osbf_gpu_box_filter_3d(osbf_ctx* ctx, const double* d_in, double* d_out, int width,
                                  int height, int depth, int radius, int iterations,
                                  void* stream) {
    return filter3d(ctx, false, d_in, d_out, width, height, depth, radius, iterations, stream);
}

osbf_status osbf_gpu_osbf_3d_host(osbf_ctx* ctx, const double* h_in, double* h_out, int width,
                                 int height, int depth, int radius, int iterations) {
    return filter3d_host(ctx, true, h_in, h_out, width, height, depth, radius, iterations);
}

osbf_status osbf_gpu_svt_host(osbf_ctx* ctx, const double* h_in, int width, int height, int depth,
                             double* h_cumsum) {
    if (!ctx) return fail(OSBF_ERR_INVALID_ARGUMENT, "null context");
    if (!h_in || !h_cumsum) return fail(OSBF_ERR_INVALID_ARGUMENT, "null host pointer");
    if (width < 1 || height < 1 || depth < 1)
        return fail(OSBF_ERR_INVALID_ARGUMENT, "Volume: extents must be >= 1");
    OSBF_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
    const size_t n = static_cast<size_t>(width) * height * depth;
    const size_t nt = osbf_gpu::svt_elems(width, height, depth);
    OSBF_CUDA(ctx->host_in.ensure(n * sizeof(double)), "alloc input");
    OSBF_CUDA(ctx->rowpfx.ensure(n * sizeof(double)), "alloc rows");
    OSBF_CUDA(ctx->host_out.ensure(nt * sizeof(double)), "alloc table");
    cudaStream_t s = pick_stream(ctx, ctx->stream);
    OSBF_CUDA(cudaMemcpyAsync(ctx->host_in.ptr, h_in, n * sizeof(double), cudaMemcpyHostToDevice, s),
              "H2D");
    OSBF_CUDA(osbf_gpu::svt_build(ctx->host_in.as<double>(), width, height, depth,
                                  ctx->rowpfx.as<double>(), ctx->host_out.as<double>(), s, ctx->lc),
              "svt");
    OSBF_CUDA(cudaMemcpyAsync(h_cumsum, ctx->host_out.ptr, nt * sizeof(double),
                              cudaMemcpyDeviceToHost, s),
              "D2H");
    OSBF_CUDA(cudaStreamSynchronize(s), "sync");
    return OSBF_OK;
}

osbf_status osbf_gpu_box_filter_3d_host(osbf_ctx* ctx, const double* h_in, double* h_out,
                                       int width, int height, int depth, int radius,
                                       int iterations) {
    return filter3d_host(ctx, false, h_in, h_out, width, height, depth, radius, iterations);
}

osbf_status osbf_gpu_subwindow_means(osbf_ctx* ctx, osbf_dtype in_dtype, const void* d_in,
                                     size_t in_pitch, size_t in_plane_stride, int width,
                                     int height, int batch, int radius, double* d_means,
                                     uint8_t* d_sel, osbf_mode mode, void* stream) {
    if (!ctx) return fail(OSBF_ERR_INVALID_ARGUMENT, "null context");
    osbf_status st;
    if ((st = check_geometry(width, height, batch)) != OSBF_OK) return st;
    if ((st = check_dtype(in_dtype)) != OSBF_OK) return st;
    if ((st = check_mode(mode)) != OSBF_OK) return st;
    if (radius < 1) return fail(OSBF_ERR_INVALID_ARGUMENT, "sub_windows: radius must be >= 1");
    if (!d_in) return fail(OSBF_ERR_INVALID_ARGUMENT, "null plane pointer");
    OSBF_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
    cudaStream_t s = pick_stream(ctx, stream);
    const osbf_gpu::Geometry g{width, height, batch};
    const osbf_gpu::PlaneView input{d_in, in_dtype, in_pitch, in_plane_stride};
    return one_pass(ctx, input, g, radius, nullptr, 0, 0, d_means, d_sel, mode, s);
}

osbf_status osbf_gpu_sat(osbf_ctx* ctx, osbf_dtype in_dtype, const void* d_in, size_t in_pitch,
                         size_t in_plane_stride, int width, int height, int batch,
                         double* d_cumsum, void* stream) {
    if (!ctx) return fail(OSBF_ERR_INVALID_ARGUMENT, "null context");
    osbf_status st;
    if ((st = check_geometry(width, height, batch)) != OSBF_OK) return st;
    if ((st = check_dtype(in_dtype)) != OSBF_OK) return st;
    if (!d_in || !d_cumsum) return fail(OSBF_ERR_INVALID_ARGUMENT, "null pointer");
    OSBF_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
    cudaStream_t s = pick_stream(ctx, stream);
    const osbf_gpu::Geometry g{width, height, batch};
    const osbf_gpu::PlaneView input{d_in, in_dtype, in_pitch, in_plane_stride};
    OSBF_CUDA(ctx->rowpfx.ensure(static_cast<size_t>(batch) * width * height * sizeof(double)),
              "alloc row prefix");
    OSBF_CUDA(osbf_gpu::exact_build_sat(input, g, ctx->rowpfx.as<double>(), d_cumsum, s, ctx->lc),
              "exact SAT");
    return OSBF_OK;
}

osbf_status osbf_gpu_step_band(osbf_ctx* ctx, osbf_dtype in_dtype, const void* d_in,
                               size_t in_pitch, int in_row0, int in_rows, double* d_out,
                               size_t out_pitch, int out_row0, int out_rows, int width,
                               int image_height, int radius, osbf_mode mode, void* stream) {
    return osbf_gpu_step_band_push(ctx, in_dtype, d_in, in_pitch, in_row0, in_rows, d_out,
                                   out_pitch, out_row0, out_rows, width, image_height, radius,
                                   mode, nullptr, nullptr, 0, 0, stream);
}

osbf_status osbf_gpu_step_band_push(osbf_ctx* ctx, osbf_dtype in_dtype, const void* d_in,
                                    size_t in_pitch, int in_row0, int in_rows, double* d_out,
                                    size_t out_pitch, int out_row0, int out_rows, int width,
                                    int image_height, int radius, osbf_mode mode,
                                    double* d_push_up, double* d_push_down, int push_rows,
                                    size_t push_pitch, void* stream) {
    if (!ctx) return fail(OSBF_ERR_INVALID_ARGUMENT, "null context");
    if (push_rows < 0 || push_rows > out_rows)
        return fail(OSBF_ERR_INVALID_ARGUMENT, "push_rows %d outside [0, out_rows]", push_rows);
    if (push_rows > 0 && (d_push_up || d_push_down) && push_pitch < static_cast<size_t>(width))
        return fail(OSBF_ERR_INVALID_ARGUMENT, "push pitch smaller than width");
    osbf_status st;
    if ((st = check_dtype(in_dtype)) != OSBF_OK) return st;
    if ((st = check_mode(mode)) != OSBF_OK) return st;
    if (mode != OSBF_MODE_FAST)
        return fail(OSBF_ERR_INVALID_ARGUMENT,
                    "row bands need OSBF_MODE_FAST: the exact mode's whole-image prefix is serial");
    if (width < 1 || image_height < 1 || in_rows < 1 || out_rows < 1)
        return fail(OSBF_ERR_INVALID_ARGUMENT, "ImagePlane: dimensions must be >= 1");
    if (radius < 1) return fail(OSBF_ERR_INVALID_ARGUMENT, "osbf_step: radius must be >= 1");
    if (radius > osbf_gpu::fast_generic_max_radius())
        return fail(OSBF_ERR_INVALID_ARGUMENT, "row bands support radius <= %d (got %d)",
                    osbf_gpu::fast_generic_max_radius(), radius);
    if (out_row0 < 0 || out_row0 + out_rows > image_height)
        return fail(OSBF_ERR_OUT_OF_RANGE, "output rows [%d, %d) outside the image height %d",
                    out_row0, out_row0 + out_rows, image_height);
    const int need0 = out_row0 - radius < 0 ? 0 : out_row0 - radius;
    const int need1 = out_row0 + out_rows + radius > image_height ? image_height
                                                                 : out_row0 + out_rows + radius;
    if (in_row0 > need0 || in_row0 + in_rows < need1)
        return fail(OSBF_ERR_OUT_OF_RANGE,
                    "input rows [%d, %d) do not cover the band plus halo [%d, %d)", in_row0,
                    in_row0 + in_rows, need0, need1);
    if (!d_in || !d_out) return fail(OSBF_ERR_INVALID_ARGUMENT, "null plane pointer");
    if (in_pitch < static_cast<size_t>(width) || out_pitch < static_cast<size_t>(width))
        return fail(OSBF_ERR_INVALID_ARGUMENT, "pitch smaller than width");
    OSBF_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
    osbf_gpu::Geometry g{width, out_rows, 1};
    g.img_height = image_height;
    g.in_row0 = in_row0;
    g.out_row0 = out_row0;
    g.in_rows = in_rows;
    if (push_rows > 0) {
        g.push_up = d_push_up;
        g.push_dn = d_push_down;
        g.push_rows = push_rows;
        g.push_pitch = push_pitch;
    }
    const osbf_gpu::PlaneView input{d_in, in_dtype, in_pitch, in_pitch * in_rows};
    if (radius > osbf_gpu::kFastMaxRadius) {
        OSBF_CUDA(osbf_gpu::fast_generic_step(input, g, radius, d_out, out_pitch,
                                              out_pitch * out_rows, pick_stream(ctx, stream),
                                              ctx->lc),
                  "band step");
        return OSBF_OK;
    }
    OSBF_CUDA(osbf_gpu::fast_step(input, g, radius, d_out, out_pitch, out_pitch * out_rows, nullptr,
                                  nullptr, pick_stream(ctx, stream), ctx->lc),
              "band step");
    return OSBF_OK;
}

}  // extern "C"

namespace {
// Host-buffer batch: H2D, filter(d_in, d_out, planes) on the compute stream,
// D2H.  Large batches run in chunks so the upload of chunk j+1 and the
// download of chunk j-1 (two copy streams) overlap the passes of chunk j.
template <typename Filter>
osbf_status host_batch(osbf_ctx* ctx, osbf_dtype in_dtype, const void* h_in, double* h_out,
                       int width, int height, int batch, Filter&& filter) {
    osbf_status st = OSBF_OK;
    if (!h_in || !h_out) return fail(OSBF_ERR_INVALID_ARGUMENT, "null host pointer");
    OSBF_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
    const size_t n = static_cast<size_t>(width) * height * batch;
    OSBF_CUDA(ctx->host_in.ensure(n * dtype_size(in_dtype)), "alloc input");
    OSBF_CUDA(ctx->host_out.ensure(n * sizeof(double)), "alloc output");
    cudaStream_t s = pick_stream(ctx, ctx->stream);
    const size_t plane = static_cast<size_t>(width) * height;
    const size_t in_bytes = plane * dtype_size(in_dtype);
    const char* hin = static_cast<const char*>(h_in);
    char* din = static_cast<char*>(ctx->host_in.ptr);
    double* dout = ctx->host_out.as<double>();
    // Planes are independent: large batches go through in chunks so the
    // upload of chunk j+1 and the download of chunk j-1 (two copy streams)
    // overlap the passes of chunk j (compute stream).  Results do not depend
    // on the chunking.
    const int chunks = (batch >= 4 && n * sizeof(double) >= (64u << 20)) ? (batch < 8 ? batch : 8)
                                                                           : 1;
    if (chunks == 1) {
        OSBF_CUDA(cudaMemcpyAsync(din, hin, n * dtype_size(in_dtype), cudaMemcpyHostToDevice, s),
                  "H2D");
        st = filter(din, dout, batch);
        if (st != OSBF_OK) return st;
        OSBF_CUDA(cudaMemcpyAsync(h_out, dout, n * sizeof(double), cudaMemcpyDeviceToHost, s),
                  "D2H");
        OSBF_CUDA(cudaStreamSynchronize(s), "sync");
        return OSBF_OK;
    }
    if (!ctx->copy_in)
        OSBF_CUDA(cudaStreamCreateWithFlags(&ctx->copy_in, cudaStreamNonBlocking), "stream");
    if (!ctx->copy_out)
        OSBF_CUDA(cudaStreamCreateWithFlags(&ctx->copy_out, cudaStreamNonBlocking), "stream");
    cudaEvent_t ev[2 * 8];
    int nev = 0;
    for (; nev < 2 * chunks; ++nev) {
        cudaError_t e = cudaEventCreateWithFlags(&ev[nev], cudaEventDisableTiming);
        if (e != cudaSuccess) {
            for (int i = 0; i < nev; ++i) cudaEventDestroy(ev[i]);
            return cuda_fail(e, "cudaEventCreate");
        }
    }
    auto cleanup = [&] {
        for (int i = 0; i < nev; ++i) cudaEventDestroy(ev[i]);
    };
    for (int j = 0; j < chunks && st == OSBF_OK; ++j) {
        const int b0 = static_cast<int>(static_cast<long long>(batch) * j / chunks);
        const int b1 = static_cast<int>(static_cast<long long>(batch) * (j + 1) / chunks);
        const size_t nb = static_cast<size_t>(b1 - b0);
        cudaError_t e = cudaMemcpyAsync(din + b0 * in_bytes, hin + b0 * in_bytes, nb * in_bytes,
                                        cudaMemcpyHostToDevice, ctx->copy_in);
        if (e == cudaSuccess) e = cudaEventRecord(ev[2 * j], ctx->copy_in);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ev[2 * j], 0);
        if (e != cudaSuccess) {
            st = cuda_fail(e, "H2D");
            break;
        }
        st = filter(din + b0 * in_bytes, dout + b0 * plane, b1 - b0);
        if (st != OSBF_OK) break;
        e = cudaEventRecord(ev[2 * j + 1], s);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(ctx->copy_out, ev[2 * j + 1], 0);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(h_out + b0 * plane, dout + b0 * plane, nb * plane * sizeof(double),
                                cudaMemcpyDeviceToHost, ctx->copy_out);
        if (e != cudaSuccess) st = cuda_fail(e, "D2H");
    }
    cudaError_t e1 = cudaStreamSynchronize(ctx->copy_out);
    cudaError_t e2 = cudaStreamSynchronize(s);
    cudaError_t e3 = cudaStreamSynchronize(ctx->copy_in);
    cleanup();
    if (st != OSBF_OK) return st;
    if (e1 != cudaSuccess) return cuda_fail(e1, "sync");
    if (e2 != cudaSuccess) return cuda_fail(e2, "sync");
    if (e3 != cudaSuccess) return cuda_fail(e3, "sync");
    return OSBF_OK;
}

}  // namespace

extern "C" {

osbf_status osbf_gpu_osbf_host(osbf_ctx* ctx, osbf_dtype in_dtype, const void* h_in,
                               double* h_out, int width, int height, int batch, int radius,
                               int iterations, osbf_mode mode) {
    if (!ctx) return fail(OSBF_ERR_INVALID_ARGUMENT, "null context");
    osbf_status st;
    if ((st = check_geometry(width, height, batch)) != OSBF_OK) return st;
    if ((st = check_dtype(in_dtype)) != OSBF_OK) return st;
    if (iterations < 0) return fail(OSBF_ERR_INVALID_ARGUMENT, "osbf: iterations must be >= 0");
    if (iterations > 0 && radius < 1)
        return fail(OSBF_ERR_INVALID_ARGUMENT, "osbf_step: radius must be >= 1");
    const size_t plane = static_cast<size_t>(width) * height;
    return host_batch(ctx, in_dtype, h_in, h_out, width, height, batch,
                      [&](const void* din, double* dout, int nb) {
                          return osbf_gpu_iterate(ctx, in_dtype, din, width, plane, dout, width,
                                                  plane, width, height, nb, radius, iterations,
                                                  mode, ctx->stream);
                      });
}

osbf_status osbf_gpu_box_filter_host(osbf_ctx* ctx, osbf_dtype in_dtype, const void* h_in,
                                     double* h_out, int width, int height, int batch, int radius,
                                     int iterations) {
    if (!ctx) return fail(OSBF_ERR_INVALID_ARGUMENT, "null context");
    if (radius < 1) return fail(OSBF_ERR_INVALID_ARGUMENT, "box_filter: radius must be >= 1");
    if (iterations < 0)
        return fail(OSBF_ERR_INVALID_ARGUMENT, "box_filter: iterations must be >= 0");
    osbf_status st;
    if ((st = check_geometry(width, height, batch)) != OSBF_OK) return st;
    if ((st = check_dtype(in_dtype)) != OSBF_OK) return st;
    const size_t plane = static_cast<size_t>(width) * height;
    return host_batch(ctx, in_dtype, h_in, h_out, width, height, batch,
                      [&](const void* din, double* dout, int nb) {
                          return osbf_gpu_box_filter(ctx, in_dtype, din, width, plane, dout, width,
                                                     plane, width, height, nb, radius, iterations,
                                                     ctx->stream);
                      });
}

osbf_status osbf_gpu_fast_osbf_host(osbf_ctx* ctx, osbf_dtype in_dtype, const void* h_in,
                                    double* h_out, int width, int height, int batch, int radius,
                                    int iterations) {
    if (!ctx) return fail(OSBF_ERR_INVALID_ARGUMENT, "null context");
    if (radius < 1) return fail(OSBF_ERR_INVALID_ARGUMENT, "fast_osbf: radius must be >= 1");
    if (iterations < 0) return fail(OSBF_ERR_INVALID_ARGUMENT, "fast_osbf: iterations must be >= 0");
    osbf_status st;
    if ((st = check_geometry(width, height, batch)) != OSBF_OK) return st;
    if ((st = check_dtype(in_dtype)) != OSBF_OK) return st;
    const size_t plane = static_cast<size_t>(width) * height;
    return host_batch(ctx, in_dtype, h_in, h_out, width, height, batch,
                      [&](const void* din, double* dout, int nb) {
                          return osbf_gpu_fast_osbf(ctx, in_dtype, din, width, plane, dout, width,
                                                    plane, width, height, nb, radius, iterations,
                                                    ctx->stream);
                      });
}

osbf_status osbf_gpu_osbf_step_host(osbf_ctx* ctx, const double* h_in, double* h_out, int width,
                                    int height, int radius, osbf_mode mode) {
    if (radius < 1) return fail(OSBF_ERR_INVALID_ARGUMENT, "osbf_step: radius must be >= 1");
    return osbf_gpu_osbf_host(ctx, OSBF_F64, h_in, h_out, width, height, 1, radius, 1, mode);
}

}  // extern "C"

namespace {
// filter_multichannel (filters2d.hpp:371-400) for either variant: channels
// are independent, so they run as one batched launch per pass.
osbf_status multichannel_host(osbf_ctx* ctx, const double* const* h_in, double* const* h_out,
                              int channels, int width, int height, int radius, int iterations,
                              int variant, osbf_mode mode) {  // 0 OsbfExact, 1 OsbfFast, 2 Box
    if (!ctx) return fail(OSBF_ERR_INVALID_ARGUMENT, "null context");
    // FilterConfig::validate (core.hpp:244-253), then the channel checks of
    // MultiChannelImage (core.hpp:85-92).
    if (radius < 1) return fail(OSBF_ERR_INVALID_ARGUMENT, "FilterConfig: radius must be >= 1");
    if (iterations < 0)
        return fail(OSBF_ERR_INVALID_ARGUMENT, "FilterConfig: iterations must be >= 0");
    if (channels < 1 || channels > 4)
        return fail(OSBF_ERR_INVALID_ARGUMENT, "MultiChannelImage: channel count must be in [1,4]");
    osbf_status st;
    if ((st = check_geometry(width, height, 1)) != OSBF_OK) return st;
    if (!h_in || !h_out) return fail(OSBF_ERR_INVALID_ARGUMENT, "null host pointer");
    OSBF_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
    const size_t plane = static_cast<size_t>(width) * height;
    OSBF_CUDA(ctx->host_in.ensure(plane * channels * sizeof(double)), "alloc input");
    OSBF_CUDA(ctx->host_out.ensure(plane * channels * sizeof(double)), "alloc output");
    cudaStream_t s = pick_stream(ctx, ctx->stream);
    double* din = ctx->host_in.as<double>();
    double* dout = ctx->host_out.as<double>();
    for (int c = 0; c < channels; ++c) {
        if (!h_in[c] || !h_out[c]) return fail(OSBF_ERR_INVALID_ARGUMENT, "null channel pointer");
        OSBF_CUDA(cudaMemcpyAsync(din + c * plane, h_in[c], plane * sizeof(double),
                                  cudaMemcpyHostToDevice, s),
                  "H2D");
    }
    // Channels are independent (filters2d.hpp:376-384): one batched launch.
    st = variant == 1   ? osbf_gpu_fast_osbf(ctx, OSBF_F64, din, width, plane, dout, width,
                                             plane, width, height, channels, radius,
                                             iterations, s)
         : variant == 2 ? osbf_gpu_box_filter(ctx, OSBF_F64, din, width, plane, dout, width,
                                              plane, width, height, channels, radius,
                                              iterations, s)
                        : osbf_gpu_iterate(ctx, OSBF_F64, din, width, plane, dout, width, plane,
                                           width, height, channels, radius, iterations, mode, s);
    if (st != OSBF_OK) return st;
    for (int c = 0; c < channels; ++c)
        OSBF_CUDA(cudaMemcpyAsync(h_out[c], dout + c * plane, plane * sizeof(double),
                                  cudaMemcpyDeviceToHost, s),
                  "D2H");
    OSBF_CUDA(cudaStreamSynchronize(s), "sync");
    return OSBF_OK;
}

}  // namespace

extern "C" {

osbf_status osbf_gpu_filter_multichannel_host(osbf_ctx* ctx, const double* const* h_in,
                                              double* const* h_out, int channels, int width,
                                              int height, int radius, int iterations,
                                              osbf_mode mode) {
    return multichannel_host(ctx, h_in, h_out, channels, width, height, radius, iterations, 0,
                             mode);
}

osbf_status osbf_gpu_filter_multichannel_fast_host(osbf_ctx* ctx, const double* const* h_in,
                                                   double* const* h_out, int channels, int width,
                                                   int height, int radius, int iterations) {
    return multichannel_host(ctx, h_in, h_out, channels, width, height, radius, iterations, 1,
                             OSBF_MODE_EXACT);
}

osbf_status osbf_gpu_filter_multichannel_box_host(osbf_ctx* ctx, const double* const* h_in,
                                                  double* const* h_out, int channels, int width,
                                                  int height, int radius, int iterations) {
    return multichannel_host(ctx, h_in, h_out, channels, width, height, radius, iterations, 2,
                             OSBF_MODE_EXACT);
}

osbf_status osbf_gpu_smooth_raster_host(osbf_ctx* ctx, const void* h_raster, int sample_bytes,
                                        int channels, int width, int height, osbf_filter filter,
                                        int radius, int iterations, osbf_mode mode, void* h_out,
                                        int out_sample_bytes) {
    if (!ctx) return fail(OSBF_ERR_INVALID_ARGUMENT, "null context");
    // FilterConfig::validate (core.hpp:244-253), then write_image's checks
    // (io.hpp:189-194).
    if (radius < 1) return fail(OSBF_ERR_INVALID_ARGUMENT, "FilterConfig: radius must be >= 1");
    if (iterations < 0)
        return fail(OSBF_ERR_INVALID_ARGUMENT, "FilterConfig: iterations must be >= 0");
    if (filter != OSBF_FILTER_OSBF && filter != OSBF_FILTER_FAST_OSBF && filter != OSBF_FILTER_BOX)
        return fail(OSBF_ERR_INVALID_ARGUMENT, "unknown filter");
    if (channels != 1 && channels != 3)
        return fail(OSBF_ERR_INVALID_ARGUMENT,
                    "write_image: only 1- or 3-channel images can be saved");
    if ((sample_bytes != 1 && sample_bytes != 2) || (out_sample_bytes != 1 && out_sample_bytes != 2))
        return fail(OSBF_ERR_INVALID_ARGUMENT, "write_image: bit depth must be 8 or 16");
    osbf_status st;
    if ((st = check_geometry(width, height, 1)) != OSBF_OK) return st;
    if (!h_raster || !h_out) return fail(OSBF_ERR_INVALID_ARGUMENT, "null host pointer");
    OSBF_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
    const size_t plane = static_cast<size_t>(width) * height;
    const size_t in_bytes = plane * channels * sample_bytes;
    const size_t out_bytes = plane * channels * out_sample_bytes;
    // host_in: the raster, then (multi-channel or 16-bit) its channel planes
    // (uint8 for 8-bit samples — promoted inside the first pass — fp64 for
    // 16-bit); host_out: the filtered fp64 planes, then the quantised raster.
    const size_t planes_off = (in_bytes + 255) & ~size_t(255);
    const bool direct = channels == 1 && sample_bytes == 1;  // already a uint8 plane
    const size_t plane_bytes = plane * channels * (sample_bytes == 1 ? 1 : sizeof(double));
    OSBF_CUDA(ctx->host_in.ensure(planes_off + (direct ? 0 : plane_bytes)), "alloc input");
    const size_t raster_off = plane * channels * sizeof(double);
    OSBF_CUDA(ctx->host_out.ensure(raster_off + out_bytes), "alloc output");
    cudaStream_t s = pick_stream(ctx, ctx->stream);
    char* in_base = static_cast<char*>(ctx->host_in.ptr);
    double* dout = ctx->host_out.as<double>();
    void* draster_out = static_cast<char*>(ctx->host_out.ptr) + raster_off;
    OSBF_CUDA(cudaMemcpyAsync(in_base, h_raster, in_bytes, cudaMemcpyHostToDevice, s), "H2D");
    const void* src = in_base;
    const osbf_dtype dtype = sample_bytes == 1 ? OSBF_U8 : OSBF_F64;
    if (!direct) {
        OSBF_CUDA(osbf_gpu::raster_to_planes(in_base, sample_bytes, channels, plane,
                                             in_base + planes_off, s, ctx->lc),
                  "raster_to_planes");
        src = in_base + planes_off;
    }
    // Channels are independent (filters2d.hpp:376-384): one batched launch.
    st = filter == OSBF_FILTER_FAST_OSBF
             ? osbf_gpu_fast_osbf(ctx, dtype, src, width, plane, dout, width, plane, width,
                                  height, channels, radius, iterations, s)
         : filter == OSBF_FILTER_BOX
             ? osbf_gpu_box_filter(ctx, dtype, src, width, plane, dout, width, plane, width,
                                   height, channels, radius, iterations, s)
             : osbf_gpu_iterate(ctx, dtype, src, width, plane, dout, width, plane, width, height,
                                channels, radius, iterations, mode, s);
    if (st != OSBF_OK) return st;
    OSBF_CUDA(osbf_gpu::planes_to_raster(dout, channels, plane, draster_out, out_sample_bytes, s,
                                         ctx->lc),
              "planes_to_raster");
    OSBF_CUDA(cudaMemcpyAsync(h_out, draster_out, out_bytes, cudaMemcpyDeviceToHost, s), "D2H");
    OSBF_CUDA(cudaStreamSynchronize(s), "sync");
    return OSBF_OK;
}

osbf_status osbf_gpu_sat_host(osbf_ctx* ctx, const double* h_in, int width, int height,
                              double* h_cumsum) {
    if (!ctx) return fail(OSBF_ERR_INVALID_ARGUMENT, "null context");
    osbf_status st;
    if ((st = check_geometry(width, height, 1)) != OSBF_OK) return st;
    if (!h_in || !h_cumsum) return fail(OSBF_ERR_INVALID_ARGUMENT, "null host pointer");
    OSBF_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
    const size_t plane = static_cast<size_t>(width) * height;
    const size_t ns = static_cast<size_t>(width + 1) * (height + 1);
    OSBF_CUDA(ctx->host_in.ensure(plane * sizeof(double)), "alloc input");
    OSBF_CUDA(ctx->host_out.ensure(ns * sizeof(double)), "alloc output");
    cudaStream_t s = pick_stream(ctx, ctx->stream);
    OSBF_CUDA(cudaMemcpyAsync(ctx->host_in.ptr, h_in, plane * sizeof(double), cudaMemcpyHostToDevice,
                              s),
              "H2D");
    st = osbf_gpu_sat(ctx, OSBF_F64, ctx->host_in.ptr, width, plane, width, height, 1,
                      ctx->host_out.as<double>(), s);
    if (st != OSBF_OK) return st;
    OSBF_CUDA(cudaMemcpyAsync(h_cumsum, ctx->host_out.ptr, ns * sizeof(double),
                              cudaMemcpyDeviceToHost, s),
              "D2H");
    OSBF_CUDA(cudaStreamSynchronize(s), "sync");
    return OSBF_OK;
}

}  // extern "C"
