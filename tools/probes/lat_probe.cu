// Latency probe: dependent fp64 add chains (register-only, through shared
// memory, and with an interleaved independent store) on one warp.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain_reg(double* out, long long* cyc, int n, double x) {
    double a = x, b = x * 0.5;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) a = __dadd_rn(a, b);
    }
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void chain_fma(double* out, long long* cyc, int n, double x) {
    double a = x, b = x * 0.5;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) a = __fma_rn(a, b, b);
    }
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// prefix over a shared-memory row: load (independent), add (dependent), store
__global__ void chain_smem(double* out, long long* cyc, int n, double x) {
    __shared__ double t[16 * 33];
    for (int k = threadIdx.x; k < 16 * 33; k += 32) t[k] = x + k;
    __syncwarp();
    double acc = 0;
    const int lane = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        double v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = t[k * 33 + lane];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            acc = __dadd_rn(acc, v[k]);
            t[k * 33 + lane] = acc;
        }
        __syncwarp();
    }
    long long t1 = clock64();
    out[threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void int_chain(double* out, long long* cyc, int n, double x) {
    unsigned a = __double_as_longlong(x), b = 3;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) a = a * b + 1u;
    }
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// throughput: many independent chains per SM
__global__ void dadd_tput(double* out, int n, double x) {
    double a0 = x, a1 = x + 1, a2 = x + 2, a3 = x + 3, a4 = x + 4, a5 = x + 5, a6 = x + 6, a7 = x + 7;
    const double b = x * 1e-9;
    for (int i = 0; i < n; ++i) {
        a0 = __dadd_rn(a0, b); a1 = __dadd_rn(a1, b); a2 = __dadd_rn(a2, b); a3 = __dadd_rn(a3, b);
        a4 = __dadd_rn(a4, b); a5 = __dadd_rn(a5, b); a6 = __dadd_rn(a6, b); a7 = __dadd_rn(a7, b);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

int main() {
    double* out; long long* cyc;
    cudaMalloc(&out, 1 << 26); cudaMalloc(&cyc, 64);
    const int n = 4096;
    long long c;
    auto run = [&](const char* name, void (*k)(double*, long long*, int, double), int per) {
        k<<<1, 32>>>(out, cyc, n, 1.0);
        k<<<1, 32>>>(out, cyc, n, 1.0);
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        printf("%-12s %.2f cycles per dependent op\n", name, double(c) / (double(n) * per));
    };
    run("dadd", chain_reg, 16);
    run("dfma", chain_fma, 16);
    run("lds+dadd+sts", chain_smem, 16);
    run("imad", int_chain, 16);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int dev; cudaGetDevice(&dev); int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    dadd_tput<<<sms * 8, 256>>>(out, 1000, 1.0);
    cudaEventRecord(e0);
    const int it = 20000;
    dadd_tput<<<sms * 8, 256>>>(out, it, 1.0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = double(sms) * 8 * 256 * it * 8;
    printf("dadd throughput: %.2f Tops/s = %.1f lanes/clk/SM at 1.965 GHz\n", ops / ms / 1e9,
           ops / (ms * 1e-3) / sms / 1.965e9);
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
