// FP64 microbenchmarks on one B200 (sm_100a): DFMA throughput (independent chains, full
// occupancy) -> the FP64 roofline peak; dependent-chain latencies of DFMA / DADD / DMUL /
// double division / shared-memory load (one warp, clock64).
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void k_dfma_tput(double* out, int iters, double a, double b) {
    double x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    if (s == 12345.678) out[0] = s;
}

__global__ void k_lat(long long* cyc, double* out, int iters, double a, double b, int kind) {
    __shared__ double sh[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sh[i] = (i * 7 + 1) % 1024;
    __syncthreads();
    double x = threadIdx.x * 1e-9 + 1.0;
    long long t0 = clock64();
    if (kind == 0)
        for (int i = 0; i < iters; ++i) x = fma(x, a, b);
    else if (kind == 1)
        for (int i = 0; i < iters; ++i) x = x + a;
    else if (kind == 2)
        for (int i = 0; i < iters; ++i) x = x * a;
    else if (kind == 3)
        for (int i = 0; i < iters; ++i) x = b / x;
    else
        for (int i = 0; i < iters; ++i) x = sh[(int)x & 1023];
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    if (x == 1234.5) out[0] = x;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 8);
    cudaMalloc(&cyc, 8);
    int nsm = 0, clk = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096;
    const int blocks = nsm * 8, threads = 256;
    k_dfma_tput<8><<<blocks, threads>>>(out, iters, 0.999, 1e-3);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k_dfma_tput<8><<<blocks, threads>>>(out, iters, 0.999, 1e-3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 5.0 * 2.0 * 8 * (double)iters * blocks * threads;
    printf("{\"fp64_dfma_tflops\": %.2f, \"sms\": %d, \"clock_khz\": %d", flops / (ms * 1e-3) / 1e12, nsm, clk);
    const char* names[5] = {"dfma", "dadd", "dmul", "ddiv", "lds_dep"};
    for (int kind = 0; kind < 5; ++kind) {
        const int it = kind == 3 ? 256 : 1024;
        k_lat<<<1, 32>>>(cyc, out, it, 0.999, 1e-3, kind);
        k_lat<<<1, 32>>>(cyc, out, it, 0.999, 1e-3, kind);
        long long c = 0;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        printf(", \"lat_%s_cycles\": %.1f", names[kind], (double)c / it);
    }
    printf("}\n");
    return 0;
}
