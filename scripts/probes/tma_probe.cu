// Minimal TMA probe: one 3-D box load (f64) into shared memory with mbarrier completion.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstring>

struct Maps { CUtensorMap q; CUtensorMap c; int variant; int cbytes; };

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ Maps mp, double* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    double* buf = (double*)sm;
    uint64_t* bar = (uint64_t*)(sm + 44 * 20 * 4 * 8);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(bar)), "r"(1));
        if (mp.variant != 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        else asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(bar)), "r"((mp.variant == 3 || mp.variant == 4) ? mp.cbytes : 44 * 20 * 4 * 8) : "memory");
        if (mp.variant == 5) {
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(su(buf)), "l"(&mp.c), "r"(-6), "r"(-6), "r"(0), "r"(su(bar)) : "memory");
        } else if (mp.variant == 4) {
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(su(buf)), "l"(&mp.c), "r"(-6), "r"(-6), "r"(0), "r"(su(bar)) : "memory");
        } else if (mp.variant == 3) {
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(su(buf)), "l"(&mp.c), "r"(-8), "r"(-6), "r"(su(bar)) : "memory");
        } else if (mp.variant == 2)
            asm volatile("cp.async.bulk.tensor.3d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(su(buf)), "l"(&mp.q), "r"(-6), "r"(-6), "r"(0), "r"(su(bar)) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(su(buf)), "l"(&mp.q), "r"(-6), "r"(-6), "r"(0), "r"(su(bar)) : "memory");
    }
    uint32_t done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(su(bar)), "r"(0) : "memory");
    double s = 0;
    for (int i = threadIdx.x; i < 44 * 20 * 4; i += blockDim.x) s += buf[i];
    atomicAdd(out, s);
}

int main(int argc, char** argv) {
    int variant = argc > 1 ? atoi(argv[1]) : 0;
    const int n0 = 1024, n1 = 1024;
    double* d; cudaMalloc(&d, (size_t)n0 * n1 * 4 * 8);
    cudaMemset(d, 0, (size_t)n0 * n1 * 4 * 8);
    double one = 1.0;
    for (int c = 0; c < 4; ++c) for (int j = 0; j < 14; ++j) for (int i = 0; i < 38; ++i)
        cudaMemcpy(d + (size_t)c * n0 * n1 + (size_t)j * n0 + i, &one, 8, cudaMemcpyHostToDevice);
    double* out; cudaMalloc(&out, 8); cudaMemset(out, 0, 8);
    void* fp = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled)fp;
    Maps mp; memset(&mp, 0, sizeof(mp)); mp.variant = variant;
    cuuint64_t dims[3] = {n0, n1, 4}; cuuint64_t str[2] = {(cuuint64_t)n0 * 8, (cuuint64_t)n0 * n1 * 8};
    cuuint32_t box[3] = {44, 20, 4}, es[3] = {1, 1, 1};
    CUresult r = enc(&mp.q, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    uint16_t* dc; cudaMalloc(&dc, (size_t)n0 * n1 * 2); cudaMemset(dc, 0, (size_t)n0 * n1 * 2);
    int bw = argc > 2 ? atoi(argv[2]) : 48;
    int u32 = argc > 3 ? atoi(argv[3]) : 0;
    cuuint64_t d2[2] = {(cuuint64_t)(u32 ? n0 / 2 : n0), n1}; cuuint64_t s2[1] = {(cuuint64_t)n0 * 2}; cuuint32_t b2[2] = {(cuuint32_t)bw, 20}, e2[2] = {1, 1};
    cuuint64_t d3[3] = {d2[0], d2[1], 1}; cuuint64_t s3[2] = {s2[0], s2[0] * n1}; cuuint32_t b3[3] = {b2[0], 20, 1}, e3[3] = {1, 1, 1};
    if (variant == 5) mp.c = mp.q;
    else if (variant == 4)
    r = enc(&mp.c, u32 ? CU_TENSOR_MAP_DATA_TYPE_UINT32 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, dc, d3, s3, b3, e3, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    else
    r = enc(&mp.c, u32 ? CU_TENSOR_MAP_DATA_TYPE_UINT32 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, dc, d2, s2, b2, e2, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode2 %d\n", (int)r);
    mp.cbytes = bw * 20 * (u32 ? 4 : 2);
    size_t smem = 44 * 20 * 4 * 8 + 128;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    probe<<<1, 128, smem>>>(mp, out);
    cudaError_t e = cudaDeviceSynchronize();
    double h = 0; cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
    printf("variant %d: %s sum=%g (expect %d)\n", variant, cudaGetErrorString(e), h, 32 * 14 * 4);
    return 0;
}
