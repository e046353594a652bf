// Probe: one 4-D TMA box load (fp64, box 22 x 18 x 1 x 5) into shared memory with an mbarrier,
// tensor map passed as a __grid_constant__ kernel parameter (the k_rhs3z pattern).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o tma4_probe tma4_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

struct Maps { CUtensorMap box; int ok; };

__global__ void k(const __grid_constant__ Maps maps, double* out, int x0, int y0, int z, int fence, int bx) {
    extern __shared__ __align__(128) double raw[];
    double* sm = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(raw) + 127) & ~uintptr_t(127));
    __shared__ __align__(8) unsigned long long bar;
    const unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
        if (fence) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(8u * bx * 18 * 5) : "memory");
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                     ::"r"((unsigned)__cvta_generic_to_shared(sm)), "l"(reinterpret_cast<unsigned long long>(&maps.box)),
                       "r"(x0), "r"(y0), "r"(z), "r"(0), "r"(b) : "memory");
    }
    unsigned done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(b), "r"(0u) : "memory");
    for (int i = threadIdx.x; i < bx * 18 * 5; i += blockDim.x) out[i] = sm[i];
}

int main(int argc, char** argv) {
    const int promo = argc > 1 ? atoi(argv[1]) : 3, bxw = argc > 2 ? atoi(argv[2]) : 22, x0 = argc > 3 ? atoi(argv[3]) : -3;
    const int n0 = 64, n1 = 48, n2 = 8;
    const size_t N = (size_t)n0 * n1 * n2;
    std::vector<double> h(5 * N);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
    double *d, *o;
    cudaMalloc(&d, h.size() * 8);
    cudaMalloc(&o, 256 * 18 * 5 * 8);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    using Enc = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    Maps mp;
    memset(&mp, 0, sizeof(mp));
    const cuuint64_t dim[4] = {n0, n1, n2, 5};
    const cuuint64_t str[3] = {n0 * 8, (cuuint64_t)n0 * n1 * 8, N * 8};
    const cuuint32_t box[4] = {(cuuint32_t)bxw, 18, 1, 5}, es[4] = {1, 1, 1, 1};
    CUresult r = ((Enc)fn)(&mp.box, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, d, dim, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_NONE, (CUtensorMapL2promotion)promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    for (int fence = 0; fence < 2; ++fence) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        k<<<1, 128, 64 * 1024>>>(mp, o, x0, 5, 2, fence, bxw);
        cudaError_t e = cudaDeviceSynchronize();
        printf("fence %d: %s\n", fence, cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
        std::vector<double> res(bxw * 18 * 5);
        cudaMemcpy(res.data(), o, res.size() * 8, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int c = 0; c < 5; ++c)
            for (int y = 0; y < 18; ++y)
                for (int x = 0; x < bxw; ++x) {
                    const int gx = x + x0, gy = y + 5;
                    const double want = (gx < 0) ? 0.0 : h[(size_t)c * N + (size_t)2 * n0 * n1 + (size_t)gy * n0 + gx];
                    bad += res[(c * 18 + y) * bxw + x] != want;
                }
        printf("mismatches %d\n", bad);
    }
    return 0;
}
