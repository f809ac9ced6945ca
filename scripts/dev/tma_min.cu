// Minimal TMA load test: 4-D float tensor like the solver state; argv selects the variant.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap m, float* out, int c0, int c1, int c2, int c3, int bytes, int mode)
{
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ alignas(8) unsigned long long bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(bytes) : "memory");
        if (mode == 0)
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
                ::"r"(sa(sm)), "l"(&m), "r"(sa(&bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3) : "memory");
        else
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
                ::"r"(sa(sm)), "l"(&m), "r"(sa(&bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3) : "memory");
    }
    __syncthreads();
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(sa(&bar)) : "memory");
    for (int i = threadIdx.x; i < bytes / 4; i += blockDim.x) out[i] = reinterpret_cast<float*>(sm)[i];
}

int main(int argc, char** argv)
{
    int nx = atoi(argv[1]), ny = atoi(argv[2]), nz = atoi(argv[3]), ns = atoi(argv[4]);
    int bw = atoi(argv[5]), bh = atoi(argv[6]), nf = atoi(argv[7]);
    int c0 = atoi(argv[8]), c1 = atoi(argv[9]), c2 = atoi(argv[10]), c3 = atoi(argv[11]);
    int mode = argc > 12 ? atoi(argv[12]) : 0;
    int px = (nx + 31) / 32 * 32;
    size_t plane = (size_t)px * ny, fs = plane * nz;
    float* d;
    cudaMalloc(&d, fs * ns * 4);
    float* h = (float*)malloc(fs * ns * 4);
    for (size_t i = 0; i < fs * ns; ++i) h[i] = (float)i;
    cudaMemcpy(d, h, fs * ns * 4, cudaMemcpyHostToDevice);
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    EncodeTiledFn enc = (EncodeTiledFn)p;
    CUtensorMap m;
    cuuint64_t dims[4] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz, (cuuint64_t)ns};
    cuuint64_t strides[3] = {(cuuint64_t)px * 4, plane * 4, fs * 4};
    cuuint32_t box[4] = {(cuuint32_t)bw, (cuuint32_t)bh, 1, (cuuint32_t)nf};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode=%d ", (int)r);
    int bytes = bw * bh * nf * 4;
    float* o;
    cudaMalloc(&o, bytes);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    k<<<1, 128, bytes + 256>>>(m, o, c0, c1, c2, c3, bytes, mode);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel=%s ", cudaGetErrorString(e));
    if (e == cudaSuccess) {
        float* ho = (float*)malloc(bytes);
        cudaMemcpy(ho, o, bytes, cudaMemcpyDeviceToHost);
        // check a few elements
        int bad = 0;
        for (int f = 0; f < nf; ++f)
            for (int yy = 0; yy < bh; ++yy)
                for (int xx = 0; xx < bw; ++xx) {
                    int gx = c0 + xx, gy = c1 + yy, gz = c2, gs = c3 + f;
                    float want = (gx >= 0 && gx < nx && gy >= 0 && gy < ny && gz >= 0 && gz < nz && gs < ns)
                                     ? (float)(gs * fs + gz * plane + (size_t)gy * px + gx) : 0.f;
                    if (ho[(f * bh + yy) * bw + xx] != want) ++bad;
                }
        printf("bad=%d", bad);
    }
    printf("\n");
    return 0;
}
