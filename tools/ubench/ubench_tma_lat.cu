// Latency of the first TMA load of a kernel: one 16 KB box (128 x 64 bf16, 128B
// swizzle) per CTA, 148 CTAs, clock64 from issue to mbarrier completion, for data
// resident in L2 and data in HBM only (a region not touched since an L2 flush), with
// and without a prefetch.tensormap ahead of the load, and for N back-to-back boxes.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "sm100.cuh"
using namespace sdx::sm100;

template <int NBOX, bool PREF>
__global__ void lat_kernel(const __grid_constant__ CUtensorMap tm, int row0, long long* out) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) {
        if (PREF) tma_prefetch(&tm);
        mbar_init(&bar, 1);
        fence_barrier_init();
        const long long t0 = clock64();
        mbar_expect_tx(&bar, NBOX * 16384);
        for (int i = 0; i < NBOX; ++i)
            tma_load_2d(sm + i * 16384, &tm, &bar, 0, row0 + (blockIdx.x * NBOX + i) * 128);
        mbar_wait(&bar, 0);
        const long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int NBOX, bool PREF>
void run(const CUtensorMap& tm, int row0, long long* d, const char* what, void* flush, size_t flush_bytes) {
    auto k = lat_kernel<NBOX, PREF>;
    const int smem = 1024 + NBOX * 16384;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (flush) cudaMemset(flush, 0, flush_bytes);  // evicts the matrix from L2
    k<<<148, 32, smem>>>(tm, row0, d);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    long long mn = 1LL << 60, mx = 0, sum = 0;
    for (auto x : h) { mn = x < mn ? x : mn; mx = x > mx ? x : mx; sum += x; }
    printf("%-26s boxes %d prefetch %d: min %6lld med~ %6lld max %6lld cycles\n", what, NBOX, PREF, mn, sum / 148, mx);
}

int main() {
    const int rows = 148 * 4 * 128 * 2, cols = 64;  // two disjoint halves of 148 x 4 boxes
    void* buf;
    cudaMalloc(&buf, (size_t)rows * cols * 2);
    cudaMemset(buf, 1, (size_t)rows * cols * 2);
    const size_t fl = 512ull << 20;
    void* flush;
    cudaMalloc(&flush, fl);
    long long* d;
    cudaMalloc(&d, 148 * sizeof(long long));
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    EncFn enc = (EncFn)p;
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int rep = 0; rep < 2; ++rep) {
        run<1, true>(tm, 0, d, "HBM (after L2 flush)", flush, fl);
        run<1, true>(tm, 0, d, "L2 warm", nullptr, 0);
        run<1, false>(tm, 0, d, "L2 warm", nullptr, 0);
        run<1, false>(tm, 0, d, "HBM (after L2 flush)", flush, fl);
        run<4, true>(tm, 0, d, "HBM (after L2 flush)", flush, fl);
        run<4, true>(tm, 0, d, "L2 warm", nullptr, 0);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
