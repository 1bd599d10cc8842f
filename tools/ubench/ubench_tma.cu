// TMA ingest bandwidth: each CTA streams 16 KB (128 x 64 bf16, 128B swizzle) boxes of an
// L2-resident matrix through an S-stage smem ring; a consumer warp releases each stage as
// soon as it lands.  Reports bytes/clk/SM and aggregate TB/s for several grid sizes, and
// the same with 2-CTA clusters multicasting every box to both CTAs.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "sm100.cuh"
using namespace sdx::sm100;

__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, %4}], [%2], %5;" ::
            "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
        : "memory");
}

template <int S, int MC>
__global__ void tma_kernel(const __grid_constant__ CUtensorMap tm, int rows, int iters, long long* cyc) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + S * 16384);
    uint64_t* empty = full + S;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t rank = 0;
    if (MC) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], MC ? 2 : 1); }
        fence_barrier_init();
    }
    __syncthreads();
    if (MC) { asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory"); }
    const int nbox_r = rows / 128;
    const long long t0 = clock64();
    const int unit = MC ? blockIdx.x / 2 : blockIdx.x;
    if (warp == 0 && lane == 0) {
        for (int it = 0; it < iters; ++it) {
            const int s = it % S;
            mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
            mbar_expect_tx(&full[s], 16384);
            const int box = (unit * 7 + it) % (nbox_r * 8);
            if (MC) {
                // each CTA issues half the boxes, multicast to both
                if ((it & 1) == (int)rank) tma_load_2d_mc(sm + s * 16384, &tm, &full[s], (box & 7) * 64, (box >> 3) * 128, 3);
            } else {
                tma_load_2d(sm + s * 16384, &tm, &full[s], (box & 7) * 64, (box >> 3) * 128);
            }
        }
    } else if (warp == 1 && lane == 0) {
        for (int it = 0; it < iters; ++it) {
            const int s = it % S;
            mbar_wait(&full[s], (it / S) & 1);
            if (MC) {
                // release the slot in both CTAs (the peer's multicast writes into ours too)
                mbar_arrive(&empty[s]);
                const uint32_t peer = mapa_shared(smem_u32(&empty[s]), rank ^ 1);
                mbar_arrive_cluster(peer);
            } else {
                mbar_arrive(&empty[s]);
            }
        }
    }
    __syncthreads();
    if (MC) { asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory"); }
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int S, int MC>
void run(const CUtensorMap& tm, int rows, int grid, long long* d) {
    const int iters = 2000;
    auto k = tma_kernel<S, MC>;
    const int smem = 1024 + S * 16384 + 256;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(64);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = MC ? 2 : 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaLaunchKernelEx(&cfg, k, tm, rows, iters, d);
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, k, tm, rows, iters, d);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long h[148]; cudaMemcpy(h, d, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
    long long mx = 0; for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
    const double bytes_per_cta = 16384.0 * iters;  // bytes landing in each CTA's smem
    printf("stages %d grid %3d %s: %.1f B/clk/SM landed, aggregate landed %.2f TB/s, L2 reads %.2f TB/s  (%s)\n", S, grid,
           MC ? "mcast2" : "unicast", bytes_per_cta / mx, bytes_per_cta * grid / (ms * 1e-3) / 1e12,
           bytes_per_cta * grid / (MC ? 2 : 1) / (ms * 1e-3) / 1e12, cudaGetErrorString(e));
}

int main() {
    const int rows = 8192, cols = 512;  // 8 MB bf16, L2 resident
    void* buf; cudaMalloc(&buf, (size_t)rows * cols * 2); cudaMemset(buf, 1, (size_t)rows * cols * 2);
    long long* d; cudaMalloc(&d, 148 * sizeof(long long));
    void* p = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    EncFn enc = (EncFn)p;
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int g : {148, 74, 16}) { run<4, 0>(tm, rows, g, d); run<8, 0>(tm, rows, g, d); }
    run<8, 1>(tm, rows, 148, d);
    run<4, 1>(tm, rows, 148, d);
    return 0;
}
