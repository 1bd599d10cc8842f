// Does a warp blocked in tcgen05.mma issue slow the other warps of its SM sub-partition?
// Warp 0 (SMSP 0) issues back-to-back MMAs (or idles); warps 1..7 run FFMA chains.  The
// FFMA rate of warp 4 (SMSP 0, shares with the MMA warp) vs warps 5..7 (SMSPs 1..3).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "sm100.cuh"
using namespace sdx::sm100;

__device__ __forceinline__ void umma_ss_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

template <int MMA, int N>
__global__ void __launch_bounds__(256, 1) k(long long* out, float* sink, int n_mma, int n_fma) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 49152);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
    for (int i = threadIdx.x; i < 49152 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) { mbar_init(bar, 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc(slot, 512);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    if (warp == 0) {
        if (MMA) {
            constexpr uint32_t idesc = idesc_bf16(128, N);
            const uint64_t da = desc_kmajor_sw128(smem_u32(sm));
            const uint64_t db = desc_kmajor_sw128(smem_u32(sm + 16384));
            for (int i = 0; i < n_mma; ++i) umma_ss_elect(tmem, da + 2 * (i & 3), db + 2 * (i & 3), idesc, i > 0);
            asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                         "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar)) : "memory");
            mbar_wait(bar, 0);
        }
    } else {
        float v[8];
        for (int i = 0; i < 8; ++i) v[i] = threadIdx.x * 0.001f + i;
        const long long t0 = clock64();
        for (int it = 0; it < n_fma; ++it)
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = fmaf(v[i], 0.9999f, 0.0001f);
        const long long t1 = clock64();
        float s = 0; for (int i = 0; i < 8; ++i) s += v[i];
        sink[blockIdx.x * 256 + threadIdx.x] = s;
        if ((threadIdx.x & 31) == 0) out[blockIdx.x * 8 + warp] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int MMA, int N>
void run(long long* d, float* s) {
    auto kk = k<MMA, N>;
    const int smem = 1024 + 49152 + 64;
    cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int n_fma = 20000;
    kk<<<148, 256, smem>>>(d, s, 2000, n_fma);
    kk<<<148, 256, smem>>>(d, s, 2000, n_fma);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148 * 8];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%s N=%3d: cycles per 8-FFMA iteration by warp (SMSP):", MMA ? "MMA " : "idle", N);
    for (int w = 1; w < 8; ++w) {
        double a = 0; for (int b = 0; b < 148; ++b) a += h[b * 8 + w];
        printf("  w%d(s%d) %.2f", w, w % 4, a / 148 / n_fma);
    }
    printf("  %s\n", cudaGetErrorString(e));
}

int main() {
    long long* d; float* s;
    cudaMalloc(&d, 148 * 8 * sizeof(long long));
    cudaMalloc(&s, 148 * 256 * sizeof(float));
    run<0, 128>(d, s);
    run<1, 64>(d, s);
    run<1, 128>(d, s);
    run<1, 256>(d, s);
    return 0;
}
