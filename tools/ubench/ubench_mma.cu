// tcgen05.mma issue / execution rates on one SM per CTA (148 CTAs):
//   variant 0: issued from `if (lane == 0)` (operands in per-thread registers: the
//              compiler wraps every UTCHMMA in an ELECT / R2UR.BROADCAST loop)
//   variant 1: the whole warp runs the loop (uniform operands), one lane elected
//              inside the asm (elect.sync) issues
// Shapes: SS (A, B from smem) M128 x N x K16, and TS (A from TMEM) M128 x N x K16.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "sm100.cuh"

using namespace sdx::sm100;

__device__ __forceinline__ void umma_ss_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void umma_ts_elect(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit_elect(uint64_t* bar) {
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar)) : "memory");
}

template <int VARIANT, int TS, int N, int AOFF = 0>
__global__ void __launch_bounds__(128, 1) mma_kernel(long long* out, int n_mma) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = sm;            // 128 x 64 bf16, sw128 (16 KB)
    uint8_t* sB = sm + 16384;    // 256 x 64 bf16 (32 KB)
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 16384 + 32768);
    uint64_t* ready = bar + 1;  // VARIANT 2: a completed barrier polled before every 4 MMAs
    uint64_t* sink = bar + 2;   // VARIANT 2: committed after every 4 MMAs (never completes)
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 3);
    for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_init(ready, 1);
        mbar_init(sink, 1 << 19);
        fence_barrier_init();
        mbar_arrive(ready);  // phase 0 complete
    }
    if (warp == 0) tmem_alloc(slot, 512);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    constexpr uint32_t idesc = idesc_bf16(128, N);
    const uint64_t da = desc_kmajor_sw128(smem_u32(sA) + AOFF * 128);  // AOFF: A window start row (halo conv taps)
    const uint64_t db = desc_kmajor_sw128(smem_u32(sB));
    long long t0 = 0, t1 = 0, t2 = 0;
    if (warp == 0) {
        if (VARIANT == 0) {
            if (lane == 0) {
                t0 = clock64();
                for (int i = 0; i < n_mma; ++i) {
                    const int k = i & 3;
                    if (TS) umma_ts(tmem, tmem + 256 + 8 * k, db + 2 * k, idesc, i > 0);
                    else umma_f16(tmem, da + 2 * k, db + 2 * k, idesc, i > 0);
                }
                t1 = clock64();
                umma_commit(bar);
                mbar_wait(bar, 0);
                t2 = clock64();
            }
        } else if (VARIANT == 2) {
            // the GEMM mainloop's per-stage skeleton: poll a (ready) full barrier, fence, 4 MMAs,
            // commit the stage's empty barrier
            t0 = clock64();
            for (int i = 0; i < n_mma; i += 4) {
                mbar_wait(ready, 0);
                tc_fence_after();
#pragma unroll
                for (int k = 0; k < 4; ++k) umma_ss_elect(tmem, da + 2 * k, db + 2 * k, idesc, (i + k) > 0);
                commit_elect(sink);
            }
            t1 = clock64();
            commit_elect(bar);
            mbar_wait(bar, 0);
            t2 = clock64();
        } else {
            t0 = clock64();
            for (int i = 0; i < n_mma; ++i) {
                const int k = i & 3;
                if (TS) umma_ts_elect(tmem, tmem + 256 + 8 * k, db + 2 * k, idesc, i > 0);
                else umma_ss_elect(tmem, da + 2 * k, db + 2 * k, idesc, i > 0);
            }
            t1 = clock64();
            commit_elect(bar);
            mbar_wait(bar, 0);
            t2 = clock64();
        }
        if (lane == 0) { out[blockIdx.x * 2] = t1 - t0; out[blockIdx.x * 2 + 1] = t2 - t0; }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int V, int TS, int N, int AOFF = 0>
void run(long long* d, const char* name) {
    const int n_mma = 2048;
    auto k = mma_kernel<V, TS, N, AOFF>;
    const int smem = 1024 + 16384 + 32768 + 64;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<148, 128, smem>>>(d, n_mma);
    k<<<148, 128, smem>>>(d, n_mma);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[296];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double iss = 0, tot = 0;
    for (int i = 0; i < 148; ++i) { iss += h[2 * i]; tot += h[2 * i + 1]; }
    iss /= 148; tot /= 148;
    const double floor_cyc = 128.0 * N / 256.0;
    printf("%-34s N=%3d: issue %6.1f cyc/MMA, total %6.1f cyc/MMA (floor %5.1f) -> %5.1f%% of floor rate  %s\n", name, N,
           iss / n_mma, tot / n_mma, floor_cyc, 100.0 * floor_cyc / (tot / n_mma), cudaGetErrorString(e));
}

int main() {
    long long* d;
    cudaMalloc(&d, 296 * sizeof(long long));
    run<2, 0, 64>(d, "SS GEMM stage skeleton (wait/fence/4/commit)");
    run<2, 0, 96>(d, "SS GEMM stage skeleton (wait/fence/4/commit)");
    run<2, 0, 160>(d, "SS GEMM stage skeleton (wait/fence/4/commit)");
    run<2, 0, 256>(d, "SS GEMM stage skeleton (wait/fence/4/commit)");
    run<1, 0, 96>(d, "SS warp+elect");
    run<1, 0, 64, 1>(d, "SS warp+elect A at row 1");
    run<1, 0, 64, 3>(d, "SS warp+elect A at row 3");
    run<1, 0, 64, 8>(d, "SS warp+elect A at row 8");
    run<1, 0, 128, 1>(d, "SS warp+elect A at row 1");
    run<1, 0, 16>(d, "SS warp+elect");
    run<1, 0, 32>(d, "SS warp+elect");
    run<0, 0, 64>(d, "SS lane0-divergent");
    run<1, 0, 64>(d, "SS warp+elect");
    run<0, 0, 128>(d, "SS lane0-divergent");
    run<1, 0, 128>(d, "SS warp+elect");
    run<0, 0, 160>(d, "SS lane0-divergent");
    run<1, 0, 160>(d, "SS warp+elect");
    run<0, 0, 256>(d, "SS lane0-divergent");
    run<1, 0, 256>(d, "SS warp+elect");
    run<0, 1, 64>(d, "TS lane0-divergent");
    run<1, 1, 64>(d, "TS warp+elect");
    run<0, 1, 128>(d, "TS lane0-divergent");
    run<1, 1, 128>(d, "TS warp+elect");
    run<1, 1, 256>(d, "TS warp+elect");
    return 0;
}
