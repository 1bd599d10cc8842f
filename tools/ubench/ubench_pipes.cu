// Microbenchmarks of the sm_100a pipes the attention softmax leans on: MUFU.EX2,
// FFMA2, FMNMX3, F2FP pack, and tcgen05.ld (TMEM -> registers) throughput.
// Each test: 148 x k CTAs, W warps each, long unrolled independent chains; prints
// warp-instructions per cycle per SM (clock64 around the loop, max over CTAs).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

template <int MODE>
__global__ void pipe_kernel(float* out, long long* cyc, int iters) {
    float v[16];
    for (int i = 0; i < 16; ++i) v[i] = 0.001f * (threadIdx.x + i);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (MODE == 0) v[i] = ex2(v[i]) * -0.5f;  // ex2 + fmul
            if (MODE == 1) v[i] = ex2(v[i]);
            if (MODE == 2) {  // ffma2 pairs
                if (i % 2 == 0) {
                    asm volatile("{\n\t.reg .b64 a, d;\n\tmov.b64 a, {%0,%1};\n\tfma.rn.ftz.f32x2 d, a, a, a;\n\tmov.b64 {%0,%1}, d;\n\t}" : "+f"(v[i]), "+f"(v[i+1]));
                }
            }
            if (MODE == 3) v[i] = fmaf(v[i], 0.999f, 0.001f);
            if (MODE == 4) {  // packed bf16x2 ex2: two exponentials per lane per instruction
                uint32_t x = __float_as_uint(v[i]);
                asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(x));
                v[i] = __uint_as_float(x);
            }
            if (MODE == 5) {  // packed f16x2 ex2
                uint32_t x = __float_as_uint(v[i]);
                asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(x));
                v[i] = __uint_as_float(x);
            }
        }
    }
    const long long t1 = clock64();
    float s = 0; for (int i = 0; i < 16; ++i) s += v[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    float* out; long long* cyc;
    cudaMalloc(&out, 148 * 8 * 1024 * sizeof(float));
    cudaMalloc(&cyc, 148 * 8 * sizeof(long long));
    const int iters = 4096;
    const char* names[] = {"ex2+fmul (1 MUFU + 1 FMUL per elem)", "ex2 chain", "ffma2 (per pair)", "ffma",
                           "ex2.bf16x2 (per pair)", "ex2.f16x2 (per pair)"};
    for (int mode = 0; mode < 6; ++mode) {
        for (int warps : {4, 8, 16}) {
            auto k = mode == 0 ? pipe_kernel<0> : mode == 1 ? pipe_kernel<1> : mode == 2 ? pipe_kernel<2> : mode == 3 ? pipe_kernel<3>
                   : mode == 4 ? pipe_kernel<4> : pipe_kernel<5>;
            k<<<148, warps * 32>>>(out, cyc, iters);
            cudaDeviceSynchronize();
            k<<<148, warps * 32>>>(out, cyc, iters);
            cudaDeviceSynchronize();
            long long h[148];
            cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
            long long mx = 0; for (auto x : h) mx = x > mx ? x : mx;
            const double ops = (double)iters * 16 * warps * (mode == 2 ? 0.5 : 1.0);  // warp-instr of the main op per SM
            printf("%-38s warps/SM %2d: %.3f warp-instr/clk/SM (%.1f lanes/clk/SM)\n", names[mode], warps, ops / mx,
                   32 * ops / mx);
        }
    }
    cudaError_t e = cudaGetLastError();
    printf("err: %s\n", cudaGetErrorString(e));
    return 0;
}
