// HBM-bound helper kernels of the UNet / TAESD forward (nn_kernels.cu).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace sdx {

using bf16 = __nv_bfloat16;

// GroupNorm over NHWC (optionally over the channel concat [x1 | x2]), 32
// groups, fp32 statistics, affine, optional SiLU, bf16 out [imgs][HW][C1+C2].
struct GnPlan {
    const bf16* x1;
    const bf16* x2;
    int C1, C2, HW, groups;
    float eps;
    const float *gamma, *beta;
    int silu;
    bf16* out;
    // per (image, group) sum and sum of squares, 2^-20 fixed point int64 (exact,
    // order-independent adds); zeroed by the owner before every forward.  Filled
    // by gn_stats_kernel, or by the producing GEMM epilogues when stats_fused.
    unsigned long long* acc;
    int stats_fused;
    int px_per_block, chunks;  // pixel range per block (both kernels), blocks per image
    // single-launch statistics + apply (gn_fused_kernel): grid-wide arrival counter,
    // zeroed with the arena before each forward; fused = grid fits co-resident
    unsigned long long* counter;
    int fused;
    int imgs;
    const int* rows_dev;
    // single launch, one thread-block cluster of `cluster` CTAs per image (DSMEM
    // statistics), pixel ranges streamed through shared memory in `piece`-pixel pieces
    int cluster, piece;
    long long* dbg = nullptr;  // cluster kernel phase stamps [img * cluster + rank][8] (kernel benchmarks)
};
GnPlan plan_groupnorm(const bf16* x1, int C1, const bf16* x2, int C2, int HW, int imgs, float eps, const float* gamma,
                      const float* beta, int silu, bf16* out, const int* rows_dev, unsigned long long* acc,
                      unsigned long long* counter = nullptr);
void run_groupnorm(const GnPlan& p, cudaStream_t st);
// one pass of the pair (0 statistics, 1 apply), for timing
void run_groupnorm_part(const GnPlan& p, int part, cudaStream_t st);
void free_groupnorm(GnPlan& p);
// Device buffer that subsequent cluster GroupNorm launches fill with per-CTA %globaltimer
// phase stamps (entry, after the PDL wait, first piece landed, statistics summed, cluster
// barrier, group statistics, apply done, exit); null disables.  Kernel benchmarks only.
void set_groupnorm_debug_buffer(long long* dbg);

// LayerNorm over the last dim C of [rows][C] (fp32 stats), bf16 out.
void run_layernorm(const bf16* x, int rows, int C, const float* gamma, const float* beta, float eps, bf16* out,
                   const int* rows_dev, int rows_per_unit, cudaStream_t st);

// GEGLU: out[r][j] = a[r][j] * gelu(g[r][j]) with a = in[:, :H], g = in[:, H:2H]
void run_geglu(const bf16* in, int rows, int H, bf16* out, const int* rows_dev, int rows_per_unit, cudaStream_t st);

// nearest 2x upsample, NHWC
void run_upsample2x(const bf16* in, int imgs, int H, int W, int C, bf16* out, const int* rows_dev, cudaStream_t st);

// 3x3/pad1 im2col of a small-channel NHWC input (C <= 7) into [imgs*H*W][Kp] bf16,
// column = tap*C + c, zero padded to Kp (multiple of 64).  Source is fp32 or u8
// (u8 scaled by 1/255, the TAESD input range) with an optional per-image gather.
void run_im2col3x3_f32(const float* in, int imgs, int H, int W, int C, int Kp, bf16* out, const int* rows_dev,
                       cudaStream_t st);
void run_im2col3x3_f32_gather(const float* in, long long img_stride, const int* img_src, int imgs, int H, int W, int C,
                              int Kp, int tanh_clamp, bf16* out, const int* rows_dev, cudaStream_t st);
void run_im2col3x3_u8(const uint8_t* in, long long img_stride, const int* img_src, int imgs, int H, int W, int C,
                      int Kp, bf16* out, const int* rows_dev, cudaStream_t st);

// Direct 3x3 / pad 1 conv of u8 NHWC RGB frames (scaled 1/255) to 64 bf16 channels:
// w [64][ldw] bf16 with column k = tap * 3 + c (k < 27), bias [64] or null.
// 3x3 conv (pad 1) from 64 channels NHWC bf16 to Cout = 3 channels, u8 output
// round(255 clamp(v, 0, 1)), image n written to output image img_map[n] (TAESD decoder head).
// w [Cout][3][3][64] bf16, bias fp32 (or null); images >= *rows_dev skipped.
void run_conv3x3_c64_u8(const bf16* in, int imgs, int H, int W, const bf16* w, int Cout, const float* bias,
                        uint8_t* out, const int* img_map, const int* rows_dev, cudaStream_t st);
void run_conv3x3_rgb8(const uint8_t* in, long long img_stride, const int* img_src, int imgs, int H, int W,
                      const bf16* w, int ldw, const float* bias, bf16* out, const int* rows_dev, cudaStream_t st);

// sinusoidal timestep embedding (flip_sin_to_cos, shift 0): [n][dim] bf16
void run_timestep_embedding(const int* taus, int n, int dim, bf16* out, cudaStream_t st);

// deterministic N(0, std) / constant initialisers (counter-based hash RNG)
void fill_normal_bf16(bf16* p, long long n, float std, uint64_t seed, cudaStream_t st);
void fill_normal_f32(float* p, long long n, float std, uint64_t seed, cudaStream_t st);
void fill_const_f32(float* p, long long n, float v, cudaStream_t st);

// Reorders a GEGLU projection ([2H][K] weights, [2H] bias: value rows then gate
// rows) into 16-row blocks [value 16j.. | gate 16j..] for the fused GEMM epilogue.
void run_interleave_geglu(const bf16* w, const float* b, int H, int K, bf16* wout, float* bout, cudaStream_t st);

// LayerNorm folded into the following GEMM: Wf = bf16(W * gamma) ([N][K], gamma
// over K), s[n] = sum_k Wf[n][k], c[n] = bias[n] (or 0) + sum_k W[n][k] * beta[k].
void run_ln_fold(const bf16* W, int N, int K, const float* gamma, const float* beta, const float* bias, bf16* Wf,
                 float* s, float* c, cudaStream_t st);

// elementwise: TAESD decoder input clamp  y = tanh(x / 3) * 3  (fp32 -> fp32)
void run_tanh_clamp(const float* in, float* out, long long n, cudaStream_t st);

}  // namespace sdx
