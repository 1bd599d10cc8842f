/* stagger_b200 kernel-level entry points.
 *
 * The building blocks of the batched UNet / TAESD denoiser behind
 * DenoiserBackend::predict_eps_batch (denoiser.hpp:21-39), exposed on device
 * pointers so the numerics tests can check each sm_100a kernel against a
 * PyTorch fp32 reference of the same op.  `stream` is a cudaStream_t (NULL =
 * legacy default stream).  Tensors are bf16 unless stated; layouts NHWC /
 * row-major.  Return SDX_* status codes (stagger_b200.h).
 */
#ifndef STAGGER_B200_KERNELS_H
#define STAGGER_B200_KERNELS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* C[M,N] = act(A[M,K] . B[N,K]^T * scale + bias) + residual ; tcgen05 + TMA.
 * act: 0 none, 1 SiLU, 2 ReLU, 3 GELU(erf).  out_f32: C is fp32 else bf16. */
int sdx_kernel_gemm(const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int M, int N, int K,
                    const float* bias, const void* residual, int act, int out_f32, float scale, void* stream);
/* A = [A1 | A2] concatenated along K at column K1. */
int sdx_kernel_gemm_concat(const void* A1, int64_t lda1, int K1, const void* A2, int64_t lda2, const void* B,
                           int64_t ldb, void* C, int M, int N, int K, const float* bias, int act, int out_f32,
                           void* stream);
/* 3x3 conv, pad 1, stride 1|2, NHWC, w [Cout][3][3][Cin]; implicit GEMM via 4-D TMA.
 * bias_img: optional [imgs][Cout] per-image bias (time embedding). */
int sdx_kernel_conv3x3(const void* x, int imgs, int H, int W, int Cin, const void* w, int Cout, int stride,
                       const float* bias, const float* bias_img, const void* residual, int act, void* out,
                       int out_f32, void* stream);

/* GroupNorm (32 groups) over NHWC bf16, optionally over the channel concat
 * [x1 | x2] (decoder skip joins), + SiLU when silu != 0; fp32 affine gamma/beta.
 * arena: device scratch of imgs*64 + 1 u64 (zeroed here before every pass).
 * iters > 1 repeats the pass (zero + statistics + apply) for timing. */
int sdx_kernel_groupnorm(const void* x1, int C1, const void* x2, int C2, int HW, int imgs, float eps,
                         const float* gamma, const float* beta, int silu, void* out, void* arena, int iters,
                         void* stream);

/* Flash attention, head_dim 64, tcgen05: out[img*q_len + i][64h..] = softmax(q k^T * scale) v
 * per (image, head).  Q rows [images*q_len][ld_q] (head h at q_col0 + 64h); KV rows
 * [kv_rows_total][ld_kv] with K at k_col0 + 64h and V at v_col0 + 64h; image i reads
 * KV block kv_index[i] (or i) of kv_rows_per_img rows, kv_len of them valid. */
int sdx_kernel_attention(const void* q, int64_t q_rows_total, int64_t ld_q, int q_col0, const void* kv,
                         int64_t kv_rows_total, int64_t ld_kv, int k_col0, int v_col0, void* out, int64_t ld_out,
                         int images, int heads, int q_len, int kv_len, int kv_rows_per_img, const int* kv_index,
                         float scale, void* stream);
/* Device buffer [images * cluster][8] int64 that subsequent cluster GroupNorm launches fill with
 * per-CTA %globaltimer phase stamps; null disables (kernel benchmarks only). */
int sdx_kernel_groupnorm_debug(void* dbg);
const char* sdx_kernel_last_error(void);

/* Prebuilt GEMM / conv launches for kernel benchmarks: plan once (tensor maps,
 * split-K workspace), replay `iters` times back to back on `stream`.
 * force_bn / force_splits override the cost-model tiling (0 = model; force_bn < 0 =
 * CTA-pair tile of width -force_bn); plan_info reports a CTA-pair tile as bn < 0. */
typedef struct sdx_gemm_plan sdx_gemm_plan;
int sdx_kernel_gemm_plan(const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int M, int N, int K,
                         const float* bias, const void* residual, int act, int out_f32, int force_bn,
                         int force_splits, sdx_gemm_plan** out);
int sdx_kernel_conv3x3_plan(const void* x, int imgs, int H, int W, int Cin, const void* w, int Cout, int stride,
                            const float* bias, const void* residual, int act, void* out, int out_f32, int force_bn,
                            int force_splits, sdx_gemm_plan** out_plan);
int sdx_kernel_plan_run(sdx_gemm_plan* p, int iters, void* stream);
int sdx_kernel_plan_info(sdx_gemm_plan* p, int* bn, int* splits, double* model_clk);
int sdx_kernel_plan_destroy(sdx_gemm_plan* p);
/* Device u64 buffer [grid][8] for per-CTA %globaltimer phase stamps of the next
 * GEMM launches (NULL disables); see set_gemm_debug_buffer in gemm_sm100.cuh. */
int sdx_kernel_gemm_debug(void* dbg);
/* Pipeline probe for kernel experiments (results are wrong): 0 off, 1 = TMA only
 * (no MMAs), 2 = MMA only (no loads). */
int sdx_kernel_gemm_probe(int mode);
/* Same for the attention kernel: 1 = no MMAs, 2 = no softmax exponentials. */
int sdx_kernel_attention_probe(int mode);
/* Device buffer of [10 warps][64 KV blocks][8] clock64 phase stamps of CTA 0 of the next
 * attention launches (NULL disables); see attention_sm100.cu. */
int sdx_kernel_attention_debug(void* dbg);

/* The batched UNet denoiser (random-init SD-2.1/SD-turbo topology, bf16
 * weights, fp32 accumulation) used by the pipeline's predict_eps_batch slot.
 * taus: timestep of each schedule step; forward() takes rows latents x
 * (device fp32 [rows][64][64][4], NHWC) with per-row schedule step and prompt
 * (0 condition, 1 negative) and writes eps (device fp32, same shape). */
typedef struct sdx_unet sdx_unet;
int sdx_unet_create(int rmax, const int* taus, int n_steps, uint64_t seed, int device, sdx_unet** out);
int sdx_unet_destroy(sdx_unet* u);
int sdx_unet_forward(sdx_unet* u, const float* x, int rows, const int* row_step, const int* row_prompt, float* eps,
                     void* stream);
int sdx_unet_param_count(sdx_unet* u, int* n);
int sdx_unet_param(sdx_unet* u, int i, const char** name, void** ptr, int64_t* shape, int* ndim, int* is_f32);
int sdx_unet_flops_per_row(sdx_unet* u, double* flops);
// Device ms per whole forward at `rows` rows: the forward as one CUDA graph replayed `iters`
// times back to back (tools only).
int sdx_unet_time_forward(sdx_unet* u, int rows, int iters, float* ms_per_forward);
int sdx_unet_profile(sdx_unet* u, int rows, int cap, const char** kinds, float* ms, int* count);
int sdx_unet_profile_detail(sdx_unet* u, int rows, int cap, const char** labels, double* flops, float* ms,
                            int* count);
int sdx_memcpy_d2d(void* dst, const void* src, int64_t bytes);

/* The TAESD-class tiny VAE of the pipeline's codec slot on its own (random-init,
 * seeded): encode n <= imax u8 NHWC 512x512x3 frames (device) to fp32 NHWC 64x64x4
 * latents (device), decode the reverse (u8 = round(255 clamp(x, 0, 1))).  Parameters
 * are exposed like the UNet's for the fp32 restatement test. */
typedef struct sdx_taesd sdx_taesd;
int sdx_taesd_create(int imax, uint64_t seed, int device, sdx_taesd** out);
int sdx_taesd_destroy(sdx_taesd* t);
int sdx_taesd_encode(sdx_taesd* t, const uint8_t* frames, int n, float* latents, void* stream);
int sdx_taesd_decode(sdx_taesd* t, const float* latents, int n, uint8_t* frames, void* stream);
/* Per-op device times of the encoder (decoder = 0) or decoder (1) at n live images:
 * labels[i] (valid until the next call on this thread), flops[i] at n images, ms[i]. */
int sdx_taesd_profile(sdx_taesd* t, int decoder, int n, int cap, const char** labels, double* flops, float* ms,
                      int* count);
int sdx_taesd_param_count(sdx_taesd* t, int* n);
int sdx_taesd_param(sdx_taesd* t, int i, const char** name, void** ptr, int64_t* shape, int* ndim, int* is_f32);
/* Measured denoise loop for the bench tables: one CUDA graph of [TAESD encode of
 * `frames` 512x512 frames, `calls` UNet forwards of `rows_per_call` rows, TAESD decode of
 * `frames` frames] (random-init weights, seeded), replayed `iters` times; *ms_per_iter =
 * device ms per replay (CUDA events).  Sequential denoising (engine.cpp:213-238) is
 * (1, n, 1) per frame; wait-and-batch (engine.cpp:240-309) is (n, n, n) per n frames. */
int sdx_bench_denoise_loop(int rows_per_call, int calls, int frames, int n_steps, int iters, uint64_t seed,
                           int device, double* ms_per_iter);
/* cudaProfilerStart / Stop around a region (for ncu --profile-from-start off). */
int sdx_profiler_start(void);
int sdx_profiler_stop(void);

#ifdef __cplusplus
}
#endif
#endif
