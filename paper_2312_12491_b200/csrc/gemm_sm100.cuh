// tcgen05 / TMA GEMM and implicit-GEMM 3x3 convolution for sm_100a.
//
//   C[M, N] = act( A[M, K] . B[N, K]^T * scale + bias[N] + bias_img[m / rows_per_img][N] ) + residual[M, N]
//
// A, B bf16 K-major, fp32 accumulation in TMEM, bf16 or fp32 output.
// A sources: a 2-D row-major matrix, two matrices concatenated along K
// (decoder skip concat), or an NHWC activation read through a 4-D TMA box at
// tap-shifted coordinates (implicit im2col: zero padding comes from TMA
// out-of-bounds fill, stride-2 from TMA element strides).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <memory>

namespace sdx {

enum { kActNone = 0, kActSilu = 1, kActRelu = 2, kActGelu = 3 };
enum { kAMatrix = 0, kAConcat = 1, kAConv = 2, kAHalo = 3 };

// GroupNorm statistics accumulated in the epilogue of the GEMM that produces
// the normalised tensor: per (image, group) sum and sum of squares of the
// stored (bf16-rounded) outputs as 2^-20 fixed-point int64 atomics, which are
// exact and order-independent, so the statistics are deterministic.
struct GnSink {
    unsigned long long* acc = nullptr;  // [images][groups][2]
    int c_off = 0;                      // channel offset of this tensor inside the GN input
    int cg = 1;                         // channels per group
    int groups = 32;
    long long hw = 1;                   // rows per image
};
constexpr float kGnFixedScale = 1048576.f;  // 2^20

struct GemmEpilogue {
    const float* bias = nullptr;          // [N]
    const float* bias_img = nullptr;      // [images][N] (time-embedding projection)
    long long rows_per_img = 1;
    const int* img_index = nullptr;       // image -> row of bias_img (per-row schedule step) or null
    long long bias_img_ld = 0;            // row pitch of bias_img (0 = N)
    const __nv_bfloat16* residual = nullptr;  // [M][ld_res]
    long long ld_res = 0;
    int act = kActNone;
    float scale = 1.f;
    void* out = nullptr;
    long long ld_out = 0;
    int out_f32 = 0;                      // 0 bf16, 1 fp32, 2 u8 (round(255 * clamp(v, 0, 1))), 3 fp16
    int act_after_residual = 0;           // act(acc + bias + residual) instead of act(acc + bias) + residual
    int geglu = 0;                        // B rows interleaved [16 value | 16 gate]: out[:, j] = a_j * gelu(g_j), N/2 cols
    int gelu_tanh = 0;                    // GEGLU gate as tanh-form GELU with tanh.approx (else erf GELU)
    const int* out_img_map = nullptr;     // image -> destination image block of rows_per_img rows (scatter)
    GnSink gn[2];                         // GroupNorm statistics of this output (up to two consumers)
    int n_gn = 0;
    const int* rows_dev = nullptr;        // device row-unit count (skip tiles past *rows_dev * rows_per_unit)
    long long rows_per_unit = 0;
    // LayerNorm folded into this GEMM (fast epilogue only): A holds the raw rows x, B the
    // folded weights W' = W * gamma, and the epilogue applies
    //   out = rstd_r * (acc - mean_r * ln_s[n]) + bias[n]      (bias = b + W beta)
    // with the row statistics summed from ln_nparts partials [ln_nparts][M] (sum, sumsq of
    // the bf16 A rows) written by the producer of A (row_stats_out below).
    const float2* ln_part = nullptr;
    int ln_nparts = 0;
    int ln_C = 0;
    float ln_eps = 1e-5f;
    const float* ln_s = nullptr;
    // Row statistics of this GEMM's (bf16-rounded) output for a LayerNorm-folded
    // consumer: [kRowStatParts * n_tiles][M] float2, one entry per (N tile, epilogue
    // warp of the row's quadrant) per row.
    float2* row_stats_out = nullptr;
};
constexpr int kRowStatParts = 3;  // fast-path epilogue warps per TMEM lane quadrant

// A prebuilt launch (tensor maps encoded once; replayable / graph-capturable).
struct GemmPlan {
    CUtensorMap ta, ta2, tb;
    CUtensorMap to;                     // output (bf16 [M][ld_out]) or split-K partials (fp32 [splits][M][N]) for TMA stores
    bool fast = false;                  // streamlined TMA-store epilogue (see gemm_tc_kernel)
    bool pair = false;                  // CTA-pair 2-SM MMA (M = 256 per pair; needs fast)
    int amode = kAMatrix;
    int M = 0, N = 0, K = 0, K1 = 0;   // K1: split point of the concat source
    int bn = 128;
    // conv geometry (amode == kAConv)
    int H = 0, W = 0, Cin = 0, Ho = 0, Wo = 0, stride = 1, Wt = 0, Ht = 0, Nt = 0;
    GemmEpilogue epi;
    int splits = 1;                     // split-K factor (chosen when tiles cannot fill the SMs)
    float* ws = nullptr;                // split-K fp32 partials
    std::shared_ptr<void> ws_owner;     // frees ws with the last copy of the plan
    bool valid = false;
};

// Row-major bf16 matrices: A [M][lda] (K used), B [N][ldb].
GemmPlan plan_gemm(const __nv_bfloat16* A, long long lda, const __nv_bfloat16* B, long long ldb, int M, int N, int K,
                   const GemmEpilogue& epi);
// A = [A1 (K1 cols) | A2 (K - K1 cols)] per row.
GemmPlan plan_gemm_concat(const __nv_bfloat16* A1, long long lda1, int K1, const __nv_bfloat16* A2, long long lda2,
                          const __nv_bfloat16* B, long long ldb, int M, int N, int K, const GemmEpilogue& epi);
// 3x3 conv, pad 1, stride 1 or 2: x NHWC [imgs][H][W][Cin] bf16, w [Cout][3][3][Cin] bf16,
// out NHWC [imgs][Ho][Wo][Cout].  Cin % 64 == 0.  64 -> 64 channel stride-1 convs on rows of
// >= 128 pixels (the TAESD trunk) run halo-tiled: one 3 x 130-pixel TMA box per 128-pixel output
// tile feeds all nine taps (UMMA descriptors at 128-byte pixel-row offsets) against
// weights resident in smem (SDX_CONV_HALO=0 disables).
GemmPlan plan_conv3x3(const __nv_bfloat16* x, int imgs, int H, int W, int Cin, const __nv_bfloat16* w, int Cout,
                      int stride, const GemmEpilogue& epi);

void run_gemm(const GemmPlan& p, cudaStream_t st);

// Forces the tile width / split-K factor of subsequently planned GEMMs (0 = cost
// model).  Kernel benchmarks only.
void set_gemm_tiling_override(int bn, int splits, int pair = 0);
// Device buffer [grid][16] that subsequent launches fill with %globaltimer phase
// stamps per CTA (entry, setup done, first stage landed, first tile committed,
// epilogue start / end, exit); null disables.  Kernel benchmarks only.
void set_gemm_debug_buffer(unsigned long long* dbg);
// Pipeline probes (results wrong): 1 = TMA only (no MMAs), 2 = MMA only (no loads), 4 = no epilogue work.
void set_gemm_probe_mode(int mode);
// Modelled cost (SM clocks) of one tiling; see choose_tiling in gemm_sm100.cu.
double gemm_cost(long long M, int N, int K, int bn, int splits, int out_bytes, bool residual, bool pair);

}  // namespace sdx
