// extern "C" kernel-level entry points (include/stagger_b200_kernels.h).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <string>

#include "common.cuh"
#include "attention_sm100.cuh"
#include "gemm_sm100.cuh"
#include "stagger_b200_kernels.h"

namespace {
thread_local std::string g_kerr;
template <class F>
int kguard(F&& f) {
    try {
        f();
        return SDX_OK;
    } catch (const sdx::Error& e) {
        g_kerr = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_kerr = e.what();
        return SDX_RUNTIME_ERROR;
    }
}
using bf16 = __nv_bfloat16;
}  // namespace

extern "C" {

const char* sdx_kernel_last_error(void) { return g_kerr.c_str(); }

int sdx_kernel_gemm(const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int M, int N, int K,
                    const float* bias, const void* residual, int act, int out_f32, float scale, void* stream) {
    return kguard([&] {
        sdx::GemmEpilogue e;
        e.bias = bias;
        e.residual = static_cast<const bf16*>(residual);
        e.act = act;
        e.scale = scale;
        e.out = C;
        e.out_f32 = out_f32;
        auto p = sdx::plan_gemm(static_cast<const bf16*>(A), lda, static_cast<const bf16*>(B), ldb, M, N, K, e);
        sdx::run_gemm(p, static_cast<cudaStream_t>(stream));
    });
}

int sdx_kernel_gemm_concat(const void* A1, int64_t lda1, int K1, const void* A2, int64_t lda2, const void* B,
                           int64_t ldb, void* C, int M, int N, int K, const float* bias, int act, int out_f32,
                           void* stream) {
    return kguard([&] {
        sdx::GemmEpilogue e;
        e.bias = bias;
        e.act = act;
        e.out = C;
        e.out_f32 = out_f32;
        auto p = sdx::plan_gemm_concat(static_cast<const bf16*>(A1), lda1, K1, static_cast<const bf16*>(A2), lda2,
                                       static_cast<const bf16*>(B), ldb, M, N, K, e);
        sdx::run_gemm(p, static_cast<cudaStream_t>(stream));
    });
}

int sdx_kernel_conv3x3(const void* x, int imgs, int H, int W, int Cin, const void* w, int Cout, int stride,
                       const float* bias, const float* bias_img, const void* residual, int act, void* out,
                       int out_f32, void* stream) {
    return kguard([&] {
        sdx::GemmEpilogue e;
        e.bias = bias;
        e.bias_img = bias_img;
        const int Ho = stride == 1 ? H : (H + 1) / 2;
        const int Wo = stride == 1 ? W : (W + 1) / 2;
        e.rows_per_img = static_cast<long long>(Ho) * Wo;
        e.residual = static_cast<const bf16*>(residual);
        e.act = act;
        e.out = out;
        e.out_f32 = out_f32;
        auto p = sdx::plan_conv3x3(static_cast<const bf16*>(x), imgs, H, W, Cin, static_cast<const bf16*>(w), Cout,
                                   stride, e);
        sdx::run_gemm(p, static_cast<cudaStream_t>(stream));
    });
}

int sdx_kernel_attention(const void* q, int64_t q_rows_total, int64_t ld_q, int q_col0, const void* kv,
                         int64_t kv_rows_total, int64_t ld_kv, int k_col0, int v_col0, void* out, int64_t ld_out,
                         int images, int heads, int q_len, int kv_len, int kv_rows_per_img, const int* kv_index,
                         float scale, void* stream) {
    return kguard([&] {
        auto p = sdx::plan_attention(static_cast<const bf16*>(q), q_rows_total, ld_q, q_col0,
                                     static_cast<const bf16*>(kv), kv_rows_total, ld_kv, k_col0, v_col0,
                                     static_cast<bf16*>(out), ld_out, 0, images, heads, q_len, q_len, kv_len,
                                     kv_rows_per_img, kv_index, nullptr, scale);
        sdx::run_attention(p, static_cast<cudaStream_t>(stream));
    });
}

}  // extern "C"
