// extern "C" kernel-level entry points (include/stagger_b200_kernels.h).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <string>

#include "common.cuh"
#include "attention_sm100.cuh"
#include "gemm_sm100.cuh"
#include "stagger_b200_kernels.h"
#include "taesd.cuh"
#include "unet.cuh"
#include <memory>
#include <numeric>
#include <vector>

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

int sdx_kernel_groupnorm_debug(void* dbg) {
    return kguard([&] { sdx::set_groupnorm_debug_buffer(static_cast<long long*>(dbg)); });
}

int sdx_kernel_groupnorm(const void* x1, int C1, const void* x2, int C2, int HW, int imgs, float eps,
                         const float* gamma, const float* beta, int silu, void* out, void* arena, int iters,
                         void* stream) {
    return kguard([&] {
        if (!arena || imgs < 1 || HW < 1 || iters < 1) sdx::raise(SDX_INVALID_ARGUMENT, "groupnorm: bad arguments");
        auto* acc = static_cast<unsigned long long*>(arena);
        auto p = sdx::plan_groupnorm(static_cast<const bf16*>(x1), C1, static_cast<const bf16*>(x2), C2, HW, imgs, eps,
                                     gamma, beta, silu, static_cast<bf16*>(out), nullptr, acc,
                                     acc + static_cast<long long>(imgs) * 64);
        const auto st = static_cast<cudaStream_t>(stream);
        // timing breakdown knob (tools/gn_bench.py): bit 0 zero, bit 1 statistics, bit 2 apply
        const char* pe = std::getenv("SDX_GN_PARTS");
        const int parts = pe ? std::atoi(pe) : 7;
        for (int i = 0; i < iters; ++i) {
            if (parts & 1)
                SDX_CUDA(cudaMemsetAsync(acc, 0, sizeof(unsigned long long) * (static_cast<size_t>(imgs) * 64 + 1), st));
            if ((parts & 6) == 6) {
                sdx::run_groupnorm(p, st);
            } else if (parts & 6) {
                auto q = p;
                q.stats_fused = (parts & 2) ? 0 : 1;
                sdx::run_groupnorm_part(q, (parts & 2) ? 0 : 1, st);
            }
        }
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

struct sdx_gemm_plan {
    sdx::GemmPlan p;
};

namespace {
struct TilingOverride {
    // bn < 0: CTA-pair tile of width -bn
    TilingOverride(int bn, int s) { sdx::set_gemm_tiling_override(bn < 0 ? -bn : bn, s, bn < 0 ? 1 : 0); }
    ~TilingOverride() { sdx::set_gemm_tiling_override(0, 0, 0); }
};
}  // namespace

int sdx_kernel_gemm_plan(const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int M, int N, int K,
                         const float* bias, const void* residual, int act, int out_f32, int force_bn,
                         int force_splits, sdx_gemm_plan** out) {
    return kguard([&] {
        sdx::GemmEpilogue e;
        e.bias = bias;
        e.residual = static_cast<const bf16*>(residual);
        e.act = act;
        e.out = C;
        e.out_f32 = out_f32;
        TilingOverride ov(force_bn, force_splits);
        auto* h = new sdx_gemm_plan{sdx::plan_gemm(static_cast<const bf16*>(A), lda, static_cast<const bf16*>(B), ldb,
                                                   M, N, K, e)};
        *out = h;
    });
}

int sdx_kernel_conv3x3_plan(const void* x, int imgs, int H, int W, int Cin, const void* w, int Cout, int stride,
                            const float* bias, const void* residual, int act, void* out, int out_f32, int force_bn,
                            int force_splits, sdx_gemm_plan** out_plan) {
    return kguard([&] {
        sdx::GemmEpilogue e;
        e.bias = bias;
        e.residual = static_cast<const bf16*>(residual);
        e.act = act;
        e.out = out;
        e.out_f32 = out_f32;
        TilingOverride ov(force_bn, force_splits);
        *out_plan = new sdx_gemm_plan{sdx::plan_conv3x3(static_cast<const bf16*>(x), imgs, H, W, Cin,
                                                        static_cast<const bf16*>(w), Cout, stride, e)};
    });
}

int sdx_kernel_plan_run(sdx_gemm_plan* p, int iters, void* stream) {
    return kguard([&] {
        if (!p) sdx::raise(SDX_INVALID_ARGUMENT, "null plan");
        for (int i = 0; i < iters; ++i) sdx::run_gemm(p->p, static_cast<cudaStream_t>(stream));
    });
}

int sdx_kernel_plan_info(sdx_gemm_plan* p, int* bn, int* splits, double* model_clk) {
    return kguard([&] {
        if (!p) sdx::raise(SDX_INVALID_ARGUMENT, "null plan");
        *bn = p->p.pair ? -p->p.bn : p->p.bn;
        *splits = p->p.splits;
        const int ob = p->p.epi.out_f32 == 1 ? 4 : (p->p.epi.out_f32 == 2 ? 1 : 2);
        *model_clk = sdx::gemm_cost(p->p.M, p->p.N, p->p.K, p->p.bn, p->p.splits, ob, p->p.epi.residual != nullptr,
                                    p->p.pair);
    });
}

int sdx_kernel_gemm_debug(void* dbg) {
    return kguard([&] { sdx::set_gemm_debug_buffer(static_cast<unsigned long long*>(dbg)); });
}

int sdx_kernel_gemm_probe(int mode) {
    return kguard([&] { sdx::set_gemm_probe_mode(mode); });
}

int sdx_kernel_attention_probe(int mode) {
    return kguard([&] { sdx::set_attention_probe_mode(mode); });
}
int sdx_kernel_attention_debug(void* dbg) {
    return kguard([&] { sdx::set_attention_debug_buffer(static_cast<long long*>(dbg)); });
}

int sdx_kernel_plan_destroy(sdx_gemm_plan* p) {
    return kguard([&] { delete p; });
}

// ---- TAESD codec on its own (numerics tests / kernel tools) -------------------------
struct sdx_taesd {
    sdx::TAESD* t = nullptr;
    int imax = 0;
    int *src = nullptr, *dst = nullptr, *enc_cnt = nullptr, *dec_cnt = nullptr;
    uint8_t *frames_in = nullptr, *frames_out = nullptr;
    float *lat_out = nullptr, *lat_in = nullptr;
};

int sdx_taesd_create(int imax, uint64_t seed, int device, sdx_taesd** out) {
    return kguard([&] {
        if (imax < 1) sdx::raise(SDX_INVALID_ARGUMENT, "taesd: imax must be >= 1");
        SDX_CUDA(cudaSetDevice(device));
        auto* h = new sdx_taesd;
        h->imax = imax;
        const size_t fb = 512ull * 512 * 3, lb = 64ull * 64 * 4;
        h->src = sdx::dev_alloc<int>(imax);
        h->dst = sdx::dev_alloc<int>(imax);
        h->enc_cnt = sdx::dev_alloc<int>(1);
        h->dec_cnt = sdx::dev_alloc<int>(1);
        h->frames_in = sdx::dev_alloc<uint8_t>(fb * imax);
        h->frames_out = sdx::dev_alloc<uint8_t>(fb * imax);
        h->lat_out = sdx::dev_alloc<float>(lb * imax);
        h->lat_in = sdx::dev_alloc<float>(lb * imax);
        std::vector<int> iota(static_cast<size_t>(imax));
        std::iota(iota.begin(), iota.end(), 0);
        SDX_CUDA(cudaMemcpy(h->src, iota.data(), sizeof(int) * imax, cudaMemcpyHostToDevice));
        SDX_CUDA(cudaMemcpy(h->dst, iota.data(), sizeof(int) * imax, cudaMemcpyHostToDevice));
        sdx::TaesdIO io;
        io.frames = h->frames_in;
        io.frame_stride = static_cast<long long>(fb);
        io.enc_src = h->src;
        io.enc_count = h->enc_cnt;
        io.latent_out = h->lat_out;
        io.enc_dst = h->dst;
        io.latent_in = h->lat_in;
        io.dec_src = h->src;
        io.dec_count = h->dec_cnt;
        io.frames_out = h->frames_out;
        io.dec_dst = h->dst;
        h->t = new sdx::TAESD(imax, seed, io, nullptr);
        *out = h;
    });
}

int sdx_taesd_destroy(sdx_taesd* h) {
    return kguard([&] {
        if (!h) return;
        delete h->t;
        for (void* p : {static_cast<void*>(h->src), static_cast<void*>(h->dst), static_cast<void*>(h->enc_cnt),
                        static_cast<void*>(h->dec_cnt), static_cast<void*>(h->frames_in),
                        static_cast<void*>(h->frames_out), static_cast<void*>(h->lat_out), static_cast<void*>(h->lat_in)})
            sdx::dev_free(p);
        delete h;
    });
}

int sdx_taesd_encode(sdx_taesd* h, const uint8_t* frames, int n, float* latents, void* stream) {
    return kguard([&] {
        if (!h || n < 1 || n > h->imax) sdx::raise(SDX_INVALID_ARGUMENT, "taesd_encode: 1 <= n <= imax");
        auto st = static_cast<cudaStream_t>(stream);
        SDX_CUDA(cudaMemcpyAsync(h->frames_in, frames, 512ull * 512 * 3 * n, cudaMemcpyDeviceToDevice, st));
        SDX_CUDA(cudaMemcpyAsync(h->enc_cnt, &n, sizeof(int), cudaMemcpyHostToDevice, st));
        h->t->encode(st);
        SDX_CUDA(cudaMemcpyAsync(latents, h->lat_out, 64ull * 64 * 4 * sizeof(float) * n, cudaMemcpyDeviceToDevice, st));
        SDX_CUDA(cudaStreamSynchronize(st));
    });
}

int sdx_taesd_decode(sdx_taesd* h, const float* latents, int n, uint8_t* frames, void* stream) {
    return kguard([&] {
        if (!h || n < 1 || n > h->imax) sdx::raise(SDX_INVALID_ARGUMENT, "taesd_decode: 1 <= n <= imax");
        auto st = static_cast<cudaStream_t>(stream);
        SDX_CUDA(cudaMemcpyAsync(h->lat_in, latents, 64ull * 64 * 4 * sizeof(float) * n, cudaMemcpyDeviceToDevice, st));
        SDX_CUDA(cudaMemcpyAsync(h->dec_cnt, &n, sizeof(int), cudaMemcpyHostToDevice, st));
        h->t->decode(st);
        SDX_CUDA(cudaMemcpyAsync(frames, h->frames_out, 512ull * 512 * 3 * n, cudaMemcpyDeviceToDevice, st));
        SDX_CUDA(cudaStreamSynchronize(st));
    });
}

// Per-op device times of the encoder (decoder = 0) or decoder (1) at n live images.
int sdx_taesd_profile(sdx_taesd* h, int decoder, int n, int cap, const char** labels, double* flops, float* ms,
                      int* count) {
    return kguard([&] {
        if (!h || n < 1 || n > h->imax) sdx::raise(SDX_INVALID_ARGUMENT, "taesd_profile: 1 <= n <= imax");
        static thread_local std::vector<std::tuple<std::string, double, float>> res;
        SDX_CUDA(cudaMemcpy(decoder ? h->dec_cnt : h->enc_cnt, &n, sizeof(int), cudaMemcpyHostToDevice));
        h->t->profile(decoder != 0, &res);
        const int k = static_cast<int>(res.size());
        for (int i = 0; i < k && i < cap; ++i) {
            labels[i] = std::get<0>(res[static_cast<size_t>(i)]).c_str();
            flops[i] = std::get<1>(res[static_cast<size_t>(i)]) * n;
            ms[i] = std::get<2>(res[static_cast<size_t>(i)]);
        }
        *count = k;
    });
}

int sdx_taesd_param_count(sdx_taesd* h, int* n) {
    return kguard([&] { *n = static_cast<int>(h->t->params().size()); });
}

int sdx_taesd_param(sdx_taesd* h, int i, const char** name, void** ptr, int64_t* shape, int* ndim, int* is_f32) {
    return kguard([&] {
        const auto& p = h->t->params().at(static_cast<size_t>(i));
        *name = p.name.c_str();
        *ptr = p.ptr;
        *ndim = static_cast<int>(p.shape.size());
        for (size_t k = 0; k < p.shape.size() && k < 4; ++k) shape[k] = p.shape[k];
        *is_f32 = p.f32 ? 1 : 0;
    });
}

struct sdx_unet {
    sdx::UNet* net;
};

int sdx_unet_create(int rmax, const int* taus, int n_steps, uint64_t seed, int device, sdx_unet** out) {
    return kguard([&] {
        SDX_CUDA(cudaSetDevice(device));
        sdx::UNetConfig c;
        c.rmax = rmax;
        c.taus.assign(taus, taus + n_steps);
        c.seed = seed;
        *out = new sdx_unet{new sdx::UNet(c, nullptr)};
    });
}

int sdx_unet_destroy(sdx_unet* u) {
    return kguard([&] {
        if (u) delete u->net;
        delete u;
    });
}

int sdx_unet_forward(sdx_unet* u, const float* x, int rows, const int* row_step, const int* row_prompt, float* eps,
                     void* stream) {
    return kguard([&] {
        auto* n = u->net;
        const int R = n->config().rmax;
        if (rows < 1 || rows > R) sdx::raise(SDX_INVALID_ARGUMENT, "unet: rows out of range");
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const size_t elems = static_cast<size_t>(rows) * 64 * 64 * 4;
        if (x) SDX_CUDA(cudaMemcpyAsync(n->input(), x, elems * sizeof(float), cudaMemcpyDeviceToDevice, st));
        if (row_step) SDX_CUDA(cudaMemcpyAsync(n->row_step(), row_step, sizeof(int) * rows, cudaMemcpyHostToDevice, st));
        if (row_prompt)
            SDX_CUDA(cudaMemcpyAsync(n->row_prompt(), row_prompt, sizeof(int) * rows, cudaMemcpyHostToDevice, st));
        static thread_local int* d_rows = nullptr;
        if (!d_rows) SDX_CUDA(cudaMalloc(&d_rows, sizeof(int)));
        SDX_CUDA(cudaMemcpyAsync(d_rows, &rows, sizeof(int), cudaMemcpyHostToDevice, st));
        n->forward(d_rows, st);
        if (eps) SDX_CUDA(cudaMemcpyAsync(eps, n->output(), elems * sizeof(float), cudaMemcpyDeviceToDevice, st));
        SDX_CUDA(cudaStreamSynchronize(st));
    });
}

// Device time of whole forwards at `rows` rows: one forward captured in a CUDA graph,
// replayed `iters` times back to back (weights stream from HBM every forward, as in
// the pipeline: 1.7 GB of them do not stay in the 126 MB L2), CUDA events around
// the replays.  Kernel benchmarks / tools only.
int sdx_unet_time_forward(sdx_unet* u, int rows, int iters, float* ms_per_forward) {
    return kguard([&] {
        auto* n = u->net;
        if (rows < 1 || rows > n->config().rmax || iters < 1) sdx::raise(SDX_INVALID_ARGUMENT, "unet: bad rows/iters");
        cudaStream_t st;
        SDX_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        int* d_rows = nullptr;
        SDX_CUDA(cudaMalloc(&d_rows, sizeof(int)));
        SDX_CUDA(cudaMemcpy(d_rows, &rows, sizeof(int), cudaMemcpyHostToDevice));
        n->forward(d_rows, st);  // warm-up outside the graph
        SDX_CUDA(cudaStreamSynchronize(st));
        cudaGraph_t g;
        cudaGraphExec_t ge;
        SDX_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        n->forward(d_rows, st);
        SDX_CUDA(cudaStreamEndCapture(st, &g));
        SDX_CUDA(cudaGraphInstantiate(&ge, g, 0));
        SDX_CUDA(cudaGraphLaunch(ge, st));
        SDX_CUDA(cudaStreamSynchronize(st));
        cudaEvent_t e0, e1;
        SDX_CUDA(cudaEventCreate(&e0));
        SDX_CUDA(cudaEventCreate(&e1));
        SDX_CUDA(cudaEventRecord(e0, st));
        for (int i = 0; i < iters; ++i) SDX_CUDA(cudaGraphLaunch(ge, st));
        SDX_CUDA(cudaEventRecord(e1, st));
        SDX_CUDA(cudaEventSynchronize(e1));
        float ms = 0.f;
        SDX_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        *ms_per_forward = ms / static_cast<float>(iters);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
        cudaFree(d_rows);
        cudaStreamDestroy(st);
    });
}

int sdx_unet_param_count(sdx_unet* u, int* n) {
    return kguard([&] { *n = static_cast<int>(u->net->params().size()); });
}

int sdx_unet_param(sdx_unet* u, int i, const char** name, void** ptr, int64_t* shape, int* ndim, int* is_f32) {
    return kguard([&] {
        const auto& p = u->net->params().at(static_cast<size_t>(i));
        *name = p.name.c_str();
        *ptr = p.ptr;
        *ndim = static_cast<int>(p.shape.size());
        for (size_t k = 0; k < p.shape.size() && k < 4; ++k) shape[k] = p.shape[k];
        *is_f32 = p.f32 ? 1 : 0;
    });
}

int sdx_unet_flops_per_row(sdx_unet* u, double* flops) {
    return kguard([&] { *flops = u->net->flops_per_row(); });
}

// Per-op device times of one forward at `rows` rows: kinds[i] (static strings) and ms[i].
int sdx_unet_profile(sdx_unet* u, int rows, int cap, const char** kinds, float* ms, int* count) {
    return kguard([&] {
        static thread_local int* d_rows = nullptr;
        static thread_local std::vector<std::pair<std::string, float>> res;
        if (!d_rows) SDX_CUDA(cudaMalloc(&d_rows, sizeof(int)));
        SDX_CUDA(cudaMemcpy(d_rows, &rows, sizeof(int), cudaMemcpyHostToDevice));
        u->net->forward_profiled(d_rows, nullptr, &res);
        const int n = static_cast<int>(res.size());
        for (int i = 0; i < n && i < cap; ++i) {
            kinds[i] = res[static_cast<size_t>(i)].first.c_str();
            ms[i] = res[static_cast<size_t>(i)].second;
        }
        *count = n;
    });
}

// Same, with each op's label (kind + GEMM/attention shape) and algorithmic FLOPs at rmax rows.
int sdx_unet_profile_detail(sdx_unet* u, int rows, int cap, const char** labels, double* flops, float* ms,
                            int* count) {
    return kguard([&] {
        static thread_local int* d_rows = nullptr;
        static thread_local std::vector<std::pair<std::string, float>> res;
        if (!d_rows) SDX_CUDA(cudaMalloc(&d_rows, sizeof(int)));
        SDX_CUDA(cudaMemcpy(d_rows, &rows, sizeof(int), cudaMemcpyHostToDevice));
        u->net->forward_profiled(d_rows, nullptr, &res);
        const int n = static_cast<int>(res.size());
        for (int i = 0; i < n && i < cap; ++i) {
            labels[i] = u->net->op_label(static_cast<size_t>(i)).c_str();
            flops[i] = u->net->op_flops(static_cast<size_t>(i));
            ms[i] = res[static_cast<size_t>(i)].second;
        }
        *count = n;
    });
}

int sdx_memcpy_d2d(void* dst, const void* src, int64_t bytes) {
    return kguard([&] { SDX_CUDA(cudaMemcpy(dst, src, static_cast<size_t>(bytes), cudaMemcpyDeviceToDevice)); });
}

}  // extern "C"

#include <cuda_profiler_api.h>

extern "C" {
// Bracket a region for `ncu --profile-from-start off` (bench.py --profile-window).
int sdx_profiler_start(void) { return kguard([&] { SDX_CUDA(cudaProfilerStart()); }); }
int sdx_profiler_stop(void) { return kguard([&] { SDX_CUDA(cudaProfilerStop()); }); }

// Measured denoise loops for the bench tables (bench.cpp:225-244, engine.cpp:213-309):
// one CUDA graph of [TAESD encode of `frames` frames, `calls` UNet calls of
// `rows_per_call` rows, TAESD decode of `frames` frames], replayed `iters` times and
// timed with CUDA events.  sequential = (1 row, n calls, 1 frame) per frame;
// wait-and-batch = (n rows, n calls, n frames) per n frames.
int sdx_bench_denoise_loop(int rows_per_call, int calls, int frames, int n_steps, int iters, uint64_t seed,
                           int device, double* ms_per_iter) {
    return kguard([&] {
        if (rows_per_call < 1 || calls < 1 || frames < 1 || n_steps < 1 || iters < 1 || !ms_per_iter)
            sdx::raise(SDX_INVALID_ARGUMENT, "bench_denoise_loop: bad arguments");
        SDX_CUDA(cudaSetDevice(device));
        std::vector<sdx_step> steps(static_cast<size_t>(n_steps));
        if (sdx_build_schedule(n_steps, 1000, 1.0, steps.data()) != 0)
            sdx::raise(SDX_INVALID_ARGUMENT, sdx_precompute_error());
        sdx::UNetConfig c;
        c.rmax = rows_per_call;
        for (const auto& s : steps) c.taus.push_back(s.tau);
        c.seed = seed;
        sdx_taesd* t = nullptr;
        if (sdx_taesd_create(frames, seed ^ 0x7AE5DULL, device, &t) != SDX_OK) sdx::raise(SDX_CUDA_ERROR, g_kerr);
        std::unique_ptr<sdx_taesd, int (*)(sdx_taesd*)> tguard(t, sdx_taesd_destroy);
        sdx::UNet net(c, nullptr);
        int* d_rows = sdx::dev_alloc<int>(1);
        std::vector<int> hs(static_cast<size_t>(rows_per_call)), hp(static_cast<size_t>(rows_per_call), 0);
        for (int r = 0; r < rows_per_call; ++r) hs[static_cast<size_t>(r)] = r % n_steps;
        SDX_CUDA(cudaMemcpy(net.row_step(), hs.data(), sizeof(int) * hs.size(), cudaMemcpyHostToDevice));
        SDX_CUDA(cudaMemcpy(net.row_prompt(), hp.data(), sizeof(int) * hp.size(), cudaMemcpyHostToDevice));
        SDX_CUDA(cudaMemcpy(d_rows, &rows_per_call, sizeof(int), cudaMemcpyHostToDevice));
        SDX_CUDA(cudaMemcpy(t->enc_cnt, &frames, sizeof(int), cudaMemcpyHostToDevice));
        SDX_CUDA(cudaMemcpy(t->dec_cnt, &frames, sizeof(int), cudaMemcpyHostToDevice));
        SDX_CUDA(cudaMemset(t->frames_in, 77, 512ull * 512 * 3 * frames));
        const size_t lat = 64ull * 64 * 4 * sizeof(float);
        const size_t moved = lat * static_cast<size_t>(std::min(rows_per_call, frames));
        cudaStream_t st = nullptr;
        SDX_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        auto body = [&] {
            t->t->encode(st);
            SDX_CUDA(cudaMemcpyAsync(net.input(), t->lat_out, moved, cudaMemcpyDeviceToDevice, st));
            for (int i = 0; i < calls; ++i) net.forward(d_rows, st);
            SDX_CUDA(cudaMemcpyAsync(t->lat_in, net.output(), moved, cudaMemcpyDeviceToDevice, st));
            t->t->decode(st);
        };
        body();  // plans, first-launch attributes
        SDX_CUDA(cudaStreamSynchronize(st));
        cudaGraph_t g = nullptr;
        cudaGraphExec_t ge = nullptr;
        SDX_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        body();
        SDX_CUDA(cudaStreamEndCapture(st, &g));
        SDX_CUDA(cudaGraphInstantiate(&ge, g, 0));
        for (int i = 0; i < 3; ++i) SDX_CUDA(cudaGraphLaunch(ge, st));
        cudaEvent_t e0, e1;
        SDX_CUDA(cudaEventCreate(&e0));
        SDX_CUDA(cudaEventCreate(&e1));
        SDX_CUDA(cudaEventRecord(e0, st));
        for (int i = 0; i < iters; ++i) SDX_CUDA(cudaGraphLaunch(ge, st));
        SDX_CUDA(cudaEventRecord(e1, st));
        SDX_CUDA(cudaEventSynchronize(e1));
        float ms = 0.f;
        SDX_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        *ms_per_iter = static_cast<double>(ms) / iters;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
        cudaStreamDestroy(st);
        sdx::dev_free(d_rows);
    });
}

}
