// Random-init SD-2.1 / SD-turbo-class UNet (the Stream Batch denoiser behind
// DenoiserBackend::predict_eps_batch, denoiser.hpp:21-39) on the sm_100a
// kernels: tcgen05 implicit-GEMM convs and GEMMs, tcgen05 flash attention,
// fused GroupNorm/SiLU, per-row time embedding as a conv1 epilogue bias.
//
// Topology (diffusers UNet2DConditionModel, stabilityai/sd-turbo config):
// block_out_channels (320, 640, 1280, 1280), 2 resnets per down block, 3 per
// up block, attention at the three top levels with head_dim 64, linear
// proj_in/out, GEGLU feed-forward, cross-attention dim 1024, 77 context tokens,
// GroupNorm(32), latent 4x64x64 (512x512 frames).
//
// All launches are planned once for `rmax` rows; the live row count is read
// from device memory (rows_dev) so tiles of rows that do not exist this tick
// do no work and the forward is graph-capturable.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <deque>
#include <functional>
#include <map>
#include <string>
#include <vector>

#include "attention_sm100.cuh"
#include "gemm_sm100.cuh"
#include "nn_kernels.cuh"

namespace sdx {

struct UNetConfig {
    int rmax = 8;
    std::vector<int> taus;  // timestep of each schedule step (row_step indexes this)
    int n_prompts = 2;      // 0: condition, 1: negative
    uint64_t seed = 1234;
    int H = 64, W = 64;
    int ctx_len = 77, ctx_dim = 1024;
    int levels_channels[4] = {320, 640, 1280, 1280};
};

struct Param {
    std::string name;
    void* ptr;
    std::vector<long long> shape;
    bool f32;
};

class UNet {
  public:
    UNet(const UNetConfig& cfg, cudaStream_t st);
    ~UNet();
    UNet(const UNet&) = delete;
    UNet& operator=(const UNet&) = delete;

    float* input() { return x_in_; }          // fp32 [rmax][H][W][4]
    float* output() { return eps_; }          // fp32 [rmax][H][W][4]
    int* row_step() { return row_step_; }     // device [rmax]: schedule step of each row
    int* row_prompt() { return row_prompt_; } // device [rmax]: prompt of each row
    bf16* context(int p) { return ctx_ + static_cast<long long>(p) * cfg_.ctx_len * cfg_.ctx_dim; }
    // Recompute the per-prompt cross-attention K/V cache after context() changed.
    void refresh_context(cudaStream_t st);
    void forward(const int* rows_dev, cudaStream_t st);
    const std::vector<Param>& params() const { return params_; }
    double flops_per_row() const { return flops_per_row_; }
    int launches_per_forward() const {
        int n = 0;
        for (const auto& op : ops_) n += op.kind != "join";
        return n;
    }
    const UNetConfig& config() const { return cfg_; }
    // Device time of each op class accumulated by forward_profiled (ms).
    void forward_profiled(const int* rows_dev, cudaStream_t st, std::vector<std::pair<std::string, float>>* out);
    // Per-op label (kind + shape) and FLOPs at rmax rows, in launch order.
    const std::string& op_label(size_t i) const { return ops_[i].label.empty() ? ops_[i].kind : ops_[i].label; }
    double op_flops(size_t i) const { return ops_[i].flops; }

  private:
    struct Op {
        std::string kind;
        std::function<void(cudaStream_t)> fn;
        std::string label;   // kind + shape (profiling)
        double flops = 0;    // algorithmic FLOPs at rmax rows (tensor ops)
        // forked ops (fn runs on the side stream): rejoins the caller's stream when the op is
        // run on its own (per-op profile); in the forward a separate "join" op does that
        std::function<void(cudaStream_t)> join;
    };
    cudaStream_t side_ = nullptr;           // resblock shortcut GEMMs run here, concurrent with GN/conv1/GN
    std::vector<cudaEvent_t> fork_events_;
    bf16* wbf(const std::string& name, std::vector<long long> shape, float std);
    float* wf32(const std::string& name, std::vector<long long> shape, float std, float constant);
    bf16* act(long long elems);
    float* actf(long long elems);
    bf16* resblock(const bf16* x, int Cx, const bf16* skip, int Cs, int Cout, int H, int W, const std::string& nm);
    bf16* transformer(const bf16* x, int C, int H, int W, const std::string& nm);
    bf16* downsample(const bf16* x, int C, int H, int W, const std::string& nm);
    bf16* upsample(const bf16* x, int C, int H, int W, const std::string& nm);
    void gemm_op(const std::string& kind, const GemmPlan& p);
    // GroupNorm over [x1 | x2]: statistics fused into the producing GEMMs' epilogues
    GnPlan groupnorm(const bf16* x1, int C1, const bf16* x2, int C2, int HW, float eps, const float* g,
                     const float* b, int silu, bf16* out);
    std::deque<GemmPlan> plans_;                 // stable storage: ops and GN sinks point into it
    std::map<const void*, GemmPlan*> produced_;  // output tensor -> producing GEMM
    unsigned long long* gn_acc_ = nullptr;       // fixed-point GN statistics arena, zeroed per forward
    size_t gn_acc_elems_ = 0, gn_acc_used_ = 0;

    UNetConfig cfg_;
    std::vector<Param> params_;
    std::vector<void*> allocs_;
    std::vector<GnPlan> gns_;
    std::vector<Op> ops_;
    std::vector<Op> ctx_ops_;
    uint64_t param_counter_ = 0;
    int R_ = 0;
    const int* rows_dev_ = nullptr;    // = rows_buf_: the live row count every planned op reads
    float* x_in_ = nullptr;
    float* eps_ = nullptr;
    int* row_step_ = nullptr;
    int* row_prompt_ = nullptr;
    bf16* ctx_ = nullptr;
    float* temb_table_ = nullptr;  // [n_steps][20160] per-step resnet time-embedding biases
    bf16* temb_w_ = nullptr;       // [20160][1280] all resnets' time_emb_proj weights, build order
    float* temb_b_ = nullptr;
    long long temb_used_ = 0;
    double flops_per_row_ = 0;
    int* rows_buf_ = nullptr;  // [0] live rows (copied from the engine each forward), [1] = rmax
};

}  // namespace sdx
