// TAESD encoder / decoder build + launch (see taesd.cuh).
#include "taesd.cuh"

#include <cmath>

#include "common.cuh"

namespace sdx {

namespace {
constexpr int kRes[4] = {512, 256, 128, 64};
constexpr int kC = 64;
}  // namespace

bf16* TAESD::wbf(const std::string& name, std::vector<long long> shape, float std) {
    long long n = 1;
    for (auto s : shape) n *= s;
    bf16* p = dev_alloc<bf16>(static_cast<size_t>(n));
    allocs_.push_back(p);
    fill_normal_bf16(p, n, std, seed_ * 7919ULL + (++counter_), nullptr);
    params_.push_back(Param{name, p, shape, false});
    return p;
}

float* TAESD::wf32(const std::string& name, std::vector<long long> shape, float std) {
    long long n = 1;
    for (auto s : shape) n *= s;
    float* p = dev_alloc<float>(static_cast<size_t>(n));
    allocs_.push_back(p);
    fill_normal_f32(p, n, std, seed_ * 7919ULL + (++counter_), nullptr);
    params_.push_back(Param{name, p, shape, true});
    return p;
}

void TAESD::conv(std::vector<Op>& ops, double& flops, const bf16* x, int H, int stride, const std::string& nm,
                 bool bias, int act, const bf16* residual, bf16* out, const int* count) {
    GemmEpilogue e;
    e.bias = bias ? wf32(nm + ".b", {kC}, 0.02f) : nullptr;
    e.act = act;
    e.residual = residual;
    e.act_after_residual = residual != nullptr;
    e.out = out;
    const int Ho = stride == 1 ? H : H / 2;
    e.rows_dev = count;
    e.rows_per_unit = static_cast<long long>(Ho) * Ho;
    bf16* w = wbf(nm + ".w", {kC, 3, 3, kC}, std::sqrt(2.f / (9.f * kC)));
    GemmPlan p = plan_conv3x3(x, imax_, H, H, kC, w, kC, stride, e);
    const double f = 2.0 * Ho * Ho * kC * 9.0 * kC;
    ops.push_back(Op{"conv3x3", [p](cudaStream_t s) { run_gemm(p, s); },
                     "conv3x3 " + std::to_string(Ho) + "^2 s" + std::to_string(stride) + " bn=" + std::to_string(p.bn) +
                         (p.amode == kAHalo ? " halo" : ""),
                     f});
    flops += f;
}

int TAESD::block(std::vector<Op>& ops, double& flops, int r, int in, const std::string& nm, const int* count) {
    const int a = (in + 1) % 3, b = (in + 2) % 3;
    const int H = kRes[r];
    conv(ops, flops, buf(r, in), H, 1, nm + ".c0", true, kActRelu, nullptr, buf(r, a), count);
    conv(ops, flops, buf(r, a), H, 1, nm + ".c1", true, kActRelu, nullptr, buf(r, b), count);
    conv(ops, flops, buf(r, b), H, 1, nm + ".c2", true, kActRelu, buf(r, in), buf(r, a), count);  // relu(conv + x)
    return a;
}

TAESD::TAESD(int imax, uint64_t seed, const TaesdIO& io, cudaStream_t st) : imax_(imax), seed_(seed) {
    const int sets = io.separate_decoder_buffers && io.frames && io.latent_in ? 2 : 1;
    for (int set = 0; set < 2; ++set)
        for (int r = 0; r < 4; ++r)
            for (int k = 0; k < 3; ++k) {
                if (set < sets) {
                    bufs_[set][r][k] = dev_alloc<bf16>(static_cast<size_t>(imax) * kRes[r] * kRes[r] * kC);
                    allocs_.push_back(bufs_[set][r][k]);
                } else {
                    bufs_[set][r][k] = bufs_[0][r][k];
                }
            }
    a0_ = dev_alloc<bf16>(static_cast<size_t>(imax) * 64 * 64 * 64);  // decoder conv_in im2col (64x64 latents)
    allocs_.push_back(a0_);

    // ---------------- encoder ----------------
    if (io.frames) {
        const int* cnt = io.enc_count;
        {
            // first layer (3 -> 64) as a direct CUDA-core conv of the u8 frames
            const float* b = wf32("enc.conv_in.b", {kC}, 0.02f);
            const bf16* w = wbf("enc.conv_in.w", {kC, 64}, std::sqrt(2.f / 27.f));  // cols >= 27 unused
            const uint8_t* fr = io.frames;
            const long long fs = io.frame_stride;
            const int* src = io.enc_src;
            const int im = imax_;
            bf16* o = buf(0, 0);
            enc_.push_back(Op{"conv_in", [=](cudaStream_t s) {
                                  run_conv3x3_rgb8(fr, fs, src, im, 512, 512, w, 64, b, o, cnt, s);
                              }, "conv_in 512^2 rgb8", 2.0 * 512 * 512 * kC * 27});
            enc_flops_ += 2.0 * 512 * 512 * kC * 27;
        }
        int cur = block(enc_, enc_flops_, 0, 0, "enc.b0", cnt);
        for (int r = 1; r < 4; ++r) {
            conv(enc_, enc_flops_, buf(r - 1, cur), kRes[r - 1], 2, "enc.down" + std::to_string(r), false, kActNone,
                 nullptr, buf(r, 0), cnt);
            cur = 0;
            for (int j = 0; j < 3; ++j) cur = block(enc_, enc_flops_, r, cur, "enc.b" + std::to_string(r) + std::to_string(j), cnt);
        }
        {
            GemmEpilogue e;
            e.bias = wf32("enc.conv_out.b", {4}, 0.02f);
            e.out = io.latent_out;
            e.out_f32 = 1;
            e.out_img_map = io.enc_dst;
            e.rows_per_img = 64 * 64;
            e.rows_dev = cnt;
            e.rows_per_unit = 64 * 64;
            bf16* w = wbf("enc.conv_out.w", {4, 3, 3, kC}, std::sqrt(1.f / (9.f * kC)));
            GemmPlan p = plan_conv3x3(buf(3, cur), imax_, 64, 64, kC, w, 4, 1, e);
            enc_.push_back(Op{"conv_out", [p](cudaStream_t s) { run_gemm(p, s); }, "conv_out 64^2 64->4",
                              2.0 * 64 * 64 * 4 * 9.0 * kC});
            enc_flops_ += 2.0 * 64 * 64 * 4 * 9.0 * kC;
        }
    }
    // ---------------- decoder ----------------
    set_ = 1;
    if (io.latent_in) {
        const int* cnt = io.dec_count;
        {
            const float* li = io.latent_in;
            const int* src = io.dec_src;
            const int im = imax_;
            bf16* a0 = a0_;
            dec_.push_back(Op{"im2col", [=](cudaStream_t s) {
                                  run_im2col3x3_f32_gather(li, 64 * 64 * 4, src, im, 64, 64, 4, 64, 1, a0, cnt, s);
                              }, "im2col 64^2", 0.0});
        }
        {
            GemmEpilogue e;
            e.bias = wf32("dec.conv_in.b", {kC}, 0.02f);
            e.act = kActRelu;
            e.out = buf(3, 0);
            e.rows_dev = cnt;
            e.rows_per_unit = 64 * 64;
            bf16* w = wbf("dec.conv_in.w", {kC, 64}, std::sqrt(2.f / 36.f));
            GemmPlan p = plan_gemm(a0_, 64, w, 64, imax_ * 64 * 64, kC, 64, e);
            dec_.push_back(Op{"conv_in", [p](cudaStream_t s) { run_gemm(p, s); }, "conv_in 64^2 4->64",
                              2.0 * 64 * 64 * kC * 36});
            dec_flops_ += 2.0 * 64 * 64 * kC * 36;
        }
        int cur = 0;
        for (int j = 0; j < 3; ++j) cur = block(dec_, dec_flops_, 3, cur, "dec.b3" + std::to_string(j), cnt);
        for (int r = 2; r >= 0; --r) {
            // Upsample 2x into buffer 2 of the next resolution, then conv (no bias) into buffer 0
            const bf16* src = buf(r + 1, cur);
            bf16* up = buf(r, 2);
            const int Hs = kRes[r + 1];
            const int im = imax_;
            dec_.push_back(Op{"upsample", [=](cudaStream_t s) { run_upsample2x(src, im, Hs, Hs, kC, up, cnt, s); },
                              "upsample " + std::to_string(Hs) + "^2->" + std::to_string(2 * Hs) + "^2", 0.0});
            conv(dec_, dec_flops_, up, kRes[r], 1, "dec.up" + std::to_string(r), false, kActNone, nullptr, buf(r, 0), cnt);
            cur = 0;
            const int nblocks = r == 0 ? 1 : 3;
            for (int j = 0; j < nblocks; ++j)
                cur = block(dec_, dec_flops_, r, cur, "dec.b" + std::to_string(r) + std::to_string(j), cnt);
        }
        {
            // 64 -> 3 head as a CUDA-core conv (a tensor-core tile would pad N to 64)
            const float* b = wf32("dec.conv_out.b", {3}, 0.02f);
            const bf16* w = wbf("dec.conv_out.w", {3, 3, 3, kC}, std::sqrt(1.f / (9.f * kC)));
            const bf16* x = buf(0, cur);
            uint8_t* fo = io.frames_out;
            const int* map = io.dec_dst;
            const int im = imax_;
            dec_.push_back(Op{"conv_out", [=](cudaStream_t s) { run_conv3x3_c64_u8(x, im, 512, 512, w, 3, b, fo, map, cnt, s); },
                              "conv_out 512^2 64->3 u8", 2.0 * 512 * 512 * 3 * 9.0 * kC});
            dec_flops_ += 2.0 * 512 * 512 * 3 * 9.0 * kC;
        }
    }
    set_ = 0;
    SDX_CUDA(cudaStreamSynchronize(st));
    SDX_CUDA(cudaDeviceSynchronize());
}

TAESD::~TAESD() {
    cudaDeviceSynchronize();
    for (void* p : allocs_) dev_free(p);
}

void TAESD::encode(cudaStream_t st) {
    for (auto& op : enc_) op.fn(st);
}

void TAESD::decode(cudaStream_t st) {
    for (auto& op : dec_) op.fn(st);
}

void TAESD::profile(bool decoder, std::vector<std::tuple<std::string, double, float>>* out) {
    constexpr int kReps = 10;
    std::vector<Op>& ops = decoder ? dec_ : enc_;
    cudaStream_t cs;
    SDX_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaEvent_t e0, e1;
    SDX_CUDA(cudaEventCreate(&e0));
    SDX_CUDA(cudaEventCreate(&e1));
    for (auto& op : ops) op.fn(cs);
    SDX_CUDA(cudaStreamSynchronize(cs));
    out->clear();
    for (auto& op : ops) {
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        SDX_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        for (int r = 0; r < kReps; ++r) op.fn(cs);
        SDX_CUDA(cudaStreamEndCapture(cs, &graph));
        SDX_CUDA(cudaGraphInstantiate(&exec, graph, 0));
        SDX_CUDA(cudaGraphLaunch(exec, cs));
        SDX_CUDA(cudaEventRecord(e0, cs));
        SDX_CUDA(cudaGraphLaunch(exec, cs));
        SDX_CUDA(cudaEventRecord(e1, cs));
        SDX_CUDA(cudaEventSynchronize(e1));
        float ms = 0.f;
        SDX_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        out->emplace_back(op.label, op.flops, ms / kReps);
        cudaGraphExecDestroy(exec);
        cudaGraphDestroy(graph);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(cs);
}

}  // namespace sdx
