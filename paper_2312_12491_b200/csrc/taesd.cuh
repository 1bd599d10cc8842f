// TAESD-class tiny VAE (the LatentCodec slot, codec.hpp:11-30) on the sm_100a
// implicit-GEMM conv kernels: 3x512x512 u8 frames <-> 4x64x64 fp32 latents.
//
// Topology (madebyollin/taesd): encoder conv(3,64) Block, 3 x [conv s2 (no
// bias), 3 Blocks], conv(64,4); decoder Clamp(tanh(x/3)*3), conv(4,64), ReLU,
// 3 Blocks, 3 x [Upsample 2x, conv (no bias), Block(s)], conv(64,3).
// Block(64): conv-ReLU-conv-ReLU-conv, + identity, ReLU (fused in the last
// conv's epilogue).  Random-init weights; activations bf16 NHWC ping-ponged
// through three buffers per resolution.
//
// Encode gathers the frames of the streams that ingest this iteration
// (device list) and scatters latents to their engine slots; decode gathers
// the emitted latents and scatters u8 frames to their streams' output slots.
// Both read the live image count from device memory.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <functional>
#include <string>
#include <tuple>
#include <vector>

#include "gemm_sm100.cuh"
#include "nn_kernels.cuh"
#include "unet.cuh"

namespace sdx {

struct TaesdIO {
    // encoder
    const uint8_t* frames = nullptr;  // [.][512*512*3] u8
    long long frame_stride = 0;
    const int* enc_src = nullptr;     // device [imax]: frame index of each encoded image
    const int* enc_count = nullptr;   // device: live images
    float* latent_out = nullptr;      // fp32 [.][64*64*4]
    const int* enc_dst = nullptr;     // device [imax]: latent block of each encoded image
    // decoder
    const float* latent_in = nullptr;  // fp32 [.][64*64*4]
    const int* dec_src = nullptr;
    const int* dec_count = nullptr;
    uint8_t* frames_out = nullptr;     // [.][512*512*3] u8
    const int* dec_dst = nullptr;
    // decoder activations in their own buffers, so a decode may run on another
    // stream concurrently with the next encode
    bool separate_decoder_buffers = false;
};

class TAESD {
  public:
    TAESD(int imax, uint64_t seed, const TaesdIO& io, cudaStream_t st);
    ~TAESD();
    TAESD(const TAESD&) = delete;
    TAESD& operator=(const TAESD&) = delete;
    void encode(cudaStream_t st);
    void decode(cudaStream_t st);
    const std::vector<Param>& params() const { return params_; }
    double enc_flops_per_image() const { return enc_flops_; }
    double dec_flops_per_image() const { return dec_flops_; }
    int launches_per_encode() const { return static_cast<int>(enc_.size()); }
    int launches_per_decode() const { return static_cast<int>(dec_.size()); }
    // Per-op device times of the encoder (decoder=false) or decoder at the live image
    // count already set on the device: each op alone, 10 back-to-back repetitions in one
    // CUDA graph (as UNet::forward_profiled).  out: (label, flops per image, ms).
    void profile(bool decoder, std::vector<std::tuple<std::string, double, float>>* out);

  private:
    struct Op {
        std::string kind;
        std::function<void(cudaStream_t)> fn;
        std::string label;  // kind + resolution (per-op profile)
        double flops = 0;   // per image
    };
    bf16* wbf(const std::string& name, std::vector<long long> shape, float std);
    float* wf32(const std::string& name, std::vector<long long> shape, float std);
    void conv(std::vector<Op>& ops, double& flops, const bf16* x, int H, int stride, const std::string& nm, bool bias,
              int act, const bf16* residual, bf16* out, const int* count);
    // returns the buffer index holding the output
    int block(std::vector<Op>& ops, double& flops, int res_idx, int in, const std::string& nm, const int* count);
    bf16* buf(int res_idx, int k) { return bufs_[set_][res_idx][k]; }

    int imax_;
    uint64_t seed_, counter_ = 0;
    std::vector<Param> params_;
    std::vector<void*> allocs_;
    bf16* bufs_[2][4][3] = {};  // [encoder, decoder][resolution 512, 256, 128, 64][3]
    int set_ = 0;
    bf16* a0_ = nullptr;  // im2col scratch [imax*512*512][64]
    std::vector<Op> enc_, dec_;
    double enc_flops_ = 0, dec_flops_ = 0;
};

}  // namespace sdx
