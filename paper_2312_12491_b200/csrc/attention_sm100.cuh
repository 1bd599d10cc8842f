// tcgen05 flash attention, head_dim 64 (attention_sm100.cu).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace sdx {

struct AttnArgs {
    int q_col0, k_col0, v_col0;   // column of head 0 inside the Q / KV matrices
    __nv_bfloat16* out;
    long long ld_out;
    int out_col0;
    int q_len, q_rows_per_img;    // queries per image and their row stride in Q
    int kv_len, kv_rows_per_img;  // keys per image (or per prompt) and row stride in KV
    const int* kv_index;          // image -> KV block (prompt index for cross-attention) or null = image
    const int* rows_dev;          // live image count (device) or null
    float scale;
    int xmode;                    // experiments only: 1 = no MMAs, 2 = no softmax math (pipeline probes)
    int heads;                    // set by run_attention
    int single, unit_base, pair_base;  // CTAs >= pair_base run single-tile units (the tail); single/unit_base unused
    long long* dbg;               // experiments only: clock64 phase stamps of CTA 0 (null = off)
    const __nv_bfloat16* q;       // Q rows for the TMEM-resident A operand (attn_ts_kernel)
    long long q_rows_total, ld_q;
};

// Pipeline probe for kernel experiments (results wrong): 0 off, 1 no MMAs, 2 no softmax math.
void set_attention_probe_mode(int mode);
// Experiments: device buffer of [10 warps][64 blocks][8] clock64 stamps for CTA 0 (null = off).
void set_attention_debug_buffer(long long* dbg);

struct AttnPlan {
    CUtensorMap tq, tkv;
    AttnArgs a;
    int images = 0, heads = 0;
    bool valid = false;
};

// Q: [q_rows_total][ld_q] bf16 (head h at column q_col0 + 64h); KV: [kv_rows_total][ld_kv]
// (K head h at k_col0 + 64h, V at v_col0 + 64h); out [.][ld_out] at out_col0 + 64h.
AttnPlan plan_attention(const __nv_bfloat16* q, long long q_rows_total, long long ld_q, int q_col0,
                        const __nv_bfloat16* kv, long long kv_rows_total, long long ld_kv, int k_col0, int v_col0,
                        __nv_bfloat16* out, long long ld_out, int out_col0, int images, int heads, int q_len,
                        int q_rows_per_img, int kv_len, int kv_rows_per_img, const int* kv_index, const int* rows_dev,
                        float scale);
void run_attention(const AttnPlan& p, cudaStream_t st);

}  // namespace sdx
