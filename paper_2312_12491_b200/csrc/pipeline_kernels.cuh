// Control-block -> UNet / TAESD glue kernels (pipeline_kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include "device_ctl.cuh"

namespace sdx {

struct CodecLists {
    int* enc_src;     // [S] global frame index (ring_slot * S + stream) of each encoded frame
    int* enc_dst;     // [S] latent slot block (stream * n + slot)
    int* n_ingest;
    int* dec_src;     // [S] emitted-latent index (stream)
    int* dec_dst;     // [S] output frame index (ring_slot * S + stream)
    int* n_emit;
    int* row_step;    // UNet [rmax] or null
    int* row_prompt;  // UNet [rmax]
};

// x0[enc_dst[i]] = staged[enc_src[i]] for the n_ingest encoded frames (staged latents
// indexed like enc_src: ring_slot * S + stream)
void launch_enc_gather(const CodecLists& L, int S, const float* staged, float* x0, long long d, cudaStream_t st);
void launch_ctl_lists(const StreamCtl* ctl, int S, int n, int ring_slot, const RowDesc* rows, const int* n_rows,
                      const CodecLists& L, cudaStream_t st);
void launch_unet_prep(const StreamCtl* ctl, const RowDesc* rows, const int* n_rows, int rmax, int n, long long d,
                      const float* x_cur, const float* x0, const float* eps_cached, const StepScalars* tbl, float* out,
                      cudaStream_t st);

}  // namespace sdx
