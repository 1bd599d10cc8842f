// Device-side glue between the engine control block and the UNet / TAESD
// stages of one pipeline iteration (no host round trip):
//   ctl_lists  : compact lists of the streams that ingest (encoder gather /
//                latent-slot scatter) and that emit (decoder gather / output
//                scatter) this iteration, and the UNet's per-row schedule step and
//                prompt from the row table (engine.cpp:90-118)
//   unet_prep  : the batched denoiser input, one row per RowDesc: the slot's
//                current latent, or x_tau0 = sqrt(a0) x0 + sqrt(b0) eps_cached[0]
//                for the frame ingested this iteration (engine.cpp:69)
#include <cuda_runtime.h>

#include "common.cuh"
#include "device_ctl.cuh"
#include "pipeline_kernels.cuh"

namespace sdx {

namespace {

__global__ void ctl_lists_kernel(const StreamCtl* __restrict__ ctl, int S, int n, int ring_slot,
                                 const RowDesc* __restrict__ rows, const int* __restrict__ n_rows, CodecLists L) {
    __shared__ int scan_i[1024], scan_e[1024];
    const int s = threadIdx.x;
    const bool ing = s < S && ctl[s].ingest_slot >= 0;
    const bool emi = s < S && ctl[s].tick_now && ctl[s].emit_slot >= 0;
    scan_i[s] = ing;
    scan_e[s] = emi;
    __syncthreads();
    for (int off = 1; off < blockDim.x; off <<= 1) {
        const int vi = s >= off ? scan_i[s - off] : 0;
        const int ve = s >= off ? scan_e[s - off] : 0;
        __syncthreads();
        scan_i[s] += vi;
        scan_e[s] += ve;
        __syncthreads();
    }
    if (ing) {
        const int k = scan_i[s] - 1;
        L.enc_src[k] = ring_slot * S + s;
        L.enc_dst[k] = s * n + ctl[s].ingest_slot;
    }
    if (emi) {
        const int k = scan_e[s] - 1;
        L.dec_src[k] = s;
        L.dec_dst[k] = ring_slot * S + s;
    }
    if (s == blockDim.x - 1) {
        *L.n_ingest = scan_i[s];
        *L.n_emit = scan_e[s];
    }
    if (L.row_step) {
        const int R = *n_rows;
        for (int r = s; r < R; r += blockDim.x) {
            L.row_step[r] = rows[r].step;
            L.row_prompt[r] = rows[r].kind == 0 ? 0 : 1;
        }
    }
}

__global__ void unet_prep_kernel(const StreamCtl* __restrict__ ctl, const RowDesc* __restrict__ rows,
                                 const int* __restrict__ n_rows, int n, long long d, const float* __restrict__ x_cur,
                                 const float* __restrict__ x0, const float* __restrict__ eps_cached,
                                 const StepScalars* __restrict__ tbl, float* __restrict__ out) {
    const int r = blockIdx.y;
    if (r >= *n_rows) return;
    const RowDesc rd = rows[r];
    const bool entering = ctl[rd.stream].slot[rd.slot].entering != 0;
    const long long sd = static_cast<long long>(rd.stream) * n + rd.slot;
    const float4* xc = reinterpret_cast<const float4*>(x_cur + sd * d);
    const float4* xz = reinterpret_cast<const float4*>(x0 + sd * d);
    const float4* e0 = reinterpret_cast<const float4*>(eps_cached + static_cast<long long>(rd.stream) * n * d);
    float4* o = reinterpret_cast<float4*>(out + static_cast<long long>(r) * d);
    const float sa = tbl[0].f_sa, sb = tbl[0].f_sb;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < d / 4;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        float4 v;
        if (entering) {
            const float4 a = xz[i], b = e0[i];
            v = make_float4(sa * a.x + sb * b.x, sa * a.y + sb * b.y, sa * a.z + sb * b.z, sa * a.w + sb * b.w);
        } else {
            v = xc[i];
        }
        o[i] = v;
    }
}

}  // namespace

namespace {
// Latents of the ingesting streams out of the per-frame encoder staging
// (encoded ahead of the iteration): x0[enc_dst[i]] = staged[enc_src[i]].
__global__ void enc_gather_kernel(CodecLists L, const float* __restrict__ staged, float* __restrict__ x0, long long d) {
    const int i = blockIdx.y;
    if (i >= *L.n_ingest) return;
    const float4* src = reinterpret_cast<const float4*>(staged + static_cast<long long>(L.enc_src[i]) * d);
    float4* dst = reinterpret_cast<float4*>(x0 + static_cast<long long>(L.enc_dst[i]) * d);
    for (long long j = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; j < d / 4;
         j += static_cast<long long>(gridDim.x) * blockDim.x)
        dst[j] = src[j];
}

}  // namespace

void launch_enc_gather(const CodecLists& L, int S, const float* staged, float* x0, long long d, cudaStream_t st) {
    enc_gather_kernel<<<dim3(8, S), 256, 0, st>>>(L, staged, x0, d);
    SDX_LAUNCH_CHECK();
}

void launch_ctl_lists(const StreamCtl* ctl, int S, int n, int ring_slot, const RowDesc* rows, const int* n_rows,
                      const CodecLists& L, cudaStream_t st) {
    int threads = 32;
    while (threads < S) threads <<= 1;
    ctl_lists_kernel<<<1, threads, 0, st>>>(ctl, S, n, ring_slot, rows, n_rows, L);
    SDX_LAUNCH_CHECK();
}

void launch_unet_prep(const StreamCtl* ctl, const RowDesc* rows, const int* n_rows, int rmax, int n, long long d,
                      const float* x_cur, const float* x0, const float* eps_cached, const StepScalars* tbl, float* out,
                      cudaStream_t st) {
    dim3 grid(static_cast<unsigned>((d / 4 + 255) / 256), rmax);
    unet_prep_kernel<<<grid, 256, 0, st>>>(ctl, rows, n_rows, n, d, x_cur, x0, eps_cached, tbl, out);
    SDX_LAUNCH_CHECK();
}

}  // namespace sdx
