// Launch interfaces of the HBM-bound engine / SSF kernels (kernels_core.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "device_ctl.cuh"

namespace sdx {

enum { kIngestHost = 0, kIngestAlways = 1, kIngestSsf = 2 };

struct StepArgs {
    int n;
    long long d;
    int guidance;
    double gamma, delta;
    const StepScalars* tbl;     // [n + 1], tbl[n] = terminal (alpha 1, beta 0)
    float* x_cur;               // [S][n][d]
    const float* x0;            // [S][n][d]
    float* x0ref;               // [S][n][d] (onetime) or null
    const float* eps_cached;    // [S][n][d]
    const float* cond;          // analytic means
    long long cond_stream_stride, cond_slot_stride;
    const float* neg;           // [S][d] or null
    const float* eps_ext;       // [rows][eps_ext_stride] external (UNet) eps, or null -> analytic
    long long eps_ext_stride;
    const int* slot_row_c;      // [S][kMaxSteps] row of each slot's conditional eps
    const int* slot_row_n;      // [S][kMaxSteps] negative / init row or -1
    float* emitted;             // [S][d]
    StreamCtl* ctl;
    float* xfa_eps;             // cross-frame attention: [S][n][d] guided eps, or null (off)
    double* xfa_dots;           // [S][n][n] latent dot products
};

struct SsfArgs {
    const uint8_t* frames;      // [S] frames, frame_stride bytes apart
    long long frame_stride;
    const uint8_t* ref;         // [S][D]
    long long D;
    double eta;
    int max_skip;
    StreamCtl* ctl;
    unsigned long long* mt_state;  // [S][312]
    int* dec_out;                  // optional: decision of stream 0 (standalone gate)
    double* sim_out;               // optional: cosine of stream 0
};

struct CommitArgs {
    const uint8_t* frames;
    long long frame_stride;
    uint8_t* ref;               // null: no SSF
    long long D;
    float* x0;                  // null: codec is not identity
    int n;
    long long d;
    const StreamCtl* ctl;
};

void launch_ctl_begin(StreamCtl* ctl, int S, int n, int guidance, int ingest_mode, long long host_seq,
                      int frame_present, RowDesc* rows, int* n_rows, int* slot_row_c, int* slot_row_n,
                      cudaStream_t st);
void launch_step(const StepArgs& a, int S, cudaStream_t st);
void launch_ctl_end(StreamCtl* ctl, int S, int n, int guidance, LogEntry* log, int frame_present,
                    cudaStream_t st);
void launch_ssf_reduce(const SsfArgs& a, int S, cudaStream_t st);
void launch_commit_encode(const CommitArgs& a, int S, cudaStream_t st);

}  // namespace sdx
