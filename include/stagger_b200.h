/* stagger_b200 — C-ABI of the B200-native streaming denoise loop.
 *
 * Drop-in boundary for the reference `stagger` hot path
 * (/root/reference/proj/core).  Plain pointers and sizes only; no torch or
 * CUDA types cross this boundary (streams are created and owned inside).
 * Every entry point returns an SDX_* status; the message of the last failure
 * on the calling thread is available from sdx_last_error().  The C++ drop-in
 * headers (include/stagger_b200/...) turn the codes back into the
 * reference's exception types (invalid_argument / logic_error / runtime_error).
 *
 * Which reference interface each group replaces:
 *   sdx_engine_*    stagger::StreamBatchEngine      engine.hpp:58-97, engine.cpp:36-211
 *                   + DenoiserBackend::predict_eps_batch (denoiser.hpp:21-39) as the
 *                   batched device denoiser inside tick()
 *   sdx_ssf_*       stagger::SsfState                ssf.hpp:25-42, ssf.cpp:34-54
 *   sdx_pipeline_*  stagger::run_pipeline (deterministic mode) + EngineStage +
 *                   BoundedQueue                     pipeline.hpp:31-32, pipeline.cpp:39-214,
 *                                                    queue.hpp:16-118
 *   sdx_host_*      pinned frame rings (no reference counterpart: the reference's
 *                   queues hold std::vector payloads)
 * Threading: every handle is single-owner, not thread-safe,
 * exactly like the reference objects.
 */
#ifndef STAGGER_B200_H
#define STAGGER_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SDX_ABI_VERSION 1

enum {
    SDX_OK = 0,
    SDX_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
    SDX_LOGIC_ERROR = 2,      /* std::logic_error */
    SDX_RUNTIME_ERROR = 3,    /* std::runtime_error (e.g. non-finite emission) */
    SDX_CUDA_ERROR = 4,
    SDX_UNSUPPORTED = 5
};

enum { SDX_GUIDANCE_NONE = 0, SDX_GUIDANCE_CFG = 1, SDX_GUIDANCE_SELF_NEGATIVE = 2,
       SDX_GUIDANCE_ONETIME_NEGATIVE = 3 };
enum { SDX_LCM_EXACT = 0, SDX_LCM_BOUNDARY_APPROX = 1 };
/* Denoiser behind predict_eps_batch: the reference's closed-form Gaussian model
 * (the parity denoiser, denoiser.cpp:26-43) or the random-init UNet. */
enum { SDX_BACKEND_ANALYTIC = 0, SDX_BACKEND_UNET = 2 };
/* Frame <-> latent codec: identity (codec.cpp:82-96, u8 frame -> f32 latent of the
 * same length) or the TAESD-class tiny VAE (3x512x512 u8 <-> 4x64x64 latent). */
enum { SDX_CODEC_IDENTITY = 0, SDX_CODEC_TAESD = 2 };
enum { SDX_GATE_PROCESS = 0, SDX_GATE_SKIP = 1 };

/* Mirror of stagger::EngineConfig (core.hpp:41-69), field for field, with the
 * string enums as ints.  Synthetic-backend timing fields are omitted: the
 * busy-wait timing probe (denoiser.cpp:54-73) has no device counterpart. */
typedef struct sdx_config {
    int n_steps;
    int guidance_mode;
    double gamma;
    double delta;
    int ssf_enabled;
    double eta;
    uint64_t seed;
    int cross_frame_attention; /* Stream Batch attention mix, engine.cpp:139-149 / attention.cpp:12-95 */
    int d_latent;
    int t_grid;
    double entry_strength;
    int backend;
    double data_variance;
    int lcm_mode;
    int codec;
    int queue_capacity;
} sdx_config;

/* stagger::ScheduleStep (schedule.hpp:14-24). */
typedef struct sdx_step {
    int tau;
    double alpha;
    double beta;
} sdx_step;

/* stagger::TickResult + EmittedFrame scalars (engine.hpp:30-41). */
typedef struct sdx_tick_result {
    int64_t emitted_seq; /* -1: nothing emitted this tick */
    int64_t ingest_tick;
    int64_t emit_tick;
    uint64_t denoiser_calls;
    uint64_t element_evals;
} sdx_tick_result;

const char* sdx_last_error(void);
int sdx_abi_version(void);
int sdx_device_count(int* count);

/* ---- StreamBatchEngine --------------------------------------------------
 * Host-driven: ingest() uploads x0 (+ its condition) into the frame's device
 * slot; tick() runs ONE fused device step over every in-flight frame (batched
 * denoiser, R-CFG / CFG combine, onetime init, LCM consistency update, cached
 * re-noise) and copies the emitted x0_hat back when one completes.
 * steps / eps_cached are the PrecomputeCache (precompute.hpp:16-21): n steps and
 * n x d_latent cached noise, uploaded once to HBM.  neg_condition is the
 * negative mean (cfg / onetime_negative) or NULL. */
typedef struct sdx_engine sdx_engine;
int sdx_engine_create(const sdx_config* cfg, const sdx_step* steps, int n_steps,
                      const double* eps_cached, const double* neg_condition, int device,
                      sdx_engine** out);
int sdx_engine_destroy(sdx_engine* e);
int sdx_engine_ingest(sdx_engine* e, int64_t seq_id, const double* x0, const double* cond);
int sdx_engine_tick(sdx_engine* e, sdx_tick_result* out, double* x0_hat /* d or NULL */);
int sdx_engine_ticks_completed(sdx_engine* e, int64_t* ticks);
int sdx_engine_inflight(sdx_engine* e, int* count);
int sdx_engine_step_indices(sdx_engine* e, int* out /* >= n_steps */, int* count);
int sdx_engine_min_inflight_seq(sdx_engine* e, int64_t* seq /* INT64_MAX when idle */);
int sdx_engine_counters(sdx_engine* e, uint64_t* calls, uint64_t* element_evals);
int sdx_engine_reset_counters(sdx_engine* e);
/* Device time of the last tick's kernels (CUDA events on the engine stream). */
int sdx_engine_last_tick_ms(sdx_engine* e, float* ms);

/* ---- SsfState -------------------------------------------------------------
 * Frames are u8 payloads (the frame format): the three dot products are exact
 * integer sums, so cosine, skip probability and the MT19937-64 uniform draw
 * are bit-identical to the reference's fp64 path on the same integer values.
 * max_skip <= 0 is the reference; > 0 is the cfg3 extension (forced process
 * after max_skip consecutive skips, the uniform is still drawn). */
typedef struct sdx_ssf sdx_ssf;
int sdx_ssf_create(double eta, uint64_t rng_seed, int max_skip, int64_t frame_bytes, int device,
                   sdx_ssf** out);
int sdx_ssf_destroy(sdx_ssf* s);
/* Gates nframes consecutive frames (host u8, nframes x frame_bytes) in order;
 * decisions[i] = SDX_GATE_PROCESS / SDX_GATE_SKIP; sims[i] (optional) the fp64
 * cosine (NaN for a first frame). */
int sdx_ssf_gate(sdx_ssf* s, const uint8_t* frames, int nframes, int* decisions, double* sims);
int sdx_ssf_counters(sdx_ssf* s, uint64_t* examined, uint64_t* skipped);

/* ---- run_pipeline (deterministic mode), S independent streams -------------
 * One push() = one iteration of the reference loop (pipeline.cpp:193-210) for
 * every stream: H2D of the frame, device SSF gate, encode, ingest-or-skip,
 * one batched tick over all streams' rows, decode, output ring.  Skip/run
 * decisions never return to the host before the next launch; the host reads
 * the device decision log asynchronously to order its sink (duplicates at
 * their sequence position, pipeline.cpp:102-116).
 * Frames are u8 of frame_bytes; outputs are f32 latents (identity codec,
 * d_latent floats) or u8 frames (TAESD codec, frame_bytes).  eps_cached is
 * S x n x d, cond is S x d (analytic mean) and neg S x d or NULL. */
typedef struct sdx_pipeline_config {
    sdx_config engine;
    int n_streams;
    int64_t frame_bytes;
    int max_skip;
    int ring_depth;   /* in-flight iterations between host and device, >= 2 */
    int graph;        /* capture one iteration in a CUDA graph (1) or launch eagerly (0) */
} sdx_pipeline_config;

typedef struct sdx_report { /* stagger::MetricsReport (metrics.hpp:12-41), per stream */
    uint64_t frames_in, frames_out, duplicates, stale_skips, input_drops, output_drops;
    uint64_t ticks, denoiser_calls, element_evals;
    uint64_t ssf_examined, ssf_skipped;
    double skip_rate, latency_ticks_mean;
    int64_t latency_ticks_min, latency_ticks_max;
    double mean_frame_time_ms, throughput_fps, wall_ms;
    int incomplete;
} sdx_report;

typedef struct sdx_pipeline sdx_pipeline;
int sdx_pipeline_create(const sdx_pipeline_config* cfg, const sdx_step* steps,
                        const double* eps_cached, const double* cond, const double* neg,
                        int device, sdx_pipeline** out);
int sdx_pipeline_destroy(sdx_pipeline* p);
/* frames: S x frame_bytes host u8.  Pinned memory (sdx_host_alloc) is copied to
 * HBM in place instead of through a staging buffer; either way the call returns
 * only after the frames have been read, so the caller may refill its buffer at
 * once.  The frames get the source sequence ids 0,1,2,... in push order. */
int sdx_pipeline_push(sdx_pipeline* p, const uint8_t* frames);
/* As push, with the S frames' source sequence ids (Frame::seq_id, pipeline.cpp:176):
 * sink frames, duplicates and the trace carry these ids.  Per stream the ids of
 * processed frames must strictly increase (engine.cpp:59-60, else the stream is
 * flagged incomplete with the reference's message); gaps are allowed (input drops). */
int sdx_pipeline_push_seq(sdx_pipeline* p, const uint8_t* frames, const int64_t* seq_ids);
/* Live loop without input (pipeline.cpp:235-245 ticks whenever the engine is not
 * idle): runs one frame-less iteration (a tick, no ingest) unless every stream is
 * known to be idle; *ran tells which. */
int sdx_pipeline_tick(sdx_pipeline* p, int* ran);
/* *idle = 1 when no stream has a frame in flight (processed iterations only count
 * once the device finished them; unfinished frame pushes count as busy). */
int sdx_pipeline_idle(sdx_pipeline* p, int* idle);
/* Source exhausted: keep ticking until every engine is idle, flush skips. */
int sdx_pipeline_finish(sdx_pipeline* p);
/* Next sink frame of stream s in sink order; *has = 0 when none is ready.
 * payload receives the output (f32 x d_latent or u8 x frame_bytes). */
int sdx_pipeline_pop(sdx_pipeline* p, int stream, int64_t* seq_id, void* payload, int* has);
int sdx_pipeline_report(sdx_pipeline* p, int stream, sdx_report* out);
/* Per-stream gate decisions of every examined frame so far (in seq order). */
int sdx_pipeline_decisions(sdx_pipeline* p, int stream, int* out, int cap, int* count);
int sdx_pipeline_sync(sdx_pipeline* p);
/* Per-tick trace of stream `stream` (the engine's TickLogEntry log, engine.hpp:43-50,
 * engine.cpp:181-192): one entry per tick; ingested / emitted are -1 for "none";
 * calls / element_evals are the tick's denoiser counters; elapsed_ns is the device
 * time of the iteration when stage profiling is on, else 0.  Entries beyond `cap` are
 * counted but not copied.  The first 2^20 ticks of a run are kept. */
typedef struct sdx_trace_entry {
    int64_t tick, ingested, emitted;
    uint64_t calls, element_evals;
    int64_t elapsed_ns;
} sdx_trace_entry;
int sdx_pipeline_trace(sdx_pipeline* p, int stream, sdx_trace_entry* out, int cap, int* count);
/* Error message of an incomplete stream ("" when complete). */
const char* sdx_pipeline_error_message(sdx_pipeline* p, int stream);
/* Benchmark path: stage ring_depth iterations of frames (ring_depth x S x
 * frame_bytes) in HBM once, then push_resident() runs one full iteration per
 * call reading them in place (no H2D; output D2H only when copy_outputs). */
int sdx_pipeline_upload_resident(sdx_pipeline* p, const uint8_t* frames, int count);
int sdx_pipeline_push_resident(sdx_pipeline* p, int copy_outputs);
/* Per-kernel timing with CUDA events on the pipeline stream (resets the
 * accumulators); kernel_times returns the summed device ms and launch counts of
 * the SSF reduction and of the fused step kernel since set_profile(1), and the
 * number of library kernel launches issued. */
int sdx_pipeline_set_profile(sdx_pipeline* p, int on);
/* ms6: summed device ms per stage over the profiled iterations:
 * [0] SSF gate, [1] control + reference commit, [2] encode (TAESD), [3] batched
 * denoiser (UNet), [4] fused step + control end, [5] decode (TAESD). */
int sdx_pipeline_stage_times(sdx_pipeline* p, double* ms6, int64_t* iterations, int64_t* total_launches);
/* Algorithmic FLOPs: UNet per denoiser row, TAESD encode + decode per frame (0 if absent). */
int sdx_pipeline_flops(sdx_pipeline* p, double* unet_per_row, double* codec_per_frame);
int sdx_pipeline_device_time_ms(sdx_pipeline* p, float* ms); /* since last reset */
int sdx_pipeline_reset_timer(sdx_pipeline* p);

/* ---- host precompute (PrecomputeCache, precompute.cpp:7-21) ---------------
 * derive_seed (rng.cpp:14-20), build_schedule (schedule.cpp:29-58), Rng +
 * sample_gaussian (rng.hpp:19-49, rng.cpp:7-12) and the n x d noise cache from
 * Rng(derive_seed(seed, kStreamNoiseCache)).  Host fp64, bit-identical to the
 * reference; errors via sdx_precompute_error(). */
uint64_t sdx_derive_seed(uint64_t seed, uint64_t tag);
int sdx_build_schedule(int n, int t_grid, double entry_strength, sdx_step* out);
int sdx_sample_gaussian(uint64_t seed, int64_t d, double* out);
int sdx_build_noise_cache(uint64_t seed, int n, int64_t d, double* out);
const char* sdx_precompute_error(void);

/* ---- pinned host memory -------------------------------------------------- */
int sdx_host_alloc(size_t bytes, void** out);
int sdx_host_free(void* p);

#ifdef __cplusplus
}
#endif
#endif /* STAGGER_B200_H */
