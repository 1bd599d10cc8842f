/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the streaming denoise path.
 *
 * A plain-C restatement of the reference `stagger` hot path
 * (/root/reference/proj/core), fp64 like the reference.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it, and only as the checker or the CPU baseline; the product
 * (paper_2312_12491_b200/) never links or calls it.
 *
 * Pinned against: the reference's golden vectors (test_scheduler.cpp,
 * test_guidance.cpp, test_ssf.cpp, test_runtime.cpp — ported into
 * tests/test_oracle.py) and against the reference itself compiled from its
 * own sources (oracle/_ref/libstagger_ref.so, see oracle/Makefile).
 */
#ifndef STAGGER_ORACLE_H
#define STAGGER_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- RNG (rng.hpp:19-62, rng.cpp:7-20) -------------------------------- */
typedef struct orc_rng {
    uint64_t mt[312];
    int mti;
    double spare;
    int has_spare;
} orc_rng;

void orc_rng_init(orc_rng* r, uint64_t seed);
uint64_t orc_rng_next_u64(orc_rng* r);
double orc_rng_uniform(orc_rng* r);
double orc_rng_gaussian(orc_rng* r);
uint64_t orc_derive_seed(uint64_t seed, uint64_t tag);
void orc_rng_uniforms(uint64_t seed, int n, double* out);
void orc_rng_u64(uint64_t seed, int n, uint64_t* out);
int orc_sample_gaussian(uint64_t seed, int d, double* out);

/* ---- schedule (schedule.cpp:15-107) ---------------------------------- */
int orc_build_schedule(int n, int t_grid, double entry, int* taus, double* alphas,
                       double* betas);
void orc_lcm_coefficients(int tau, double alpha, double beta, int mode, double* c_skip,
                          double* c_out);

/* ---- SSF (ssf.cpp:8-54) ------------------------------------------------ */
double orc_cosine(const double* a, const double* b, int d);
double orc_skip_probability(double sim, double eta);

/* Gate state; max_skip <= 0 is exactly the reference SsfState.  max_skip > 0
 * is the cfg3 extension (no reference counterpart): the uniform
 * is still drawn, and after max_skip consecutive skips the next would-be skip
 * is forced to process. */
typedef struct orc_ssf orc_ssf;
int orc_ssf_create(double eta, uint64_t rng_seed, int max_skip, orc_ssf** out);
void orc_ssf_destroy(orc_ssf* s);
int orc_ssf_gate(orc_ssf* s, const double* payload, int d); /* 0 process, 1 skip, <0 error */
void orc_ssf_counters(orc_ssf* s, uint64_t* examined, uint64_t* skipped);

/* ---- engine (engine.cpp:36-238) ---------------------------------------- */
typedef struct orc_cfg {
    int n_steps;
    int guidance_mode; /* 0 none, 1 cfg, 2 self_negative, 3 onetime_negative */
    double gamma;
    double delta;
    int ssf_enabled;
    double eta;
    uint64_t seed;
    int d_latent;
    int t_grid;
    double entry_strength;
    double data_variance;
    int lcm_mode; /* 0 exact, 1 boundary_approx */
    int codec;    /* 0 identity (only identity is restated) */
    int queue_capacity;
    int cross_frame_attention; /* engine.cpp:139-149, attention.cpp:12-95 */
} orc_cfg;

typedef struct orc_engine orc_engine;
int orc_engine_create(const orc_cfg* c, const double* cond, const double* neg, orc_engine** out);
void orc_engine_destroy(orc_engine* e);
int orc_engine_ingest(orc_engine* e, int64_t seq, const double* x0);
int orc_engine_tick(orc_engine* e, int64_t* emitted_seq, double* x0_hat, int64_t* ingest_tick,
                    int64_t* emit_tick, uint64_t* calls, uint64_t* evals);
int orc_engine_idle(orc_engine* e);
int64_t orc_engine_ticks(orc_engine* e);
int orc_engine_inflight(orc_engine* e);
int64_t orc_engine_min_inflight_seq(orc_engine* e);
int orc_engine_step_indices(orc_engine* e, int* out);
void orc_engine_counters(orc_engine* e, uint64_t* calls, uint64_t* evals);
void orc_engine_eps_cached(orc_engine* e, int step, double* out);
int orc_sequential(const orc_cfg* c, const double* cond, const double* neg, const double* x0,
                   double* out);

/* ---- deterministic pipeline (pipeline.cpp:152-341) --------------------- */
typedef struct orc_report {
    uint64_t frames_in, frames_out, duplicates, stale_skips, input_drops, output_drops;
    uint64_t ticks, denoiser_calls, element_evals;
    uint64_t ssf_examined, ssf_skipped;
    double skip_rate, latency_ticks_mean;
    int64_t latency_ticks_min, latency_ticks_max;
    double mean_frame_time_ms, throughput_fps, wall_ms;
    int incomplete;
} orc_report;

int orc_run_pipeline(const orc_cfg* c, const double* cond, const double* neg,
                     const double* frames, int nframes, int d, int max_skip, int64_t* out_seq,
                     double* out_payload, int out_cap, int* n_out, int* decisions,
                     orc_report* report);

int orc_stream_frames(int kind, int d, uint64_t seed, int nframes, double* out);

const char* orc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
