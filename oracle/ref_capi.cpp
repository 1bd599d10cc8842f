// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference `stagger` core, compiled from
// /root/reference/proj/core/src/*.cpp with -Dstagger=stagger_ref (see
// oracle/Makefile).  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs load the resulting
// oracle/_ref/libstagger_ref.so, as the checker or as the CPU baseline.
//
// Every entry point mirrors one reference call:
//   ref_derive_seed        -> stagger::derive_seed            (rng.cpp:14-20)
//   ref_rng_uniforms       -> stagger::Rng::uniform           (rng.hpp:26-28)
//   ref_sample_gaussian    -> stagger::sample_gaussian        (rng.cpp:7-12)
//   ref_build_schedule     -> stagger::build_schedule         (schedule.cpp:29-58)
//   ref_lcm_coefficients   -> stagger::lcm_coefficients       (schedule.cpp:80-89)
//   ref_engine_*           -> stagger::StreamBatchEngine      (engine.cpp:36-211)
//   ref_sequential         -> stagger::run_sequential_reference (engine.cpp:213-238)
//   ref_ssf_*              -> stagger::SsfState               (ssf.cpp:34-54)
//   ref_cosine             -> stagger::cosine_similarity      (ssf.cpp:8-20)
//   ref_run_pipeline       -> stagger::run_pipeline           (pipeline.cpp:152-341)
// Status codes: 0 ok, 1 invalid_argument, 2 logic_error, 3 runtime_error, 5 other.
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "stagger/engine.hpp"
#include "stagger/guidance.hpp"
#include "stagger/metrics.hpp"
#include "stagger/pipeline.hpp"
#include "stagger/precompute.hpp"
#include "stagger/rng.hpp"
#include "stagger/schedule.hpp"
#include "stagger/ssf.hpp"
#include "stagger/stream_gen.hpp"

namespace S = stagger_ref;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 5;
    }
}

}  // namespace

extern "C" {

// Plain-C mirror of the EngineConfig fields the hot path reads (core.hpp:41-69).
struct ref_cfg {
    int n_steps;
    int guidance_mode;  // 0 none, 1 cfg, 2 self_negative, 3 onetime_negative
    double gamma;
    double delta;
    int ssf_enabled;
    double eta;
    uint64_t seed;
    int d_latent;
    int t_grid;
    double entry_strength;
    double data_variance;
    int lcm_mode;  // 0 exact, 1 boundary_approx
    int codec;     // 0 identity, 1 affine
    int queue_capacity;
    int cross_frame_attention;
};

const char* ref_last_error() { return g_err.c_str(); }

static S::EngineConfig to_cfg(const ref_cfg* c, const double* cond, const double* neg) {
    S::EngineConfig cfg;
    cfg.n_steps = c->n_steps;
    cfg.guidance_mode = static_cast<S::GuidanceMode>(c->guidance_mode);
    cfg.gamma = c->gamma;
    cfg.delta = c->delta;
    cfg.ssf_enabled = c->ssf_enabled != 0;
    cfg.eta = c->eta;
    cfg.seed = c->seed;
    cfg.d_latent = c->d_latent;
    cfg.t_grid = c->t_grid;
    cfg.entry_strength = c->entry_strength;
    cfg.data_variance = c->data_variance;
    cfg.lcm_mode = c->lcm_mode == 1 ? "boundary_approx" : "exact";
    cfg.codec = c->codec == 1 ? "affine" : "identity";
    cfg.queue_capacity = c->queue_capacity;
    cfg.cross_frame_attention = c->cross_frame_attention != 0;
    if (cond) cfg.condition.assign(cond, cond + c->d_latent);
    if (neg) cfg.negative_condition.assign(neg, neg + c->d_latent);
    return cfg;
}

uint64_t ref_derive_seed(uint64_t seed, uint64_t tag) { return S::derive_seed(seed, tag); }

void ref_rng_uniforms(uint64_t seed, int n, double* out) {
    S::Rng rng(seed);
    for (int i = 0; i < n; ++i) out[i] = rng.uniform();
}

void ref_rng_u64(uint64_t seed, int n, uint64_t* out) {
    S::Rng rng(seed);
    for (int i = 0; i < n; ++i) out[i] = rng.next_u64();
}

int ref_sample_gaussian(uint64_t seed, int d, double* out) {
    return guarded([&] {
        S::Rng rng(seed);
        const auto v = S::sample_gaussian(rng, static_cast<size_t>(d));
        std::memcpy(out, v.data(), sizeof(double) * v.size());
    });
}

int ref_build_schedule(int n, int t_grid, double entry, int* taus, double* alphas,
                       double* betas) {
    return guarded([&] {
        const auto s = S::build_schedule(n, t_grid, entry);
        for (int i = 0; i < n; ++i) {
            taus[i] = s.steps[size_t(i)].tau;
            alphas[i] = s.steps[size_t(i)].alpha;
            betas[i] = s.steps[size_t(i)].beta;
        }
    });
}

void ref_lcm_coefficients(int tau, double alpha, double beta, int mode, double* c_skip,
                          double* c_out) {
    S::LcmParams p;
    p.mode = mode == 1 ? S::LcmParams::Mode::boundary_approx : S::LcmParams::Mode::exact;
    const auto [a, b] = S::lcm_coefficients(S::ScheduleStep{tau, alpha, beta}, p);
    *c_skip = a;
    *c_out = b;
}

double ref_cosine(const double* a, const double* b, int d) {
    return S::cosine_similarity(S::Latent(a, a + d), S::Latent(b, b + d));
}

double ref_skip_probability(double sim, double eta) { return S::skip_probability(sim, eta); }

// ---- engine -----------------------------------------------------------------

struct ref_engine {
    S::EngineConfig cfg;
    S::Condition cond;
    std::unique_ptr<S::StreamBatchEngine> engine;
    std::shared_ptr<S::DenoiserBackend> backend;
};

int ref_engine_create(const ref_cfg* c, const double* cond, const double* neg,
                      ref_engine** out) {
    return guarded([&] {
        auto e = std::make_unique<ref_engine>();
        e->cfg = to_cfg(c, nullptr, neg);
        e->cond = S::Condition{"cond", S::Latent(cond, cond + c->d_latent)};
        std::vector<S::Condition> conds{e->cond};
        if (neg) conds.push_back(S::Condition{"negative", e->cfg.negative_condition});
        auto cache = S::build_precompute(e->cfg, conds);
        e->backend = S::make_backend(e->cfg);
        e->engine = std::make_unique<S::StreamBatchEngine>(e->cfg, std::move(cache), e->backend);
        *out = e.release();
    });
}

void ref_engine_destroy(ref_engine* e) { delete e; }

int ref_engine_ingest(ref_engine* e, int64_t seq, const double* x0) {
    return guarded([&] {
        e->engine->ingest(seq, S::Latent(x0, x0 + e->cfg.d_latent), e->cond);
    });
}

// emitted_seq = -1 when nothing emitted.  x0_hat receives d doubles on emission.
int ref_engine_tick(ref_engine* e, int64_t* emitted_seq, double* x0_hat, int64_t* ingest_tick,
                    int64_t* emit_tick, uint64_t* calls, uint64_t* evals) {
    return guarded([&] {
        const auto r = e->engine->tick();
        *emitted_seq = -1;
        if (r.emitted) {
            *emitted_seq = r.emitted->seq_id;
            std::memcpy(x0_hat, r.emitted->x0_hat.data(), sizeof(double) * r.emitted->x0_hat.size());
            *ingest_tick = r.emitted->ingest_tick;
            *emit_tick = r.emitted->emit_tick;
        }
        *calls = r.denoiser_calls;
        *evals = r.element_evals;
    });
}

int ref_engine_idle(ref_engine* e) { return e->engine->idle() ? 1 : 0; }
int64_t ref_engine_ticks(ref_engine* e) { return e->engine->ticks_completed(); }
int ref_engine_inflight(ref_engine* e) { return int(e->engine->inflight_size()); }
int64_t ref_engine_min_inflight_seq(ref_engine* e) {
    const auto s = e->engine->min_inflight_seq();
    return s ? *s : INT64_MAX;
}
int ref_engine_step_indices(ref_engine* e, int* out) {
    const auto v = e->engine->step_indices();
    for (size_t i = 0; i < v.size(); ++i) out[i] = v[i];
    return int(v.size());
}
void ref_engine_counters(ref_engine* e, uint64_t* calls, uint64_t* evals) {
    *calls = e->engine->backend().counters().calls;
    *evals = e->engine->backend().counters().element_evals;
}
void ref_engine_eps_cached(ref_engine* e, int step, double* out) {
    const auto& v = e->engine->cache().eps_cached[size_t(step)];
    std::memcpy(out, v.data(), sizeof(double) * v.size());
}

int ref_sequential(const ref_cfg* c, const double* cond, const double* neg, const double* x0,
                   double* out) {
    return guarded([&] {
        const auto cfg = to_cfg(c, nullptr, neg);
        S::Condition cd{"cond", S::Latent(cond, cond + c->d_latent)};
        std::vector<S::Condition> conds{cd};
        auto cache = S::build_precompute(cfg, conds);
        S::AnalyticGaussianModel backend(cfg.data_variance);
        const auto g = S::guidance_from_config(cfg);
        const auto v = S::run_sequential_reference(S::Latent(x0, x0 + c->d_latent), cd, cache,
                                                   backend, g);
        std::memcpy(out, v.data(), sizeof(double) * v.size());
    });
}

// ---- SSF --------------------------------------------------------------------

struct ref_ssf {
    S::SsfState state;
};

int ref_ssf_create(double eta, uint64_t rng_seed, ref_ssf** out) {
    return guarded([&] { *out = new ref_ssf{S::SsfState(eta, S::Rng(rng_seed))}; });
}
void ref_ssf_destroy(ref_ssf* s) { delete s; }

// returns 0 process, 1 skip, <0 error
int ref_ssf_gate(ref_ssf* s, const double* payload, int d) {
    int decision = 0;
    const int st = guarded([&] {
        S::Frame f;
        f.payload.assign(payload, payload + d);
        decision = s->state.gate(f) == S::GateDecision::skip ? 1 : 0;
    });
    return st == 0 ? decision : -st;
}
void ref_ssf_counters(ref_ssf* s, uint64_t* examined, uint64_t* skipped) {
    *examined = s->state.examined();
    *skipped = s->state.skipped();
}

// ---- pipeline ---------------------------------------------------------------

// Runs the deterministic pipeline over nframes frames of d doubles each.
// Writes the sink sequence (seq ids + payloads, up to out_cap frames) and the
// report JSON (report_to_json, metrics.cpp:10-36).  cond may be null (then the
// seed-derived condition is used, pipeline.cpp:30-34).
int ref_run_pipeline(const ref_cfg* c, const double* cond, const double* neg,
                     const double* frames, int nframes, int d, int64_t* out_seq,
                     double* out_payload, int out_cap, int* n_out, char* report,
                     int report_cap) {
    return guarded([&] {
        const auto cfg = to_cfg(c, cond, neg);
        std::vector<S::Frame> fs(static_cast<size_t>(nframes));
        for (int i = 0; i < nframes; ++i) {
            fs[size_t(i)].seq_id = i;
            fs[size_t(i)].payload.assign(frames + size_t(i) * size_t(d),
                                         frames + size_t(i + 1) * size_t(d));
        }
        int count = 0;
        auto sink = [&](const S::Frame& f) {
            if (count < out_cap) {
                out_seq[count] = f.seq_id;
                if (out_payload)
                    std::memcpy(out_payload + size_t(count) * f.payload.size(), f.payload.data(),
                                sizeof(double) * f.payload.size());
            }
            ++count;
        };
        const auto r = S::run_pipeline(cfg, S::vector_source(std::move(fs)), sink);
        *n_out = count;
        const auto j = S::report_to_json(r);
        std::strncpy(report, j.c_str(), size_t(report_cap) - 1);
        report[report_cap - 1] = '\0';
    });
}

// StreamGenerator frames (stream_gen.cpp:53-71): kind 0 static, 1 dynamic, 2 periodic.
int ref_stream_frames(int kind, int d, uint64_t seed, int nframes, double* out) {
    return guarded([&] {
        S::StreamGenerator gen(static_cast<S::StreamGenerator::Kind>(kind), d, seed);
        for (int i = 0; i < nframes; ++i) {
            const auto f = gen.next();
            std::memcpy(out + size_t(i) * size_t(d), f.payload.data(), sizeof(double) * size_t(d));
        }
    });
}

}  // extern "C"
