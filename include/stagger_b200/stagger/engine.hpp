// Drop-in for stagger/engine.hpp (engine.hpp:30-97): the staggered stream-batch
// engine on the GPU.  ingest() uploads x0 and its condition into the frame's
// HBM slot; tick() runs one fused device step over every in-flight frame
// (batched denoiser rows, CFG / R-CFG combine, onetime init, LCM consistency
// update, cached re-noise) and copies the emitted x0_hat back.
#pragma once

#include <chrono>
#include <cstdint>
#include <memory>
#include <optional>
#include <vector>

#include "stagger/denoiser.hpp"
#include "stagger/precompute.hpp"

namespace stagger {

struct EmittedFrame {
    std::int64_t seq_id = 0;
    Latent x0_hat;
    std::int64_t ingest_tick = 0;
    std::int64_t emit_tick = 0;
};

struct TickResult {
    std::optional<EmittedFrame> emitted;
    std::uint64_t denoiser_calls = 0;
    std::uint64_t element_evals = 0;
};

struct TickLogEntry {
    std::int64_t tick = 0;
    std::optional<std::int64_t> ingested;
    std::optional<std::int64_t> emitted;
    std::uint64_t denoiser_calls = 0;
    std::uint64_t element_evals = 0;
    std::int64_t elapsed_ns = 0;  // device time of the tick (CUDA events)
};

class StreamBatchEngine {
  public:
    StreamBatchEngine(const EngineConfig& cfg, PrecomputeCache cache, std::shared_ptr<DenoiserBackend> backend,
                      int device = 0)
        : cfg_(validated(cfg)), cache_(std::move(cache)), backend_(std::move(backend)) {
        if (!backend_) throw std::invalid_argument("StreamBatchEngine: null backend");
        if (cache_.schedule.n() != cfg_.n_steps)
            throw std::invalid_argument("StreamBatchEngine: schedule length != n_steps");
        if (cache_.eps_cached.size() != static_cast<size_t>(cfg_.n_steps))
            throw std::invalid_argument("StreamBatchEngine: noise cache length != n_steps");
        std::vector<sdx_step> steps;
        for (const auto& s : cache_.schedule.steps) steps.push_back(sdx_step{s.tau, s.alpha, s.beta});
        std::vector<double> eps;
        for (const auto& e : cache_.eps_cached) {
            if (e.size() != static_cast<size_t>(cfg_.d_latent))
                throw std::invalid_argument("StreamBatchEngine: noise cache width != d_latent");
            eps.insert(eps.end(), e.begin(), e.end());
        }
        sdx_config c = detail::to_c(cfg_);
        c.lcm_mode = cache_.lcm.mode == LcmParams::Mode::boundary_approx ? SDX_LCM_BOUNDARY_APPROX : SDX_LCM_EXACT;
        const double* neg = cfg_.negative_condition.empty() ? nullptr : cfg_.negative_condition.data();
        detail::check(sdx_engine_create(&c, steps.data(), static_cast<int>(steps.size()), eps.data(), neg, device, &h_));
    }
    ~StreamBatchEngine() {
        if (h_) sdx_engine_destroy(h_);
    }
    StreamBatchEngine(const StreamBatchEngine&) = delete;
    StreamBatchEngine& operator=(const StreamBatchEngine&) = delete;

    void ingest(std::int64_t seq_id, Latent x0, Condition cond) {
        if (x0.size() != static_cast<size_t>(cfg_.d_latent))
            throw std::invalid_argument("ingest: latent length != d_latent");
        if (cond.embedding.size() != static_cast<size_t>(cfg_.d_latent))
            throw std::invalid_argument("ingest: condition embedding length != d_latent");
        detail::check(sdx_engine_ingest(h_, seq_id, x0.data(), cond.embedding.data()));
        ingested_since_tick_ = seq_id;
    }

    TickResult tick() {
        sdx_tick_result r{};
        Latent out(static_cast<size_t>(cfg_.d_latent));
        detail::check(sdx_engine_tick(h_, &r, out.data()));
        TickResult res;
        res.denoiser_calls = r.denoiser_calls;
        res.element_evals = r.element_evals;
        backend_->account(r.element_evals);
        if (r.emitted_seq >= 0) res.emitted = EmittedFrame{r.emitted_seq, std::move(out), r.ingest_tick, r.emit_tick};
        if (logging_) {
            TickLogEntry e;
            e.tick = ticks_completed();
            e.ingested = ingested_since_tick_;
            if (res.emitted) e.emitted = res.emitted->seq_id;
            e.denoiser_calls = res.denoiser_calls;
            e.element_evals = res.element_evals;
            float ms = 0.f;
            sdx_engine_last_tick_ms(h_, &ms);
            e.elapsed_ns = static_cast<std::int64_t>(ms * 1e6);
            log_.push_back(e);
        }
        ingested_since_tick_.reset();
        return res;
    }

    std::size_t inflight_size() const {
        int n = 0;
        detail::check(sdx_engine_inflight(h_, &n));
        return static_cast<std::size_t>(n);
    }
    bool idle() const { return inflight_size() == 0; }
    std::int64_t ticks_completed() const {
        int64_t t = 0;
        detail::check(sdx_engine_ticks_completed(h_, &t));
        return t;
    }
    std::vector<int> step_indices() const {
        std::vector<int> v(static_cast<size_t>(cfg_.n_steps) + 1);
        int n = 0;
        detail::check(sdx_engine_step_indices(h_, v.data(), &n));
        v.resize(static_cast<size_t>(n));
        return v;
    }
    std::optional<std::int64_t> min_inflight_seq() const {
        int64_t s = 0;
        detail::check(sdx_engine_min_inflight_seq(h_, &s));
        if (s == INT64_MAX) return std::nullopt;
        return s;
    }
    const std::vector<TickLogEntry>& log() const { return log_; }
    void set_logging(bool on) { logging_ = on; }
    const PrecomputeCache& cache() const { return cache_; }
    DenoiserBackend& backend() { return *backend_; }

  private:
    EngineConfig cfg_;
    PrecomputeCache cache_;
    std::shared_ptr<DenoiserBackend> backend_;
    sdx_engine* h_ = nullptr;
    std::optional<std::int64_t> ingested_since_tick_;
    bool logging_ = true;
    std::vector<TickLogEntry> log_;
};

}  // namespace stagger
