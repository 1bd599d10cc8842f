// Drop-in for stagger/pipeline.hpp (pipeline.hpp:23-32): run_pipeline in
// deterministic mode on the device pipeline (sdx_pipeline_*): device SSF gate,
// encode, batched tick, decode; the sink receives frames in sequence order with
// skipped frames replayed as duplicates of the last output (pipeline.cpp:102-116).
// Frame payloads are u8-valued; outputs are the decoded latents (identity
// codec) or u8 frames (TAESD codec) as doubles.
#pragma once

#include <cstring>
#include <string>
#include <vector>

#include "stagger/metrics.hpp"
#include "stagger/precompute.hpp"
#include "stagger/ssf.hpp"
#include "stagger/stream_gen.hpp"

namespace stagger {

struct PipelineOptions {
    bool threaded = false;     // the device pipeline is asynchronous by construction; only
    bool strict_fifo = true;   // the deterministic contract is offered
    std::string trace_path;
    double pace_us = 0.0;
    int max_skip = 0;          // SSF forced-process extension (0 = reference behaviour)
    int device = 0;
};

inline MetricsReport run_pipeline(const EngineConfig& raw_cfg, FrameSource source, FrameSink sink,
                                  const PipelineOptions& opts = {}) {
    const EngineConfig cfg = validated(raw_cfg);
    if (opts.threaded) throw std::invalid_argument("run_pipeline: threaded mode is not built on the B200 path");
    MetricsReport report;
    report.mode = "deterministic";
    Latent cond = cfg.condition;
    if (cond.empty()) {  // resolve_condition (pipeline.cpp:30-34)
        Rng rng(derive_seed(cfg.seed, kStreamCondition));
        cond = sample_gaussian(rng, static_cast<size_t>(cfg.d_latent));
    }
    const auto cache = build_precompute(cfg, {});
    std::vector<sdx_step> steps;
    for (const auto& s : cache.schedule.steps) steps.push_back(sdx_step{s.tau, s.alpha, s.beta});
    std::vector<double> eps;
    for (const auto& e : cache.eps_cached) eps.insert(eps.end(), e.begin(), e.end());
    sdx_pipeline* p = nullptr;
    int64_t frame_bytes = -1;
    const bool taesd = cfg.codec == "taesd";
    std::vector<std::uint8_t> out_buf;
    auto drain = [&]() {
        int has = 1;
        while (true) {
            int64_t seq = 0;
            detail::check(sdx_pipeline_pop(p, 0, &seq, out_buf.data(), &has));
            if (!has) break;
            Frame f;
            f.seq_id = seq;
            if (taesd) {
                f.payload.assign(out_buf.begin(), out_buf.end());
            } else {
                const float* fp = reinterpret_cast<const float*>(out_buf.data());
                f.payload.assign(fp, fp + cfg.d_latent);
            }
            sink(f);
        }
    };
    try {
        while (auto f = source()) {
            const auto u8 = detail::to_u8(f->payload);
            if (!p) {
                frame_bytes = static_cast<int64_t>(u8.size());
                sdx_pipeline_config pc{};
                pc.engine = detail::to_c(cfg);
                pc.n_streams = 1;
                pc.frame_bytes = frame_bytes;
                pc.max_skip = opts.max_skip;
                pc.ring_depth = 4;
                detail::check(sdx_pipeline_create(&pc, steps.data(), eps.data(), cond.data(),
                                                  cfg.negative_condition.empty() ? nullptr : cfg.negative_condition.data(),
                                                  opts.device, &p));
                out_buf.resize(taesd ? static_cast<size_t>(frame_bytes) : static_cast<size_t>(cfg.d_latent) * 4);
            }
            if (static_cast<int64_t>(u8.size()) != frame_bytes)
                throw std::invalid_argument("ingest: latent length != d_latent");
            detail::check(sdx_pipeline_push(p, u8.data()));
            drain();
        }
        if (p) {
            detail::check(sdx_pipeline_finish(p));
            drain();
        }
    } catch (const std::exception& e) {
        report.incomplete = true;
        report.error = e.what();
    }
    if (p) {
        sdx_report r{};
        sdx_pipeline_sync(p);
        detail::check(sdx_pipeline_report(p, 0, &r));
        report.frames_in = r.frames_in;
        report.frames_out = r.frames_out;
        report.duplicates = r.duplicates;
        report.stale_skips = r.stale_skips;
        report.input_drops = r.input_drops;
        report.output_drops = r.output_drops;
        report.ticks = r.ticks;
        report.denoiser_calls = r.denoiser_calls;
        report.element_evals = r.element_evals;
        const double unit_cost = cfg.cost_per_element_us > 0.0 ? cfg.cost_per_element_us : 1.0;
        report.work_units = static_cast<double>(r.element_evals) * unit_cost;
        report.ssf_examined = r.ssf_examined;
        report.ssf_skipped = r.ssf_skipped;
        report.skip_rate = r.skip_rate;
        report.latency_ticks_mean = r.latency_ticks_mean;
        report.latency_ticks_min = r.latency_ticks_min;
        report.latency_ticks_max = r.latency_ticks_max;
        report.mean_frame_time_ms = r.mean_frame_time_ms;
        report.throughput_fps = r.throughput_fps;
        report.wall_ms = r.wall_ms;
        if (r.incomplete && !report.incomplete) {
            report.incomplete = true;
            report.error = sdx_pipeline_error_message(p, 0);
        }
        sdx_pipeline_destroy(p);
    }
    return report;
}

}  // namespace stagger
