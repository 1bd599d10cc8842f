// Drop-in for stagger/pipeline.hpp (pipeline.hpp:11-32, pipeline.cpp:152-340):
// run_pipeline on the device pipeline (sdx_pipeline_*): device SSF gate,
// encode, batched tick, decode; the sink receives frames in sequence order with
// skipped frames replayed as duplicates of the last output (pipeline.cpp:102-116).
// Frame payloads are u8-valued; outputs are the decoded latents (identity
// codec) or u8 frames (TAESD codec) as doubles.
//
// Deterministic mode (default) drives source -> push -> drain on the calling
// thread.  Threaded mode (pipeline.cpp:215-286) runs the reference's three
// stages on three host threads joined by BoundedQueues: pre (source -> input
// queue, drop-oldest, optional pacing), engine (freshest-wins or strict-FIFO
// dequeue -> sdx_pipeline_push -> ordered outputs into the output queue) and
// post (output queue -> sink).  trace_path writes the per-tick JSON-lines trace
// (pipeline.cpp:135-148) from the device pipeline's tick log.
#pragma once

#include <atomic>
#include <chrono>
#include <cstring>
#include <exception>
#include <fstream>
#include <string>
#include <thread>
#include <vector>

#include "stagger/metrics.hpp"
#include "stagger/precompute.hpp"
#include "stagger/queue.hpp"
#include "stagger/ssf.hpp"
#include "stagger/stream_gen.hpp"

namespace stagger {

struct PipelineOptions {
    bool threaded = false;
    bool strict_fifo = true;   // forced true in deterministic mode
    std::string trace_path;    // JSON-lines tick trace, empty = off
    double pace_us = 0.0;      // source pacing (threaded mode only)
    int max_skip = 0;          // SSF forced-process extension (0 = reference behaviour)
    int device = 0;
};

namespace detail {

// write_trace (pipeline.cpp:135-148): one JSON object per tick, keys in the
// reference's order, null for "no frame".
inline void write_trace(sdx_pipeline* p, const std::string& path) {
    int n = 0;
    check(sdx_pipeline_trace(p, 0, nullptr, 0, &n));
    std::vector<sdx_trace_entry> v(static_cast<size_t>(n));
    if (n > 0) check(sdx_pipeline_trace(p, 0, v.data(), n, &n));
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("run_pipeline: cannot open trace path " + path);
    for (const auto& e : v) {
        out << "{\"tick\":" << e.tick << ",\"ingested\":";
        if (e.ingested >= 0) out << e.ingested; else out << "null";
        out << ",\"emitted\":";
        if (e.emitted >= 0) out << e.emitted; else out << "null";
        out << ",\"calls\":" << e.calls << ",\"element_evals\":" << e.element_evals << ",\"elapsed_ns\":" << e.elapsed_ns
            << "}\n";
    }
}

// The device pipeline of one stream plus the host-side state both modes share.
struct DevicePipeline {
    EngineConfig cfg;
    PipelineOptions opts;
    std::vector<sdx_step> steps;
    std::vector<double> eps;
    Latent cond;
    sdx_pipeline* p = nullptr;
    int64_t frame_bytes = -1;
    bool taesd = false;
    std::vector<std::uint8_t> out_buf;

    DevicePipeline(const EngineConfig& c, const PipelineOptions& o) : cfg(c), opts(o) {
        cond = cfg.condition;
        if (cond.empty()) {  // resolve_condition (pipeline.cpp:30-34)
            Rng rng(derive_seed(cfg.seed, kStreamCondition));
            cond = sample_gaussian(rng, static_cast<size_t>(cfg.d_latent));
        }
        const auto cache = build_precompute(cfg, {});
        for (const auto& s : cache.schedule.steps) steps.push_back(sdx_step{s.tau, s.alpha, s.beta});
        for (const auto& e : cache.eps_cached) eps.insert(eps.end(), e.begin(), e.end());
        taesd = cfg.codec == "taesd";
    }
    ~DevicePipeline() {
        if (p) sdx_pipeline_destroy(p);
    }
    void push(const std::vector<std::uint8_t>& u8, std::int64_t seq_id) {
        if (!p) {
            frame_bytes = static_cast<int64_t>(u8.size());
            sdx_pipeline_config pc{};
            pc.engine = to_c(cfg);
            pc.n_streams = 1;
            pc.frame_bytes = frame_bytes;
            pc.max_skip = opts.max_skip;
            pc.ring_depth = 4;
            check(sdx_pipeline_create(&pc, steps.data(), eps.data(), cond.data(),
                                      cfg.negative_condition.empty() ? nullptr : cfg.negative_condition.data(),
                                      opts.device, &p));
            out_buf.resize(taesd ? static_cast<size_t>(frame_bytes) : static_cast<size_t>(cfg.d_latent) * 4);
        }
        if (static_cast<int64_t>(u8.size()) != frame_bytes) throw std::invalid_argument("ingest: latent length != d_latent");
        check(sdx_pipeline_push_seq(p, u8.data(), &seq_id));
    }
    // a tick without input while frames are in flight; false when idle (nothing launched)
    bool tick() {
        if (!p) return false;
        int ran = 0;
        check(sdx_pipeline_tick(p, &ran));
        return ran != 0;
    }
    // every output frame the pipeline has ordered so far, in sequence order
    template <class F>
    void drain(F&& emit) {
        if (!p) return;
        int has = 1;
        while (true) {
            int64_t seq = 0;
            check(sdx_pipeline_pop(p, 0, &seq, out_buf.data(), &has));
            if (!has) break;
            Frame f;
            f.seq_id = seq;
            if (taesd) {
                f.payload.assign(out_buf.begin(), out_buf.end());
            } else {
                const float* fp = reinterpret_cast<const float*>(out_buf.data());
                f.payload.assign(fp, fp + cfg.d_latent);
            }
            emit(std::move(f));
        }
    }
    void finish() {
        if (p) check(sdx_pipeline_finish(p));
    }
    void fill_report(MetricsReport& report) {
        if (!p) return;
        sdx_report r{};
        sdx_pipeline_sync(p);
        check(sdx_pipeline_report(p, 0, &r));
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
    }
};

}  // namespace detail

inline MetricsReport run_pipeline(const EngineConfig& raw_cfg, FrameSource source, FrameSink sink,
                                  const PipelineOptions& opts = {}) {
    const EngineConfig cfg = validated(raw_cfg);
    MetricsReport report;
    report.mode = opts.threaded ? "threaded" : "deterministic";
    detail::DevicePipeline dp(cfg, opts);
    std::uint64_t host_in_drops = 0, host_out_drops = 0;
    const auto wall0 = std::chrono::steady_clock::now();
    if (!opts.threaded) {
        try {
            while (auto f = source()) {
                dp.push(detail::to_u8(f->payload), f->seq_id);
                dp.drain([&](Frame&& o) { sink(o); });
            }
            dp.finish();
            dp.drain([&](Frame&& o) { sink(o); });
        } catch (const std::exception& e) {
            report.incomplete = true;
            report.error = e.what();
        }
    } else {
        struct InputItem {
            std::int64_t seq;
            std::vector<std::uint8_t> u8;
        };
        const std::size_t cap = static_cast<std::size_t>(cfg.queue_capacity > 0 ? cfg.queue_capacity : 8);
        BoundedQueue<InputItem> in_q(cap);
        BoundedQueue<Frame> out_q(cap * 8);  // pipeline.cpp:158-160
        std::exception_ptr pre_err, engine_err, post_err;
        std::thread pre([&] {
            try {
                while (auto f = source()) {
                    in_q.enqueue(InputItem{f->seq_id, detail::to_u8(f->payload)});
                    if (opts.pace_us > 0.0)
                        std::this_thread::sleep_for(std::chrono::duration<double, std::micro>(opts.pace_us));
                }
            } catch (...) {
                pre_err = std::current_exception();
            }
            in_q.close();
        });
        std::thread engine([&] {
            try {
                bool busy = false;  // frames may be in flight: tick without waiting for input
                while (true) {
                    // freshest-wins unless strict FIFO (pipeline.cpp:236-241); block only when idle
                    std::optional<InputItem> item;
                    if (busy) item = opts.strict_fifo ? in_q.dequeue_fifo() : in_q.dequeue_latest();
                    else item = in_q.wait_dequeue(!opts.strict_fifo, std::chrono::microseconds(200));
                    if (item) {
                        dp.push(item->u8, item->seq);
                        busy = true;
                        dp.drain([&](Frame&& o) { out_q.enqueue(std::move(o)); });
                    } else if (in_q.closed() && in_q.empty()) {
                        dp.finish();
                        dp.drain([&](Frame&& o) { out_q.enqueue(std::move(o)); });
                        break;
                    } else if (busy) {
                        // no input waiting: the reference still ticks the non-idle engine
                        busy = dp.tick();
                        dp.drain([&](Frame&& o) { out_q.enqueue(std::move(o)); });
                    }
                }
            } catch (...) {
                engine_err = std::current_exception();
            }
            out_q.close();
        });
        std::thread post([&] {
            try {
                while (true) {
                    auto of = out_q.wait_dequeue(false, std::chrono::microseconds(200));
                    if (of) sink(*of);
                    else if (out_q.closed() && out_q.empty()) break;
                }
            } catch (...) {
                post_err = std::current_exception();
            }
        });
        pre.join();
        engine.join();
        post.join();
        host_in_drops = in_q.dropped();
        host_out_drops = out_q.dropped();
        for (auto err : {pre_err, engine_err, post_err}) {
            if (!err) continue;
            report.incomplete = true;
            try {
                std::rethrow_exception(err);
            } catch (const std::exception& e) {
                if (report.error.empty()) report.error = e.what();
            }
        }
    }
    const double wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - wall0).count();
    try {
        const bool incomplete = report.incomplete;
        const std::string err = report.error;
        dp.fill_report(report);
        if (incomplete) {
            report.incomplete = true;
            report.error = err;
        }
        if (opts.threaded) {
            // host queues: frames dropped before reaching the device pipeline; the
            // device pipeline's own frames_in counts only the frames it received
            report.input_drops += host_in_drops;
            report.output_drops += host_out_drops;
            report.frames_in += host_in_drops;
            report.wall_ms = wall_ms;
            const double frames = static_cast<double>(report.frames_out);
            report.throughput_fps = wall_ms > 0.0 ? frames / (wall_ms * 1e-3) : 0.0;
            report.mean_frame_time_ms = frames > 0.0 ? wall_ms / frames : 0.0;
        }
        if (!opts.trace_path.empty() && dp.p) detail::write_trace(dp.p, opts.trace_path);
    } catch (const std::exception& e) {
        report.incomplete = true;
        if (report.error.empty()) report.error = e.what();
    }
    return report;
}

}  // namespace stagger
