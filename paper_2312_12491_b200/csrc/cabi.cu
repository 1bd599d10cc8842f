// extern "C" boundary (include/stagger_b200.h): status codes + thread-local
// error text around the C++ runtime.
#include <cuda_runtime.h>

#include <cstring>
#include <exception>
#include <new>
#include <string>

#include "runtime.cuh"
#include "stagger_b200.h"

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return SDX_OK;
    } catch (const sdx::Error& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "out of host memory";
        return SDX_RUNTIME_ERROR;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SDX_RUNTIME_ERROR;
    }
}

#define NEED(p)                                                             \
    do {                                                                    \
        if (!(p)) sdx::raise(SDX_INVALID_ARGUMENT, "null argument: " #p);   \
    } while (0)
}  // namespace

struct sdx_engine {
    sdx::Engine impl;
};
struct sdx_ssf {
    sdx::Ssf impl;
};
struct sdx_pipeline {
    sdx::Pipeline impl;
};

extern "C" {

const char* sdx_last_error(void) { return g_err.c_str(); }
int sdx_abi_version(void) { return SDX_ABI_VERSION; }

int sdx_device_count(int* count) {
    return guarded([&] {
        NEED(count);
        SDX_CUDA(cudaGetDeviceCount(count));
    });
}

// ---- engine ----
int sdx_engine_create(const sdx_config* cfg, const sdx_step* steps, int n_steps, const double* eps_cached,
                      const double* neg_condition, int device, sdx_engine** out) {
    return guarded([&] {
        NEED(cfg);
        NEED(steps);
        NEED(out);
        *out = new sdx_engine{sdx::Engine(*cfg, steps, n_steps, eps_cached, neg_condition, device)};
    });
}
int sdx_engine_destroy(sdx_engine* e) {
    return guarded([&] { delete e; });
}
int sdx_engine_ingest(sdx_engine* e, int64_t seq_id, const double* x0, const double* cond) {
    return guarded([&] {
        NEED(e);
        e->impl.ingest(seq_id, x0, cond);
    });
}
int sdx_engine_tick(sdx_engine* e, sdx_tick_result* out, double* x0_hat) {
    return guarded([&] {
        NEED(e);
        NEED(out);
        *out = e->impl.tick(x0_hat);
    });
}
int sdx_engine_ticks_completed(sdx_engine* e, int64_t* ticks) {
    return guarded([&] {
        NEED(e);
        NEED(ticks);
        *ticks = e->impl.mirror().ticks();
    });
}
int sdx_engine_inflight(sdx_engine* e, int* count) {
    return guarded([&] {
        NEED(e);
        NEED(count);
        *count = e->impl.mirror().inflight();
    });
}
int sdx_engine_step_indices(sdx_engine* e, int* out, int* count) {
    return guarded([&] {
        NEED(e);
        NEED(count);
        const auto v = e->impl.mirror().step_indices();
        if (out) std::memcpy(out, v.data(), v.size() * sizeof(int));
        *count = static_cast<int>(v.size());
    });
}
int sdx_engine_min_inflight_seq(sdx_engine* e, int64_t* seq) {
    return guarded([&] {
        NEED(e);
        NEED(seq);
        *seq = e->impl.mirror().min_inflight_seq();
    });
}
int sdx_engine_counters(sdx_engine* e, uint64_t* calls, uint64_t* element_evals) {
    return guarded([&] {
        NEED(e);
        if (calls) *calls = e->impl.mirror().calls;
        if (element_evals) *element_evals = e->impl.mirror().evals;
    });
}
int sdx_engine_reset_counters(sdx_engine* e) {
    return guarded([&] {
        NEED(e);
        e->impl.reset_counters();
    });
}
int sdx_engine_last_tick_ms(sdx_engine* e, float* ms) {
    return guarded([&] {
        NEED(e);
        NEED(ms);
        *ms = e->impl.last_tick_ms();
    });
}

// ---- ssf ----
int sdx_ssf_create(double eta, uint64_t rng_seed, int max_skip, int64_t frame_bytes, int device, sdx_ssf** out) {
    return guarded([&] {
        NEED(out);
        *out = new sdx_ssf{sdx::Ssf(eta, rng_seed, max_skip, frame_bytes, device)};
    });
}
int sdx_ssf_destroy(sdx_ssf* s) {
    return guarded([&] { delete s; });
}
int sdx_ssf_gate(sdx_ssf* s, const uint8_t* frames, int nframes, int* decisions, double* sims) {
    return guarded([&] {
        NEED(s);
        NEED(frames);
        s->impl.gate(frames, nframes, decisions, sims);
    });
}
int sdx_ssf_counters(sdx_ssf* s, uint64_t* examined, uint64_t* skipped) {
    return guarded([&] {
        NEED(s);
        if (examined) *examined = s->impl.examined();
        if (skipped) *skipped = s->impl.skipped();
    });
}

// ---- pipeline ----
int sdx_pipeline_create(const sdx_pipeline_config* cfg, const sdx_step* steps, const double* eps_cached,
                        const double* cond, const double* neg, int device, sdx_pipeline** out) {
    return guarded([&] {
        NEED(cfg);
        NEED(steps);
        NEED(eps_cached);
        NEED(cond);
        NEED(out);
        *out = new sdx_pipeline{sdx::Pipeline(*cfg, steps, eps_cached, cond, neg, device)};
    });
}
int sdx_pipeline_destroy(sdx_pipeline* p) {
    return guarded([&] { delete p; });
}
int sdx_pipeline_push(sdx_pipeline* p, const uint8_t* frames) {
    return guarded([&] {
        NEED(p);
        NEED(frames);
        p->impl.push(frames);
    });
}
int sdx_pipeline_push_seq(sdx_pipeline* p, const uint8_t* frames, const int64_t* seq_ids) {
    return guarded([&] {
        NEED(p);
        NEED(frames);
        NEED(seq_ids);
        p->impl.push(frames, seq_ids);
    });
}
int sdx_pipeline_tick(sdx_pipeline* p, int* ran) {
    return guarded([&] {
        NEED(p);
        const bool r = p->impl.tick_idle();
        if (ran) *ran = r ? 1 : 0;
    });
}
int sdx_pipeline_idle(sdx_pipeline* p, int* idle) {
    return guarded([&] {
        NEED(p);
        NEED(idle);
        *idle = p->impl.idle() ? 1 : 0;
    });
}
int sdx_pipeline_finish(sdx_pipeline* p) {
    return guarded([&] {
        NEED(p);
        p->impl.finish();
    });
}
int sdx_pipeline_pop(sdx_pipeline* p, int stream, int64_t* seq_id, void* payload, int* has) {
    return guarded([&] {
        NEED(p);
        NEED(seq_id);
        NEED(has);
        *has = p->impl.pop(stream, seq_id, payload) ? 1 : 0;
    });
}
int sdx_pipeline_report(sdx_pipeline* p, int stream, sdx_report* out) {
    return guarded([&] {
        NEED(p);
        NEED(out);
        *out = p->impl.report(stream);
    });
}
int sdx_pipeline_decisions(sdx_pipeline* p, int stream, int* out, int cap, int* count) {
    return guarded([&] {
        NEED(p);
        NEED(count);
        const auto& v = p->impl.decisions(stream);
        const int n = static_cast<int>(v.size());
        if (out) std::memcpy(out, v.data(), sizeof(int) * static_cast<size_t>(n < cap ? n : cap));
        *count = n;
    });
}
int sdx_pipeline_trace(sdx_pipeline* p, int stream, sdx_trace_entry* out, int cap, int* count) {
    return guarded([&] {
        NEED(p);
        NEED(count);
        const auto& v = p->impl.trace(stream);
        const int n = static_cast<int>(v.size());
        if (out && cap > 0) std::memcpy(out, v.data(), sizeof(sdx_trace_entry) * static_cast<size_t>(n < cap ? n : cap));
        *count = n;
    });
}
int sdx_pipeline_sync(sdx_pipeline* p) {
    return guarded([&] {
        NEED(p);
        p->impl.sync();
    });
}
const char* sdx_pipeline_error_message(sdx_pipeline* p, int stream) {
    static thread_local std::string msg;
    msg.clear();
    guarded([&] {
        NEED(p);
        msg = p->impl.error(stream);
    });
    return msg.c_str();
}
int sdx_pipeline_device_time_ms(sdx_pipeline* p, float* ms) {
    return guarded([&] {
        NEED(p);
        NEED(ms);
        *ms = p->impl.device_time_ms();
    });
}
int sdx_pipeline_reset_timer(sdx_pipeline* p) {
    return guarded([&] {
        NEED(p);
        p->impl.reset_timer();
    });
}
int sdx_pipeline_upload_resident(sdx_pipeline* p, const uint8_t* frames, int count) {
    return guarded([&] {
        NEED(p);
        NEED(frames);
        p->impl.upload_resident(frames, count);
    });
}
int sdx_pipeline_push_resident(sdx_pipeline* p, int copy_outputs) {
    return guarded([&] {
        NEED(p);
        p->impl.push_resident(copy_outputs != 0);
    });
}

int sdx_pipeline_set_profile(sdx_pipeline* p, int on) {
    return guarded([&] {
        NEED(p);
        p->impl.set_profile(on != 0);
    });
}
int sdx_pipeline_stage_times(sdx_pipeline* p, double* ms6, int64_t* iterations, int64_t* total_launches) {
    return guarded([&] {
        NEED(p);
        NEED(ms6);
        long long it = 0;
        p->impl.stage_times(ms6, &it);
        if (iterations) *iterations = it;
        if (total_launches) *total_launches = p->impl.launches();
    });
}
int sdx_pipeline_flops(sdx_pipeline* p, double* unet_per_row, double* codec_per_frame) {
    return guarded([&] {
        NEED(p);
        if (unet_per_row) *unet_per_row = p->impl.unet_flops_per_row();
        if (codec_per_frame) *codec_per_frame = p->impl.taesd_flops();
    });
}

// ---- pinned host memory ----
int sdx_host_alloc(size_t bytes, void** out) {
    return guarded([&] {
        NEED(out);
        SDX_CUDA(cudaMallocHost(out, bytes));
    });
}
int sdx_host_free(void* p) {
    return guarded([&] {
        if (p) SDX_CUDA(cudaFreeHost(p));
    });
}

}  // extern "C"
