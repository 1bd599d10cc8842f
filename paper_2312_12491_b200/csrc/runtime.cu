// Host runtime: device-state owners and the host mirror of the reference's
// engine / pipeline bookkeeping.  See runtime.cuh.
#include "runtime.cuh"

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <sstream>

namespace sdx {

// ---------------------------------------------------------------------------
// EngineMirror — StreamBatchEngine bookkeeping (engine.cpp:53-211)
// ---------------------------------------------------------------------------

void EngineMirror::check_ingest(int64_t seq) const {
    if (seq <= last_seq_) raise(SDX_INVALID_ARGUMENT, "ingest: seq ids must strictly increase");
    for (const auto& f : inflight_)
        if (f.step == 0) raise(SDX_LOGIC_ERROR, "ingest: step-0 slot already occupied, tick first");
}

void EngineMirror::ingest(int64_t seq) {
    inflight_.push_back(Frame{seq, 0, ticks_});
    last_seq_ = seq;
    pending_ = true;
    pending_seq_ = seq;
}

EngineMirror::TickOut EngineMirror::tick() {
    if (inflight_.empty()) raise(SDX_LOGIC_ERROR, "tick: no in-flight frames");
    TickOut out;
    const uint64_t b = inflight_.size();
    out.rows = b;
    if (guidance_ == SDX_GUIDANCE_CFG) out.rows += b;
    if (guidance_ == SDX_GUIDANCE_ONETIME_NEGATIVE && pending_) out.rows += 1;
    ticks_ += 1;
    calls += 1;
    evals += out.rows;
    size_t emit_index = inflight_.size();
    for (size_t i = 0; i < inflight_.size(); ++i) {
        auto& f = inflight_[i];
        f.step += 1;
        if (f.step == n_) {
            out.emitted = true;
            out.seq = f.seq;
            out.ingest_tick = f.ingest_tick;
            out.emit_tick = ticks_;
            emit_index = i;
        }
    }
    if (emit_index < inflight_.size()) inflight_.erase(inflight_.begin() + static_cast<long>(emit_index));
    pending_ = false;
    pending_seq_ = -1;
    return out;
}

std::vector<int> EngineMirror::step_indices() const {
    std::vector<int> v;
    for (const auto& f : inflight_) v.push_back(f.step);
    std::sort(v.begin(), v.end());
    return v;
}

int64_t EngineMirror::min_inflight_seq() const {
    int64_t m = INT64_MAX;
    for (const auto& f : inflight_) m = std::min(m, f.seq);
    return m;
}

// ---------------------------------------------------------------------------
// step table + device engine
// ---------------------------------------------------------------------------

std::vector<StepScalars> make_step_table(const sdx_step* steps, int n, int lcm_mode, double var) {
    std::vector<StepScalars> t(static_cast<size_t>(n) + 1);
    for (int i = 0; i <= n; ++i) {
        const bool term = i == n;
        const int tau = term ? 0 : steps[i].tau;
        const double alpha = term ? 1.0 : steps[i].alpha;
        const double beta = term ? 0.0 : steps[i].beta;
        StepScalars& s = t[static_cast<size_t>(i)];
        s.tau = tau;
        s.alpha = alpha;
        s.beta = beta;
        s.sa = std::sqrt(alpha);
        s.sb = std::sqrt(beta);
        // lcm_coefficients (schedule.cpp:80-89), sigma_data 0.5, s 10
        if (lcm_mode == SDX_LCM_BOUNDARY_APPROX) {
            s.c_skip = tau == 0 ? 1.0 : 0.0;
            s.c_out = tau == 0 ? 0.0 : 1.0;
        } else {
            const double st = 10.0 * tau;
            const double sig2 = 0.25;
            s.c_skip = sig2 / (st * st + sig2);
            s.c_out = 0.5 * st / std::sqrt(sig2 + st * st);
        }
        s.an_scale = std::sqrt(beta) / (alpha * var + beta);
        s.pad = 0;
        s.f_sa = static_cast<float>(s.sa);
        s.f_sb = static_cast<float>(s.sb);
        s.f_isa = static_cast<float>(1.0 / s.sa);
        s.f_isb = beta > 0.0 ? static_cast<float>(1.0 / s.sb) : 0.f;
        s.f_cs = static_cast<float>(s.c_skip);
        s.f_co = static_cast<float>(s.c_out);
        s.f_an = static_cast<float>(s.an_scale);
        s.f_beta = static_cast<float>(beta);
    }
    return t;
}

void DeviceEngine::init(int S_, int n_, long long d_, int guidance_, double gamma_, double delta_,
                        const std::vector<StepScalars>& table, bool per_slot_cond_, bool cross_frame) {
    S = S_;
    n = n_;
    d = d_;
    guidance = guidance_;
    gamma = gamma_;
    delta = delta_;
    per_slot_cond = per_slot_cond_;
    const size_t sn = static_cast<size_t>(S) * n;
    const size_t snd = sn * static_cast<size_t>(d);
    tbl = dev_alloc<StepScalars>(table.size());
    SDX_CUDA(cudaMemcpy(tbl, table.data(), sizeof(StepScalars) * table.size(), cudaMemcpyHostToDevice));
    x_cur = dev_alloc<float>(snd);
    x0 = dev_alloc<float>(snd);
    if (guidance == SDX_GUIDANCE_ONETIME_NEGATIVE) x0ref = dev_alloc<float>(snd);
    eps_cached = dev_alloc<float>(snd);
    cond = dev_alloc<float>(per_slot_cond ? snd : static_cast<size_t>(S) * d);
    if (guidance == SDX_GUIDANCE_CFG || guidance == SDX_GUIDANCE_ONETIME_NEGATIVE)
        neg = dev_alloc<float>(static_cast<size_t>(S) * d);
    emitted = dev_alloc<float>(static_cast<size_t>(S) * d);
    SDX_CUDA(cudaMemset(x_cur, 0, snd * sizeof(float)));
    SDX_CUDA(cudaMemset(x0, 0, snd * sizeof(float)));
    SDX_CUDA(cudaMemset(emitted, 0, static_cast<size_t>(S) * d * sizeof(float)));
    ctl = dev_alloc<StreamCtl>(static_cast<size_t>(S));
    std::vector<StreamCtl> h(static_cast<size_t>(S));
    for (auto& c : h) {
        std::memset(&c, 0, sizeof c);
        c.last_seq = -1;
        c.ingest_slot = -1;
        c.emit_slot = -1;
        c.emit_seq = -1;
        c.mti = 312;
        c.decision = SDX_GATE_PROCESS;
        for (auto& sl : c.slot) sl.seq = -1;
    }
    SDX_CUDA(cudaMemcpy(ctl, h.data(), sizeof(StreamCtl) * h.size(), cudaMemcpyHostToDevice));
    const int rmax = S * 2 * n + S;
    rows = dev_alloc<RowDesc>(static_cast<size_t>(rmax));
    n_rows = dev_alloc<int>(1);
    slot_row_c = dev_alloc<int>(static_cast<size_t>(S) * kMaxSteps);
    slot_row_n = dev_alloc<int>(static_cast<size_t>(S) * kMaxSteps);
    log = dev_alloc<LogEntry>(static_cast<size_t>(S));
    if (cross_frame) {
        xfa_eps = dev_alloc<float>(snd);
        xfa_dots = dev_alloc<double>(static_cast<size_t>(S) * n * n);
    }
}

void DeviceEngine::release() {
    for (void* p : {static_cast<void*>(tbl), static_cast<void*>(x_cur), static_cast<void*>(x0),
                    static_cast<void*>(x0ref), static_cast<void*>(eps_cached), static_cast<void*>(cond),
                    static_cast<void*>(neg), static_cast<void*>(emitted), static_cast<void*>(ctl),
                    static_cast<void*>(rows), static_cast<void*>(n_rows), static_cast<void*>(slot_row_c),
                    static_cast<void*>(slot_row_n), static_cast<void*>(log), static_cast<void*>(xfa_eps),
                    static_cast<void*>(xfa_dots)})
        dev_free(p);
    tbl = nullptr;
}

StepArgs DeviceEngine::step_args() const {
    StepArgs a{};
    a.n = n;
    a.d = d;
    a.guidance = guidance;
    a.gamma = gamma;
    a.delta = delta;
    a.tbl = tbl;
    a.x_cur = x_cur;
    a.x0 = x0;
    a.x0ref = x0ref;
    a.eps_cached = eps_cached;
    a.cond = cond;
    a.cond_stream_stride = per_slot_cond ? static_cast<long long>(n) * d : d;
    a.cond_slot_stride = per_slot_cond ? d : 0;
    a.neg = neg;
    a.eps_ext = nullptr;
    a.eps_ext_stride = 0;
    a.slot_row_c = slot_row_c;
    a.slot_row_n = slot_row_n;
    a.emitted = emitted;
    a.ctl = ctl;
    a.xfa_eps = xfa_eps;
    a.xfa_dots = xfa_dots;
    return a;
}

static void upload_f32(float* dst, const double* src, size_t count, cudaStream_t st) {
    std::vector<float> tmp(count);
    for (size_t i = 0; i < count; ++i) tmp[i] = static_cast<float>(src[i]);
    // pageable source: the call returns once the bytes are staged
    SDX_CUDA(cudaMemcpyAsync(dst, tmp.data(), count * sizeof(float), cudaMemcpyHostToDevice, st));
    SDX_CUDA(cudaStreamSynchronize(st));
}

static std::string config_errors(const sdx_config& c) {
    // validate_config (core.cpp:26-60); all violations joined (core.cpp:62-69)
    std::vector<std::string> e;
    if (c.n_steps < 1) e.push_back("n_steps must be >= 1");
    if (!(c.eta >= 0.0 && c.eta < 1.0)) e.push_back("eta out of range: must lie in [0,1) so 1-eta stays positive");
    if (!(c.gamma >= 0.0)) e.push_back("gamma must be >= 0");
    if (!(c.delta >= 0.0 && c.delta <= 1.0)) e.push_back("delta must lie in [0,1]");
    if (c.d_latent < 1) e.push_back("d_latent must be >= 1");
    if (c.t_grid < 1) e.push_back("t_grid must be >= 1");
    if (c.n_steps > c.t_grid) e.push_back("n_steps must not exceed t_grid");
    if (!(c.entry_strength > 0.0 && c.entry_strength <= 1.0)) e.push_back("entry_strength must lie in (0,1]");
    if (c.backend != SDX_BACKEND_ANALYTIC && c.backend != SDX_BACKEND_UNET)
        e.push_back("backend must be analytic or unet");
    if (!(c.data_variance > 0.0)) e.push_back("data_variance must be > 0");
    if (c.lcm_mode != SDX_LCM_EXACT && c.lcm_mode != SDX_LCM_BOUNDARY_APPROX)
        e.push_back("lcm_mode must be \"exact\" or \"boundary_approx\"");
    if (c.codec != SDX_CODEC_IDENTITY && c.codec != SDX_CODEC_TAESD) e.push_back("codec must be identity or taesd");
    if (c.queue_capacity < 1) e.push_back("queue_capacity must be >= 1");
    if (c.n_steps > kMaxSteps) e.push_back("n_steps exceeds the device slot table (64)");
    if (e.empty()) return {};
    std::ostringstream o;
    o << "invalid config:";
    for (const auto& m : e) o << "\n  - " << m;
    return o.str();
}

// ---------------------------------------------------------------------------
// Engine
// ---------------------------------------------------------------------------

Engine::Engine(const sdx_config& cfg, const sdx_step* steps, int n, const double* eps_cached,
               const double* neg, int device)
    : cfg_(cfg), device_(device), mirror_(cfg.n_steps, cfg.guidance_mode) {
    const std::string errs = config_errors(cfg);
    if (!errs.empty()) raise(SDX_INVALID_ARGUMENT, errs);
    if (cfg.backend != SDX_BACKEND_ANALYTIC)
        raise(SDX_UNSUPPORTED, "engine API: the UNet backend runs through sdx_pipeline");
    if (n != cfg.n_steps) raise(SDX_INVALID_ARGUMENT, "StreamBatchEngine: schedule length != n_steps");
    if (!eps_cached) raise(SDX_INVALID_ARGUMENT, "StreamBatchEngine: noise cache length != n_steps");
    const bool needs_neg = cfg.guidance_mode == SDX_GUIDANCE_CFG || cfg.guidance_mode == SDX_GUIDANCE_ONETIME_NEGATIVE;
    if (needs_neg && !neg) raise(SDX_INVALID_ARGUMENT, "StreamBatchEngine: guidance mode requires negative_cond");
    for (int i = 0; i < n; ++i)
        if (!(steps[i].alpha > 0.0)) raise(SDX_INVALID_ARGUMENT, "predict_x0: singular step (alpha = 0)");
    SDX_CUDA(cudaSetDevice(device_));
    SDX_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    SDX_CUDA(cudaEventCreate(&ev0_));
    SDX_CUDA(cudaEventCreate(&ev1_));
    const auto table = make_step_table(steps, n, cfg.lcm_mode, cfg.data_variance);
    dev_.init(1, n, cfg.d_latent, cfg.guidance_mode, cfg.gamma, cfg.delta, table, /*per_slot_cond=*/true,
              cfg.cross_frame_attention != 0);
    const size_t d = static_cast<size_t>(cfg.d_latent);
    upload_f32(dev_.eps_cached, eps_cached, static_cast<size_t>(n) * d, stream_);
    if (dev_.neg && neg) upload_f32(dev_.neg, neg, d, stream_);
    slot_cond_.resize(static_cast<size_t>(n));
    SDX_CUDA(cudaMallocHost(&h_stage_, sizeof(float) * d));
    SDX_CUDA(cudaMallocHost(&h_log_, sizeof(LogEntry)));
}

Engine::~Engine() {
    cudaSetDevice(device_);
    if (stream_) cudaStreamSynchronize(stream_);
    dev_.release();
    if (h_stage_) cudaFreeHost(h_stage_);
    if (h_log_) cudaFreeHost(h_log_);
    if (ev0_) cudaEventDestroy(ev0_);
    if (ev1_) cudaEventDestroy(ev1_);
    if (stream_) cudaStreamDestroy(stream_);
}

void Engine::ingest(int64_t seq, const double* x0, const double* cond) {
    const size_t d = static_cast<size_t>(cfg_.d_latent);
    if (!x0 || !cond) raise(SDX_INVALID_ARGUMENT, "ingest: latent length != d_latent");
    for (size_t i = 0; i < d; ++i)
        if (!std::isfinite(x0[i])) raise(SDX_INVALID_ARGUMENT, "ingest: non-finite latent");
    mirror_.check_ingest(seq);
    SDX_CUDA(cudaSetDevice(device_));
    const int slot = static_cast<int>(mirror_.ticks() % cfg_.n_steps);
    upload_f32(dev_.x0 + static_cast<size_t>(slot) * d, x0, d, stream_);
    auto& last = slot_cond_[static_cast<size_t>(slot)];
    bool same = last.size() == d;
    for (size_t i = 0; same && i < d; ++i) same = last[i] == static_cast<float>(cond[i]);
    if (!same) {
        last.resize(d);
        for (size_t i = 0; i < d; ++i) last[i] = static_cast<float>(cond[i]);
        SDX_CUDA(cudaMemcpyAsync(dev_.cond + static_cast<size_t>(slot) * d, last.data(), d * sizeof(float),
                                 cudaMemcpyHostToDevice, stream_));
    }
    mirror_.ingest(seq);
}

sdx_tick_result Engine::tick(double* x0_hat) {
    const bool pend = mirror_.pending_ingest();
    const int64_t pseq = mirror_.pending_seq();
    const auto t = mirror_.tick();  // throws logic_error on an empty engine
    SDX_CUDA(cudaSetDevice(device_));
    const int n = cfg_.n_steps;
    SDX_CUDA(cudaEventRecord(ev0_, stream_));
    launch_ctl_begin(dev_.ctl, 1, n, cfg_.guidance_mode, kIngestHost, pend ? pseq : -1, 0, nullptr, nullptr,
                     nullptr, nullptr, stream_);
    launch_step(dev_.step_args(), 1, stream_);
    launch_ctl_end(dev_.ctl, 1, n, cfg_.guidance_mode, dev_.log, 0, stream_);
    SDX_CUDA(cudaEventRecord(ev1_, stream_));
    timed_ = true;
    sdx_tick_result r{};
    r.emitted_seq = -1;
    r.denoiser_calls = 1;
    r.element_evals = t.rows;
    if (t.emitted) {
        const size_t d = static_cast<size_t>(cfg_.d_latent);
        SDX_CUDA(cudaMemcpyAsync(h_log_, dev_.log, sizeof(LogEntry), cudaMemcpyDeviceToHost, stream_));
        SDX_CUDA(cudaMemcpyAsync(h_stage_, dev_.emitted, d * sizeof(float), cudaMemcpyDeviceToHost, stream_));
        SDX_CUDA(cudaStreamSynchronize(stream_));
        if (h_log_->emit_seq != t.seq) raise(SDX_RUNTIME_ERROR, "device/host engine mirror diverged");
        if (h_log_->nonfinite) raise(SDX_RUNTIME_ERROR, "tick: non-finite latent at emission");
        if (x0_hat)
            for (size_t i = 0; i < d; ++i) x0_hat[i] = static_cast<double>(h_stage_[i]);
        r.emitted_seq = t.seq;
        r.ingest_tick = t.ingest_tick;
        r.emit_tick = t.emit_tick;
    }
    float ms = 0.f;
    SDX_CUDA(cudaEventSynchronize(ev1_));
    SDX_CUDA(cudaEventElapsedTime(&ms, ev0_, ev1_));
    last_ms_ = ms;
    return r;
}

// ---------------------------------------------------------------------------
// MT19937-64 seeding (std::mt19937_64)
// ---------------------------------------------------------------------------

void mt_seed_words(uint64_t seed, unsigned long long* mt) {
    mt[0] = seed;
    for (int i = 1; i < 312; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i;
}

// ---------------------------------------------------------------------------
// Ssf
// ---------------------------------------------------------------------------

Ssf::Ssf(double eta, uint64_t seed, int max_skip, int64_t frame_bytes, int device)
    : eta_(eta), max_skip_(max_skip), D_(frame_bytes), device_(device) {
    if (!(eta >= 0.0 && eta < 1.0)) raise(SDX_INVALID_ARGUMENT, "SsfState: eta must lie in [0,1)");
    if (frame_bytes < 1) raise(SDX_INVALID_ARGUMENT, "SsfState: frame_bytes must be >= 1");
    SDX_CUDA(cudaSetDevice(device_));
    SDX_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    const int64_t pad = (D_ + 15) / 16 * 16;
    batch_ = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(64, (64LL << 20) / pad)));
    d_frames_ = dev_alloc<uint8_t>(static_cast<size_t>(pad) * batch_);
    d_ref_ = dev_alloc<uint8_t>(static_cast<size_t>(pad));
    SDX_CUDA(cudaMemset(d_ref_, 0, static_cast<size_t>(pad)));
    ctl_ = dev_alloc<StreamCtl>(1);
    StreamCtl h;
    std::memset(&h, 0, sizeof h);
    h.mti = 312;
    h.decision = SDX_GATE_PROCESS;
    for (auto& sl : h.slot) sl.seq = -1;
    SDX_CUDA(cudaMemcpy(ctl_, &h, sizeof h, cudaMemcpyHostToDevice));
    mt_ = dev_alloc<unsigned long long>(312);
    unsigned long long words[312];
    mt_seed_words(seed, words);
    SDX_CUDA(cudaMemcpy(mt_, words, sizeof words, cudaMemcpyHostToDevice));
    dec_ = dev_alloc<int>(static_cast<size_t>(batch_));
    sims_ = dev_alloc<double>(static_cast<size_t>(batch_));
}

Ssf::~Ssf() {
    cudaSetDevice(device_);
    if (stream_) cudaStreamSynchronize(stream_);
    dev_free(d_frames_);
    dev_free(d_ref_);
    dev_free(ctl_);
    dev_free(mt_);
    dev_free(dec_);
    dev_free(sims_);
    if (stream_) cudaStreamDestroy(stream_);
}

void Ssf::gate(const uint8_t* frames, int nframes, int* decisions, double* sims) {
    SDX_CUDA(cudaSetDevice(device_));
    const int64_t pad = (D_ + 15) / 16 * 16;
    std::vector<int> hd(static_cast<size_t>(batch_));
    std::vector<double> hs(static_cast<size_t>(batch_));
    for (int base = 0; base < nframes; base += batch_) {
        const int cnt = std::min(batch_, nframes - base);
        for (int i = 0; i < cnt; ++i)
            SDX_CUDA(cudaMemcpyAsync(d_frames_ + static_cast<size_t>(i) * pad,
                                     frames + static_cast<size_t>(base + i) * D_, static_cast<size_t>(D_),
                                     cudaMemcpyHostToDevice, stream_));
        for (int i = 0; i < cnt; ++i) {
            SsfArgs a{};
            a.frames = d_frames_ + static_cast<size_t>(i) * pad;
            a.frame_stride = pad;
            a.ref = d_ref_;
            a.D = D_;
            a.eta = eta_;
            a.max_skip = max_skip_;
            a.ctl = ctl_;
            a.mt_state = mt_;
            a.dec_out = dec_ + i;
            a.sim_out = sims_ + i;
            launch_ssf_reduce(a, 1, stream_);
            CommitArgs ca{};
            ca.frames = a.frames;
            ca.frame_stride = pad;
            ca.ref = d_ref_;
            ca.D = D_;
            ca.x0 = nullptr;
            ca.ctl = ctl_;
            launch_commit_encode(ca, 1, stream_);
        }
        SDX_CUDA(cudaMemcpyAsync(hd.data(), dec_, sizeof(int) * cnt, cudaMemcpyDeviceToHost, stream_));
        SDX_CUDA(cudaMemcpyAsync(hs.data(), sims_, sizeof(double) * cnt, cudaMemcpyDeviceToHost, stream_));
        SDX_CUDA(cudaStreamSynchronize(stream_));
        for (int i = 0; i < cnt; ++i) {
            examined_ += 1;
            if (hd[static_cast<size_t>(i)] == SDX_GATE_SKIP) skipped_ += 1;
            if (decisions) decisions[base + i] = hd[static_cast<size_t>(i)];
            if (sims) sims[base + i] = hs[static_cast<size_t>(i)];
        }
    }
}

// ---------------------------------------------------------------------------
// Pipeline
// ---------------------------------------------------------------------------

Pipeline::Pipeline(const sdx_pipeline_config& cfg, const sdx_step* steps, const double* eps_cached,
                   const double* cond, const double* neg, int device)
    : cfg_(cfg), S_(cfg.n_streams), n_(cfg.engine.n_steps), K_(std::max(2, cfg.ring_depth)),
      D_(cfg.frame_bytes), d_(cfg.engine.d_latent), device_(device) {
    const auto& e = cfg.engine;
    const std::string errs = config_errors(e);
    if (!errs.empty()) raise(SDX_INVALID_ARGUMENT, errs);
    if (S_ < 1 || S_ > 1024) raise(SDX_INVALID_ARGUMENT, "n_streams must lie in [1,1024]");
    if (e.codec == SDX_CODEC_IDENTITY && D_ != d_)
        raise(SDX_INVALID_ARGUMENT, "LatentCodec::encode: dim mismatch");
    if (e.codec == SDX_CODEC_TAESD && (D_ != 3LL * 512 * 512 || d_ != 4LL * 64 * 64))
        raise(SDX_INVALID_ARGUMENT, "TAESD codec: frames are 3x512x512 u8 and latents 4x64x64");
    if (e.backend == SDX_BACKEND_UNET && d_ != 4LL * 64 * 64)
        raise(SDX_INVALID_ARGUMENT, "UNet backend: d_latent must be 4x64x64 = 16384");
    const bool needs_neg = e.guidance_mode == SDX_GUIDANCE_CFG || e.guidance_mode == SDX_GUIDANCE_ONETIME_NEGATIVE;
    if (needs_neg && !neg)
        raise(SDX_INVALID_ARGUMENT,
              "invalid config:\n  - negative_condition is required for cfg/onetime_negative modes");
    for (int i = 0; i < n_; ++i)
        if (!(steps[i].alpha > 0.0)) raise(SDX_INVALID_ARGUMENT, "predict_x0: singular step (alpha = 0)");
    SDX_CUDA(cudaSetDevice(device_));
    SDX_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    SDX_CUDA(cudaStreamCreateWithFlags(&copy_, cudaStreamNonBlocking));
    const auto table = make_step_table(steps, n_, e.lcm_mode, e.data_variance);
    dev_.init(S_, n_, d_, e.guidance_mode, e.gamma, e.delta, table, /*per_slot_cond=*/false,
              e.cross_frame_attention != 0);
    const size_t d = static_cast<size_t>(d_);
    upload_f32(dev_.eps_cached, eps_cached, static_cast<size_t>(S_) * n_ * d, stream_);
    upload_f32(dev_.cond, cond, static_cast<size_t>(S_) * d, stream_);
    if (dev_.neg && neg) upload_f32(dev_.neg, neg, static_cast<size_t>(S_) * d, stream_);
    pad_ = (D_ + 15) / 16 * 16;
    d_in_ = dev_alloc<uint8_t>(static_cast<size_t>(K_) * S_ * pad_);
    if (e.ssf_enabled) {
        d_ref_ = dev_alloc<uint8_t>(static_cast<size_t>(S_) * pad_);
        SDX_CUDA(cudaMemset(d_ref_, 0, static_cast<size_t>(S_) * pad_));
        mt_ = dev_alloc<unsigned long long>(static_cast<size_t>(S_) * 312);
        std::vector<unsigned long long> words(static_cast<size_t>(S_) * 312);
        for (int s = 0; s < S_; ++s) {
            // per-stream SSF Rng(derive_seed(seed_s, kStreamSsf)), pipeline.cpp:166-167
            uint64_t z = (e.seed + static_cast<uint64_t>(s)) + 0x9e3779b97f4a7c15ULL * (2 + 1);
            z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
            z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
            z = z ^ (z >> 31);
            mt_seed_words(z, words.data() + static_cast<size_t>(s) * 312);
        }
        SDX_CUDA(cudaMemcpy(mt_, words.data(), words.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice));
    }
    const bool taesd = e.codec == SDX_CODEC_TAESD;
    out_bytes_ = taesd ? static_cast<size_t>(D_) : d * sizeof(float);
    if (taesd || e.backend == SDX_BACKEND_UNET) {
        lists_buf_ = dev_alloc<int>(static_cast<size_t>(4 * S_ + 2));
        SDX_CUDA(cudaMemset(lists_buf_, 0, sizeof(int) * (4 * S_ + 2)));
        lists_.enc_src = lists_buf_;
        lists_.enc_dst = lists_buf_ + S_;
        lists_.dec_src = lists_buf_ + 2 * S_;
        lists_.dec_dst = lists_buf_ + 3 * S_;
        lists_.n_ingest = lists_buf_ + 4 * S_;
        lists_.n_emit = lists_buf_ + 4 * S_ + 1;
    }
    if (e.backend == SDX_BACKEND_UNET) {
        // rows per stream: n (none / self), 2n (cfg), n + 1 (onetime)  (engine.cpp:97-118)
        const int per = e.guidance_mode == SDX_GUIDANCE_CFG ? 2 * n_
                        : e.guidance_mode == SDX_GUIDANCE_ONETIME_NEGATIVE ? n_ + 1 : n_;
        unet_rmax_ = S_ * per;
        UNetConfig uc;
        uc.rmax = unet_rmax_;
        for (int i = 0; i < n_; ++i) uc.taus.push_back(steps[i].tau);
        uc.seed = e.seed ^ 0x5EEDULL;
        unet_ = std::make_unique<UNet>(uc, stream_);
        lists_.row_step = unet_->row_step();
        lists_.row_prompt = unet_->row_prompt();
    }
    if (taesd) {
        d_out_ = dev_alloc<uint8_t>(static_cast<size_t>(K_) * S_ * D_);
        TaesdIO io;
        io.frames = d_in_;
        io.frame_stride = pad_;
        // the encoder always encodes all S frames of a ring slot into enc_stage_ (identity
        // lists of that slot, copied into enc_lists_ first); the iteration gathers
        const int nl2 = 2 * S_ + 1;
        enc_stage_ = dev_alloc<float>(static_cast<size_t>(K_) * S_ * d);
        enc_lists_ = dev_alloc<int>(static_cast<size_t>(nl2));
        spec_lists_ = dev_alloc<int>(static_cast<size_t>(K_) * nl2);
        {
            std::vector<int> hl(static_cast<size_t>(K_) * nl2);
            for (int k = 0; k < K_; ++k) {
                for (int s2 = 0; s2 < S_; ++s2) {
                    hl[static_cast<size_t>(k) * nl2 + s2] = k * S_ + s2;       // src frame
                    hl[static_cast<size_t>(k) * nl2 + S_ + s2] = k * S_ + s2;  // dst staging block
                }
                hl[static_cast<size_t>(k) * nl2 + 2 * S_] = S_;
            }
            SDX_CUDA(cudaMemcpy(spec_lists_, hl.data(), sizeof(int) * hl.size(), cudaMemcpyHostToDevice));
            SDX_CUDA(cudaMemcpy(enc_lists_, hl.data(), sizeof(int) * nl2, cudaMemcpyHostToDevice));
        }
        io.enc_src = enc_lists_;
        io.enc_count = enc_lists_ + 2 * S_;
        io.latent_out = enc_stage_;
        io.enc_dst = enc_lists_ + S_;
        // the decoder reads its own copy of the emitted latents and codec lists
        // (staged per ring slot by the main part of the iteration)
        const int nl = 4 * S_ + 2;
        stage_lat_ = dev_alloc<float>(static_cast<size_t>(K_) * S_ * d);
        stage_lists_ = dev_alloc<int>(static_cast<size_t>(K_) * nl);
        dec_in_ = dev_alloc<float>(static_cast<size_t>(S_) * d);
        dec_lists_ = dev_alloc<int>(static_cast<size_t>(nl));
        SDX_CUDA(cudaMemset(stage_lists_, 0, sizeof(int) * K_ * nl));
        SDX_CUDA(cudaMemset(dec_lists_, 0, sizeof(int) * nl));
        io.latent_in = dec_in_;
        io.dec_src = dec_lists_ + 2 * S_;
        io.dec_count = dec_lists_ + 4 * S_ + 1;
        io.frames_out = d_out_;
        io.dec_dst = dec_lists_ + 3 * S_;
        const char* ov = std::getenv("SDX_DECODE_OVERLAP");
        overlap_ = !(ov && ov[0] == '0');
        const char* oe = std::getenv("SDX_ENCODE_OVERLAP");
        enc_overlap_ = !(oe && oe[0] == '0');
        io.separate_decoder_buffers = overlap_ || enc_overlap_;
        taesd_ = std::make_unique<TAESD>(S_, e.seed ^ 0x7AE5DULL, io, stream_);
        if (overlap_) {
            SDX_CUDA(cudaStreamCreateWithFlags(&dec_stream_, cudaStreamNonBlocking));
            main_done_.resize(static_cast<size_t>(K_));
            for (auto& ev : main_done_) SDX_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            SDX_CUDA(cudaEventCreateWithFlags(&dec_join_, cudaEventDisableTiming));
        }
        if (enc_overlap_) {
            SDX_CUDA(cudaStreamCreateWithFlags(&enc_stream_, cudaStreamNonBlocking));
            enc_done_.resize(static_cast<size_t>(K_));
            for (auto& ev : enc_done_) SDX_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        }
    }
    SDX_CUDA(cudaMallocHost(&h_in_, static_cast<size_t>(K_) * S_ * D_));
    SDX_CUDA(cudaMallocHost(&h_out_, static_cast<size_t>(K_) * S_ * out_bytes_));
    SDX_CUDA(cudaMallocHost(&h_log_, static_cast<size_t>(K_) * S_ * sizeof(LogEntry)));
    done_.resize(static_cast<size_t>(K_));
    h2d_.resize(static_cast<size_t>(K_));
    for (int k = 0; k < K_; ++k) {
        SDX_CUDA(cudaEventCreateWithFlags(&done_[static_cast<size_t>(k)], cudaEventDisableTiming));
        SDX_CUDA(cudaEventCreateWithFlags(&h2d_[static_cast<size_t>(k)], cudaEventDisableTiming));
    }
    SDX_CUDA(cudaEventCreate(&t0_));
    SDX_CUDA(cudaEventCreate(&t1_));
    st_.resize(static_cast<size_t>(S_));
    for (auto& h : st_) h.eng = std::make_unique<EngineMirror>(n_, e.guidance_mode);
}

Pipeline::~Pipeline() {
    cudaSetDevice(device_);
    if (stream_) cudaStreamSynchronize(stream_);
    if (copy_) cudaStreamSynchronize(copy_);
    if (dec_stream_) cudaStreamSynchronize(dec_stream_);
    if (enc_stream_) cudaStreamSynchronize(enc_stream_);
    for (auto gexec : graphs_)
        if (gexec) cudaGraphExecDestroy(gexec);
    for (auto gexec : enc_graphs_)
        if (gexec) cudaGraphExecDestroy(gexec);
    for (auto gexec : dec_graphs_)
        if (gexec) cudaGraphExecDestroy(gexec);
    taesd_.reset();
    unet_.reset();
    dev_free(lists_buf_);
    dev_free(d_out_);
    dev_free(stage_lat_);
    dev_free(stage_lists_);
    dev_free(dec_in_);
    dev_free(dec_lists_);
    for (auto ev : main_done_) cudaEventDestroy(ev);
    if (dec_join_) cudaEventDestroy(dec_join_);
    if (dec_stream_) cudaStreamDestroy(dec_stream_);
    dev_free(enc_stage_);
    dev_free(enc_lists_);
    dev_free(spec_lists_);
    for (auto ev : enc_done_) cudaEventDestroy(ev);
    if (enc_stream_) cudaStreamDestroy(enc_stream_);
    dev_.release();
    dev_free(d_in_);
    dev_free(d_ref_);
    dev_free(mt_);
    if (h_in_) cudaFreeHost(h_in_);
    if (h_out_) cudaFreeHost(h_out_);
    if (h_log_) cudaFreeHost(h_log_);
    for (auto ev : done_) cudaEventDestroy(ev);
    for (auto ev : h2d_) cudaEventDestroy(ev);
    for (auto ev : kt_) cudaEventDestroy(ev);
    if (t0_) cudaEventDestroy(t0_);
    if (t1_) cudaEventDestroy(t1_);
    if (stream_) cudaStreamDestroy(stream_);
    if (copy_) cudaStreamDestroy(copy_);
}

void Pipeline::launch_iteration(int k, bool frame_present) {
    const auto& e = cfg_.engine;
    uint8_t* frames = d_in_ + static_cast<size_t>(k) * S_ * pad_;
    const bool taesd = e.codec == SDX_CODEC_TAESD;
    const bool unet = e.backend == SDX_BACKEND_UNET;
    auto mark = [&](int i) {
        if (profile_) SDX_CUDA(cudaEventRecord(kt_[static_cast<size_t>(k) * kMarks + i], stream_));
    };
    mark(0);
    if (frame_present) {
        if (e.ssf_enabled) {
            SsfArgs a{};
            a.frames = frames;
            a.frame_stride = pad_;
            a.ref = d_ref_;
            a.D = D_;
            a.eta = e.eta;
            a.max_skip = cfg_.max_skip;
            a.ctl = dev_.ctl;
            a.mt_state = mt_;
            launch_ssf_reduce(a, S_, stream_);
            launches_ += 1;
        }
        mark(1);
        launch_ctl_begin(dev_.ctl, S_, n_, e.guidance_mode, e.ssf_enabled ? kIngestSsf : kIngestAlways, -1, 1,
                         dev_.rows, dev_.n_rows, dev_.slot_row_c, dev_.slot_row_n, stream_);
        launches_ += 1;
        if (e.ssf_enabled || !taesd) {
            CommitArgs ca{};
            ca.frames = frames;
            ca.frame_stride = pad_;
            ca.ref = e.ssf_enabled ? d_ref_ : nullptr;
            ca.D = D_;
            ca.x0 = taesd ? nullptr : dev_.x0;
            ca.n = n_;
            ca.d = d_;
            ca.ctl = dev_.ctl;
            launch_commit_encode(ca, S_, stream_);
            launches_ += 1;
        }
    } else {
        mark(1);
        launch_ctl_begin(dev_.ctl, S_, n_, e.guidance_mode, kIngestAlways, -1, 0, dev_.rows, dev_.n_rows,
                         dev_.slot_row_c, dev_.slot_row_n, stream_);
        launches_ += 1;
    }
    if (taesd || unet) {
        launch_ctl_lists(dev_.ctl, S_, n_, k, dev_.rows, dev_.n_rows, lists_, stream_);
        launches_ += 1;
    }
    mark(2);
    if (taesd && frame_present) {
        if (!(enc_overlap_ && !profile_)) launch_encode(k, stream_);  // else encoded ahead (run_encode)
        launch_enc_gather(lists_, S_, enc_stage_, dev_.x0, d_, stream_);
        launches_ += 1;
    }
    mark(3);
    StepArgs sa = dev_.step_args();
    if (unet) {
        launch_unet_prep(dev_.ctl, dev_.rows, dev_.n_rows, unet_rmax_, n_, d_, dev_.x_cur, dev_.x0, dev_.eps_cached,
                         dev_.tbl, unet_->input(), stream_);
        unet_->forward(dev_.n_rows, stream_);
        launches_ += 1 + unet_->launches_per_forward();
        sa.eps_ext = unet_->output();
        sa.eps_ext_stride = d_;
    }
    mark(4);
    launch_step(sa, S_, stream_);
    launch_ctl_end(dev_.ctl, S_, n_, e.guidance_mode, dev_.log, frame_present ? 1 : 0, stream_);
    launches_ += 2;
    mark(5);
    if (taesd) {
        // stage this slot's emitted latents and codec lists for its decode
        const int nl = 4 * S_ + 2;
        SDX_CUDA(cudaMemcpyAsync(stage_lat_ + static_cast<size_t>(k) * S_ * d_, dev_.emitted,
                                 sizeof(float) * S_ * d_, cudaMemcpyDeviceToDevice, stream_));
        SDX_CUDA(cudaMemcpyAsync(stage_lists_ + static_cast<size_t>(k) * nl, lists_buf_, sizeof(int) * nl,
                                 cudaMemcpyDeviceToDevice, stream_));
        if (!(overlap_ && !profile_)) launch_decode(k, stream_);
    }
    mark(6);
    SDX_CUDA(cudaMemcpyAsync(h_log_ + static_cast<size_t>(k) * S_, dev_.log, sizeof(LogEntry) * S_,
                             cudaMemcpyDeviceToHost, stream_));
    if (!taesd && (!resident_ || copy_outputs_))
        SDX_CUDA(cudaMemcpyAsync(h_out_ + static_cast<size_t>(k) * S_ * out_bytes_, dev_.emitted, out_bytes_ * S_,
                                 cudaMemcpyDeviceToHost, stream_));
}

// Decode of ring slot k (TAESD codec): the staged latents and lists into the
// decoder's inputs, the decoder, the frames back to the host.
void Pipeline::launch_decode(int k, cudaStream_t s) {
    const int nl = 4 * S_ + 2;
    SDX_CUDA(cudaMemcpyAsync(dec_in_, stage_lat_ + static_cast<size_t>(k) * S_ * d_, sizeof(float) * S_ * d_,
                             cudaMemcpyDeviceToDevice, s));
    SDX_CUDA(cudaMemcpyAsync(dec_lists_, stage_lists_ + static_cast<size_t>(k) * nl, sizeof(int) * nl,
                             cudaMemcpyDeviceToDevice, s));
    taesd_->decode(s);
    launches_ += taesd_->launches_per_decode();
    if (!resident_ || copy_outputs_)
        SDX_CUDA(cudaMemcpyAsync(h_out_ + static_cast<size_t>(k) * S_ * out_bytes_,
                                 d_out_ + static_cast<size_t>(k) * S_ * out_bytes_, out_bytes_ * S_,
                                 cudaMemcpyDeviceToHost, s));
}

// Encode all S frames of ring slot k into enc_stage_ (its identity lists first).
void Pipeline::launch_encode(int k, cudaStream_t s) {
    const int nl2 = 2 * S_ + 1;
    SDX_CUDA(cudaMemcpyAsync(enc_lists_, spec_lists_ + static_cast<size_t>(k) * nl2, sizeof(int) * nl2,
                             cudaMemcpyDeviceToDevice, s));
    taesd_->encode(s);
    launches_ += taesd_->launches_per_encode();
}

// Encode ahead: slot k's frames on enc_stream_ once they are in HBM (h2d_[k]),
// overlapping the iterations still running; the iteration waits enc_done_[k].
void Pipeline::run_encode(int k) {
    SDX_CUDA(cudaStreamWaitEvent(enc_stream_, h2d_[static_cast<size_t>(k)], 0));
    if (!cfg_.graph) {
        launch_encode(k, enc_stream_);
    } else {
        if (enc_graphs_.size() < static_cast<size_t>(K_)) enc_graphs_.assign(static_cast<size_t>(K_), nullptr);
        if (!enc_graphs_[static_cast<size_t>(k)]) {
            const long long before = launches_;
            cudaGraph_t g = nullptr;
            SDX_CUDA(cudaStreamBeginCapture(enc_stream_, cudaStreamCaptureModeThreadLocal));
            launch_encode(k, enc_stream_);
            SDX_CUDA(cudaStreamEndCapture(enc_stream_, &g));
            SDX_CUDA(cudaGraphInstantiate(&enc_graphs_[static_cast<size_t>(k)], g, 0));
            SDX_CUDA(cudaGraphDestroy(g));
            enc_graph_launches_ = launches_ - before;
            launches_ = before;
        }
        SDX_CUDA(cudaGraphLaunch(enc_graphs_[static_cast<size_t>(k)], enc_stream_));
        launches_ += enc_graph_launches_;
    }
    SDX_CUDA(cudaEventRecord(enc_done_[static_cast<size_t>(k)], enc_stream_));
}

// Make stream_ wait for every decode issued so far (timer marks, sync).
void Pipeline::join_decode() {
    // the encode-ahead stream never runs past the main stream's waits, so joining the
    // decode stream (which waits for the main stream) covers it as well
    if (!dec_stream_) return;
    SDX_CUDA(cudaEventRecord(dec_join_, dec_stream_));
    SDX_CUDA(cudaStreamWaitEvent(stream_, dec_join_, 0));
}

// One iteration on ring slot k: wait for the slot's H2D, run the iteration
// (replaying its CUDA graph when graphs are enabled), mark completion.
void Pipeline::run_iteration(int k, bool frame_present) {
    if (frame_present) SDX_CUDA(cudaStreamWaitEvent(stream_, h2d_[static_cast<size_t>(k)], 0));
    if (frame_present && taesd_ && enc_overlap_ && !profile_) {
        run_encode(k);
        SDX_CUDA(cudaStreamWaitEvent(stream_, enc_done_[static_cast<size_t>(k)], 0));
    }
    const bool use_graph = cfg_.graph && !profile_;
    if (!use_graph) {
        launch_iteration(k, frame_present);
    } else {
        // one graph per (ring slot, output-copy variant, frame present): pointers differ per slot
        const int key = (k * 2 + ((!resident_ || copy_outputs_) ? 1 : 0)) * 2 + (frame_present ? 1 : 0);
        if (graphs_.size() < static_cast<size_t>(4 * K_)) {
            graphs_.assign(static_cast<size_t>(4 * K_), nullptr);
            graph_launches_.assign(static_cast<size_t>(4 * K_), 0);
        }
        if (!graphs_[static_cast<size_t>(key)]) {
            const long long before = launches_;
            cudaGraph_t g = nullptr;
            SDX_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
            launch_iteration(k, frame_present);
            SDX_CUDA(cudaStreamEndCapture(stream_, &g));
            SDX_CUDA(cudaGraphInstantiate(&graphs_[static_cast<size_t>(key)], g, 0));
            SDX_CUDA(cudaGraphDestroy(g));
            graph_launches_[static_cast<size_t>(key)] = launches_ - before;
            launches_ = before;
        }
        SDX_CUDA(cudaGraphLaunch(graphs_[static_cast<size_t>(key)], stream_));
        launches_ += graph_launches_[static_cast<size_t>(key)];
    }
    if (taesd_ && overlap_ && !profile_) {
        // the decode of slot k overlaps the next iteration's main part
        SDX_CUDA(cudaEventRecord(main_done_[static_cast<size_t>(k)], stream_));
        SDX_CUDA(cudaStreamWaitEvent(dec_stream_, main_done_[static_cast<size_t>(k)], 0));
        if (!cfg_.graph) {
            launch_decode(k, dec_stream_);
        } else {
            const int key = k * 2 + ((!resident_ || copy_outputs_) ? 1 : 0);
            if (dec_graphs_.size() < static_cast<size_t>(2 * K_)) {
                dec_graphs_.assign(static_cast<size_t>(2 * K_), nullptr);
                dec_graph_launches_.assign(static_cast<size_t>(2 * K_), 0);
            }
            if (!dec_graphs_[static_cast<size_t>(key)]) {
                const long long before = launches_;
                cudaGraph_t g = nullptr;
                SDX_CUDA(cudaStreamBeginCapture(dec_stream_, cudaStreamCaptureModeThreadLocal));
                launch_decode(k, dec_stream_);
                SDX_CUDA(cudaStreamEndCapture(dec_stream_, &g));
                SDX_CUDA(cudaGraphInstantiate(&dec_graphs_[static_cast<size_t>(key)], g, 0));
                SDX_CUDA(cudaGraphDestroy(g));
                dec_graph_launches_[static_cast<size_t>(key)] = launches_ - before;
                launches_ = before;
            }
            SDX_CUDA(cudaGraphLaunch(dec_graphs_[static_cast<size_t>(key)], dec_stream_));
            launches_ += dec_graph_launches_[static_cast<size_t>(key)];
        }
        SDX_CUDA(cudaEventRecord(done_[static_cast<size_t>(k)], dec_stream_));
    } else {
        SDX_CUDA(cudaEventRecord(done_[static_cast<size_t>(k)], stream_));
    }
}

std::shared_ptr<std::vector<uint8_t>> Pipeline::acquire_buffer() {
    // recycle output buffers nobody references any more (no page faults per frame)
    for (auto& b : pool_)
        if (b.use_count() == 1) return b;
    pool_.push_back(std::make_shared<std::vector<uint8_t>>(out_bytes_));
    return pool_.back();
}

int64_t Pipeline::src_of(const StreamHost& h, int64_t dev_seq) {
    return h.src_ids[static_cast<size_t>(dev_seq - h.src_base)];
}

// Drop the source ids no future output can refer to: below every pending skip,
// every in-flight frame and every frame not yet processed.
void Pipeline::trim_src(StreamHost& h) {
    int64_t keep = static_cast<int64_t>(h.frames_in);
    if (!h.pending_skips.empty()) keep = std::min(keep, h.pending_skips.front());
    keep = std::min(keep, h.eng->min_inflight_seq());
    while (h.src_base < keep && !h.src_ids.empty()) {
        h.src_ids.pop_front();
        h.src_base += 1;
    }
}

void Pipeline::flush_below(StreamHost& h, int64_t limit, std::vector<Out>& staged) {
    // EngineStage::flush_skips_below (pipeline.cpp:102-116); limit is a device frame index
    while (!h.pending_skips.empty() && h.pending_skips.front() < limit) {
        const int64_t seq = h.pending_skips.front();
        h.pending_skips.pop_front();
        if (!h.has_output) {
            h.stale += 1;
            continue;
        }
        h.duplicates += 1;
        staged.push_back(Out{src_of(h, seq), h.last_output});
    }
}

void Pipeline::process(int k, bool frame_present) {
    const auto& e = cfg_.engine;
    if (profile_) {
        for (int i = 0; i + 1 < kMarks; ++i) {
            float ms = 0.f;
            SDX_CUDA(cudaEventElapsedTime(&ms, kt_[static_cast<size_t>(k) * kMarks + i],
                                          kt_[static_cast<size_t>(k) * kMarks + i + 1]));
            ktime_[i] += ms;
        }
        kcount_ += 1;
    }
    const size_t cap8 = static_cast<size_t>(e.queue_capacity) * 8;
    int64_t iter_ns = 0;  // device time of this iteration (stage profiling only)
    if (profile_) {
        float ms = 0.f;
        SDX_CUDA(cudaEventElapsedTime(&ms, kt_[static_cast<size_t>(k) * kMarks], kt_[static_cast<size_t>(k) * kMarks + kMarks - 1]));
        iter_ns = static_cast<int64_t>(static_cast<double>(ms) * 1e6);
    }
    for (int s = 0; s < S_; ++s) {
        StreamHost& h = st_[static_cast<size_t>(s)];
        if (h.incomplete) continue;
        const LogEntry& L = h_log_[static_cast<size_t>(k) * S_ + s];
        std::vector<Out> staged;
        if (frame_present) {
            h.frames_in += 1;
            const bool skip = e.ssf_enabled && L.decision == SDX_GATE_SKIP;
            if (e.ssf_enabled) {
                h.examined += 1;
                if (skip) h.skipped += 1;
                h.decisions.push_back(L.decision);
            }
            if (skip) {
                h.pending_skips.push_back(L.seq_in);
            } else {
                // StreamBatchEngine::ingest (engine.cpp:59-60) on the source id
                const int64_t src = src_of(h, L.seq_in);
                if (src <= h.last_src) {
                    h.incomplete = true;
                    h.error = "ingest: seq ids must strictly increase";
                    continue;
                }
                h.last_src = src;
                h.eng->ingest(L.seq_in);
            }
        }
        const bool ingested_now = frame_present && !(e.ssf_enabled && L.decision == SDX_GATE_SKIP);
        if (!h.eng->idle()) {
            const uint64_t calls0 = h.eng->calls, evals0 = h.eng->evals;
            const auto t = h.eng->tick();
            if (h.trace.size() < (size_t(1) << 20))
                h.trace.push_back(sdx_trace_entry{h.eng->ticks(), ingested_now ? src_of(h, L.seq_in) : -1,
                                                  t.emitted ? src_of(h, t.seq) : -1, h.eng->calls - calls0,
                                                  h.eng->evals - evals0, iter_ns});
            if (t.emitted != (L.emit_seq >= 0) || (t.emitted && t.seq != L.emit_seq)) {
                h.incomplete = true;
                h.error = "device/host engine mirror diverged";
                continue;
            }
            if (t.emitted) {
                if (L.nonfinite) {
                    h.incomplete = true;
                    h.error = "tick: non-finite latent at emission";
                    continue;
                }
                flush_below(h, t.seq, staged);
                // benchmark path without output copies: order only, no payload
                std::shared_ptr<std::vector<uint8_t>> payload;
                if (!resident_ || copy_outputs_) {
                    payload = acquire_buffer();
                    std::memcpy(payload->data(), h_out_ + (static_cast<size_t>(k) * S_ + s) * out_bytes_, out_bytes_);
                }
                h.lats.push_back(t.emit_tick - t.ingest_tick);
                h.last_output = payload;
                h.has_output = true;
                staged.push_back(Out{src_of(h, t.seq), payload});
            }
        }
        flush_below(h, h.eng->min_inflight_seq(), staged);
        trim_src(h);
        // out_q: bounded drop-oldest (queue.hpp:23-34), drained every iteration
        size_t first = 0;
        if (staged.size() > cap8) {
            first = staged.size() - cap8;
            h.output_drops += first;
        }
        for (size_t i = first; i < staged.size(); ++i) {
            h.sink.push_back(staged[i]);
            h.frames_out += 1;
        }
    }
}

void Pipeline::drain_completed(bool block_all) {
    while (!inflight_.empty()) {
        const auto [k, fp] = inflight_.front();
        cudaEvent_t ev = done_[static_cast<size_t>(k)];
        if (block_all) {
            SDX_CUDA(cudaEventSynchronize(ev));
        } else {
            const cudaError_t q = cudaEventQuery(ev);
            if (q == cudaErrorNotReady) return;
            SDX_CUDA(q);
        }
        process(k, fp);
        inflight_.pop_front();
    }
}

void Pipeline::push(const uint8_t* frames, const int64_t* seq_ids) {
    SDX_CUDA(cudaSetDevice(device_));
    const int k = static_cast<int>(iter_ % K_);
    while (static_cast<int>(inflight_.size()) >= K_) {
        const auto [kk, fp] = inflight_.front();
        SDX_CUDA(cudaEventSynchronize(done_[static_cast<size_t>(kk)]));
        process(kk, fp);
        inflight_.pop_front();
    }
    for (int s = 0; s < S_; ++s) {
        // the device numbers each stream's frames 0,1,2,... (ctl_begin_kernel); the
        // source ids are mapped back when the host orders the sink
        StreamHost& h = st_[static_cast<size_t>(s)];
        h.src_ids.push_back(seq_ids ? seq_ids[s] : frames_pushed_);
    }
    frames_pushed_ += 1;
    if (frames) {
        resident_ = false;
        const uint8_t* src = frames;
        cudaPointerAttributes attr{};
        const bool pinned = cudaPointerGetAttributes(&attr, frames) == cudaSuccess && attr.type == cudaMemoryTypeHost;
        cudaGetLastError();
        if (!pinned) {
            uint8_t* stage = h_in_ + static_cast<size_t>(k) * S_ * D_;
            std::memcpy(stage, frames, static_cast<size_t>(S_) * D_);
            src = stage;
        }
        if (pad_ == D_) {
            SDX_CUDA(cudaMemcpyAsync(d_in_ + static_cast<size_t>(k) * S_ * pad_, src, static_cast<size_t>(S_) * D_,
                                     cudaMemcpyHostToDevice, copy_));
        } else {
            SDX_CUDA(cudaMemcpy2DAsync(d_in_ + static_cast<size_t>(k) * S_ * pad_, static_cast<size_t>(pad_), src,
                                       static_cast<size_t>(D_), static_cast<size_t>(D_), static_cast<size_t>(S_),
                                       cudaMemcpyHostToDevice, copy_));
        }
        SDX_CUDA(cudaEventRecord(h2d_[static_cast<size_t>(k)], copy_));
        // a pinned caller buffer is read in place: return only once the copy is done,
        // so the caller may refill it right away (the copy is not queued behind compute)
        if (pinned) SDX_CUDA(cudaEventSynchronize(h2d_[static_cast<size_t>(k)]));
    } else {
        // resident mode: frames already in ring slot k (upload_resident)
        SDX_CUDA(cudaEventRecord(h2d_[static_cast<size_t>(k)], stream_));
    }
    run_iteration(k, true);
    inflight_.push_back({k, true});
    iter_ += 1;
    drain_completed(false);
}

bool Pipeline::idle() {
    SDX_CUDA(cudaSetDevice(device_));
    drain_completed(false);
    for (const auto& [k, fp] : inflight_)
        if (fp) return false;  // an unprocessed frame may have been ingested
    for (const auto& h : st_)
        if (!h.incomplete && !h.eng->idle()) return false;
    return true;
}

bool Pipeline::tick_idle() {
    if (idle()) return false;
    const int k = static_cast<int>(iter_ % K_);
    while (static_cast<int>(inflight_.size()) >= K_) {
        const auto [kk, fp] = inflight_.front();
        SDX_CUDA(cudaEventSynchronize(done_[static_cast<size_t>(kk)]));
        process(kk, fp);
        inflight_.pop_front();
    }
    run_iteration(k, false);
    inflight_.push_back({k, false});
    iter_ += 1;
    drain_completed(false);
    return true;
}

void Pipeline::upload_resident(const uint8_t* frames, int count) {
    // Stage `count` iterations' frames into the device ring (<= K) so timed
    // pushes run with inputs already in HBM.
    SDX_CUDA(cudaSetDevice(device_));
    if (count > K_) raise(SDX_INVALID_ARGUMENT, "upload_resident: count exceeds ring_depth");
    sync();
    for (int k = 0; k < count; ++k)
        SDX_CUDA(cudaMemcpy2D(d_in_ + static_cast<size_t>(k) * S_ * pad_, static_cast<size_t>(pad_),
                              frames + static_cast<size_t>(k) * S_ * D_, static_cast<size_t>(D_),
                              static_cast<size_t>(D_), static_cast<size_t>(S_), cudaMemcpyHostToDevice));
    resident_count_ = count;
}

void Pipeline::push_resident(bool copy_outputs) {
    if (resident_count_ < 1) raise(SDX_LOGIC_ERROR, "push_resident: no resident frames uploaded");
    // ring slot k holds resident frame (iter % resident_count); keep them by
    // pinning K == resident_count usage
    resident_ = true;
    copy_outputs_ = copy_outputs;
    const int64_t saved = iter_;
    (void)saved;
    if (resident_count_ != K_) raise(SDX_LOGIC_ERROR, "push_resident: upload exactly ring_depth frames");
    push(nullptr);
}

void Pipeline::finish() {
    SDX_CUDA(cudaSetDevice(device_));
    drain_completed(true);
    int rem = 0;
    for (auto& h : st_) {
        if (h.incomplete || h.eng->idle()) continue;
        const auto steps = h.eng->step_indices();
        rem = std::max(rem, n_ - steps.front());
    }
    for (int i = 0; i < rem; ++i) {
        const int k = static_cast<int>(iter_ % K_);
        while (static_cast<int>(inflight_.size()) >= K_) drain_completed(true);
        run_iteration(k, false);
        inflight_.push_back({k, false});
        iter_ += 1;
    }
    drain_completed(true);
    for (auto& h : st_) {
        if (h.incomplete) continue;
        std::vector<Out> staged;
        flush_below(h, INT64_MAX, staged);  // EngineStage::finish (pipeline.cpp:84-86)
        for (auto& o : staged) {
            h.sink.push_back(o);
            h.frames_out += 1;
        }
    }
}

bool Pipeline::pop(int stream, int64_t* seq, void* payload) {
    if (stream < 0 || stream >= S_) raise(SDX_INVALID_ARGUMENT, "pop: stream index out of range");
    auto& h = st_[static_cast<size_t>(stream)];
    if (h.sink.empty()) drain_completed(false);
    if (h.sink.empty()) return false;
    const Out o = h.sink.front();
    h.sink.pop_front();
    *seq = o.seq;
    if (payload && o.payload) std::memcpy(payload, o.payload->data(), o.payload->size());
    return true;
}

const Pipeline::StreamHost& Pipeline::host(int stream) const {
    if (stream < 0 || stream >= S_) raise(SDX_INVALID_ARGUMENT, "pipeline: stream index out of range");
    return st_[static_cast<size_t>(stream)];
}

sdx_report Pipeline::report(int stream) const {
    if (stream < 0 || stream >= S_) raise(SDX_INVALID_ARGUMENT, "report: stream index out of range");
    const auto& h = st_[static_cast<size_t>(stream)];
    sdx_report r{};
    r.frames_in = h.frames_in;
    r.frames_out = h.frames_out;
    r.duplicates = h.duplicates;
    r.stale_skips = h.stale;
    r.input_drops = 0;
    r.output_drops = h.output_drops;
    r.ticks = static_cast<uint64_t>(h.eng->ticks());
    r.denoiser_calls = h.eng->calls;
    r.element_evals = h.eng->evals;
    if (cfg_.engine.ssf_enabled) {
        r.ssf_examined = h.examined;
        r.ssf_skipped = h.skipped;
        r.skip_rate = h.examined == 0 ? 0.0 : static_cast<double>(h.skipped) / static_cast<double>(h.examined);
    }
    if (!h.lats.empty()) {
        int64_t lo = h.lats[0], hi = h.lats[0], sum = 0;
        for (auto l : h.lats) {
            lo = std::min(lo, l);
            hi = std::max(hi, l);
            sum += l;
        }
        r.latency_ticks_min = lo;
        r.latency_ticks_max = hi;
        r.latency_ticks_mean = static_cast<double>(sum) / static_cast<double>(h.lats.size());
    }
    if (r.frames_out > 0) {
        r.mean_frame_time_ms = static_cast<double>(r.ticks) / static_cast<double>(r.frames_out);
        r.throughput_fps = 1000.0 / r.mean_frame_time_ms;
        r.wall_ms = static_cast<double>(r.ticks);
    }
    r.incomplete = h.incomplete ? 1 : 0;
    return r;
}

const std::string& Pipeline::error(int stream) const { return st_[static_cast<size_t>(stream)].error; }

void Pipeline::sync() {
    SDX_CUDA(cudaSetDevice(device_));
    drain_completed(true);
    join_decode();
    SDX_CUDA(cudaStreamSynchronize(stream_));
}

void Pipeline::reset_timer() {
    SDX_CUDA(cudaSetDevice(device_));
    join_decode();
    SDX_CUDA(cudaEventRecord(t0_, stream_));
}

void Pipeline::set_profile(bool on) {
    SDX_CUDA(cudaSetDevice(device_));
    sync();
    if (on && kt_.empty()) {
        kt_.resize(static_cast<size_t>(K_) * kMarks);
        for (auto& ev : kt_) SDX_CUDA(cudaEventCreate(&ev));
    }
    profile_ = on;
    for (auto& t : ktime_) t = 0.0;
    kcount_ = 0;
    launches_ = 0;
}

void Pipeline::stage_times(double* ms, long long* iters) const {
    for (int i = 0; i + 1 < kMarks; ++i) ms[i] = ktime_[i];
    *iters = kcount_;
}

float Pipeline::device_time_ms() {
    SDX_CUDA(cudaSetDevice(device_));
    join_decode();
    SDX_CUDA(cudaEventRecord(t1_, stream_));
    SDX_CUDA(cudaEventSynchronize(t1_));
    float ms = 0.f;
    SDX_CUDA(cudaEventElapsedTime(&ms, t0_, t1_));
    return ms;
}

}  // namespace sdx
