// C++ drop-in parity test: the reference's own test cases (test_stream_batch.cpp,
// test_ssf.cpp, test_runtime.cpp) written against the B200 drop-in headers
// (include/stagger_b200/stagger/*.hpp, namespace stagger, device execution) and
// checked against the CPU oracle (oracle/stagger_oracle.h, pinned bit-for-bit to
// the reference build).  Run by tests/test_dropin_gpu.py on a B200.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <map>
#include <random>
#include <string>
#include <vector>

#include "stagger/engine.hpp"
#include "stagger/pipeline.hpp"
#include "stagger/ssf.hpp"
#include "stagger_oracle.h"

using namespace stagger;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        ++g_checks;                                                              \
        if (!(cond)) {                                                           \
            ++g_fail;                                                            \
            std::fprintf(stderr, "%s:%d CHECK failed: %s\n", __FILE__, __LINE__, #cond); \
        }                                                                        \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                   \
    do {                                           \
        bool thrown = false;                       \
        try {                                      \
            expr;                                  \
        } catch (const T&) {                       \
            thrown = true;                         \
        } catch (...) {                            \
        }                                          \
        CHECK(thrown);                             \
    } while (0)

static double max_abs_diff(const Latent& a, const Latent& b) {
    double m = 0.0;
    for (size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a[i] - b[i]));
    return m;
}

static orc_cfg ocfg(const EngineConfig& c) {
    orc_cfg o{};
    o.n_steps = c.n_steps;
    o.guidance_mode = static_cast<int>(c.guidance_mode);
    o.gamma = c.gamma;
    o.delta = c.delta;
    o.ssf_enabled = c.ssf_enabled;
    o.eta = c.eta;
    o.seed = c.seed;
    o.d_latent = c.d_latent;
    o.t_grid = c.t_grid;
    o.entry_strength = c.entry_strength;
    o.data_variance = c.data_variance;
    o.lcm_mode = c.lcm_mode == "boundary_approx" ? 1 : 0;
    o.codec = 0;
    o.queue_capacity = c.queue_capacity;
    return o;
}

// test_stream_batch.cpp:250-282 — engine output equals the sequential oracle
static void stream_batch_oracle_equivalence() {
    for (int n : {1, 2, 4, 10}) {
        for (auto mode : {GuidanceMode::none, GuidanceMode::self_negative, GuidanceMode::cfg,
                          GuidanceMode::onetime_negative}) {
            EngineConfig cfg;
            cfg.n_steps = n;
            cfg.guidance_mode = mode;
            Rng crng(derive_seed(0, kStreamCondition));
            const Condition cond{"c", sample_gaussian(crng, 8)};
            Rng nrng(derive_seed(0, kStreamCondition + 1));
            const Latent neg = sample_gaussian(nrng, 8);
            if (mode == GuidanceMode::cfg || mode == GuidanceMode::onetime_negative) cfg.negative_condition = neg;
            auto backend = make_backend(cfg);
            StreamBatchEngine engine(cfg, build_precompute(cfg, {cond}), backend);
            Rng rng(13);
            std::vector<Latent> inputs;
            for (int f = 0; f < 25; ++f) inputs.push_back(sample_gaussian(rng, 8));
            std::map<std::int64_t, Latent> out;
            std::int64_t seq = 0;
            for (const auto& x0 : inputs) {
                engine.ingest(seq++, x0, cond);
                if (auto r = engine.tick(); r.emitted) {
                    CHECK(r.denoiser_calls == 1);
                    CHECK(r.emitted->emit_tick - r.emitted->ingest_tick == n);
                    out[r.emitted->seq_id] = r.emitted->x0_hat;
                }
            }
            while (!engine.idle())
                if (auto r = engine.tick(); r.emitted) out[r.emitted->seq_id] = r.emitted->x0_hat;
            CHECK(out.size() == inputs.size());
            const orc_cfg oc = ocfg(cfg);
            double worst = 0.0;
            for (std::int64_t f = 0; f < std::int64_t(inputs.size()); ++f) {
                Latent ref(8);
                CHECK(orc_sequential(&oc, cond.embedding.data(),
                                     cfg.negative_condition.empty() ? nullptr : cfg.negative_condition.data(),
                                     inputs[size_t(f)].data(), ref.data()) == 0);
                worst = std::max(worst, max_abs_diff(out.at(f), ref));
            }
            CHECK(worst <= 1e-3);
            // per-frame call contracts {n, 2n, n, n+1} (test_stream_batch.cpp:224-248)
            const std::uint64_t per = mode == GuidanceMode::cfg ? 2u * n
                                      : mode == GuidanceMode::onetime_negative ? n + 1u : std::uint64_t(n);
            CHECK(backend->counters().element_evals == per * inputs.size());
            CHECK(engine.log().size() == size_t(engine.ticks_completed()));
        }
    }
}

// test_stream_batch.cpp:284-308 — cross-frame attention changes outputs but not the contract;
// the drop-in engine (device, fp32) also matches the C restatement with it on
static void stream_batch_cross_frame() {
    const int n = 4;
    auto run = [&](bool mixed, std::map<std::int64_t, Latent>* out, orc_engine** oe) {
        EngineConfig cfg;
        cfg.n_steps = n;
        cfg.cross_frame_attention = mixed;
        Rng crng(derive_seed(0, kStreamCondition));
        const Condition cond{"c", sample_gaussian(crng, 8)};
        StreamBatchEngine engine(cfg, build_precompute(cfg, {cond}), make_backend(cfg));
        orc_cfg oc = ocfg(cfg);
        oc.cross_frame_attention = mixed ? 1 : 0;
        CHECK(orc_engine_create(&oc, cond.embedding.data(), nullptr, oe) == 0);
        Rng rng(14);
        std::int64_t seq = 0;
        double worst = 0.0;
        auto tick = [&]() {
            const auto r = engine.tick();
            std::int64_t es = -1, it = 0, et = 0;
            std::uint64_t c = 0, ev = 0;
            Latent ref(8);
            CHECK(orc_engine_tick(*oe, &es, ref.data(), &it, &et, &c, &ev) == 0);
            CHECK(bool(r.emitted) == (es >= 0));
            if (r.emitted) {
                CHECK(r.emitted->seq_id == es && r.emitted->emit_tick - r.emitted->ingest_tick == n);
                worst = std::max(worst, max_abs_diff(r.emitted->x0_hat, ref));
                (*out)[r.emitted->seq_id] = r.emitted->x0_hat;
            }
        };
        for (int f = 0; f < 12; ++f) {
            const Latent x0 = sample_gaussian(rng, 8);
            engine.ingest(seq, x0, cond);
            CHECK(orc_engine_ingest(*oe, seq, x0.data()) == 0);
            ++seq;
            tick();
        }
        while (!engine.idle()) tick();
        CHECK(worst <= 1e-3);
        orc_engine_destroy(*oe);
    };
    std::map<std::int64_t, Latent> base, attn;
    orc_engine* oe = nullptr;
    run(false, &base, &oe);
    run(true, &attn, &oe);
    CHECK(base.size() == attn.size() && base.size() == 12);
    double diff = 0.0;
    for (const auto& [seq, v] : base) diff = std::max(diff, max_abs_diff(v, attn.at(seq)));
    CHECK(diff > 1e-9);  // documented non-equivalence when the mix is on
}

// test_stream_batch.cpp:62-97 — error contract
static void stream_batch_errors() {
    EngineConfig cfg;
    cfg.n_steps = 4;
    const Condition cond{"c", Latent(8, 0.5)};
    StreamBatchEngine engine(cfg, build_precompute(cfg, {cond}), make_backend(cfg));
    CHECK_THROWS_AS(engine.tick(), std::logic_error);
    engine.ingest(5, Latent(8, 1.0), cond);
    CHECK_THROWS_AS(engine.ingest(6, Latent(8, 1.0), cond), std::logic_error);
    engine.tick();
    CHECK_THROWS_AS(engine.ingest(5, Latent(8, 1.0), cond), std::invalid_argument);
    CHECK(engine.step_indices() == std::vector<int>{1});
    CHECK(engine.min_inflight_seq() == std::optional<std::int64_t>(5));
    EngineConfig bad = cfg;
    bad.eta = 1.0;
    CHECK_THROWS_AS(validated(bad), std::invalid_argument);
}

static std::vector<Frame> u8_frames(int kind, int d, std::uint64_t seed, int n) {
    std::mt19937_64 g(seed);
    std::vector<Frame> out;
    Latent base(static_cast<size_t>(d));
    for (auto& x : base) x = double(g() % 256);
    for (int i = 0; i < n; ++i) {
        Frame f;
        f.seq_id = i;
        if (kind == 0) {
            f.payload = base;
        } else if (kind == 1) {
            f.payload.resize(size_t(d));
            for (auto& x : f.payload) x = double(g() % 256);
        } else {
            if (i % 13 == 12)
                for (auto& x : base) x = double(g() % 256);
            f.payload = base;
            for (int k = 0; k < d / 40; ++k) f.payload[g() % size_t(d)] = double(g() % 256);
        }
        out.push_back(f);
    }
    return out;
}

// test_runtime.cpp:169-211 / 228-242 — pipeline contracts against the oracle pipeline
static void runtime_pipeline() {
    for (int kind : {0, 1, 2}) {
        for (int n : {1, 4}) {
            EngineConfig cfg;
            cfg.n_steps = n;
            cfg.ssf_enabled = true;
            cfg.eta = 0.98;
            cfg.seed = 5 + kind;
            cfg.d_latent = 1024;
            const auto frames = u8_frames(kind, 1024, 77 + kind, 60);
            std::vector<Frame> got;
            const auto rep = run_pipeline(cfg, vector_source(frames), [&](const Frame& f) { got.push_back(f); });
            CHECK(!rep.incomplete);
            // oracle
            std::vector<double> flat;
            for (const auto& f : frames) flat.insert(flat.end(), f.payload.begin(), f.payload.end());
            std::vector<std::int64_t> oseq(200);
            std::vector<double> opay(200 * 1024);
            int n_out = 0;
            orc_report orep{};
            const orc_cfg oc = ocfg(cfg);
            CHECK(orc_run_pipeline(&oc, nullptr, nullptr, flat.data(), 60, 1024, 0, oseq.data(), opay.data(), 200,
                                   &n_out, nullptr, &orep) == 0);
            CHECK(int(got.size()) == n_out);
            double worst = 0.0;
            for (int i = 0; i < n_out && i < int(got.size()); ++i) {
                CHECK(got[size_t(i)].seq_id == oseq[size_t(i)]);
                Latent ref(opay.begin() + i * 1024, opay.begin() + (i + 1) * 1024);
                worst = std::max(worst, max_abs_diff(got[size_t(i)].payload, ref));
            }
            CHECK(worst <= 1e-3);
            CHECK(rep.ssf_skipped == orep.ssf_skipped && rep.duplicates == orep.duplicates);
            CHECK(rep.element_evals == orep.element_evals && rep.ticks == orep.ticks);
            CHECK(rep.latency_ticks_max == orep.latency_ticks_max);
            if (kind == 0) CHECK(rep.ssf_skipped == 59 && rep.duplicates == 59);
            // the sink carries the SOURCE's seq ids (pipeline.cpp:176), here 1000 + 3 i:
            // same frames, same order, ids mapped through the source
            std::vector<Frame> sparse = frames;
            for (size_t i = 0; i < sparse.size(); ++i) sparse[i].seq_id = 1000 + 3 * std::int64_t(i);
            std::vector<Frame> got2;
            const auto rep2 = run_pipeline(cfg, vector_source(sparse), [&](const Frame& f) { got2.push_back(f); });
            CHECK(!rep2.incomplete && got2.size() == got.size());
            bool mapped = got2.size() == got.size();
            for (size_t i = 0; mapped && i < got2.size(); ++i)
                mapped = got2[i].seq_id == 1000 + 3 * got[i].seq_id && got2[i].payload == got[i].payload;
            CHECK(mapped);
        }
    }
    // a processed frame whose source id does not increase -> ingest error, incomplete
    // (engine.cpp:59-60 "ingest: seq ids must strictly increase")
    {
        EngineConfig cfg;
        cfg.n_steps = 2;
        cfg.d_latent = 256;
        auto frames = u8_frames(1, 256, 5, 6);
        frames[4].seq_id = 2;
        const auto rep = run_pipeline(cfg, vector_source(frames), [](const Frame&) {});
        CHECK(rep.incomplete && rep.error.find("strictly increase") != std::string::npos);
    }
    // byte-identical deterministic reports (test_runtime.cpp:228-242)
    EngineConfig cfg;
    cfg.n_steps = 4;
    cfg.ssf_enabled = true;
    cfg.seed = 31;
    cfg.d_latent = 512;
    const auto frames = u8_frames(2, 512, 3, 80);
    const auto a = report_to_json(run_pipeline(cfg, vector_source(frames), [](const Frame&) {}));
    const auto b = report_to_json(run_pipeline(cfg, vector_source(frames), [](const Frame&) {}));
    CHECK(a == b);
    CHECK(a.find("\"schema_version\": 1") != std::string::npos);
    // stage failure -> partial report flagged incomplete (test_runtime.cpp:303-316)
    std::int64_t seq = 0;
    EngineConfig c2;
    c2.n_steps = 2;
    auto source = [&seq]() -> std::optional<Frame> {
        if (seq >= 8) return std::nullopt;
        Frame f;
        f.seq_id = seq++;
        f.payload = seq < 5 ? Latent(8, 5.0) : Latent(3, 5.0);
        return f;
    };
    const auto r = run_pipeline(c2, source, [](const Frame&) {});
    CHECK(r.incomplete && !r.error.empty());
}

// test_runtime.cpp:145-167 — tick trace: one JSON line per tick; test_runtime.cpp:263-301 —
// threaded mode (three host threads, bounded queues): strict FIFO delivers every frame in
// order with no drops; freshest-wins keeps sink ids strictly increasing and never drops at
// the output
static void runtime_trace_and_threaded() {
    {
        EngineConfig cfg;
        cfg.n_steps = 2;
        cfg.d_latent = 256;
        const auto frames = u8_frames(1, 256, 9, 10);
        PipelineOptions opts;
        opts.trace_path = "/tmp/stagger_b200_trace_test.jsonl";
        const auto rep = run_pipeline(cfg, vector_source(frames), [](const Frame&) {}, opts);
        CHECK(!rep.incomplete);
        std::ifstream in(opts.trace_path);
        CHECK(in.good());
        std::string line;
        std::uint64_t lines = 0;
        std::int64_t last_tick = 0;
        bool keys = true;
        while (std::getline(in, line)) {
            keys = keys && line.find("\"tick\":") != std::string::npos && line.find("\"element_evals\":") != std::string::npos &&
                   line.find("\"ingested\":") != std::string::npos && line.find("\"emitted\":") != std::string::npos;
            const std::int64_t t = std::atoll(line.c_str() + 8);
            keys = keys && t == last_tick + 1;
            last_tick = t;
            ++lines;
        }
        CHECK(keys);
        CHECK(lines == rep.ticks && lines > 0);
        std::remove(opts.trace_path.c_str());
    }
    {
        EngineConfig cfg;
        cfg.n_steps = 4;
        cfg.seed = 41;
        cfg.d_latent = 512;
        cfg.queue_capacity = 256;  // strict FIFO timing-style run: no drops
        PipelineOptions opts;
        opts.threaded = true;
        opts.strict_fifo = true;
        std::vector<Frame> got;
        const auto frames = u8_frames(2, 512, 41, 200);
        const auto rep = run_pipeline(cfg, vector_source(frames), [&](const Frame& f) { got.push_back(f); }, opts);
        CHECK(!rep.incomplete);
        CHECK(rep.mode == "threaded");
        CHECK(got.size() == 200);
        CHECK(rep.input_drops == 0);
        bool inc = true;
        for (size_t i = 1; i < got.size(); ++i) inc = inc && got[i].seq_id > got[i - 1].seq_id;
        CHECK(inc);
        CHECK(rep.wall_ms > 0.0);
        // same frames deterministically: identical outputs (the device pipeline is the same)
        std::vector<Frame> ref;
        run_pipeline(cfg, vector_source(frames), [&](const Frame& f) { ref.push_back(f); });
        bool same = ref.size() == got.size();
        for (size_t i = 0; same && i < got.size(); ++i)
            same = got[i].seq_id == ref[i].seq_id && got[i].payload == ref[i].payload;
        CHECK(same);
    }
    {
        EngineConfig cfg;
        cfg.n_steps = 2;
        cfg.seed = 43;
        cfg.d_latent = 4096;
        cfg.queue_capacity = 2;
        PipelineOptions opts;
        opts.threaded = true;
        opts.strict_fifo = false;  // freshest-wins
        std::vector<Frame> got;
        auto frames = u8_frames(2, 4096, 43, 300);
        for (size_t i = 0; i < frames.size(); ++i) frames[i].seq_id = 7 + 5 * std::int64_t(i);
        const auto rep = run_pipeline(cfg, vector_source(frames), [&](const Frame& f) { got.push_back(f); }, opts);
        CHECK(!rep.incomplete);
        CHECK(rep.output_drops == 0);
        CHECK(rep.frames_in == 300);
        CHECK(rep.frames_out + rep.input_drops >= 300 - 2 * 4);
        CHECK(!got.empty());
        bool inc = true, known = true;
        for (size_t i = 1; i < got.size(); ++i) inc = inc && got[i].seq_id > got[i - 1].seq_id;
        // every sink id is one of the source's ids (input drops leave gaps, never renumber)
        for (const auto& f : got) known = known && f.seq_id >= 7 && (f.seq_id - 7) % 5 == 0 && f.seq_id < 7 + 5 * 300;
        CHECK(inc);
        CHECK(known);
        // the last frame is never dropped by freshest-wins: it reaches the sink
        CHECK(got.back().seq_id == 7 + 5 * 299);
    }
}

// test_ssf.cpp:97-156 — device gate
static void ssf_gate() {
    SsfState state(0.98, Rng(2));
    Frame f;
    f.payload = {1.0, 200.0, 5.0, 2.0};
    CHECK(state.gate(f) == GateDecision::process);
    int skips = 0;
    for (int i = 0; i < 300; ++i) skips += state.gate(f) == GateDecision::skip;
    CHECK(skips == 300 && state.examined() == 301 && state.skipped() == 300);
    // identical seeds -> identical decisions, equal to the oracle gate
    const auto frames = u8_frames(2, 2048, 9, 200);
    SsfState a(0.98, Rng(8));
    orc_ssf* o = nullptr;
    orc_ssf_create(0.98, 8, 0, &o);
    for (const auto& fr : frames) {
        const int od = orc_ssf_gate(o, fr.payload.data(), int(fr.payload.size()));
        CHECK((a.gate(fr) == GateDecision::skip) == (od == 1));
    }
    orc_ssf_destroy(o);
    CHECK_THROWS_AS(SsfState(1.0, Rng(1)), std::invalid_argument);
    Frame bad;
    bad.payload = {0.5, 1.0};
    SsfState s2(0.9, Rng(3));
    CHECK_THROWS_AS(s2.gate(bad), std::invalid_argument);
}

int main() {
    stream_batch_oracle_equivalence();
    stream_batch_cross_frame();
    stream_batch_errors();
    runtime_pipeline();
    runtime_trace_and_threaded();
    ssf_gate();
    std::printf("%d checks, %d failed\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
