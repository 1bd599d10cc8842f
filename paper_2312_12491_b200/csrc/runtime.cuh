// Host runtime of the B200 streaming denoise loop: device-state owners for
// the engine, the SSF gate and the multi-stream pipeline, plus the host
// mirror of the reference's engine/pipeline bookkeeping.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <deque>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "common.cuh"
#include "device_ctl.cuh"
#include "kernels_core.cuh"
#include "pipeline_kernels.cuh"
#include "taesd.cuh"
#include "unet.cuh"

namespace sdx {

// Host mirror of StreamBatchEngine's frame bookkeeping (engine.cpp:53-211):
// which frames are in flight at which step.  It never touches latents; the
// device holds those.  Used for argument validation with the reference's
// exception semantics and to order the pipeline sink without reading data.
class EngineMirror {
  public:
    struct Frame {
        int64_t seq;
        int step;
        int64_t ingest_tick;
    };
    struct TickOut {
        bool emitted = false;
        int64_t seq = -1, ingest_tick = 0, emit_tick = 0;
        uint64_t rows = 0;
    };

    EngineMirror(int n, int guidance) : n_(n), guidance_(guidance) {}

    void check_ingest(int64_t seq) const;
    void ingest(int64_t seq);
    TickOut tick();
    bool idle() const { return inflight_.empty(); }
    int64_t ticks() const { return ticks_; }
    int inflight() const { return static_cast<int>(inflight_.size()); }
    std::vector<int> step_indices() const;
    int64_t min_inflight_seq() const;  // INT64_MAX when idle
    uint64_t calls = 0, evals = 0;
    bool pending_ingest() const { return pending_; }
    int64_t pending_seq() const { return pending_seq_; }

  private:
    int n_, guidance_;
    std::vector<Frame> inflight_;
    int64_t ticks_ = 0, last_seq_ = -1;
    bool pending_ = false;
    int64_t pending_seq_ = -1;
};

// Device-resident state of S streams sharing one batched denoiser call.
struct DeviceEngine {
    int S = 0, n = 0;
    long long d = 0;
    int guidance = 0;
    double gamma = 1.4, delta = 1.0;
    bool per_slot_cond = false;
    StepScalars* tbl = nullptr;
    float *x_cur = nullptr, *x0 = nullptr, *x0ref = nullptr, *eps_cached = nullptr;
    float *cond = nullptr, *neg = nullptr, *emitted = nullptr;
    StreamCtl* ctl = nullptr;
    RowDesc* rows = nullptr;
    int* n_rows = nullptr;
    int *slot_row_c = nullptr, *slot_row_n = nullptr;
    LogEntry* log = nullptr;  // [S]
    float* xfa_eps = nullptr;     // cross-frame attention buffers (null when off)
    double* xfa_dots = nullptr;

    void init(int S_, int n_, long long d_, int guidance_, double gamma_, double delta_,
              const std::vector<StepScalars>& table, bool per_slot_cond_, bool cross_frame = false);
    void release();
    StepArgs step_args() const;
};

std::vector<StepScalars> make_step_table(const sdx_step* steps, int n, int lcm_mode, double data_variance);

class Engine {
  public:
    Engine(const sdx_config& cfg, const sdx_step* steps, int n, const double* eps_cached,
           const double* neg, int device);
    ~Engine();
    void ingest(int64_t seq, const double* x0, const double* cond);
    sdx_tick_result tick(double* x0_hat);
    EngineMirror& mirror() { return mirror_; }
    float last_tick_ms() const { return last_ms_; }
    void reset_counters() { mirror_.calls = 0; mirror_.evals = 0; }

  private:
    sdx_config cfg_;
    int device_;
    cudaStream_t stream_ = nullptr;
    cudaEvent_t ev0_ = nullptr, ev1_ = nullptr;
    DeviceEngine dev_;
    EngineMirror mirror_;
    float* h_stage_ = nullptr;  // pinned, 2 x d floats
    LogEntry* h_log_ = nullptr;
    std::vector<std::vector<float>> slot_cond_;  // last condition uploaded per slot
    float last_ms_ = 0.f;
    bool timed_ = false;
};

class Ssf {
  public:
    Ssf(double eta, uint64_t seed, int max_skip, int64_t frame_bytes, int device);
    ~Ssf();
    void gate(const uint8_t* frames, int nframes, int* decisions, double* sims);
    uint64_t examined() const { return examined_; }
    uint64_t skipped() const { return skipped_; }

  private:
    double eta_;
    int max_skip_;
    int64_t D_;
    int device_;
    cudaStream_t stream_ = nullptr;
    uint8_t *d_frames_ = nullptr, *d_ref_ = nullptr;
    StreamCtl* ctl_ = nullptr;
    unsigned long long* mt_ = nullptr;
    int* dec_ = nullptr;
    double* sims_ = nullptr;
    int batch_ = 0;
    uint64_t examined_ = 0, skipped_ = 0;
};

// Initial MT19937-64 state words for seed (std::mt19937_64 seeding).
void mt_seed_words(uint64_t seed, unsigned long long* out312);

class Pipeline {
  public:
    Pipeline(const sdx_pipeline_config& cfg, const sdx_step* steps, const double* eps_cached,
             const double* cond, const double* neg, int device);
    ~Pipeline();
    // seq_ids: the S source sequence ids of this push's frames (NULL: the frame index)
    void push(const uint8_t* frames, const int64_t* seq_ids = nullptr);
    // One frame-less iteration (a tick with no ingest) when some stream may still
    // have frames in flight; returns false, without launching, when every stream is
    // known to be idle.  The threaded live loop calls it when no input is waiting
    // (pipeline.cpp:235-245 ticks whenever the engine is not idle).
    bool tick_idle();
    bool idle();
    void upload_resident(const uint8_t* frames, int count);
    void push_resident(bool copy_outputs);
    void finish();
    const std::string& error(int stream) const;
    bool pop(int stream, int64_t* seq, void* payload);
    sdx_report report(int stream) const;
    const std::vector<int>& decisions(int stream) const { return host(stream).decisions; }
    const std::vector<sdx_trace_entry>& trace(int stream) const { return host(stream).trace; }
    void sync();
    void reset_timer();
    float device_time_ms();
    // Per-stage device time (CUDA events on the pipeline stream between the
    // stages of every iteration), accumulated while profiling:
    // [0] SSF, [1] control + commit, [2] encode, [3] denoiser (UNet), [4] step +
    // control end, [5] decode.
    static constexpr int kMarks = 7;
    void set_profile(bool on);
    void stage_times(double* ms, long long* iters) const;
    long long launches() const { return launches_; }
    double unet_flops_per_row() const { return unet_ ? unet_->flops_per_row() : 0.0; }
    double taesd_flops() const { return taesd_ ? taesd_->enc_flops_per_image() + taesd_->dec_flops_per_image() : 0.0; }

  private:
    struct Out {
        int64_t seq;
        std::shared_ptr<std::vector<uint8_t>> payload;
    };
    struct StreamHost;
    const StreamHost& host(int stream) const;
    struct StreamHost {
        std::unique_ptr<EngineMirror> eng;
        std::deque<int64_t> pending_skips;
        std::shared_ptr<std::vector<uint8_t>> last_output;  // null in the no-copy benchmark mode
        bool has_output = false;  // EngineStage::last_output_ engaged (pipeline.cpp:106)
        // source sequence ids by device frame index (the device numbers the frames of a
        // stream 0,1,2,...); src_base is the device index of src_ids.front()
        std::deque<int64_t> src_ids;
        int64_t src_base = 0;
        int64_t last_src = INT64_MIN;  // last ingested source id (engine.cpp:59-60)
        std::deque<Out> sink;
        std::vector<int64_t> lats;
        std::vector<int> decisions;
        std::vector<sdx_trace_entry> trace;  // one per tick (TickLogEntry), first 2^20 kept
        uint64_t frames_in = 0, frames_out = 0, duplicates = 0, stale = 0, output_drops = 0;
        uint64_t examined = 0, skipped = 0;
        bool incomplete = false;
        std::string error;
    };
    void launch_iteration(int k, bool frame_present);
    void launch_decode(int k, cudaStream_t s);
    void launch_encode(int k, cudaStream_t s);
    void run_encode(int k);
    void run_iteration(int k, bool frame_present);
    void join_decode();
    void process(int k, bool frame_present);
    std::vector<cudaGraphExec_t> graphs_;     // [ring slot][output-copy variant][frame present]
    std::vector<long long> graph_launches_;
    void drain_completed(bool block_all);
    void flush_below(StreamHost& h, int64_t limit, std::vector<Out>& staged);
    static int64_t src_of(const StreamHost& h, int64_t dev_seq);
    static void trim_src(StreamHost& h);
    std::shared_ptr<std::vector<uint8_t>> acquire_buffer();
    std::vector<std::shared_ptr<std::vector<uint8_t>>> pool_;

    sdx_pipeline_config cfg_;
    int S_, n_, K_;
    int64_t D_;
    long long d_;
    size_t out_bytes_;
    int device_;
    cudaStream_t stream_ = nullptr, copy_ = nullptr;
    DeviceEngine dev_;
    int64_t pad_ = 0;
    bool resident_ = false, copy_outputs_ = true;
    int resident_count_ = 0;
    std::vector<cudaEvent_t> h2d_;
    uint8_t *d_in_ = nullptr, *d_ref_ = nullptr;
    unsigned long long* mt_ = nullptr;
    uint8_t *h_in_ = nullptr, *h_out_ = nullptr;
    LogEntry* h_log_ = nullptr;
    std::vector<cudaEvent_t> done_;
    std::deque<std::pair<int, bool>> inflight_;  // (ring slot, frame_present)
    int64_t iter_ = 0;
    int64_t frames_pushed_ = 0;  // frame-present iterations (the device frame index)
    std::vector<StreamHost> st_;
    cudaEvent_t t0_ = nullptr, t1_ = nullptr;
    bool profile_ = false;
    std::vector<cudaEvent_t> kt_;  // [K][kMarks]
    double ktime_[kMarks - 1] = {};
    long long kcount_ = 0;
    long long launches_ = 0;
    // UNet backend / TAESD codec
    std::unique_ptr<UNet> unet_;
    std::unique_ptr<TAESD> taesd_;
    int unet_rmax_ = 0;
    int* lists_buf_ = nullptr;
    CodecLists lists_{};
    uint8_t* d_out_ = nullptr;  // [K][S][frame_bytes] decoded frames (TAESD)
    // Decode overlap (TAESD codec): iteration t's decode runs on dec_stream_
    // while iteration t+1's SSF / encode / UNet / step run on stream_.  The
    // main graph stages the emitted latents and codec lists per ring slot; the
    // decode graph copies them into the decoder's fixed inputs, decodes, and
    // reads the frames back; done_[k] is recorded after it.
    bool overlap_ = false;
    cudaStream_t dec_stream_ = nullptr;
    std::vector<cudaEvent_t> main_done_;  // [K] main part of slot k finished
    cudaEvent_t dec_join_ = nullptr;
    float* stage_lat_ = nullptr;   // [K][S][d] emitted latents
    int* stage_lists_ = nullptr;   // [K][4S+2] codec lists
    float* dec_in_ = nullptr;      // [S][d] decoder input
    int* dec_lists_ = nullptr;     // [4S+2]
    std::vector<cudaGraphExec_t> dec_graphs_;  // [ring slot][output-copy variant]
    std::vector<long long> dec_graph_launches_;
    // Encode ahead (TAESD codec): the frames of ring slot k are encoded on enc_stream_
    // as soon as they are in HBM, all S of them, into enc_stage_ (indexed like the
    // ring, slot * S + stream) while the previous iterations run; the iteration then
    // only gathers its ingesting streams' latents into x0 (it waits enc_done_[k]).
    bool enc_overlap_ = false;
    cudaStream_t enc_stream_ = nullptr;
    std::vector<cudaEvent_t> enc_done_;  // [K]
    float* enc_stage_ = nullptr;          // [K*S][d]
    int* enc_lists_ = nullptr;            // [2S+1] encoder's src / dst / count
    int* spec_lists_ = nullptr;           // [K][2S+1] per-slot identity lists
    std::vector<cudaGraphExec_t> enc_graphs_;  // [ring slot]
    long long enc_graph_launches_ = 0;
};

}  // namespace sdx
