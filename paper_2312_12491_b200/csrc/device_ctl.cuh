// Device-resident control state of the stream-batch engine.
//
// The reference keeps its engine bookkeeping in host objects
// (InFlightFrame list, engine.hpp:18-28; SsfState, ssf.hpp:25-42).  Here the
// same state lives in HBM so the skip/run decision, the ingest and the
// emission are decided on the device and never round-trip to the host before
// the next launch.  The host keeps a mirror (runtime.cu) that it advances
// from the asynchronously-read decision log.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace sdx {

// One in-flight frame slot.  A frame ingested when `ticks` ticks have
// completed lives in slot ticks % n for exactly n ticks (engine.hpp:52-57:
// latency is n tick boundaries), so slots never collide.
struct SlotCtl {
    long long seq;          // -1: empty
    long long ingest_tick;
    int init;               // onetime_negative x0_ref initialised (GuidanceState)
    int entering;           // ingested this iteration: the step kernel forms x_tau0
};

struct StreamCtl {
    long long ticks;        // ticks completed (StreamBatchEngine::ticks_)
    long long iter;         // pipeline iterations run
    long long last_seq;
    int count;              // frames in flight
    int tick_now;           // this iteration runs a tick
    int ingest_slot;        // slot that received a frame this iteration, -1 none
    int emit_slot;          // slot whose frame completes this tick, -1 none
    long long ingest_seq;
    long long emit_seq;
    long long emit_ingest_tick;
    int rows;               // denoiser rows of this tick (evals delta)
    int nonfinite;          // set by the step kernel if the emitted x0_hat is non-finite
    unsigned long long calls, evals;
    // ---- SSF gate state (SsfState) ----
    int has_ref;
    int skip_run;           // consecutive skips (max_skip extension)
    int decision;           // SDX_GATE_* of the frame examined this iteration
    int mti;                // MT19937-64 position
    unsigned long long examined, skipped;
    unsigned long long ref_norm2;        // exact sum of squares of the reference frame
    unsigned long long acc_dot, acc_aa;  // reduction accumulators (reset by the tail)
    unsigned int ticket;                 // last-block detection
    unsigned int pad0;
    double sim;
    int row_base;           // first denoiser row of this stream in the batched call
    int pad1;
    SlotCtl slot[kMaxSteps];
};

// One entry per stream per iteration; copied to a pinned host ring.
struct LogEntry {
    long long seq_in;       // frame pushed this iteration (-1 during finish)
    long long emit_seq;     // -1 none
    long long emit_ingest_tick;
    long long ticks_after;
    double sim;
    int decision;           // SDX_GATE_* (process when SSF is off)
    int ingested;
    int ticked;
    int nonfinite;
    int rows;
    int pad;
};

// Batched-denoiser row descriptor (the `xs/ss/cs` vectors assembled in
// engine.cpp:90-118).  kind: 0 cond row, 1 negative row (cfg), 2 onetime init row.
struct RowDesc {
    int stream;
    int slot;
    int step;
    int kind;
};

}  // namespace sdx
