// sm_100a kernels of the streaming denoise loop's HBM-bound path:
//   * ctl_begin / ctl_end : device-side engine bookkeeping (ingest, row
//     assembly, emission, counters, decision log)        engine.cpp:53-195
//   * step kernel         : fused analytic denoiser + CFG / R-CFG combine +
//     onetime x0_ref init + LCM consistency update + cached re-noise, one
//     pass over every in-flight row                     engine.cpp:78-173,
//                                                       guidance.cpp:19-48,
//                                                       schedule.cpp:60-107,
//                                                       denoiser.cpp:26-43
//   * SSF reduce + tail   : exact integer cosine sums (dp4a), fp64 tail,
//     device MT19937-64 uniform, gate decision          ssf.cpp:8-54, rng.hpp:26-28
//   * commit/encode       : reference-frame update on process + identity encode
//                                                       ssf.cpp:52, codec.cpp:82-86
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "common.cuh"
#include "device_ctl.cuh"
#include "kernels_core.cuh"

namespace sdx {

// ---------------------------------------------------------------------------
// control: begin of an iteration
// ---------------------------------------------------------------------------

// One thread per stream (S <= 1024).  ingest source: host argument (engine
// API) or the SSF decision (pipeline).  Also assigns the batched-denoiser
// rows: per stream, conditional rows for every in-flight frame, then the
// negative rows (cfg) or the one onetime init row (engine.cpp:90-118); the
// streams' row ranges are concatenated with a block scan.
__global__ void ctl_begin_kernel(StreamCtl* __restrict__ ctl, int S, int n, int guidance,
                                 int ingest_mode, long long host_seq, int frame_present,
                                 RowDesc* __restrict__ rows, int* __restrict__ n_rows,
                                 int* __restrict__ slot_row_c, int* __restrict__ slot_row_n) {
    __shared__ int scan[1024];
    const int s = threadIdx.x;
    int my_rows = 0;
    StreamCtl* c = (s < S) ? &ctl[s] : nullptr;
    if (c) {
        int ingest = 0;
        long long seq = -1;
        if (ingest_mode == kIngestHost) {
            ingest = host_seq >= 0;
            seq = host_seq;
        } else if (frame_present) {
            seq = c->iter;  // pipeline seq ids are the frame index (vector_source order)
            ingest = (ingest_mode == kIngestAlways) ? 1 : (c->decision == SDX_GATE_PROCESS);
        }
        c->ingest_seq = frame_present || ingest_mode == kIngestHost ? seq : -1;
        c->ingest_slot = -1;
        if (ingest) {
            const int slot = static_cast<int>(c->ticks % n);
            c->slot[slot].seq = seq;
            c->slot[slot].ingest_tick = c->ticks;
            c->slot[slot].init = 0;
            c->slot[slot].entering = 1;
            c->count += 1;
            c->last_seq = seq;
            c->ingest_slot = slot;
        }
        c->tick_now = c->count > 0;
        c->emit_slot = -1;
        c->emit_seq = -1;
        c->nonfinite = 0;
        c->rows = 0;
        if (c->tick_now) {
            const int es = static_cast<int>((c->ticks + 1) % n);
            if (c->slot[es].seq >= 0 && c->slot[es].ingest_tick == c->ticks - n + 1) {
                c->emit_slot = es;
                c->emit_seq = c->slot[es].seq;
                c->emit_ingest_tick = c->slot[es].ingest_tick;
            }
            const int b = c->count;
            int extra = 0;
            if (guidance == SDX_GUIDANCE_CFG) extra = b;
            if (guidance == SDX_GUIDANCE_ONETIME_NEGATIVE && c->ingest_slot >= 0) extra = 1;
            my_rows = b + extra;
            c->rows = my_rows;
            c->calls += 1;
            c->evals += static_cast<unsigned long long>(my_rows);
        }
    }
    // exclusive scan of rows over streams
    scan[threadIdx.x] = my_rows;
    __syncthreads();
    for (int off = 1; off < blockDim.x; off <<= 1) {
        const int v = threadIdx.x >= off ? scan[threadIdx.x - off] : 0;
        __syncthreads();
        scan[threadIdx.x] += v;
        __syncthreads();
    }
    const int base = scan[threadIdx.x] - my_rows;
    if (c) {
        c->row_base = base;
        if (rows && c->tick_now) {
            // cond rows oldest first (highest step) -> stable, deterministic order
            int r = base;
            const int b = c->count;
            for (int age = n - 1; age >= 0; --age) {
                const int slot = static_cast<int>(((c->ticks - age) % n + n) % n);
                if (c->slot[slot].seq < 0 || c->slot[slot].ingest_tick != c->ticks - age) continue;
                rows[r] = RowDesc{s, slot, age, 0};
                if (slot_row_c) {
                    slot_row_c[s * kMaxSteps + slot] = r;
                    slot_row_n[s * kMaxSteps + slot] = -1;
                }
                ++r;
            }
            if (guidance == SDX_GUIDANCE_CFG) {
                for (int i = 0; i < b; ++i) {
                    RowDesc d = rows[base + i];
                    d.kind = 1;
                    if (slot_row_n) slot_row_n[s * kMaxSteps + d.slot] = r;
                    rows[r++] = d;
                }
            } else if (guidance == SDX_GUIDANCE_ONETIME_NEGATIVE && c->ingest_slot >= 0) {
                if (slot_row_n) slot_row_n[s * kMaxSteps + c->ingest_slot] = r;
                rows[r++] = RowDesc{s, c->ingest_slot, 0, 2};
            }
        }
    }
    if (n_rows && threadIdx.x == blockDim.x - 1) *n_rows = scan[threadIdx.x];
}

// ---------------------------------------------------------------------------
// control: end of an iteration
// ---------------------------------------------------------------------------

__global__ void ctl_end_kernel(StreamCtl* __restrict__ ctl, int S, int n, int guidance,
                               LogEntry* __restrict__ log, int frame_present) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S) return;
    StreamCtl& c = ctl[s];
    LogEntry e;
    e.seq_in = frame_present ? c.iter : -1;
    e.decision = c.decision;
    e.ingested = c.ingest_slot >= 0;
    e.ticked = c.tick_now;
    e.rows = c.rows;
    e.sim = c.sim;
    e.nonfinite = c.nonfinite;
    e.emit_seq = c.emit_seq;
    e.emit_ingest_tick = c.emit_ingest_tick;
    if (c.tick_now) {
        for (int k = 0; k < n; ++k) {
            c.slot[k].entering = 0;
            if (guidance == SDX_GUIDANCE_ONETIME_NEGATIVE && c.slot[k].seq >= 0) c.slot[k].init = 1;
        }
        c.ticks += 1;
        if (c.emit_slot >= 0) {
            c.slot[c.emit_slot].seq = -1;
            c.count -= 1;
        }
    }
    e.ticks_after = c.ticks;
    e.pad = 0;
    if (frame_present) c.iter += 1;
    if (log) log[s] = e;
}

// ---------------------------------------------------------------------------
// SSF
// ---------------------------------------------------------------------------

namespace {
constexpr unsigned long long kMtA = 0xB5026F5AA96619E9ULL;
constexpr unsigned long long kMtUM = 0xFFFFFFFF80000000ULL;
constexpr unsigned long long kMtLM = 0x7FFFFFFFULL;

__device__ __forceinline__ unsigned long long mt_mix(unsigned long long cur, unsigned long long nxt,
                                                     unsigned long long far) {
    const unsigned long long y = (cur & kMtUM) | (nxt & kMtLM);
    return far ^ (y >> 1) ^ ((y & 1ULL) ? kMtA : 0ULL);
}

// Block-cooperative MT19937-64 twist of one 312-word state held in smem.
__device__ void mt_twist_block(unsigned long long* mt) {
    unsigned long long v = 0;
    const int t = threadIdx.x;
    // phase 1: i in [0,156) reads only old words
    for (int base = 0; base < 156; base += blockDim.x) {
        const int i = base + t;
        if (i < 156) v = mt_mix(mt[i], mt[i + 1], mt[i + 156]);
        __syncthreads();
        if (i < 156) mt[i] = v;
        __syncthreads();
    }
    // phase 2: i in [156,311) reads old mt[i], mt[i+1] and new mt[i-156]
    for (int base = 156; base < 311; base += blockDim.x) {
        const int i = base + t;
        if (i < 311) v = mt_mix(mt[i], mt[i + 1], mt[i - 156]);
        __syncthreads();
        if (i < 311) mt[i] = v;
        __syncthreads();
    }
    if (t == 0) mt[311] = mt_mix(mt[311], mt[0], mt[155]);
    __syncthreads();
}

__device__ __forceinline__ unsigned long long mt_temper(unsigned long long x) {
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}
}  // namespace

// grid (blocks_per_stream, S), block 256.  Frame and reference are u8; the
// sums a.b and a.a are exact (dp4a into u32 per 16-byte vector, u64 beyond).
__global__ void __launch_bounds__(256) ssf_reduce_kernel(SsfArgs a) {
    const int s = blockIdx.y;
    StreamCtl& c = a.ctl[s];
    const uint8_t* __restrict__ f = a.frames + static_cast<long long>(s) * a.frame_stride;
    const uint8_t* __restrict__ r = a.ref + static_cast<long long>(s) * a.frame_stride;
    const long long nvec = a.D >> 4;
    const uint4* __restrict__ fv = reinterpret_cast<const uint4*>(f);
    const uint4* __restrict__ rv = reinterpret_cast<const uint4*>(r);
    unsigned long long dot = 0, aa = 0;
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    // 2-way unrolled to keep two 16-byte loads per operand in flight
    for (; i + stride < nvec; i += 2 * stride) {
        const uint4 x0 = __ldcs(fv + i), y0 = __ldcs(rv + i);
        const uint4 x1 = __ldcs(fv + i + stride), y1 = __ldcs(rv + i + stride);
        unsigned int d0 = __dp4a(x0.x, y0.x, 0u);
        d0 = __dp4a(x0.y, y0.y, d0);
        d0 = __dp4a(x0.z, y0.z, d0);
        d0 = __dp4a(x0.w, y0.w, d0);
        unsigned int a0 = __dp4a(x0.x, x0.x, 0u);
        a0 = __dp4a(x0.y, x0.y, a0);
        a0 = __dp4a(x0.z, x0.z, a0);
        a0 = __dp4a(x0.w, x0.w, a0);
        unsigned int d1 = __dp4a(x1.x, y1.x, 0u);
        d1 = __dp4a(x1.y, y1.y, d1);
        d1 = __dp4a(x1.z, y1.z, d1);
        d1 = __dp4a(x1.w, y1.w, d1);
        unsigned int a1 = __dp4a(x1.x, x1.x, 0u);
        a1 = __dp4a(x1.y, x1.y, a1);
        a1 = __dp4a(x1.z, x1.z, a1);
        a1 = __dp4a(x1.w, x1.w, a1);
        dot += static_cast<unsigned long long>(d0) + d1;
        aa += static_cast<unsigned long long>(a0) + a1;
    }
    for (; i < nvec; i += stride) {
        const uint4 x0 = __ldcs(fv + i), y0 = __ldcs(rv + i);
        unsigned int d0 = __dp4a(x0.x, y0.x, 0u);
        d0 = __dp4a(x0.y, y0.y, d0);
        d0 = __dp4a(x0.z, y0.z, d0);
        d0 = __dp4a(x0.w, y0.w, d0);
        unsigned int a0 = __dp4a(x0.x, x0.x, 0u);
        a0 = __dp4a(x0.y, x0.y, a0);
        a0 = __dp4a(x0.z, x0.z, a0);
        a0 = __dp4a(x0.w, x0.w, a0);
        dot += d0;
        aa += a0;
    }
    if (blockIdx.x == 0) {  // tail bytes
        for (long long k = (nvec << 4) + threadIdx.x; k < a.D; k += blockDim.x) {
            dot += static_cast<unsigned long long>(f[k]) * r[k];
            aa += static_cast<unsigned long long>(f[k]) * f[k];
        }
    }
    // warp + block reduction
    for (int o = 16; o > 0; o >>= 1) {
        dot += __shfl_xor_sync(0xffffffffu, dot, o);
        aa += __shfl_xor_sync(0xffffffffu, aa, o);
    }
    __shared__ unsigned long long sd[8], sa[8];
    __shared__ unsigned int last;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        sd[w] = dot;
        sa[w] = aa;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long td = 0, ta = 0;
        for (int k = 0; k < (blockDim.x >> 5); ++k) {
            td += sd[k];
            ta += sa[k];
        }
        atomicAdd(&c.acc_dot, td);
        atomicAdd(&c.acc_aa, ta);
        __threadfence();
        const unsigned int t = atomicAdd(&c.ticket, 1u);
        last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!last) return;

    // ---- tail: one block per stream ----
    __threadfence();
    __shared__ unsigned long long mt[312];
    __shared__ int need_draw;
    __shared__ unsigned long long tot_dot, tot_aa;
    if (threadIdx.x == 0) {
        tot_dot = atomicAdd(&c.acc_dot, 0ULL);
        tot_aa = atomicAdd(&c.acc_aa, 0ULL);
        need_draw = c.has_ref;
    }
    __syncthreads();
    const unsigned long long dot_t = tot_dot, aa_t = tot_aa;
    unsigned long long* gstate = a.mt_state + static_cast<long long>(s) * 312;
    if (need_draw && c.mti >= 312) {
        for (int k = threadIdx.x; k < 312; k += blockDim.x) mt[k] = gstate[k];
        __syncthreads();
        mt_twist_block(mt);
        for (int k = threadIdx.x; k < 312; k += blockDim.x) gstate[k] = mt[k];
        __syncthreads();
        if (threadIdx.x == 0) c.mti = 0;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        c.examined += 1;
        c.acc_dot = 0;
        c.acc_aa = 0;
        c.ticket = 0;
        if (!c.has_ref) {  // first frame: nothing to compare against (ssf.cpp:41-44)
            c.has_ref = 1;
            c.ref_norm2 = aa_t;
            c.skip_run = 0;
            c.decision = SDX_GATE_PROCESS;
            c.sim = __longlong_as_double(0x7ff8000000000000LL);
        } else {
            // cosine_similarity (ssf.cpp:8-20): a = frame, b = reference
            const double na = __dsqrt_rn(static_cast<double>(aa_t));
            const double nb = __dsqrt_rn(static_cast<double>(c.ref_norm2));
            double sim = 0.0;
            if (!(na < 1e-12 || nb < 1e-12)) sim = __ddiv_rn(static_cast<double>(dot_t), __dmul_rn(na, nb));
            // skip_probability (ssf.cpp:26-32)
            double p = __ddiv_rn(__dsub_rn(sim, a.eta), __dsub_rn(1.0, a.eta));
            p = p <= 0.0 ? 0.0 : (p >= 1.0 ? 1.0 : p);
            // Rng::uniform (rng.hpp:26-28) on the device MT19937-64 stream
            const unsigned long long x = mt_temper(gstate[c.mti]);
            c.mti += 1;
            const double u = static_cast<double>(x >> 11) * 0x1.0p-53;
            int skip = u < p;
            if (skip && a.max_skip > 0 && c.skip_run >= a.max_skip) skip = 0;
            c.sim = sim;
            if (skip) {
                c.skipped += 1;
                c.skip_run += 1;
                c.decision = SDX_GATE_SKIP;
            } else {
                c.skip_run = 0;
                c.ref_norm2 = aa_t;
                c.decision = SDX_GATE_PROCESS;
            }
        }
        if (a.dec_out) a.dec_out[0] = c.decision;
        if (a.sim_out) a.sim_out[0] = c.sim;
    }
}

// Reference-frame update on process (ref := frame) fused with the identity
// encode of the ingested frame into its latent slot (u8 -> f32).
__global__ void __launch_bounds__(256) commit_encode_kernel(CommitArgs a) {
    const int s = blockIdx.y;
    const StreamCtl& c = a.ctl[s];
    const bool commit = a.ref != nullptr && c.decision == SDX_GATE_PROCESS;
    const int slot = c.ingest_slot;
    const bool encode = a.x0 != nullptr && slot >= 0;
    if (!commit && !encode) return;
    const uint8_t* __restrict__ f = a.frames + static_cast<long long>(s) * a.frame_stride;
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    if (commit) {
        const long long nvec = a.D >> 4;
        const uint4* fv = reinterpret_cast<const uint4*>(f);
        uint8_t* rs = a.ref + static_cast<long long>(s) * a.frame_stride;
        uint4* rv = reinterpret_cast<uint4*>(rs);
        for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < nvec; i += stride)
            rv[i] = fv[i];
        for (long long k = (nvec << 4) + static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; k < a.D;
             k += stride)
            rs[k] = f[k];
    }
    if (encode) {
        float* x0 = a.x0 + (static_cast<long long>(s) * a.n + slot) * a.d;
        for (long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; k < a.d; k += stride)
            x0[k] = static_cast<float>(f[k]);
    }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------

void launch_ctl_begin(StreamCtl* ctl, int S, int n, int guidance, int ingest_mode, long long host_seq,
                      int frame_present, RowDesc* rows, int* n_rows, int* slot_row_c, int* slot_row_n,
                      cudaStream_t st) {
    int threads = 32;
    while (threads < S) threads <<= 1;
    ctl_begin_kernel<<<1, threads, 0, st>>>(ctl, S, n, guidance, ingest_mode, host_seq, frame_present, rows,
                                            n_rows, slot_row_c, slot_row_n);
    SDX_LAUNCH_CHECK();
}

void launch_ctl_end(StreamCtl* ctl, int S, int n, int guidance, LogEntry* log, int frame_present,
                    cudaStream_t st) {
    ctl_end_kernel<<<(S + 127) / 128, 128, 0, st>>>(ctl, S, n, guidance, log, frame_present);
    SDX_LAUNCH_CHECK();
}

void launch_ssf_reduce(const SsfArgs& a, int S, cudaStream_t st) {
    const long long nvec = a.D >> 4;
    long long per_stream = (2LL * kSmCount * 2 + S - 1) / S;  // ~4 waves of 256-thread blocks over the chip
    const long long useful = (nvec + 255) / 256;
    if (per_stream > useful) per_stream = useful;
    if (per_stream < 1) per_stream = 1;
    dim3 grid(static_cast<unsigned>(per_stream), S);
    ssf_reduce_kernel<<<grid, 256, 0, st>>>(a);
    SDX_LAUNCH_CHECK();
}

void launch_commit_encode(const CommitArgs& a, int S, cudaStream_t st) {
    const long long work = a.D > a.d ? a.D / 16 : a.d;
    long long per_stream = (work + 255) / 256;
    const long long cap = (4LL * kSmCount + S - 1) / S;
    if (per_stream > cap) per_stream = cap;
    if (per_stream < 1) per_stream = 1;
    dim3 grid(static_cast<unsigned>(per_stream), S);
    commit_encode_kernel<<<grid, 256, 0, st>>>(a);
    SDX_LAUNCH_CHECK();
}

}  // namespace sdx
