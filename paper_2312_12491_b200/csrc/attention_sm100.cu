// Flash attention (head_dim 64) on tcgen05 / TMEM / TMA for the UNet's
// self- and cross-attention (the Stream Batch denoiser's attention blocks).
//
// One CTA = 128 queries of one (image row, head).  Warp roles:
//   warp 0      TMA producer: Q once, K/V blocks of 128 keys into a 2-deep ring
//   warp 1      TMEM alloc + MMA issuer: S = Q K^T (M128 N128 K64) into one of two
//               TMEM S buffers; O_part = P V (M128 N64 K128, V as an MN-major
//               operand) into a TMEM O_part buffer
//   warps 2..5  softmax: one query row per thread (TMEM lane), online max/sum
//               in fp32 (exp2), P written to smem as bf16 in the 128-byte
//               swizzled K-major layout, O accumulated in registers
// Keys past kv_len and queries past q_len are masked (cross-attention pads 77
// keys to 128; the 8x8 level has 64 tokens per image).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "attention_sm100.cuh"
#include "common.cuh"
#include "sm100.cuh"

namespace sdx {

using namespace sm100;

namespace {

constexpr int BQ = 128, BKV = 128, HD = 64;
constexpr uint32_t TILE_BYTES = 128 * 64 * 2;  // one 128-row x 64-col bf16 tile (16 KB)
// P buffers per q tile: with 2, the softmax of block j+1 writes P while PV(j) still
// reads the other buffer (it waits only for PV(j-1)), but the K/V ring must shrink to
// 2 to fit in shared memory; measured on B200 (tools/attn_probe.py, 4 x 4096 x 5
// heads): PB=2/KVS=2 210.7 us vs PB=1/KVS=4 190.2 us, so one buffer.
constexpr int PB = 1;
constexpr int KVS = PB == 2 ? 2 : 4;  // K/V ring depth
// How far QK^T may run ahead of PV per tile (S_t(j+1) also needs s_free: S_t(j) read
// into registers).  2 lets S(j+1) overlap the softmax of block j; measured equal to 1
// (190.7 vs 190.2 us, tools/attn_probe.py): the softmax warps, not the MMA order, set
// the pace.
constexpr int kSAhead = 1;
constexpr int KVS_TS = 5;
constexpr bool kStaggerTiles = true;
// attn_ts_kernel<POLY>: one exp2 pair in POLY (pairs 1, 1 + POLY, ...) on the FMA-pipe
// polynomial, 0 = all on the MUFU; SDX_ATTN_POLY picks the instantiation (default kPolyDefault)
constexpr int kPolyDefault = 3;  // K/V ring of the TMEM-P kernel (no P buffers in smem)

// Blocking wait with a suspend-time hint: the warp sleeps in the barrier unit instead of
// re-polling, so waiting warps leave the issue slots of their SM sub-partition to the
// softmax warps sharing it (the slowest of a tile's four softmax warps sets its pace).
__device__ __forceinline__ void wait_bar(uint64_t* bar, uint32_t phase) {
    const uint32_t a = smem_u32(bar);
    uint32_t done = 0;
    const long long t0 = clock64();
    while (true) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 1000000;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(a), "r"(phase)
            : "memory");
        if (done) return;
        if (clock64() - t0 > (1LL << 33)) {
            printf("sdx attention: mbarrier watchdog (block %d,%d,%d thread %d)\n", blockIdx.x, blockIdx.y,
                   blockIdx.z, threadIdx.x);
            asm volatile("trap;");
        }
    }
}

// non-blocking probe of an mbarrier phase
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t phase) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    return done != 0;
}

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
        "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
        "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
        "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15]))
        : "memory");
}

// Two 128-query tiles per CTA (256 queries of one image/head) share every K/V
// block.  10 warps: 0 TMA, 1 MMA, 2..5 softmax of tile 0, 6..9 softmax of tile 1.
// TMEM per tile: S [128 cols] + O [64 cols]; O accumulates across KV blocks in
// TMEM and is rescaled only when a row max grows by more than 2^8 (lazy
// rescaling), so P = exp2(s - m_used) stays <= 256 and never overflows.
__global__ void __launch_bounds__(320, 1)
    attn_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tkv, AttnArgs a) {
    // Work unit -> (image, head, first q tile, tiles).  Pair units (two 128-query tiles sharing
    // every K/V block) cover the full waves; a remainder that would leave most SMs idle in a
    // last wave runs as single-tile units: CTAs >= a.pair_base of the same launch (the block
    // scheduler issues them after the pair CTAs, so they fill the tail).
    const int npairs = (a.q_len + 2 * BQ - 1) / (2 * BQ);
    const bool single = static_cast<int>(blockIdx.x) >= a.pair_base;
    const int lin = single ? static_cast<int>(blockIdx.x) - a.pair_base : static_cast<int>(blockIdx.x);
    const int plin = single ? a.pair_base + lin / 2 : lin;  // linear pair index, q pair fastest
    const int qp = plin % npairs;
    const int head = (plin / npairs) % a.heads;
    const int img = plin / (npairs * a.heads);
    const int q_first = qp * 2 * BQ + (single ? (lin & 1) * BQ : 0);  // first query of this unit
    if (threadIdx.x == 0) pdl_launch();
    const bool has1 = !single && q_first + BQ < a.q_len;  // second tile holds live queries

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;                       // 2 x 16 KB
    uint8_t* sK = sQ + 2 * TILE_BYTES;        // KVS x 16 KB
    uint8_t* sV = sK + KVS * TILE_BYTES;      // KVS x 16 KB
    uint8_t* sP = sV + KVS * TILE_BYTES;      // [2 tiles][PB] x 32 KB (two 64-key atoms each)
    uint64_t* bars = reinterpret_cast<uint64_t*>(sP + 4 * PB * TILE_BYTES);
    uint64_t* q_full = bars + 0;
    uint64_t* kv_full = bars + 1;          // [KVS]
    uint64_t* kv_empty = kv_full + KVS;    // [KVS]
    uint64_t* s_full = kv_empty + KVS;     // [2] per tile
    uint64_t* p_full = s_full + 2;         // [2 tiles][PB]: P buffer written
    uint64_t* pv_done = p_full + 2 * PB;   // [2 tiles][PB]: PV that read the P buffer done
    uint64_t* s_free = pv_done + 2 * PB;   // [2] per tile: S read out of TMEM (next S may overwrite it)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_free + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nkv = (a.kv_len + BKV - 1) / BKV;
    const int q_row0 = img * a.q_rows_per_img + q_first;
    const int prompt = a.kv_index ? a.kv_index[img] : img;
    const int kv_row0 = prompt * a.kv_rows_per_img;

    if (threadIdx.x == 0) {
        tma_prefetch(&tq);
        tma_prefetch(&tkv);
        mbar_init(q_full, 1);
        for (int i = 0; i < KVS; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&s_free[i], 4);  // one arrival per softmax warp
        }
        for (int i = 0; i < 2 * PB; ++i) {
            mbar_init(&p_full[i], 128);
            mbar_init(&pv_done[i], 1);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // TMEM columns: tile t: S at t*192, O at t*192 + 128
    pdl_wait();  // setup above overlaps the previous kernel (PDL)
    const bool live = !(a.rows_dev && img >= *a.rows_dev);

    if (!live) {
    } else if (warp == 0) {
        if (lane == 0) {
            mbar_expect_tx(q_full, (has1 ? 2 : 1) * TILE_BYTES);
            tma_load_2d(sQ, &tq, q_full, a.q_col0 + head * HD, q_row0);
            if (has1) tma_load_2d(sQ + TILE_BYTES, &tq, q_full, a.q_col0 + head * HD, q_row0 + BQ);
            for (int j = 0; j < nkv; ++j) {
                const int b = j % KVS;
                wait_bar(&kv_empty[b], ((j / KVS) & 1) ^ 1);
                mbar_expect_tx(&kv_full[b], 2 * TILE_BYTES);
                tma_load_2d(sK + b * TILE_BYTES, &tkv, &kv_full[b], a.k_col0 + head * HD, kv_row0 + j * BKV);
                tma_load_2d(sV + b * TILE_BYTES, &tkv, &kv_full[b], a.v_col0 + head * HD, kv_row0 + j * BKV);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc_s = idesc_bf16(128, 128);
            constexpr uint32_t idesc_o = idesc_bf16(128, 64, 0, 1);  // B (= V) MN-major
            const int ntile = has1 ? 2 : 1;
            wait_bar(q_full, 0);
            tc_fence_after();
            auto issue_s = [&](int t, int j) {
                const uint64_t dq = desc_kmajor_sw128(smem_u32(sQ + t * TILE_BYTES));
                const uint64_t dk = desc_kmajor_sw128(smem_u32(sK + (j % KVS) * TILE_BYTES));
#pragma unroll
                for (int k = 0; k < ((a.xmode == 1 || a.xmode == 6 || a.xmode == 7) ? 0 : HD / 16); ++k)
                    umma_f16(tmem + t * 192, dq + 2 * k, dk + 2 * k, idesc_s, k != 0);
                umma_commit(&s_full[t]);
            };
            auto issue_pv = [&](int t, int j) {
                const uint32_t pbase = smem_u32(sP + (t * PB + j % PB) * 2 * TILE_BYTES);
                const uint32_t vbase = smem_u32(sV + (j % KVS) * TILE_BYTES);
#pragma unroll
                for (int k = 0; k < ((a.xmode == 1 || a.xmode == 5 || a.xmode == 7) ? 0 : BKV / 16); ++k) {
                    const uint64_t dp = desc_kmajor_sw128(pbase + (k >> 2) * TILE_BYTES) + 2 * (k & 3);
                    const uint64_t dv = desc_mnmajor_sw128(vbase + k * 2048, 0);
                    umma_f16(tmem + t * 192 + 128, dp, dv, idesc_o, (j > 0 || k != 0) ? 1u : 0u);
                }
                umma_commit(&pv_done[t * PB + j % PB]);
            };
            wait_bar(&kv_full[0], 0);
            tc_fence_after();
            for (int t = 0; t < ntile; ++t) issue_s(t, 0);
            // Event-driven issue: per tile, S_t(j) goes out once K_j has landed and the softmax
            // has read S_t(j-1) out of TMEM (s_free), PV_t(j) once P_t(j) is in smem (p_full).
            // The barriers are polled without blocking, so one tile's softmax never stalls
            // the other tile's MMAs; K/V slot j is released after both tiles' PV(j).
            int ns[2] = {1, ntile > 1 ? 1 : nkv};   // next S block per tile
            int np[2] = {0, ntile > 1 ? 0 : nkv};   // next PV block per tile
            int released = 0;                        // K/V blocks released so far
            const long long t0 = clock64();
            while (released < nkv) {
                bool progress = false;
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    if (ns[t] < nkv && ns[t] - np[t] <= kSAhead && mbar_test(&kv_full[ns[t] % KVS], (ns[t] / KVS) & 1) &&
                        mbar_test(&s_free[t], (ns[t] - 1) & 1)) {
                        tc_fence_after();
                        issue_s(t, ns[t]);
                        ++ns[t];
                        progress = true;
                    }
                    if (np[t] < ns[t] && mbar_test(&p_full[t * PB + np[t] % PB], (np[t] / PB) & 1)) {
                        tc_fence_after();
                        issue_pv(t, np[t]);
                        ++np[t];
                        progress = true;
                    }
                }
                const int done = np[0] < np[1] ? np[0] : np[1];
                while (released < done) umma_commit(&kv_empty[released++ % KVS]);
                if (!progress && clock64() - t0 > (1LL << 34)) {
                    printf("sdx attention: MMA issue watchdog (block %d)\n", blockIdx.x);
                    asm volatile("trap;");
                }
            }
        }
        __syncwarp();
    } else {
        const int t = (warp - 2) >> 2;  // q tile of this softmax warpgroup
        const int q = warp & 3;
        const int r = q * 32 + lane;
        if (t == 0 || has1) {
            const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
            const uint32_t s_addr = tmem + lane_off + t * 192;
            const uint32_t o_addr = s_addr + 128;
            const float sl2 = a.scale * 1.4426950408889634f;
            float m_used = -INFINITY, l = 0.f;
            for (int j = 0; j < nkv; ++j) {
                uint8_t* prow = sP + (t * PB + j % PB) * 2 * TILE_BYTES;
                wait_bar(&s_full[t], j & 1);
                tc_fence_after();
                uint32_t sr[128];
                if (a.xmode == 7) {  // probe: synchronisation skeleton only (no S read)
#pragma unroll
                    for (int i = 0; i < 128; ++i) sr[i] = 0u;
                } else {
                    tmem_ld32_nowait(s_addr + 0, sr);
                    tmem_ld32_nowait(s_addr + 32, sr + 32);
                    tmem_ld32_nowait(s_addr + 64, sr + 64);
                    tmem_ld32_nowait(s_addr + 96, sr + 96);
                    tmem_wait_ld();
                }
                // S is in registers: the next QK^T may overwrite the TMEM S buffer
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&s_free[t]);
                const int kv_valid = a.kv_len - j * BKV;
                if (kv_valid < BKV) {  // partial last block: masked keys read as -inf
#pragma unroll
                    for (int i = 0; i < BKV; ++i)
                        if (i >= kv_valid) sr[i] = 0xff800000u;
                }
                // row max: 8 independent chains, then a tree
                float mx8[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) mx8[k] = __uint_as_float(sr[k]);
#pragma unroll
                for (int i = 8; i < BKV; i += 8) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) mx8[k] = fmaxf(mx8[k], __uint_as_float(sr[i + k]));
                }
                const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                       fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
                const float m_row = mx * sl2;
                // PV(j - PB) finished reading this P buffer
                if (j >= PB) wait_bar(&pv_done[t * PB + j % PB], ((j - PB) / PB) & 1);
                if (m_row > m_used + 8.f) {
                    // lazy rescale: new reference max for this row
                    const float m_new = m_row;
                    const float corr = ex2(m_used - m_new);  // m_used = -inf -> 0
                    if (j > 0) {
                        // O_t is final through block j-1 once PV(j-1) is done
                        if (PB > 1) wait_bar(&pv_done[t * PB + (j - 1) % PB], ((j - 1) / PB) & 1);
                        tc_fence_after();
#pragma unroll
                        for (int c = 0; c < HD; c += 16) {
                            float v[16];
                            tmem_ld16(o_addr + c, v);
#pragma unroll
                            for (int i = 0; i < 16; ++i) v[i] *= corr;
                            tmem_st16(o_addr + c, v);
                        }
                    }
                    l *= corr;
                    m_used = m_new;
                }
                // p = exp2(s * scale_log2 - m_used) (exp2(-inf) = 0 for masked keys), 8 partial sums
                float sum8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                const float nm = -m_used;
#pragma unroll
                for (int c = 0; c < ((a.xmode == 2 || a.xmode == 7) ? 0 : BKV); c += 16) {
                    uint32_t pk[8];
#pragma unroll
                    for (int i = 0; i < 16; i += 2) {
                        const float p0 = ex2(fmaf(__uint_as_float(sr[c + i]), sl2, nm));
                        const float p1 = ex2(fmaf(__uint_as_float(sr[c + i + 1]), sl2, nm));
                        sum8[i >> 1] += p0 + p1;
                        pk[i / 2] = pack_bf16(p0, p1);
                    }
                    uint8_t* atom = prow + (c >> 6) * TILE_BYTES + r * 128;
                    const int ch0 = ((c & 63) >> 3);
                    *reinterpret_cast<uint4*>(atom + (((ch0) ^ (r & 7)) << 4)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                    *reinterpret_cast<uint4*>(atom + (((ch0 + 1) ^ (r & 7)) << 4)) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
                }
                l += ((sum8[0] + sum8[1]) + (sum8[2] + sum8[3])) + ((sum8[4] + sum8[5]) + (sum8[6] + sum8[7]));
                fence_async_smem();
                tc_fence_before();
                mbar_arrive(&p_full[t * PB + j % PB]);
            }
            wait_bar(&pv_done[t * PB + (nkv - 1) % PB], ((nkv - 1) / PB) & 1);
            tc_fence_after();
            const int qi = q_first + t * BQ + r;
            float o[HD];
#pragma unroll
            for (int c = 0; c < HD; c += 16) tmem_ld16(o_addr + c, o + c);
            if (qi < a.q_len) {
                const float inv = 1.f / l;
                __nv_bfloat16* op = a.out + static_cast<long long>(q_row0 + t * BQ + r) * a.ld_out + a.out_col0 + head * HD;
#pragma unroll
                for (int c = 0; c < HD; c += 8) {
                    uint4 w;
                    w.x = pack_bf16(o[c] * inv, o[c + 1] * inv);
                    w.y = pack_bf16(o[c + 2] * inv, o[c + 3] * inv);
                    w.z = pack_bf16(o[c + 4] * inv, o[c + 5] * inv);
                    w.w = pack_bf16(o[c + 6] * inv, o[c + 7] * inv);
                    *reinterpret_cast<uint4*>(op + c) = w;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ---- P in TMEM (FA4-style TS-MMA) -------------------------------------------------------
// The MMA warp runs converged and one lane, elected inside the asm, issues each
// tcgen05 op: with warp-uniform operands ptxas emits a plain UTCHMMA instead of an
// ELECT / R2UR.BROADCAST loop around it, which costs ~50 cycles per MMA
// (tools/ubench/ubench_mma.cu: an M128 N64 TS-MMA issues every 51 cycles from a
// divergent lane, every 32 = the tensor-pipe floor from the converged warp).
__device__ __forceinline__ void tmem_st16u(uint32_t taddr, const uint32_t* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float fmax3f(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
// (d0, d1) = (a0, a1) * s + (c, c) on the packed fp32 pipe (FFMA2)
__device__ __forceinline__ void ffma2_bc(float& d0, float& d1, float a0, float a1, float s, float c) {
    asm("{\n\t.reg .b64 va, vs, vc, vd;\n\t"
        "mov.b64 va, {%2, %3};\n\t"
        "mov.b64 vs, {%4, %4};\n\t"
        "mov.b64 vc, {%5, %5};\n\t"
        "fma.rn.ftz.f32x2 vd, va, vs, vc;\n\t"
        "mov.b64 {%0, %1}, vd;\n\t}"
        : "=f"(d0), "=f"(d1)
        : "f"(a0), "f"(a1), "f"(s), "f"(c));
}
// (d0, d1) += (a0, a1) (FADD2)
__device__ __forceinline__ void fadd2_acc(float& d0, float& d1, float a0, float a1) {
    asm("{\n\t.reg .b64 va, vd;\n\t"
        "mov.b64 va, {%2, %3};\n\t"
        "mov.b64 vd, {%0, %1};\n\t"
        "add.rn.ftz.f32x2 vd, vd, va;\n\t"
        "mov.b64 {%0, %1}, vd;\n\t}"
        : "+f"(d0), "+f"(d1)
        : "f"(a0), "f"(a1));
}

// exp2 of a pair on the FMA pipe (FA4's emulation): 2^x = 2^round(x) * 2^f, f in [-0.5, 0.5],
// 2^f by a degree-3 polynomial (relative error 7.7e-5, below the bf16 rounding of P), the
// integer part added to the exponent bits.  round(x) comes from the 1.5 * 2^23 trick, whose
// low mantissa bits hold it.  x is clamped at -126 (exp2(-inf) for masked keys -> ~1e-38).
__device__ __forceinline__ void ex2_poly2(float& p0, float& p1, float x0, float x1) {
    x0 = fmaxf(x0, -126.f);
    x1 = fmaxf(x1, -126.f);
    uint32_t t0, t1;
    asm("{\n\t.reg .b64 vx, vm, vt, vxi, vf, vp, vc3, vc2, vc1, vc0;\n\t"
        "mov.b64 vx, {%4, %5};\n\t"
        "mov.b64 vm, {%6, %6};\n\t"
        "add.rn.ftz.f32x2 vt, vx, vm;\n\t"
        "sub.rn.ftz.f32x2 vxi, vt, vm;\n\t"
        "sub.rn.ftz.f32x2 vf, vx, vxi;\n\t"
        "mov.b64 vc3, {%7, %7};\n\t"
        "mov.b64 vc2, {%8, %8};\n\t"
        "mov.b64 vc1, {%9, %9};\n\t"
        "mov.b64 vc0, {%10, %10};\n\t"
        "fma.rn.ftz.f32x2 vp, vf, vc3, vc2;\n\t"
        "fma.rn.ftz.f32x2 vp, vp, vf, vc1;\n\t"
        "fma.rn.ftz.f32x2 vp, vp, vf, vc0;\n\t"
        "mov.b64 {%0, %1}, vp;\n\t"
        "mov.b64 {%2, %3}, vt;\n\t}"
        : "=f"(p0), "=f"(p1), "=r"(t0), "=r"(t1)
        : "f"(x0), "f"(x1), "f"(12582912.f), "f"(0.05508877f), "f"(0.24260466f), "f"(0.69327628f), "f"(0.9999289f));
    p0 = __uint_as_float(__float_as_uint(p0) + (t0 << 23));
    p1 = __uint_as_float(__float_as_uint(p1) + (t1 << 23));
}

// Two 128-query tiles per CTA, as attn_kernel, with P in tensor memory.  Per tile t:
// S_t (fp32, 128 columns), O_t (64), P_t (bf16 pairs, 64) are TMEM-resident, so
//   * S_t(j+1) = Q_t K(j+1)^T is issued as soon as the softmax has read S_t(j) into
//     registers (s_free) and overlaps the exponentials of block j;
//   * the softmax writes P_t(j) with tcgen05.st and PV_t(j) reads it as the A operand
//     (TS-MMA): no P in shared memory, no proxy fence; the only wait before writing
//     P_t(j) is PV_t(j-1) having read P_t(j-1) (pv_done), long done by then.
// Q and K/V come in by TMA (S = Q K^T is an SS-MMA: M128 N128 runs at the tensor-pipe
// floor).  TMEM: S_t at 128 t, O_t at 256 + 64 t, P_t at 384 + 64 t.
// 11 warps: 0 TMA, 1 + t the MMA issuer of tile t (a tcgen05.mma issue blocks about as
// long as the MMA runs, so one issuer per tile keeps one tile's S(j+1) from queueing
// behind the other tile's PV), 3..6 softmax of tile 0, 7..10 softmax of tile 1.
template <int POLY>
__global__ void __launch_bounds__(352, 1)
    attn_ts_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tkv, AttnArgs a) {
    const int npairs = (a.q_len + 2 * BQ - 1) / (2 * BQ);
    const bool single = static_cast<int>(blockIdx.x) >= a.pair_base;
    const int lin = single ? static_cast<int>(blockIdx.x) - a.pair_base : static_cast<int>(blockIdx.x);
    const int plin = single ? a.pair_base + lin / 2 : lin;
    const int qp = plin % npairs;
    const int head = (plin / npairs) % a.heads;
    const int img = plin / (npairs * a.heads);
    const int q_first = qp * 2 * BQ + (single ? (lin & 1) * BQ : 0);
    if (threadIdx.x == 0) pdl_launch();
    const bool has1 = !single && q_first + BQ < a.q_len;

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;                        // 2 x 16 KB
    uint8_t* sK = sQ + 2 * TILE_BYTES;         // KVS_TS x 16 KB
    uint8_t* sV = sK + KVS_TS * TILE_BYTES;    // KVS_TS x 16 KB
    uint64_t* bars = reinterpret_cast<uint64_t*>(sV + KVS_TS * TILE_BYTES);
    uint64_t* q_full = bars + 0;
    uint64_t* kv_full = bars + 1;            // [KVS_TS]
    uint64_t* kv_empty = kv_full + KVS_TS;   // [KVS_TS]
    uint64_t* s_full = kv_empty + KVS_TS;    // [2] S_t(j) in TMEM
    uint64_t* s_free = s_full + 2;           // [2] S_t(j) read by the softmax (S_t(j+1) may overwrite)
    uint64_t* p_full = s_free + 2;           // [2] P_t(j) in TMEM
    uint64_t* pv_done = p_full + 2;          // [2] PV_t(j) complete (P_t free, O_t final through j)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nkv = (a.kv_len + BKV - 1) / BKV;
    const int q_row0 = img * a.q_rows_per_img + q_first;
    const int prompt = a.kv_index ? a.kv_index[img] : img;
    const int kv_row0 = prompt * a.kv_rows_per_img;

    if (threadIdx.x == 0) {
        tma_prefetch(&tq);
        tma_prefetch(&tkv);
        mbar_init(q_full, 1);
        for (int i = 0; i < KVS_TS; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], has1 ? 2 : 1);  // released by each tile's MMA issuer
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&s_free[i], 4);  // one arrival per softmax warp
            mbar_init(&p_full[i], 4);
            mbar_init(&pv_done[i], 1);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();
    const bool live = !(a.rows_dev && img >= *a.rows_dev);
    long long* dbg = (a.dbg && blockIdx.x == 0 && lane == 0) ? a.dbg + warp * 64 * 8 : nullptr;
    if (dbg && warp == 0) a.dbg[7] = clock64();

    if (!live) {
    } else if (warp == 0) {
        if (lane == 0) {
            mbar_expect_tx(q_full, (has1 ? 2 : 1) * TILE_BYTES);
            tma_load_2d(sQ, &tq, q_full, a.q_col0 + head * HD, q_row0);
            if (has1) tma_load_2d(sQ + TILE_BYTES, &tq, q_full, a.q_col0 + head * HD, q_row0 + BQ);
            for (int j = 0; j < nkv; ++j) {
                const int b = j % KVS_TS;
                wait_bar(&kv_empty[b], ((j / KVS_TS) & 1) ^ 1);
                mbar_expect_tx(&kv_full[b], 2 * TILE_BYTES);
                tma_load_2d(sK + b * TILE_BYTES, &tkv, &kv_full[b], a.k_col0 + head * HD, kv_row0 + j * BKV);
                tma_load_2d(sV + b * TILE_BYTES, &tkv, &kv_full[b], a.v_col0 + head * HD, kv_row0 + j * BKV);
            }
        }
    } else if (warp == 1 || warp == 2) {
        // MMA issuer of tile t: converged warp, every issue / commit through one elected lane
        const int t = warp - 1;
        if (t == 0 || has1) {
            constexpr uint32_t idesc_s = idesc_bf16(128, 128);
            constexpr uint32_t idesc_o = idesc_bf16(128, 64, 0, 1);  // B (= V) MN-major
            const uint64_t dq = desc_kmajor_sw128(smem_u32(sQ + t * TILE_BYTES));
            auto issue_s = [&](int j) {
                const uint64_t dk = desc_kmajor_sw128(smem_u32(sK + (j % KVS_TS) * TILE_BYTES));
#pragma unroll
                for (int k = 0; k < HD / 16; ++k) umma_f16_el(tmem + t * 128, dq + 2 * k, dk + 2 * k, idesc_s, k != 0);
                umma_commit_el(&s_full[t]);
            };
            wait_bar(q_full, 0);
            wait_bar(&kv_full[0], 0);
            tc_fence_after();
            issue_s(0);
            for (int j = 0; j < nkv; ++j) {
                if (j + 1 < nkv) {
                    // S_t(j+1) once the softmax holds S_t(j) in registers and K(j+1) has landed
                    wait_bar(&s_free[t], j & 1);
                    wait_bar(&kv_full[(j + 1) % KVS_TS], ((j + 1) / KVS_TS) & 1);
                    tc_fence_after();
                    issue_s(j + 1);
                    if (dbg && j < 64) dbg[j * 8 + 1] = clock64();
                }
                wait_bar(&p_full[t], j & 1);
                if (dbg && j < 64) dbg[j * 8 + 0] = clock64();
                tc_fence_after();
                const uint32_t vbase = smem_u32(sV + (j % KVS_TS) * TILE_BYTES);
#pragma unroll
                for (int k = 0; k < BKV / 16; ++k)  // P: 16 keys = 8 packed columns per MMA
                    umma_ts_el(tmem + 256 + t * 64, tmem + 384 + t * 64 + 8 * k,
                               desc_mnmajor_sw128(vbase + k * 2048, 0), idesc_o, (j > 0 || k != 0) ? 1u : 0u);
                umma_commit_el(&pv_done[t]);
                umma_commit_el(&kv_empty[j % KVS_TS]);
                if (dbg && j < 64) dbg[j * 8 + 2] = clock64();
            }
        }
    } else {
        const int t = (warp - 3) >> 2;  // q tile of this softmax warpgroup
        const int q = warp & 3;         // TMEM lane quarter this warp may access
        const int r = q * 32 + lane;
        if (t == 0 || has1) {
            const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
            const uint32_t s_addr = tmem + lane_off + t * 128;
            const uint32_t o_addr = tmem + lane_off + 256 + t * 64;
            const uint32_t p_addr = tmem + lane_off + 384 + t * 64;
            const float sl2 = a.scale * 1.4426950408889634f;
            float m_used = -INFINITY, l0 = 0.f, l1 = 0.f;
            for (int j = 0; j < nkv; ++j) {
                long long* dj = (dbg && j < 64) ? dbg + j * 8 : nullptr;
                if (dj) dj[0] = clock64();
                wait_bar(&s_full[t], j & 1);
                if (dj) dj[1] = clock64();
                tc_fence_after();
                uint32_t sr[128];
                tmem_ld32_nowait(s_addr + 0, sr);
                tmem_ld32_nowait(s_addr + 32, sr + 32);
                tmem_ld32_nowait(s_addr + 64, sr + 64);
                tmem_ld32_nowait(s_addr + 96, sr + 96);
                tmem_wait_ld32(sr);
                tmem_wait_ld32(sr + 32);
                tmem_wait_ld32(sr + 64);
                tmem_wait_ld32(sr + 96);
                // S_t(j) is in registers: S_t(j+1) may overwrite the TMEM columns
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&s_free[t]);
                if (dj) dj[2] = clock64();
                const int kv_valid = a.kv_len - j * BKV;
                if (kv_valid < BKV) {  // partial last block: masked keys read as -inf
#pragma unroll
                    for (int i = 0; i < BKV; ++i)
                        if (i >= kv_valid) sr[i] = 0xff800000u;
                }
                // row max: 4 chains of 3-input max, then a tree
                float mx4[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) mx4[k] = fmaxf(__uint_as_float(sr[k]), __uint_as_float(sr[4 + k]));
#pragma unroll
                for (int i = 8; i < BKV; i += 8) {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        mx4[k] = fmax3f(mx4[k], __uint_as_float(sr[i + k]), __uint_as_float(sr[i + 4 + k]));
                }
                const float m_row = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * sl2;
                // PV_t(j-1) done: P_t is free and O_t final through block j-1
                if (j > 0) wait_bar(&pv_done[t], (j - 1) & 1);
                tc_fence_after();
                // lazy rescale (warp-uniform: the TMEM accesses are warp-collective): move the
                // reference max only when some row's max grew by more than 2^8
                if (__any_sync(0xffffffffu, m_row > m_used + 8.f)) {
                    const float m_new = fmaxf(m_used, m_row);
                    const float corr = ex2(m_used - m_new);  // m_used = -inf -> 0
                    if (j > 0) {
#pragma unroll
                        for (int c = 0; c < HD; c += 16) {
                            float v[16];
                            tmem_ld16(o_addr + c, v);
#pragma unroll
                            for (int i = 0; i < 16; ++i) v[i] *= corr;
                            tmem_st16(o_addr + c, v);
                        }
                    }
                    l0 *= corr;
                    l1 *= corr;
                    m_used = m_new;
                }
                // stagger the tiles once: tile 1 starts its first exponentials when tile 0 has
                // finished its own, so one tile's exponentials overlap the other's S load,
                // max and PV wait instead of both tiles contending for the MUFU at once
                if (t == 1 && j == 0 && kStaggerTiles) wait_bar(&p_full[0], 0);
                if (dj) dj[3] = clock64();
                // P = exp2(s * scale_log2 - m_used) as packed bf16 into TMEM (exp2(-inf) = 0)
                const float nm = -m_used;
#pragma unroll
                for (int c = 0; c < BKV; c += 32) {
                    uint32_t pk[16];
#pragma unroll
                    for (int i = 0; i < 32; i += 2) {
                        float x0, x1, p0, p1;
                        ffma2_bc(x0, x1, __uint_as_float(sr[c + i]), __uint_as_float(sr[c + i + 1]), sl2, nm);
                        if (POLY > 0 && (i / 2) % POLY == 1) {
                            ex2_poly2(p0, p1, x0, x1);  // FMA pipe: unloads the MUFU (16 ex2 / clk / SM)
                        } else {
                            p0 = ex2(x0);
                            p1 = ex2(x1);
                        }
                        fadd2_acc(l0, l1, p0, p1);
                        pk[i / 2] = pack_bf16(p0, p1);
                    }
                    tmem_st16u(p_addr + (c >> 1), pk);
                }
                tmem_wait_st();
                if (dj) dj[4] = clock64();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&p_full[t]);
            }
            wait_bar(&pv_done[t], (nkv - 1) & 1);
            tc_fence_after();
            const int qi = q_first + t * BQ + r;
            float o[HD];
#pragma unroll
            for (int c = 0; c < HD; c += 16) tmem_ld16(o_addr + c, o + c);
            if (qi < a.q_len) {
                const float inv = 1.f / (l0 + l1);
                __nv_bfloat16* op = a.out + static_cast<long long>(q_row0 + t * BQ + r) * a.ld_out + a.out_col0 + head * HD;
#pragma unroll
                for (int c = 0; c < HD; c += 8) {
                    uint4 w;
                    w.x = pack_bf16(o[c] * inv, o[c + 1] * inv);
                    w.y = pack_bf16(o[c + 2] * inv, o[c + 3] * inv);
                    w.z = pack_bf16(o[c + 4] * inv, o[c + 5] * inv);
                    w.w = pack_bf16(o[c + 6] * inv, o[c + 7] * inv);
                    *reinterpret_cast<uint4*>(op + c) = w;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

void encode_rows(CUtensorMap* m, const void* ptr, long long rows, long long cols, long long ld) {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            raise(SDX_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 2)};
    const cuuint32_t box[2] = {64, 128};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) raise(SDX_CUDA_ERROR, "attention tensor map encode failed");
}

}  // namespace

AttnPlan plan_attention(const __nv_bfloat16* q, long long q_rows_total, long long ld_q, int q_col0,
                        const __nv_bfloat16* kv, long long kv_rows_total, long long ld_kv, int k_col0, int v_col0,
                        __nv_bfloat16* out, long long ld_out, int out_col0, int images, int heads, int q_len,
                        int q_rows_per_img, int kv_len, int kv_rows_per_img, const int* kv_index, const int* rows_dev,
                        float scale) {
    AttnPlan p;
    encode_rows(&p.tq, q, q_rows_total, ld_q, ld_q);
    encode_rows(&p.tkv, kv, kv_rows_total, ld_kv, ld_kv);
    p.a.q_col0 = q_col0;
    p.a.q = q;
    p.a.q_rows_total = q_rows_total;
    p.a.ld_q = ld_q;
    p.a.k_col0 = k_col0;
    p.a.v_col0 = v_col0;
    p.a.out = out;
    p.a.ld_out = ld_out;
    p.a.out_col0 = out_col0;
    p.a.q_len = q_len;
    p.a.q_rows_per_img = q_rows_per_img;
    p.a.kv_len = kv_len;
    p.a.kv_rows_per_img = kv_rows_per_img;
    p.a.kv_index = kv_index;
    p.a.rows_dev = rows_dev;
    p.a.scale = scale;
    p.images = images;
    p.heads = heads;
    p.valid = true;
    return p;
}

namespace {
int g_attn_xmode = 0;
long long* g_attn_dbg = nullptr;
}
void set_attention_probe_mode(int mode) { g_attn_xmode = mode; }
void set_attention_debug_buffer(long long* dbg) { g_attn_dbg = dbg; }

// SDX_ATTN_TS=0: the P-in-shared-memory kernel (attn_kernel) instead of attn_ts_kernel
static bool attn_ts_enabled() {
    static const bool on = [] {
        const char* v = std::getenv("SDX_ATTN_TS");
        return !(v && v[0] == '0');
    }();
    return on;
}

static int attn_poly() {
    static const int v = [] {
        const char* e = std::getenv("SDX_ATTN_POLY");
        return e ? std::atoi(e) : kPolyDefault;
    }();
    return v;
}

void run_attention(const AttnPlan& p, cudaStream_t st) {
    const bool ts = attn_ts_enabled() && g_attn_xmode == 0;
    const int poly = attn_poly();
    auto ts_kern = poly == 2 ? attn_ts_kernel<2> : poly == 3 ? attn_ts_kernel<3> : poly == 4 ? attn_ts_kernel<4>
                 : poly == 6 ? attn_ts_kernel<6> : attn_ts_kernel<0>;
    const size_t smem = ts ? (2 + 2 * KVS_TS) * TILE_BYTES + 1024 + 256 : (2 + 2 * KVS + 4 * PB) * TILE_BYTES + 1024 + 256;
    if (ts) ensure_kernel_attrs(ts_kern, smem);
    else ensure_kernel_attrs(attn_kernel, smem);
    AttnArgs a = p.a;
    a.xmode = g_attn_xmode;
    a.dbg = g_attn_dbg;
    a.heads = p.heads;
    const int npairs = (p.a.q_len + 2 * BQ - 1) / (2 * BQ);
    const int total = npairs * p.heads * p.images;
    // full waves of pair units; a remainder of R pairs becomes 2R single-tile units when those
    // fit one wave (a last wave of R << 148 pair CTAs would leave the GPU mostly idle)
    int full = total;
    if (total > kSmCount && (total % kSmCount) * 2 <= kSmCount)
        full = (total / kSmCount) * kSmCount;
    // one launch: CTAs [0, full) run pair units, [full, full + 2 (total - full)) single-tile units
    a.single = 0;
    a.unit_base = 0;
    a.pair_base = full;
    launch_pdl(ts ? ts_kern : attn_kernel, dim3(full + 2 * (total - full)), dim3(ts ? 352 : 320), smem, st, p.tq,
               p.tkv, a);
}

}  // namespace sdx
