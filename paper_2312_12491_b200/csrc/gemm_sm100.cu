// tcgen05 / TMA GEMM + implicit-GEMM conv3x3 (see gemm_sm100.cuh).
//
// Persistent CTAs (one per SM) walking 128 x BN output tiles, 6 warps:
//   warp 0      TMA producer (one elected lane): A and B K-slices (64 wide,
//               128-byte swizzle) into a STAGES-deep smem ring (full/empty mbarriers)
//   warp 1      TMEM allocation + MMA issuer (one lane): 4 x tcgen05.mma
//               (M=128, N=BN, K=16) per stage, tcgen05.commit frees the stage
//   warps 2..9  epilogue (two per TMEM lane quadrant): tcgen05.ld 32 lanes x 16 columns, bias / per-image
//               bias / activation / residual in fp32, bf16 or fp32 stores
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include "gemm_sm100.cuh"
#include "sm100.cuh"

namespace sdx {

using namespace sm100;

namespace {

unsigned long long* g_dbg = nullptr;  // phase timestamps of the next launches (kernel benchmarks)
int g_xmode = 0;                      // pipeline probe mode of the next launches (experiments)

struct GemmArgs {
    int M, N, K, K1, amode;
    int Ho, Wo, Cin, stride, Wt, Ht, Nt;
    int splits;   // split-K factor (> 1: raw fp32 partials to ws, epilogue in splitk_reduce)
    float* ws;    // [splits][M][N]
    unsigned long long* dbg;  // optional per-CTA phase timestamps [grid][16] (kernel benchmarks)
    int xmode;                // experiments only: 1 = no MMAs issued, 2 = no TMA loads, 4 = no epilogue (probes)
    int wpre;                 // first B slices issued before the PDL wait
    GemmEpilogue epi;
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t) : : "memory");
    return t;
}

// GEGLU gate: exact erf GELU, or the tanh form with the hardware tanh.approx
// (|err| <= ~1e-3 absolute vs erf GELU, ~6x below the bf16 rounding of the output;
// one SFU op instead of erff's ~25 FMA-pipe instructions, which bound the K=320
// GEGLU epilogue).
__device__ __forceinline__ float geglu_gate(float x, int tanh_form) {
    if (!tanh_form) return 0.5f * x * (1.f + erff(x * 0.70710678118654752f));
    float th;
    asm("tanh.approx.f32 %0, %1;" : "=f"(th) : "f"(0.7978845608028654f * fmaf(0.044715f * x, x * x, x)));
    return 0.5f * x * (1.f + th);
}

__device__ __forceinline__ void wait_bounded(uint64_t* bar, uint32_t phase) {
    // mbarrier wait with a watchdog: a protocol bug traps instead of hanging the GPU
    const uint32_t a = smem_u32(bar);
    uint32_t done = 0;
    long long t0 = 0;  // read only once the first try fails (off the common path)
    while (true) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(a), "r"(phase)
            : "memory");
        if (done) return;
        if (t0 == 0) {
            t0 = clock64();
        } else if (clock64() - t0 > (1LL << 33)) {
            printf("sdx gemm: mbarrier watchdog fired (block %d,%d thread %d)\n", blockIdx.x, blockIdx.y,
                   threadIdx.x);
            asm volatile("trap;");
        }
    }
}

__device__ __forceinline__ float act_fn(float v, int act) {
    switch (act) {
        case kActSilu: return v / (1.f + __expf(-v));
        case kActRelu: return fmaxf(v, 0.f);
        case kActGelu: return 0.5f * v * (1.f + erff(v * 0.70710678118654752f));
        default: return v;
    }
}

// GroupNorm statistics of one 32-row x 32-column epilogue chunk (fast path):
// per group the sum and sum of squares of the stored (bf16-rounded) values of
// the warp's 32 rows (one image: rows per image are multiples of 32), reduced
// over the warp with shuffles, one 2^-20 fixed-point int64 atomic per (group,
// moment) — exact, order-independent, so deterministic.
__device__ __forceinline__ void gn_sink_chunk(const GemmEpilogue& e, int ngn, const float* v, int col0, int row0,
                                              bool live, int lane) {
    float r[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) r[i] = live ? __bfloat162float(__float2bfloat16(v[i])) : 0.f;
#pragma unroll 1
    for (int kk = 0; kk < ngn; ++kk) {
        const GnSink sk = kk == 0 ? e.gn[0] : e.gn[1];
        const int c0 = sk.c_off + col0;
        const int g0 = c0 / sk.cg, g1 = (c0 + 31) / sk.cg;
        const long long img = row0 / sk.hw;
#pragma unroll 1
        for (int gi = g0; gi <= g1; ++gi) {
            const int lo = gi * sk.cg - c0, hi = lo + sk.cg;
            float a = 0.f, b = 0.f;
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const float x = (i >= lo && i < hi) ? r[i] : 0.f;
                a += x;
                b = fmaf(x, x, b);
            }
#pragma unroll
            for (int off = 16; off; off >>= 1) {
                a += __shfl_xor_sync(0xffffffffu, a, off);
                b += __shfl_xor_sync(0xffffffffu, b, off);
            }
            if (lane == 0) {
                unsigned long long* acc = sk.acc + (img * sk.groups + gi) * 2;
                atomicAdd(acc, static_cast<unsigned long long>(__float2ll_rn(a * kGnFixedScale)));
                atomicAdd(acc + 1, static_cast<unsigned long long>(__float2ll_rn(b * kGnFixedScale)));
            }
        }
    }
}

// Persistent: grid = min(tiles, SMs); tiles in (m, n) order with n fastest so
// consecutive tiles share the A block in L2.  Two TMEM accumulators let the
// epilogue of tile i overlap the MMAs of tile i+1.
//
// PAIR: a cluster of two CTAs on one TPC runs 2-SM MMAs (cta_group::2, M = 256):
// each CTA stages its own 128 A rows and half of the BN B rows, the leader
// issues the MMAs, every CTA's TMEM holds its 128 output rows x BN and runs its
// own epilogue.  Halves the per-SM B traffic (L2 and smem) of a 256 x BN tile.
// Epilogue warps: 12 (3 per TMEM lane quadrant, 2 KB smem box each) on the fast path,
// whose small-K GEMMs are epilogue-bound; 8 (4 KB fp32 slabs) on the general path.
// The halo conv (TAESD, N = 64) runs its fast epilogue with 8 warps: the CTA's warps spread over
// the SM's 4 sub-partitions, whose register files bound the registers per thread (14 warps: 128,
// with spills; 10 warps: 168, none).  Measured: TAESD encode / decode 4-5% faster, while the
// UNet's K = 320 GEMMs keep the 12 warps they need (8 warps: 0.6% slower per forward).
template <bool FAST, bool HALO = false>
struct EpiCfg {
    static_assert(kRowStatParts * 4 == 12, "row-statistics partials = fast-path epilogue warps per quadrant");
    static constexpr int kWarps = FAST && !HALO ? 12 : 8;
    static constexpr int kSlab = FAST ? 2048 : 4096;
    static constexpr int kThreads = 64 + 32 * kWarps;
};

template <int BN, int STAGES, int AMODE, bool FAST, bool PAIR>
__global__ void __launch_bounds__(EpiCfg<FAST, AMODE == kAHalo>::kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap ta2,
                   const __grid_constant__ CUtensorMap tb, const __grid_constant__ CUtensorMap to, const GemmArgs g) {
    static_assert(!PAIR || FAST, "CTA-pair GEMM uses the fast epilogue");
    constexpr int BM = 128, BK = 64;
    constexpr int BNL = PAIR ? BN / 2 : BN;  // B rows staged by this CTA
    constexpr bool HALO = AMODE == kAHalo;
    // halo mode: an A stage is one 3 x 130-pixel x 64-channel box (1024-aligned), B (9 taps x BN
    // rows) stays resident for the whole kernel
    constexpr uint32_t HALO_TX = 3 * 130 * 128;
    constexpr uint32_t A_BYTES = HALO ? ((HALO_TX + 1023) / 1024) * 1024 : BM * BK * 2;
    constexpr uint32_t B_BYTES = BNL * BK * 2;
    constexpr uint32_t TMEM_COLS = (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128 : (2 * BN <= 256) ? 256 : 512;

    if (threadIdx.x == 0) pdl_launch();
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_BYTES;
    constexpr int NEPI = EpiCfg<FAST, AMODE == kAHalo>::kWarps, SLAB = EpiCfg<FAST, AMODE == kAHalo>::kSlab;
    uint8_t* slabs = sB + (HALO ? 9 : STAGES) * B_BYTES;  // NEPI epilogue warps x SLAB (1024-aligned)
    uint64_t* full = reinterpret_cast<uint64_t*>(slabs + NEPI * SLAB);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;   // [2]
    uint64_t* tempty = tfull + 2;       // [2]
    uint64_t* bfull = tempty + 2;       // halo mode: resident B landed
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int nk = g.K / BK;
    unsigned long long* dbg = g.dbg ? g.dbg + blockIdx.x * 16 : nullptr;
    if (dbg && threadIdx.x == 0) dbg[0] = gtimer();

    if (warp == 0 && lane == 0) {
        tma_prefetch(&ta);
        if (AMODE == kAConcat) tma_prefetch(&ta2);
        tma_prefetch(&tb);
        if (FAST) tma_prefetch(&to);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(bfull, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], (PAIR ? 2 : 1) * NEPI);  // one arrival per epilogue warp (of both CTAs)
        }
        fence_barrier_init();
    }
    const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
    if (warp == 1) {
        if (PAIR) tmem_alloc_pair(tmem_slot, TMEM_COLS);
        else tmem_alloc(tmem_slot, TMEM_COLS);
    }
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync();  // peer barriers initialised before any cross-CTA signal
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (dbg && threadIdx.x == 0) dbg[1] = gtimer();
    constexpr int MU = PAIR ? 2 * BM : BM;  // rows per work unit (a CTA pair covers 256)
    const int n_tiles = (g.N + BN - 1) / BN;
    const int splits = g.splits;
    const int ustart = PAIR ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
    const int ustep = PAIR ? static_cast<int>(gridDim.x >> 1) : static_cast<int>(gridDim.x);
    // Weights are never written by earlier kernels of the stream, so their first loads are
    // issued before the PDL wait and overlap the previous kernel's tail: the resident
    // 9-tap B of the halo conv, or the B slices of this CTA's first work unit (at the
    // planned row count) for the first min(STAGES, slices) stages, each with an expect_tx
    // but no arrival (the A load after the wait arrives; a unit the live row count drops
    // arrives without A and drains).
    int npre = 0;
    if (warp == 0 && lane == 0 && g.xmode == 0) {
        if (HALO) {
            mbar_expect_tx(bfull, 9 * B_BYTES);
            for (int tap = 0; tap < 9; ++tap) tma_load_2d(sB + tap * B_BYTES, &tb, bfull, tap * BK, 0);
        } else if (!PAIR && g.wpre) {
            const int total_max = ((g.M + MU - 1) / MU) * n_tiles * splits;
            if (ustart < total_max) {
                const int t = ustart / splits, sp = ustart - t * splits;
                const int kb0 = sp * nk / splits, kb1 = (sp + 1) * nk / splits;
                const int n0 = (t % n_tiles) * BN;
                npre = kb1 - kb0 < STAGES ? kb1 - kb0 : STAGES;
                for (int i = 0; i < npre; ++i) {
                    mbar_expect_tx_only(&full[i], B_BYTES);
                    tma_load_2d(sB + i * B_BYTES, &tb, &full[i], (kb0 + i) * BK, n0);
                }
            }
        }
    }
    // everything above overlaps the previous kernel's tail (PDL); from here on
    // memory written by earlier kernels (incl. the live row count) is read
    pdl_wait();
    int m_eff = g.M;
    if (g.epi.rows_dev) {
        const long long lim = static_cast<long long>(*g.epi.rows_dev) * g.epi.rows_per_unit;
        if (lim < m_eff) m_eff = static_cast<int>(lim);
    }
    const int m_tiles = (m_eff + MU - 1) / MU;  // device-decided batch: only live rows' tiles
    const int total = m_tiles * n_tiles * splits;  // work units: (tile, K split); CTAs past it idle

    if (HALO && warp == 0) {
        if (lane == 0) {
            if (g.xmode != 0) {  // probes: the resident B was not prefetched
                mbar_expect_tx(bfull, 9 * B_BYTES);
                for (int tap = 0; tap < 9; ++tap) tma_load_2d(sB + tap * B_BYTES, &tb, bfull, tap * BK, 0);
            }
            uint32_t it = 0;
            const int hw = g.Ho * g.Wo;
            for (int u = ustart; u < total; u += ustep, ++it) {
                const int m0 = u * BM;  // n_tiles == splits == 1
                const int cn0 = m0 / hw;
                const int rem = m0 - cn0 * hw;
                const int cy0 = rem / g.Wo, cx0 = rem - cy0 * g.Wo;
                const int s = it % STAGES;
                wait_bounded(&empty[s], ((it / STAGES) & 1) ^ 1);
                mbar_expect_tx(&full[s], HALO_TX);
                tma_load_4d(sA + s * A_BYTES, &ta, &full[s], 0, cx0 - 1, cy0 - 1, cn0);
            }
        }
    } else if (HALO && warp == 1) {
        {  // converged warp, elected-lane issue (sm100.cuh)
            constexpr uint32_t idesc = idesc_bf16(BM, BN);
            wait_bounded(bfull, 0);
            uint32_t it = 0;
            for (int u = ustart; u < total; u += ustep, ++it) {
                const uint32_t acc = it & 1;
                wait_bounded(&tempty[acc], ((it >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t dtm = tmem + acc * BN;
                const int s = it % STAGES;
                wait_bounded(&full[s], (it / STAGES) & 1);
                tc_fence_after();
                // descriptors: the A window of a tap is the stage's box shifted by whole 128-byte
                // rows, and the start address sits in the descriptor's low bits (16-byte units), so
                // every tap's descriptor is the base one plus a constant; the fully unrolled tap
                // loop issues the 36 MMAs back to back
                const uint64_t da0 = desc_kmajor_sw128(smem_u32(sA + s * A_BYTES));
                const uint64_t db0 = desc_kmajor_sw128(smem_u32(sB));
#pragma unroll
                for (int tap = 0; tap < 9; ++tap) {
                    const int dy = tap / 3, dx = tap - dy * 3;
                    // output pixel i of the tile reads halo pixel (dy, i + dx): 128 consecutive rows
                    // the SW128 XOR pattern follows the absolute smem address bits (as the TMA wrote
                    // it), so a start at any 128-byte row needs no descriptor base offset
                    const uint64_t da = da0 + static_cast<uint64_t>((dy * 130 + dx) * 128 / 16);
                    const uint64_t db = db0 + static_cast<uint64_t>(tap * B_BYTES / 16);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
                        umma_f16_el(dtm, da + 2 * k, db + 2 * k, idesc, (tap != 0 || k != 0) ? 1u : 0u);
                }
                umma_commit_el(&empty[s]);
                umma_commit_el(&tfull[acc]);
            }
        }
        __syncwarp();
    } else if (warp == 0) {
        if (lane == 0) {
            // Lean issue loop (this single thread paces the TMA stream; its per-slice issue
            // latency bounded the convs): stage ring position and conv tap / channel-block
            // coordinates advance incrementally, no divisions per K slice.
            const int cblocks = AMODE == kAConv ? g.Cin / BK : 1;
            int s = 0;
            uint32_t ph = 0, it = 0;
            if (npre > 0 && ustart >= total) {
                // the live row count dropped this CTA's first unit: drain the prefetched B
                for (int i = 0; i < npre; ++i) mbar_arrive(&full[i]);
                for (int i = 0; i < npre; ++i) wait_bounded(&full[i], 0);
            }
            for (int u = ustart; u < total; u += ustep) {
                const int t = u / splits, sp = u - t * splits;
                const int kb0 = sp * nk / splits, kb1 = (sp + 1) * nk / splits;
                const int m0 = (t / n_tiles) * MU + static_cast<int>(rank) * BM;
                const int n0 = (t % n_tiles) * BN + static_cast<int>(rank) * BNL;
                int cn0 = 0, ax = 0, ay = 0, cb = 0, dx = 0;
                if (AMODE == kAConv) {
                    const int hw = g.Ho * g.Wo;
                    cn0 = m0 / hw;
                    const int rem = m0 - cn0 * hw;
                    const int cy0 = rem / g.Wo, cx0 = rem - cy0 * g.Wo;
                    const int tap = kb0 / cblocks, dy = tap / 3;
                    cb = kb0 - tap * cblocks;
                    dx = tap - dy * 3;
                    ax = cx0 * g.stride + dx - 1;  // box origin of the current tap
                    ay = cy0 * g.stride + dy - 1;
                }
                const int k1b = AMODE == kAConcat ? g.K1 / BK : 0;
                for (int kb = kb0; kb < kb1; ++kb, ++it) {
                    wait_bounded(&empty[s], ph ^ 1);
                    uint8_t* dA = sA + s * A_BYTES;
                    if (g.xmode == 2) {  // probe: skip the loads
                        if (rank == 0) mbar_arrive(&full[s]);
                    } else {
                        const CUtensorMap* amap = (AMODE == kAConcat && kb >= k1b) ? &ta2 : &ta;
                        const int ac0 = AMODE == kAConv ? cb * BK : (AMODE == kAConcat && kb >= k1b ? kb - k1b : kb) * BK;
                        if constexpr (PAIR) {
                            // both CTAs' loads complete on the leader's full barrier
                            const uint32_t fb = mapa_shared(smem_u32(&full[s]), 0);
                            if (rank == 0) mbar_expect_tx(&full[s], 2 * (A_BYTES + B_BYTES));
                            if (AMODE == kAConv) tma_load_4d_pair(dA, amap, fb, ac0, ax, ay, cn0);
                            else tma_load_2d_pair(dA, amap, fb, ac0, m0);
                            tma_load_2d_pair(sB + s * B_BYTES, &tb, fb, kb * BK, n0);
                        } else {
                            const bool bpre = static_cast<int>(it) < npre;  // B already in flight (prefetched)
                            mbar_expect_tx(&full[s], bpre ? A_BYTES : A_BYTES + B_BYTES);
                            if (AMODE == kAConv) tma_load_4d(dA, amap, &full[s], ac0, ax, ay, cn0);
                            else tma_load_2d(dA, amap, &full[s], ac0, m0);
                            if (!bpre) tma_load_2d(sB + s * B_BYTES, &tb, &full[s], kb * BK, n0);
                        }
                    }
                    if (AMODE == kAConv && ++cb == cblocks) {  // next tap
                        cb = 0;
                        if (++dx == 3) {
                            dx = 0;
                            ax -= 2;
                            ay += 1;
                        } else {
                            ax += 1;
                        }
                    }
                    if (++s == STAGES) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (rank == 0) {  // converged warp, elected-lane issue; CTA pair: only the leader issues
            constexpr uint32_t idesc = idesc_bf16(PAIR ? 2 * BM : BM, BN);
            uint32_t it = 0, lt = 0, ph = 0;
            int s = 0;  // stage ring position (advanced incrementally, as the producer's)
            // stage descriptors = stage-0 descriptors + the stage offset (16-byte units)
            const uint64_t da0 = desc_kmajor_sw128(smem_u32(sA)), db0 = desc_kmajor_sw128(smem_u32(sB));
            for (int u = ustart; u < total; u += ustep, ++lt) {
                const int sp = u % splits;
                const int kb0 = sp * nk / splits, kb1 = (sp + 1) * nk / splits;
                const uint32_t acc = lt & 1;
                wait_bounded(&tempty[acc], ((lt >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t dtm = tmem + acc * BN;
                for (int kb = kb0; kb < kb1; ++kb, ++it) {
                    wait_bounded(&full[s], ph);
                    if (dbg && it == 0 && lane == 0) dbg[2] = gtimer();
                    tc_fence_after();
                    const uint64_t da = da0 + static_cast<uint64_t>(s) * (A_BYTES >> 4);
                    const uint64_t db = db0 + static_cast<uint64_t>(s) * (B_BYTES >> 4);
#pragma unroll
                    for (int k = 0; k < (g.xmode == 1 ? 0 : BK / 16); ++k) {  // +32 B per K=16 step in the swizzle atom
                        if (PAIR) umma_f16_pair_el(dtm, da + 2 * k, db + 2 * k, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
                        else umma_f16_el(dtm, da + 2 * k, db + 2 * k, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
                    }
                    if (PAIR) umma_commit_pair_el(&empty[s], 3);
                    else umma_commit_el(&empty[s]);
                    if (++s == STAGES) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                if (PAIR) umma_commit_pair_el(&tfull[acc], 3);
                else umma_commit_el(&tfull[acc]);
                if (dbg && lt == 0 && lane == 0) dbg[3] = gtimer();
            }
        }
        __syncwarp();
    } else if constexpr (FAST) {
        // Streamlined epilogue (bf16 output, or the fp32 split-K partials): each
        // thread owns one TMEM lane = one output row; per 32-column chunk
        // tcgen05.ld -> scale / bias / per-image bias / ReLU / residual in
        // registers -> 64-byte rows into a 64B-swizzled smem box -> one TMA
        // store per warp (OOB rows / columns clipped by the tensor map).  The
        // residual row segment is fetched before the TMEM load.
        const int q = warp & 3;
        const int part = (warp - 2) >> 2;  // which of the quadrant's NEPI/4 warps
        constexpr int CSTEP = 32 * (NEPI / 4);
        const bool raw = splits > 1;
        const float e_scale = raw ? 1.f : g.epi.scale;
        const float* e_bias = raw ? nullptr : g.epi.bias;
        const float* e_bimg = raw ? nullptr : g.epi.bias_img;
        const long long e_rpi = g.epi.rows_per_img;
        const int* e_imgidx = g.epi.img_index;
        const long long e_bimg_ld = g.epi.bias_img_ld ? g.epi.bias_img_ld : g.N;
        const __nv_bfloat16* e_res = raw ? nullptr : g.epi.residual;
        const long long e_ldres = g.epi.ld_res;
        const bool e_relu = !raw && g.epi.act == kActRelu;
        const bool e_aar = !raw && g.epi.act_after_residual;
        const bool e_geglu = !raw && g.epi.geglu;
        const int e_ngn = raw ? 0 : g.epi.n_gn;
        const float2* e_lnp = raw ? nullptr : g.epi.ln_part;
        const float* e_lns = g.epi.ln_s;
        float2* e_rso = raw ? nullptr : g.epi.row_stats_out;
        uint8_t* slab = slabs + (warp - 2) * SLAB;
        const uint32_t slab_s = smem_u32(slab);
        uint32_t lt = 0;
        for (int u = ustart; u < total; u += ustep, ++lt) {
            const int t = u / splits;
            const int sp = u - t * splits;
            const uint32_t acc = lt & 1;
            const int m0 = (t / n_tiles) * MU + static_cast<int>(rank) * BM;
            const int n0 = (t % n_tiles) * BN;
            const int row0 = m0 + q * 32;
            const int row = row0 + lane;
            // per-row operands that do not depend on the accumulator are fetched before
            // waiting for it, so their latency hides under this tile's MMAs
            const float* bimg = nullptr;
            if (e_bimg && row < m_eff) {
                const long long im = static_cast<long long>(row) / e_rpi;
                bimg = e_bimg + (e_imgidx ? e_imgidx[im] : im) * e_bimg_ld;
            }
            // folded LayerNorm: this row's mean / rstd from the producer's partials
            float ln_mean = 0.f, ln_rstd = 1.f;
            if (e_lnp) {
                float s1 = 0.f, s2 = 0.f;
                if (row < m_eff) {
                    for (int pi = 0; pi < g.epi.ln_nparts; ++pi) {
                        const float2 pv = e_lnp[static_cast<long long>(pi) * g.M + row];
                        s1 += pv.x;
                        s2 += pv.y;
                    }
                }
                const float inv_c = 1.f / static_cast<float>(g.epi.ln_C);
                ln_mean = s1 * inv_c;
                const float var = fmaxf(s2 * inv_c - ln_mean * ln_mean, 0.f);
                ln_rstd = rsqrtf(var + g.epi.ln_eps);
            }
            // residual: the first chunk's row segment is requested before waiting for
            // the accumulator (its latency hides under this tile's MMAs)
            const __nv_bfloat16* res_row = e_res ? e_res + static_cast<long long>(row < m_eff ? row : 0) * e_ldres : nullptr;
            uint4 rq[4];
            if (res_row && n0 + part * 32 < g.N) {
#pragma unroll
                for (int i = 0; i < 4; ++i) rq[i] = reinterpret_cast<const uint4*>(res_row + n0 + part * 32)[i];
            }
            wait_bounded(&tfull[acc], (lt >> 1) & 1);
            if (dbg && lt == 0 && warp == 2 && lane == 0) dbg[4] = gtimer();
            tc_fence_after();
            if (g.xmode == 4) {  // probe: no epilogue work (results wrong)
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (PAIR) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));
                    else mbar_arrive(&tempty[acc]);
                }
                continue;
            }
            float rs_sum = 0.f, rs_sq = 0.f;  // row statistics of this tile's stored values
            const uint32_t tbase = tmem + acc * BN + (static_cast<uint32_t>(q * 32) << 16);
#pragma unroll 1
            int kc = 0;
            for (int c = part * 32; c < BN; c += CSTEP, ++kc) {
                const int col0 = n0 + c;
                if (col0 >= g.N) break;  // warp-uniform; N % 32 == 0 on this path
                if (res_row && kc > 0) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) rq[i] = reinterpret_cast<const uint4*>(res_row + col0)[i];
                }
                uint32_t r[32];
                tmem_ld32_nowait(tbase + c, r);
                tmem_wait_ld32(r);
                const bool dstamp = dbg && lt == 0 && warp == 2 && lane == 0;
                if (dstamp && kc < 3) dbg[7 + 3 * kc] = gtimer();
                float v[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]) * e_scale;
                if (e_lnp) {
#pragma unroll
                    for (int i = 0; i < 32; i += 4) {
                        const float4 sv = *reinterpret_cast<const float4*>(e_lns + col0 + i);
                        v[i] = ln_rstd * fmaf(-ln_mean, sv.x, v[i]);
                        v[i + 1] = ln_rstd * fmaf(-ln_mean, sv.y, v[i + 1]);
                        v[i + 2] = ln_rstd * fmaf(-ln_mean, sv.z, v[i + 2]);
                        v[i + 3] = ln_rstd * fmaf(-ln_mean, sv.w, v[i + 3]);
                    }
                }
                if (e_bias) {
#pragma unroll
                    for (int i = 0; i < 32; i += 4) {
                        const float4 b = *reinterpret_cast<const float4*>(e_bias + col0 + i);
                        v[i] += b.x; v[i + 1] += b.y; v[i + 2] += b.z; v[i + 3] += b.w;
                    }
                }
                if (bimg) {
#pragma unroll
                    for (int i = 0; i < 32; i += 4) {
                        const float4 b = *reinterpret_cast<const float4*>(bimg + col0 + i);
                        v[i] += b.x; v[i + 1] += b.y; v[i + 2] += b.z; v[i + 3] += b.w;
                    }
                }
                if (e_relu && !e_aar) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
                }
                if (e_res) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&rq[i]);
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const float2 f = __bfloat1622float2(h2[j]);
                            v[8 * i + 2 * j] += f.x;
                            v[8 * i + 2 * j + 1] += f.y;
                        }
                    }
                }
                if (e_relu && e_aar) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
                }
                if (e_ngn > 0) gn_sink_chunk(g.epi, e_ngn, v, col0, row0, row < m_eff, lane);
                if (e_rso) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const float x = __bfloat162float(__float2bfloat16(v[i]));
                        rs_sum += x;
                        rs_sq = fmaf(x, x, rs_sq);
                    }
                }
                const int sw = (lane >> 1) & 3;  // 64-byte swizzle: 16 B chunk j of row r at r*64 + ((j ^ (r>>1 & 3)) * 16)
                if (raw) {
                    // fp32 partials: two 16-column boxes through the warp's 2 KB buffer
#pragma unroll
                    for (int hb = 0; hb < 2; ++hb) {
                        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                        __syncwarp();
                        uint8_t* rowp = slab + lane * 64;
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            *reinterpret_cast<float4*>(rowp + ((j ^ sw) << 4)) =
                                make_float4(v[16 * hb + 4 * j], v[16 * hb + 4 * j + 1], v[16 * hb + 4 * j + 2], v[16 * hb + 4 * j + 3]);
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        __syncwarp();
                        if (lane == 0) {
                            asm volatile(
                                "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                                    reinterpret_cast<uint64_t>(&to)),
                                "r"(col0 + 16 * hb), "r"(row0), "r"(sp), "r"(slab_s)
                                : "memory");
                            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                        }
                    }
                } else if (e_geglu) {
                    // interleaved [16 value | 16 gate] columns -> 16 outputs; 32-byte rows, 32B swizzle
                    if (g.epi.gelu_tanh) {
#pragma unroll
                        for (int i = 0; i < 16; ++i) v[i] *= geglu_gate(v[16 + i], 1);
                    } else {
#pragma unroll
                        for (int i = 0; i < 16; ++i) v[i] *= geglu_gate(v[16 + i], 0);
                    }
                    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    __syncwarp();
                    uint8_t* rowp = slab + lane * 32;
                    const int sw2 = (lane >> 2) & 1;
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        uint4 o;
                        o.x = pack_bf16(v[8 * j], v[8 * j + 1]);
                        o.y = pack_bf16(v[8 * j + 2], v[8 * j + 3]);
                        o.z = pack_bf16(v[8 * j + 4], v[8 * j + 5]);
                        o.w = pack_bf16(v[8 * j + 6], v[8 * j + 7]);
                        *reinterpret_cast<uint4*>(rowp + ((j ^ sw2) << 4)) = o;
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) {
                        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                                         reinterpret_cast<uint64_t>(&to)),
                                     "r"(col0 / 2), "r"(row0), "r"(slab_s)
                                     : "memory");
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                } else {
                    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    __syncwarp();
                    uint8_t* rowp = slab + lane * 64;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        uint4 o;
                        o.x = pack_bf16(v[8 * j], v[8 * j + 1]);
                        o.y = pack_bf16(v[8 * j + 2], v[8 * j + 3]);
                        o.z = pack_bf16(v[8 * j + 4], v[8 * j + 5]);
                        o.w = pack_bf16(v[8 * j + 6], v[8 * j + 7]);
                        *reinterpret_cast<uint4*>(rowp + ((j ^ sw) << 4)) = o;
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) {
                        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                                         reinterpret_cast<uint64_t>(&to)),
                                     "r"(col0), "r"(row0), "r"(slab_s)
                                     : "memory");
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                }
                if (dstamp && kc < 3) dbg[9 + 3 * kc] = gtimer();
            }
            if (e_rso && row < m_eff)
                e_rso[static_cast<long long>(kRowStatParts * (t % n_tiles) + part) * g.M + row] = make_float2(rs_sum, rs_sq);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (PAIR) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));  // the leader's barrier
                else mbar_arrive(&tempty[acc]);
            }
            if (dbg && lt == 0 && warp == 2 && lane == 0) dbg[5] = gtimer();
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        __syncwarp();
    } else {
        // epilogue warps 2..9 -> TMEM lane quadrant warp % 4 (two warps per quadrant
        // split the 32-column chunks).  Per chunk: phase 1: tcgen05.ld 32 fp32 of the
        // thread's row, scale + bias + per-image bias (+ fused GEGLU), staged in this
        // warp's XOR-swizzled smem slab;  phase 2: the warp re-reads the slab so 4 lanes
        // cover one row's 32 columns, adds the residual, applies the activation,
        // accumulates GroupNorm statistics and writes 16-byte coalesced stores.
        // Every epilogue field is read into a scalar once (param space; no local copy).
        const int q = warp & 3;
        const int half = (warp - 2) >> 2;
        const bool raw = splits > 1;  // split-K partials: plain fp32 sums, splitk_reduce finishes
        const float e_scale = raw ? 1.f : g.epi.scale;
        const float* e_bias = raw ? nullptr : g.epi.bias;
        const float* e_bimg = raw ? nullptr : g.epi.bias_img;
        const long long e_rpi = g.epi.rows_per_img;
        const int* e_imgidx = g.epi.img_index;
        const long long e_bimg_ld = g.epi.bias_img_ld ? g.epi.bias_img_ld : g.N;
        const __nv_bfloat16* e_res = raw ? nullptr : g.epi.residual;
        const long long e_ldres = g.epi.ld_res;
        const int e_act = raw ? kActNone : g.epi.act;
        const bool e_aar = !raw && g.epi.act_after_residual;
        const int e_outk = raw ? 1 : g.epi.out_f32;
        const long long e_ldo = raw ? g.N : g.epi.ld_out;
        const int* e_omap = raw ? nullptr : g.epi.out_img_map;
        const bool e_geglu = !raw && g.epi.geglu;
        const int e_ngn = raw ? 0 : g.epi.n_gn;
        float* slab = reinterpret_cast<float*>(slabs + (warp - 2) * 4096);
        uint32_t lt = 0;
        for (int u = blockIdx.x; u < total; u += gridDim.x, ++lt) {
            const int t = u / splits;
            void* e_out = raw ? static_cast<void*>(g.ws + static_cast<long long>(u % splits) * g.M * g.N) : g.epi.out;
            const uint32_t acc = lt & 1;
            const int m0 = (t / n_tiles) * BM;
            const int n0 = (t % n_tiles) * BN;
            wait_bounded(&tfull[acc], (lt >> 1) & 1);
            if (dbg && lt == 0 && warp == 2 && lane == 0) dbg[4] = gtimer();
            tc_fence_after();
            const int row = m0 + q * 32 + lane;
            const float* bimg = nullptr;
            if (e_bimg && row < m_eff) {
                const long long im = static_cast<long long>(row) / e_rpi;
                bimg = e_bimg + (e_imgidx ? e_imgidx[im] : im) * e_bimg_ld;
            }
            const uint32_t tbase = tmem + acc * BN + (static_cast<uint32_t>(q * 32) << 16);
#pragma unroll 1
            for (int c = half * 32; c < BN; c += 64) {
                const int col0 = n0 + c;
                if (col0 >= g.N) continue;  // warp-uniform (columns past N hold no data)
                // phase-2 geometry: lane -> (row, 8 columns); 4 lanes per row (2 for GEGLU's 16 outputs)
                const int lpr_shift = e_geglu ? 1 : 2;
                const int pc = (lane & ((1 << lpr_shift) - 1)) * 8;
                const int nout = e_geglu ? g.N / 2 : g.N;
                const int gcol = (e_geglu ? col0 / 2 : col0) + pc;
                // residual rows of all passes are fetched before the TMEM load so
                // their latency overlaps the accumulator read-out
                uint4 resv[4];
                if (e_res) {
#pragma unroll
                    for (int ps = 0; ps < 4; ++ps) {
                        const int grow = m0 + q * 32 + ps * 8 + (lane >> 2);
                        resv[ps] = make_uint4(0u, 0u, 0u, 0u);
                        if (grow < m_eff && gcol + 8 <= nout)
                            resv[ps] = *reinterpret_cast<const uint4*>(e_res + static_cast<long long>(grow) * e_ldres + gcol);
                    }
                }
                uint32_t r[32];
                tmem_ld32_nowait(tbase + c, r);
                tmem_wait_ld();
                const bool dstamp = dbg && lt == 0 && warp == 2 && lane == 0;
                if (dstamp) dbg[7 + 3 * (c / 64)] = gtimer();
                const bool vec_ok = col0 + 32 <= g.N;
                float v[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]) * e_scale;
                if (e_bias) {
                    if (vec_ok) {
#pragma unroll
                        for (int i = 0; i < 32; i += 4) {
                            const float4 b = *reinterpret_cast<const float4*>(e_bias + col0 + i);
                            v[i] += b.x; v[i + 1] += b.y; v[i + 2] += b.z; v[i + 3] += b.w;
                        }
                    } else {
                        for (int i = 0; i < 32; ++i)
                            if (col0 + i < g.N) v[i] += e_bias[col0 + i];
                    }
                }
                if (bimg) {
                    for (int i = 0; i < 32; ++i)
                        if (col0 + i < g.N) v[i] += bimg[col0 + i];
                }
                if (e_geglu) {  // interleaved [16 value | 16 gate] columns -> 16 outputs
#pragma unroll
                    for (int i = 0; i < 16; ++i) v[i] *= geglu_gate(v[16 + i], g.epi.gelu_tanh);
                }
                __syncwarp();
                // slab row = 8 x 16-byte chunks, chunk index XOR (row % 8): conflict-free both ways
                float* srow = slab + lane * 32;
#pragma unroll
                for (int i = 0; i < 32; i += 4)
                    *reinterpret_cast<float4*>(srow + (((i >> 2) ^ (lane & 7)) << 2)) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
                __syncwarp();
                if (dstamp) dbg[8 + 3 * (c / 64)] = gtimer();
                // GroupNorm partial sums of this lane's 8 columns (<= 2 groups per sink)
                float ga0 = 0.f, gq0 = 0.f, ga1 = 0.f, gq1 = 0.f, gb0 = 0.f, gr0 = 0.f, gb1 = 0.f, gr1 = 0.f;
                int gsplit0 = 8, gsplit1 = 8;
                if (e_ngn > 0) {
                    const int ch0 = g.epi.gn[0].c_off + gcol;
                    gsplit0 = (ch0 / g.epi.gn[0].cg + 1) * g.epi.gn[0].cg - ch0;
                }
                if (e_ngn > 1) {
                    const int ch0 = g.epi.gn[1].c_off + gcol;
                    gsplit1 = (ch0 / g.epi.gn[1].cg + 1) * g.epi.gn[1].cg - ch0;
                }
#pragma unroll
                for (int ps = 0; ps < 4; ++ps) {
                    if (e_geglu && ps >= 2) break;
                    const int lr = ps * (32 >> lpr_shift) + (lane >> lpr_shift);
                    const int grow = m0 + q * 32 + lr;
                    if (grow >= m_eff || gcol >= nout) continue;
                    const float* sr = slab + lr * 32;
                    float w8[8];
                    const float4 a0 = *reinterpret_cast<const float4*>(sr + ((((pc >> 2)) ^ (lr & 7)) << 2));
                    const float4 a1 = *reinterpret_cast<const float4*>(sr + ((((pc >> 2) + 1) ^ (lr & 7)) << 2));
                    w8[0] = a0.x; w8[1] = a0.y; w8[2] = a0.z; w8[3] = a0.w;
                    w8[4] = a1.x; w8[5] = a1.y; w8[6] = a1.z; w8[7] = a1.w;
                    const bool full8 = gcol + 8 <= nout;
                    if (!e_aar && e_act != kActNone) {
#pragma unroll
                        for (int i = 0; i < 8; ++i) w8[i] = act_fn(w8[i], e_act);
                    }
                    if (e_res) {
                        const __nv_bfloat16* rp = e_res + static_cast<long long>(grow) * e_ldres + gcol;
                        if (full8) {
                            const uint4 rv = resv[ps];
                            const __nv_bfloat16* rb = reinterpret_cast<const __nv_bfloat16*>(&rv);
#pragma unroll
                            for (int i = 0; i < 8; ++i) w8[i] += __bfloat162float(rb[i]);
                        } else {
                            for (int i = 0; i < 8 && gcol + i < nout; ++i) w8[i] += __bfloat162float(rp[i]);
                        }
                    }
                    if (e_aar && e_act != kActNone) {
#pragma unroll
                        for (int i = 0; i < 8; ++i) w8[i] = act_fn(w8[i], e_act);
                    }
                    if (e_ngn > 0) {
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const float rv = (gcol + i < nout) ? __bfloat162float(__float2bfloat16(w8[i])) : 0.f;
                            if (i < gsplit0) { ga0 += rv; gq0 += rv * rv; } else { ga1 += rv; gq1 += rv * rv; }
                            if (e_ngn > 1) {
                                if (i < gsplit1) { gb0 += rv; gr0 += rv * rv; } else { gb1 += rv; gr1 += rv * rv; }
                            }
                        }
                    }
                    long long orow = grow;
                    if (e_omap) {
                        const long long im = static_cast<long long>(grow) / e_rpi;
                        orow = static_cast<long long>(e_omap[im]) * e_rpi + (grow - im * e_rpi);
                    }
                    if (e_outk == 1) {
                        float* op = reinterpret_cast<float*>(e_out) + orow * e_ldo + gcol;
                        if (full8) {
                            *reinterpret_cast<float4*>(op) = make_float4(w8[0], w8[1], w8[2], w8[3]);
                            *reinterpret_cast<float4*>(op + 4) = make_float4(w8[4], w8[5], w8[6], w8[7]);
                        } else {
                            for (int i = 0; i < 8 && gcol + i < nout; ++i) op[i] = w8[i];
                        }
                    } else if (e_outk == 2) {
                        uint8_t* op = reinterpret_cast<uint8_t*>(e_out) + orow * e_ldo + gcol;
                        for (int i = 0; i < 8 && gcol + i < nout; ++i)
                            op[i] = static_cast<uint8_t>(__float2int_rn(fminf(fmaxf(w8[i], 0.f), 1.f) * 255.f));
                    } else if (e_outk == 3) {  // fp16 (attention operands)
                        __half* op = reinterpret_cast<__half*>(e_out) + orow * e_ldo + gcol;
                        if (full8) {
                            uint4 o;
                            __half2* h2 = reinterpret_cast<__half2*>(&o);
                            h2[0] = __floats2half2_rn(w8[0], w8[1]);
                            h2[1] = __floats2half2_rn(w8[2], w8[3]);
                            h2[2] = __floats2half2_rn(w8[4], w8[5]);
                            h2[3] = __floats2half2_rn(w8[6], w8[7]);
                            *reinterpret_cast<uint4*>(op) = o;
                        } else {
                            for (int i = 0; i < 8 && gcol + i < nout; ++i) op[i] = __float2half_rn(w8[i]);
                        }
                    } else {
                        __nv_bfloat16* op = reinterpret_cast<__nv_bfloat16*>(e_out) + orow * e_ldo + gcol;
                        if (full8) {
                            uint4 o;
                            o.x = pack_bf16(w8[0], w8[1]);
                            o.y = pack_bf16(w8[2], w8[3]);
                            o.z = pack_bf16(w8[4], w8[5]);
                            o.w = pack_bf16(w8[6], w8[7]);
                            *reinterpret_cast<uint4*>(op) = o;
                        } else {
                            for (int i = 0; i < 8 && gcol + i < nout; ++i) op[i] = __float2bfloat16(w8[i]);
                        }
                    }
                }
                if (dstamp) dbg[9 + 3 * (c / 64)] = gtimer();
                // lanes sharing columns (lane bits 2..4) combine; lanes 0..3 add one
                // fixed-point atomic per (group, moment)
                if (e_ngn > 0) {
                    float gv[8] = {ga0, gq0, ga1, gq1, gb0, gr0, gb1, gr1};
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        gv[j] += __shfl_xor_sync(0xffffffffu, gv[j], 4);
                        gv[j] += __shfl_xor_sync(0xffffffffu, gv[j], 8);
                        gv[j] += __shfl_xor_sync(0xffffffffu, gv[j], 16);
                    }
                    const int wrow0 = m0 + q * 32;
                    if (lane < 4 && gcol < nout && wrow0 < m_eff) {
#pragma unroll
                        for (int kk = 0; kk < 2; ++kk) {
                            if (kk >= e_ngn) break;
                            const GnSink sk = kk == 0 ? g.epi.gn[0] : g.epi.gn[1];
                            const int split = kk == 0 ? gsplit0 : gsplit1;
                            const long long img = wrow0 / sk.hw;
                            const int g0 = (sk.c_off + gcol) / sk.cg;
                            unsigned long long* a0 = sk.acc + (img * sk.groups + g0) * 2;
                            atomicAdd(a0, static_cast<unsigned long long>(__float2ll_rn(gv[4 * kk] * kGnFixedScale)));
                            atomicAdd(a0 + 1, static_cast<unsigned long long>(__float2ll_rn(gv[4 * kk + 1] * kGnFixedScale)));
                            if (split < 8 && g0 + 1 < sk.groups) {
                                atomicAdd(a0 + 2, static_cast<unsigned long long>(__float2ll_rn(gv[4 * kk + 2] * kGnFixedScale)));
                                atomicAdd(a0 + 3, static_cast<unsigned long long>(__float2ll_rn(gv[4 * kk + 3] * kGnFixedScale)));
                            }
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            if (dbg && lt == 0 && warp == 2 && lane == 0) dbg[5] = gtimer();
        }
    }
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync();  // no CTA leaves while its peer may still signal it
    if (dbg && threadIdx.x == 0) dbg[6] = gtimer();
    if (warp == 1) {
        tc_fence_after();
        if (PAIR) tmem_dealloc_pair(tmem, TMEM_COLS);
        else tmem_dealloc(tmem, TMEM_COLS);
    }
}

// Split-K finish: sum the fp32 partials (fixed split order, so the result is
// deterministic) and apply the full epilogue.  One thread = 8 columns of one
// row; the partials of up to 4 splits are in flight at once (L2-resident,
// __ldcg), residual / bias / output are 16-byte vectors.
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const float* __restrict__ ws, int splits, int M, int N,
                                                            const GemmEpilogue e) {
    pdl_launch();
    pdl_wait();
    int m_eff = M;
    if (e.rows_dev) {
        const long long lim = static_cast<long long>(*e.rows_dev) * e.rows_per_unit;
        if (lim < m_eff) m_eff = static_cast<int>(lim);
    }
    const int nv = (N + 7) / 8;
    const long long total = static_cast<long long>(m_eff) * nv;
    const long long plane = static_cast<long long>(M) * N;
    const bool vec = (N % 8) == 0;
    for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int row = static_cast<int>(idx / nv);
        const int col = static_cast<int>(idx % nv) * 8;
        const int cnt = N - col < 8 ? N - col : 8;
        const float* base = ws + static_cast<long long>(row) * N + col;
        float w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (vec) {
            for (int s0 = 0; s0 < splits; s0 += 4) {
                float4 a[4], b[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (s0 + j < splits) {
                        a[j] = __ldcg(reinterpret_cast<const float4*>(base + (s0 + j) * plane));
                        b[j] = __ldcg(reinterpret_cast<const float4*>(base + (s0 + j) * plane + 4));
                    }
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (s0 + j < splits) {
                        w[0] += a[j].x; w[1] += a[j].y; w[2] += a[j].z; w[3] += a[j].w;
                        w[4] += b[j].x; w[5] += b[j].y; w[6] += b[j].z; w[7] += b[j].w;
                    }
                }
            }
        } else {
            for (int sp = 0; sp < splits; ++sp)
                for (int i = 0; i < cnt; ++i) w[i] += base[sp * plane + i];
        }
        float rsd[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (e.residual) {
            const __nv_bfloat16* rp = e.residual + static_cast<long long>(row) * e.ld_res + col;
            if (cnt == 8 && (e.ld_res % 8) == 0) {
                const uint4 rv = *reinterpret_cast<const uint4*>(rp);
                const __nv_bfloat16* rb = reinterpret_cast<const __nv_bfloat16*>(&rv);
#pragma unroll
                for (int i = 0; i < 8; ++i) rsd[i] = __bfloat162float(rb[i]);
            } else {
                for (int i = 0; i < cnt; ++i) rsd[i] = __bfloat162float(rp[i]);
            }
        }
        float bs[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (e.bias) {
            if (cnt == 8) {
                const float4 b0 = *reinterpret_cast<const float4*>(e.bias + col);
                const float4 b1 = *reinterpret_cast<const float4*>(e.bias + col + 4);
                bs[0] = b0.x; bs[1] = b0.y; bs[2] = b0.z; bs[3] = b0.w;
                bs[4] = b1.x; bs[5] = b1.y; bs[6] = b1.z; bs[7] = b1.w;
            } else {
                for (int i = 0; i < cnt; ++i) bs[i] = e.bias[col + i];
            }
        }
        const long long im = row / e.rows_per_img;
        const float* bimg = e.bias_img ? e.bias_img + (e.img_index ? e.img_index[im] : im) * (e.bias_img_ld ? e.bias_img_ld : N)
                                       : nullptr;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            float x = w[i] * e.scale + bs[i];
            if (bimg && i < cnt) x += bimg[col + i];
            if (!e.act_after_residual) x = act_fn(x, e.act);
            x += rsd[i];
            if (e.act_after_residual) x = act_fn(x, e.act);
            w[i] = x;
        }
        for (int kk = 0; kk < e.n_gn; ++kk) {  // GroupNorm statistics of the stored values
            const GnSink& sk = e.gn[kk];
            const int ch0 = sk.c_off + col;
            const int g0 = ch0 / sk.cg;
            const int b = (g0 + 1) * sk.cg - ch0;
            float a[4] = {0.f, 0.f, 0.f, 0.f};
            for (int i = 0; i < cnt; ++i) {
                const float r = __bfloat162float(__float2bfloat16(w[i]));
                const int hi = i >= b ? 2 : 0;
                a[hi] += r;
                a[hi + 1] += r * r;
            }
            const long long img = row / sk.hw;
            unsigned long long* a0 = sk.acc + (img * sk.groups + g0) * 2;
            atomicAdd(a0, static_cast<unsigned long long>(__float2ll_rn(a[0] * kGnFixedScale)));
            atomicAdd(a0 + 1, static_cast<unsigned long long>(__float2ll_rn(a[1] * kGnFixedScale)));
            if (b < cnt && g0 + 1 < sk.groups) {
                atomicAdd(a0 + 2, static_cast<unsigned long long>(__float2ll_rn(a[2] * kGnFixedScale)));
                atomicAdd(a0 + 3, static_cast<unsigned long long>(__float2ll_rn(a[3] * kGnFixedScale)));
            }
        }
        long long orow = row;
        if (e.out_img_map) orow = static_cast<long long>(e.out_img_map[im]) * e.rows_per_img + (row - im * e.rows_per_img);
        const bool ovec = cnt == 8 && (e.ld_out % 8) == 0;
        if (e.out_f32 == 1) {
            float* op = reinterpret_cast<float*>(e.out) + orow * e.ld_out + col;
            if (ovec) {
                *reinterpret_cast<float4*>(op) = make_float4(w[0], w[1], w[2], w[3]);
                *reinterpret_cast<float4*>(op + 4) = make_float4(w[4], w[5], w[6], w[7]);
            } else {
                for (int i = 0; i < cnt; ++i) op[i] = w[i];
            }
        } else if (e.out_f32 == 2) {
            uint8_t* op = reinterpret_cast<uint8_t*>(e.out) + orow * e.ld_out + col;
            for (int i = 0; i < cnt; ++i) op[i] = static_cast<uint8_t>(__float2int_rn(fminf(fmaxf(w[i], 0.f), 1.f) * 255.f));
        } else if (e.out_f32 == 3) {
            __half* op = reinterpret_cast<__half*>(e.out) + orow * e.ld_out + col;
            for (int i = 0; i < cnt; ++i) op[i] = __float2half_rn(w[i]);
        } else {
            __nv_bfloat16* op = reinterpret_cast<__nv_bfloat16*>(e.out) + orow * e.ld_out + col;
            if (ovec) {
                uint4 o;
                o.x = pack_bf16(w[0], w[1]);
                o.y = pack_bf16(w[2], w[3]);
                o.z = pack_bf16(w[4], w[5]);
                o.w = pack_bf16(w[6], w[7]);
                *reinterpret_cast<uint4*>(op) = o;
            } else {
                for (int i = 0; i < cnt; ++i) op[i] = __float2bfloat16(w[i]);
            }
        }
    }
}

// ---- host: tensor maps ------------------------------------------------------

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    if (!fn) raise(SDX_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
    return fn;
}

void encode(CUtensorMap* m, const void* ptr, int rank, const cuuint64_t* dims, const cuuint64_t* strides_bytes,
            const cuuint32_t* box, const cuuint32_t* estrides,
            CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
            CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
    const CUresult r = encode_fn()(m, dt, rank, const_cast<void*>(ptr), dims, strides_bytes, box, estrides,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) raise(SDX_CUDA_ERROR, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
}

void encode_2d(CUtensorMap* m, const void* ptr, long long rows, long long cols, long long ld, int box_rows) {
    if ((ld * 2) % 16 != 0) raise(SDX_INVALID_ARGUMENT, "gemm: row pitch must be a multiple of 16 bytes");
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 2)};
    const cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_rows)};
    const cuuint32_t es[2] = {1, 1};
    encode(m, ptr, 2, dims, strides, box, es);
}

// smem: 1 KB alignment pad + STAGES x (A 16 KB + B BNL x 128 B) + 8 epilogue slabs of
// 4 KB + barriers; as many stages (<= 8) as fit in 227 KB.
template <int BN, bool PAIR, int AMODE, bool FAST>
constexpr int stages_for() {
    if (AMODE == kAHalo) return 2;  // 2 x 49 KB halo boxes next to 72 KB of resident weights
    constexpr int bnl = PAIR ? BN / 2 : BN;
    constexpr int slabs = EpiCfg<FAST, AMODE == kAHalo>::kWarps * EpiCfg<FAST, AMODE == kAHalo>::kSlab;
    constexpr int st = (232448 - 1024 - slabs - 256) / (128 * 64 * 2 + bnl * 64 * 2);
    return st > 8 ? 8 : st;
}

template <int BN, bool PAIR, int AMODE, bool FAST>
size_t smem_for() {
    constexpr int slabs = EpiCfg<FAST, AMODE == kAHalo>::kWarps * EpiCfg<FAST, AMODE == kAHalo>::kSlab;
    if (AMODE == kAHalo) return 1024 + 2 * 50176 + 9 * BN * 64 * 2 + slabs + 256;
    constexpr int bnl = PAIR ? BN / 2 : BN;
    return 1024 + static_cast<size_t>(stages_for<BN, PAIR, AMODE, FAST>()) * (128 * 64 * 2 + bnl * 64 * 2) + slabs + 256;
}

template <int BN, int AMODE, bool FAST, bool PAIR>
void launch_t(const GemmPlan& p, cudaStream_t st) {
    constexpr int S = stages_for<BN, PAIR, AMODE, FAST>();
    auto k = gemm_tc_kernel<BN, S, AMODE, FAST, PAIR>;
    const size_t smem = smem_for<BN, PAIR, AMODE, FAST>();
    ensure_kernel_attrs(k, smem);
    GemmArgs g{};
    g.M = p.M;
    g.N = p.N;
    g.K = p.K;
    g.K1 = p.K1;
    g.amode = p.amode;
    g.Ho = p.Ho;
    g.Wo = p.Wo;
    g.Cin = p.Cin;
    g.stride = p.stride;
    g.Wt = p.Wt;
    g.Ht = p.Ht;
    g.Nt = p.Nt;
    g.epi = p.epi;
    g.splits = p.splits;
    g.ws = p.ws;
    g.dbg = g_dbg;
    g.xmode = g_xmode;
    // SDX_WPREFETCH=0: no weight loads before the PDL wait
    static const int wpre = [] {
        const char* v = std::getenv("SDX_WPREFETCH");
        return v && v[0] == '0' ? 0 : 1;
    }();
    g.wpre = wpre;
    const int n_tiles = (p.N + BN - 1) / BN;
    if (PAIR) {
        const int pairs = ((p.M + 255) / 256) * n_tiles * p.splits;
        const int np = pairs < kSmCount / 2 ? pairs : kSmCount / 2;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(2 * np);
        cfg.blockDim = dim3(EpiCfg<FAST, AMODE == kAHalo>::kThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
        cfg.attrs = at;
        cfg.numAttrs = 2;
        SDX_CUDA(cudaLaunchKernelEx(&cfg, k, p.ta, p.ta2, p.tb, p.to, g));
    } else {
        const int units = n_tiles * ((p.M + 127) / 128) * p.splits;
        dim3 grid(units < kSmCount ? units : kSmCount);
        launch_pdl(k, grid, dim3(EpiCfg<FAST, AMODE == kAHalo>::kThreads), smem, st, p.ta, p.ta2, p.tb, p.to, g);
    }
    if (p.splits > 1) {
        const long long work = static_cast<long long>(p.M) * ((p.N + 7) / 8);
        long long blocks = (work + 255) / 256;
        if (blocks > 4LL * kSmCount) blocks = 4LL * kSmCount;
        launch_pdl(splitk_reduce_kernel, dim3(static_cast<unsigned>(blocks)), dim3(256), 0, st,
                   static_cast<const float*>(p.ws), p.splits, p.M, p.N, p.epi);
    }
}

template <int AMODE, bool FAST>
void launch_mode(const GemmPlan& p, cudaStream_t st) {
    if constexpr (FAST) {
        if (p.pair) {
            switch (p.bn) {
                case 128: launch_t<128, AMODE, true, true>(p, st); return;
                case 160: launch_t<160, AMODE, true, true>(p, st); return;
                case 192: launch_t<192, AMODE, true, true>(p, st); return;
                case 224: launch_t<224, AMODE, true, true>(p, st); return;
                case 256: launch_t<256, AMODE, true, true>(p, st); return;
                default: raise(SDX_LOGIC_ERROR, "gemm: unsupported CTA-pair tile width");
            }
        }
    }
    switch (p.bn) {
        case 64: launch_t<64, AMODE, FAST, false>(p, st); break;
        case 96: launch_t<96, AMODE, FAST, false>(p, st); break;
        case 128: launch_t<128, AMODE, FAST, false>(p, st); break;
        case 160: launch_t<160, AMODE, FAST, false>(p, st); break;
        case 192: launch_t<192, AMODE, FAST, false>(p, st); break;
        case 224: launch_t<224, AMODE, FAST, false>(p, st); break;
        default: launch_t<256, AMODE, FAST, false>(p, st); break;
    }
}

}  // namespace

namespace {
int g_force_bn = 0, g_force_splits = 0, g_force_pair = 0;  // tiling override (kernel benchmarks only)
}  // namespace

void set_gemm_debug_buffer(unsigned long long* dbg) { g_dbg = dbg; }
void set_gemm_probe_mode(int mode) { g_xmode = mode; }

void set_gemm_tiling_override(int bn, int splits, int pair) {
    g_force_bn = bn;
    g_force_splits = splits;
    g_force_pair = pair;
}

// Tile width BN (UMMA N) and split-K factor from a cost model of the
// persistent kernel, in SM clocks:
//   per 64-deep K slice   max(MMA 2*BN, smem fill (128 + BN) rows of 128 B) + barrier round trip
//   per tile epilogue     output (+ residual) bytes at ~48 B/clk/SM, overlapping the next mainloop
//   per CTA               ceil(units / 148) x max(mainloop, epilogue) + pipeline fill + last epilogue
//   split-K               + fp32 partial traffic and the reduce kernel
// Tile cost model (SM clocks) of the persistent kernel, calibrated on B200:
//   per 64-deep K slice  max(MMA 2*BN, smem 2*(128 + BNL)) + barrier round trip, where
//                        BNL = B rows staged per CTA (BN, or BN/2 for a CTA pair) and every
//                        staged byte is written by TMA and read by the tensor core through
//                        the 128 B/clk smem port
//   per tile epilogue    output (+ residual) bytes at ~16 B/clk/SM, overlapping the next mainloop
//   per CTA              ceil(units / slots) x max(mainloop, epilogue) + pipeline fill + last epilogue
//   split-K              + fp32 partial traffic and the reduce kernel
double gemm_cost(long long M, int N, int K, int bn, int splits, int out_bytes, bool residual, bool pair) {
    // Constants fitted (tools/fit_tiling.py) to a graph-timed sweep of every (BN, split-K,
    // pair) candidate on the UNet's GEMM / conv shapes at 2, 4 and 8 rows on B200
    // (tools/gemm_sweep.py, SDX_SWEEP_JSON): the objective is the summed measured time of
    // the candidate the model picks, 1.6% above the per-shape optimum.  Cycles:
    //   slice  = one 64-deep K slice through the MMA pipe (floor ~ the per-instruction cost
    //            of tcgen05.mma, which barely grows with N up to 224)
    //   epi    = one tile's epilogue + tile hand-off; both overlap across tiles
    //   split  = fp32 partial traffic and the reduce kernel; pair = cluster overheads
    constexpr double a0 = 411.0, a1 = 1.06, a2 = 1.66, a3 = 31.7;
    constexpr double e0 = 0.016, e1 = 13300.0, c0 = 8830.0, p0 = 10800.0, s0 = 2520.0, s1 = 14.4;
    const long long mu = pair ? 256 : 128;
    const long long slots = pair ? kSmCount / 2 : kSmCount;
    const long long mt = (M + mu - 1) / mu, nt = (N + bn - 1) / bn;
    const long long units = mt * nt * splits;
    const int nk = K / 64;
    const double bnl = pair ? bn / 2.0 : bn;
    const double nku = static_cast<double>((nk + splits - 1) / splits);
    const double slice = std::max({a0, a1 * bn, a2 * (128.0 + bnl)}) + a3;
    const double ml = nku * slice;
    const double eb = splits > 1 ? 4.0 : out_bytes + (residual ? 2.0 : 0.0);
    const double epi = e0 * 128.0 * bn * eb / 16.0 + e1;
    const double per_cta = static_cast<double>((units + slots - 1) / slots);
    double t = per_cta * std::max(ml, epi) + c0 + std::min(ml, epi);
    if (pair) t += p0;
    if (splits > 1) {
        const double bytes = static_cast<double>(M) * N * (4.0 * splits + out_bytes + (residual ? 2.0 : 0.0));
        t += s0 + bytes / (kSmCount * s1);
    }
    return t;
}

namespace {
bool aligned16(const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; }

// Epilogue the plan can use: 0 general, 1 fast bf16, 2 fast GEGLU, 3 fast split-K partials.
// Fast: bf16 output (or fp32 partials), N % 32 == 0, no scatter, activation none or
// ReLU, 16-byte aligned vectors.
int epilogue_kind(const GemmPlan& p, int splits) {
    const GemmEpilogue& e = p.epi;
    if (p.N % 32 != 0) return 0;
    if (splits > 1) return 3;
    if (e.out_f32 != 0 || e.out_img_map) return 0;
    if (e.act != kActNone && e.act != kActRelu) return 0;
    if (e.ld_out % 8 != 0 || !aligned16(e.out)) return 0;
    if (e.geglu) {
        if (p.N % 64 != 0 || e.residual || e.bias_img || e.act != kActNone || (e.bias && !aligned16(e.bias))) return 0;
        return 2;
    }
    if (e.residual && (e.ld_res % 8 != 0 || !aligned16(e.residual))) return 0;
    if (e.bias && !aligned16(e.bias)) return 0;
    if (e.bias_img && (!aligned16(e.bias_img) || (e.bias_img_ld ? e.bias_img_ld : p.N) % 4 != 0)) return 0;
    return 1;
}
}  // namespace

// Tile width, split-K factor and CTA pairing from gemm_cost.  CTA pairs need the
// fast epilogue; GEGLU and LayerNorm-folded GEMMs stay single-pass (no split-K).
void choose_tiling(GemmPlan& p) {
    static const int cand[] = {64, 96, 128, 160, 192, 224, 256};
    const int nk = p.K / 64;
    const int out_bytes = p.epi.out_f32 == 1 ? 4 : (p.epi.out_f32 == 2 ? 1 : 2);
    const bool res = p.epi.residual != nullptr;
    const bool single = p.epi.geglu || p.epi.ln_part || p.epi.row_stats_out;
    static const bool pair_on = [] {
        const char* v = std::getenv("SDX_GEMM_PAIR");
        return !(v && v[0] == '0');
    }();
    int best_bn = 64, best_s = 1;
    bool best_pair = false;
    double best = -1.0;
    for (int pr = 0; pr < 2; ++pr) {
        if (pr && !pair_on) break;
        for (int bn : cand) {
            if (p.N <= 64 && bn > 64) break;
            if (pr && bn < 128) continue;
            const int smax = single ? 1 : (nk / 4 < 16 ? nk / 4 : 16);
            for (int s = 1; s <= (smax > 1 ? smax : 1); ++s) {
                if (pr && epilogue_kind(p, s) == 0) continue;
                // CTA pairs only for long-K layers: measured on the UNet shapes (tools/gemm_sweep.py)
                // they win for K >= 11520 (1280+ input channels of a 3x3 conv) and lose 10-20%
                // below that (cluster launch / sync overheads outweigh the halved B traffic)
                if (pr && p.K < 11520) continue;
                const double c = gemm_cost(p.M, p.N, p.K, bn, s, out_bytes, res, pr != 0);
                if (best < 0 || c < best * 0.999) {
                    best = c;
                    best_bn = bn;
                    best_s = s;
                    best_pair = pr != 0;
                }
            }
        }
    }
    if (g_force_bn) {
        best_bn = g_force_bn;
        best_pair = g_force_pair && best_bn >= 128 && best_bn % 32 == 0;
    }
    if (g_force_splits) best_s = g_force_splits;
    if (best_pair && epilogue_kind(p, best_s) == 0) best_pair = false;
    p.bn = best_bn;
    p.splits = best_s;
    p.pair = best_pair;
    if (p.splits > 1) {
        float* ws = dev_alloc<float>(static_cast<size_t>(p.splits) * p.M * p.N);
        p.ws = ws;
        p.ws_owner = std::shared_ptr<void>(ws, [](void* q) { cudaFree(q); });
    }
}

// Output tensor map of the fast epilogue (if the plan qualifies).
void choose_epilogue_impl(GemmPlan& p) {
    const GemmEpilogue& e = p.epi;
    const int kind = epilogue_kind(p, p.splits);
    p.fast = kind != 0;
    if (kind == 3) {
        const cuuint64_t dims[3] = {static_cast<cuuint64_t>(p.N), static_cast<cuuint64_t>(p.M),
                                    static_cast<cuuint64_t>(p.splits)};
        const cuuint64_t strides[2] = {static_cast<cuuint64_t>(p.N) * 4, static_cast<cuuint64_t>(p.M) * p.N * 4};
        const cuuint32_t box[3] = {16, 32, 1};
        const cuuint32_t es[3] = {1, 1, 1};
        encode(&p.to, p.ws, 3, dims, strides, box, es, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, CU_TENSOR_MAP_SWIZZLE_64B);
    } else if (kind == 2) {
        const cuuint64_t dims[2] = {static_cast<cuuint64_t>(p.N / 2), static_cast<cuuint64_t>(p.M)};
        const cuuint64_t strides[1] = {static_cast<cuuint64_t>(e.ld_out) * 2};
        const cuuint32_t box[2] = {16, 32};
        const cuuint32_t es[2] = {1, 1};
        encode(&p.to, e.out, 2, dims, strides, box, es, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, CU_TENSOR_MAP_SWIZZLE_32B);
    } else if (kind == 1) {
        const cuuint64_t dims[2] = {static_cast<cuuint64_t>(p.N), static_cast<cuuint64_t>(p.M)};
        const cuuint64_t strides[1] = {static_cast<cuuint64_t>(e.ld_out) * 2};
        const cuuint32_t box[2] = {32, 32};
        const cuuint32_t es[2] = {1, 1};
        encode(&p.to, e.out, 2, dims, strides, box, es, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, CU_TENSOR_MAP_SWIZZLE_64B);
    }
    if (p.pair && !p.fast) raise(SDX_LOGIC_ERROR, "gemm: CTA pair without the fast epilogue");
}

void choose_epilogue(GemmPlan& p) {
    choose_epilogue_impl(p);
    if ((p.epi.ln_part || p.epi.row_stats_out) && !(p.fast && p.splits == 1))
        raise(SDX_INVALID_ARGUMENT, "gemm: LayerNorm folding needs the fast single-pass epilogue");
}

GemmPlan plan_gemm(const __nv_bfloat16* A, long long lda, const __nv_bfloat16* B, long long ldb, int M, int N, int K,
                   const GemmEpilogue& epi) {
    if (K % 64 != 0) raise(SDX_INVALID_ARGUMENT, "gemm: K must be a multiple of 64");
    if (epi.geglu && epi.residual) raise(SDX_INVALID_ARGUMENT, "gemm: GEGLU epilogue takes no residual");
    GemmPlan p;
    p.amode = kAMatrix;
    p.M = M;
    p.N = N;
    p.K = K;
    p.epi = epi;
    if (p.epi.ld_out == 0) p.epi.ld_out = N;
    if (p.epi.residual && p.epi.ld_res == 0) p.epi.ld_res = N;
    choose_tiling(p);
    encode_2d(&p.ta, A, M, K, lda, 128);
    p.ta2 = p.ta;
    encode_2d(&p.tb, B, N, K, ldb, p.pair ? p.bn / 2 : p.bn);
    choose_epilogue(p);
    p.valid = true;
    return p;
}

GemmPlan plan_gemm_concat(const __nv_bfloat16* A1, long long lda1, int K1, const __nv_bfloat16* A2, long long lda2,
                          const __nv_bfloat16* B, long long ldb, int M, int N, int K, const GemmEpilogue& epi) {
    if (K % 64 != 0 || K1 % 64 != 0) raise(SDX_INVALID_ARGUMENT, "gemm: K, K1 must be multiples of 64");
    GemmPlan p;
    p.amode = kAConcat;
    p.M = M;
    p.N = N;
    p.K = K;
    p.K1 = K1;
    p.epi = epi;
    if (p.epi.ld_out == 0) p.epi.ld_out = N;
    if (p.epi.residual && p.epi.ld_res == 0) p.epi.ld_res = N;
    choose_tiling(p);
    encode_2d(&p.ta, A1, M, K1, lda1, 128);
    encode_2d(&p.ta2, A2, M, K - K1, lda2, 128);
    encode_2d(&p.tb, B, N, K, ldb, p.pair ? p.bn / 2 : p.bn);
    choose_epilogue(p);
    p.valid = true;
    return p;
}

GemmPlan plan_conv3x3(const __nv_bfloat16* x, int imgs, int H, int W, int Cin, const __nv_bfloat16* w, int Cout,
                      int stride, const GemmEpilogue& epi) {
    if (Cin % 64 != 0) raise(SDX_INVALID_ARGUMENT, "conv3x3: Cin must be a multiple of 64");
    if (stride != 1 && stride != 2) raise(SDX_INVALID_ARGUMENT, "conv3x3: stride must be 1 or 2");
    GemmPlan p;
    p.amode = kAConv;
    p.H = H;
    p.W = W;
    p.Cin = Cin;
    p.stride = stride;
    p.Ho = stride == 1 ? H : (H + 1) / 2;
    p.Wo = stride == 1 ? W : (W + 1) / 2;
    p.Wt = p.Wo < 128 ? p.Wo : 128;
    if (128 % p.Wt != 0 || (p.Wo > 128 && p.Wo % 128 != 0))
        raise(SDX_INVALID_ARGUMENT, "conv3x3: output width must divide or be a multiple of 128");
    p.Ht = 128 / p.Wt;
    if (p.Ht > p.Ho) p.Ht = p.Ho;
    p.Nt = 128 / (p.Wt * p.Ht);
    if (p.Wt * p.Ht * p.Nt != 128 || (p.Ho % p.Ht) != 0)
        raise(SDX_INVALID_ARGUMENT, "conv3x3: unsupported output tile geometry");
    p.M = imgs * p.Ho * p.Wo;
    p.N = Cout;
    p.K = 9 * Cin;
    p.epi = epi;
    if (p.epi.ld_out == 0) p.epi.ld_out = Cout;
    if (p.epi.residual && p.epi.ld_res == 0) p.epi.ld_res = Cout;
    choose_tiling(p);
    const cuuint64_t dims[4] = {static_cast<cuuint64_t>(Cin), static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H),
                                static_cast<cuuint64_t>(imgs)};
    const cuuint64_t strides[3] = {static_cast<cuuint64_t>(Cin) * 2, static_cast<cuuint64_t>(W) * Cin * 2,
                                   static_cast<cuuint64_t>(H) * W * Cin * 2};
    const cuuint32_t box[4] = {64, static_cast<cuuint32_t>(p.Wt * stride), static_cast<cuuint32_t>(p.Ht * stride),
                               static_cast<cuuint32_t>(p.Nt)};
    const cuuint32_t es[4] = {1, static_cast<cuuint32_t>(stride), static_cast<cuuint32_t>(stride), 1};
    encode(&p.ta, x, 4, dims, strides, box, es);
    p.ta2 = p.ta;
    encode_2d(&p.tb, w, Cout, 9LL * Cin, 9LL * Cin, p.pair ? p.bn / 2 : p.bn);
    choose_epilogue(p);
    static const bool halo_on = [] {
        const char* v = std::getenv("SDX_CONV_HALO");
        return !(v && v[0] == '0');
    }();
    const bool halo_epi_ok = p.fast ? Cout == 64 : (p.epi.n_gn == 0 && !p.epi.geglu);  // narrow heads: general epilogue
    if (halo_on && Cin == 64 && Cout <= 64 && stride == 1 && W % 128 == 0 && halo_epi_ok && !p.epi.ln_part &&
        !p.epi.row_stats_out && g_force_bn == 0) {
        // halo-tiled: 128-pixel row segments, one 3 x 130 x 64 box per tile, resident weights
        p.amode = kAHalo;
        p.bn = 64;
        p.splits = 1;
        p.pair = false;
        p.ws = nullptr;
        p.ws_owner.reset();
        const cuuint32_t hbox[4] = {64, 130, 3, 1};
        const cuuint32_t hes[4] = {1, 1, 1, 1};
        encode(&p.ta, x, 4, dims, strides, hbox, hes);
        encode_2d(&p.tb, w, Cout, 9LL * Cin, 9LL * Cin, 64);
        choose_epilogue(p);
    }
    p.valid = true;
    return p;
}

void run_gemm(const GemmPlan& p, cudaStream_t st) {
    if (!p.valid) raise(SDX_LOGIC_ERROR, "run_gemm: invalid plan");
    if (p.amode == kAHalo) {
        if (p.fast) launch_t<64, kAHalo, true, false>(p, st);
        else launch_t<64, kAHalo, false, false>(p, st);
        return;
    }
    if (p.fast) {
        switch (p.amode) {
            case kAConcat: launch_mode<kAConcat, true>(p, st); break;
            case kAConv: launch_mode<kAConv, true>(p, st); break;
            default: launch_mode<kAMatrix, true>(p, st); break;
        }
    } else {
        switch (p.amode) {
            case kAConcat: launch_mode<kAConcat, false>(p, st); break;
            case kAConv: launch_mode<kAConv, false>(p, st); break;
            default: launch_mode<kAMatrix, false>(p, st); break;
        }
    }
}

}  // namespace sdx
