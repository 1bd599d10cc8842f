// HBM-bound helper kernels of the UNet / TAESD forward: GroupNorm (+SiLU,
// +channel concat), LayerNorm, GEGLU, nearest upsample, small-channel
// im2col, timestep embedding, initialisers.  All vectorised over 8 bf16
// channels (16 B) of NHWC activations; statistics in fp32.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "nn_kernels.cuh"

namespace sdx {

namespace {

__device__ __forceinline__ void load8(const bf16* p, float* v) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(h[i]);
        v[2 * i] = f.x;
        v[2 * i + 1] = f.y;
    }
}

__device__ __forceinline__ void unpack8(const uint4& u, float* v) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(h[i]);
        v[2 * i] = f.x;
        v[2 * i + 1] = f.y;
    }
}

// GroupNorm statistics of one octet: per-channel sum and sum of squares (3
// instructions per value; the split into the octet's <= 2 groups is done once).
__device__ __forceinline__ void gn_acc8(const uint4& u, float* as, float* aq) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float lo = __uint_as_float(w[i] << 16), hi = __uint_as_float(w[i] & 0xffff0000u);
        as[2 * i] += lo;
        aq[2 * i] = fmaf(lo, lo, aq[2 * i]);
        as[2 * i + 1] += hi;
        aq[2 * i + 1] = fmaf(hi, hi, aq[2 * i + 1]);
    }
}
__device__ __forceinline__ void gn_split8(const float* as, const float* aq, int split, float& s0, float& q0, float& s1,
                                          float& q1) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        if (i < split) {
            s0 += as[i];
            q0 += aq[i];
        } else {
            s1 += as[i];
            q1 += aq[i];
        }
    }
}

// y = GN(x) -> (SiLU) for 8 values: SiLU(y) = y * (0.5 + 0.5 tanh(y / 2)) with one
// packed tanh.approx.f16x2 per 2 values (the SFU pipe, 16 ops/clk/SM, bounds the
// apply pass with exp + reciprocal); |rel err| ~1e-3, below the bf16 output rounding.
__device__ __forceinline__ void gn_affine8(float* v, const float* sc, const float* sh, int silu) {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = fmaf(v[i], sc[i], sh[i]);
    if (!silu) return;
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
        const __half2 h = __floats2half2_rn(0.5f * v[i], 0.5f * v[i + 1]);
        uint32_t hu = *reinterpret_cast<const uint32_t*>(&h), tu;
        asm("tanh.approx.f16x2 %0, %1;" : "=r"(tu) : "r"(hu));
        const float2 t = __half22float2(*reinterpret_cast<const __half2*>(&tu));
        v[i] *= fmaf(0.5f, t.x, 0.5f);
        v[i + 1] *= fmaf(0.5f, t.y, 0.5f);
    }
}

__device__ __forceinline__ void store8(bf16* p, const float* v) {
    uint4 u;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    *reinterpret_cast<uint4*>(p) = u;
}

// ---- GroupNorm ----------------------------------------------------------------

// Thread layout of both GroupNorm kernels: blockDim = noct x PY, thread
// (ox, py) owns channel octet ox (8 channels, <= 2 groups since Ct/32 >= 8) and
// walks the pixels py, py + PY, ... of its block's pixel range, 8 independent
// 16-byte loads in flight.
__device__ __forceinline__ const bf16* gn_src(const GnPlan& p, int img, int px, int c) {
    return c < p.C1 ? p.x1 + (static_cast<long long>(img) * p.HW + px) * p.C1 + c
                    : p.x2 + (static_cast<long long>(img) * p.HW + px) * p.C2 + (c - p.C1);
}

// Statistics: per block fp32 sums over its pixel range (fixed-order smem
// reduction), then one 2^-20 fixed-point int64 atomic per (group, moment) into
// p.acc — integer adds are associative, so the totals are deterministic and no
// block has to wait for the others.
// Statistics of this block's pixel range: fp32 partial sums (fixed-order smem
// reduction), then one 2^-20 fixed-point int64 atomic per (group, moment) into
// p.acc — integer adds are associative, so the totals are deterministic.
__device__ __forceinline__ void gn_block_stats(const GnPlan& p, int img, float* sm) {
    const int Ct = p.C1 + p.C2;
    const int noct = Ct / 8;
    const int PY = blockDim.x / noct;
    const int ox = threadIdx.x % noct, py = threadIdx.x / noct;
    const int cg = Ct / p.groups;
    const int c = ox * 8;
    const int g0 = c / cg, split = (g0 + 1) * cg - c;
    const int px0 = blockIdx.x * p.px_per_block;
    const int px1 = min(p.HW, px0 + p.px_per_block);
    float as[8] = {}, aq[8] = {};  // per-channel sums; split into the <= 2 groups once at the end
    if (py < PY) {
        for (int base = px0 + py; base < px1; base += 8 * PY) {
            uint4 raw[8];  // packed bf16: 32 registers for 8 loads in flight
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int px = base + k * PY;
                raw[k] = px < px1 ? *reinterpret_cast<const uint4*>(gn_src(p, img, px, c)) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) gn_acc8(raw[k], as, aq);
        }
    }
    float s0 = 0.f, q0 = 0.f, s1 = 0.f, q1 = 0.f;
    gn_split8(as, aq, split, s0, q0, s1, q1);
    // fixed-order reduction: per octet over pixel lanes, then per group over octets
    float* mine = sm + (static_cast<long long>(py) * noct + ox) * 4;
    if (py < PY) {
        mine[0] = s0;
        mine[1] = q0;
        mine[2] = s1;
        mine[3] = q1;
    }
    __syncthreads();
    float red[4] = {0.f, 0.f, 0.f, 0.f};
    if (threadIdx.x < noct)
        for (int y = 0; y < PY; ++y)
            for (int j = 0; j < 4; ++j) red[j] += sm[(static_cast<long long>(y) * noct + threadIdx.x) * 4 + j];
    __syncthreads();
    if (threadIdx.x < noct)
        for (int j = 0; j < 4; ++j) sm[threadIdx.x * 4 + j] = red[j];
    __syncthreads();
    for (int g = threadIdx.x; g < p.groups; g += blockDim.x) {
        float a = 0.f, b = 0.f;
        const int o0 = (g * cg) / 8, o1 = ((g + 1) * cg - 1) / 8;
        for (int o = o0; o <= o1; ++o) {
            const int og0 = (o * 8) / cg;
            const int part = og0 == g ? 0 : 2;  // this octet's first or second group
            a += sm[o * 4 + part];
            b += sm[o * 4 + part + 1];
        }
        unsigned long long* acc = p.acc + (static_cast<long long>(img) * p.groups + g) * 2;
        atomicAdd(acc, static_cast<unsigned long long>(__float2ll_rn(a * 1048576.f)));
        atomicAdd(acc + 1, static_cast<unsigned long long>(__float2ll_rn(b * 1048576.f)));
    }
}

// y = GN(x) (+ SiLU) over this block's pixel range, (mean, rstd) in fp64 from the sums.
// The first batch of pixels is requested before the group statistics are derived,
// so the load latency overlaps the fp64 math and the barrier.
__device__ __forceinline__ void gn_block_apply(const GnPlan& p, int img, float (*st)[2]) {
    const int Ct = p.C1 + p.C2;
    const int noct = Ct / 8;
    const int PY = blockDim.x / noct;
    const int ox = threadIdx.x % noct, py = threadIdx.x / noct;
    const int cg = Ct / p.groups;
    const int c = ox * 8;
    const int px0 = blockIdx.x * p.px_per_block;
    const int px1 = min(p.HW, px0 + p.px_per_block);
    uint4 raw[8];  // packed bf16
    int base = px0 + py;
    if (py < PY) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int px = base + k * PY;
            if (px < px1) raw[k] = *reinterpret_cast<const uint4*>(gn_src(p, img, px, c));
        }
    }
    for (int g = threadIdx.x; g < p.groups; g += blockDim.x) {
        const double inv = 1.0 / 1048576.0;
        const double n = static_cast<double>(cg) * p.HW;
        const unsigned long long* acc = p.acc + (static_cast<long long>(img) * p.groups + g) * 2;
        const double m = static_cast<double>(static_cast<long long>(__ldcg(acc))) * inv / n;
        double var = static_cast<double>(static_cast<long long>(__ldcg(acc + 1))) * inv / n - m * m;
        if (var < 0) var = 0;
        st[g][0] = static_cast<float>(m);
        st[g][1] = static_cast<float>(1.0 / sqrt(var + p.eps));
    }
    __syncthreads();
    if (py >= PY) return;
    const int g0 = c / cg, split = (g0 + 1) * cg - c;
    const float m0 = st[g0][0], r0 = st[g0][1];
    const float m1 = split < 8 ? st[g0 + 1][0] : 0.f, r1 = split < 8 ? st[g0 + 1][1] : 0.f;
    float sc[8], sh[8];  // y = x * sc + sh
    {
        const float4 ga = *reinterpret_cast<const float4*>(p.gamma + c), gb = *reinterpret_cast<const float4*>(p.gamma + c + 4);
        const float4 ba = *reinterpret_cast<const float4*>(p.beta + c), bb = *reinterpret_cast<const float4*>(p.beta + c + 4);
        const float gam[8] = {ga.x, ga.y, ga.z, ga.w, gb.x, gb.y, gb.z, gb.w};
        const float bet[8] = {ba.x, ba.y, ba.z, ba.w, bb.x, bb.y, bb.z, bb.w};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float m = i < split ? m0 : m1, r = i < split ? r0 : r1;
            sc[i] = r * gam[i];
            sh[i] = bet[i] - m * r * gam[i];
        }
    }
    while (true) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int px = base + k * PY;
            if (px >= px1) continue;
            float v[8];
            unpack8(raw[k], v);
            gn_affine8(v, sc, sh, p.silu);
            store8(p.out + (static_cast<long long>(img) * p.HW + px) * Ct + c, v);
        }
        base += 8 * PY;
        if (base >= px1) break;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int px = base + k * PY;
            if (px < px1) raw[k] = *reinterpret_cast<const uint4*>(gn_src(p, img, px, c));
        }
    }
}

__global__ void __launch_bounds__(320, 3) gn_stats_kernel(GnPlan p) {
    pdl_launch();
    pdl_wait();
    const int img = blockIdx.y;
    if (p.rows_dev && img >= *p.rows_dev) return;
    extern __shared__ float sm[];  // [PY][noct][4]
    gn_block_stats(p, img, sm);
}

__global__ void __launch_bounds__(320, 3) gn_apply_kernel(GnPlan p) {
    pdl_launch();
    pdl_wait();
    const int img = blockIdx.y;
    if (p.rows_dev && img >= *p.rows_dev) return;
    __shared__ float st[64][2];
    gn_block_apply(p, img, st);
}

// Statistics and apply in one launch: every block adds its partial sums, then
// waits on a grid-wide arrival counter (zeroed with the statistics arena before
// each forward) until all blocks have added theirs.  The plan sizes the grid
// to be co-resident (occupancy-checked), so the wait cannot deadlock; phase 2
// re-reads the tensor from L2.
__global__ void __launch_bounds__(320) gn_fused_kernel(GnPlan p) {
    pdl_launch();
    pdl_wait();
    const int img = blockIdx.y;
    const bool live = !(p.rows_dev && img >= *p.rows_dev);
    extern __shared__ float sm[];  // [PY][noct][4]
    if (live) gn_block_stats(p, img, sm);
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(p.counter, 1ull);
        const unsigned long long target = static_cast<unsigned long long>(gridDim.x) * gridDim.y;
        if (live) {
            const long long t0 = clock64();
            while (true) {
                unsigned long long v;
                asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p.counter) : "memory");
                if (v >= target) break;
                __nanosleep(64);
                if (clock64() - t0 > (1LL << 34)) {
                    printf("sdx groupnorm: grid barrier watchdog (block %d,%d)\n", blockIdx.x, blockIdx.y);
                    asm volatile("trap;");
                }
            }
        }
    }
    __syncthreads();
    if (!live) return;
    gn_block_apply(p, img, reinterpret_cast<float (*)[2]>(sm));
}

// One launch per GroupNorm, one thread-block cluster per image.  Each CTA owns
// a contiguous pixel range of its image and streams it through two 100 KB
// shared-memory buffers with bulk async copies (cp.async.bulk, mbarrier
// completion; x1 and x2 rows are each one contiguous block), summing
// (sum, sum of squares) per channel octet.  The block's per-group partials
// (fixed-order fp32 reduction) are published by a cluster barrier; every CTA
// adds the cluster's partials of each group in rank order over DSMEM in fp64,
// so all CTAs derive bit-identical statistics.  The apply pass reads the range
// from shared memory when it fit (<= 2 pieces) or streams it again (L2), and
// stores y = GN(x) (+ SiLU) with 16-byte vector stores.  No statistics arena,
// no atomics, no second launch.
constexpr int kGnBufBytes = 100 * 1024;

__device__ __forceinline__ float ld_dsmem_f32(const float* local, uint32_t rank) {
    uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(local)), r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    float v;
    // not volatile: independent remote loads may be issued back to back (ordering against
    // the partials' producers comes from the cluster barrier before the first call)
    asm("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(r));
    return v;
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src), "r"(bytes), "r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
                 : "memory");
}

__device__ __forceinline__ void gn_mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "GNW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 10000000;\n\t"
        "@!p bra GNW_%=;\n\t}" ::"r"(a),
        "r"(parity)
        : "memory");
}

__global__ void __launch_bounds__(320, 1) gn_cluster_kernel(GnPlan p) {
    extern __shared__ __align__(128) uint8_t gbuf[];  // [2][kGnBufBytes]
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ float sm[320 * 4];
    __shared__ float gpart[64];  // this CTA's (sum, sum of squares) per group
    __shared__ float st[32][2];
    pdl_launch();
    long long* dbg = (p.dbg && threadIdx.x == 0) ? p.dbg + (blockIdx.y * gridDim.x + blockIdx.x) * 8 : nullptr;
    auto stamp = [&](int i) {
        if (dbg) {
            long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t) : : "memory");
            dbg[i] = t;
        }
    };
    stamp(0);
    const int img = blockIdx.y;
    const int Ct = p.C1 + p.C2;
    const int noct = Ct / 8;
    const int PY = blockDim.x / noct;
    const int ox = threadIdx.x % noct, py = threadIdx.x / noct;
    const int cg = Ct / p.groups;
    const int c = ox * 8;
    const int g0 = c / cg, split = (g0 + 1) * cg - c;
    const int px0 = blockIdx.x * p.px_per_block;
    const int px1 = min(p.HW, px0 + p.px_per_block);
    const int npx = max(0, px1 - px0);
    const int P = p.piece;
    const int np = (npx + P - 1) / P;
    const bool resident = np <= 2;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(&bar[0]))));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(&bar[1]))));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    pdl_wait();
    stamp(1);
    if (p.rows_dev && img >= *p.rows_dev) return;  // the whole cluster shares the image
    // load sequence number L: buffer L & 1, parity (L >> 1) & 1; phase A loads the
    // pieces as L = 0 .. np-1, a non-resident phase B again as L = np .. 2np-1
    auto issue = [&](int L, int piece) {
        const int a0 = px0 + piece * P;
        const int n = min(P, px1 - a0);
        uint8_t* dst = gbuf + (L & 1) * kGnBufBytes;
        const uint32_t b1 = static_cast<uint32_t>(n) * p.C1 * 2, b2 = static_cast<uint32_t>(n) * p.C2 * 2;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(&bar[L & 1]))),
                     "r"(b1 + b2)
                     : "memory");
        bulk_g2s(dst, p.x1 + (static_cast<long long>(img) * p.HW + a0) * p.C1, b1, &bar[L & 1]);
        if (p.C2) bulk_g2s(dst + b1, p.x2 + (static_cast<long long>(img) * p.HW + a0) * p.C2, b2, &bar[L & 1]);
    };
    // this thread's octet of local pixel pl of a piece of n pixels in buffer buf,
    // and the byte step to pixel pl + PY
    const bool in1 = c < p.C1;
    auto octet_ptr = [&](const uint8_t* buf, int n, int pl) -> const uint8_t* {
        return in1 ? buf + (pl * p.C1 + c) * 2 : buf + (n * p.C1 + pl * p.C2 + (c - p.C1)) * 2;
    };
    auto octet_step = [&](int) -> int { return PY * (in1 ? p.C1 : p.C2) * 2; };
    if (threadIdx.x == 0) {
        if (np > 0) issue(0, 0);
        if (np > 1) issue(1, 1);
    }
    float as[8] = {}, aq[8] = {};
    for (int i = 0; i < np; ++i) {
        gn_mbar_wait(&bar[i & 1], (i >> 1) & 1);
        if (i == 0) stamp(2);
        const uint8_t* buf = gbuf + (i & 1) * kGnBufBytes;
        const int n = min(P, px1 - (px0 + i * P));
        const uint8_t* q = octet_ptr(buf, n, py);
        const int step = octet_step(n);
        for (int pl = py; pl < n; pl += PY, q += step) gn_acc8(*reinterpret_cast<const uint4*>(q), as, aq);
        if (!resident) {
            __syncthreads();  // buffer consumed
            if (threadIdx.x == 0) {
                if (i + 2 < np) issue(i + 2, i + 2);
                else issue(i + 2, i + 2 - np);  // phase B's first two pieces
            }
        }
    }
    float s0 = 0.f, q0 = 0.f, s1 = 0.f, q1 = 0.f;
    gn_split8(as, aq, split, s0, q0, s1, q1);
    float* mine = sm + (py * noct + ox) * 4;
    mine[0] = s0;
    mine[1] = q0;
    mine[2] = s1;
    mine[3] = q1;
    __syncthreads();
    float red[4] = {0.f, 0.f, 0.f, 0.f};
    if (threadIdx.x < noct)
        for (int y = 0; y < PY; ++y)
            for (int j = 0; j < 4; ++j) red[j] += sm[(y * noct + threadIdx.x) * 4 + j];
    __syncthreads();
    if (threadIdx.x < noct)
        for (int j = 0; j < 4; ++j) sm[threadIdx.x * 4 + j] = red[j];
    __syncthreads();
    for (int g = threadIdx.x; g < p.groups; g += blockDim.x) {
        float a = 0.f, b = 0.f;
        const int o0 = (g * cg) / 8, o1 = ((g + 1) * cg - 1) / 8;
        for (int o = o0; o <= o1; ++o) {
            const int part = (o * 8) / cg == g ? 0 : 2;
            a += sm[o * 4 + part];
            b += sm[o * 4 + part + 1];
        }
        gpart[2 * g] = a;
        gpart[2 * g + 1] = b;
    }
    stamp(3);
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    stamp(4);
    if (threadIdx.x < p.groups) {
        const int g = threadIdx.x;
        // all ranks' partials requested at once (independent DSMEM loads, <= 16 ranks), then
        // added in rank order: one remote round trip instead of one per rank
        float pa[16], pb[16];
        const uint32_t nr = gridDim.x;  // grid.x == cluster size
#pragma unroll
        for (uint32_t r = 0; r < 16; ++r) {
            pa[r] = r < nr ? ld_dsmem_f32(&gpart[2 * g], r) : 0.f;
            pb[r] = r < nr ? ld_dsmem_f32(&gpart[2 * g + 1], r) : 0.f;
        }
        double a = 0.0, b = 0.0;
#pragma unroll
        for (uint32_t r = 0; r < 16; ++r) {
            a += static_cast<double>(pa[r]);
            b += static_cast<double>(pb[r]);
        }
        const double n = static_cast<double>(cg) * p.HW;
        const double m = a / n;
        double var = b / n - m * m;
        if (var < 0) var = 0;
        st[g][0] = static_cast<float>(m);
        st[g][1] = static_cast<float>(1.0 / sqrt(var + p.eps));
    }
    // remote reads issued: release the partials (the matching wait is at exit)
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    __syncthreads();
    stamp(5);
    const float m0 = st[g0][0], r0 = st[g0][1];
    const float m1 = split < 8 ? st[g0 + 1][0] : 0.f, r1 = split < 8 ? st[g0 + 1][1] : 0.f;
    float sc[8], sh[8];
    {
        const float4 ga = *reinterpret_cast<const float4*>(p.gamma + c), gb = *reinterpret_cast<const float4*>(p.gamma + c + 4);
        const float4 ba = *reinterpret_cast<const float4*>(p.beta + c), bb = *reinterpret_cast<const float4*>(p.beta + c + 4);
        const float gam[8] = {ga.x, ga.y, ga.z, ga.w, gb.x, gb.y, gb.z, gb.w};
        const float bet[8] = {ba.x, ba.y, ba.z, ba.w, bb.x, bb.y, bb.z, bb.w};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float m = i < split ? m0 : m1, r = i < split ? r0 : r1;
            sc[i] = r * gam[i];
            sh[i] = bet[i] - m * r * gam[i];
        }
    }
    for (int i = 0; i < np; ++i) {
        const int L = resident ? i : np + i;
        if (!resident) gn_mbar_wait(&bar[L & 1], (L >> 1) & 1);
        const uint8_t* buf = gbuf + (L & 1) * kGnBufBytes;
        const int a0 = px0 + i * P;
        const int n = min(P, px1 - a0);
        const uint8_t* q = octet_ptr(buf, n, py);
        const int step = octet_step(n);
        bf16* o = p.out + (static_cast<long long>(img) * p.HW + a0 + py) * Ct + c;
        for (int pl = py; pl < n; pl += PY, q += step, o += static_cast<long long>(PY) * Ct) {
            float v[8];
            unpack8(*reinterpret_cast<const uint4*>(q), v);
            gn_affine8(v, sc, sh, p.silu);
            store8(o, v);
        }
        if (!resident && i + 2 < np) {
            __syncthreads();
            if (threadIdx.x == 0) issue(L + 2, i + 2);
        }
    }
    stamp(6);
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    stamp(7);
}

// ---- LayerNorm (one warp per row) ------------------------------------------------

template <int MAXV>
__global__ void layernorm_kernel(const bf16* __restrict__ x, int rows, int C, const float* __restrict__ gamma,
                                 const float* __restrict__ beta, float eps, bf16* __restrict__ out,
                                 const int* rows_dev, int rows_per_unit) {
    pdl_launch();
    pdl_wait();
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    int lim = rows;
    if (rows_dev) lim = min(lim, *rows_dev * rows_per_unit);
    if (warp >= lim) return;
    const bf16* xr = x + static_cast<long long>(warp) * C;
    const int noct = C / 8;
    float v[MAXV][8];
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < MAXV; ++k) {
        const int o = lane + 32 * k;
        if (o < noct) {
            load8(xr + o * 8, v[k]);
#pragma unroll
            for (int i = 0; i < 8; ++i) s += v[k][i];
        }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    const float mean = s / C;
    float q = 0.f;
#pragma unroll
    for (int k = 0; k < MAXV; ++k) {
        const int o = lane + 32 * k;
        if (o < noct) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const float d = v[k][i] - mean;
                q += d * d;
            }
        }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) q += __shfl_xor_sync(0xffffffffu, q, off);
    const float rstd = rsqrtf(q / C + eps);
    bf16* orow = out + static_cast<long long>(warp) * C;
#pragma unroll
    for (int k = 0; k < MAXV; ++k) {
        const int o = lane + 32 * k;
        if (o < noct) {
            float y[8];
#pragma unroll
            for (int i = 0; i < 8; i += 4) {
                const float4 gm = *reinterpret_cast<const float4*>(gamma + o * 8 + i);
                const float4 bt = *reinterpret_cast<const float4*>(beta + o * 8 + i);
                y[i] = (v[k][i] - mean) * rstd * gm.x + bt.x;
                y[i + 1] = (v[k][i + 1] - mean) * rstd * gm.y + bt.y;
                y[i + 2] = (v[k][i + 2] - mean) * rstd * gm.z + bt.z;
                y[i + 3] = (v[k][i + 3] - mean) * rstd * gm.w + bt.w;
            }
            store8(orow + o * 8, y);
        }
    }
}

// ---- GEGLU ----------------------------------------------------------------------

__global__ void geglu_kernel(const bf16* __restrict__ in, int rows, int H, bf16* __restrict__ out,
                             const int* rows_dev, int rows_per_unit) {
    pdl_launch();
    pdl_wait();
    int lim = rows;
    if (rows_dev) lim = min(lim, *rows_dev * rows_per_unit);
    const int noct = H / 8;
    const long long total = static_cast<long long>(lim) * noct;
    for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long r = idx / noct;
        const int c = static_cast<int>(idx % noct) * 8;
        float a[8], g[8], y[8];
        load8(in + r * 2 * H + c, a);
        load8(in + r * 2 * H + H + c, g);
#pragma unroll
        for (int i = 0; i < 8; ++i) y[i] = a[i] * 0.5f * g[i] * (1.f + erff(g[i] * 0.70710678118654752f));
        store8(out + r * H + c, y);
    }
}

// ---- nearest upsample -------------------------------------------------------------

__global__ void upsample_kernel(const bf16* __restrict__ in, int imgs, int H, int W, int C, bf16* __restrict__ out,
                                const int* rows_dev) {
    pdl_launch();
    pdl_wait();
    int lim = imgs;
    if (rows_dev) lim = min(lim, *rows_dev);
    const int noct = C / 8;
    const long long total = static_cast<long long>(lim) * 4 * H * W * noct;
    for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(idx % noct) * 8;
        long long pix = idx / noct;
        const int ox = static_cast<int>(pix % (2 * W));
        pix /= 2 * W;
        const int oy = static_cast<int>(pix % (2 * H));
        const long long n = pix / (2 * H);
        const uint4 v = *reinterpret_cast<const uint4*>(in + ((n * H + oy / 2) * W + ox / 2) * C + c);
        *reinterpret_cast<uint4*>(out + ((n * 2 * H + oy) * 2 * W + ox) * C + c) = v;
    }
}

// ---- im2col for small-channel first convolutions ------------------------------------

template <typename T>
__global__ void im2col_kernel(const T* __restrict__ in, long long img_stride, const int* img_src, int imgs, int H,
                              int W, int C, int Kp, float scale, int tclamp, bf16* __restrict__ out,
                              const int* rows_dev) {
    pdl_launch();
    pdl_wait();
    int lim = imgs;
    if (rows_dev) lim = min(lim, *rows_dev);
    const int noct = Kp / 8;
    const long long total = static_cast<long long>(lim) * H * W * noct;
    for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int k0 = static_cast<int>(idx % noct) * 8;
        const long long pix = idx / noct;
        const int x = static_cast<int>(pix % W);
        const int y = static_cast<int>((pix / W) % H);
        const int n = static_cast<int>(pix / (static_cast<long long>(W) * H));
        const int src_img = img_src ? img_src[n] : n;
        const T* base = in + static_cast<long long>(src_img) * img_stride;
        float v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int k = k0 + i;
            float val = 0.f;
            if (k < 9 * C) {
                const int tap = k / C, c = k - tap * C;
                const int yy = y + tap / 3 - 1, xx = x + tap % 3 - 1;
                if (yy >= 0 && yy < H && xx >= 0 && xx < W)
                    val = static_cast<float>(base[(static_cast<long long>(yy) * W + xx) * C + c]) * scale;
                if (tclamp) val = tanhf(val / 3.f) * 3.f;  // TAESD decoder input Clamp
            }
            v[i] = val;
        }
        store8(out + pix * Kp + k0, v);
    }
}

// ---- warp-level tensor-core helpers (mma.sync m16n8k16, bf16 in, fp32 accumulate) ----------
// Used by the TAESD head/tail convs, whose 3-channel side is far below a tcgen05 tile
// (N >= 16 pads 3 to 16+ and the MMA cost is set by the 128-row A operand read).
__device__ __forceinline__ void mma_bf16_16816(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldmatrix_x4(uint32_t* r, const void* smem_row) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem_row))));
}
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&h);
}

// ---- 3x3 conv of u8 RGB frames, 3 -> 64 channels (the TAESD encoder's first layer) -------
// Implicit GEMM on mma.sync.  Persistent blocks (the weights' B fragments are loaded into
// registers once per block) walk tiles of one image row x 256 pixels; 8 warps x 2
// fragments of 16 pixels; K = 27 (tap * 3 + channel, as the im2col layout; padded to 32
// with zero weights), N = 64 (8 n-tiles).  A fragments are gathered in registers straight
// from a 3-row u8 tile (u8 / 255 -> bf16, zero padding).  The fp32 results (+ bias) are
// staged as bf16 in shared memory and written with 16-byte coalesced stores: the kernel
// is bound by its 128 B/pixel output.
constexpr int kRgbTileW = 256;

__global__ void __launch_bounds__(256, 2) conv3x3_rgb8_kernel(const uint8_t* __restrict__ in, long long img_stride,
                                                              const int* img_src, int imgs, int H, int W,
                                                              const bf16* __restrict__ w, int ldw,
                                                              const float* __restrict__ bias, bf16* __restrict__ out,
                                                              const int* rows_dev) {
    constexpr int RS = (kRgbTileW + 2) * 3 + 2;  // row tile stride (bytes)
    __shared__ uint8_t rowt[3][RS];
    __shared__ __align__(16) uint8_t ot[kRgbTileW * 128];  // [pixel][8 chunks x 16 B], chunk ^ (pixel & 7)
    pdl_launch();
    pdl_wait();
    const int live = rows_dev ? min(imgs, *rows_dev) : imgs;
    const int xt = (W + kRgbTileW - 1) / kRgbTileW;
    const int ntiles = live * H * xt;
    if (static_cast<int>(blockIdx.x) >= ntiles) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, q = lane & 3;
    // B fragments: n-tile j, k-step s -> (k = 16 s + 2 q + {0, 1} (+8), co = 8 j + g)
    uint32_t bf[8][2][2];
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int s = 0; s < 2; ++s)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int k = 16 * s + 2 * q + 8 * h;
                const bf16* wr = w + static_cast<long long>(8 * j + g) * ldw;
                const float w0 = k < 27 ? __bfloat162float(wr[k]) : 0.f;
                const float w1 = k + 1 < 27 ? __bfloat162float(wr[k + 1]) : 0.f;
                bf[j][s][h] = pack_bf16x2(w0, w1);
            }
    float bv[8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        bv[j][0] = bias ? bias[8 * j + 2 * q] : 0.f;
        bv[j][1] = bias ? bias[8 * j + 2 * q + 1] : 0.f;
    }
    // this lane's 8 im2col columns per K-step (k = 16 s + 2 q + {0, 1} + {0, 8}) as offsets
    // into the flattened row tile (dy * RS + dx * 3 + channel); k >= 27: zero weight
    int koff[2][4];
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            int k = 16 * s + 2 * q + (e & 1) + 8 * (e >> 1);
            k = k < 27 ? k : 26;  // any in-tile offset: its weight is zero
            const int tap = k / 3, ch = k - tap * 3, dy = tap / 3, dx = tap - dy * 3;
            koff[s][e] = dy * RS + dx * 3 + ch;
        }
    const bool vec = (W * 3) % 4 == 0 && (reinterpret_cast<uintptr_t>(in) & 3) == 0 && img_stride % 4 == 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int n = tile / (H * xt), rem = tile - n * H * xt, y = rem / xt, x0 = (rem - y * xt) * kRgbTileW;
        const uint8_t* base = in + static_cast<long long>(img_src ? img_src[n] : n) * img_stride;
        {
            // 3 rows of bytes [(x0 - 1) * 3, (x0 + 257) * 3) with 4-byte loads (rows are W * 3
            // bytes, a multiple of 4 on the vector path: a word is all in the row or all out)
            const int b0 = (x0 - 1) * 3;
            const int w0 = (b0 - 3) / 4;  // floor(b0 / 4) for b0 >= -3
            const int nw = ((x0 + kRgbTileW + 1) * 3 + 3) / 4 - w0;
            for (int i = threadIdx.x; i < 3 * nw; i += blockDim.x) {
                const int r = i / nw, wi = w0 + i % nw, yy = y - 1 + r;
                const bool rin = yy >= 0 && yy < H;
                uint32_t v = 0;
                if (vec) {
                    if (rin && wi >= 0 && 4 * wi < W * 3)
                        v = *reinterpret_cast<const uint32_t*>(base + static_cast<long long>(yy) * W * 3 + 4 * wi);
                } else if (rin) {
                    for (int e2 = 0; e2 < 4; ++e2) {
                        const int o = 4 * wi + e2;
                        if (o >= 0 && o < W * 3) v |= static_cast<uint32_t>(base[static_cast<long long>(yy) * W * 3 + o]) << (8 * e2);
                    }
                }
#pragma unroll
                for (int e2 = 0; e2 < 4; ++e2) {
                    const int j = 4 * wi + e2 - b0;
                    if (j >= 0 && j < (kRgbTileW + 2) * 3) rowt[r][j] = static_cast<uint8_t>(v >> (8 * e2));
                }
            }
        }
        __syncthreads();
        const uint8_t* rt = &rowt[0][0];
#pragma unroll
        for (int f = 0; f < 2; ++f) {
            const int p0 = warp * 32 + f * 16;  // first pixel of the fragment (tile column)
            uint32_t af[2][4];
#pragma unroll
            for (int s = 0; s < 2; ++s)
#pragma unroll
                for (int h = 0; h < 2; ++h) {  // h: pixel p0 + g (+8)
                    const uint8_t* pp = rt + (p0 + g + 8 * h) * 3;
                    af[s][h] = pack_bf16x2(pp[koff[s][0]] * (1.f / 255.f), pp[koff[s][1]] * (1.f / 255.f));
                    af[s][2 + h] = pack_bf16x2(pp[koff[s][2]] * (1.f / 255.f), pp[koff[s][3]] * (1.f / 255.f));
                }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                float d[4] = {bv[j][0], bv[j][1], bv[j][0], bv[j][1]};
                mma_bf16_16816(d, af[0], bf[j][0][0], bf[j][0][1]);
                mma_bf16_16816(d, af[1], bf[j][1][0], bf[j][1][1]);
                // columns 8 j + 2 q, +1 of pixels p0 + g and p0 + g + 8: 4 bytes in chunk j
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int px = p0 + g + 8 * h;
                    *reinterpret_cast<uint32_t*>(ot + px * 128 + ((j ^ (px & 7)) << 4) + q * 4) =
                        pack_bf16x2(d[2 * h], d[2 * h + 1]);
                }
            }
        }
        __syncthreads();
        bf16* orow = out + (static_cast<long long>(n) * H + y) * W * 64;
        const int npx = min(kRgbTileW, W - x0);
        for (int i = threadIdx.x; i < npx * 8; i += blockDim.x) {
            const int px = i >> 3, ch = i & 7;
            *reinterpret_cast<uint4*>(orow + static_cast<long long>(x0 + px) * 64 + ch * 8) =
                *reinterpret_cast<const uint4*>(ot + px * 128 + ((ch ^ (px & 7)) << 4));
        }
        // the next tile's row loads overwrite rowt only after this barrier; ot is rewritten
        // after the next tile's first barrier, once every thread has passed this store loop
    }
}

// ---- 3x3 conv, 64 -> 3 channels, u8 output (TAESD decoder head) --------------------------
// Implicit GEMM on mma.sync (a tcgen05 tile would pad N = 3 to 64 and cost twice a full
// 64 -> 64 conv).  Persistent blocks (B fragments of the weights in registers, loaded once)
// walk tiles of 4 output rows x 128 columns, 8 warps; the 6 x 130 x 64 bf16 input tile
// sits in smem with the 16-byte chunks of each pixel XOR-swizzled by (column % 8), so the
// ldmatrix rows (16 consecutive pixels) hit distinct banks.  Each warp owns half a row: 4
// fragments of 16 pixels accumulated as 4 independent chains of 9 taps x 4 K-steps of
// m16n8k16 with the 3 (padded to 8) output channels.  fp32 accumulation, then
// round(255 * clamp(v, 0, 1)) like the GEMM u8 epilogue, staged in smem and written with
// coalesced 4-byte stores.  Two blocks per SM overlap one block's tile load with the
// other's math.
constexpr int kHeadRows = 4;
constexpr int kHeadTileBytes = (kHeadRows + 2) * 130 * 128;

template <int CO>
__global__ void __launch_bounds__(64 * kHeadRows, 2) conv3x3_c64_u8_kernel(const bf16* __restrict__ in, int imgs, int H,
                                                                           int W, const bf16* __restrict__ w,
                                                                           const float* __restrict__ bias,
                                                                           uint8_t* __restrict__ out, const int* img_map,
                                                                           const int* rows_dev) {
    extern __shared__ __align__(16) uint8_t tile[];  // [rows + 2][130][8 chunks x 16 B], swizzled
    __shared__ __align__(16) uint8_t ob[kHeadRows][128 * CO + 4];
    static_assert(CO <= 8, "head conv: <= 8 output channels");
    pdl_launch();
    pdl_wait();
    const int live = rows_dev ? min(imgs, *rows_dev) : imgs;
    const int xt = (W + 127) / 128, yt = (H + kHeadRows - 1) / kHeadRows;
    const int ntiles = live * yt * xt;
    if (static_cast<int>(blockIdx.x) >= ntiles) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, q = lane & 3;
    // B fragments: tap t, K-step s (channels 16 s ..), h: k = 16 s + 2 q + 8 h + {0, 1}, co = g
    uint32_t bf[9][4][2];
#pragma unroll
    for (int t = 0; t < 9; ++t)
#pragma unroll
        for (int s = 0; s < 4; ++s)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int ci = 16 * s + 2 * q + 8 * h;
                const bf16* wr = w + (static_cast<long long>(g) * 9 + t) * 64 + ci;
                bf[t][s][h] = g < CO ? pack_bf16x2(__bfloat162float(wr[0]), __bfloat162float(wr[1])) : 0u;
            }
    const float bias0 = (bias && 2 * q < CO) ? bias[2 * q] : 0.f;
    const float bias1 = (bias && 2 * q + 1 < CO) ? bias[2 * q + 1] : 0.f;
    const int ty = warp >> 1, half = warp & 1;
    // ldmatrix.x4 row address of this lane: fragment row (lane & 15), chunk half (lane >> 4)
    const int lrow = lane & 15, lchunk = lane >> 4;
    for (int tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
        const int n = tl / (yt * xt), rem = tl - n * yt * xt, by = rem / xt;
        const int y0 = by * kHeadRows, x0 = (rem - by * xt) * 128;
        const bf16* base = in + static_cast<long long>(n) * H * W * 64;
        // the whole tile in flight at once: 16-byte cp.async (zero-filled outside the image)
        for (int i = threadIdx.x; i < (kHeadRows + 2) * 130 * 8; i += blockDim.x) {
            const int k = i & 7, col = (i >> 3) % 130, r = i / (130 * 8);
            const int yy = y0 - 1 + r, xx = x0 - 1 + col;
            const bool inb = yy >= 0 && yy < H && xx >= 0 && xx < W;
            const bf16* src = inb ? base + (static_cast<long long>(yy) * W + xx) * 64 + k * 8 : base;
            const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(tile + ((r * 130 + col) * 8 + (k ^ (col & 7))) * 16));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(inb ? 16 : 0) : "memory");
        }
        asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        // the warp's 4 fragments (16 columns each) accumulate independently: 4 MMA chains in
        // flight per warp instead of one dependent chain of 36
        float d[4][4];
#pragma unroll
        for (int f = 0; f < 4; ++f) {
            d[f][0] = bias0;
            d[f][1] = bias1;
            d[f][2] = bias0;
            d[f][3] = bias1;
        }
#pragma unroll
        for (int t = 0; t < 9; ++t) {
            const int dy = t / 3, dx = t - dy * 3;
#pragma unroll
            for (int s = 0; s < 4; ++s) {
#pragma unroll
                for (int f = 0; f < 4; ++f) {
                    const int col = half * 64 + f * 16 + lrow + dx;
                    uint32_t af[4];
                    // matrices: (rows 0-7, k 0-7), (rows 8-15, k 0-7), (rows 0-7, k 8-15), (rows 8-15, k 8-15)
                    ldmatrix_x4(af, tile + ((ty + dy) * 130 + col) * 128 + (((2 * s + lchunk) ^ (col & 7)) << 4));
                    mma_bf16_16816(d[f], af, bf[t][s][0], bf[t][s][1]);
                }
            }
        }
#pragma unroll
        for (int f = 0; f < 4; ++f) {
            const int c0 = half * 64 + f * 16;
            // d[f]: (pixel c0 + g, channels 2q, 2q+1), (pixel c0 + g + 8, same)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int px = c0 + g + 8 * h;
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int o = 2 * q + e;
                    if (o < CO)
                        ob[ty][px * CO + o] = static_cast<uint8_t>(__float2int_rn(fminf(fmaxf(d[f][2 * h + e], 0.f), 1.f) * 255.f));
                }
            }
        }
        __syncthreads();  // tile consumed, ob complete
        // coalesced write-out: each row of the block is 128 * CO contiguous bytes
        const int nx = min(128, W - x0);
        for (int r = 0; r < kHeadRows; ++r) {
            const int y = y0 + r;
            if (y >= H) break;
            uint8_t* orow = out + ((static_cast<long long>(img_map ? img_map[n] : n) * H + y) * W + x0) * CO;
            if (nx == 128 && (128 * CO) % 4 == 0 && (reinterpret_cast<uintptr_t>(orow) & 3) == 0) {
                for (int i = threadIdx.x; i < 32 * CO; i += blockDim.x)
                    reinterpret_cast<uint32_t*>(orow)[i] = *reinterpret_cast<const uint32_t*>(&ob[r][4 * i]);
            } else {
                for (int i = threadIdx.x; i < nx * CO; i += blockDim.x) orow[i] = ob[r][i];
            }
        }
        __syncthreads();  // ob read before the next tile's fragments overwrite it
    }
}

// ---- timestep embedding ------------------------------------------------------------

__global__ void temb_kernel(const int* taus, int n, int dim, bf16* out) {
    const int r = blockIdx.x;
    const int half = dim / 2;
    for (int j = threadIdx.x; j < dim; j += blockDim.x) {
        const int k = j < half ? j : j - half;
        const float f = expf(-logf(10000.f) * k / half);
        const float a = static_cast<float>(taus[r]) * f;
        out[static_cast<long long>(r) * dim + j] = __float2bfloat16(j < half ? cosf(a) : sinf(a));
    }
}

// ---- init -----------------------------------------------------------------------------

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

__device__ __forceinline__ float hash_normal(uint64_t seed, long long i) {
    const uint64_t a = mix64(seed ^ mix64(static_cast<uint64_t>(i)));
    const float u1 = (static_cast<float>(a >> 40) + 0.5f) * (1.f / 16777216.f);
    const float u2 = static_cast<float>((a >> 16) & 0xFFFFFF) * (1.f / 16777216.f);
    return sqrtf(-2.f * logf(u1)) * cospif(2.f * u2);
}

__global__ void fill_normal_bf16_kernel(bf16* p, long long n, float std, uint64_t seed) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        p[i] = __float2bfloat16(std * hash_normal(seed, i));
}
__global__ void fill_normal_f32_kernel(float* p, long long n, float std, uint64_t seed) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        p[i] = std * hash_normal(seed, i);
}
__global__ void fill_const_kernel(float* p, long long n, float v) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        p[i] = v;
}
__global__ void tanh_clamp_kernel(const float* in, float* out, long long n) {
    pdl_launch();
    pdl_wait();
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        out[i] = tanhf(in[i] / 3.f) * 3.f;
}

unsigned grid_for(long long work, int threads) {
    long long b = (work + threads - 1) / threads;
    if (b > 148LL * 16) b = 148LL * 16;
    if (b < 1) b = 1;
    return static_cast<unsigned>(b);
}

}  // namespace

GnPlan plan_groupnorm(const bf16* x1, int C1, const bf16* x2, int C2, int HW, int imgs, float eps, const float* gamma,
                      const float* beta, int silu_, bf16* out, const int* rows_dev, unsigned long long* acc,
                      unsigned long long* counter) {
    GnPlan p{};
    p.x1 = x1;
    p.x2 = x2;
    p.C1 = C1;
    p.C2 = x2 ? C2 : 0;
    p.HW = HW;
    p.groups = 32;
    p.eps = eps;
    p.gamma = gamma;
    p.beta = beta;
    p.silu = silu_;
    p.out = out;
    p.imgs = imgs;
    p.rows_dev = rows_dev;
    p.acc = acc;
    p.stats_fused = 0;
    const int Ct = p.C1 + p.C2;
    if (Ct % 8 != 0 || Ct % p.groups != 0 || (p.C2 && p.C1 % 8 != 0))
        raise(SDX_INVALID_ARGUMENT, "groupnorm: channels must be multiples of 8 and 32");
    if (Ct / 8 > 320) raise(SDX_INVALID_ARGUMENT, "groupnorm: more than 2560 channels");
    // each thread owns one aligned channel octet, which must span <= 2 groups
    if (Ct / p.groups < 8 && Ct / p.groups != 4) raise(SDX_INVALID_ARGUMENT, "groupnorm: channels per group must be 4 or >= 8");
    if (!acc) raise(SDX_INVALID_ARGUMENT, "groupnorm: statistics arena required");
    // one wave: as many blocks as are co-resident (occupancy of the heavier
    // apply kernel), split evenly over the images; every thread >= 8 pixels
    const int noct = Ct / 8;
    const int PY = noct >= 256 ? 1 : 256 / noct;
    static int resident[321] = {};  // per thread count
    const int thr = noct * PY;
    if (!resident[noct]) {
        int a = 0, b = 0;
        SDX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, gn_apply_kernel, thr, 0));
        SDX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, gn_stats_kernel, thr, static_cast<size_t>(thr) * 16));
        resident[noct] = std::max(1, std::min(a, b)) * 148;
    }
    int blocks_per_img = std::max(1, resident[noct] / imgs);
    // whole batches of 8 pixels per thread: a partial second batch costs a full load round trip
    int ppb = (HW + blocks_per_img - 1) / blocks_per_img;
    ppb = (ppb + 8 * PY - 1) / (8 * PY) * (8 * PY);
    p.px_per_block = ppb;
    p.chunks = (HW + ppb - 1) / ppb;
    // Cluster variant: one launch, one CTA cluster per image (16 CTAs up to 4 images,
    // else 8 so the clusters are co-resident).  It uses imgs x 16|8 SMs, so it wins
    // while each CTA's range is small (tools/gn_bench.py on B200: up to ~200 KB per
    // CTA at <= 4 images, ~48 KB at 8); larger tensors take the statistics + apply
    // pair over all SMs.  SDX_GN_CLUSTER_MAX (elements per image) overrides.
    {
        const char* cs = std::getenv("SDX_GN_CLUSTER_SIZE");
        const int csize = cs ? std::atoi(cs) : (imgs <= 4 ? 16 : 8);
        const long long per_cta = static_cast<long long>(HW) * Ct * 2 / std::max(1, csize);
        bool use = per_cta <= (imgs <= 4 ? 200 * 1024 : 48 * 1024);
        if (const char* ce = std::getenv("SDX_GN_CLUSTER_MAX")) use = static_cast<long long>(HW) * Ct <= std::atoll(ce);
        if (use && csize >= 1 && csize <= 16) {
            p.cluster = csize;
            p.px_per_block = (HW + csize - 1) / csize;
            p.chunks = csize;
            p.piece = kGnBufBytes / (Ct * 2);
            return p;
        }
    }
    // single-launch variant: grid must be co-resident -> grow the pixel range per block
    p.counter = counter;
    p.fused = 0;
    if (counter) {
        // opt in with SDX_GN_SINGLE=1: measured slower at 4 rows (0.66 -> 1.04 ms per forward),
        // the co-residency limit forces fewer, longer blocks and the barrier wait is exposed
        static const bool on = [] {
            const char* v = std::getenv("SDX_GN_SINGLE");
            return v && v[0] == '1';
        }();
        const int threads = noct * PY;
        const size_t smem = static_cast<size_t>(threads) * 4 * sizeof(float);
        int per_sm = 0;
        SDX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gn_fused_kernel, threads, smem));
        const long long cap = static_cast<long long>(per_sm) * 148;
        if (on && cap > 0) {
            int fppb = ppb;
            while (static_cast<long long>((HW + fppb - 1) / fppb) * imgs > cap) fppb += 8 * PY;
            p.fused = 1;
            p.px_per_block = fppb;
            p.chunks = (HW + fppb - 1) / fppb;
        }
    }
    return p;
}

void free_groupnorm(GnPlan&) {}

namespace {
long long* g_gn_dbg = nullptr;
}
void set_groupnorm_debug_buffer(long long* dbg) { g_gn_dbg = dbg; }

void run_groupnorm(const GnPlan& p_in, cudaStream_t st) {
    GnPlan p = p_in;
    p.dbg = g_gn_dbg;
    const int Ct = p.C1 + p.C2;
    const int noct = Ct / 8;
    if (p.cluster) {
        ensure_kernel_attrs(gn_cluster_kernel, 2 * kGnBufBytes, /*nonportable_cluster=*/true);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(p.cluster, p.imgs);
        cfg.blockDim = dim3(noct * std::max(1, 320 / noct));
        cfg.dynamicSmemBytes = 2 * kGnBufBytes;
        cfg.stream = st;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
        at[1].id = cudaLaunchAttributeClusterDimension;
        at[1].val.clusterDim.x = p.cluster;
        at[1].val.clusterDim.y = 1;
        at[1].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 2;
        SDX_CUDA(cudaLaunchKernelEx(&cfg, gn_cluster_kernel, p));
        return;
    }
    const int PY = noct >= 256 ? 1 : 256 / noct;
    const int threads = noct * PY;
    if (p.fused && !p.stats_fused) {
        launch_pdl(gn_fused_kernel, dim3(p.chunks, p.imgs), dim3(threads), static_cast<size_t>(threads) * 4 * sizeof(float),
                   st, p);
        return;
    }
    if (!p.stats_fused) {  // statistics not accumulated by the producer: standalone pass
        launch_pdl(gn_stats_kernel, dim3(p.chunks, p.imgs), dim3(threads), static_cast<size_t>(threads) * 4 * sizeof(float), st, p);
    }
    launch_pdl(gn_apply_kernel, dim3(p.chunks, p.imgs), dim3(threads), 0, st, p);
}

void run_groupnorm_part(const GnPlan& p, int part, cudaStream_t st) {
    const int noct = (p.C1 + p.C2) / 8;
    const int PY = noct >= 256 ? 1 : 256 / noct;
    const int threads = noct * PY;
    if (part == 0)
        launch_pdl(gn_stats_kernel, dim3(p.chunks, p.imgs), dim3(threads), static_cast<size_t>(threads) * 4 * sizeof(float), st, p);
    else
        launch_pdl(gn_apply_kernel, dim3(p.chunks, p.imgs), dim3(threads), 0, st, p);
}

void run_layernorm(const bf16* x, int rows, int C, const float* gamma, const float* beta, float eps, bf16* out,
                   const int* rows_dev, int rows_per_unit, cudaStream_t st) {
    const int noct = C / 8;
    const unsigned blocks = static_cast<unsigned>((rows + 7) / 8);
    if (noct <= 32) launch_pdl(layernorm_kernel<1>, dim3(blocks), dim3(256), 0, st, x, rows, C, gamma, beta, eps, out, rows_dev, rows_per_unit);
    else if (noct <= 64) launch_pdl(layernorm_kernel<2>, dim3(blocks), dim3(256), 0, st, x, rows, C, gamma, beta, eps, out, rows_dev, rows_per_unit);
    else if (noct <= 160) launch_pdl(layernorm_kernel<5>, dim3(blocks), dim3(256), 0, st, x, rows, C, gamma, beta, eps, out, rows_dev, rows_per_unit);
    else raise(SDX_INVALID_ARGUMENT, "layernorm: C too large");
}

void run_geglu(const bf16* in, int rows, int H, bf16* out, const int* rows_dev, int rows_per_unit, cudaStream_t st) {
    launch_pdl(geglu_kernel, dim3(grid_for(static_cast<long long>(rows) * H / 8, 256)), dim3(256), 0, st, in, rows, H, out,
               rows_dev, rows_per_unit);
}

void run_upsample2x(const bf16* in, int imgs, int H, int W, int C, bf16* out, const int* rows_dev, cudaStream_t st) {
    launch_pdl(upsample_kernel, dim3(grid_for(static_cast<long long>(imgs) * 4 * H * W * C / 8, 256)), dim3(256), 0, st,
               in, imgs, H, W, C, out, rows_dev);
}

void run_im2col3x3_f32(const float* in, int imgs, int H, int W, int C, int Kp, bf16* out, const int* rows_dev,
                       cudaStream_t st) {
    launch_pdl(im2col_kernel<float>, dim3(grid_for(static_cast<long long>(imgs) * H * W * Kp / 8, 256)), dim3(256), 0, st,
               in, static_cast<long long>(H) * W * C, static_cast<const int*>(nullptr), imgs, H, W, C, Kp, 1.f, 0, out,
               rows_dev);
}

void run_im2col3x3_f32_gather(const float* in, long long img_stride, const int* img_src, int imgs, int H, int W, int C,
                              int Kp, int tanh_clamp, bf16* out, const int* rows_dev, cudaStream_t st) {
    launch_pdl(im2col_kernel<float>, dim3(grid_for(static_cast<long long>(imgs) * H * W * Kp / 8, 256)), dim3(256), 0, st,
               in, img_stride, img_src, imgs, H, W, C, Kp, 1.f, tanh_clamp, out, rows_dev);
}

void run_im2col3x3_u8(const uint8_t* in, long long img_stride, const int* img_src, int imgs, int H, int W, int C,
                      int Kp, bf16* out, const int* rows_dev, cudaStream_t st) {
    launch_pdl(im2col_kernel<uint8_t>, dim3(grid_for(static_cast<long long>(imgs) * H * W * Kp / 8, 256)), dim3(256), 0,
               st, in, img_stride, img_src, imgs, H, W, C, Kp, 1.f / 255.f, 0, out, rows_dev);
}

void run_conv3x3_rgb8(const uint8_t* in, long long img_stride, const int* img_src, int imgs, int H, int W,
                      const bf16* w, int ldw, const float* bias, bf16* out, const int* rows_dev, cudaStream_t st) {
    if (ldw < 27) raise(SDX_INVALID_ARGUMENT, "conv3x3_rgb8: weight row shorter than 27");
    const long long tiles = static_cast<long long>(imgs) * H * ((W + kRgbTileW - 1) / kRgbTileW);
    const int grid = static_cast<int>(std::min<long long>(tiles, 2LL * kSmCount));
    launch_pdl(conv3x3_rgb8_kernel, dim3(grid), dim3(256), 0, st, in, img_stride, img_src, imgs, H, W, w, ldw, bias,
               out, rows_dev);
}

void run_conv3x3_c64_u8(const bf16* in, int imgs, int H, int W, const bf16* w, int Cout, const float* bias,
                        uint8_t* out, const int* img_map, const int* rows_dev, cudaStream_t st) {
    if (Cout != 3) raise(SDX_INVALID_ARGUMENT, "conv3x3_c64_u8: 3 output channels");
    ensure_kernel_attrs(conv3x3_c64_u8_kernel<3>, kHeadTileBytes);
    const long long tiles = static_cast<long long>(imgs) * ((H + kHeadRows - 1) / kHeadRows) * ((W + 127) / 128);
    const int grid = static_cast<int>(std::min<long long>(tiles, 2LL * kSmCount));
    launch_pdl(conv3x3_c64_u8_kernel<3>, dim3(grid), dim3(64 * kHeadRows), static_cast<size_t>(kHeadTileBytes), st, in,
               imgs, H, W, w, bias, out, img_map, rows_dev);
}

void run_timestep_embedding(const int* taus, int n, int dim, bf16* out, cudaStream_t st) {
    temb_kernel<<<n, 128, 0, st>>>(taus, n, dim, out);
    SDX_LAUNCH_CHECK();
}

void fill_normal_bf16(bf16* p, long long n, float std, uint64_t seed, cudaStream_t st) {
    fill_normal_bf16_kernel<<<grid_for(n, 256), 256, 0, st>>>(p, n, std, seed);
    SDX_LAUNCH_CHECK();
}
void fill_normal_f32(float* p, long long n, float std, uint64_t seed, cudaStream_t st) {
    fill_normal_f32_kernel<<<grid_for(n, 256), 256, 0, st>>>(p, n, std, seed);
    SDX_LAUNCH_CHECK();
}
void fill_const_f32(float* p, long long n, float v, cudaStream_t st) {
    fill_const_kernel<<<grid_for(n, 256), 256, 0, st>>>(p, n, v);
    SDX_LAUNCH_CHECK();
}
__global__ void interleave_geglu_kernel(const bf16* w, const float* b, int H, int K, bf16* wout, float* bout) {
    const int r = blockIdx.x;  // destination row
    const int blk = r >> 5, wi = r & 31;
    const int src = wi < 16 ? blk * 16 + wi : H + blk * 16 + (wi - 16);
    for (int k = threadIdx.x; k < K; k += blockDim.x) wout[static_cast<long long>(r) * K + k] = w[static_cast<long long>(src) * K + k];
    if (threadIdx.x == 0) bout[r] = b[src];
}

// LayerNorm folding into the next GEMM: W' = bf16(W * gamma) per input column,
// s[n] = sum_k W'[n][k] (fp32 of the bf16 values the MMA sees), c[n] = bias[n] +
// sum_k W[n][k] * beta[k].  One block per output row, fixed-order reductions.
__global__ void ln_fold_kernel(const bf16* __restrict__ W, int K, const float* __restrict__ gamma,
                               const float* __restrict__ beta, const float* __restrict__ bias, bf16* __restrict__ Wf,
                               float* __restrict__ s, float* __restrict__ c) {
    const int n = blockIdx.x;
    float a = 0.f, b = 0.f;
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
        const float w = __bfloat162float(W[static_cast<long long>(n) * K + k]);
        const bf16 wf = __float2bfloat16(w * gamma[k]);
        Wf[static_cast<long long>(n) * K + k] = wf;
        a += __bfloat162float(wf);
        b += w * beta[k];
    }
    __shared__ float ra[256], rb[256];
    ra[threadIdx.x] = a;
    rb[threadIdx.x] = b;
    __syncthreads();
    for (int off = blockDim.x / 2; off; off >>= 1) {
        if (static_cast<int>(threadIdx.x) < off) {
            ra[threadIdx.x] += ra[threadIdx.x + off];
            rb[threadIdx.x] += rb[threadIdx.x + off];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        s[n] = ra[0];
        c[n] = (bias ? bias[n] : 0.f) + rb[0];
    }
}

void run_ln_fold(const bf16* W, int N, int K, const float* gamma, const float* beta, const float* bias, bf16* Wf,
                 float* s, float* c, cudaStream_t st) {
    ln_fold_kernel<<<N, 256, 0, st>>>(W, K, gamma, beta, bias, Wf, s, c);
    SDX_LAUNCH_CHECK();
}

void run_interleave_geglu(const bf16* w, const float* b, int H, int K, bf16* wout, float* bout, cudaStream_t st) {
    interleave_geglu_kernel<<<2 * H, 128, 0, st>>>(w, b, H, K, wout, bout);
    SDX_LAUNCH_CHECK();
}

void run_tanh_clamp(const float* in, float* out, long long n, cudaStream_t st) {
    launch_pdl(tanh_clamp_kernel, dim3(grid_for(n, 256)), dim3(256), 0, st, in, out, n);
}

}  // namespace sdx
