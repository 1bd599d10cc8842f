// Fused stream-batch step (one launch per tick over every in-flight row of
// every stream):
//   denoiser rows   AnalyticGaussianModel::do_predict  denoiser.cpp:26-43
//                   (or external eps rows from the UNet)
//   guidance        cfg_combine / virtual_residual_noise / rcfg_combine
//                                                      guidance.cpp:19-48, engine.cpp:17-32
//   onetime init    predict_x0 on the negative row    engine.cpp:122-126
//   LCM update      consistency_step + forward_diffuse schedule.cpp:60-107
//   entry noising   forward_diffuse(x0, steps[0], eps_cached[0]) for the
//                   frame ingested this iteration      engine.cpp:69
// HBM-bound: fp32 storage and math (inverse sqrt(alpha)/sqrt(beta)
// precomputed in fp64 on the host), float4 streaming loads, 2 vectors per
// thread in flight, one template instance per guidance mode so unused
// operands are never loaded.
#include <cuda_runtime.h>

#include "common.cuh"
#include "device_ctl.cuh"
#include "kernels_core.cuh"

namespace sdx {

namespace {

template <int kMode, bool kExt>
struct Lane {
    float4 x, mu, ng, ref, ren, ec, en;
};

__device__ __forceinline__ float4 ld4(const float* p) { return __ldcs(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ void st4(float* p, float4 v) { __stcs(reinterpret_cast<float4*>(p), v); }

// guided eps of one element (combine_row, engine.cpp:17-32)
template <int kMode, bool kExt>
__device__ __forceinline__ float combine1(float x, float mu, float ng, float ref, float ec_in, float en_in,
                                          const StepScalars& st, const StepScalars& st0, float gamma, float delta,
                                          bool init_now, float* x0ref_out) {
    const float ec = kExt ? ec_in : st.f_an * (x - st.f_sa * mu);
    float eps = ec;
    if (kMode == SDX_GUIDANCE_CFG) {
        const float en = kExt ? en_in : st.f_an * (x - st.f_sa * ng);
        eps = en + gamma * (ec - en);
    } else if (kMode == SDX_GUIDANCE_SELF_NEGATIVE || kMode == SDX_GUIDANCE_ONETIME_NEGATIVE) {
        float xr = ref;
        if (kMode == SDX_GUIDANCE_ONETIME_NEGATIVE && init_now) {
            const float en = kExt ? en_in : st0.f_an * (x - st0.f_sa * ng);
            xr = (x - st0.f_sb * en) * st0.f_isa;
            *x0ref_out = xr;
        }
        if (st.f_beta > 0.f) {
            const float dv = delta * ((x - st.f_sa * xr) * st.f_isb);
            eps = dv + gamma * (ec - dv);
        }
    }
    return eps;
}

// consistency_step + re-noise (schedule.cpp:91-107)
__device__ __forceinline__ float update1(float x, float eps, float ren, const StepScalars& st, const StepScalars& nx,
                                         bool terminal) {
    const float px0 = (x - st.f_sb * eps) * st.f_isa;
    const float xh = st.f_cs * x + st.f_co * px0;
    return terminal ? xh : nx.f_sa * xh + nx.f_sb * ren;
}

template <int kMode, bool kExt>
__device__ __forceinline__ float step1(float x, float mu, float ng, float ref, float ren, float ec_in, float en_in,
                                       const StepScalars& st, const StepScalars& st0, const StepScalars& nx,
                                       float gamma, float delta, bool init_now, bool terminal, float* x0ref_out) {
    return update1(x, combine1<kMode, kExt>(x, mu, ng, ref, ec_in, en_in, st, st0, gamma, delta, init_now, x0ref_out),
                   ren, st, nx, terminal);
}

#define SDX_COMP(c) c
template <int kMode, bool kExt>
__device__ __forceinline__ float4 step4(const float4 x, const float4 mu, const float4 ng, const float4 ref,
                                        const float4 ren, const float4 ec, const float4 en, const StepScalars& st,
                                        const StepScalars& st0, const StepScalars& nx, float g, float dl,
                                        bool init_now, bool terminal, float4* xr) {
    float4 y;
    y.x = step1<kMode, kExt>(x.x, mu.x, ng.x, ref.x, ren.x, ec.x, en.x, st, st0, nx, g, dl, init_now, terminal, &xr->x);
    y.y = step1<kMode, kExt>(x.y, mu.y, ng.y, ref.y, ren.y, ec.y, en.y, st, st0, nx, g, dl, init_now, terminal, &xr->y);
    y.z = step1<kMode, kExt>(x.z, mu.z, ng.z, ref.z, ren.z, ec.z, en.z, st, st0, nx, g, dl, init_now, terminal, &xr->z);
    y.w = step1<kMode, kExt>(x.w, mu.w, ng.w, ref.w, ren.w, ec.w, en.w, st, st0, nx, g, dl, init_now, terminal, &xr->w);
    return y;
}

__device__ __forceinline__ bool finite4(float4 v) {
    return isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w);
}

// Vectorised path: d % 4 == 0.  grid (chunks, n slots, S streams).
template <int kMode, bool kExt>
__global__ void __launch_bounds__(256) step_vec_kernel(StepArgs a) {
    constexpr int U = 2;  // float4 per operand per thread in flight
    const int s = blockIdx.z;
    const int slot = blockIdx.y;
    const StreamCtl* cp = a.ctl + s;
    if (!cp->tick_now) return;
    const SlotCtl sc = cp->slot[slot];
    if (sc.seq < 0) return;
    const int step = static_cast<int>(cp->ticks - sc.ingest_tick);
    const bool terminal = step + 1 >= a.n;
    const bool entering = sc.entering != 0;
    const bool init_now = kMode == SDX_GUIDANCE_ONETIME_NEGATIVE && sc.init == 0;
    const StepScalars st = a.tbl[step];
    const StepScalars st0 = a.tbl[0];
    const StepScalars nx = a.tbl[terminal ? a.n : step + 1];
    const float g = static_cast<float>(a.gamma), dl = static_cast<float>(a.delta);

    const long long d = a.d;
    const long long sd = static_cast<long long>(s) * a.n + slot;
    const float* x0 = a.x0 + sd * d;
    float* xcur = a.x_cur + sd * d;
    float* x0ref = a.x0ref ? a.x0ref + sd * d : nullptr;
    const float* e0 = a.eps_cached + (static_cast<long long>(s) * a.n) * d;
    const float* ren = terminal ? nullptr : a.eps_cached + (static_cast<long long>(s) * a.n + step + 1) * d;
    const float* mu = a.cond + s * a.cond_stream_stride + slot * a.cond_slot_stride;
    const float* ng = a.neg ? a.neg + static_cast<long long>(s) * d : nullptr;
    float* out = terminal ? a.emitted + static_cast<long long>(s) * d : xcur;
    const float* ecr = nullptr;
    const float* enr = nullptr;
    if (kExt) {
        ecr = a.eps_ext + static_cast<long long>(a.slot_row_c[s * kMaxSteps + slot]) * a.eps_ext_stride;
        const int rn = a.slot_row_n[s * kMaxSteps + slot];
        enr = rn >= 0 ? a.eps_ext + static_cast<long long>(rn) * a.eps_ext_stride : nullptr;
    }

    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    int bad = 0;
    const long long per_iter = static_cast<long long>(gridDim.x) * blockDim.x * 4 * U;
    for (long long base = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) * 4; base < d;
         base += per_iter) {
        float4 vx[U], vmu[U], vng[U], vref[U], vren[U], vec[U], ven[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long i = base + static_cast<long long>(u) * gridDim.x * blockDim.x * 4;
            const bool ok = i < d;
            vx[u] = vmu[u] = vng[u] = vref[u] = vren[u] = vec[u] = ven[u] = z4;
            if (!ok) continue;
            if (entering) {
                const float4 a0 = ld4(x0 + i), b0 = ldg4(e0 + i);
                vx[u] = make_float4(st0.f_sa * a0.x + st0.f_sb * b0.x, st0.f_sa * a0.y + st0.f_sb * b0.y,
                                    st0.f_sa * a0.z + st0.f_sb * b0.z, st0.f_sa * a0.w + st0.f_sb * b0.w);
                if (kMode == SDX_GUIDANCE_SELF_NEGATIVE) vref[u] = a0;
            } else {
                vx[u] = ld4(xcur + i);
                if (kMode == SDX_GUIDANCE_SELF_NEGATIVE) vref[u] = ld4(x0 + i);
            }
            if (kMode == SDX_GUIDANCE_ONETIME_NEGATIVE && !init_now) vref[u] = ld4(x0ref + i);
            if (!kExt) vmu[u] = ldg4(mu + i);
            if (!kExt && (kMode == SDX_GUIDANCE_CFG || (kMode == SDX_GUIDANCE_ONETIME_NEGATIVE && init_now)))
                vng[u] = ldg4(ng + i);
            if (!terminal) vren[u] = ldg4(ren + i);
            if (kExt) {
                vec[u] = ld4(ecr + i);
                if (enr) ven[u] = ld4(enr + i);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long i = base + static_cast<long long>(u) * gridDim.x * blockDim.x * 4;
            if (i >= d) continue;
            float4 xr = z4;
            const float4 y = step4<kMode, kExt>(vx[u], vmu[u], vng[u], vref[u], vren[u], vec[u], ven[u], st, st0,
                                                nx, g, dl, init_now, terminal, &xr);
            if (kMode == SDX_GUIDANCE_ONETIME_NEGATIVE && init_now) st4(x0ref + i, xr);
            if (terminal && !finite4(y)) bad = 1;
            st4(out + i, y);
        }
    }
    if (terminal) {
        bad = __syncthreads_or(bad);
        if (bad && threadIdx.x == 0) atomicOr(&a.ctl[s].nonfinite, 1);
    }
}

// Scalar path for d % 4 != 0 (reference tests use d = 3, 8, ...).
template <int kMode, bool kExt>
__global__ void __launch_bounds__(256) step_scalar_kernel(StepArgs a) {
    const int s = blockIdx.z;
    const int slot = blockIdx.y;
    const StreamCtl* cp = a.ctl + s;
    if (!cp->tick_now) return;
    const SlotCtl sc = cp->slot[slot];
    if (sc.seq < 0) return;
    const int step = static_cast<int>(cp->ticks - sc.ingest_tick);
    const bool terminal = step + 1 >= a.n;
    const bool entering = sc.entering != 0;
    const bool init_now = kMode == SDX_GUIDANCE_ONETIME_NEGATIVE && sc.init == 0;
    const StepScalars st = a.tbl[step];
    const StepScalars st0 = a.tbl[0];
    const StepScalars nx = a.tbl[terminal ? a.n : step + 1];
    const float g = static_cast<float>(a.gamma), dl = static_cast<float>(a.delta);
    const long long d = a.d;
    const long long sd = static_cast<long long>(s) * a.n + slot;
    const float* x0 = a.x0 + sd * d;
    float* xcur = a.x_cur + sd * d;
    float* x0ref = a.x0ref ? a.x0ref + sd * d : nullptr;
    const float* e0 = a.eps_cached + (static_cast<long long>(s) * a.n) * d;
    const float* ren = terminal ? nullptr : a.eps_cached + (static_cast<long long>(s) * a.n + step + 1) * d;
    const float* mu = a.cond + s * a.cond_stream_stride + slot * a.cond_slot_stride;
    const float* ng = a.neg ? a.neg + static_cast<long long>(s) * d : nullptr;
    float* out = terminal ? a.emitted + static_cast<long long>(s) * d : xcur;
    const float* ecr = nullptr;
    const float* enr = nullptr;
    if (kExt) {
        ecr = a.eps_ext + static_cast<long long>(a.slot_row_c[s * kMaxSteps + slot]) * a.eps_ext_stride;
        const int rn = a.slot_row_n[s * kMaxSteps + slot];
        enr = rn >= 0 ? a.eps_ext + static_cast<long long>(rn) * a.eps_ext_stride : nullptr;
    }
    int bad = 0;
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < d;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const float x = entering ? st0.f_sa * x0[i] + st0.f_sb * e0[i] : xcur[i];
        float ref = 0.f;
        if (kMode == SDX_GUIDANCE_SELF_NEGATIVE) ref = x0[i];
        if (kMode == SDX_GUIDANCE_ONETIME_NEGATIVE && !init_now) ref = x0ref[i];
        const float m = kExt ? 0.f : mu[i];
        const float n_ = (!kExt && ng) ? ng[i] : 0.f;
        const float r = terminal ? 0.f : ren[i];
        const float ec = kExt ? ecr[i] : 0.f;
        const float en = (kExt && enr) ? enr[i] : 0.f;
        float xr = 0.f;
        const float y = step1<kMode, kExt>(x, m, n_, ref, r, ec, en, st, st0, nx, g, dl, init_now, terminal, &xr);
        if (kMode == SDX_GUIDANCE_ONETIME_NEGATIVE && init_now) x0ref[i] = xr;
        if (terminal && !isfinite(y)) bad = 1;
        out[i] = y;
    }
    if (terminal) {
        bad = __syncthreads_or(bad);
        if (bad && threadIdx.x == 0) atomicOr(&a.ctl[s].nonfinite, 1);
    }
}

// ---- cross-frame (Stream Batch) attention, engine.cpp:139-149 / attention.cpp:12-95 ----
// With kAttentionTokens identical token rows per frame (lift_tokens), attention of
// frame i's latent over the in-flight latents (keys) and guided eps (values)
// reduces to eps_i <- sum_f softmax_f(x_i . x_f / sqrt(d)) eps_f; unlift_tokens
// averages identical rows.  Three launches per tick: guided eps (+ entry noising
// into x_cur), the fp64 dot table, then the mix + consistency step.

// 1. guided eps of every in-flight slot into xfa_eps; the entering frame's x into x_cur
template <int kMode, bool kExt>
__global__ void __launch_bounds__(256) xfa_eps_kernel(StepArgs a) {
    const int s = blockIdx.z, slot = blockIdx.y;
    const StreamCtl* cp = a.ctl + s;
    if (!cp->tick_now) return;
    const SlotCtl sc = cp->slot[slot];
    if (sc.seq < 0) return;
    const int step = static_cast<int>(cp->ticks - sc.ingest_tick);
    const bool entering = sc.entering != 0;
    const bool init_now = kMode == SDX_GUIDANCE_ONETIME_NEGATIVE && sc.init == 0;
    const StepScalars st = a.tbl[step];
    const StepScalars st0 = a.tbl[0];
    const float g = static_cast<float>(a.gamma), dl = static_cast<float>(a.delta);
    const long long d = a.d;
    const long long sd = static_cast<long long>(s) * a.n + slot;
    const float* x0 = a.x0 + sd * d;
    float* xcur = a.x_cur + sd * d;
    float* x0ref = a.x0ref ? a.x0ref + sd * d : nullptr;
    float* eo = a.xfa_eps + sd * d;
    const float* e0 = a.eps_cached + (static_cast<long long>(s) * a.n) * d;
    const float* mu = a.cond + s * a.cond_stream_stride + slot * a.cond_slot_stride;
    const float* ng = a.neg ? a.neg + static_cast<long long>(s) * d : nullptr;
    const float* ecr = nullptr;
    const float* enr = nullptr;
    if (kExt) {
        ecr = a.eps_ext + static_cast<long long>(a.slot_row_c[s * kMaxSteps + slot]) * a.eps_ext_stride;
        const int rn = a.slot_row_n[s * kMaxSteps + slot];
        enr = rn >= 0 ? a.eps_ext + static_cast<long long>(rn) * a.eps_ext_stride : nullptr;
    }
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < d;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const float x = entering ? st0.f_sa * x0[i] + st0.f_sb * e0[i] : xcur[i];
        if (entering) xcur[i] = x;
        float ref = 0.f;
        if (kMode == SDX_GUIDANCE_SELF_NEGATIVE) ref = x0[i];
        if (kMode == SDX_GUIDANCE_ONETIME_NEGATIVE && !init_now) ref = x0ref[i];
        const float m = kExt ? 0.f : mu[i];
        const float n_ = (!kExt && ng) ? ng[i] : 0.f;
        const float ec = kExt ? ecr[i] : 0.f;
        const float en = (kExt && enr) ? enr[i] : 0.f;
        float xr = 0.f;
        eo[i] = combine1<kMode, kExt>(x, m, n_, ref, ec, en, st, st0, g, dl, init_now, &xr);
        if (kMode == SDX_GUIDANCE_ONETIME_NEGATIVE && init_now) x0ref[i] = xr;
    }
}

// 2. dots[s][i][f] = x_i . x_f in fp64 for every in-flight slot pair (one block per pair)
__global__ void __launch_bounds__(256) xfa_dots_kernel(StepArgs a) {
    const int s = blockIdx.z, i = blockIdx.y, f = blockIdx.x;
    const StreamCtl* cp = a.ctl + s;
    if (!cp->tick_now || cp->slot[i].seq < 0 || cp->slot[f].seq < 0) return;
    const long long d = a.d;
    const float* xi = a.x_cur + (static_cast<long long>(s) * a.n + i) * d;
    const float* xf = a.x_cur + (static_cast<long long>(s) * a.n + f) * d;
    double acc = 0.0;
    for (long long k = threadIdx.x; k < d; k += blockDim.x) acc += static_cast<double>(xi[k]) * xf[k];
    __shared__ double red[256];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int off = blockDim.x / 2; off; off >>= 1) {
        if (static_cast<int>(threadIdx.x) < off) red[threadIdx.x] += red[threadIdx.x + off];
        __syncthreads();
    }
    if (threadIdx.x == 0) a.xfa_dots[(static_cast<long long>(s) * a.n + i) * a.n + f] = red[0];
}

// 3. eps_i <- sum_f w_if eps_f (softmax in fp64 over the in-flight slots), then the
//    consistency step / emission exactly as the fused step kernel
template <int kMode>
__global__ void __launch_bounds__(256) xfa_step_kernel(StepArgs a) {
    const int s = blockIdx.z, slot = blockIdx.y;
    const StreamCtl* cp = a.ctl + s;
    if (!cp->tick_now) return;
    const SlotCtl sc = cp->slot[slot];
    if (sc.seq < 0) return;
    __shared__ float w[kMaxSteps];
    if (threadIdx.x == 0) {
        const double* dots = a.xfa_dots + (static_cast<long long>(s) * a.n + slot) * a.n;
        const double inv_sqrt_d = 1.0 / sqrt(static_cast<double>(a.d));
        double mx = -INFINITY;
        for (int f = 0; f < a.n; ++f)
            if (cp->slot[f].seq >= 0) mx = fmax(mx, dots[f] * inv_sqrt_d);
        double den = 0.0;
        for (int f = 0; f < a.n; ++f)
            if (cp->slot[f].seq >= 0) den += exp(dots[f] * inv_sqrt_d - mx);
        for (int f = 0; f < a.n; ++f)
            w[f] = cp->slot[f].seq >= 0 ? static_cast<float>(exp(dots[f] * inv_sqrt_d - mx) / den) : 0.f;
    }
    __syncthreads();
    const int step = static_cast<int>(cp->ticks - sc.ingest_tick);
    const bool terminal = step + 1 >= a.n;
    const StepScalars st = a.tbl[step];
    const StepScalars nx = a.tbl[terminal ? a.n : step + 1];
    const long long d = a.d;
    const long long sd = static_cast<long long>(s) * a.n + slot;
    float* xcur = a.x_cur + sd * d;
    const float* ren = terminal ? nullptr : a.eps_cached + (static_cast<long long>(s) * a.n + step + 1) * d;
    float* out = terminal ? a.emitted + static_cast<long long>(s) * d : xcur;
    const float* eps_s = a.xfa_eps + static_cast<long long>(s) * a.n * d;
    int bad = 0;
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < d;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        float e = 0.f;
        for (int f = 0; f < a.n; ++f)
            if (w[f] != 0.f) e = fmaf(w[f], eps_s[static_cast<long long>(f) * d + i], e);
        const float y = update1(xcur[i], e, terminal ? 0.f : ren[i], st, nx, terminal);
        if (terminal && !isfinite(y)) bad = 1;
        out[i] = y;
    }
    if (terminal) {
        bad = __syncthreads_or(bad);
        if (bad && threadIdx.x == 0) atomicOr(&a.ctl[s].nonfinite, 1);
    }
}

template <int kMode, bool kExt>
void launch_xfa(const StepArgs& a, int S, cudaStream_t st) {
    long long blocks = (a.d + 255) / 256;
    if (blocks > 1024) blocks = 1024;
    const dim3 grid(static_cast<unsigned>(blocks), a.n, S);
    xfa_eps_kernel<kMode, kExt><<<grid, 256, 0, st>>>(a);
    xfa_dots_kernel<<<dim3(a.n, a.n, S), 256, 0, st>>>(a);
    xfa_step_kernel<kMode><<<grid, 256, 0, st>>>(a);
}

template <int kMode, bool kExt>
void launch_mode(const StepArgs& a, int S, cudaStream_t st) {
    if (a.xfa_eps) {
        launch_xfa<kMode, kExt>(a, S, st);
        return;
    }
    const int threads = 256;
    const bool vec = (a.d % 4) == 0;
    const long long per_block = threads * (vec ? 8 : 1);
    long long blocks = (a.d + per_block - 1) / per_block;
    if (blocks < 1) blocks = 1;
    if (blocks > 65535) blocks = 65535;
    dim3 grid(static_cast<unsigned>(blocks), a.n, S);
    if (vec) step_vec_kernel<kMode, kExt><<<grid, threads, 0, st>>>(a);
    else step_scalar_kernel<kMode, kExt><<<grid, threads, 0, st>>>(a);
}

template <bool kExt>
void launch_ext(const StepArgs& a, int S, cudaStream_t st) {
    switch (a.guidance) {
        case SDX_GUIDANCE_NONE: launch_mode<SDX_GUIDANCE_NONE, kExt>(a, S, st); break;
        case SDX_GUIDANCE_CFG: launch_mode<SDX_GUIDANCE_CFG, kExt>(a, S, st); break;
        case SDX_GUIDANCE_SELF_NEGATIVE: launch_mode<SDX_GUIDANCE_SELF_NEGATIVE, kExt>(a, S, st); break;
        default: launch_mode<SDX_GUIDANCE_ONETIME_NEGATIVE, kExt>(a, S, st); break;
    }
}

}  // namespace

void launch_step(const StepArgs& a, int S, cudaStream_t st) {
    if (a.eps_ext) launch_ext<true>(a, S, st);
    else launch_ext<false>(a, S, st);
    SDX_LAUNCH_CHECK();
}

}  // namespace sdx
