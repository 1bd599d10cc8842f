// tcgen05 / TMA GEMM + implicit-GEMM conv3x3 (see gemm_sm100.cuh).
//
// One 128 x BN output tile per CTA, 6 warps:
//   warp 0      TMA producer (one elected lane): A and B K-slices (64 wide,
//               128-byte swizzle) into a STAGES-deep smem ring (full/empty mbarriers)
//   warp 1      TMEM allocation + MMA issuer (one lane): 4 x tcgen05.mma
//               (M=128, N=BN, K=16) per stage, tcgen05.commit frees the stage
//   warps 2..5  epilogue: tcgen05.ld 32 lanes x 16 columns, bias / per-image
//               bias / activation / residual in fp32, bf16 or fp32 stores
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include "gemm_sm100.cuh"
#include "sm100.cuh"

namespace sdx {

using namespace sm100;

namespace {

struct GemmArgs {
    int M, N, K, K1, amode;
    int Ho, Wo, Cin, stride, Wt, Ht, Nt;
    GemmEpilogue epi;
};

__device__ __forceinline__ void wait_bounded(uint64_t* bar, uint32_t phase) {
    // mbarrier wait with a watchdog: a protocol bug traps instead of hanging the GPU
    const uint32_t a = smem_u32(bar);
    uint32_t done = 0;
    long long t0 = clock64();
    while (true) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(a), "r"(phase)
            : "memory");
        if (done) return;
        if (clock64() - t0 > (1LL << 33)) {
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

// bias / per-image bias / residual / activation on 16 accumulator columns of
// one row, then a bf16, fp32 or u8 store.
__device__ __forceinline__ void epilogue16(const GemmEpilogue& e, int N, long long row, long long orow, int col0,
                                           const float* bimg, float* v) {
    const bool full16 = col0 + 16 <= N;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const int col = col0 + i;
        float x = v[i] * e.scale;
        if (full16 || col < N) {
            if (e.bias) x += e.bias[col];
            if (bimg) x += bimg[col];
        }
        v[i] = x;
    }
    if (!e.act_after_residual) {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = act_fn(v[i], e.act);
    }
    if (e.residual) {
        const __nv_bfloat16* rp = e.residual + row * e.ld_res + col0;
        if (full16) {
            const uint4 r0 = *reinterpret_cast<const uint4*>(rp);
            const uint4 r1 = *reinterpret_cast<const uint4*>(rp + 8);
            const __nv_bfloat16* rb0 = reinterpret_cast<const __nv_bfloat16*>(&r0);
            const __nv_bfloat16* rb1 = reinterpret_cast<const __nv_bfloat16*>(&r1);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                v[i] += __bfloat162float(rb0[i]);
                v[8 + i] += __bfloat162float(rb1[i]);
            }
        } else {
            for (int i = 0; i < 16 && col0 + i < N; ++i) v[i] += __bfloat162float(rp[i]);
        }
    }
    if (e.act_after_residual) {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = act_fn(v[i], e.act);
    }
    if (e.out_f32 == 1) {
        float* op = reinterpret_cast<float*>(e.out) + orow * e.ld_out + col0;
        if (full16) {
#pragma unroll
            for (int i = 0; i < 16; i += 4) *reinterpret_cast<float4*>(op + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
        } else {
            for (int i = 0; i < 16 && col0 + i < N; ++i) op[i] = v[i];
        }
    } else if (e.out_f32 == 2) {
        uint8_t* op = reinterpret_cast<uint8_t*>(e.out) + orow * e.ld_out + col0;
        for (int i = 0; i < 16 && col0 + i < N; ++i)
            op[i] = static_cast<uint8_t>(__float2int_rn(fminf(fmaxf(v[i], 0.f), 1.f) * 255.f));
    } else {
        __nv_bfloat16* op = reinterpret_cast<__nv_bfloat16*>(e.out) + orow * e.ld_out + col0;
        if (full16) {
            uint4 o0, o1;
            o0.x = pack_bf16(v[0], v[1]);
            o0.y = pack_bf16(v[2], v[3]);
            o0.z = pack_bf16(v[4], v[5]);
            o0.w = pack_bf16(v[6], v[7]);
            o1.x = pack_bf16(v[8], v[9]);
            o1.y = pack_bf16(v[10], v[11]);
            o1.z = pack_bf16(v[12], v[13]);
            o1.w = pack_bf16(v[14], v[15]);
            *reinterpret_cast<uint4*>(op) = o0;
            *reinterpret_cast<uint4*>(op + 8) = o1;
        } else {
            for (int i = 0; i < 16 && col0 + i < N; ++i) op[i] = __float2bfloat16(v[i]);
        }
    }
}

template <int BN, int STAGES, int AMODE>
__global__ void __launch_bounds__(192, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap ta2,
                   const __grid_constant__ CUtensorMap tb, const GemmArgs g) {
    constexpr int BM = 128, BK = 64;
    constexpr uint32_t A_BYTES = BM * BK * 2;
    constexpr uint32_t B_BYTES = BN * BK * 2;
    constexpr uint32_t TMEM_COLS = BN < 32 ? 32 : BN;

    const int n_tile = blockIdx.x;
    const int m_tile = blockIdx.y;
    const int m0 = m_tile * BM;
    const int n0 = n_tile * BN;
    int m_eff = g.M;
    if (g.epi.rows_dev) {
        const long long lim = static_cast<long long>(*g.epi.rows_dev) * g.epi.rows_per_unit;
        if (lim < m_eff) m_eff = static_cast<int>(lim);
    }
    if (m0 >= m_eff) return;  // device-decided batch: rows past the live count do no work

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* done = empty + STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int nk = g.K / BK;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&ta);
        if (AMODE == kAConcat) tma_prefetch(&ta2);
        tma_prefetch(&tb);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // conv tile origin in output space
            int cn0 = 0, cy0 = 0, cx0 = 0;
            if (AMODE == kAConv) {
                const int hw = g.Ho * g.Wo;
                cn0 = m0 / hw;
                const int rem = m0 - cn0 * hw;
                cy0 = rem / g.Wo;
                cx0 = rem - cy0 * g.Wo;
            }
            const int cblocks = AMODE == kAConv ? g.Cin / BK : 1;
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % STAGES;
                const uint32_t ph = (kb / STAGES) & 1;
                wait_bounded(&empty[s], ph ^ 1);
                mbar_expect_tx(&full[s], A_BYTES + B_BYTES);
                uint8_t* dA = sA + s * A_BYTES;
                if (AMODE == kAMatrix) {
                    tma_load_2d(dA, &ta, &full[s], kb * BK, m0);
                } else if (AMODE == kAConcat) {
                    const int k1b = g.K1 / BK;
                    if (kb < k1b) tma_load_2d(dA, &ta, &full[s], kb * BK, m0);
                    else tma_load_2d(dA, &ta2, &full[s], (kb - k1b) * BK, m0);
                } else {
                    const int tap = kb / cblocks;
                    const int cb = kb - tap * cblocks;
                    const int dy = tap / 3, dx = tap - dy * 3;
                    tma_load_4d(dA, &ta, &full[s], cb * BK, cx0 * g.stride + dx - 1, cy0 * g.stride + dy - 1, cn0);
                }
                tma_load_2d(sB + s * B_BYTES, &tb, &full[s], kb * BK, n0);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_bf16(BM, BN);
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % STAGES;
                const uint32_t ph = (kb / STAGES) & 1;
                wait_bounded(&full[s], ph);
                tc_fence_after();
                const uint64_t da = desc_kmajor_sw128(smem_u32(sA + s * A_BYTES));
                const uint64_t db = desc_kmajor_sw128(smem_u32(sB + s * B_BYTES));
#pragma unroll
                for (int k = 0; k < BK / 16; ++k)  // +32 bytes per K=16 step inside the swizzle atom
                    umma_f16(tmem, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
                umma_commit(&empty[s]);
            }
            umma_commit(done);
        }
        __syncwarp();
    } else {
        // epilogue warps 2..5 -> TMEM lane quadrants 2,3,0,1
        const int q = warp & 3;
        wait_bounded(done, 0);
        tc_fence_after();
        const int row = m0 + q * 32 + lane;
        const bool row_ok = row < m_eff;
        const GemmEpilogue& e = g.epi;
        const float* bimg = nullptr;
        long long orow = row;  // destination row (scatter by image when out_img_map is set)
        if (row_ok) {
            const long long im = static_cast<long long>(row) / e.rows_per_img;
            if (e.bias_img)
                bimg = e.bias_img + (e.img_index ? e.img_index[im] : im) * (e.bias_img_ld ? e.bias_img_ld : g.N);
            if (e.out_img_map) orow = static_cast<long long>(e.out_img_map[im]) * e.rows_per_img + (row - im * e.rows_per_img);
        }
#pragma unroll 1
        for (int c = 0; c < BN; c += 16) {
            float v[16];
            tmem_ld16(tmem + (static_cast<uint32_t>(q * 32) << 16) + c, v);
            const int col0 = n0 + c;
            if (!row_ok || col0 >= g.N) continue;
            epilogue16(e, g.N, row, orow, col0, bimg, v);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, TMEM_COLS);
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
            const cuuint32_t* box, const cuuint32_t* estrides) {
    const CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(ptr), dims,
                                   strides_bytes, box, estrides, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
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

int pick_bn(int N) {
    if (N <= 64) return 64;
    if (N % 256 == 0 || N > 640) return 256;
    return 128;
}

template <int BN>
constexpr int stages_for() {
    return BN == 256 ? 4 : 6;
}

template <int BN>
size_t smem_for() {
    return static_cast<size_t>(stages_for<BN>()) * (128 * 64 * 2 + BN * 64 * 2) + 1024 + 256;
}

template <int BN, int AMODE>
void launch_t(const GemmPlan& p, cudaStream_t st) {
    constexpr int S = stages_for<BN>();
    auto k = gemm_tc_kernel<BN, S, AMODE>;
    static bool attr = false;
    const size_t smem = smem_for<BN>();
    if (!attr) {
        SDX_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        attr = true;
    }
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
    dim3 grid((p.N + BN - 1) / BN, (p.M + 127) / 128);
    k<<<grid, 192, smem, st>>>(p.ta, p.ta2, p.tb, g);
    SDX_LAUNCH_CHECK();
}

template <int AMODE>
void launch_mode(const GemmPlan& p, cudaStream_t st) {
    switch (p.bn) {
        case 64: launch_t<64, AMODE>(p, st); break;
        case 256: launch_t<256, AMODE>(p, st); break;
        default: launch_t<128, AMODE>(p, st); break;
    }
}

}  // namespace

GemmPlan plan_gemm(const __nv_bfloat16* A, long long lda, const __nv_bfloat16* B, long long ldb, int M, int N, int K,
                   const GemmEpilogue& epi) {
    if (K % 64 != 0) raise(SDX_INVALID_ARGUMENT, "gemm: K must be a multiple of 64");
    GemmPlan p;
    p.amode = kAMatrix;
    p.M = M;
    p.N = N;
    p.K = K;
    p.bn = pick_bn(N);
    encode_2d(&p.ta, A, M, K, lda, 128);
    p.ta2 = p.ta;
    encode_2d(&p.tb, B, N, K, ldb, p.bn);
    p.epi = epi;
    if (p.epi.ld_out == 0) p.epi.ld_out = N;
    if (p.epi.residual && p.epi.ld_res == 0) p.epi.ld_res = N;
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
    p.bn = pick_bn(N);
    encode_2d(&p.ta, A1, M, K1, lda1, 128);
    encode_2d(&p.ta2, A2, M, K - K1, lda2, 128);
    encode_2d(&p.tb, B, N, K, ldb, p.bn);
    p.epi = epi;
    if (p.epi.ld_out == 0) p.epi.ld_out = N;
    if (p.epi.residual && p.epi.ld_res == 0) p.epi.ld_res = N;
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
    p.bn = pick_bn(Cout);
    const cuuint64_t dims[4] = {static_cast<cuuint64_t>(Cin), static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H),
                                static_cast<cuuint64_t>(imgs)};
    const cuuint64_t strides[3] = {static_cast<cuuint64_t>(Cin) * 2, static_cast<cuuint64_t>(W) * Cin * 2,
                                   static_cast<cuuint64_t>(H) * W * Cin * 2};
    const cuuint32_t box[4] = {64, static_cast<cuuint32_t>(p.Wt * stride), static_cast<cuuint32_t>(p.Ht * stride),
                               static_cast<cuuint32_t>(p.Nt)};
    const cuuint32_t es[4] = {1, static_cast<cuuint32_t>(stride), static_cast<cuuint32_t>(stride), 1};
    encode(&p.ta, x, 4, dims, strides, box, es);
    p.ta2 = p.ta;
    encode_2d(&p.tb, w, Cout, 9LL * Cin, 9LL * Cin, p.bn);
    p.epi = epi;
    if (p.epi.ld_out == 0) p.epi.ld_out = Cout;
    if (p.epi.residual && p.epi.ld_res == 0) p.epi.ld_res = Cout;
    p.valid = true;
    return p;
}

void run_gemm(const GemmPlan& p, cudaStream_t st) {
    if (!p.valid) raise(SDX_LOGIC_ERROR, "run_gemm: invalid plan");
    switch (p.amode) {
        case kAConcat: launch_mode<kAConcat>(p, st); break;
        case kAConv: launch_mode<kAConv>(p, st); break;
        default: launch_mode<kAMatrix>(p, st); break;
    }
}

}  // namespace sdx
