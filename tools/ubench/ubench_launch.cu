// Kernel-boundary cost inside a CUDA graph: 100 back-to-back launches of a
// near-empty kernel shaped like the UNet's GEMMs (148 CTAs, 448 threads), with
// and without programmatic dependent launch (PDL), with a large dynamic smem
// footprint (one CTA per SM, so the next kernel's CTAs cannot co-reside), with
// a TMEM alloc/dealloc, and with a dependent global read after griddepcontrol.wait.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <bool TMEM, bool READ>
__global__ void k_empty(float* buf, int n) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    extern __shared__ uint8_t sm[];
    __shared__ uint32_t slot;
    if (TMEM && threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&slot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    __syncthreads();
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (READ) {
        // one dependent read + write per CTA (what the next kernel consumes)
        if (threadIdx.x == 0) buf[blockIdx.x] = buf[(blockIdx.x + 1) % gridDim.x] + 1.f;
    }
    if (threadIdx.x == 0) sm[0] = 1;
    __syncthreads();
    if (TMEM && threadIdx.x < 32) {
        const uint32_t t = slot;
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(t) : "memory");
    }
}

template <bool TMEM, bool READ>
float run(int smem, bool pdl, float* buf) {
    auto kern = k_empty<TMEM, READ>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148);
    cfg.blockDim = dim3(448);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const int N = 100;
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < N; ++i) cudaLaunchKernelEx(&cfg, kern, buf, 148);
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, st);
    cudaStreamSynchronize(st);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a, st);
        cudaGraphLaunch(ge, st);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
    }
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaStreamDestroy(st);
    return best * 1000.f / N;
}

int main() {
    float* buf;
    cudaMalloc(&buf, 4096 * sizeof(float));
    cudaMemset(buf, 0, 4096 * sizeof(float));
    for (int pdl = 0; pdl < 2; ++pdl) {
        for (int smem : {1024, 100 * 1024, 200 * 1024}) {
            printf("pdl %d smem %3d KB: plain %.2f us, +read %.2f us, +tmem %.2f us, +tmem+read %.2f us per launch\n", pdl,
                   smem / 1024, run<false, false>(smem, pdl, buf), run<false, true>(smem, pdl, buf),
                   run<true, false>(smem, pdl, buf), run<true, true>(smem, pdl, buf));
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
