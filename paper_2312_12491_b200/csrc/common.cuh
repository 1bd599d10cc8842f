// Shared helpers for the sm_100a streaming-denoise library.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>
#include <stdexcept>
#include <string>

#include "stagger_b200.h"

namespace sdx {

// Status-carrying exception used inside the library; the C-ABI layer turns it
// into an SDX_* return code plus a thread-local message.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void raise(int code, const std::string& msg) { throw Error(code, msg); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess)
        raise(SDX_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file +
                                  ":" + std::to_string(line) + ")");
}

#define SDX_CUDA(x) ::sdx::cuda_check((x), #x, __FILE__, __LINE__)
#define SDX_LAUNCH_CHECK() ::sdx::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

// ---- programmatic dependent launch (PDL) ---------------------------------------
// Kernels of the denoiser forward are launched with programmatic stream
// serialisation: a kernel may start (prologue, TMEM alloc, descriptor and
// weight prefetch) while its predecessor drains.  Every such kernel calls
// pdl_launch() early and pdl_wait() before touching memory written by earlier
// kernels (and before finishing), so ordering stays transitive.  SDX_PDL=0
// disables it (plain stream order).
inline bool pdl_enabled() {
    static const bool on = [] {
        const char* v = std::getenv("SDX_PDL");
        return !(v && v[0] == '0');
    }();
    return on;
}

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cuda_check(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...), "cudaLaunchKernelEx", __FILE__, __LINE__);
}

// Kernel attributes (dynamic smem above 48 KB, non-portable cluster sizes) belong
// to a device context: set them once per (kernel, device), under a lock, before the
// kernel's first launch on that device.  Pipelines on several GPUs in one process
// and concurrent plan creation on several threads are both safe.
template <typename... KArgs>
inline void ensure_kernel_attrs(void (*kern)(KArgs...), size_t smem, bool nonportable_cluster = false) {
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice", __FILE__, __LINE__);
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> done;  // value: smem set + 1
    std::lock_guard<std::mutex> lk(mu);
    size_t& have = done[{reinterpret_cast<const void*>(kern), dev}];
    if (have > smem) return;
    if (nonportable_cluster)
        cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
                   "cudaFuncSetAttribute", __FILE__, __LINE__);
    cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
               "cudaFuncSetAttribute", __FILE__, __LINE__);
    have = smem + 1;
}

#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#endif

constexpr int kMaxSteps = 64;     // n_steps upper bound for device slot tables
constexpr int kSmCount = 148;     // B200

template <class T>
inline T* dev_alloc(size_t count) {
    if (count == 0) return nullptr;
    void* p = nullptr;
    SDX_CUDA(cudaMalloc(&p, count * sizeof(T)));
    return static_cast<T*>(p);
}

inline void dev_free(void* p) {
    if (p) cudaFree(p);
}

// Per-step scalar table, computed on the host in fp64 from build_schedule /
// lcm_coefficients (schedule.cpp:29-107) and consumed in fp64 on device.
struct StepScalars {
    double sa, sb;          // sqrt(alpha), sqrt(beta)
    double c_skip, c_out;   // LCM output parameterisation at this step
    double an_scale;        // analytic denoiser: sqrt(beta) / (alpha*var + beta)
    double beta;            // raw beta (R-CFG falls back to eps_cond when beta <= 0)
    double alpha;
    int tau;
    int pad;
    // fp32 copies for the device step (inverses precomputed in fp64)
    float f_sa, f_sb, f_isa, f_isb, f_cs, f_co, f_an, f_beta;
};

}  // namespace sdx
