// Shared plumbing for libmmb200: error reporting and launch helpers.
#pragma once
#include <cuda_runtime.h>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <string>
#include <utility>

#include "mmb200.h"

namespace mm {

void set_error(const char* fmt, ...);

enum Status { kOk = 0, kArg = -1, kCuda = -2, kNccl = -3, kUnsupported = -4 };

inline int cuda_status(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return kOk;
    set_error("%s: %s", what, cudaGetErrorString(e));
    return kCuda;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int num_sms();

// programmatic dependent launch on (default) or off (MM_NO_PDL=1, diagnostics)
bool pdl_enabled();

// every kernel launch of the library (bench.py's gpu_launches; mm_launch_count)
extern std::atomic<unsigned long long> g_launches;

// Programmatic dependent launch: every kernel of the library is launched with
// programmatic stream serialization, waits (griddepcontrol.wait) before its
// first global-memory access and signals launch_dependents when its main work
// is issued, so the next kernel's launch and prologue (barrier init, TMEM
// allocation, descriptor prefetch) overlap this kernel's tail.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_cluster(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                      cudaStream_t s, unsigned cluster_x, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = cluster_x;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = cluster_x > 1 ? 2 : 1;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args&&... args) {
    return launch_pdl_cluster(kern, grid, block, smem, s, 1u, std::forward<Args>(args)...);
}

}  // namespace mm

#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// Small memory-bound kernels release their dependent right after their own
// wait: the next kernel (typically a GEMM, one 225 KB CTA per SM) then gets
// its CTAs resident beside this grid's blocks and runs its prologue (barrier
// init, TMEM allocation, descriptor prefetch, weight-tile prefetch) before
// its griddepcontrol.wait -- which still waits for this whole grid.
__device__ __forceinline__ void pdl_wait_release() {
    pdl_wait();
    pdl_trigger();
}
// Device-side bounds / invariant checks of the debug build
// (tools/build_variant.py dbg --all -DMM_DEBUG_BOUNDS): the failing condition
// is printed and the kernel traps, so the launch's stream reports an error.
// compute-sanitizer is closed on the GPU pool; the GPU test suite runs
// against this build instead (profiles/r02_debug_bounds.txt).
#ifdef MM_DEBUG_BOUNDS
#include <cstdio>
#define MM_DCHECK(cond)                                                                      \
    do {                                                                                     \
        if (!(cond)) {                                                                       \
            printf("MM_DCHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__,     \
                   (int)blockIdx.x, (int)threadIdx.x, #cond);                                \
            __trap();                                                                        \
        }                                                                                    \
    } while (0)
#else
#define MM_DCHECK(cond) \
    do {                \
    } while (0)
#endif
#endif

#define MM_CHECK_ARG(cond, ...)              \
    do {                                     \
        if (!(cond)) {                       \
            mm::set_error(__VA_ARGS__);      \
            return mm::kArg;                 \
        }                                    \
    } while (0)

#define MM_CUDA_TRY(expr)                                         \
    do {                                                          \
        cudaError_t _e = (expr);                                  \
        if (_e != cudaSuccess) return mm::cuda_status(_e, #expr); \
    } while (0)

#define MM_LAUNCH_CHECK(name) MM_CUDA_TRY(cudaGetLastError())
