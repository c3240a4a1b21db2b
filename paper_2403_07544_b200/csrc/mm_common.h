// Shared plumbing for libmmb200: error reporting and launch helpers.
#pragma once
#include <cuda_runtime.h>
#include <cstdarg>
#include <cstdio>
#include <string>

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

}  // namespace mm

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
