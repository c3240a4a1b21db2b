// Element-wise Adam step and bf16 packing shared by K3 (sync_update.cu) and
// the fused peer exchange + update (peer.cu): one definition, so both paths
// produce bit-identical parameters.
#pragma once
#include <cuda_bf16.h>

#include "mmb200.h"

// Every operation is an explicitly rounded intrinsic: no FMA contraction is
// left to the compiler, so each inlined copy (the update kernels, the GEMM's
// MM_EPI_F32_ADAM epilogue) computes the same bits.
__device__ __forceinline__ void adam_elem(float g, float& p, float& m, float& v, float step_size,
                                          float inv_sqrt_bc2, const mm_adam_hyper& hp) {
    if (hp.weight_decay != 0.f) g = __fmaf_rn(hp.weight_decay, p, g);
    // torch.optim.Adam (single-tensor path): lerp for m, mul/addcmul for v,
    // denom = sqrt(v)/sqrt(bc2) + eps, p -= step_size * m / denom
    m = __fmaf_rn(hp.one_minus_beta1, __fsub_rn(g, m), m);
    v = __fmaf_rn(hp.one_minus_beta2, __fmul_rn(g, g), __fmul_rn(hp.beta2, v));
    const float denom = __fmaf_rn(__fsqrt_rn(v), inv_sqrt_bc2, hp.eps);
    p = __fmaf_rn(-step_size, __fdiv_rn(m, denom), p);
}
// Algorithm 1's rescale: the group sum / n ready members, times the loss unscale
__device__ __forceinline__ float adam_grad(float sum, float n, float unscale) {
    return __fmul_rn(__fdiv_rn(sum, n), unscale);
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}
