// Element-wise Adam step and bf16 packing shared by K3 (sync_update.cu) and
// the fused peer exchange + update (peer.cu): one definition, so both paths
// produce bit-identical parameters.
#pragma once
#include <cuda_bf16.h>

#include "mmb200.h"

__device__ __forceinline__ void adam_elem(float g, float& p, float& m, float& v, float step_size,
                                          float inv_sqrt_bc2, const mm_adam_hyper& hp) {
    if (hp.weight_decay != 0.f) g = fmaf(hp.weight_decay, p, g);
    // torch.optim.Adam (single-tensor path): lerp for m, mul/addcmul for v,
    // denom = sqrt(v)/sqrt(bc2) + eps, p -= step_size * m / denom
    m = fmaf(hp.one_minus_beta1, g - m, m);
    v = fmaf(hp.one_minus_beta2, g * g, hp.beta2 * v);
    const float denom = sqrtf(v) * inv_sqrt_bc2 + hp.eps;
    p = p - step_size * __fdiv_rn(m, denom);
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}
