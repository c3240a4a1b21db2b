// K5: packed varlen multi-head attention for short NMT sentences (lengths
// 4..256), head_dim 64.  One CTA per (sequence, head); the sequence's K / V
// (and Q / dO in backward) are staged in shared memory as bf16 pairs with a
// 33-word row pitch so lane-parallel row accesses are bank-conflict free.
// Softmax statistics are fp32; the forward saves the natural-log LSE per
// (head, query) for the backward's recomputation.  Attention is <1 % of the
// step's FLOPs at these lengths, so this kernel is sized for
// latency (thousands of small CTAs), not for the tensor pipe.
#include <cuda_bf16.h>

#include <algorithm>

#include "mm_common.h"

namespace {

constexpr int kHd = 64;       // head dim
constexpr int kWords = 32;    // bf16 pairs per head row
constexpr int kPitch = 33;    // padded smem row pitch (words)
constexpr int kWarps = 4;

__device__ __forceinline__ float2 unpack(uint32_t w) {
    return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
}
__device__ __forceinline__ uint32_t pack(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float dot_row(const uint32_t* a, const uint32_t* b) {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < kWords; ++w) {
        const float2 x = unpack(a[w]), y = unpack(b[w]);
        s = fmaf(x.x, y.x, s);
        s = fmaf(x.y, y.y, s);
    }
    return s;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// rows [0, n) of a head slice -> smem with pitch kPitch (words)
__device__ __forceinline__ void stage(uint32_t* dst, const uint16_t* src, int64_t ld, int n) {
    for (int idx = threadIdx.x; idx < n * kWords; idx += blockDim.x) {
        const int r = idx / kWords, w = idx % kWords;
        dst[r * kPitch + w] = reinterpret_cast<const uint32_t*>(src + r * ld)[w];
    }
}

__global__ void __launch_bounds__(kWarps * 32) attn_fwd_kernel(const mm_attn_args a) {
    extern __shared__ uint32_t sm[];
    const int seq = blockIdx.x, h = blockIdx.y;
    const int q0 = a.cu_q[seq], lq = a.cu_q[seq + 1] - q0;
    const int k0 = a.cu_k[seq], lk = a.cu_k[seq + 1] - k0;
    uint32_t* Ks = sm;
    uint32_t* Vs = Ks + a.max_k * kPitch;
    uint32_t* Qs = Vs + a.max_k * kPitch;             // per-warp query row
    float* Ps = reinterpret_cast<float*>(Qs + kWarps * kWords);  // per-warp probs
    stage(Ks, a.k + int64_t(k0) * a.ldk + h * kHd, a.ldk, lk);
    stage(Vs, a.v + int64_t(k0) * a.ldv + h * kHd, a.ldv, lk);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t* qrow = Qs + warp * kWords;
    float* P = Ps + warp * a.max_k;
    for (int i = warp; i < lq; i += kWarps) {
        qrow[lane] = reinterpret_cast<const uint32_t*>(a.q + int64_t(q0 + i) * a.ldq + h * kHd)[lane];
        __syncwarp();
        const int kend = a.causal ? min(lk, i + 1) : lk;
        float mx = -INFINITY;
        for (int j = lane; j < kend; j += 32) {
            const float s = dot_row(qrow, Ks + j * kPitch) * a.scale;
            P[j] = s;
            mx = fmaxf(mx, s);
        }
        mx = warp_max(mx);
        float sum = 0.f;
        for (int j = lane; j < kend; j += 32) {
            const float e = __expf(P[j] - mx);
            P[j] = e;
            sum += e;
        }
        sum = warp_sum(sum);
        __syncwarp();
        float ox = 0.f, oy = 0.f;
        for (int j = 0; j < kend; ++j) {
            const float2 v = unpack(Vs[j * kPitch + lane]);
            ox = fmaf(P[j], v.x, ox);
            oy = fmaf(P[j], v.y, oy);
        }
        const float inv = 1.f / sum;
        reinterpret_cast<uint32_t*>(a.o + int64_t(q0 + i) * a.ldo + h * kHd)[lane] =
            pack(ox * inv, oy * inv);
        if (lane == 0) a.lse[int64_t(h) * a.total_q + q0 + i] = mx + __logf(sum);
        __syncwarp();
    }
}

__global__ void __launch_bounds__(kWarps * 32) attn_bwd_kernel(const mm_attn_args a) {
    extern __shared__ uint32_t sm[];
    const int seq = blockIdx.x, h = blockIdx.y;
    const int q0 = a.cu_q[seq], lq = a.cu_q[seq + 1] - q0;
    const int k0 = a.cu_k[seq], lk = a.cu_k[seq + 1] - k0;
    const int mrow = max(a.max_q, a.max_k);
    uint32_t* Qs = sm;
    uint32_t* dOs = Qs + a.max_q * kPitch;
    uint32_t* Ks = dOs + a.max_q * kPitch;
    uint32_t* Vs = Ks + a.max_k * kPitch;
    float* lse = reinterpret_cast<float*>(Vs + a.max_k * kPitch);
    float* Dd = lse + a.max_q;
    float* Pw = Dd + a.max_q;            // per warp: P then DS, mrow each
    stage(Qs, a.q + int64_t(q0) * a.ldq + h * kHd, a.ldq, lq);
    stage(dOs, a.d_o + int64_t(q0) * a.ldo + h * kHd, a.ldo, lq);
    stage(Ks, a.k + int64_t(k0) * a.ldk + h * kHd, a.ldk, lk);
    stage(Vs, a.v + int64_t(k0) * a.ldv + h * kHd, a.ldv, lk);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < lq; i += blockDim.x) lse[i] = a.lse[int64_t(h) * a.total_q + q0 + i];
    __syncthreads();
    float* P = Pw + warp * 2 * mrow;
    float* DS = P + mrow;
    // phase A: D_i = sum_j p_ij dp_ij computed exactly in fp32 (not from the
    // bf16-rounded O: dp - D cancels strongly in cross attention), then
    // dQ_i = scale * sum_j p_ij (dp_ij - D_i) K_j
    for (int i = warp; i < lq; i += kWarps) {
        const int kend = a.causal ? min(lk, i + 1) : lk;
        const uint32_t* qi = Qs + i * kPitch;
        const uint32_t* di = dOs + i * kPitch;
        float part = 0.f;
        for (int j = lane; j < kend; j += 32) {
            const float p = __expf(dot_row(qi, Ks + j * kPitch) * a.scale - lse[i]);
            const float dp = dot_row(di, Vs + j * kPitch);
            P[j] = p;
            DS[j] = dp;
            part = fmaf(p, dp, part);
        }
        const float Di = warp_sum(part);
        if (lane == 0) Dd[i] = Di;
        for (int j = lane; j < kend; j += 32) DS[j] = P[j] * (DS[j] - Di);
        __syncwarp();
        float gx = 0.f, gy = 0.f;
        for (int j = 0; j < kend; ++j) {
            const float2 kk = unpack(Ks[j * kPitch + lane]);
            gx = fmaf(DS[j], kk.x, gx);
            gy = fmaf(DS[j], kk.y, gy);
        }
        reinterpret_cast<uint32_t*>(a.dq + int64_t(q0 + i) * a.ld_dq + h * kHd)[lane] =
            pack(gx * a.scale, gy * a.scale);
        __syncwarp();
    }
    __syncthreads();  // every D_i is needed by every warp in phase B
    // phase B: dV_j = sum_i p_ij dO_i ; dK_j = scale * sum_i ds_ij Q_i
    for (int j = warp; j < lk; j += kWarps) {
        const int ibeg = a.causal ? j : 0;
        const uint32_t* kj = Ks + j * kPitch;
        const uint32_t* vj = Vs + j * kPitch;
        for (int i = ibeg + lane; i < lq; i += 32) {
            const float p = __expf(dot_row(Qs + i * kPitch, kj) * a.scale - lse[i]);
            const float dp = dot_row(dOs + i * kPitch, vj);
            P[i] = p;
            DS[i] = p * (dp - Dd[i]);
        }
        __syncwarp();
        float vx = 0.f, vy = 0.f, kx = 0.f, ky = 0.f;
        for (int i = ibeg; i < lq; ++i) {
            const float2 d = unpack(dOs[i * kPitch + lane]);
            const float2 q = unpack(Qs[i * kPitch + lane]);
            vx = fmaf(P[i], d.x, vx);
            vy = fmaf(P[i], d.y, vy);
            kx = fmaf(DS[i], q.x, kx);
            ky = fmaf(DS[i], q.y, ky);
        }
        reinterpret_cast<uint32_t*>(a.dv + int64_t(k0 + j) * a.ld_dv + h * kHd)[lane] = pack(vx, vy);
        reinterpret_cast<uint32_t*>(a.dk + int64_t(k0 + j) * a.ld_dk + h * kHd)[lane] =
            pack(kx * a.scale, ky * a.scale);
        __syncwarp();
    }
}

size_t fwd_smem(const mm_attn_args& a) {
    return (size_t(2) * a.max_k * kPitch + kWarps * kWords) * 4 + size_t(kWarps) * a.max_k * 4;
}
size_t bwd_smem(const mm_attn_args& a) {
    const int mrow = std::max(a.max_q, a.max_k);
    return (size_t(2) * a.max_q * kPitch + size_t(2) * a.max_k * kPitch) * 4 +
           size_t(2) * a.max_q * 4 + size_t(kWarps) * 2 * mrow * 4;
}

int check(const mm_attn_args* a, bool bwd) {
    MM_CHECK_ARG(a != nullptr, "args is NULL");
    MM_CHECK_ARG(a->head_dim == kHd, "head_dim must be 64 (got %d)", a->head_dim);
    MM_CHECK_ARG(a->q && a->k && a->v && a->o && a->lse && a->cu_q && a->cu_k, "NULL tensor");
    MM_CHECK_ARG(a->n_seq >= 0 && a->heads > 0 && a->max_q > 0 && a->max_k > 0, "bad sizes");
    MM_CHECK_ARG(a->max_q <= 1024 && a->max_k <= 1024, "sequence longer than 1024");
    MM_CHECK_ARG(!bwd || (a->d_o && a->dq && a->dk && a->dv), "NULL gradient tensor");
    return 0;
}

}  // namespace

extern "C" int mm_attention_fwd(const mm_attn_args* a, void* stream) {
    if (int st = check(a, false)) return st;
    if (a->n_seq == 0) return 0;
    const size_t smem = fwd_smem(*a);
    MM_CUDA_TRY(cudaFuncSetAttribute(attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
    attn_fwd_kernel<<<dim3(a->n_seq, a->heads), kWarps * 32, smem, mm::as_stream(stream)>>>(*a);
    MM_LAUNCH_CHECK("attn_fwd_kernel");
    return 0;
}

extern "C" int mm_attention_bwd(const mm_attn_args* a, void* stream) {
    if (int st = check(a, true)) return st;
    if (a->n_seq == 0) return 0;
    const size_t smem = bwd_smem(*a);
    MM_CHECK_ARG(smem <= 227 * 1024, "attention backward needs %zu B of smem", smem);
    MM_CUDA_TRY(cudaFuncSetAttribute(attn_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
    attn_bwd_kernel<<<dim3(a->n_seq, a->heads), kWarps * 32, smem, mm::as_stream(stream)>>>(*a);
    MM_LAUNCH_CHECK("attn_bwd_kernel");
    return 0;
}
