// K5 for head_dim below 64: config 1's true shape (d_model 64, 4 heads,
// head_dim 16 -- BASELINE configs[0], the reference's CPU-runnable case),
// which the tcgen05 kernels (64-column head boxes) do not take.
//
// Same contract as mm_attention_fwd / _bwd (include/mmb200.h): packed
// varlen sequences (cu_q / cu_k), top-left causal mask (query i sees keys
// j <= i, as oracle/transformer.py's triu(1) fill), natural-log LSE per
// (head, query), dQ / dK / dV overwritten.  Softmax of one query row of the
// reference's attention (oracle/transformer.py _attention, replacing the toy
// model's layer of syncsim.py:34-87).
//
// At these sizes (sentences of <= 32 tokens, 16-wide heads) a step is a few
// thousand dot products of 16 elements: CUDA-core fp32 kernels, one CTA per
// (sequence, head), a warp per query row (forward, dQ) or key row (dK, dV),
// lanes across keys / queries for the scores and across head dimensions for
// the products.  Everything stays fp32 (P and dS are not rounded to bf16),
// D_i = sum_j p_ij dp_ij is exact, and every sum has a fixed order:
// bitwise reproducible, no atomics.
#include <cuda_bf16.h>

#include <cmath>

#include "mm_common.h"

namespace {

constexpr int kWarps = 8;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ float bf(uint16_t h) { return __uint_as_float(uint32_t(h) << 16); }

__device__ __forceinline__ uint16_t to_bf(float f) {
    const __nv_bfloat16 b = __float2bfloat16_rn(f);
    return *reinterpret_cast<const uint16_t*>(&b);
}

__device__ __forceinline__ float wsum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

__device__ __forceinline__ float wmax(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(kFull, v, o));
    return v;
}

// one head row (HD bf16, 16-byte aligned) into fp32 registers
template <int HD>
__device__ __forceinline__ void load_row(const uint16_t* p, float (&r)[HD]) {
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
        const uint4 u = reinterpret_cast<const uint4*>(p)[i];
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            r[8 * i + 2 * j] = __uint_as_float(w[j] << 16);
            r[8 * i + 2 * j + 1] = __uint_as_float(w[j] & 0xffff0000u);
        }
    }
}

// the sequence's rows of one head into shared memory (n rows of HD bf16)
template <int HD>
__device__ __forceinline__ void stage_rows(uint16_t* dst, const uint16_t* src, int64_t ld, int n) {
    for (int t = threadIdx.x; t < n * (HD / 8); t += blockDim.x) {
        const int r = t / (HD / 8), c = t - r * (HD / 8);
        reinterpret_cast<uint4*>(dst + r * HD)[c] = reinterpret_cast<const uint4*>(src + int64_t(r) * ld)[c];
    }
}

template <int HD>
__device__ __forceinline__ float dot(const float (&a)[HD], const float (&b)[HD]) {
    float t = 0.f;
#pragma unroll
    for (int d = 0; d < HD; ++d) t = fmaf(a[d], b[d], t);
    return t;
}

// forward: warp per query row; lanes take 32 keys per chunk (scores, online
// softmax in the exp2 domain), then lane d < HD accumulates o[d] over the
// chunk's keys in key order
template <int HD>
__global__ void __launch_bounds__(kWarps * 32) attn_small_fwd_kernel(const mm_attn_args a) {
    extern __shared__ uint4 smem_fwd[];  // K then V rows of this (sequence, head)
    pdl_wait_release();
    const int s = blockIdx.x, h = blockIdx.y;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int q0 = a.cu_q[s], lq = a.cu_q[s + 1] - q0;
    const int k0 = a.cu_k[s], lk = a.cu_k[s + 1] - k0;
    MM_DCHECK(q0 >= 0 && lq >= 0 && q0 + lq <= a.total_q && k0 >= 0 && lk >= 0 && k0 + lk <= a.total_k);
    MM_DCHECK(lk <= a.max_k);
    uint16_t* sk = reinterpret_cast<uint16_t*>(smem_fwd);
    uint16_t* sv = sk + a.max_k * HD;
    stage_rows<HD>(sk, a.k + int64_t(k0) * a.ldk + h * HD, a.ldk, lk);
    stage_rows<HD>(sv, a.v + int64_t(k0) * a.ldv + h * HD, a.ldv, lk);
    __syncthreads();
    const float sl2 = a.scale * kLog2e;
    for (int i = warp; i < lq; i += kWarps) {
        float q[HD];
        load_row<HD>(a.q + int64_t(q0 + i) * a.ldq + h * HD, q);
        const int nk = a.causal ? min(lk, i + 1) : lk;
        float m = -INFINITY, l = 0.f, acc = 0.f;
        for (int c = 0; c < nk; c += 32) {
            const int j = c + lane;
            float sc = -INFINITY;
            if (j < nk) {
                float k[HD];
                load_row<HD>(sk + j * HD, k);
                sc = dot<HD>(q, k) * sl2;
            }
            const float mn = fmaxf(m, wmax(sc));  // finite: key c is live
            const float corr = exp2f(m - mn);
            const float p = j < nk ? exp2f(sc - mn) : 0.f;
            l = l * corr + wsum(p);
            acc *= corr;
            const int cnt = min(32, nk - c);
            const uint16_t* vb = sv + c * HD + (lane < HD ? lane : 0);
            for (int u = 0; u < cnt; ++u) {
                const float pu = __shfl_sync(kFull, p, u);
                acc = fmaf(pu, bf(vb[u * HD]), acc);
            }
            m = mn;
        }
        if (lane < HD) a.o[int64_t(q0 + i) * a.ldo + h * HD + lane] = to_bf(nk ? acc / l : 0.f);
        if (lane == 0) a.lse[int64_t(h) * a.total_q + q0 + i] = nk ? (m + log2f(l)) * kLn2 : 0.f;
    }
}

// backward, one CTA per (sequence, head):
//   phase A (warp per query i): D_i = sum_j p_ij dp_ij (fp32, exact), then
//            dQ_i = scale * sum_j ds_ij k_j, ds_ij = p_ij (dp_ij - D_i);
//   phase B (warp per key j): dV_j = sum_i p_ij dO_i, dK_j = scale * sum_i ds_ij q_i,
//            with D_i and the log2-domain LSE from phase A in shared memory.
template <int HD>
__global__ void __launch_bounds__(kWarps * 32) attn_small_bwd_kernel(const mm_attn_args a) {
    __shared__ float d_s[256], lse_s[256];
    extern __shared__ uint4 smem_bwd[];  // K, V, Q, dO rows of this (sequence, head)
    pdl_wait_release();
    const int s = blockIdx.x, h = blockIdx.y;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int q0 = a.cu_q[s], lq = a.cu_q[s + 1] - q0;
    const int k0 = a.cu_k[s], lk = a.cu_k[s + 1] - k0;
    MM_DCHECK(lq <= 256 && lk <= 256 && q0 >= 0 && lq >= 0 && q0 + lq <= a.total_q && k0 >= 0 &&
              lk >= 0 && k0 + lk <= a.total_k && lq <= a.max_q && lk <= a.max_k);
    uint16_t* sk = reinterpret_cast<uint16_t*>(smem_bwd);
    uint16_t* sv = sk + a.max_k * HD;
    uint16_t* sq = sv + a.max_k * HD;
    uint16_t* sg = sq + a.max_q * HD;
    stage_rows<HD>(sk, a.k + int64_t(k0) * a.ldk + h * HD, a.ldk, lk);
    stage_rows<HD>(sv, a.v + int64_t(k0) * a.ldv + h * HD, a.ldv, lk);
    stage_rows<HD>(sq, a.q + int64_t(q0) * a.ldq + h * HD, a.ldq, lq);
    stage_rows<HD>(sg, a.d_o + int64_t(q0) * a.ldo + h * HD, a.ldo, lq);
    __syncthreads();
    const float sl2 = a.scale * kLog2e;
    const int hl = lane < HD ? lane : 0;
    for (int i = warp; i < lq; i += kWarps) {
        float q[HD], g[HD];
        load_row<HD>(sq + i * HD, q);
        load_row<HD>(sg + i * HD, g);
        const float lse2 = a.lse[int64_t(h) * a.total_q + q0 + i] * kLog2e;
        const int nk = a.causal ? min(lk, i + 1) : lk;
        float dsum = 0.f;
        for (int c = 0; c < nk; c += 32) {
            const int j = c + lane;
            if (j < nk) {
                float k[HD], v[HD];
                load_row<HD>(sk + j * HD, k);
                load_row<HD>(sv + j * HD, v);
                dsum += exp2f(dot<HD>(q, k) * sl2 - lse2) * dot<HD>(g, v);
            }
        }
        const float D = wsum(dsum);
        float dq = 0.f;
        for (int c = 0; c < nk; c += 32) {
            const int j = c + lane;
            float ds = 0.f;
            if (j < nk) {
                float k[HD], v[HD];
                load_row<HD>(sk + j * HD, k);
                load_row<HD>(sv + j * HD, v);
                const float p = exp2f(dot<HD>(q, k) * sl2 - lse2);
                ds = p * (dot<HD>(g, v) - D);
            }
            const int cnt = min(32, nk - c);
            const uint16_t* kb = sk + c * HD + hl;
            for (int u = 0; u < cnt; ++u) dq = fmaf(__shfl_sync(kFull, ds, u), bf(kb[u * HD]), dq);
        }
        if (lane < HD) a.dq[int64_t(q0 + i) * a.ld_dq + h * HD + lane] = to_bf(dq * a.scale);
        if (lane == 0) {
            d_s[i] = D;
            lse_s[i] = lse2;
        }
    }
    __syncthreads();
    for (int j = warp; j < lk; j += kWarps) {
        float k[HD], v[HD];
        load_row<HD>(sk + j * HD, k);
        load_row<HD>(sv + j * HD, v);
        const int i0 = a.causal ? j : 0;  // queries that see key j
        float dv = 0.f, dk = 0.f;
        for (int c = i0; c < lq; c += 32) {
            const int i = c + lane;
            float p = 0.f, ds = 0.f;
            if (i < lq) {
                float q[HD], g[HD];
                load_row<HD>(sq + i * HD, q);
                load_row<HD>(sg + i * HD, g);
                p = exp2f(dot<HD>(q, k) * sl2 - lse_s[i]);
                ds = p * (dot<HD>(g, v) - d_s[i]);
            }
            const int cnt = min(32, lq - c);
            const uint16_t* qb = sq + c * HD + hl;
            const uint16_t* gb = sg + c * HD + hl;
            for (int u = 0; u < cnt; ++u) {
                dv = fmaf(__shfl_sync(kFull, p, u), bf(gb[u * HD]), dv);
                dk = fmaf(__shfl_sync(kFull, ds, u), bf(qb[u * HD]), dk);
            }
        }
        if (lane < HD) {
            a.dv[int64_t(k0 + j) * a.ld_dv + h * HD + lane] = to_bf(dv);
            a.dk[int64_t(k0 + j) * a.ld_dk + h * HD + lane] = to_bf(dk * a.scale);
        }
    }
}

template <int HD>
int launch(const mm_attn_args* a, cudaStream_t s, bool bwd) {
    if (a->n_seq == 0) return 0;
    const dim3 grid(a->n_seq, a->heads), blk(kWarps * 32);
    const size_t row = HD * sizeof(uint16_t);
    if (bwd) {
        const size_t smem = (2 * size_t(a->max_k) + 2 * size_t(a->max_q)) * row;  // <= 64 KB
        MM_CUDA_TRY(cudaFuncSetAttribute(attn_small_bwd_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem)));
        MM_CUDA_TRY(mm::launch_pdl(attn_small_bwd_kernel<HD>, grid, blk, smem, s, *a));
        MM_LAUNCH_CHECK("attn_small_bwd_kernel");
    } else {
        const size_t smem = 2 * size_t(a->max_k) * row;
        MM_CUDA_TRY(mm::launch_pdl(attn_small_fwd_kernel<HD>, grid, blk, smem, s, *a));
        MM_LAUNCH_CHECK("attn_small_fwd_kernel");
    }
    return 0;
}

}  // namespace

// called by mm_attention_fwd / _bwd (attention.cu) after their argument check
int mm_attention_small(const mm_attn_args* a, void* stream, bool bwd) {
    MM_CHECK_ARG(a->n_seq >= 0 && a->n_seq <= 65535 * 1024, "bad sequence count %d", a->n_seq);
    const cudaStream_t s = mm::as_stream(stream);
    switch (a->head_dim) {
        case 16: return launch<16>(a, s, bwd);
        case 32: return launch<32>(a, s, bwd);
        default:
            mm::set_error("attention: head_dim %d unsupported (16, 32 or 64)", a->head_dim);
            return mm::kUnsupported;
    }
}
