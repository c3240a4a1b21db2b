// K5: packed varlen multi-head attention on tensor cores for short NMT
// sentences (lengths up to 256), head_dim 64, bf16 in / out, fp32 softmax.
//
// Warp-level bf16 MMA (mma.sync m16n8k16, fp32 accumulate) with ldmatrix
// fragment loads from padded shared memory (72-element pitch: conflict-free
// 16-byte rows).  Attention is ~1 % of the step's FLOPs at these lengths
// (SURVEY §2.3 K5): the kernels are sized for latency -- whole sequences
// resident in smem, thousands of small CTAs -- not for the tcgen05 pipe.
//
// Work unit: CTA = (group of consecutive sequences, head).  The host packs
// short sentences so one CTA's tile holds up to `cap` rows per side; every
// sequence sits at a 32-row-aligned, zero-padded offset, and warps take
// 16-row tiles of any sequence in the group round-robin.
// forward : per query tile, online softmax over 32-key blocks (exp2 domain),
//           O normalised once, natural-log LSE saved per (head, query).
// backward: phase A (query tiles): D_i = sum_j p_ij dp_ij in fp32 (exact --
//           not from the bf16-rounded O), then dQ = scale * dS K;
//           phase B (key tiles): dV = P^T dO, dK = scale * dS^T Q,
//           recomputing P / dP transposed.
// Probabilities and dS enter the second MMA as a bf16 hi + lo pair (two MMAs),
// so the products keep ~16 mantissa bits instead of bf16's 8.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "mm_common.h"
#include "tc_ptx.cuh"

namespace {

constexpr int kHd = 64;
constexpr int kP = 72;  // smem row pitch (bf16 elements)
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const uint16_t* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(smem_u32(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const uint16_t* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(smem_u32(p)));
}
__device__ __forceinline__ void mma(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                    uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// 2^x on the SFU, flush-to-zero (exp2f without fast-math adds subnormal
// handling around MUFU.EX2); -inf -> +0
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ uint32_t pack(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float quad_max(float v) {
    v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 1));
    return fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 2));
}
__device__ __forceinline__ float quad_sum(float v) {
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    return v + __shfl_xor_sync(0xffffffffu, v, 2);
}

// rows [0, n) of a 64-wide head slice -> smem (pitch kP), rows [n, npad) zeroed.
// cp.async (16 B, L2-only) so every copy of the CTA is in flight at once; the
// caller waits with cp_async_wait_all() + __syncthreads().
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(valid ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_all;" ::: "memory");
}
__device__ __forceinline__ void stage(uint16_t* dst, const uint16_t* src, int64_t ld, int n,
                                      int npad, int tid, int nthr) {
    for (int idx = tid; idx < npad * 8; idx += nthr) {
        const int r = idx >> 3, c = idx & 7;
        const bool valid = r < n;
        cp_async16(dst + r * kP + c * 8, valid ? src + r * ld + c * 8 : src, valid);
    }
}

// A fragments (16 rows x 64 cols, 4 k-steps) of a row-major smem tile
__device__ __forceinline__ void load_a(uint32_t (&f)[4][4], const uint16_t* base, int lane) {
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
        ldsm_x4(f[kk], base + (lane & 15) * kP + kk * 16 + (lane >> 4) * 8);
}

// acc[nt] (+)= A(16x64) * B^T where B rows n0..n0+31 (row-major [n][k], k = 64)
__device__ __forceinline__ void mma_abt(float (&acc)[4][4], const uint32_t (&a)[4][4],
                                        const uint16_t* b, int n0, int lane) {
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
#pragma unroll
        for (int kk2 = 0; kk2 < 2; ++kk2) {
            uint32_t r[4];
            ldsm_x4(r, b + (n0 + nt * 8 + (lane & 7)) * kP + kk2 * 32 + (lane >> 3) * 8);
            mma(acc[nt], a[2 * kk2], r[0], r[1]);
            mma(acc[nt], a[2 * kk2 + 1], r[2], r[3]);
        }
    }
}

// out[8][4] (+)= P(16 x 32, fp32 accumulators -> bf16 A fragments) * B where
// B rows k0..k0+31 are row-major [k][n] (n = 64): ldmatrix.trans fragments
__device__ __forceinline__ void mma_pb(float (&out)[8][4], const float (&p)[4][4],
                                       const uint16_t* b, int k0, int lane) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const float v[8] = {p[2 * j][0], p[2 * j][1], p[2 * j][2], p[2 * j][3],
                            p[2 * j + 1][0], p[2 * j + 1][1], p[2 * j + 1][2], p[2 * j + 1][3]};
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            hi[i] = pack(v[2 * i], v[2 * i + 1]);
            const float h0 = __uint_as_float(hi[i] << 16), h1 = __uint_as_float(hi[i] & 0xffff0000u);
            lo[i] = pack(v[2 * i] - h0, v[2 * i + 1] - h1);
        }
#pragma unroll
        for (int np = 0; np < 4; ++np) {
            uint32_t r[4];
            ldsm_x4_t(r, b + (k0 + j * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * kP + np * 16 +
                             (lane >> 4) * 8);
            mma(out[2 * np], hi, r[0], r[1]);
            mma(out[2 * np + 1], hi, r[2], r[3]);
            mma(out[2 * np], lo, r[0], r[1]);
            mma(out[2 * np + 1], lo, r[2], r[3]);
        }
    }
}

__device__ __forceinline__ void zero(float (&x)[4][4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i][0] = x[i][1] = x[i][2] = x[i][3] = 0.f;
}

// ---------------------------------------------------------------------------
constexpr int kMaxSeqPerGroup = 16;

struct Group {
    int n;                       // sequences in the group
    int q0[kMaxSeqPerGroup], lq[kMaxSeqPerGroup], qoff[kMaxSeqPerGroup];
    int k0[kMaxSeqPerGroup], lk[kMaxSeqPerGroup], koff[kMaxSeqPerGroup];
};

// called by warp 0: lane i loads sequence i of the group, offsets by warp scan
__device__ __forceinline__ void load_group(Group& G, const mm_attn_args& a, int lane) {
    const int first = a.groups[2 * blockIdx.y], n = a.groups[2 * blockIdx.y + 1];
    int q0 = 0, lq = 0, k0 = 0, lk = 0;
    if (lane < n) {
        q0 = a.cu_q[first + lane];
        lq = a.cu_q[first + lane + 1] - q0;
        k0 = a.cu_k[first + lane];
        lk = a.cu_k[first + lane + 1] - k0;
    }
    int pq = (lq + 31) & ~31, pk = (lk + 31) & ~31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {  // inclusive scan
        const int xq = __shfl_up_sync(0xffffffffu, pq, o), xk = __shfl_up_sync(0xffffffffu, pk, o);
        if (lane >= o) { pq += xq; pk += xk; }
    }
    if (lane < n) {
        G.q0[lane] = q0; G.lq[lane] = lq; G.k0[lane] = k0; G.lk[lane] = lk;
        G.qoff[lane] = pq - ((lq + 31) & ~31);
        G.koff[lane] = pk - ((lk + 31) & ~31);
    }
    if (lane == 0) G.n = n;
}

// tile -> (sequence, 16-row tile start); tiles enumerate the group's
// sequences in order (lens = G.lq for query tiles, G.lk for key tiles)
__device__ __forceinline__ bool tile_of(const Group& G, const int* lens, int tile, int& s,
                                        int& r0) {
    for (s = 0; s < G.n; ++s) {
        const int nt = (lens[s] + 15) >> 4;
        if (tile < nt) {
            r0 = tile * 16;
            return true;
        }
        tile -= nt;
    }
    return false;
}

__device__ __forceinline__ int n_tiles(const Group& G, const int* lens) {
    int t = 0;
    for (int s = 0; s < G.n; ++s) t += (lens[s] + 15) >> 4;
    return t;
}

__device__ void stage_group(uint16_t* Qs, uint16_t* Ks, uint16_t* Vs, uint16_t* dOs,
                            const Group& G, const mm_attn_args& a, int h, int nthr) {
    for (int i = 0; i < G.n; ++i) {
        const int pq = (G.lq[i] + 31) & ~31, pk = (G.lk[i] + 31) & ~31;
        if (Qs) stage(Qs + G.qoff[i] * kP, a.q + int64_t(G.q0[i]) * a.ldq + h * kHd, a.ldq, G.lq[i], pq, threadIdx.x, nthr);
        if (dOs) stage(dOs + G.qoff[i] * kP, a.d_o + int64_t(G.q0[i]) * a.ldo + h * kHd, a.ldo, G.lq[i], pq, threadIdx.x, nthr);
        stage(Ks + G.koff[i] * kP, a.k + int64_t(G.k0[i]) * a.ldk + h * kHd, a.ldk, G.lk[i], pk, threadIdx.x, nthr);
        stage(Vs + G.koff[i] * kP, a.v + int64_t(G.k0[i]) * a.ldv + h * kHd, a.ldv, G.lk[i], pk, threadIdx.x, nthr);
    }
}

constexpr int kFwdWarps = 4;

__global__ void __launch_bounds__(kFwdWarps * 32) attn_fwd_kernel(const mm_attn_args a) {
    extern __shared__ __align__(16) uint16_t sm[];
    __shared__ Group G;
    const int h = blockIdx.x;  // heads fastest: a group's CTAs run together and share its rows' DRAM pages
    // the group table and sequence offsets come from the step's host upload,
    // not from the previous kernel: read them before griddepcontrol.wait
    if (threadIdx.x < 32) load_group(G, a, threadIdx.x);
    if (a.flags & 1) {  // groups of <= 128 rows per side went to the tcgen05 kernel
        const int first = a.groups[2 * blockIdx.y], n = a.groups[2 * blockIdx.y + 1];
        if (a.cu_q[first + n] - a.cu_q[first] <= 128 && a.cu_k[first + n] - a.cu_k[first] <= 128) return;
    }
    pdl_wait_release();
    __syncthreads();
    uint16_t* Qs = sm;
    uint16_t* Ks = Qs + a.cap * kP;
    uint16_t* Vs = Ks + a.cap * kP;
    stage_group(Qs, Ks, Vs, nullptr, G, a, h, kFwdWarps * 32);
    cp_async_wait_all();
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const float c = a.scale * kLog2e;
    const int ntiles = n_tiles(G, G.lq);
    for (int tile = warp; tile < ntiles; tile += kFwdWarps) {
        int sidx, r0;
        tile_of(G, G.lq, tile, sidx, r0);
        const int lq = G.lq[sidx], lk = G.lk[sidx], q0 = G.q0[sidx];
        const uint16_t* Kseq = Ks + G.koff[sidx] * kP;
        const uint16_t* Vseq = Vs + G.koff[sidx] * kP;
        uint32_t qf[4][4];
        load_a(qf, Qs + (G.qoff[sidx] + r0) * kP, lane);
        const int row0 = r0 + g, row1 = row0 + 8;
        const int kend = a.causal ? min(lk, r0 + 16) : lk;
        float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
        float o[8][4];
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
        for (int kb = 0; kb < kend; kb += 32) {
            float s[4][4];
            zero(s);
            mma_abt(s, qf, Kseq, kb, lane);
            float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
            for (int nt = 0; nt < 4; ++nt)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int key = kb + nt * 8 + 2 * t + (e & 1);
                    const int row = e < 2 ? row0 : row1;
                    float v = s[nt][e] * c;
                    if (key >= lk || (a.causal && key > row)) v = -INFINITY;
                    s[nt][e] = v;
                    mx[e >> 1] = fmaxf(mx[e >> 1], v);
                }
            float corr[2], mref[2];
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const float mn = fmaxf(m[i], quad_max(mx[i]));
                mref[i] = mn == -INFINITY ? 0.f : mn;
                corr[i] = ex2(m[i] - mref[i]);  // m = -inf -> 0
                m[i] = mn;
            }
            float sum[2] = {0.f, 0.f};
#pragma unroll
            for (int nt = 0; nt < 4; ++nt)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float p = ex2(s[nt][e] - mref[e >> 1]);
                    s[nt][e] = p;
                    sum[e >> 1] += p;
                }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                o[i][0] *= corr[0]; o[i][1] *= corr[0];
                o[i][2] *= corr[1]; o[i][3] *= corr[1];
            }
            l[0] = l[0] * corr[0] + sum[0];
            l[1] = l[1] * corr[1] + sum[1];
            mma_pb(o, s, Vseq, kb, lane);
        }
        l[0] = quad_sum(l[0]);
        l[1] = quad_sum(l[1]);
        const float inv0 = 1.f / l[0], inv1 = 1.f / l[1];
        uint16_t* out0 = a.o + int64_t(q0 + row0) * a.ldo + h * kHd;
        uint16_t* out1 = a.o + int64_t(q0 + row1) * a.ldo + h * kHd;
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
            if (row0 < lq)
                *reinterpret_cast<uint32_t*>(out0 + nt * 8 + 2 * t) = pack(o[nt][0] * inv0, o[nt][1] * inv0);
            if (row1 < lq)
                *reinterpret_cast<uint32_t*>(out1 + nt * 8 + 2 * t) = pack(o[nt][2] * inv1, o[nt][3] * inv1);
        }
        if (t == 0) {
            if (row0 < lq) a.lse[int64_t(h) * a.total_q + q0 + row0] = (m[0] + log2f(l[0])) * kLn2;
            if (row1 < lq) a.lse[int64_t(h) * a.total_q + q0 + row1] = (m[1] + log2f(l[1])) * kLn2;
        }
    }
}

// ---------------------------------------------------------------------------
constexpr int kBwdWarps = 8;

#ifdef MM_ATTN_TRACE  // diagnostics build: per-CTA phase stamps of the last backward launch
__device__ unsigned long long g_attn_trace[8192 * 4];
#define ATTN_STAMP(i)                                                                         \
    do {                                                                                      \
        if (threadIdx.x == 0) {                                                               \
            unsigned long long t_;                                                            \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                            \
            const int cta_ = blockIdx.y * gridDim.x + blockIdx.x;                             \
            if (cta_ < 8192) g_attn_trace[cta_ * 4 + (i)] = t_;                               \
        }                                                                                     \
    } while (0)
#define ATTN_STAMP_LANE0(i)                                                                   \
    do {                                                                                      \
        if ((threadIdx.x & 31) == 0) {                                                        \
            unsigned long long t_;                                                            \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                            \
            const int cta_ = blockIdx.y * gridDim.x + blockIdx.x;                             \
            if (cta_ < 8192) g_attn_trace[cta_ * 4 + (i)] = t_;                               \
        }                                                                                     \
    } while (0)
#else
#define ATTN_STAMP_LANE0(i) \
    do {                    \
    } while (0)
#define ATTN_STAMP(i) \
    do {              \
    } while (0)
#endif

__global__ void __launch_bounds__(kBwdWarps * 32, 2) attn_bwd_kernel(const mm_attn_args a) {
    extern __shared__ __align__(16) uint16_t sm[];
    __shared__ Group G;
    const int h = blockIdx.x;  // heads fastest: a group's CTAs run together and share its rows' DRAM pages
    if (threadIdx.x < 32) load_group(G, a, threadIdx.x);  // host-uploaded: before the wait
    if (a.flags & 1) {  // groups of <= 128 rows per side went to the tcgen05 kernel
        const int first = a.groups[2 * blockIdx.y], n = a.groups[2 * blockIdx.y + 1];
        if (a.cu_q[first + n] - a.cu_q[first] <= 128 && a.cu_k[first + n] - a.cu_k[first] <= 128) return;
    }
    pdl_wait_release();
    ATTN_STAMP(0);
    __syncthreads();
    uint16_t* Qs = sm;
    uint16_t* dOs = Qs + a.cap * kP;
    uint16_t* Ks = dOs + a.cap * kP;
    uint16_t* Vs = Ks + a.cap * kP;
    float* lse2 = reinterpret_cast<float*>(Vs + a.cap * kP);  // lse * log2(e), per smem row
    float* Dd = lse2 + a.cap;
    const int nthr = kBwdWarps * 32;
    stage_group(Qs, Ks, Vs, dOs, G, a, h, nthr);
    for (int i = 0; i < G.n; ++i) {
        const int pq = (G.lq[i] + 31) & ~31;
        for (int r = threadIdx.x; r < pq; r += nthr) {
            // lse rides the same cp.async batch (4-byte copies); padding rows 0
            if (r < G.lq[i]) cp_async4(lse2 + G.qoff[i] + r, a.lse + int64_t(h) * a.total_q + G.q0[i] + r);
            else lse2[G.qoff[i] + r] = 0.f;
            // phase A writes D only for rows of its 16-row tiles; phase B reads
            // it for every row of a 32-row block (as 0 * (dP - D) past lq), so
            // the padding rows must hold a finite value, not stale smem
            Dd[G.qoff[i] + r] = 0.f;
        }
    }
    cp_async_wait_all();
    __syncthreads();
    for (int r = threadIdx.x; r < a.cap; r += nthr) lse2[r] *= kLog2e;  // natural log -> log2 domain
    __syncthreads();
    ATTN_STAMP(1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const float c = a.scale * kLog2e;

    // ---------------- phase A: D and dQ (warps over 16-query tiles)
    const int nqt = n_tiles(G, G.lq);
    for (int tile = warp; tile < nqt; tile += kBwdWarps) {
        int sidx, qt;
        tile_of(G, G.lq, tile, sidx, qt);
        const int lq = G.lq[sidx], lk = G.lk[sidx], q0 = G.q0[sidx], qo = G.qoff[sidx];
        const uint16_t* Kseq = Ks + G.koff[sidx] * kP;
        const uint16_t* Vseq = Vs + G.koff[sidx] * kP;
        uint32_t qf[4][4], df[4][4];
        load_a(qf, Qs + (qo + qt) * kP, lane);
        load_a(df, dOs + (qo + qt) * kP, lane);
        const int row0 = qt + g, row1 = row0 + 8;
        const float l20 = lse2[qo + row0], l21 = lse2[qo + row1];
        const int kend = a.causal ? min(lk, qt + 16) : lk;
        float dpart[2] = {0.f, 0.f};
        for (int pass = 0; pass < 2; ++pass) {
            float dq[8][4];
#pragma unroll
            for (int i = 0; i < 8; ++i) dq[i][0] = dq[i][1] = dq[i][2] = dq[i][3] = 0.f;
            const float D0 = dpart[0], D1 = dpart[1];
            for (int kb = 0; kb < kend; kb += 32) {
                float s[4][4], dp[4][4];
                zero(s);
                zero(dp);
                mma_abt(s, qf, Kseq, kb, lane);
                mma_abt(dp, df, Vseq, kb, lane);
                // a block fully inside the sequence (and below the causal
                // diagonal of both rows) needs no per-element masks
                const bool full = kb + 32 <= lk && row1 < lq && (!a.causal || kb + 31 <= row0);
#pragma unroll
                for (int nt = 0; nt < 4; ++nt)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        float p = ex2(s[nt][e] * c - (e < 2 ? l20 : l21));
                        if (!full) {
                            const int key = kb + nt * 8 + 2 * t + (e & 1);
                            const int row = e < 2 ? row0 : row1;
                            if (key >= lk || (a.causal && key > row) || row >= lq) p = 0.f;
                        }
                        if (pass == 0) dpart[e >> 1] = fmaf(p, dp[nt][e], dpart[e >> 1]);
                        else s[nt][e] = p * (dp[nt][e] - (e < 2 ? D0 : D1));  // dS
                    }
                if (pass == 1) mma_pb(dq, s, Kseq, kb, lane);
            }
            if (pass == 0) {
                dpart[0] = quad_sum(dpart[0]);
                dpart[1] = quad_sum(dpart[1]);
                if (t == 0) {
                    Dd[qo + row0] = dpart[0];
                    Dd[qo + row1] = dpart[1];
                }
            } else {
                uint16_t* o0 = a.dq + int64_t(q0 + row0) * a.ld_dq + h * kHd;
                uint16_t* o1 = a.dq + int64_t(q0 + row1) * a.ld_dq + h * kHd;
#pragma unroll
                for (int nt = 0; nt < 8; ++nt) {
                    if (row0 < lq)
                        *reinterpret_cast<uint32_t*>(o0 + nt * 8 + 2 * t) =
                            pack(dq[nt][0] * a.scale, dq[nt][1] * a.scale);
                    if (row1 < lq)
                        *reinterpret_cast<uint32_t*>(o1 + nt * 8 + 2 * t) =
                            pack(dq[nt][2] * a.scale, dq[nt][3] * a.scale);
                }
            }
        }
    }
    __syncthreads();
    ATTN_STAMP(2);

    // ---------------- phase B: dK, dV (warps over 16-key tiles)
    const int nkt = n_tiles(G, G.lk);
    for (int tile = warp; tile < nkt; tile += kBwdWarps) {
        int sidx, kt;
        tile_of(G, G.lk, tile, sidx, kt);
        const int lq = G.lq[sidx], lk = G.lk[sidx], k0 = G.k0[sidx], qo = G.qoff[sidx];
        const uint16_t* Qseq = Qs + qo * kP;
        const uint16_t* dOseq = dOs + qo * kP;
        uint32_t kf[4][4];
        load_a(kf, Ks + (G.koff[sidx] + kt) * kP, lane);
        const int key0 = kt + g, key1 = key0 + 8;
        const int qbeg = a.causal ? (kt & ~31) : 0;
        // two passes keep the live set under 128 registers: pass 0 dV = P^T dO,
        // pass 1 dK = dS^T Q (S^T recomputed; the MMAs are cheap here)
        for (int pass = 0; pass < 2; ++pass) {
            float acc[8][4];
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
            uint32_t vf[4][4];
            if (pass == 1) load_a(vf, Vs + (G.koff[sidx] + kt) * kP, lane);
            for (int qb = qbeg; qb < lq; qb += 32) {
                float st[4][4], dpt[4][4];
                zero(st);
                mma_abt(st, kf, Qseq, qb, lane);    // S^T = K Q^T
                if (pass == 1) {
                    zero(dpt);
                    mma_abt(dpt, vf, dOseq, qb, lane);  // dP^T = V dO^T
                }
#pragma unroll
                for (int nt = 0; nt < 4; ++nt)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int q = qb + nt * 8 + 2 * t + (e & 1);
                        const int key = e < 2 ? key0 : key1;
                        float p = 0.f;
                        if (q < lq && key < lk && !(a.causal && key > q))
                            p = ex2(st[nt][e] * c - lse2[qo + q]);
                        if (pass == 0) st[nt][e] = p;
                        else dpt[nt][e] = p * (dpt[nt][e] - Dd[qo + q]);
                    }
                if (pass == 0) mma_pb(acc, st, dOseq, qb, lane);   // dV += P^T dO
                else mma_pb(acc, dpt, Qseq, qb, lane);              // dK += dS^T Q
            }
            const float sc = pass == 0 ? 1.f : a.scale;
            uint16_t* base = pass == 0 ? a.dv : a.dk;
            const int64_t ld = pass == 0 ? a.ld_dv : a.ld_dk;
            uint16_t* o0 = base + int64_t(k0 + key0) * ld + h * kHd;
            uint16_t* o1 = base + int64_t(k0 + key1) * ld + h * kHd;
#pragma unroll
            for (int nt = 0; nt < 8; ++nt) {
                if (key0 < lk)
                    *reinterpret_cast<uint32_t*>(o0 + nt * 8 + 2 * t) = pack(acc[nt][0] * sc, acc[nt][1] * sc);
                if (key1 < lk)
                    *reinterpret_cast<uint32_t*>(o1 + nt * 8 + 2 * t) = pack(acc[nt][2] * sc, acc[nt][3] * sc);
            }
        }
    }
    __syncthreads();
    ATTN_STAMP(3);
}

// ===========================================================================
// Backward on tcgen05 (groups whose sequences fit one 128-row block per side)
//
// One CTA per (head, group): TMA stages the group's Q, K, V, dO rows (one
// 128-row x 64-column SW128 box each -- rows past the group are other
// tokens, masked by sequence id); the MMA warp computes S = Q K^T and
// dP = dO V^T into TMEM (128 columns each); eight warps turn them into P, the
// exact fp32 D_i = sum_j P_ij dP_ij and dS = P (dP - D), written to shared
// memory as bf16 hi + lo pairs in the SW128 K-major layout -- the same bytes
// serve as the K-major A of dQ = dS K and as the MN-major A of dV = P^T dO and
// dK = dS^T Q -- then the MMA warp issues the three products (hi and lo) into
// TMEM and the eight warps scale, convert and store dQ / dK / dV.  Sequence
// masks come from the group's offsets (no padding rows).
namespace tca {

constexpr int kRows = 128;
constexpr int kTile = kRows * 128;         // 128 rows x 64 bf16 (one SW128 box)
constexpr int kPTile = 2 * kTile;          // 128 rows x 128 keys (two 64-key regions)
constexpr int kEpiW0 = 2, kEpiW = 16;  // 4 warps per TMEM lane quarter, 32 keys each
constexpr int kThreads = (kEpiW0 + kEpiW) * 32;
constexpr int kSmemBytes = 4 * kTile + 4 * kPTile + 4096 + 1024;  // + meta + alignment

struct alignas(64) BwdParams {
    CUtensorMap mq, mk, mv, mdo;
    const int32_t* cu_q;
    const int32_t* cu_k;
    const int32_t* groups;
    const float* lse;
    uint16_t* dq;
    uint16_t* dk;
    uint16_t* dv;
    int64_t ld_dq, ld_dk, ld_dv;
    int total_q, causal;
    float scale;
    int n_groups, heads;
    int early_qkv;  // Q / K / V may be loaded before griddepcontrol.wait (mm_attn_args.flags & 2)
    int long_skip;  // long kernel: long groups before this one belong to an earlier launch
};

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}

// 32 values of a row (4 16-byte chunks from chunk c0) as bf16 hi (+ lo
// residual) into a SW128 K-major region: row r at r*128, 16-byte chunk c at
// (c ^ (r & 7)) * 16
__device__ __forceinline__ void store_row_hilo(uint8_t* hi, uint8_t* lo, int r, int c0, const float* v) {
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
        uint32_t h[4], l[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float a = v[cc * 8 + 2 * e], b = v[cc * 8 + 2 * e + 1];
            h[e] = pack_bf16(a, b);
            const float ah = __uint_as_float(h[e] << 16), bh = __uint_as_float(h[e] & 0xffff0000u);
            l[e] = pack_bf16(a - ah, b - bh);
        }
        const int off = r * 128 + (((c0 + cc) ^ (r & 7)) * 16);
        *reinterpret_cast<uint4*>(hi + off) = make_uint4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<uint4*>(lo + off) = make_uint4(l[0], l[1], l[2], l[3]);
    }
}

// bf16 hi only: dS for the dK / dQ products (as FlashAttention stores it)
__device__ __forceinline__ void store_row_hi(uint8_t* hi, int r, int c0, const float* v) {
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
        uint32_t h[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) h[e] = pack_bf16(v[cc * 8 + 2 * e], v[cc * 8 + 2 * e + 1]);
        const int off = r * 128 + (((c0 + cc) ^ (r & 7)) * 16);
        *reinterpret_cast<uint4*>(hi + off) = make_uint4(h[0], h[1], h[2], h[3]);
    }
}

// dS = P (dP - D) enters dK = dS^T Q and dQ = dS K as bf16 (FlashAttention's
// choice): its rounding (2^-9 relative) matches that of the bf16 dq / dk / dv
// outputs themselves; -DMM_ATTN_DS_LO=1 restores the hi + lo pair (two more
// MMA chains and a quarter of the smem stores: 16 vs 13.5 us per config-3
// launch).  P keeps hi + lo: dropping it moved the cross / causal blocks
// past 2e-3.
#ifndef MM_ATTN_DS_LO
#define MM_ATTN_DS_LO 0
#endif
constexpr bool kDsLo = MM_ATTN_DS_LO != 0;
// forward O = P V with P as bf16 hi + lo (default); -DMM_ATTN_FWD_P_LO=0
// stores P as bf16 only: 8.4 -> 7.5 us per launch, but three oracle / block
// tests then exceed their bounds and the step time does not move
#ifndef MM_ATTN_FWD_P_LO
#define MM_ATTN_FWD_P_LO 1
#endif
constexpr bool kFwdPLo = MM_ATTN_FWD_P_LO != 0;

__device__ __forceinline__ uint64_t desc(const void* p, uint32_t lbo) {
    return tc::umma_desc_sw128(tc::smem_u32(p), lbo, 1024);
}

// -DMM_ATTN_WAITPROF (diagnostics build, tools/attn_waitprof.py): per-CTA
// clock64 totals of the MMA warp's waits for tiles / P and the epilogue's
// waits for S / the gradient MMAs
#ifdef MM_ATTN_WAITPROF
__device__ unsigned long long g_wp[148 * 8];
#define WP_BEGIN(t) const long long t = clock64()
#define WP_ADD(i, t)                                                                        \
    do {                                                                                    \
        if ((threadIdx.x & 31) == 0 && blockIdx.x < 148)                                    \
            atomicAdd(&g_wp[blockIdx.x * 8 + (i)], (unsigned long long)(clock64() - (t)));  \
    } while (0)
#else
#define WP_BEGIN(t) do { } while (0)
#define WP_ADD(i, t) do { } while (0)
#endif
// Persistent: CTA b takes units (group, head) b, b + grid, ... (heads fastest);
// the producer loads unit n+1's tiles as soon as unit n's MMAs have consumed
// them (g_bar), so the TMA latency hides behind unit n's output phase; TMEM
// is double-buffered by unit parity (unit n+1's S / dP cannot overwrite the
// dV / dK / dQ of unit n that the warps are still reading).
__global__ void __launch_bounds__(kThreads, 1) attn_bwd_tc_kernel(const __grid_constant__ BwdParams p) {
    extern __shared__ uint8_t smraw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    uint8_t* Qs = sm;
    uint8_t* Ks = Qs + kTile;
    uint8_t* Vs = Ks + kTile;
    uint8_t* dOs = Vs + kTile;
    uint8_t* Ph = dOs + kTile;   // regions: keys 0-63 at +0, keys 64-127 at +kTile
    uint8_t* Pl = Ph + kPTile;
    uint8_t* Sh = Pl + kPTile;   // dS hi
    uint8_t* Sl = Sh + kPTile;   // dS lo
    float* dpart = reinterpret_cast<float*>(Sl + kPTile);  // [4][128] D partials
    uint64_t* bars = reinterpret_cast<uint64_t*>(dpart + 4 * kRows);
    uint64_t* tma_bar = bars;
    uint64_t* s_bar = bars + 1;
    uint64_t* p_bar = bars + 2;
    uint64_t* g_bar = bars + 3;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4);

    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
    const int lane = threadIdx.x & 31;
    const int units = p.n_groups * p.heads;
    if (warp == 1 && lane == 0) {
        tc::mbar_init(tma_bar, 1);
        tc::mbar_init(s_bar, 1);
        tc::mbar_init(p_bar, kEpiW);
        tc::mbar_init(g_bar, 1);
        tc::fence_barrier_init();
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem0 = *tmem_slot;
    ATTN_STAMP(0);
    // unit -> group metadata (host-uploaded: may be read before griddepcontrol.wait)
    struct U { int first, nseq, q_lo, nq, k_lo, nk, h; };
    auto unit = [&](int u) -> U {
        U x;
        const int grp = u / p.heads;
        x.h = u - grp * p.heads;
        x.first = p.groups[2 * grp];
        x.nseq = p.groups[2 * grp + 1];
        x.q_lo = p.cu_q[x.first];
        x.nq = p.cu_q[x.first + x.nseq] - x.q_lo;
        x.k_lo = p.cu_k[x.first];
        x.nk = p.cu_k[x.first + x.nseq] - x.k_lo;
        MM_DCHECK(x.nseq >= 1 && x.q_lo >= 0 && x.nq >= 0 && x.q_lo + x.nq <= p.total_q && x.k_lo >= 0 && x.nk >= 0);
        return x;
    };
    auto mine = [&](const U& x) { return x.nq <= kRows && x.nk <= kRows; };  // else: mma.sync kernel

    if (warp == 0) {
        if (lane == 0) {
            // the forward pass's Q / K / V can be in flight before the previous
            // kernel (which produced dO) has finished
            bool waited = !p.early_qkv;
            if (waited) pdl_wait();
            int n = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x) {
                const U x = unit(u);
                if (!mine(x)) continue;
                if (n > 0) tc::mbar_wait(g_bar, (n - 1) & 1);  // unit n-1's MMAs consumed the tiles
                tc::mbar_expect_tx(tma_bar, 4 * kTile);
                tc::tma_load_2d(Qs, &p.mq, tma_bar, x.h * 64, x.q_lo);
                tc::tma_load_2d(Ks, &p.mk, tma_bar, x.h * 64, x.k_lo);
                tc::tma_load_2d(Vs, &p.mv, tma_bar, x.h * 64, x.k_lo);
                if (!waited) {
                    pdl_wait();
                    waited = true;
                }
                tc::tma_load_2d(dOs, &p.mdo, tma_bar, x.h * 64, x.q_lo);
                ++n;
            }
            if (!waited) pdl_wait();
        }
    } else if (warp == 1) {
        int n = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x) {
            const U x = unit(u);
            if (!mine(x)) continue;
            const uint32_t tmem = tmem0 + (n & 1) * 256;
            // ---- S = Q K^T (cols 0-127), dP = dO V^T (cols 128-255)
            WP_BEGIN(w0_);
            tc::mbar_wait(tma_bar, n & 1);
            WP_ADD(0, w0_);
            tc::tc_fence_after();
            constexpr uint32_t id_s = tc::idesc_bf16_f32(128, 128, 0, 0);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                tc::mma_bf16_elect<1>(tmem, desc(Qs + kk * 32, 16), desc(Ks + kk * 32, 16), id_s, kk > 0);
                tc::mma_bf16_elect<1>(tmem + 128, desc(dOs + kk * 32, 16), desc(Vs + kk * 32, 16), id_s, kk > 0);
            }
            tc::mma_commit_elect<1>(s_bar);
            // ---- dV = P^T dO (cols 0-63), dK = dS^T Q (64-127), dQ = dS K (128-191)
            WP_BEGIN(w1_);
            tc::mbar_wait(p_bar, n & 1);
            WP_ADD(1, w1_);
            tc::tc_fence_after();
            constexpr uint32_t id_mn = tc::idesc_bf16_f32(128, 64, 1, 1);  // A and B MN-major
            constexpr uint32_t id_km = tc::idesc_bf16_f32(128, 64, 0, 1);  // A K-major, B MN-major
#pragma unroll
            for (int part = 0; part < 2; ++part) {  // bf16 hi, then lo
                const uint8_t* P = part ? Pl : Ph;
                const uint8_t* S = part ? Sl : Sh;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {  // K = 128 query rows
                    const uint32_t acc = (part > 0 || kk > 0) ? 1u : 0u;
                    tc::mma_bf16_elect<1>(tmem + 0, desc(P + kk * 2048, kTile), desc(dOs + kk * 2048, kTile), id_mn, acc);
                    if (kDsLo || part == 0)
                        tc::mma_bf16_elect<1>(tmem + 64, desc(S + kk * 2048, kTile), desc(Qs + kk * 2048, kTile), id_mn, acc);
                }
                if (kDsLo || part == 0) {
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {  // K = 128 keys
                        const uint32_t acc = (part > 0 || kk > 0) ? 1u : 0u;
                        tc::mma_bf16_elect<1>(tmem + 128, desc(S + (kk >> 2) * kTile + (kk & 3) * 32, 16),
                                              desc(Ks + kk * 2048, kTile), id_km, acc);
                    }
                }
            }
            tc::mma_commit_elect<1>(g_bar);
            ++n;
        }
    } else {
        // ---- sixteen warps: warp%4 = TMEM lane quarter (query rows), kc = 32-key chunk
        const int quarter = warp & 3, kc = (warp - kEpiW0) >> 2;
        const int i = quarter * 32 + lane;  // query row within the group
        const float c = p.scale * kLog2e;
        pdl_wait();
        // this row's metadata of a unit -- group -> sequence offsets -> the
        // row's key range and lse, a chain of dependent global loads -- is
        // fetched for the next unit while the current unit's gradient MMAs
        // run, off the per-unit critical path
        struct RowMeta {
            U x;
            int u, klo, khi;
            float lse;
        };
        auto fetch = [&](int u, RowMeta& m) {  // m.u = units: no unit left
            for (; u < units; u += gridDim.x) {
                m.x = unit(u);
                if (mine(m.x)) break;
            }
            m.u = u;
            m.klo = m.khi = 0;
            m.lse = 0.f;
            if (u >= units || i >= m.x.nq) return;
            // the row's keys: one contiguous range of the group's key rows (its
            // own sequence; causal: up to its position)
            for (int s2 = 0; s2 < m.x.nseq; ++s2) {
                const int a = p.cu_q[m.x.first + s2] - m.x.q_lo, b = p.cu_q[m.x.first + s2 + 1] - m.x.q_lo;
                if (i >= a && i < b) {
                    m.klo = p.cu_k[m.x.first + s2] - m.x.k_lo;
                    m.khi = p.causal ? m.klo + (i - a) + 1 : p.cu_k[m.x.first + s2 + 1] - m.x.k_lo;
                }
            }
            m.lse = p.lse[int64_t(m.x.h) * p.total_q + m.x.q_lo + i];
        };
        RowMeta cur;
        fetch(blockIdx.x, cur);
        int n = 0;
        while (cur.u < units) {
            const U x = cur.x;
            const uint32_t trow = tmem0 + (n & 1) * 256 + (static_cast<uint32_t>(quarter * 32) << 16);
            const bool vrow = i < x.nq;
            const int klo = cur.klo, khi = cur.khi;
            const float l2 = cur.lse * kLog2e;
            WP_BEGIN(w2_);
            tc::mbar_wait(s_bar, n & 1);
            if (warp == kEpiW0) WP_ADD(2, w2_);
            tc::tc_fence_after();
            if (warp == kEpiW0) ATTN_STAMP_LANE0(1);
            const int key0 = kc * 32;
            float pv[32], dpv[32];
            // a chunk no row of this warp attends to is all zeros (warp-uniform skip)
            const bool any = __any_sync(0xffffffffu, klo < key0 + 32 && khi > key0);
            if (any) {
                uint32_t sv[32], dv[32];
                tc::tmem_ld_32x32(trow + key0, sv);
                tc::tmem_ld_32x32(trow + 128 + key0, dv);
                tc::tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const int key = key0 + j;
                    pv[j] = (key >= klo && key < khi) ? ex2(fmaf(__uint_as_float(sv[j]), c, -l2)) : 0.f;
                    dpv[j] = __uint_as_float(dv[j]);
                }
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) pv[j] = dpv[j] = 0.f;
            }
            float dsum = 0.f;
#pragma unroll
            for (int j = 0; j < 32; ++j) dsum = fmaf(pv[j], dpv[j], dsum);
            dpart[kc * kRows + i] = dsum;
            tc::named_barrier_sync(1, kEpiW * 32);
            const float D = (dpart[i] + dpart[kRows + i]) + (dpart[2 * kRows + i] + dpart[3 * kRows + i]);
#pragma unroll
            for (int j = 0; j < 32; ++j) dpv[j] = pv[j] * (dpv[j] - D);  // dS
            // keys kc*32..+32: region kc/2, 16-byte chunks (kc&1)*4 .. +4 of the row
            store_row_hilo(Ph + (kc >> 1) * kTile, Pl + (kc >> 1) * kTile, i, (kc & 1) * 4, pv);
            if (kDsLo) store_row_hilo(Sh + (kc >> 1) * kTile, Sl + (kc >> 1) * kTile, i, (kc & 1) * 4, dpv);
            else store_row_hi(Sh + (kc >> 1) * kTile, i, (kc & 1) * 4, dpv);
            tc::fence_proxy_async_smem();  // generic stores -> visible to the tensor core
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(p_bar);
            if (warp == kEpiW0) ATTN_STAMP_LANE0(2);
            RowMeta nxt;
            fetch(cur.u + gridDim.x, nxt);
            // ---- gradients out of TMEM: this warp's 16 of each output's 64 columns,
            // all three loaded before one wait (the stores' source registers are
            // not reused by a following TMEM load)
            WP_BEGIN(w3_);
            tc::mbar_wait(g_bar, n & 1);
            if (warp == kEpiW0) WP_ADD(3, w3_);
            tc::tc_fence_after();
            uint32_t gv[3][16];
            tc::tmem_ld_32x16(trow + 0 + kc * 16, gv[0]);    // dV: TMEM lane = key row
            tc::tmem_ld_32x16(trow + 64 + kc * 16, gv[1]);   // dK
            tc::tmem_ld_32x16(trow + 128 + kc * 16, gv[2]);  // dQ: TMEM lane = query row
            tc::tmem_ld_wait();
            auto emit = [&](const uint32_t (&v)[16], uint16_t* base, int64_t ld, int row_lo, bool vr, float sc) {
                if (!vr) return;
                uint4* dst = reinterpret_cast<uint4*>(base + int64_t(row_lo + i) * ld + x.h * 64 + kc * 16);
#pragma unroll
                for (int q = 0; q < 2; ++q)
                    dst[q] = make_uint4(pack_bf16(__uint_as_float(v[8 * q + 0]) * sc, __uint_as_float(v[8 * q + 1]) * sc),
                                        pack_bf16(__uint_as_float(v[8 * q + 2]) * sc, __uint_as_float(v[8 * q + 3]) * sc),
                                        pack_bf16(__uint_as_float(v[8 * q + 4]) * sc, __uint_as_float(v[8 * q + 5]) * sc),
                                        pack_bf16(__uint_as_float(v[8 * q + 6]) * sc, __uint_as_float(v[8 * q + 7]) * sc));
            };
            emit(gv[0], p.dv, p.ld_dv, x.k_lo, i < x.nk, 1.f);
            emit(gv[1], p.dk, p.ld_dk, x.k_lo, i < x.nk, p.scale);
            emit(gv[2], p.dq, p.ld_dq, x.q_lo, vrow, p.scale);
            if (warp == kEpiW0) ATTN_STAMP_LANE0(3);
            tc::tc_fence_before();
            cur = nxt;
            ++n;
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc::tc_fence_after();
        tc::tmem_dealloc(tmem0, 512);
    }
}

// ---------------------------------------------------------------------------
// Forward on tcgen05: S = Q K^T in TMEM, eight warps (two per TMEM lane
// quarter, 64 keys each) build P = softmax(S) as bf16 hi + lo over the dead
// Q / K tiles, O = P V (hi and lo) in TMEM, then O and lse out.  80 KB of
// shared memory: two CTAs per SM.
constexpr int kFwdEpiW = 8;
constexpr int kFwdThreads = (kEpiW0 + kFwdEpiW) * 32;
constexpr int kFwdSmemBytes = 3 * kTile + kPTile + 2048 + 1024;  // Q K V, P lo (2 regions), meta, align

struct alignas(64) FwdParams {
    CUtensorMap mq, mk, mv;
    const int32_t* cu_q;
    const int32_t* cu_k;
    const int32_t* groups;
    float* lse;
    uint16_t* o;
    int64_t ldo;
    int total_q, causal;
    float scale;
    int early_kv;  // K / V may be loaded before griddepcontrol.wait (mm_attn_args.flags & 4)
    int n_groups, heads, long_skip;  // long kernel: the table to scan (see collect_long)
};

__global__ void __launch_bounds__(kFwdThreads, 2) attn_fwd_tc_kernel(const __grid_constant__ FwdParams p) {
    extern __shared__ uint8_t smraw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    uint8_t* Qs = sm;             // Q, K: after S = Q K^T, the P hi regions (keys 0-63, 64-127)
    uint8_t* Ks = Qs + kTile;
    uint8_t* Vs = Ks + kTile;
    uint8_t* Pl = Vs + kTile;     // P lo: two regions
    uint8_t* Ph = Qs;
    float* red = reinterpret_cast<float*>(Pl + kPTile);  // [2][128] row partials
    uint64_t* bars = reinterpret_cast<uint64_t*>(red + 2 * kRows);
    uint64_t* tma_bar = bars;
    uint64_t* s_bar = bars + 1;
    uint64_t* p_bar = bars + 2;
    uint64_t* o_bar = bars + 3;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4);

    const int h = blockIdx.x, grp = blockIdx.y;
    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
    const int lane = threadIdx.x & 31;
    const int first = p.groups[2 * grp], nseq = p.groups[2 * grp + 1];
    const int q_lo = p.cu_q[first], nq = p.cu_q[first + nseq] - q_lo;
    const int k_lo = p.cu_k[first], nk = p.cu_k[first + nseq] - k_lo;
    MM_DCHECK(nseq >= 1 && q_lo >= 0 && nq >= 1 && q_lo + nq <= p.total_q && k_lo >= 0 && nk >= 0 && nq <= 2 * kRows && nk <= 2 * kRows);
    if (nq > kRows || nk > kRows) return;  // the mma.sync kernel's group
    if (warp == 1 && lane == 0) {
        tc::mbar_init(tma_bar, 1);
        tc::mbar_init(s_bar, 1);
        tc::mbar_init(p_bar, kFwdEpiW);
        tc::mbar_init(o_bar, 1);
        tc::fence_barrier_init();
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, 256);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            if (!p.early_kv) pdl_wait();
            tc::mbar_expect_tx(tma_bar, 3 * kTile);
            tc::tma_load_2d(Ks, &p.mk, tma_bar, h * 64, k_lo);
            tc::tma_load_2d(Vs, &p.mv, tma_bar, h * 64, k_lo);
            if (p.early_kv) pdl_wait();  // (cross attention: only Q is the previous kernel's)
            tc::tma_load_2d(Qs, &p.mq, tma_bar, h * 64, q_lo);
        }
    } else if (warp == 1) {
        tc::mbar_wait(tma_bar, 0);
        tc::tc_fence_after();
        constexpr uint32_t id_s = tc::idesc_bf16_f32(128, 128, 0, 0);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
            tc::mma_bf16_elect<1>(tmem, desc(Qs + kk * 32, 16), desc(Ks + kk * 32, 16), id_s, kk > 0);
        tc::mma_commit_elect<1>(s_bar);
        tc::mbar_wait(p_bar, 0);
        tc::tc_fence_after();
        constexpr uint32_t id_o = tc::idesc_bf16_f32(128, 64, 0, 1);  // P K-major, V MN-major
#pragma unroll
        for (int part = 0; part < (kFwdPLo ? 2 : 1); ++part) {
            const uint8_t* P = part ? Pl : Ph;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
                tc::mma_bf16_elect<1>(tmem + 128, desc(P + (kk >> 2) * kTile + (kk & 3) * 32, 16),
                                      desc(Vs + kk * 2048, kTile), id_o, (part > 0 || kk > 0) ? 1u : 0u);
        }
        tc::mma_commit_elect<1>(o_bar);
    } else {
        const int quarter = warp & 3, kh = (warp - kEpiW0) >> 2;
        const int i = quarter * 32 + lane;
        const bool vrow = i < nq;
        int klo = 0, khi = 0;
        if (vrow) {
            for (int s2 = 0; s2 < nseq; ++s2) {
                const int a = p.cu_q[first + s2] - q_lo, b = p.cu_q[first + s2 + 1] - q_lo;
                if (i >= a && i < b) {
                    klo = p.cu_k[first + s2] - k_lo;
                    khi = p.causal ? klo + (i - a) + 1 : p.cu_k[first + s2 + 1] - k_lo;
                }
            }
        }
        const float c = p.scale * kLog2e;
        tc::mbar_wait(s_bar, 0);
        tc::tc_fence_after();
        const uint32_t trow = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
        float pv[64];
        float mx = -INFINITY;
        bool live[2];  // warp-uniform: some row of this warp attends to the 32-key chunk
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
            const int key0 = kh * 64 + ch * 32;
            live[ch] = __any_sync(0xffffffffu, klo < key0 + 32 && khi > key0);
            if (live[ch]) {
                uint32_t sv[32];
                tc::tmem_ld_32x32(trow + key0, sv);
                tc::tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const int key = key0 + j;
                    const float v = (key >= klo && key < khi) ? __uint_as_float(sv[j]) * c : -INFINITY;
                    pv[ch * 32 + j] = v;
                    mx = fmaxf(mx, v);
                }
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) pv[ch * 32 + j] = -INFINITY;
            }
        }
        red[kh * kRows + i] = mx;
        tc::named_barrier_sync(1, kFwdEpiW * 32);
        const float m = fmaxf(red[i], red[kRows + i]);
        const float mref = m == -INFINITY ? 0.f : m;
        float sum = 0.f;
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
            if (live[ch]) {  // dead chunks stay 0 without spending the SFU
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    pv[ch * 32 + j] = ex2(pv[ch * 32 + j] - mref);  // -inf -> 0
                    sum += pv[ch * 32 + j];
                }
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) pv[ch * 32 + j] = 0.f;
            }
        }
        tc::named_barrier_sync(1, kFwdEpiW * 32);  // every max read before the slots are reused
        red[kh * kRows + i] = sum;
        tc::named_barrier_sync(1, kFwdEpiW * 32);
        const float l = red[i] + red[kRows + i];
        const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll
        for (int j = 0; j < 64; ++j) pv[j] *= inv;
        // P over the (consumed) Q / K tiles: keys kh*64.. = region kh
        if (kFwdPLo) {
            store_row_hilo(Ph + kh * kTile, Pl + kh * kTile, i, 0, pv);
            store_row_hilo(Ph + kh * kTile, Pl + kh * kTile, i, 4, pv + 32);
        } else {
            store_row_hi(Ph + kh * kTile, i, 0, pv);
            store_row_hi(Ph + kh * kTile, i, 4, pv + 32);
        }
        tc::fence_proxy_async_smem();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(p_bar);
        if (vrow && kh == 0) p.lse[int64_t(h) * p.total_q + q_lo + i] = (mref + log2f(l)) * kLn2;
        tc::mbar_wait(o_bar, 0);
        tc::tc_fence_after();
        uint32_t v[32];
        tc::tmem_ld_32x32(trow + 128 + kh * 32, v);
        tc::tmem_ld_wait();
        if (vrow) {
            uint4* dst = reinterpret_cast<uint4*>(p.o + int64_t(q_lo + i) * p.ldo + h * 64 + kh * 32);
#pragma unroll
            for (int q = 0; q < 4; ++q)
                dst[q] = make_uint4(pack_bf16(__uint_as_float(v[8 * q + 0]), __uint_as_float(v[8 * q + 1])),
                                    pack_bf16(__uint_as_float(v[8 * q + 2]), __uint_as_float(v[8 * q + 3])),
                                    pack_bf16(__uint_as_float(v[8 * q + 4]), __uint_as_float(v[8 * q + 5])),
                                    pack_bf16(__uint_as_float(v[8 * q + 6]), __uint_as_float(v[8 * q + 7])));
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc::tc_fence_after();
        tc::tmem_dealloc(tmem, 256);
    }
}

// ---------------------------------------------------------------------------
// Groups with a sequence longer than 128 rows (config 5's length tail, up to
// 256 per side): the unpadded table gives such a sequence a group of its own.
//
// Forward: one CTA per (head, group, 128-query block); S = Q K^T over all of
// the group's keys in ONE MMA chain (N = 256 when nk > 128: K as two stacked
// 128-row SW128 boxes is one 256-row K-major operand), sixteen warps (four
// per TMEM lane quarter, 64 keys each) form P = softmax(S) as bf16 hi + lo in
// four 64-key regions, O = P V (K = 256) into TMEM, then O and lse out.
// 208 KB of shared memory, 512 TMEM columns (S 256 + O 64): one CTA per SM.
constexpr int kLongW = 16;
constexpr int kLongThreads = (kEpiW0 + kLongW) * 32;
constexpr int kLongList = (1024 + 32) * 4;  // list of long groups (kMaxLong) + chunk counts
constexpr int kLongFwdSmem = kTile /*Q*/ + 2 * kTile /*K*/ + 2 * kTile /*V*/ + 8 * kTile /*P hi+lo*/ + 4096 + kLongList + 1024;

__device__ __forceinline__ bool long_group(int nq, int nk) { return nq > kRows || nk > kRows; }

// Long groups are rare (config 5: a few per table of ~150), so the long
// kernels run one wave of persistent CTAs instead of one CTA per (head, group
// [, query block]) -- that grid was ~4800 CTAs of 208 KB shared memory, one
// per SM at a time, nearly all exiting at once: ~40 us of CTA turnover per
// launch.  Every CTA lists the table's long groups in table order (one
// parallel pass over the table, a ballot prefix per chunk), from the
// skip-th on and at most kMaxLong of them (the launcher covers the rest with
// further launches), and walks its units of that list.
constexpr int kMaxLong = 1024;
// upper bound on a table's long groups: each holds a sequence of > 128 rows
inline int long_bound(int n_groups, int total_q, int total_k) {
    return static_cast<int>(std::min<int64_t>(n_groups, int64_t(total_q) / (kRows + 1) + int64_t(total_k) / (kRows + 1)));
}

template <int NT>
__device__ int collect_long(const int32_t* groups, const int32_t* cu_q, const int32_t* cu_k, int n_groups,
                            int skip, int* list, int* wsum) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int base = 0;  // long groups in earlier chunks
    for (int g0 = 0; g0 < n_groups; g0 += NT) {
        const int g = g0 + static_cast<int>(threadIdx.x);
        bool lg = false;
        if (g < n_groups) {
            const int first = groups[2 * g], nseq = groups[2 * g + 1];
            lg = long_group(cu_q[first + nseq] - cu_q[first], cu_k[first + nseq] - cu_k[first]);
        }
        const unsigned b = __ballot_sync(0xffffffffu, lg);
        if (lane == 0) wsum[warp] = __popc(b);
        __syncthreads();
        int before = base, total = 0;
#pragma unroll
        for (int w = 0; w < NT / 32; ++w) {
            before += w < warp ? wsum[w] : 0;
            total += wsum[w];
        }
        if (lg) {
            const int idx = before + __popc(b & ((1u << lane) - 1u)) - skip;
            if (idx >= 0 && idx < kMaxLong) list[idx] = g;
        }
        base += total;
        __syncthreads();  // wsum reused by the next chunk; list complete after the last
    }
    return min(max(base - skip, 0), kMaxLong);
}

__global__ void __launch_bounds__(kLongThreads, 1) attn_fwd_long_kernel(const __grid_constant__ FwdParams p) {
    extern __shared__ uint8_t smraw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    uint8_t* Qs = sm;
    uint8_t* Ks = Qs + kTile;        // keys 0-127, 128-255
    uint8_t* Vs = Ks + 2 * kTile;
    uint8_t* Ph = Vs + 2 * kTile;    // 4 regions of 64 keys
    uint8_t* Pl = Ph + 4 * kTile;
    float* red = reinterpret_cast<float*>(Pl + 4 * kTile);  // [4][128] row partials
    uint64_t* bars = reinterpret_cast<uint64_t*>(red + 4 * kRows);
    uint64_t* tma_bar = bars;
    uint64_t* s_bar = bars + 1;
    uint64_t* p_bar = bars + 2;
    uint64_t* o_bar = bars + 3;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4);
    int* list = reinterpret_cast<int*>(sm + 13 * kTile + 4096);  // [kMaxLong] + [32] chunk counts

    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
    const int lane = threadIdx.x & 31;
    const int n_long = collect_long<kLongThreads>(p.groups, p.cu_q, p.cu_k, p.n_groups, p.long_skip, list,
                                                  list + kMaxLong);
    const int per = p.heads * 2;  // units of a long group: (head, 128-query block)
    if (static_cast<int>(blockIdx.x) >= n_long * per) return;
    if (warp == 1 && lane == 0) {
        tc::mbar_init(tma_bar, 1);
        tc::mbar_init(s_bar, 1);
        tc::mbar_init(p_bar, kLongW);
        tc::mbar_init(o_bar, 1);
        tc::fence_barrier_init();
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    uint32_t n = 0;  // units done: barrier parity
    for (int u = blockIdx.x; u < n_long * per; u += gridDim.x) {
    const int grp = list[u / per], h = (u % per) >> 1, qb = u & 1;
    const int first = p.groups[2 * grp], nseq = p.groups[2 * grp + 1];
    const int q_lo = p.cu_q[first], nq = p.cu_q[first + nseq] - q_lo;
    const int k_lo = p.cu_k[first], nk = p.cu_k[first + nseq] - k_lo;
    MM_DCHECK(nseq >= 1 && q_lo >= 0 && nq >= 1 && q_lo + nq <= p.total_q && k_lo >= 0 && nk >= 0 && nq <= 2 * kRows && nk <= 2 * kRows);
    if (qb * kRows >= nq) continue;  // no second query block (uniform over the CTA)
    const int q0 = qb * kRows;
    const int nkb = nk > kRows ? 2 : 1;
    if (warp == 0) {
        if (lane == 0) {
            if (n == 0) pdl_wait();
            tc::mbar_expect_tx(tma_bar, (1 + 2 * nkb) * kTile);
            tc::tma_load_2d(Qs, &p.mq, tma_bar, h * 64, q_lo + q0);
            for (int b = 0; b < nkb; ++b) {
                tc::tma_load_2d(Ks + b * kTile, &p.mk, tma_bar, h * 64, k_lo + b * kRows);
                tc::tma_load_2d(Vs + b * kTile, &p.mv, tma_bar, h * 64, k_lo + b * kRows);
            }
        }
    } else if (warp == 1) {
        tc::mbar_wait(tma_bar, n & 1);
        tc::tc_fence_after();
        constexpr uint32_t id_s1 = tc::idesc_bf16_f32(128, 128, 0, 0);
        constexpr uint32_t id_s2 = tc::idesc_bf16_f32(128, 256, 0, 0);
        const uint32_t id_s = nkb == 2 ? id_s2 : id_s1;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
            tc::mma_bf16_elect<1>(tmem, desc(Qs + kk * 32, 16), desc(Ks + kk * 32, 16), id_s, kk > 0);
        tc::mma_commit_elect<1>(s_bar);
        tc::mbar_wait(p_bar, n & 1);
        tc::tc_fence_after();
        constexpr uint32_t id_o = tc::idesc_bf16_f32(128, 64, 0, 1);  // P K-major, V MN-major
        for (int part = 0; part < 2; ++part) {
            const uint8_t* P = part ? Pl : Ph;
            for (int kk = 0; kk < 8 * nkb; ++kk)  // K = 16 keys per step
                tc::mma_bf16_elect<1>(tmem + 256, desc(P + (kk >> 2) * kTile + (kk & 3) * 32, 16),
                                      desc(Vs + kk * 2048, 2 * kTile), id_o, (part > 0 || kk > 0) ? 1u : 0u);
        }
        tc::mma_commit_elect<1>(o_bar);
    } else {
        const int quarter = warp & 3, kc = (warp - kEpiW0) >> 2;  // keys kc*64 .. +64
        const int i = q0 + quarter * 32 + lane;                    // query row within the group
        const bool vrow = i < nq;
        int klo = 0, khi = 0;
        if (vrow) {
            for (int s2 = 0; s2 < nseq; ++s2) {
                const int a = p.cu_q[first + s2] - q_lo, b = p.cu_q[first + s2 + 1] - q_lo;
                if (i >= a && i < b) {
                    klo = p.cu_k[first + s2] - k_lo;
                    khi = p.causal ? klo + (i - a) + 1 : p.cu_k[first + s2 + 1] - k_lo;
                }
            }
        }
        const int rl = quarter * 32 + lane;  // TMEM lane
        const float c = p.scale * kLog2e;
        tc::mbar_wait(s_bar, n & 1);
        tc::tc_fence_after();
        const uint32_t trow = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
        float pv[64];
        float mx = -INFINITY;
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
            const int key0 = kc * 64 + ch * 32;
            if (key0 < nkb * kRows && __any_sync(0xffffffffu, klo < key0 + 32 && khi > key0)) {
                uint32_t sv[32];
                tc::tmem_ld_32x32(trow + key0, sv);
                tc::tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const int key = key0 + j;
                    const float v = (key >= klo && key < khi) ? __uint_as_float(sv[j]) * c : -INFINITY;
                    pv[ch * 32 + j] = v;
                    mx = fmaxf(mx, v);
                }
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) pv[ch * 32 + j] = -INFINITY;
            }
        }
        red[kc * kRows + rl] = mx;
        tc::named_barrier_sync(1, kLongW * 32);
        const float m = fmaxf(fmaxf(red[rl], red[kRows + rl]), fmaxf(red[2 * kRows + rl], red[3 * kRows + rl]));
        const float mref = m == -INFINITY ? 0.f : m;
        float sum = 0.f;
#pragma unroll
        for (int j = 0; j < 64; ++j) {
            pv[j] = ex2(pv[j] - mref);
            sum += pv[j];
        }
        tc::named_barrier_sync(1, kLongW * 32);
        red[kc * kRows + rl] = sum;
        tc::named_barrier_sync(1, kLongW * 32);
        const float l = (red[rl] + red[kRows + rl]) + (red[2 * kRows + rl] + red[3 * kRows + rl]);
        const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll
        for (int j = 0; j < 64; ++j) pv[j] *= inv;
        store_row_hilo(Ph + kc * kTile, Pl + kc * kTile, rl, 0, pv);
        store_row_hilo(Ph + kc * kTile, Pl + kc * kTile, rl, 4, pv + 32);
        tc::fence_proxy_async_smem();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(p_bar);
        if (vrow && kc == 0) p.lse[int64_t(h) * p.total_q + q_lo + i] = (mref + log2f(l)) * kLn2;
        tc::mbar_wait(o_bar, n & 1);
        tc::tc_fence_after();
        uint32_t v[16];
        tc::tmem_ld_32x16(trow + 256 + kc * 16, v);
        tc::tmem_ld_wait();
        if (vrow) {
            uint4* dst = reinterpret_cast<uint4*>(p.o + int64_t(q_lo + i) * p.ldo + h * 64 + kc * 16);
#pragma unroll
            for (int q = 0; q < 2; ++q)
                dst[q] = make_uint4(pack_bf16(__uint_as_float(v[8 * q + 0]), __uint_as_float(v[8 * q + 1])),
                                    pack_bf16(__uint_as_float(v[8 * q + 2]), __uint_as_float(v[8 * q + 3])),
                                    pack_bf16(__uint_as_float(v[8 * q + 4]), __uint_as_float(v[8 * q + 5])),
                                    pack_bf16(__uint_as_float(v[8 * q + 6]), __uint_as_float(v[8 * q + 7])));
        }
    }
    // unit done: its TMEM reads and MMAs are complete before the next unit's
    // loads and MMAs reuse shared memory and TMEM
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    ++n;
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc::tc_fence_after();
        tc::tmem_dealloc(tmem, 512);
    }
}

// Backward of a long group: one CTA per (head, group); the group's keys in
// <= 2 blocks j of 128, its queries in <= 2 blocks i.  D_i = sum_k P dP needs
// every key block of row i, so pass 1 computes S_ij / dP_ij for all j and
// accumulates D_i (fixed j order); pass 2 loops j outer, i inner: S_ij, dP_ij
// again, P_ij (bf16 hi + lo) and dS_ij = P (dP - D_i) (bf16) into shared
// memory, then dV_j += P^T dO_i, dK_j += dS^T Q_i (accumulated over i in
// TMEM, emitted after the i loop) and dQ_i += dS K_j (both dQ blocks live in
// TMEM until the end).  TMEM: S 128 + dP 128 + dV_j 64 + dK_j 64 + dQ 2 x 64.
// One control thread issues the TMA loads and MMAs strictly in order; these
// groups are rare, so the phases are not overlapped.
constexpr int kLongBwdSmem = 2 * kTile /*K*/ + 2 * kTile /*V*/ + kTile /*Q_i*/ + kTile /*dO_i*/ +
                             2 * kPTile /*P hi+lo*/ + kPTile /*dS*/ + 4096 + kLongList + 1024;

__global__ void __launch_bounds__(kLongThreads, 1) attn_bwd_long_kernel(const __grid_constant__ BwdParams p) {
    extern __shared__ uint8_t smraw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    uint8_t* Ks = sm;
    uint8_t* Vs = Ks + 2 * kTile;
    uint8_t* Qs = Vs + 2 * kTile;
    uint8_t* dOs = Qs + kTile;
    uint8_t* Ph = dOs + kTile;
    uint8_t* Pl = Ph + kPTile;
    uint8_t* Sh = Pl + kPTile;
    float* dpart = reinterpret_cast<float*>(Sh + kPTile);  // [4][128]
    float* Dv = dpart + 4 * kRows;                           // [2][128]
    uint64_t* bars = reinterpret_cast<uint64_t*>(Dv + 2 * kRows);
    uint64_t* tma_bar = bars;
    uint64_t* s_bar = bars + 1;  // S / dP in TMEM
    uint64_t* e_bar = bars + 2;  // warps done with S / dP (pass 1) or with dV / dK (emit)
    uint64_t* p_bar = bars + 3;  // P / dS in shared memory
    uint64_t* g_bar = bars + 4;  // gradient MMAs of an (i, j) tile done
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 5);
    int* list = reinterpret_cast<int*>(Sh + kPTile + 4096);  // [kMaxLong] + [32] chunk counts

    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
    const int lane = threadIdx.x & 31;
    const int n_long = collect_long<kLongThreads>(p.groups, p.cu_q, p.cu_k, p.n_groups, p.long_skip, list,
                                                  list + kMaxLong);
    if (static_cast<int>(blockIdx.x) >= n_long * p.heads) return;
    if (warp == 1 && lane == 0) {
        tc::mbar_init(tma_bar, 1);
        tc::mbar_init(s_bar, 1);
        tc::mbar_init(e_bar, kLongW);
        tc::mbar_init(p_bar, kLongW);
        tc::mbar_init(g_bar, 1);
        tc::fence_barrier_init();
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    constexpr uint32_t T_S = 0, T_DP = 128, T_DV = 256, T_DK = 320, T_DQ = 384;
    // barrier phase counts, running over this CTA's units
    uint32_t n_tma = 0, n_s = 0, n_e = 0, n_p = 0, n_g = 0;
    for (int u = blockIdx.x; u < n_long * p.heads; u += gridDim.x) {
    const int grp = list[u / p.heads], h = u % p.heads;
    const int first = p.groups[2 * grp], nseq = p.groups[2 * grp + 1];
    const int q_lo = p.cu_q[first], nq = p.cu_q[first + nseq] - q_lo;
    const int k_lo = p.cu_k[first], nk = p.cu_k[first + nseq] - k_lo;
    MM_DCHECK(nseq >= 1 && q_lo >= 0 && nq >= 1 && q_lo + nq <= p.total_q && k_lo >= 0 && nk >= 0 && nq <= 2 * kRows && nk <= 2 * kRows);
    const int nqb = nq > kRows ? 2 : 1, nkb = nk > kRows ? 2 : 1;
    if (warp == 1) {
        // ------------------------------------------------ control: TMA + MMA, in order
        if (n_tma == 0) pdl_wait();
        auto load_qi = [&](int i, bool kv) {
            if (lane == 0) {
                tc::mbar_expect_tx(tma_bar, (2 + (kv ? 2 * nkb : 0)) * kTile);
                tc::tma_load_2d(Qs, &p.mq, tma_bar, h * 64, q_lo + i * kRows);
                tc::tma_load_2d(dOs, &p.mdo, tma_bar, h * 64, q_lo + i * kRows);
                if (kv)
                    for (int b = 0; b < nkb; ++b) {
                        tc::tma_load_2d(Ks + b * kTile, &p.mk, tma_bar, h * 64, k_lo + b * kRows);
                        tc::tma_load_2d(Vs + b * kTile, &p.mv, tma_bar, h * 64, k_lo + b * kRows);
                    }
            }
            __syncwarp();
            tc::mbar_wait(tma_bar, (n_tma++) & 1);
            tc::tc_fence_after();
        };
        constexpr uint32_t id_s = tc::idesc_bf16_f32(128, 128, 0, 0);
        auto s_dp = [&](int j) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                tc::mma_bf16_elect<1>(tmem + T_S, desc(Qs + kk * 32, 16), desc(Ks + j * kTile + kk * 32, 16), id_s, kk > 0);
                tc::mma_bf16_elect<1>(tmem + T_DP, desc(dOs + kk * 32, 16), desc(Vs + j * kTile + kk * 32, 16), id_s, kk > 0);
            }
            tc::mma_commit_elect<1>(s_bar);
            ++n_s;
        };
        // pass 1: D_i over every key block
        for (int i = 0; i < nqb; ++i) {
            load_qi(i, i == 0);
            for (int j = 0; j < nkb; ++j) {
                s_dp(j);
                tc::mbar_wait(e_bar, (n_e++) & 1);  // warps read S / dP
                tc::tc_fence_after();
            }
        }
        // pass 2
        constexpr uint32_t id_mn = tc::idesc_bf16_f32(128, 64, 1, 1);
        constexpr uint32_t id_km = tc::idesc_bf16_f32(128, 64, 0, 1);
        int loaded = nqb == 1 ? 0 : -1;  // block of Q / dO in shared memory
        for (int j = 0; j < nkb; ++j) {
            for (int i = 0; i < nqb; ++i) {
                if (loaded != i) {
                    load_qi(i, false);
                    loaded = i;
                }
                s_dp(j);
                tc::mbar_wait(p_bar, (n_p++) & 1);  // P / dS staged
                tc::tc_fence_after();
                for (int part = 0; part < 2; ++part) {
                    const uint8_t* P = part ? Pl : Ph;
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {  // K = 128 query rows
                        const uint32_t acc_v = (i > 0 || part > 0 || kk > 0) ? 1u : 0u;
                        tc::mma_bf16_elect<1>(tmem + T_DV, desc(P + kk * 2048, kTile), desc(dOs + kk * 2048, kTile), id_mn, acc_v);
                        if (part == 0)
                            tc::mma_bf16_elect<1>(tmem + T_DK, desc(Sh + kk * 2048, kTile), desc(Qs + kk * 2048, kTile), id_mn,
                                                  (i > 0 || kk > 0) ? 1u : 0u);
                    }
                }
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)  // K = 128 keys
                    tc::mma_bf16_elect<1>(tmem + T_DQ + i * 64, desc(Sh + (kk >> 2) * kTile + (kk & 3) * 32, 16),
                                          desc(Ks + j * kTile + kk * 2048, 2 * kTile), id_km, (j > 0 || kk > 0) ? 1u : 0u);
                tc::mma_commit_elect<1>(g_bar);
                tc::mbar_wait(g_bar, (n_g++) & 1);  // smem P / dS and Q / dO free again
                tc::tc_fence_after();
            }
            tc::mbar_wait(e_bar, (n_e++) & 1);  // dV_j / dK_j emitted
            tc::tc_fence_after();
        }
    } else if (warp >= kEpiW0) {
        const int quarter = warp & 3, kc = (warp - kEpiW0) >> 2;  // keys kc*32 .. +32 of a block
        const int rl = quarter * 32 + lane;
        const uint32_t trow = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
        const float c = p.scale * kLog2e;
        // this row's key range (group coordinates) for query block i
        auto range = [&](int i, int& klo, int& khi, float& l2) {
            const int qi = i * kRows + rl;
            klo = khi = 0;
            l2 = 0.f;
            if (qi >= nq) return false;
            for (int s2 = 0; s2 < nseq; ++s2) {
                const int a = p.cu_q[first + s2] - q_lo, b = p.cu_q[first + s2 + 1] - q_lo;
                if (qi >= a && qi < b) {
                    klo = p.cu_k[first + s2] - k_lo;
                    khi = p.causal ? klo + (qi - a) + 1 : p.cu_k[first + s2 + 1] - k_lo;
                }
            }
            l2 = p.lse[int64_t(h) * p.total_q + q_lo + qi] * kLog2e;
            return true;
        };
        // P (this warp's 32 keys of block j) and dP out of TMEM
        auto load_p = [&](int j, int klo, int khi, float l2, float (&pv)[32], float (&dpv)[32]) {
            const int key0 = j * kRows + kc * 32;
            if (__any_sync(0xffffffffu, klo < key0 + 32 && khi > key0)) {
                uint32_t sv[32], dv[32];
                tc::tmem_ld_32x32(trow + T_S + kc * 32, sv);
                tc::tmem_ld_32x32(trow + T_DP + kc * 32, dv);
                tc::tmem_ld_wait();
#pragma unroll
                for (int jj = 0; jj < 32; ++jj) {
                    const int key = key0 + jj;
                    pv[jj] = (key >= klo && key < khi) ? ex2(fmaf(__uint_as_float(sv[jj]), c, -l2)) : 0.f;
                    dpv[jj] = __uint_as_float(dv[jj]);
                }
            } else {
#pragma unroll
                for (int jj = 0; jj < 32; ++jj) pv[jj] = dpv[jj] = 0.f;
            }
        };
        // pass 1: D_i = sum over key blocks (j order) of sum_k P dP
        for (int i = 0; i < nqb; ++i) {
            int klo, khi;
            float l2;
            range(i, klo, khi, l2);
            for (int j = 0; j < nkb; ++j) {
                tc::mbar_wait(s_bar, (n_s++) & 1);
                tc::tc_fence_after();
                float pv[32], dpv[32];
                load_p(j, klo, khi, l2, pv, dpv);
                float dsum = 0.f;
#pragma unroll
                for (int jj = 0; jj < 32; ++jj) dsum = fmaf(pv[jj], dpv[jj], dsum);
                dpart[kc * kRows + rl] = dsum;
                tc::tc_fence_before();
                tc::named_barrier_sync(1, kLongW * 32);
                if (kc == 0) {
                    const float t = (dpart[rl] + dpart[kRows + rl]) + (dpart[2 * kRows + rl] + dpart[3 * kRows + rl]);
                    Dv[i * kRows + rl] = j == 0 ? t : Dv[i * kRows + rl] + t;
                }
                tc::named_barrier_sync(1, kLongW * 32);
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(e_bar);
            }
        }
        // pass 2
        auto emit = [&](uint32_t col, uint16_t* base, int64_t ld, int row, bool vr, float sc) {
            uint32_t v[16];
            tc::tmem_ld_32x16(trow + col + kc * 16, v);
            tc::tmem_ld_wait();
            if (!vr) return;
            uint4* dst = reinterpret_cast<uint4*>(base + int64_t(row) * ld + h * 64 + kc * 16);
#pragma unroll
            for (int q = 0; q < 2; ++q)
                dst[q] = make_uint4(pack_bf16(__uint_as_float(v[8 * q + 0]) * sc, __uint_as_float(v[8 * q + 1]) * sc),
                                    pack_bf16(__uint_as_float(v[8 * q + 2]) * sc, __uint_as_float(v[8 * q + 3]) * sc),
                                    pack_bf16(__uint_as_float(v[8 * q + 4]) * sc, __uint_as_float(v[8 * q + 5]) * sc),
                                    pack_bf16(__uint_as_float(v[8 * q + 6]) * sc, __uint_as_float(v[8 * q + 7]) * sc));
        };
        for (int j = 0; j < nkb; ++j) {
            for (int i = 0; i < nqb; ++i) {
                int klo, khi;
                float l2;
                range(i, klo, khi, l2);
                tc::mbar_wait(s_bar, (n_s++) & 1);
                tc::tc_fence_after();
                float pv[32], dpv[32];
                load_p(j, klo, khi, l2, pv, dpv);
                const float D = Dv[i * kRows + rl];
#pragma unroll
                for (int jj = 0; jj < 32; ++jj) dpv[jj] = pv[jj] * (dpv[jj] - D);  // dS
                store_row_hilo(Ph + (kc >> 1) * kTile, Pl + (kc >> 1) * kTile, rl, (kc & 1) * 4, pv);
                store_row_hi(Sh + (kc >> 1) * kTile, rl, (kc & 1) * 4, dpv);
                tc::fence_proxy_async_smem();
                tc::tc_fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(p_bar);
                tc::mbar_wait(g_bar, (n_g++) & 1);  // this tile's gradient MMAs done
                tc::tc_fence_after();
            }
            // dV_j, dK_j: TMEM lane = key row of block j
            const int key = j * kRows + rl;
            emit(T_DV, p.dv, p.ld_dv, k_lo + key, key < nk, 1.f);
            emit(T_DK, p.dk, p.ld_dk, k_lo + key, key < nk, p.scale);
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(e_bar);
        }
        for (int i = 0; i < nqb; ++i) {
            const int qi = i * kRows + rl;
            emit(T_DQ + i * 64, p.dq, p.ld_dq, q_lo + qi, qi < nq, p.scale);
        }
    }
    // unit done (every role's phase counts advanced alike): TMEM reads and
    // MMAs complete before the next unit reuses shared memory and TMEM
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc::tc_fence_after();
        tc::tmem_dealloc(tmem, 512);
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* ptr = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    });
    return fn;
}

// [rows, 64-column head slices] bf16 view with row stride ld: 128-row x 64-col SW128 boxes
int head_map(CUtensorMap* m, const void* base, int64_t rows, int64_t ld, int64_t cols) {
    auto enc = encoder();
    if (!enc) {
        mm::set_error("cuTensorMapEncodeTiled unavailable");
        return mm::kCuda;
    }
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 2)};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        mm::set_error("attention tensor map (%d): rows=%lld ld=%lld", (int)r, (long long)rows, (long long)ld);
        return mm::kCuda;
    }
    return 0;
}

}  // namespace tca

size_t fwd_smem(const mm_attn_args& a) { return size_t(3) * a.cap * kP * 2; }
size_t bwd_smem(const mm_attn_args& a) { return size_t(4) * a.cap * kP * 2 + size_t(2) * a.cap * 4; }

int check(const mm_attn_args* a, bool bwd) {
    MM_CHECK_ARG(a != nullptr, "args is NULL");
    MM_CHECK_ARG(a->head_dim == kHd || a->head_dim == 16 || a->head_dim == 32,
                 "head_dim must be 16, 32 or 64 (got %d)", a->head_dim);
    MM_CHECK_ARG(a->q && a->k && a->v && a->o && a->lse && a->cu_q && a->cu_k, "NULL tensor");
    MM_CHECK_ARG(a->n_seq >= 0 && a->heads > 0 && a->max_q > 0 && a->max_k > 0, "bad sizes");
    MM_CHECK_ARG(a->max_q <= 256 && a->max_k <= 256, "sequence longer than 256");
    MM_CHECK_ARG(a->groups && a->n_groups > 0 && a->cap >= 32 && a->cap % 32 == 0 && a->cap <= 256,
                 "bad attention work groups (cap %d)", a->cap);
    MM_CHECK_ARG((a->ldq | a->ldk | a->ldv | a->ldo) % 8 == 0, "row strides must be multiples of 8");
    MM_CHECK_ARG(!bwd || (a->d_o && a->dq && a->dk && a->dv), "NULL gradient tensor");
    return 0;
}

}  // namespace

// head_dim 16 / 32 (config 1's true shape): CUDA-core kernels, attn_small.cu
int mm_attention_small(const mm_attn_args* a, void* stream, bool bwd);

#ifdef MM_ATTN_TRACE
extern "C" int mm_attn_trace_read(unsigned long long* host, int n) {
    MM_CUDA_TRY(cudaMemcpyFromSymbol(host, g_attn_trace, sizeof(unsigned long long) * n));
    return 0;
}
#endif

extern "C" int mm_attention_fwd(const mm_attn_args* a, void* stream) {
    if (int st = check(a, false)) return st;
    if (a->n_seq == 0) return 0;
    if (a->head_dim != kHd) return mm_attention_small(a, stream, false);
    // On the padded (32-row aligned) groups the tcgen05 forward lost to the
    // mma.sync kernel (13.1 vs 10.0 us: 83 KB of smem and 256 TMEM columns
    // allow two CTAs per SM against four).
    // With the unpadded group table (fewer, fuller units) the tcgen05 forward
    // wins whenever its units fit one wave at two CTAs per SM (config 3 self
    // attention: 8.3 vs 10.0 us); beyond that (config-3 cross attention: 40+
    // groups x 8 heads) the mma.sync kernel's four CTAs per SM win (9.5 vs
    // 11.7 us).  MM_ATTN_TC_FWD=1 / 0 forces either kernel (tests, A/B).
    // Every group runs on tcgen05 by default now (groups past 128 rows in
    // attn_fwd_long_kernel); MM_ATTN_TC_FWD=0 restores the mma.sync kernel for
    // all groups, MM_ATTN_TC_FWD=auto the previous one-wave rule (A/B).
    const char* tcf = std::getenv("MM_ATTN_TC_FWD");
    const bool have_tcg = a->tc_groups != nullptr && a->n_tc_groups > 0;
    const bool auto_rule = tcf && std::strcmp(tcf, "auto") == 0;
    const bool use_tc = (tcf && !auto_rule) ? tcf[0] == '1'
                        : have_tcg && (!auto_rule || int64_t(a->n_tc_groups) * a->heads <= 2 * int64_t(mm::num_sms()));
    mm_attn_args b = *a;
    if (use_tc && a->total_k > 0) {
        tca::FwdParams fp{};
        const int64_t cols = int64_t(a->heads) * kHd;
        if (int st = tca::head_map(&fp.mq, a->q, a->total_q, a->ldq, cols)) return st;
        if (int st = tca::head_map(&fp.mk, a->k, a->total_k, a->ldk, cols)) return st;
        if (int st = tca::head_map(&fp.mv, a->v, a->total_k, a->ldv, cols)) return st;
        const bool tcg = a->tc_groups != nullptr && a->n_tc_groups > 0;  // unpadded packing
        fp.cu_q = a->cu_q; fp.cu_k = a->cu_k; fp.groups = tcg ? a->tc_groups : a->groups; fp.lse = a->lse;
        fp.o = a->o; fp.ldo = a->ldo;
        fp.total_q = a->total_q; fp.causal = a->causal; fp.scale = a->scale;
        fp.early_kv = (a->flags & 4) != 0;
        static bool attr = false;
        if (!attr) {
            MM_CUDA_TRY(cudaFuncSetAttribute(tca::attn_fwd_tc_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, tca::kFwdSmemBytes));
            attr = true;
        }
        MM_CUDA_TRY(mm::launch_pdl(tca::attn_fwd_tc_kernel, dim3(a->heads, tcg ? a->n_tc_groups : a->n_groups),
                                   dim3(tca::kFwdThreads),
                                   tca::kFwdSmemBytes, mm::as_stream(stream), fp));
        MM_LAUNCH_CHECK("attn_fwd_tc_kernel");
        if (a->cap <= tca::kRows) return 0;
        if (tcg && !std::getenv("MM_ATTN_LONG_MMA_SYNC")) {
            // groups with a sequence past 128 rows: tcgen05, one CTA per 128-query block
            static bool attr_l = false;
            if (!attr_l) {
                MM_CUDA_TRY(cudaFuncSetAttribute(tca::attn_fwd_long_kernel,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, tca::kLongFwdSmem));
                attr_l = true;
            }
            fp.n_groups = a->n_tc_groups;
            fp.heads = a->heads;
            const int bound = tca::long_bound(a->n_tc_groups, a->total_q, a->total_k);
            for (int skip = 0; skip < bound; skip += tca::kMaxLong) {  // one launch unless > kMaxLong
                fp.long_skip = skip;
                const int64_t units = int64_t(std::min(bound - skip, tca::kMaxLong)) * a->heads * 2;
                MM_CUDA_TRY(mm::launch_pdl(tca::attn_fwd_long_kernel, dim3(int(std::min<int64_t>(units, mm::num_sms()))),
                                           dim3(tca::kLongThreads), tca::kLongFwdSmem, mm::as_stream(stream), fp));
                MM_LAUNCH_CHECK("attn_fwd_long_kernel");
            }
            return 0;
        }
        b.flags = 1;  // the mma.sync kernel takes only groups with a longer sequence
    }
    a = &b;
    const size_t smem = fwd_smem(*a);
    MM_CUDA_TRY(cudaFuncSetAttribute(attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
    MM_CUDA_TRY(mm::launch_pdl(attn_fwd_kernel, dim3(a->heads, a->n_groups), dim3(kFwdWarps * 32),
                               smem, mm::as_stream(stream), *a));
    MM_LAUNCH_CHECK("attn_fwd_kernel");
    return 0;
}

extern "C" int mm_attention_bwd(const mm_attn_args* a, void* stream) {
    if (int st = check(a, true)) return st;
    if (a->n_seq == 0) return 0;
    if (a->head_dim != kHd) return mm_attention_small(a, stream, true);
    static const bool mma_sync_only = std::getenv("MM_ATTN_MMA_SYNC") != nullptr;  // diagnostics
    if (!mma_sync_only && a->total_k > 0) {
        // tcgen05 kernel for every group that fits one 128-row block per side
        tca::BwdParams bp{};
        const int64_t cols = int64_t(a->heads) * kHd;
        if (int st = tca::head_map(&bp.mq, a->q, a->total_q, a->ldq, cols)) return st;
        if (int st = tca::head_map(&bp.mk, a->k, a->total_k, a->ldk, cols)) return st;
        if (int st = tca::head_map(&bp.mv, a->v, a->total_k, a->ldv, cols)) return st;
        if (int st = tca::head_map(&bp.mdo, a->d_o, a->total_q, a->ldo, cols)) return st;
        // unpadded groups when the caller built them: a unit is one 128-row
        // TMA box per side, so the mma.sync kernels' 32-row padding only
        // multiplies the units (config 3: ~35 instead of 56 groups per table)
        const bool tcg = a->tc_groups != nullptr && a->n_tc_groups > 0;
        bp.cu_q = a->cu_q; bp.cu_k = a->cu_k; bp.groups = tcg ? a->tc_groups : a->groups; bp.lse = a->lse;
        bp.dq = a->dq; bp.dk = a->dk; bp.dv = a->dv;
        bp.ld_dq = a->ld_dq; bp.ld_dk = a->ld_dk; bp.ld_dv = a->ld_dv;
        bp.total_q = a->total_q; bp.causal = a->causal; bp.scale = a->scale;
        bp.n_groups = tcg ? a->n_tc_groups : a->n_groups; bp.heads = a->heads;
        bp.early_qkv = (a->flags & 2) != 0;
        static bool attr = false;
        if (!attr) {
            MM_CUDA_TRY(cudaFuncSetAttribute(tca::attn_bwd_tc_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, tca::kSmemBytes));
            attr = true;
        }
        const int units = bp.n_groups * a->heads;
        MM_CUDA_TRY(mm::launch_pdl(tca::attn_bwd_tc_kernel, dim3(std::min(units, mm::num_sms())),
                                   dim3(tca::kThreads), tca::kSmemBytes, mm::as_stream(stream), bp));
        MM_LAUNCH_CHECK("attn_bwd_tc_kernel");
        if (a->cap <= tca::kRows) return 0;
        if (tcg && !std::getenv("MM_ATTN_LONG_MMA_SYNC")) {
            static bool attr_l = false;
            if (!attr_l) {
                MM_CUDA_TRY(cudaFuncSetAttribute(tca::attn_bwd_long_kernel,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, tca::kLongBwdSmem));
                attr_l = true;
            }
            const int bound = tca::long_bound(bp.n_groups, a->total_q, a->total_k);
            for (int skip = 0; skip < bound; skip += tca::kMaxLong) {
                bp.long_skip = skip;
                const int64_t units = int64_t(std::min(bound - skip, tca::kMaxLong)) * a->heads;
                MM_CUDA_TRY(mm::launch_pdl(tca::attn_bwd_long_kernel, dim3(int(std::min<int64_t>(units, mm::num_sms()))),
                                           dim3(tca::kLongThreads), tca::kLongBwdSmem, mm::as_stream(stream), bp));
                MM_LAUNCH_CHECK("attn_bwd_long_kernel");
            }
            return 0;
        }
    }
    // groups with a sequence longer than 128 rows (or the diagnostics path):
    // the mma.sync kernel, skipping groups the tcgen05 kernel took
    mm_attn_args b = *a;
    b.flags = (!mma_sync_only && a->total_k > 0) ? 1 : 0;
    a = &b;
    const size_t smem = bwd_smem(*a);
    MM_CHECK_ARG(smem <= 227 * 1024, "attention backward needs %zu B of smem", smem);
    MM_CUDA_TRY(cudaFuncSetAttribute(attn_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
    MM_CUDA_TRY(mm::launch_pdl(attn_bwd_kernel, dim3(a->heads, a->n_groups), dim3(kBwdWarps * 32),
                               smem, mm::as_stream(stream), *a));
    MM_LAUNCH_CHECK("attn_bwd_kernel");
    return 0;
}

#ifdef MM_ATTN_WAITPROF
extern "C" int mm_attn_wp_read(unsigned long long* host, int zero) {
    if (zero) {
        static unsigned long long z[148 * 8] = {};
        MM_CUDA_TRY(cudaMemcpyToSymbol(tca::g_wp, z, sizeof(z)));
        return 0;
    }
    MM_CUDA_TRY(cudaMemcpyFromSymbol(host, tca::g_wp, sizeof(unsigned long long) * 148 * 8));
    return 0;
}
#endif
