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
#include <cuda_bf16.h>

#include <algorithm>

#include "mm_common.h"

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
#else
#define ATTN_STAMP(i) \
    do {              \
    } while (0)
#endif

__global__ void __launch_bounds__(kBwdWarps * 32, 2) attn_bwd_kernel(const mm_attn_args a) {
    extern __shared__ __align__(16) uint16_t sm[];
    __shared__ Group G;
    const int h = blockIdx.x;  // heads fastest: a group's CTAs run together and share its rows' DRAM pages
    if (threadIdx.x < 32) load_group(G, a, threadIdx.x);  // host-uploaded: before the wait
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

size_t fwd_smem(const mm_attn_args& a) { return size_t(3) * a.cap * kP * 2; }
size_t bwd_smem(const mm_attn_args& a) { return size_t(4) * a.cap * kP * 2 + size_t(2) * a.cap * 4; }

int check(const mm_attn_args* a, bool bwd) {
    MM_CHECK_ARG(a != nullptr, "args is NULL");
    MM_CHECK_ARG(a->head_dim == kHd, "head_dim must be 64 (got %d)", a->head_dim);
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

#ifdef MM_ATTN_TRACE
extern "C" int mm_attn_trace_read(unsigned long long* host, int n) {
    MM_CUDA_TRY(cudaMemcpyFromSymbol(host, g_attn_trace, sizeof(unsigned long long) * n));
    return 0;
}
#endif

extern "C" int mm_attention_fwd(const mm_attn_args* a, void* stream) {
    if (int st = check(a, false)) return st;
    if (a->n_seq == 0) return 0;
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
    const size_t smem = bwd_smem(*a);
    MM_CHECK_ARG(smem <= 227 * 1024, "attention backward needs %zu B of smem", smem);
    MM_CUDA_TRY(cudaFuncSetAttribute(attn_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
    MM_CUDA_TRY(mm::launch_pdl(attn_bwd_kernel, dim3(a->heads, a->n_groups), dim3(kBwdWarps * 32),
                               smem, mm::as_stream(stream), *a));
    MM_LAUNCH_CHECK("attn_bwd_kernel");
    return 0;
}
