// K6 LayerNorm, K8 embedding gather / scatter-add, K7 softmax cross-entropy,
// and the bias-gradient column sums.  All HBM-bound: warp-per-row mappings
// with 128-bit vector accesses and warp-shuffle reductions.
#ifndef MM_LN_FWD_WARPS
// rows (warps) per CTA of the row-per-warp LayerNorm forward
#define MM_LN_FWD_WARPS 4
#endif
#ifndef MM_LN_BWD_PREFETCH
#define MM_LN_BWD_PREFETCH 1
#endif
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>

#include "mm_common.h"
#include "tc_ptx.cuh"

namespace {

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
__device__ __forceinline__ float bf2f(uint16_t h) { return __uint_as_float(uint32_t(h) << 16); }
__device__ __forceinline__ uint16_t f2bf(float f) {
    __nv_bfloat16 h = __float2bfloat16_rn(f);
    return *reinterpret_cast<uint16_t*>(&h);
}
// two floats -> packed bf16x2 in one conversion instruction (F2FP) instead
// of two single conversions; same round-to-nearest-even bits
__device__ __forceinline__ uint32_t pack2(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}

// ----------------------------------------------------------------------------
// LayerNorm: a warp owns R rows at a time (all their loads issued before any
// reduction, for memory-level parallelism); lane owns columns
// {4*lane + 128*i}, COLS/128 float4 per row in registers.
constexpr int kLnRows = 2;

template <int COLS>
__global__ void __launch_bounds__(256) ln_fwd_kernel(const float* __restrict__ x,
                                                     const float* __restrict__ gamma,
                                                     const float* __restrict__ beta,
                                                     uint16_t* __restrict__ y, float* mean_out,
                                                     float* rstd_out, int64_t rows, float eps) {
    pdl_wait_release();
    // COLS = 64 (config 1): one float4 per lane on half the warp, the other
    // lanes hold zeros and stay out of the variance and the stores
    constexpr int V = (COLS + 127) / 128;
    const int lane = threadIdx.x & 31;
    auto live = [&](int i) { return COLS % 128 == 0 || lane + 32 * i < COLS / 4; };
    const int64_t row0 = (int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5)) * kLnRows;
    float4 v[kLnRows][V];
#pragma unroll
    for (int r = 0; r < kLnRows; ++r) {
        const int64_t row = min(row0 + r, rows - 1);
        const float4* xr = reinterpret_cast<const float4*>(x + row * COLS);
#pragma unroll
        for (int i = 0; i < V; ++i) v[r][i] = live(i) ? xr[lane + 32 * i] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int r = 0; r < kLnRows; ++r) {
        const int64_t row = row0 + r;
        float s = 0.f;
#pragma unroll
        for (int i = 0; i < V; ++i) s += v[r][i].x + v[r][i].y + v[r][i].z + v[r][i].w;
        const float mu = warp_sum(s) * (1.f / COLS);
        float q = 0.f;
#pragma unroll
        for (int i = 0; i < V; ++i) {
            if (!live(i)) continue;
            const float a = v[r][i].x - mu, b = v[r][i].y - mu, c = v[r][i].z - mu, d = v[r][i].w - mu;
            q += a * a + b * b + c * c + d * d;
        }
        const float rs = rsqrtf(warp_sum(q) * (1.f / COLS) + eps);
        if (row >= rows) continue;
        uint2* yr = reinterpret_cast<uint2*>(y + row * COLS);
#pragma unroll
        for (int i = 0; i < V; ++i) {
            if (!live(i)) continue;
            const int c = 4 * lane + 128 * i;
            const float4 g = __ldg(reinterpret_cast<const float4*>(gamma + c));
            const float4 bb = __ldg(reinterpret_cast<const float4*>(beta + c));
            uint2 o;
            o.x = pack2((v[r][i].x - mu) * rs * g.x + bb.x, (v[r][i].y - mu) * rs * g.y + bb.y);
            o.y = pack2((v[r][i].z - mu) * rs * g.z + bb.z, (v[r][i].w - mu) * rs * g.w + bb.w);
            yr[lane + 32 * i] = o;
        }
        if (lane == 0) {
            mean_out[row] = mu;
            rstd_out[row] = rs;
        }
    }
}

// Backward: dxhat = dy*gamma; dx_ln = rstd*(dxhat - mean(dxhat) - xhat*mean(dxhat*xhat)).
// dx += dx_ln (residual-stream gradient, fp32) and its bf16 copy is written;
// dgamma += sum(dy*xhat), dbeta += sum(dy) accumulated per lane across the
// block's rows, reduced over warps in smem, one atomicAdd per column per block.
template <int COLS>
__global__ void __launch_bounds__(256, (COLS <= 512 ? 2 : 1)) ln_bwd_kernel(const float* __restrict__ dy,
                                                     const float* __restrict__ x,
                                                     const float* __restrict__ gamma,
                                                     const float* __restrict__ mean,
                                                     const float* __restrict__ rstd, float* dx,
                                                     uint16_t* dx_bf16, float* dgamma,
                                                     float* dbeta, int64_t rows) {
    pdl_wait_release();
    constexpr int V = (COLS + 127) / 128;  // COLS = 64: half the lanes live (see ln_fwd_kernel)
    constexpr int R = COLS <= 512 ? kLnRows : 1;  // rows per warp batch (register budget)
    __shared__ float red_g[8][COLS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    auto lane_on = [&](int i) { return COLS % 128 == 0 || lane + 32 * i < COLS / 4; };
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 ag[V], ab[V];
#pragma unroll
    for (int i = 0; i < V; ++i) ag[i] = ab[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    const int64_t stride = int64_t(gridDim.x) * 8 * R;
    for (int64_t row0 = (int64_t(blockIdx.x) * 8 + warp) * R; row0 < rows; row0 += stride) {
        // wide rows (one row per warp batch): the residual-gradient row is
        // fetched with dy and x, one DRAM round trip per row instead of two
        constexpr bool kPreDx = R == 1;
        float4 d[R][V], xv[R][V], opre[kPreDx ? V : 1];
        float mu[R], rs[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {  // every dy / x load of the batch first
            const int64_t row = min(row0 + r, rows - 1);
            mu[r] = mean[row];
            rs[r] = rstd[row];
            const float4* dyr = reinterpret_cast<const float4*>(dy + row * COLS);
            const float4* xr = reinterpret_cast<const float4*>(x + row * COLS);
#pragma unroll
            for (int i = 0; i < V; ++i) {
                d[r][i] = lane_on(i) ? dyr[lane + 32 * i] : z4;
                xv[r][i] = lane_on(i) ? xr[lane + 32 * i] : z4;
            }
            if constexpr (kPreDx) {
                const float4* dxr = reinterpret_cast<const float4*>(dx + row * COLS);
#pragma unroll
                for (int i = 0; i < V; ++i) opre[i] = lane_on(i) ? dxr[lane + 32 * i] : z4;
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int64_t row = row0 + r;
            const bool live = row < rows;
            float s1 = 0.f, s2 = 0.f;
#pragma unroll
            for (int i = 0; i < V; ++i) {
                float4& xh = xv[r][i];
                xh = make_float4((xh.x - mu[r]) * rs[r], (xh.y - mu[r]) * rs[r],
                                 (xh.z - mu[r]) * rs[r], (xh.w - mu[r]) * rs[r]);
                const float4 gm = lane_on(i) ? __ldg(reinterpret_cast<const float4*>(gamma + 4 * lane + 128 * i)) : z4;
                const float4 g = make_float4(d[r][i].x * gm.x, d[r][i].y * gm.y,
                                             d[r][i].z * gm.z, d[r][i].w * gm.w);
                s1 += g.x + g.y + g.z + g.w;
                s2 += g.x * xh.x + g.y * xh.y + g.z * xh.z + g.w * xh.w;
                if (live) {
                    ag[i].x += d[r][i].x * xh.x; ag[i].y += d[r][i].y * xh.y;
                    ag[i].z += d[r][i].z * xh.z; ag[i].w += d[r][i].w * xh.w;
                    ab[i].x += d[r][i].x; ab[i].y += d[r][i].y; ab[i].z += d[r][i].z; ab[i].w += d[r][i].w;
                }
                d[r][i] = g;  // keep dxhat
            }
            const float m1 = warp_sum(s1) * (1.f / COLS), m2 = warp_sum(s2) * (1.f / COLS);
            if (!live) continue;
            float4* dxr = reinterpret_cast<float4*>(dx + row * COLS);
            uint2* dbr = reinterpret_cast<uint2*>(dx_bf16 + row * COLS);
            float4 o[V];
#pragma unroll
            for (int i = 0; i < V; ++i) o[i] = kPreDx ? opre[kPreDx ? i : 0] : (lane_on(i) ? dxr[lane + 32 * i] : z4);
#pragma unroll
            for (int i = 0; i < V; ++i) {
                if (!lane_on(i)) continue;
                float4 w = o[i];
                w.x += rs[r] * (d[r][i].x - m1 - xv[r][i].x * m2);
                w.y += rs[r] * (d[r][i].y - m1 - xv[r][i].y * m2);
                w.z += rs[r] * (d[r][i].z - m1 - xv[r][i].z * m2);
                w.w += rs[r] * (d[r][i].w - m1 - xv[r][i].w * m2);
                dxr[lane + 32 * i] = w;
                if (dx_bf16) {
                    uint2 b;
                    b.x = pack2(w.x, w.y);
                    b.y = pack2(w.z, w.w);
                    dbr[lane + 32 * i] = b;
                }
            }
        }
    }
    // two reductions through the same smem buffer
    for (int pass = 0; pass < 2; ++pass) {
#pragma unroll
        for (int i = 0; i < V; ++i) {
            const float4 a = pass == 0 ? ag[i] : ab[i];
            if (lane_on(i)) *reinterpret_cast<float4*>(&red_g[warp][4 * lane + 128 * i]) = a;
        }
        __syncthreads();
        float* dst = pass == 0 ? dgamma : dbeta;
        for (int c = threadIdx.x; c < COLS; c += 256) {
            float sum = 0.f;
#pragma unroll
            for (int w = 0; w < 8; ++w) sum += red_g[w][c];
            atomicAdd(dst + c, sum);
        }
        __syncthreads();
    }
}

// Backward, one row per warp: dy, x AND the residual-gradient row dx are
// all requested before the first reduction (one DRAM round trip per row), and
// the dgamma / dbeta partials live in shared memory (a lane owns its columns,
// plain read-modify-write, no conflicts) instead of registers, so the kernel
// fits MINB CTAs per SM and the whole config-3 problem in one wave.
template <int COLS, int MINB>
__global__ void __launch_bounds__(256, MINB) ln_bwd_row_kernel(const float* __restrict__ dy,
                                                               const float* __restrict__ x,
                                                               const float* __restrict__ gamma,
                                                               const float* __restrict__ mean,
                                                               const float* __restrict__ rstd, float* dx,
                                                               uint16_t* dx_bf16, float* dgamma,
                                                               float* dbeta, int64_t rows) {
    constexpr int V = COLS / 128;
    extern __shared__ float4 red4[];  // [2][8 warps][COLS / 4]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float4* rg = red4 + warp * (COLS / 4);
    float4* rb = red4 + (8 + warp) * (COLS / 4);
#pragma unroll
    for (int i = 0; i < V; ++i) rg[lane + 32 * i] = rb[lane + 32 * i] = make_float4(0.f, 0.f, 0.f, 0.f);
#if MM_LN_BWD_PREFETCH
    // before griddepcontrol.wait: pull this warp's rows of the forward input x
    // and of the residual gradient dx (both written several kernels earlier;
    // an L2 prefetch is coherent whatever the previous kernel writes) into L2,
    // so their HBM fetch overlaps the producer of dy instead of following it
    for (int64_t row = int64_t(blockIdx.x) * 8 + warp; row < rows; row += int64_t(gridDim.x) * 8) {
        const float* base = (lane < 16 ? x : dx) + row * COLS;
        for (int c = (lane & 15) * 32; c < COLS; c += 16 * 32)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(base + c));
    }
#endif
    pdl_wait_release();
    for (int64_t row = int64_t(blockIdx.x) * 8 + warp; row < rows; row += int64_t(gridDim.x) * 8) {
        const float4* dyr = reinterpret_cast<const float4*>(dy + row * COLS);
        const float4* xr = reinterpret_cast<const float4*>(x + row * COLS);
        float4* dxr = reinterpret_cast<float4*>(dx + row * COLS);
        float4 d[V], xv[V], o[V];
        const float mu = mean[row], rs = rstd[row];
#pragma unroll
        for (int i = 0; i < V; ++i) {
            d[i] = __ldcs(dyr + lane + 32 * i);
            xv[i] = __ldcs(xr + lane + 32 * i);
            o[i] = __ldcs(dxr + lane + 32 * i);
        }
        float s1 = 0.f, s2 = 0.f;
#pragma unroll
        for (int i = 0; i < V; ++i) {
            float4& xh = xv[i];
            xh = make_float4((xh.x - mu) * rs, (xh.y - mu) * rs, (xh.z - mu) * rs, (xh.w - mu) * rs);
            float4 a = rg[lane + 32 * i], b = rb[lane + 32 * i];
            a.x += d[i].x * xh.x; a.y += d[i].y * xh.y; a.z += d[i].z * xh.z; a.w += d[i].w * xh.w;
            b.x += d[i].x; b.y += d[i].y; b.z += d[i].z; b.w += d[i].w;
            rg[lane + 32 * i] = a;
            rb[lane + 32 * i] = b;
            const float4 gm = __ldg(reinterpret_cast<const float4*>(gamma + 4 * lane + 128 * i));
            d[i] = make_float4(d[i].x * gm.x, d[i].y * gm.y, d[i].z * gm.z, d[i].w * gm.w);  // dxhat
            s1 += d[i].x + d[i].y + d[i].z + d[i].w;
            s2 += d[i].x * xh.x + d[i].y * xh.y + d[i].z * xh.z + d[i].w * xh.w;
        }
        const float m1 = warp_sum(s1) * (1.f / COLS), m2 = warp_sum(s2) * (1.f / COLS);
        uint2* dbr = reinterpret_cast<uint2*>(dx_bf16 + row * COLS);
#pragma unroll
        for (int i = 0; i < V; ++i) {
            float4 w = o[i];
            w.x += rs * (d[i].x - m1 - xv[i].x * m2);
            w.y += rs * (d[i].y - m1 - xv[i].y * m2);
            w.z += rs * (d[i].z - m1 - xv[i].z * m2);
            w.w += rs * (d[i].w - m1 - xv[i].w * m2);
            dxr[lane + 32 * i] = w;
            if (dx_bf16) {
                uint2 b;
                b.x = pack2(w.x, w.y);
                b.y = pack2(w.z, w.w);
                dbr[lane + 32 * i] = b;
            }
        }
    }
    __syncthreads();
    // column sums over the 8 warps, one vector atomic per 4 columns per CTA
    for (int c4 = threadIdx.x; c4 < 2 * (COLS / 4); c4 += 256) {
        const int which = c4 / (COLS / 4), c = c4 - which * (COLS / 4);
        float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            const float4 v = red4[(which * 8 + w) * (COLS / 4) + c];
            sum.x += v.x; sum.y += v.y; sum.z += v.z; sum.w += v.w;
        }
#ifndef MM_LN_DIAG_NO_COLSUM  // diagnostics only (timing A/B): drops dgamma / dbeta
        atomicAdd(reinterpret_cast<float4*>(which ? dbeta : dgamma) + c, sum);
#endif
    }
}

// ----------------------------------------------------------------------------
// LayerNorm v2 (default): one row per warp, 4-warp CTAs, every row of the
// problem in flight in one wave (4096 rows = 1024 CTAs, ~7 per SM: balanced,
// where 256 CTAs of 8 warps left half the SMs with one CTA and half with two).
// Forward: 2 KB (d = 512) of fp32 row per warp loaded at once, two-pass mean /
// variance from registers, bf16 out.
template <int COLS>
__global__ void __launch_bounds__(32 * MM_LN_FWD_WARPS) ln_fwd_v2_kernel(const float* __restrict__ x,
                                                        const float* __restrict__ gamma,
                                                        const float* __restrict__ beta,
                                                        uint16_t* __restrict__ y, float* mean_out,
                                                        float* rstd_out, int64_t rows, float eps) {
    constexpr int V = COLS / 128;
    const int lane = threadIdx.x & 31;
    const int64_t row = int64_t(blockIdx.x) * MM_LN_FWD_WARPS + (threadIdx.x >> 5);
    pdl_wait_release();
    if (row >= rows) return;
    const float4* xr = reinterpret_cast<const float4*>(x + row * COLS);
    float4 v[V];
#pragma unroll
    for (int i = 0; i < V; ++i) v[i] = __ldcs(xr + lane + 32 * i);
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < V; ++i) s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
    const float mu = warp_sum(s) * (1.f / COLS);
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < V; ++i) {
        const float a = v[i].x - mu, b = v[i].y - mu, c = v[i].z - mu, d = v[i].w - mu;
        q += (a * a + b * b) + (c * c + d * d);
    }
    const float rs = rsqrtf(warp_sum(q) * (1.f / COLS) + eps);
    uint2* yr = reinterpret_cast<uint2*>(y + row * COLS);
#pragma unroll
    for (int i = 0; i < V; ++i) {
        const int c = 4 * lane + 128 * i;
        const float4 g = __ldg(reinterpret_cast<const float4*>(gamma + c));
        const float4 bb = __ldg(reinterpret_cast<const float4*>(beta + c));
        uint2 o;
        o.x = pack2((v[i].x - mu) * rs * g.x + bb.x, (v[i].y - mu) * rs * g.y + bb.y);
        o.y = pack2((v[i].z - mu) * rs * g.z + bb.z, (v[i].w - mu) * rs * g.w + bb.w);
        yr[lane + 32 * i] = o;
    }
    if (lane == 0) {
        mean_out[row] = mu;
        rstd_out[row] = rs;
    }
}

// Backward v2: one row per warp, 8-warp CTAs at up to four per SM (<= 64
// registers: the whole config-3 problem, 4096 rows, resident in one wave).
// dy and x are loaded at once; the residual-gradient row dx is only PREFETCHED
// into L2 then (no registers held across the reductions) and read after them.
// dgamma / dbeta: per-CTA column partials in shared memory (a lane owns its
// columns, no conflicts), one float4 atomic per 4 columns per CTA.
template <int COLS>
__global__ void __launch_bounds__(256, 4) ln_bwd_v2_kernel(const float* __restrict__ dy,
                                                           const float* __restrict__ x,
                                                           const float* __restrict__ gamma,
                                                           const float* __restrict__ mean,
                                                           const float* __restrict__ rstd, float* dx,
                                                           uint16_t* dx_bf16, float* dgamma,
                                                           float* dbeta, int64_t rows) {
    constexpr int V = COLS / 128;
    __shared__ float4 red[2][8][COLS / 4];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t row = int64_t(blockIdx.x) * 8 + warp;
    pdl_wait_release();
    const bool live = row < rows;
    float4 d[V], xv[V];
    if (live) {
        const float4* dyr = reinterpret_cast<const float4*>(dy + row * COLS);
        const float4* xr = reinterpret_cast<const float4*>(x + row * COLS);
        const char* dxr = reinterpret_cast<const char*>(dx + row * COLS);
#pragma unroll
        for (int i = 0; i < V; ++i) {
            d[i] = __ldcs(dyr + lane + 32 * i);
            xv[i] = __ldcs(xr + lane + 32 * i);
        }
        if (lane < COLS * 4 / 128)  // one 128-byte line per lane
            asm volatile("prefetch.global.L2 [%0];" ::"l"(dxr + lane * 128));
    } else {
#pragma unroll
        for (int i = 0; i < V; ++i) d[i] = xv[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const float mu = live ? mean[row] : 0.f, rs = live ? rstd[row] : 0.f;
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < V; ++i) {
        float4& xh = xv[i];
        xh = make_float4((xh.x - mu) * rs, (xh.y - mu) * rs, (xh.z - mu) * rs, (xh.w - mu) * rs);
        red[0][warp][lane + 32 * i] = make_float4(d[i].x * xh.x, d[i].y * xh.y, d[i].z * xh.z, d[i].w * xh.w);
        red[1][warp][lane + 32 * i] = d[i];
        const float4 gm = __ldg(reinterpret_cast<const float4*>(gamma + 4 * lane + 128 * i));
        d[i] = make_float4(d[i].x * gm.x, d[i].y * gm.y, d[i].z * gm.z, d[i].w * gm.w);  // dxhat
        s1 += d[i].x + d[i].y + d[i].z + d[i].w;
        s2 += d[i].x * xh.x + d[i].y * xh.y + d[i].z * xh.z + d[i].w * xh.w;
    }
    const float m1 = warp_sum(s1) * (1.f / COLS), m2 = warp_sum(s2) * (1.f / COLS);
    if (live) {
        float4* dxr = reinterpret_cast<float4*>(dx + row * COLS);
        uint2* dbr = reinterpret_cast<uint2*>(dx_bf16 + row * COLS);
#pragma unroll
        for (int i = 0; i < V; ++i) {
            float4 w = dxr[lane + 32 * i];
            w.x += rs * (d[i].x - m1 - xv[i].x * m2);
            w.y += rs * (d[i].y - m1 - xv[i].y * m2);
            w.z += rs * (d[i].z - m1 - xv[i].z * m2);
            w.w += rs * (d[i].w - m1 - xv[i].w * m2);
            dxr[lane + 32 * i] = w;
            if (dx_bf16) {
                uint2 b;
                b.x = pack2(w.x, w.y);
                b.y = pack2(w.z, w.w);
                dbr[lane + 32 * i] = b;
            }
        }
    }
    __syncthreads();
    for (int c4 = threadIdx.x; c4 < 2 * (COLS / 4); c4 += 256) {
        const int which = c4 / (COLS / 4), c = c4 - which * (COLS / 4);
        float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            const float4 v = red[which][w][c];
            sum.x += v.x; sum.y += v.y; sum.z += v.z; sum.w += v.w;
        }
        atomicAdd(reinterpret_cast<float4*>(which ? dbeta : dgamma) + c, sum);
    }
}

// ----------------------------------------------------------------------------
// Embedding: out[r,:] = table[id[r],:] * scale + PE(pos[r]) (sinusoidal,
// sin on even / cos on odd columns, OpenNMT layout).  One warp per row.
__global__ void __launch_bounds__(256) embed_fwd_kernel(const int32_t* __restrict__ ids,
                                                        const int32_t* __restrict__ pos,
                                                        const uint16_t* __restrict__ table,
                                                        float* __restrict__ out, int64_t rows,
                                                        int cols, float scale) {
    pdl_wait_release();
    const int lane = threadIdx.x & 31;
    const int64_t row = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (row >= rows) return;
    const int64_t id = ids[row];
    MM_DCHECK(id >= 0 && pos[row] >= 0);
    const float p = static_cast<float>(pos[row]);
    const uint2* tr = reinterpret_cast<const uint2*>(table + id * cols);
    float4* orow = reinterpret_cast<float4*>(out + row * cols);
    const float kLog = -9.210340371976184f / static_cast<float>(cols);  // -ln(10000)/d
    for (int v = lane; v < cols / 4; v += 32) {
        const uint2 w = __ldg(tr + v);
        const int c = 4 * v;
        const float f0 = expf(kLog * static_cast<float>(c));
        const float f1 = expf(kLog * static_cast<float>(c + 2));
        float s0, c0, s1, c1;
        sincosf(p * f0, &s0, &c0);
        sincosf(p * f1, &s1, &c1);
        float4 o;
        o.x = bf2f(w.x & 0xffff) * scale + s0;
        o.y = bf2f(w.x >> 16) * scale + c0;
        o.z = bf2f(w.y & 0xffff) * scale + s1;
        o.w = bf2f(w.y >> 16) * scale + c1;
        orow[v] = o;
    }
}

__global__ void __launch_bounds__(256) embed_bwd_kernel(const int32_t* __restrict__ ids,
                                                        const float* __restrict__ dout,
                                                        float* dtable, int64_t rows, int cols,
                                                        float scale) {
    pdl_wait_release();
    const int lane = threadIdx.x & 31;
    const int64_t row = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (row >= rows) return;
    const int64_t id = ids[row];
    const float4* d = reinterpret_cast<const float4*>(dout + row * cols);
    float4* t = reinterpret_cast<float4*>(dtable + id * cols);
    for (int v = lane; v < cols / 4; v += 32) {
        float4 g = d[v];
        g.x *= scale; g.y *= scale; g.z *= scale; g.w *= scale;
        atomicAdd(t + v, g);
    }
}

// Deterministic scatter-add (mm_embed_segments tables): a warp per chunk sums
// its rows (ascending row order within the token id) and adds the sum into the
// table row when the id has one chunk, else writes the chunk's partial; a warp
// per multi-chunk id then adds the partials in chunk order.  Every table row
// has one writer per launch and a fixed summation order: no atomics, bitwise
// reproducible, and a Zipf-hot id costs one partial per 32 rows instead of
// hundreds of serialised atomics on one row.
constexpr int kEmbMaxV = 8;  // float4 per lane: cols <= 1024

// V = cols / 128 float4 per lane; R rows loaded per batch (independent loads
// in flight, summed in row order): the chunk's row indices come in with one
// coalesced load and are broadcast by shuffles, so no load waits on another
template <int V, int R, int C4 = 32 * V>  // C4 float4 per row (16: cols = 64)
__global__ void __launch_bounds__(256) embed_bwd_chunk_kernel(const int32_t* __restrict__ perm,
                                                              const int32_t* __restrict__ chunks,
                                                              int n_chunks, const float* __restrict__ dout,
                                                              float* dtable, float* scratch, float scale) {
    constexpr int cols = C4 * 4;
    pdl_wait_release();
    const int lane = threadIdx.x & 31;
    const int c = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (c >= n_chunks) return;
    const int b = chunks[3 * c], e = chunks[3 * c + 1], tgt = chunks[3 * c + 2];
    const int n = e - b;  // <= 32 (EMB_CHUNK_ROWS)
    MM_DCHECK(b >= 0 && n >= 1 && n <= 32);
    const int my_row = lane < n ? perm[b + lane] : 0;
    MM_DCHECK(my_row >= 0);
    float4 acc[V];
#pragma unroll
    for (int i = 0; i < V; ++i) acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int r0 = 0; r0 < n; r0 += R) {
        float4 g[R][V];
#pragma unroll
        for (int u = 0; u < R; ++u) {
            const int row = __shfl_sync(0xffffffffu, my_row, (r0 + u) & 31);
            const float4* d = reinterpret_cast<const float4*>(dout + int64_t(row) * cols);
#pragma unroll
            for (int i = 0; i < V; ++i) g[u][i] = r0 + u < n && (C4 == 32 * V || lane + 32 * i < C4) ? d[lane + 32 * i] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < R; ++u) {
            if (r0 + u >= n) break;
#pragma unroll
            for (int i = 0; i < V; ++i) {
                acc[i].x = fmaf(g[u][i].x, scale, acc[i].x); acc[i].y = fmaf(g[u][i].y, scale, acc[i].y);
                acc[i].z = fmaf(g[u][i].z, scale, acc[i].z); acc[i].w = fmaf(g[u][i].w, scale, acc[i].w);
            }
        }
    }
    float4* dst = tgt >= 0 ? reinterpret_cast<float4*>(dtable + int64_t(tgt) * cols)
                           : reinterpret_cast<float4*>(scratch + int64_t(-tgt - 1) * cols);
#pragma unroll
    for (int i = 0; i < V; ++i) {
        const int v = lane + 32 * i;
        if (C4 != 32 * V && v >= C4) continue;
        if (tgt >= 0) {
            float4 t = dst[v];
            t.x += acc[i].x; t.y += acc[i].y; t.z += acc[i].z; t.w += acc[i].w;
            dst[v] = t;
        } else {
            dst[v] = acc[i];
        }
    }
}

// one warp per multi-chunk id: its partials (R per batch, independent loads)
// added in chunk order, then into the table row
template <int V, int R, int C4 = 32 * V>  // C4 float4 per row (16: cols = 64)
__global__ void __launch_bounds__(256) embed_bwd_multi_kernel(const int32_t* __restrict__ multi, int n_multi,
                                                              const float* __restrict__ scratch,
                                                              float* dtable) {
    constexpr int cols = C4 * 4;
    pdl_wait_release();
    const int lane = threadIdx.x & 31;
    const int m = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (m >= n_multi) return;
    const int id = multi[3 * m], s0 = multi[3 * m + 1], ns = multi[3 * m + 2];
    MM_DCHECK(id >= 0 && s0 >= 0 && ns >= 2);
    float4 a[V];
#pragma unroll
    for (int i = 0; i < V; ++i) a[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int k0 = 0; k0 < ns; k0 += R) {
        float4 x[R][V];
#pragma unroll
        for (int u = 0; u < R; ++u)
#pragma unroll
            for (int i = 0; i < V; ++i)
                x[u][i] = k0 + u < ns && (C4 == 32 * V || lane + 32 * i < C4) ? reinterpret_cast<const float4*>(scratch + int64_t(s0 + k0 + u) * cols)[lane + 32 * i]
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < R; ++u) {
            if (k0 + u >= ns) break;
#pragma unroll
            for (int i = 0; i < V; ++i) {
                a[i].x += x[u][i].x; a[i].y += x[u][i].y; a[i].z += x[u][i].z; a[i].w += x[u][i].w;
            }
        }
    }
    float4* dst = reinterpret_cast<float4*>(dtable + int64_t(id) * cols);
#pragma unroll
    for (int i = 0; i < V; ++i) {
        if (C4 != 32 * V && lane + 32 * i >= C4) continue;
        float4 t = dst[lane + 32 * i];
        t.x += a[i].x; t.y += a[i].y; t.z += a[i].z; t.w += a[i].w;
        dst[lane + 32 * i] = t;
    }
}

template <int V, int C4 = 32 * V>
int embed_sorted_launch(const int32_t* perm, const int32_t* chunks, int n_chunks, const int32_t* multi,
                        int n_multi, const float* dout, float* dtable, float scale, float* scratch,
                        cudaStream_t s) {
    constexpr int R = V >= 8 ? 2 : (V >= 4 ? 4 : 8);
    MM_CUDA_TRY(mm::launch_pdl(embed_bwd_chunk_kernel<V, R, C4>, dim3((n_chunks + 7) / 8), dim3(256), 0, s, perm,
                               chunks, n_chunks, dout, dtable, scratch, scale));
    MM_LAUNCH_CHECK("embed_bwd_chunk_kernel");
    if (n_multi > 0) {
        MM_CUDA_TRY(mm::launch_pdl(embed_bwd_multi_kernel<V, R, C4>, dim3((n_multi + 7) / 8), dim3(256), 0, s,
                                   multi, n_multi, (const float*)scratch, dtable));
        MM_LAUNCH_CHECK("embed_bwd_multi_kernel");
    }
    return 0;
}

// ----------------------------------------------------------------------------
// Cross-entropy over bf16 logits, one CTA per row.  Pass 1: per-thread online
// (max, sum-exp) over 8-wide bf16 vectors, block-combined.  Pass 2 (row is
// L1/L2-resident): dlogits = (softmax - onehot(label)) * grad_scale in bf16.
// label < 0 marks padding: zero loss, zero gradient.
constexpr int kXentThreads = 512;
constexpr int kXentStreamMinVocab = 4096;  // below: the row-per-CTA kernel

__global__ void __launch_bounds__(kXentThreads) xent_kernel(const uint16_t* logits,
                                                            const int32_t* __restrict__ labels,
                                                            uint16_t* dlogits, float* row_loss,
                                                            float* loss_sum, int vocab,
                                                            float grad_scale) {
    pdl_wait_release();
    __shared__ float sm_m[kXentThreads / 32], sm_s[kXentThreads / 32];
    const int64_t row = blockIdx.x;
    const int label = labels[row];
    MM_DCHECK(label < vocab);
    const uint16_t* lr = logits + row * int64_t(vocab);
    uint16_t* dr = dlogits + row * int64_t(vocab);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (label < 0) {
        for (int v = threadIdx.x; v < vocab / 8; v += kXentThreads)
            reinterpret_cast<uint4*>(dr)[v] = make_uint4(0, 0, 0, 0);
        for (int c = (vocab / 8) * 8 + threadIdx.x; c < vocab; c += kXentThreads) dr[c] = 0;
        if (threadIdx.x == 0) row_loss[row] = 0.f;
        return;
    }
    float m = -INFINITY, s = 0.f;
    const int nv = vocab / 8;
    for (int v = threadIdx.x; v < nv; v += kXentThreads) {
        const uint4 w = reinterpret_cast<const uint4*>(lr)[v];
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
        float f[8];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            f[2 * e] = bf2f(ws[e] & 0xffff);
            f[2 * e + 1] = bf2f(ws[e] >> 16);
        }
        float lm = f[0];
#pragma unroll
        for (int e = 1; e < 8; ++e) lm = fmaxf(lm, f[e]);
        const float nm = fmaxf(m, lm);
        float acc = s * __expf(m - nm);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc += __expf(f[e] - nm);
        m = nm;
        s = acc;
    }
    for (int c = nv * 8 + threadIdx.x; c < vocab; c += kXentThreads) {
        const float f = bf2f(lr[c]);
        const float nm = fmaxf(m, f);
        s = s * __expf(m - nm) + __expf(f - nm);
        m = nm;
    }
    // combine (m, s) across the warp, then across warps
    float wm = warp_max(m);
    float ws_ = warp_sum(m == -INFINITY ? 0.f : s * __expf(m - wm));
    if (lane == 0) { sm_m[warp] = wm; sm_s[warp] = ws_; }
    __syncthreads();
    float gm = -INFINITY;
#pragma unroll
    for (int w = 0; w < kXentThreads / 32; ++w) gm = fmaxf(gm, sm_m[w]);
    float gs = 0.f;
#pragma unroll
    for (int w = 0; w < kXentThreads / 32; ++w) gs += sm_s[w] * __expf(sm_m[w] - gm);
    const float lse = gm + __logf(gs);
    const float inv = 1.f / gs;
    if (threadIdx.x == 0) {
        const float l = lse - bf2f(lr[label]);
        row_loss[row] = l;
        if (loss_sum) atomicAdd(loss_sum, l * grad_scale);  // token mean when scale = 1/rows
    }
    __syncthreads();  // every read of the row's label logit precedes in-place writes
    for (int v = threadIdx.x; v < nv; v += kXentThreads) {
        const uint4 w = reinterpret_cast<const uint4*>(lr)[v];
        const uint32_t wsv[4] = {w.x, w.y, w.z, w.w};
        uint32_t o[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int c = v * 8 + 2 * e;
            float p0 = __expf(bf2f(wsv[e] & 0xffff) - gm) * inv;
            float p1 = __expf(bf2f(wsv[e] >> 16) - gm) * inv;
            if (c == label) p0 -= 1.f;
            if (c + 1 == label) p1 -= 1.f;
            o[e] = pack2(p0 * grad_scale, p1 * grad_scale);
        }
        reinterpret_cast<uint4*>(dr)[v] = make_uint4(o[0], o[1], o[2], o[3]);
    }
    for (int c = nv * 8 + threadIdx.x; c < vocab; c += kXentThreads) {
        float pr = __expf(bf2f(lr[c]) - gm) * inv;
        if (c == label) pr -= 1.f;
        dr[c] = f2bf(pr * grad_scale);
    }
}

// Persistent variant (one CTA per SM, vocab <= kXentSmemVocab): each CTA
// walks rows b, b + grid, ...; a 1-D bulk copy (TMA) streams the NEXT row into
// the other half of a double-buffered smem row while the current row is
// reduced and its dlogits written, so HBM reads overlap the math.  The math is
// kept to one MUFU exp per logit (the exps stay in registers between the sum
// and the write pass -- two exps per logit are SFU-bound at ~60 us for a
// 4096 x 32000 batch on B200's 16 MUFU/clk/SM) and a packed bf16x2 max.
constexpr int kXentSmemVocab = 32768;
#ifndef MM_XENT_STREAM_THREADS
#define MM_XENT_STREAM_THREADS 512
#endif
constexpr int kXsThreads = MM_XENT_STREAM_THREADS;
#ifndef MM_XENT_BUFS
#define MM_XENT_BUFS 3
#endif
constexpr int kXentBufs = MM_XENT_BUFS;  // logit rows in flight + the one being reduced

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int NT>
__device__ __forceinline__ float xent_block_reduce(float v, float* sm, bool is_max) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = is_max ? warp_max(v) : warp_sum(v);
    __syncthreads();  // sm free (previous reduction consumed)
    if (lane == 0) sm[warp] = v;
    __syncthreads();
    float r = is_max ? -INFINITY : 0.f;
#pragma unroll
    for (int j = 0; j < NT / 32; ++j) r = is_max ? fmaxf(r, sm[j]) : r + sm[j];
    return r;
}

__global__ void __launch_bounds__(kXsThreads, 1) xent_stream_kernel(const uint16_t* logits,
                                                                      const int32_t* __restrict__ labels,
                                                                      uint16_t* dlogits, float* row_loss,
                                                                      float* loss_sum, int64_t rows,
                                                                      int vocab, float grad_scale) {
    constexpr int VPT = kXentSmemVocab / kXsThreads / 8;  // 8-logit vectors per thread
    constexpr float kL2e = 1.4426950408889634f;
    extern __shared__ __align__(128) uint8_t xsm[];
    __shared__ uint64_t bar[kXentBufs];
    __shared__ float red[kXsThreads / 32];
    uint16_t* const buf0 = reinterpret_cast<uint16_t*>(xsm);
    const uint32_t bytes = static_cast<uint32_t>(vocab) * 2u;
    const int nv = vocab / 8;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kXentBufs; ++i) tc::mbar_init(&bar[i], 1);
        tc::fence_barrier_init();
    }
    // each buffer is kXentSmemVocab wide; the tail past the vocab holds bf16
    // -inf (exp -> 0), so every thread's VPT vectors are unconditional
    for (int c = vocab + threadIdx.x; c < kXentSmemVocab; c += kXsThreads)
        for (int i = 0; i < kXentBufs; ++i) buf0[i * kXentSmemVocab + c] = 0xff80u;
    __syncthreads();
    pdl_wait_release();
    const int64_t first = blockIdx.x, step = gridDim.x;
    if (threadIdx.x == 0) {  // the first kXentBufs - 1 rows in flight
        for (int i = 0; i < kXentBufs - 1 && first + i * step < rows; ++i) {
            tc::mbar_expect_tx(&bar[i], bytes);
            tc::bulk_load_1d(buf0 + i * kXentSmemVocab, logits + (first + i * step) * int64_t(vocab), bytes, &bar[i]);
        }
    }
    int it = 0;
    for (int64_t row = first; row < rows; row += step, ++it) {
        const int b = it % kXentBufs;
        // prefetch kXentBufs - 1 rows ahead into the buffer the previous row
        // used (fully consumed before the trailing __syncthreads of the last
        // iteration)
        const int64_t ahead = row + int64_t(kXentBufs - 1) * step;
        if (threadIdx.x == 0 && ahead < rows) {
            const int nb = (it + kXentBufs - 1) % kXentBufs;
            tc::mbar_expect_tx(&bar[nb], bytes);
            tc::bulk_load_1d(buf0 + nb * kXentSmemVocab, logits + ahead * int64_t(vocab), bytes, &bar[nb]);
        }
        const int label = labels[row];
        MM_DCHECK(label < vocab);
        tc::mbar_wait(&bar[b], static_cast<uint32_t>((it / kXentBufs) & 1));
        const uint16_t* lrow = buf0 + b * kXentSmemVocab;
        const uint4* lr = reinterpret_cast<const uint4*>(lrow);
        uint4* dr = reinterpret_cast<uint4*>(dlogits + row * int64_t(vocab));
        if (label < 0) {
            for (int v = threadIdx.x; v < nv; v += kXsThreads) dr[v] = make_uint4(0, 0, 0, 0);
            if (threadIdx.x == 0) row_loss[row] = 0.f;
            __syncthreads();
            continue;
        }
        // pass 1: row max (packed bf16x2 max)
        __nv_bfloat162 m2 = __floats2bfloat162_rn(-INFINITY, -INFINITY);
#pragma unroll
        for (int i = 0; i < VPT; ++i) {
            const uint4 w = lr[threadIdx.x + i * kXsThreads];
            m2 = __hmax2(m2, __hmax2(__hmax2(*reinterpret_cast<const __nv_bfloat162*>(&w.x),
                                             *reinterpret_cast<const __nv_bfloat162*>(&w.y)),
                                     __hmax2(*reinterpret_cast<const __nv_bfloat162*>(&w.z),
                                             *reinterpret_cast<const __nv_bfloat162*>(&w.w))));
        }
        const float gm = xent_block_reduce<kXsThreads>(fmaxf(__low2float(m2), __high2float(m2)), red, true);
        const float gm2 = gm * kL2e;
        // pass 2: one exp per logit, kept in registers
        float p[VPT][8];
        float sacc = 0.f;
#pragma unroll
        for (int i = 0; i < VPT; ++i) {
            const uint4 w = lr[threadIdx.x + i * kXsThreads];
            const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                p[i][2 * e] = ex2_approx(fmaf(bf2f(ws[e] & 0xffff), kL2e, -gm2));
                p[i][2 * e + 1] = ex2_approx(fmaf(bf2f(ws[e] >> 16), kL2e, -gm2));
                sacc += p[i][2 * e] + p[i][2 * e + 1];
            }
        }
        const float gs = xent_block_reduce<kXsThreads>(sacc, red, false);
        const float sc = grad_scale / gs;
        if (threadIdx.x == 0) {
            const float l = gm + __logf(gs) - bf2f(lrow[label]);
            row_loss[row] = l;
            if (loss_sum) atomicAdd(loss_sum, l * grad_scale);  // token mean when scale = 1/rows
        }
        // pass 3: dlogits = softmax * scale, then the label's -scale
#pragma unroll
        for (int i = 0; i < VPT; ++i) {
            uint32_t o[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                __nv_bfloat162 h = __floats2bfloat162_rn(p[i][2 * e] * sc, p[i][2 * e + 1] * sc);
                o[e] = *reinterpret_cast<uint32_t*>(&h);
            }
            const int v = threadIdx.x + i * kXsThreads;
            if (v < nv) dr[v] = make_uint4(o[0], o[1], o[2], o[3]);
        }
        if (threadIdx.x == (label >> 3) % kXsThreads) {  // the thread that stored the label's vector
            const float pl = ex2_approx(fmaf(bf2f(lrow[label]), kL2e, -gm2));  // == its p, recomputed
            reinterpret_cast<uint16_t*>(dr)[label] = f2bf(pl * sc - grad_scale);
        }
        __syncthreads();  // buffer b fully read before it is refilled
    }
}

// ----------------------------------------------------------------------------
// out[c] += sum_r x[r, c] (bias gradients).  Block = 32 column octets (256
// columns, one 128-bit load per row per thread) x 8 row lanes; the grid has
// enough row slabs to fill every SM; per-block partials are reduced over the
// row lanes in smem and leave with one atomic per column.
__global__ void __launch_bounds__(256) colsum_kernel(const uint16_t* __restrict__ x, float* out,
                                                     int64_t rows, int cols, int64_t slab) {
    pdl_wait_release();
    __shared__ float red[8][256 + 8];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int c8 = blockIdx.x * 32 + tx;
    const bool live = 8 * c8 < cols;
    const int64_t r0 = int64_t(blockIdx.y) * slab;
    const int64_t r1 = min(rows, r0 + slab);
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (live) {
        const uint4* xp = reinterpret_cast<const uint4*>(x);
        const int64_t pitch = cols / 8;
#pragma unroll 2
        for (int64_t r = r0 + ty; r < r1; r += 8) {
            const uint4 w = __ldg(xp + r * pitch + c8);
            const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                acc[2 * e] += bf2f(ws[e] & 0xffff);
                acc[2 * e + 1] += bf2f(ws[e] >> 16);
            }
        }
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) red[ty][tx * 8 + e] = acc[e];
    __syncthreads();
    const int col = blockIdx.x * 256 + threadIdx.x;
    if (col < cols) {
        float s = 0.f;
#pragma unroll
        for (int y = 0; y < 8; ++y) s += red[y][threadIdx.x];
        atomicAdd(out + col, s);
    }
}

__global__ void cast_kernel(const float* __restrict__ x, uint16_t* __restrict__ y, int64_t n4) {
    pdl_wait_release();
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n4;
         i += int64_t(gridDim.x) * blockDim.x) {
        const float4 v = reinterpret_cast<const float4*>(x)[i];
        uint2 o;
        o.x = pack2(v.x, v.y);
        o.y = pack2(v.z, v.w);
        reinterpret_cast<uint2*>(y)[i] = o;
    }
}

__global__ void widen_kernel(const uint16_t* __restrict__ x, float* __restrict__ y, int64_t n4) {
    pdl_wait_release();
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n4;
         i += int64_t(gridDim.x) * blockDim.x) {
        const uint2 w = reinterpret_cast<const uint2*>(x)[i];
        reinterpret_cast<float4*>(y)[i] = make_float4(bf2f(w.x & 0xffff), bf2f(w.x >> 16),
                                                      bf2f(w.y & 0xffff), bf2f(w.y >> 16));
    }
}

}  // namespace

extern "C" int mm_layernorm_fwd(const float* x, const float* gamma, const float* beta, uint16_t* y,
                                float* mean, float* rstd, int64_t rows, int cols, float eps,
                                void* stream) {
    MM_CHECK_ARG(x && gamma && beta && y && mean && rstd, "NULL argument");
    if (rows == 0) return 0;
    const unsigned grid = static_cast<unsigned>((rows + 8 * kLnRows - 1) / (8 * kLnRows));
    auto s = mm::as_stream(stream);
    static const bool v1 = std::getenv("MM_LN_V1") != nullptr;  // A/B: the previous kernels
    if (!v1 && (cols == 512 || cols == 1024)) {
        const unsigned g2 = static_cast<unsigned>((rows + MM_LN_FWD_WARPS - 1) / MM_LN_FWD_WARPS);
        const dim3 blk(32 * MM_LN_FWD_WARPS);
        if (cols == 512)
            MM_CUDA_TRY(mm::launch_pdl(ln_fwd_v2_kernel<512>, dim3(g2), blk, 0, s, x, gamma, beta, y, mean, rstd, rows, eps));
        else
            MM_CUDA_TRY(mm::launch_pdl(ln_fwd_v2_kernel<1024>, dim3(g2), blk, 0, s, x, gamma, beta, y, mean, rstd, rows, eps));
        MM_LAUNCH_CHECK("ln_fwd_v2_kernel");
        return 0;
    }
    if (cols == 512)
        MM_CUDA_TRY(mm::launch_pdl(ln_fwd_kernel<512>, dim3(grid), dim3(256), 0, s, x, gamma, beta, y, mean, rstd, rows, eps));
    else if (cols == 1024)
        MM_CUDA_TRY(mm::launch_pdl(ln_fwd_kernel<1024>, dim3(grid), dim3(256), 0, s, x, gamma, beta, y, mean, rstd, rows, eps));
    else if (cols == 64)
        MM_CUDA_TRY(mm::launch_pdl(ln_fwd_kernel<64>, dim3(grid), dim3(256), 0, s, x, gamma, beta, y, mean, rstd, rows, eps));
    else if (cols == 128)
        MM_CUDA_TRY(mm::launch_pdl(ln_fwd_kernel<128>, dim3(grid), dim3(256), 0, s, x, gamma, beta, y, mean, rstd, rows, eps));
    else if (cols == 256)
        MM_CUDA_TRY(mm::launch_pdl(ln_fwd_kernel<256>, dim3(grid), dim3(256), 0, s, x, gamma, beta, y, mean, rstd, rows, eps));
    else {
        mm::set_error("layernorm: cols=%d unsupported (64/128/256/512/1024)", cols);
        return mm::kUnsupported;
    }
    MM_LAUNCH_CHECK("ln_fwd_kernel");
    return 0;
}

extern "C" int mm_layernorm_bwd(const float* dy, const float* x, const float* gamma,
                                const float* mean, const float* rstd, float* dx, uint16_t* dx_bf16,
                                float* dgamma, float* dbeta, int64_t rows, int cols, void* stream) {
    MM_CHECK_ARG(dy && x && gamma && mean && rstd && dx && dgamma && dbeta, "NULL argument");
    if (rows == 0) return 0;
    auto s = mm::as_stream(stream);
    static const bool old_kernel = std::getenv("MM_LN_BWD_BATCHED") != nullptr;  // A/B diagnostics
    static const bool v1 = std::getenv("MM_LN_V1") != nullptr;
    // v2 (row per warp, one wave): 8.5 vs 5.9 us back to back at 4096 x 512 --
    // the persistent row kernel below wins; kept for A/B (MM_LN_BWD_V2=1)
    static const bool bwd_v2 = std::getenv("MM_LN_BWD_V2") != nullptr;
    if (bwd_v2 && !v1 && !old_kernel && cols == 512) {  // (d = 1024 spills at 64 registers)
        const unsigned g2 = static_cast<unsigned>((rows + 7) / 8);
        MM_CUDA_TRY(mm::launch_pdl(ln_bwd_v2_kernel<512>, dim3(g2), dim3(256), 0, s, dy, x, gamma, mean, rstd, dx, dx_bf16, dgamma, dbeta, rows));
        MM_LAUNCH_CHECK("ln_bwd_v2_kernel");
        return 0;
    }
    if (cols == 512 && !old_kernel) {
        // one row per warp, 2 CTAs/SM (3 CTAs/SM = 85 registers spills: 9.3 us;
        // this 5.9 us vs 6.7 us for the batched kernel, graph back to back)
        const int per_sm = 2;
        const size_t smem = size_t(2) * 8 * cols * sizeof(float);
        const unsigned g1 = static_cast<unsigned>(
            std::min<int64_t>((rows + 7) / 8, int64_t(per_sm) * mm::num_sms()));
        static bool attr = false;
        if (!attr) {
            MM_CUDA_TRY(cudaFuncSetAttribute(ln_bwd_row_kernel<512, 2>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            attr = true;
        }
        MM_CUDA_TRY(mm::launch_pdl(ln_bwd_row_kernel<512, 2>, dim3(g1), dim3(256), smem, s, dy, x, gamma,
                                   mean, rstd, dx, dx_bf16, dgamma, dbeta, rows));
        MM_LAUNCH_CHECK("ln_bwd_row_kernel");
        return 0;
    }
    const unsigned grid = static_cast<unsigned>(
        std::min<int64_t>((rows + 8 * kLnRows - 1) / (8 * kLnRows), 4 * mm::num_sms()));
    if (cols == 512)
        MM_CUDA_TRY(mm::launch_pdl(ln_bwd_kernel<512>, dim3(grid), dim3(256), 0, s, dy, x, gamma, mean, rstd, dx, dx_bf16, dgamma, dbeta, rows));
    else if (cols == 1024)
        MM_CUDA_TRY(mm::launch_pdl(ln_bwd_kernel<1024>, dim3(grid), dim3(256), 0, s, dy, x, gamma, mean, rstd, dx, dx_bf16, dgamma, dbeta, rows));
    else if (cols == 64)
        MM_CUDA_TRY(mm::launch_pdl(ln_bwd_kernel<64>, dim3(grid), dim3(256), 0, s, dy, x, gamma, mean, rstd, dx, dx_bf16, dgamma, dbeta, rows));
    else if (cols == 128)
        MM_CUDA_TRY(mm::launch_pdl(ln_bwd_kernel<128>, dim3(grid), dim3(256), 0, s, dy, x, gamma, mean, rstd, dx, dx_bf16, dgamma, dbeta, rows));
    else if (cols == 256)
        MM_CUDA_TRY(mm::launch_pdl(ln_bwd_kernel<256>, dim3(grid), dim3(256), 0, s, dy, x, gamma, mean, rstd, dx, dx_bf16, dgamma, dbeta, rows));
    else {
        mm::set_error("layernorm: cols=%d unsupported (64/128/256/512/1024)", cols);
        return mm::kUnsupported;
    }
    MM_LAUNCH_CHECK("ln_bwd_kernel");
    return 0;
}

extern "C" int mm_embed_fwd(const int32_t* ids, const int32_t* pos, const uint16_t* table,
                            float* out, int64_t rows, int cols, float scale, void* stream) {
    MM_CHECK_ARG(ids && pos && table && out, "NULL argument");
    MM_CHECK_ARG(cols % 4 == 0, "cols must be a multiple of 4");
    if (rows == 0) return 0;
    MM_CUDA_TRY(mm::launch_pdl(embed_fwd_kernel, dim3(static_cast<unsigned>((rows + 7) / 8)), dim3(256), 0, mm::as_stream(stream), ids, pos, table, out, rows, cols, scale));
    MM_LAUNCH_CHECK("embed_fwd_kernel");
    return 0;
}

extern "C" int mm_embed_bwd(const int32_t* ids, const float* dout, float* dtable, int64_t rows,
                            int cols, float scale, void* stream) {
    MM_CHECK_ARG(ids && dout && dtable, "NULL argument");
    MM_CHECK_ARG(cols % 4 == 0, "cols must be a multiple of 4");
    if (rows == 0) return 0;
    MM_CUDA_TRY(mm::launch_pdl(embed_bwd_kernel, dim3(static_cast<unsigned>((rows + 7) / 8)), dim3(256), 0, mm::as_stream(stream), ids, dout, dtable, rows, cols, scale));
    MM_LAUNCH_CHECK("embed_bwd_kernel");
    return 0;
}

extern "C" int mm_embed_bwd_sorted(const int32_t* table, int64_t rows, int n_chunks, int n_multi,
                                   const float* dout, float* dtable, int cols, float scale,
                                   float* scratch, void* stream) {
    MM_CHECK_ARG(table && dout && dtable && (n_multi == 0 || scratch), "NULL argument");
    MM_CHECK_ARG(cols == 64 || cols == 128 || cols == 256 || cols == 512 || cols == 1024,
                 "cols %d: 64, 128, 256, 512 or 1024", cols);
    if (rows == 0 || n_chunks == 0) return 0;
    const int32_t* perm = table;
    const int32_t* chunks = table + rows;
    const int32_t* multi = chunks + int64_t(3) * n_chunks;
    auto s = mm::as_stream(stream);
    switch (cols) {
        case 64: return embed_sorted_launch<1, 16>(perm, chunks, n_chunks, multi, n_multi, dout, dtable, scale, scratch, s);
        case 128: return embed_sorted_launch<1>(perm, chunks, n_chunks, multi, n_multi, dout, dtable, scale, scratch, s);
        case 256: return embed_sorted_launch<2>(perm, chunks, n_chunks, multi, n_multi, dout, dtable, scale, scratch, s);
        case 512: return embed_sorted_launch<4>(perm, chunks, n_chunks, multi, n_multi, dout, dtable, scale, scratch, s);
        default: return embed_sorted_launch<8>(perm, chunks, n_chunks, multi, n_multi, dout, dtable, scale, scratch, s);
    }
}

extern "C" int mm_xent_fwd_bwd(const uint16_t* logits, const int32_t* labels, uint16_t* dlogits,
                               float* row_loss, float* loss_sum, int64_t rows, int vocab,
                               float grad_scale, void* stream) {
    MM_CHECK_ARG(logits && labels && dlogits && row_loss, "NULL argument");
    MM_CHECK_ARG(vocab % 8 == 0, "vocab must be a multiple of 8");
    if (rows == 0) return 0;
    static const bool force_rowwise = std::getenv("MM_XENT_ROWWISE") != nullptr;  // diagnostics
    // short rows (config 1's V1000): one CTA per row -- the streamed kernel's
    // per-row TMA round trip dominates there (365 us for 16K rows x 1000 in
    // one config-1 step, profiles/r02_launch_summary_c1.txt)
    if (vocab >= kXentStreamMinVocab && vocab <= kXentSmemVocab && !force_rowwise) {
        const size_t smem = size_t(kXentBufs) * kXentSmemVocab * 2;
        MM_CUDA_TRY(cudaFuncSetAttribute(xent_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem)));
        const unsigned grid = static_cast<unsigned>(std::min<int64_t>(rows, mm::num_sms()));
        MM_CUDA_TRY(mm::launch_pdl(xent_stream_kernel, dim3(grid), dim3(kXsThreads), smem,
                                   mm::as_stream(stream), logits, labels, dlogits, row_loss, loss_sum,
                                   rows, vocab, grad_scale));
    } else {
        MM_CUDA_TRY(mm::launch_pdl(xent_kernel, dim3(static_cast<unsigned>(rows)), dim3(kXentThreads), 0, mm::as_stream(stream), logits, labels, dlogits, row_loss, loss_sum, vocab, grad_scale));
    }
    MM_LAUNCH_CHECK("xent_kernel");
    return 0;
}

extern "C" int mm_colsum_bf16(const uint16_t* x, float* out, int64_t rows, int cols,
                              void* stream) {
    MM_CHECK_ARG(x && out && cols % 8 == 0, "cols must be a multiple of 8");
    if (rows == 0) return 0;
    const int64_t gx = (cols + 255) / 256;
    int64_t slabs = std::max<int64_t>(1, std::min<int64_t>((rows + 15) / 16, (2 * mm::num_sms() + gx - 1) / gx));
    const int64_t slab = (rows + slabs - 1) / slabs;
    slabs = (rows + slab - 1) / slab;
    dim3 grid(static_cast<unsigned>(gx), static_cast<unsigned>(slabs));
    MM_CUDA_TRY(mm::launch_pdl(colsum_kernel, dim3(grid), dim3(256), 0, mm::as_stream(stream), x, out, rows, cols, slab));
    MM_LAUNCH_CHECK("colsum_kernel");
    return 0;
}

extern "C" int mm_cast_bf16_f32(const uint16_t* x, float* y, int64_t n, void* stream) {
    MM_CHECK_ARG(x && y && n % 4 == 0, "n must be a multiple of 4");
    if (n == 0) return 0;
    const int64_t n4 = n / 4;
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>((n4 + 255) / 256, 8 * mm::num_sms()));
    MM_CUDA_TRY(mm::launch_pdl(widen_kernel, dim3(grid), dim3(256), 0, mm::as_stream(stream), x, y, n4));
    MM_LAUNCH_CHECK("widen_kernel");
    return 0;
}

extern "C" int mm_cast_f32_bf16(const float* x, uint16_t* y, int64_t n, void* stream) {
    MM_CHECK_ARG(x && y && n % 4 == 0, "n must be a multiple of 4");
    if (n == 0) return 0;
    const int64_t n4 = n / 4;
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>((n4 + 255) / 256, 8 * mm::num_sms()));
    MM_CUDA_TRY(mm::launch_pdl(cast_kernel, dim3(grid), dim3(256), 0, mm::as_stream(stream), x, y, n4));
    MM_LAUNCH_CHECK("cast_kernel");
    return 0;
}
