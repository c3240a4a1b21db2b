// K4: bf16 GEMM on 5th-generation tensor cores (tcgen05), sm_100a.
//
//   D[M,N] = A[M,K] * B[N,K]^T      (fp32 accumulate in TMEM)
//
// One persistent CTA per SM walks a static list of work units (output tile x
// K split).  Warp roles (192 threads):
//   warp 0      TMA producer: A/B tiles -> 128B-swizzled smem ring (mbarrier
//               complete_tx), one elected lane
//   warp 1      MMA issuer: one elected lane issues tcgen05.mma (M=128, N=BN,
//               K=16) from smem descriptors into a double-buffered TMEM
//               accumulator, tcgen05.commit releases smem stages / signals the
//               epilogue; this warp also owns the TMEM allocation
//   warps 2..5  epilogue: tcgen05.ld (32 lanes x 32 columns per access),
//               fused bias (warp-shuffle broadcast) / ReLU / ReLU-backward
//               mask / residual add, staged through a per-warp swizzled smem
//               box and written by TMA (cp.async.bulk.tensor store; fp32
//               accumulation -- wgrad into the grad bucket, split-K partials --
//               uses the TMA reduce-add, so no read-modify-write or atomics)
// Operands may be K-major or MN-major (transpose bits of the instruction
// descriptor), which is what lets forward, dgrad and wgrad all run without a
// transpose pass:
//   forward  Y  = X  W^T : A = X  (K-major), B = W (K-major)
//   dgrad    dX = dY W   : A = dY (K-major), B = W (MN-major)
//   wgrad    dW = dY^T X : A = dY (MN-major), B = X (MN-major), fp32 accumulate
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "mm_common.h"
#include "tc_ptx.cuh"

namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // one 128-byte swizzle row of bf16
constexpr int UMMA_K = 16;
constexpr int kEpiWarp0 = 2;
#ifndef MM_GEMM_EPI_WARPS
#define MM_GEMM_EPI_WARPS 8
#endif
#ifndef MM_GEMM_EPI_BUFS
// one staging box per epilogue warp: the 32 KB saved buy every tile shape one
// more mainloop stage (BN = 128: 6 instead of 5), which outweighs waiting for
// the previous box's TMA store to be read (config 3: 3.53 vs 3.61 ms/step)
#define MM_GEMM_EPI_BUFS 1
#endif
#ifndef MM_GEMM_MAX_STAGES
#define MM_GEMM_MAX_STAGES 8
#endif
// epilogue warps: 4 per "column slice" (one per TMEM lane quarter); with 8,
// two slices each take half of the tile's columns
constexpr int kEpiWarps = MM_GEMM_EPI_WARPS;
constexpr int kSlices = kEpiWarps / 4;
#ifndef MM_GEMM_WIDE_LAST
#define MM_GEMM_WIDE_LAST 1
#endif
#ifndef MM_GEMM_RESID_TMEM
// residual tile of single-CTA 128-wide tiles parked in TMEM columns 256..383
#define MM_GEMM_RESID_TMEM 1
#endif
#ifndef MM_GEMM_BN64
// 64-wide single-CTA tiles (diagnostics build: MM_GEMM_OVERRIDE "...=1:64"):
// twice the tiles of a narrow GEMM, so a CTA's first epilogue overlaps its
// second tile's mainloop
#define MM_GEMM_BN64 0
#endif
#ifndef MM_GEMM_EPI_BUFS256P
// CTA-pair 256-wide tiles (generator, grouped weight gradients)
#define MM_GEMM_EPI_BUFS256P MM_GEMM_EPI_BUFS
#endif
#ifndef MM_GEMM_EPI_BUFS128
// single-CTA 128-wide tiles (the small forward / dgrad GEMMs): staging boxes
// per epilogue warp.  2 measured slower in the step (3.579 vs 3.525 ms: one
// mainloop stage fewer), so it follows MM_GEMM_EPI_BUFS
#define MM_GEMM_EPI_BUFS128 MM_GEMM_EPI_BUFS
#endif
constexpr int kBiasWarp = kEpiWarp0 + kEpiWarps;  // first of the bias-gradient warps
// bias-gradient warps: second consumer of every smem stage; each sums 16 of
// the stage's 64 K-rows (one warp summing all 64 was slower than a 256-wide
// MMA k-block and gated the pipeline: +46 % on the generator wgrad)
constexpr int kBiasWarps = 4;
constexpr int kThreads = (kBiasWarp + kBiasWarps) * 32;
constexpr int kMaxProbs = 48;  // problems per grouped launch (kernel parameter space: ~21 KB of 32 KB)

constexpr int kEpiBufBytes = 32 * 128;                    // 32 rows x 128 B box

constexpr int kSmemLimit = 232448;

// CG = CTAs per MMA: 1, or 2 for a CTA pair (cta_group::2) computing a
// (2*BM) x BN tile -- each CTA holds its BM rows of A and BN/2 rows of B, so
// per-SM shared-memory traffic per MMA drops by a quarter (BN=128) to a half.
template <int BN, int CG, int CN = 1, int RT = 0>
struct Cfg {
    static constexpr int kEpiBufs = (BN == 128 && CG == 1 && CN == 1) ? MM_GEMM_EPI_BUFS128
                                    : (BN == 256 && CG == 2) ? MM_GEMM_EPI_BUFS256P
                                                             : MM_GEMM_EPI_BUFS;
    static constexpr int kEpiSmem = kEpiWarps * kEpiBufs * kEpiBufBytes;
    static constexpr int kBRows = BN / CG;             // B rows (N) staged by one CTA
    static constexpr int kABytes = BM * BK * 2;
    static constexpr int kBBytes = kBRows * BK * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kTxBytes = kStageBytes * CG;  // bytes counted on the MMA CTA's barrier
    static constexpr int kBarBytes = 512;
    // fused LayerNorm (cluster of CN CTAs along N): per-row partials of the two
    // column halves [2][BM] and the CTA's exchanged row sums [2 parities][BM]
    static constexpr int kLnBytes = CN > 1 ? 4 * BM * 8 : 0;  // float2 [2][BM] x 2
    static constexpr int kStagesFit = (kSmemLimit - kEpiSmem - 1024 - kBarBytes - kLnBytes) / kStageBytes;
    static constexpr int kStages = kStagesFit > MM_GEMM_MAX_STAGES ? MM_GEMM_MAX_STAGES : kStagesFit;
    // 2 accumulators (power of 2); a single-CTA 128-wide tile also parks the
    // tile's fp32 residual in columns 256..383 (loaded while the MMAs run)
    // RT = 1: the residual-epilogue instantiation (single-CTA 128-wide tiles
    // of one MM_EPI_F32_RESID problem) parks the tile's fp32 residual in TMEM
    // columns 256..383; every other launch allocates only the 256 columns of
    // its two accumulators (a 512-column allocation made the FFN-up / QKV
    // launches 0.5-2 us slower in the config-3 step, r02al)
    static constexpr bool kResidTmem = MM_GEMM_RESID_TMEM && RT && BN <= 128 && CG == 1 && CN == 1;
    static constexpr int kTmemCols = kResidTmem || 2 * BN > 256 ? 512 : 256;
    static constexpr uint32_t kResidCol = 2 * BN;
    static constexpr int kSmem = kStages * kStageBytes + kEpiSmem + 1024 + kBarBytes + kLnBytes;
    static_assert(kSmem <= kSmemLimit, "smem budget");
    static_assert(CG == 1 || kBRows % 64 == 0, "pair tiles need 64-aligned B halves");
    static_assert((3 * kStages + 6) * 8 + 4 <= kBarBytes, "barrier area");
};

// One GEMM problem of a launch: its three tensor maps (A, B, D) and its slice
// [unit_begin, unit_begin + tiles_m * tiles_n * splits) of the launch's unit list.
struct alignas(64) Prob {
    CUtensorMap ta, tb, td;
    int64_t m, n, k;
    int64_t ldd;
    void* d;
    const float* bias;
    const float* resid;
    const __nv_bfloat16* aux;
    uint32_t* relu_mask;  // [m, mask_ld] 1-bit ReLU mask (written by RELU, read by DRELU)
    int64_t mask_ld;
    float* dbias;
    int epilogue;
    int tiles_m, tiles_n, splits, kb_per_split, num_kb;
    int group_m;  // unit order: M-tiles walked in groups of group_m (L2 reuse of A)
    int resid_early;  // residual not written by the preceding kernel (see mm_gemm_args)
    int unit_begin;
};

// A launch: NP = 1 for a plain GEMM, kMaxProbs for a grouped launch (all
// problems share the operand majorness and the tile width; units of all
// problems are dealt to the persistent CTAs from one list).
// the fused LayerNorm of a MM_EPI_F32_RESID_LN launch (single problem)
struct alignas(64) LnParams {
    CUtensorMap th;  // LayerNorm output (bf16 [M, N])
    const float* gamma;
    const float* beta;
    float* mean;
    float* rstd;
    float eps;
};
template <int NP>
struct Group {
    LnParams ln;
    Prob prob[NP];
    unsigned long long* trace;  // optional per-CTA phase timestamps (diagnostics)
    // optional launch span (mm_gemm_timing): %globaltimer min over CTAs after
    // griddepcontrol.wait -> *span_lo, max over CTAs at exit -> *span_hi
    unsigned long long* span_lo;
    unsigned long long* span_hi;
    int n_probs;
    int units;
    int b_prefetch;
    int any_dbias;  // some problem fuses bias-gradient column sums (bias warp active)
};
// diagnostics build (tools/build_variant.py -DMM_GEMM_DEBUG=bits): bit 0 skip
// MMAs, bit 1 skip epilogue stores, bit 2 skip loads, bit 3 LayerNorm without the
// cluster exchange, bit 4 no LayerNorm epilogue at all
#ifndef MM_GEMM_DEBUG
#define MM_GEMM_DEBUG 0
#endif

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// trace slots per CTA: 0 entry, 1 setup done, 2 first stage full (MMA warp),
// 3 last commit issued, 4 first tfull seen (epilogue warp 2), 5 epilogue
// done (warp 2), 6 stores drained (warp 2), 7 exit
// per-k-block pipeline stamps (clock64) of CTAs 0 and 1 after the 8 x 148 phase slots:
// [cta*256 + i] producer passed the empty wait for its i-th stage fill,
// [cta*256 + 128 + i] MMA warp passed the full wait for its i-th stage
#ifdef MM_GEMM_KB_TRACE
#define MM_KB_TRACE(off, i)                                                              \
    do {                                                                                 \
        if (g.trace && blockIdx.x < 2 && (i) < 128)                                      \
            g.trace[8 * 148 + blockIdx.x * 256 + (off) + (i)] = clock64();               \
    } while (0)
#else
#define MM_KB_TRACE(off, i) \
    do {                    \
    } while (0)
#endif
#define MM_TRACE(slot)                                                                   \
    do {                                                                                 \
        if (g.trace) g.trace[blockIdx.x * 8 + (slot)] = gtime();                         \
    } while (0)

__device__ __forceinline__ float bf16_to_f(uint16_t h) {
    return __uint_as_float(static_cast<uint32_t>(h) << 16);
}

__device__ __forceinline__ uint32_t pack2(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}

// Epilogue math for one row (this thread) x 32 columns held in registers.
// ep: the problem's epilogue -- a compile-time constant in the specialised
// instantiations (EK >= 0), so only its path is compiled
__device__ __forceinline__ bool has_bias(const Prob& p, int ep) {
    return p.bias && (ep == MM_EPI_BF16 || ep == MM_EPI_BF16_RELU || ep == MM_EPI_F32 ||
                      ep == MM_EPI_F32_RESID || ep == MM_EPI_F32_RESID_LN);
}

// bv: this lane's bias value for column col0 + lane (preloaded per tile);
// resid_done: the residual is added by the caller (parked in TMEM)
__device__ __forceinline__ void epilogue_math(const Prob& p, int ep, int64_t row, int64_t col0,
                                              float (&acc)[32], float bv, bool resid_done = false) {
    if (has_bias(p, ep)) {
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j] += __shfl_sync(0xffffffffu, bv, j);
    }
    if (ep == MM_EPI_BF16_RELU) {
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j] = fmaxf(acc[j], 0.f);
    }
    if (row >= p.m) return;
    const bool full = col0 + 32 <= p.n;
    if (ep == MM_EPI_BF16_DRELU) {
        const uint16_t* aux = reinterpret_cast<const uint16_t*>(p.aux) + row * p.ldd + col0;
        if (p.relu_mask) {  // one word per row and 32 columns
            const uint32_t bits = p.relu_mask[row * p.mask_ld + (col0 >> 5)];
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (!((bits >> j) & 1u)) acc[j] = 0.f;
        } else if (full) {
            const uint4* a4 = reinterpret_cast<const uint4*>(aux);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint4 w = __ldg(a4 + q);
                const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int j = q * 8 + e * 2;
                    if (bf16_to_f(ws[e] & 0xffff) <= 0.f) acc[j] = 0.f;
                    if (bf16_to_f(ws[e] >> 16) <= 0.f) acc[j + 1] = 0.f;
                }
            }
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (col0 + j < p.n && bf16_to_f(aux[j]) <= 0.f) acc[j] = 0.f;
        }
    }
    if ((ep == MM_EPI_F32_RESID && !resid_done) || ep == MM_EPI_F32_RESID_LN) {
        const float* res = p.resid + row * p.ldd + col0;
        if (full) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                float4 r = *reinterpret_cast<const float4*>(res + q * 4);
                acc[q * 4 + 0] += r.x; acc[q * 4 + 1] += r.y;
                acc[q * 4 + 2] += r.z; acc[q * 4 + 3] += r.w;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (col0 + j < p.n) acc[j] += res[j];
        }
    }
}

// Write this thread's 32 values as row `r` of a 32-row staging box laid out
// in the tensor map's swizzle (bf16: 64 B rows, SWIZZLE_64B; fp32: 128 B
// rows, SWIZZLE_128B).  A warp's 16-byte stores then spread over all banks.
__device__ __forceinline__ void stage_row(uint8_t* buf, int r, const float (&acc)[32], bool bf16) {
    if (bf16) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint4 w;
            w.x = pack2(acc[q * 8 + 0], acc[q * 8 + 1]);
            w.y = pack2(acc[q * 8 + 2], acc[q * 8 + 3]);
            w.z = pack2(acc[q * 8 + 4], acc[q * 8 + 5]);
            w.w = pack2(acc[q * 8 + 6], acc[q * 8 + 7]);
            const int phys = q ^ ((r >> 1) & 3);
            *reinterpret_cast<uint4*>(buf + r * 64 + phys * 16) = w;
        }
    } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int phys = q ^ (r & 7);
            *reinterpret_cast<float4*>(buf + r * 128 + phys * 16) =
                make_float4(acc[q * 4], acc[q * 4 + 1], acc[q * 4 + 2], acc[q * 4 + 3]);
        }
    }
}

// Work unit: (problem, M-tile, N-tile, K-split).  Consecutive units walk M
// first, so CTAs running at the same time share the B tile in L2.
struct Unit {
    int pi, tm, tn, kb0, kb1;
};
// CN > 1 (fused LayerNorm): a unit is a 128-row block, the CN CTAs of a
// cluster take its N-tiles (cluster rank = N-tile), full K
template <int NP>
__device__ __forceinline__ Unit decode_cluster(const Group<NP>& g, int u, int crank) {
    Unit w;
    w.pi = 0;
    w.tm = u;
    w.tn = crank;
    w.kb0 = 0;
    w.kb1 = g.prob[0].num_kb;
    return w;
}
template <int NP>
__device__ __forceinline__ Unit decode(const Group<NP>& g, int u) {
    int pi = 0;
    if constexpr (NP > 1) {
#pragma unroll 1
        for (int j = 1; j < g.n_probs; ++j)
            if (u >= g.prob[j].unit_begin) pi = j;
    }
    const Prob& P = g.prob[pi];
    const int v = u - P.unit_begin;
    const int tp = v / P.splits, split = v - tp * P.splits;
    Unit w;
    w.pi = pi;
    if (P.group_m >= P.tiles_m) {  // A fits the L2 budget: M fastest over every M-tile
        w.tm = tp % P.tiles_m;
        w.tn = tp / P.tiles_m;
    } else {  // groups of group_m M-tiles, N-tiles within a group, M fastest inside
        const int per = P.group_m * P.tiles_n;
        const int grp = tp / per;
        const int first = grp * P.group_m;
        const int gm = min(P.group_m, P.tiles_m - first);
        const int r = tp - grp * per;
        w.tm = first + r % gm;
        w.tn = r / gm;
    }
    w.kb0 = split * P.kb_per_split;
    w.kb1 = min(P.num_kb, w.kb0 + P.kb_per_split);
    MM_DCHECK(v >= 0 && w.tm < P.tiles_m && w.tn < P.tiles_n && w.kb0 < w.kb1);
    return w;
}

// MC = 2 (CTA pairs only): a cluster of two pairs on adjacent N-tiles of the
// same 256-row block; each CTA fetches half of its 128 A rows and multicasts
// it to the CTA at the same pair position in the other pair, so every SM
// requests 3/4 of the operand bytes per k-block (cuBLAS's 2x2 / 2cta shape).
// EK >= 0: an instantiation for one epilogue (the single-problem launches of
// the step), whose code is a fraction of the generic kernel's -- a launch
// after another GEMM instantiation pays less instruction-fetch warm-up
template <int BN, int A_MN, int B_MN, int NP, int CG, int CN = 1, int RT = 0, int MC = 1, int EK = -1>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tcgen05_kernel(const __grid_constant__ Group<NP> g) {
    using C = Cfg<BN, CG, CN, RT>;
    static_assert(CN == 1 || (CG == 1 && NP == 1), "LayerNorm clusters: single CTAs, one problem");
    static_assert(MC == 1 || (CG == 2 && CN == 1), "A multicast: CTA pairs");
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint8_t* smem_a = smem;
    uint8_t* smem_b = smem + C::kStages * C::kABytes;
    uint8_t* smem_epi = smem + C::kStages * C::kStageBytes;  // 1024-aligned
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem_epi + C::kEpiSmem);
    uint64_t* empty_bar = full_bar + C::kStages;
    uint64_t* bias_bar = empty_bar + C::kStages;  // pair: "stage consumed by the MMA" for the bias warp
    uint64_t* tfull_bar = bias_bar + C::kStages;
    uint64_t* tempty_bar = tfull_bar + 2;
    uint64_t* xch_bar = tempty_bar + 2;  // CN > 1: row-sum exchange, one per parity
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xch_bar + 2);
    float* ln_part = reinterpret_cast<float*>(smem_epi + C::kEpiSmem + C::kBarBytes);  // [2][BM]
    float* ln_xch = ln_part + 4 * BM;                                                // float2 [2][BM]

    // warp index through a shuffle: ptxas then knows it is warp-uniform, so
    // the role branches below are uniform and their loop state (stage, phase,
    // descriptors) lives in uniform registers next to the tcgen05 operands
    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
    const int lane = threadIdx.x & 31;
    // pair rank: 0 = leader (issues the MMAs, owns the stage-full barriers);
    // MC = 2: pair pp of the cluster (its leader is cluster rank 2 pp)
    const uint32_t crank_all = CG == 2 ? tc::cluster_ctarank() : 0u;
    const uint32_t rank = crank_all & 1u;
    const uint32_t pp = MC == 2 ? (crank_all >> 1) : 0u;
    const uint32_t lead = 2u * pp;
    // empty-barrier commits: the pair (MC = 1) or both pairs, whose smem our
    // multicast A halves also fill (MC = 2); accumulator commits: the pair
    const uint16_t empty_mask = MC == 2 ? 0xF : 0x3;
    const uint16_t pair_mask = static_cast<uint16_t>(0x3u << lead);
    const int crank = CN > 1 ? static_cast<int>(tc::cluster_ctarank()) : 0;  // N-tile of a LN cluster
    auto unit_at = [&](int u) -> Unit {
        if constexpr (CN > 1) return decode_cluster(g, u, crank);
        else return decode(g, u);
    };
    // bias gradients need an MN-major A (check_args): compiled out otherwise
    const bool dbias_any = A_MN && g.any_dbias != 0;
    if (threadIdx.x == 0) MM_TRACE(0);

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < g.n_probs; ++i) {
            tc::tma_prefetch(&g.prob[i].ta);
            tc::tma_prefetch(&g.prob[i].tb);
            tc::tma_prefetch(&g.prob[i].td);
        }
    }
    if (warp == 1 && lane == 0) {
        for (int s = 0; s < C::kStages; ++s) {
            tc::mbar_init(&full_bar[s], 1);
            // MMA commit (+ bias warps); MC = 2: both pairs' MMA commits
            tc::mbar_init(&empty_bar[s], MC == 2 ? 2 : dbias_any ? 1 + kBiasWarps : 1);
            tc::mbar_init(&bias_bar[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            tc::mbar_init(&tfull_bar[a], 1);
            tc::mbar_init(&tempty_bar[a], CG * kEpiWarps);  // one arrive per epilogue warp of the pair
            tc::mbar_init(&xch_bar[a], CN);                 // one arrive per CTA of the LN cluster
        }
        tc::fence_barrier_init();
    }
    if (warp == 1) {
        if constexpr (CG == 2) tc::tmem_alloc_pair(tmem_slot, C::kTmemCols);
        else tc::tmem_alloc(tmem_slot, C::kTmemCols);
    }
    tc::tc_fence_before();
    if constexpr (CG == 2 || CN > 1) tc::cluster_sync();  // peer barriers initialised before any remote signal
    else __syncthreads();
    tc::tc_fence_after();
    // units are dealt per pair (CG = 2) or per LayerNorm cluster (CN > 1)
    const int cid = blockIdx.x / (CG * CN * MC), ncta = gridDim.x / (CG * CN * MC);
    const uint32_t tmem_base = *tmem_slot;
    if (tmem_base != 0) __trap();  // the MMA issuer addresses TMEM by column offset
    if (threadIdx.x == 0) MM_TRACE(1);
    // griddepcontrol.wait: roles that read or write global memory wait for the
    // previous kernel; everything above (barrier init, TMEM allocation,
    // descriptor prefetch) and the B prefetch below overlap its tail

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            // stage completion is counted on the leader's full barrier
            const uint32_t full_leader = CG == 2 ? tc::mapa_u32(tc::smem_u32(full_bar), lead) : 0u;
            auto load = [&](uint8_t* dst, const CUtensorMap* map, int stage, int c0, int c1) {
                if constexpr (CG == 2) tc::tma_load_2d_pair(dst, map, full_leader + stage * 8, c0, c1);
                else tc::tma_load_2d(dst, map, &full_bar[stage], c0, c1);
            };
            // MC = 2: this CTA's 64-row half pp of its 128 A rows, to both pairs
            const uint16_t a_mask = static_cast<uint16_t>((1u << rank) | (1u << (2u + rank)));
            auto load_a = [&](const Prob& P, int stage, int m0, int k0) {
                uint8_t* sa = smem_a + stage * C::kABytes;
                if constexpr (MC == 2) {
                    const int h = static_cast<int>(pp);
                    if (A_MN) tc::tma_load_2d_pair_mc(sa + h * 64 * BK * 2, &P.ta, full_leader + stage * 8,
                                                      m0 + h * 64, k0, a_mask);
                    else tc::tma_load_2d_pair_mc(sa + h * 64 * 128, &P.ta, full_leader + stage * 8,
                                                 k0, m0 + h * 64, a_mask);
                } else if (A_MN) {
#pragma unroll
                    for (int c = 0; c < BM / 64; ++c) load(sa + c * 64 * BK * 2, &P.ta, stage, m0 + c * 64, k0);
                } else {
                    load(sa, &P.ta, stage, k0, m0);
                }
            };
            auto load_b = [&](const Prob& P, int stage, int n0, int k0) {
                uint8_t* sb = smem_b + stage * C::kBBytes;
                if (B_MN) {
#pragma unroll
                    for (int c = 0; c < C::kBRows / 64; ++c)
                        load(sb + c * 64 * BK * 2, &P.tb, stage, n0 + c * 64, k0);
                } else {
                    load(sb, &P.tb, stage, k0, n0);
                }
            };
            auto expect = [&](int stage) {
                if (rank == 0) tc::mbar_expect_tx(&full_bar[stage], C::kTxBytes);
            };
            // B stages of the first unit that do not depend on the previous kernel
            int pre = 0;
            if (g.b_prefetch && cid < g.units && !(MM_GEMM_DEBUG & 4)) {
                const Unit w = unit_at(cid);
                const Prob& P = g.prob[w.pi];
                pre = min(C::kStages, w.kb1 - w.kb0);
                const int tn = MC == 2 ? 2 * w.tn + static_cast<int>(pp) : w.tn;
                for (int i = 0; i < pre; ++i) {
                    expect(i);
                    load_b(P, i, tn * BN + rank * C::kBRows, (w.kb0 + i) * BK);
                }
            }
            pdl_wait();
            if (g.span_lo) atomicMin(g.span_lo, gtime());
            int stage = 0;
            uint32_t phase = 0;
            int issued = 0;
            for (int u = cid; u < g.units; u += ncta) {
                const Unit w = unit_at(u);
                const Prob& P = g.prob[w.pi];
                const int tn = MC == 2 ? 2 * w.tn + static_cast<int>(pp) : w.tn;
                const int m0 = w.tm * (BM * CG) + rank * BM, n0 = tn * BN + rank * C::kBRows;
                for (int kb = w.kb0; kb < w.kb1; ++kb, ++issued) {
                    if (issued < pre) {  // expect_tx and B already issued
                        load_a(P, stage, m0, kb * BK);
                    } else {
                        tc::mbar_wait(&empty_bar[stage], phase ^ 1);
                        MM_KB_TRACE(0, issued);
                        if (MM_GEMM_DEBUG & 4) {  // diagnostics: no loads, MMAs on stale smem
                            if (rank == 0) tc::mbar_arrive(&full_bar[stage]);
                        } else {
                            expect(stage);
                            load_a(P, stage, m0, kb * BK);
                            load_b(P, stage, n0, kb * BK);
                        }
                    }
                    if (++stage == C::kStages) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        // (pair: the leader issues for both CTAs; the peer's warp 1 only owns
        // its half of the TMEM allocation).  The warp stays converged and one
        // lane is elected inside each MMA (see tc::mma_bf16_elect); operand
        // descriptors are the stage-0 descriptor plus the stage/K offset in
        // the 14-bit start-address field (smem addresses < 256 KB: no carry).
        // The accumulator address is the column offset alone: TMEM is
        // allocated at column 0 because one GEMM CTA fills an SM's shared
        // memory (checked at allocation).
        constexpr uint32_t idesc = tc::idesc_bf16_f32(BM * CG, BN, A_MN, B_MN);
        const uint64_t a_desc0 = A_MN ? tc::umma_desc_sw128(tc::smem_u32(smem_a), 64 * BK * 2, 1024)
                                      : tc::umma_desc_sw128(tc::smem_u32(smem_a), 16, 1024);
        const uint64_t b_desc0 = B_MN ? tc::umma_desc_sw128(tc::smem_u32(smem_b), 64 * BK * 2, 1024)
                                      : tc::umma_desc_sw128(tc::smem_u32(smem_b), 16, 1024);
        // per-K-step advance (16-byte units): K-major 32 B inside the swizzled
        // row; MN-major 16 K-rows = 2 x 1024 B
        constexpr int a_kstep = A_MN ? 2048 / 16 : 32 / 16;
        constexpr int b_kstep = B_MN ? 2048 / 16 : 32 / 16;
        const uint32_t a_lo0 = static_cast<uint32_t>(a_desc0), a_hi = static_cast<uint32_t>(a_desc0 >> 32);
        const uint32_t b_lo0 = static_cast<uint32_t>(b_desc0), b_hi = static_cast<uint32_t>(b_desc0 >> 32);
        int stage = 0;
        uint32_t phase = 0;
        int local = 0;
        int consumed = 0;
        for (int u = cid; u < g.units && rank == 0; u += ncta, ++local) {
            const Unit w = unit_at(u);
            const int kb0 = w.kb0, kb1 = w.kb1;
            const int acc = local & 1;
            const uint32_t acc_phase = (local >> 1) & 1;
            if constexpr (CG == 2) tc::mbar_wait_cluster(&tempty_bar[acc], acc_phase ^ 1);
            else tc::mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
            tc::tc_fence_after();
            const uint32_t d_tmem = static_cast<uint32_t>(acc * BN);
            for (int kb = kb0; kb < kb1; ++kb, ++consumed) {
                tc::mbar_wait(&full_bar[stage], phase);
                tc::tc_fence_after();
                MM_KB_TRACE(128, consumed);
                if (consumed == 0 && lane == 0) MM_TRACE(2);
                const uint32_t a_lo = a_lo0 + static_cast<uint32_t>(stage * (C::kABytes / 16));
                const uint32_t b_lo = b_lo0 + static_cast<uint32_t>(stage * (C::kBBytes / 16));
                if (!(MM_GEMM_DEBUG & 1)) {
                    tc::mma_kblock_commit<CG, a_kstep, b_kstep>(d_tmem, a_lo, a_hi, b_lo, b_hi, idesc,
                                                                kb > kb0 ? 1u : 0u, &empty_bar[stage],
                                                                empty_mask);
                } else {
                    tc::mma_commit_elect<CG>(&empty_bar[stage], empty_mask);
                }
                MM_KB_TRACE(512, consumed);  // MMAs + commit issued
                if (CG == 2 && dbias_any) tc::mma_commit_elect<CG>(&bias_bar[stage], pair_mask);
                if (++stage == C::kStages) { stage = 0; phase ^= 1; }
            }
            tc::mma_commit_elect<CG>(&tfull_bar[acc], pair_mask);
            if (lane == 0) MM_TRACE(3);
            __syncwarp();
        }
    } else if (warp >= kBiasWarp) {
        // ------------------------------------------------------------ bias-grad warp
        // Second consumer of every smem stage.  For a wgrad (A = dY, MN-major)
        // with dbias set, dbias[m] += sum_k dY[k, m]: the tiles_n units that load
        // the same A rows share the work -- N-column tn sums the k-blocks with
        // kb % tiles_n == tn, so every k-block is summed exactly once.  Lane owns M = 4*lane..4*lane+3
        // (box lane/16, 16B chunk (lane%16)/2, half lane%2; rows are K,
        // 128B-swizzled).  Every stage is released here too (empty count 2).
        // A pair's peer cannot wait on the leader's full barrier, so there the
        // MMA's commit to bias_bar says the stage is resident (and still held:
        // the empty barrier also needs this warp's arrival).
        if (!dbias_any) goto done;
        pdl_wait();
        {
        int stage = 0;
        uint32_t phase = 0;
        for (int u = cid; u < g.units; u += ncta) {
            const Unit w = unit_at(u);
            const Prob& P = g.prob[w.pi];
            const int kb0 = w.kb0, kb1 = w.kb1, tn = w.tn;
            float* dbias = P.dbias;
            const int tiles_n = P.tiles_n;
            const bool bias_sum = A_MN && dbias != nullptr;
            float bsum[4] = {0.f, 0.f, 0.f, 0.f};
            for (int kb = kb0; kb < kb1; ++kb) {
                if constexpr (CG == 2) tc::mbar_wait(&bias_bar[stage], phase);
                else tc::mbar_wait(&full_bar[stage], phase);
                if (bias_sum && kb % tiles_n == tn) {
                    const uint8_t* box = smem_a + stage * C::kABytes + (lane >> 4) * 64 * BK * 2;
                    const int chunk = (lane & 15) >> 1, sub = (lane & 1) * 8;
                    const int r0 = (warp - kBiasWarp) * (BK / kBiasWarps);
#pragma unroll
                    for (int r = r0; r < r0 + BK / kBiasWarps; ++r) {
                        const uint2 v = *reinterpret_cast<const uint2*>(
                            box + r * 128 + ((chunk ^ (r & 7)) * 16) + sub);
                        bsum[0] += bf16_to_f(v.x & 0xffff);
                        bsum[1] += bf16_to_f(v.x >> 16);
                        bsum[2] += bf16_to_f(v.y & 0xffff);
                        bsum[3] += bf16_to_f(v.y >> 16);
                    }
                }
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&empty_bar[stage]);
                if (++stage == C::kStages) { stage = 0; phase ^= 1; }
            }
            if (bias_sum) {
                const int64_t m = int64_t(w.tm) * (BM * CG) + rank * BM + 4 * lane;
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (m + i < P.m) atomicAdd(dbias + m + i, bsum[i]);
            }
        }
        }
    done:;
    } else {
        // ------------------------------------------------------------ epilogue
        const int lane_grp = warp & 3;                   // TMEM lanes this warp may access
        const int half = (warp - kEpiWarp0) >> 2;        // which column slice of the tile
        constexpr int kChunks = BN / 32 / kSlices;       // 32-column chunks per warp
        // residual tile of this warp's rows / columns into TMEM while the
        // MMAs of the unit run (lane = row: 128 B per lane per chunk; the
        // LSU is idle during the mainloop), read back next to the
        // accumulator in the epilogue -- the add order stays
        // (acc + bias) + resid
        auto resid_to_tmem = [&](const Prob& P, int tm, int cbase) {
            const int64_t rrow = int64_t(tm) * BM + lane_grp * 32 + lane;
            const uint32_t t_res = tmem_base + (static_cast<uint32_t>(lane_grp * 32) << 16) +
                                   C::kResidCol + half * (BN / kSlices);
#pragma unroll 1
            for (int c = 0; c < kChunks; ++c) {
                const int col0 = cbase + c * 32;
                uint32_t r[32];
                if (rrow < P.m && col0 + 32 <= P.n) {
                    const float4* res = reinterpret_cast<const float4*>(P.resid + rrow * P.ldd + col0);
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const float4 x = res[q];
                        r[4 * q] = __float_as_uint(x.x); r[4 * q + 1] = __float_as_uint(x.y);
                        r[4 * q + 2] = __float_as_uint(x.z); r[4 * q + 3] = __float_as_uint(x.w);
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        r[j] = (rrow < P.m && col0 + j < P.n) ? __float_as_uint(P.resid[rrow * P.ldd + col0 + j]) : 0u;
                }
                tc::tmem_st_32x32(t_res + c * 32, r);
            }
            tc::tmem_st_wait();
        };
        // the first unit's residual before griddepcontrol.wait when the
        // caller says the previous kernel did not write it: its fetch then
        // overlaps that kernel's tail instead of this launch's mainloop
        bool resid_pre = false;
        if constexpr (C::kResidTmem) {
            if (cid < g.units) {
                const Unit w0 = unit_at(cid);
                const Prob& P0 = g.prob[w0.pi];
                if (P0.epilogue == MM_EPI_F32_RESID && P0.resid_early) {
                    resid_to_tmem(P0, w0.tm, w0.tn * BN + half * (BN / kSlices));
                    resid_pre = true;
                }
            }
        }
        pdl_wait();
        uint8_t* bufs = smem_epi + (warp - kEpiWarp0) * C::kEpiBufs * kEpiBufBytes;
        int nbuf = 0;
        int local = 0;
        int ln_round = 0;  // CN > 1: row-sum exchanges so far (two per tile)
        for (int u = cid; u < g.units; u += ncta, ++local) {
            const Unit w = unit_at(u);
            const Prob& P = g.prob[w.pi];
            const int epi = EK >= 0 ? EK : P.epilogue;
            const bool out_bf16 = epi == MM_EPI_BF16 || epi == MM_EPI_BF16_RELU || epi == MM_EPI_BF16_DRELU;
            const bool reduce = epi == MM_EPI_F32_ACCUM;
            const bool bias = has_bias(P, epi);
            const int tm = w.tm, tn = MC == 2 ? 2 * w.tn + static_cast<int>(pp) : w.tn;
            const int acc = local & 1;
            const uint32_t acc_phase = (local >> 1) & 1;
            const int cbase = tn * BN + half * (BN / kSlices);
            const bool resid_tm = C::kResidTmem && epi == MM_EPI_F32_RESID;
            // this CTA's last tile: once its accumulator is final every
            // mainloop stage is idle (no further loads; the MMAs that read
            // them have completed), so each warp stages each chunk in its own
            // box there instead of waiting for the previous box's store to be
            // read (single CTAs without bias-gradient warps)
            const bool wide = MM_GEMM_WIDE_LAST && CG == 1 && CN == 1 && !dbias_any && u + ncta >= g.units;
            if constexpr (C::kResidTmem) {
                if (resid_tm && !(local == 0 && resid_pre)) resid_to_tmem(P, tm, cbase);
            }
            // bias for this warp's columns, fetched before waiting on the MMAs
            float bv[kChunks];
#pragma unroll
            for (int c = 0; c < kChunks; ++c) {
                const int col = cbase + c * 32 + lane;
                bv[c] = (bias && col < P.n) ? __ldg(P.bias + col) : 0.f;
            }
            tc::mbar_wait(&tfull_bar[acc], acc_phase);
            tc::tc_fence_after();
            // last tile's accumulator is final: let the dependent grid launch
            // (its blocks sit in griddepcontrol.wait until this grid is done)
            if (u + ncta >= g.units) pdl_trigger();
            if (warp == kEpiWarp0 && lane == 0 && local == 0) MM_TRACE(4);
            const int row0 = tm * (BM * CG) + rank * BM + lane_grp * 32;  // this warp's first row
            const int64_t row = int64_t(row0) + lane;
            const uint32_t t_row = tmem_base + (static_cast<uint32_t>(lane_grp * 32) << 16) + acc * BN +
                                   half * (BN / kSlices);
            float xs[CN > 1 ? kChunks : 1][32];  // LayerNorm input kept in registers
#pragma unroll
            for (int c = 0; c < kChunks; ++c) {
                const int col0 = cbase + c * 32;
                if (col0 < P.n) {
                    uint32_t v[32];
                    tc::tmem_ld_32x32(t_row + c * 32, v);
                    tc::tmem_ld_wait();
                    float f[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
                    epilogue_math(P, epi, row, col0, f, bv[c], resid_tm);
                    if (epi == MM_EPI_BF16_RELU && P.relu_mask && row < P.m) {
                        // bit j = the bf16 output is non-zero.  For f = relu(.) >= 0
                        // (or NaN) that is !(f <= 2^-134): round-to-nearest-even
                        // takes exactly [0, 2^-134] to bf16 zero.  A float compare
                        // instead of a second float -> bf16 conversion per element
                        // (the conversion pipe is the bottleneck here: 13.0 vs
                        // 10.8 us for the FFN-up GEMM with / without the mask)
                        constexpr float kBf16Zero = 0x1p-134f;
                        uint32_t bits = 0;
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (col0 + j < P.n && !(f[j] <= kBf16Zero)) bits |= 1u << j;
                        P.relu_mask[row * P.mask_ld + (col0 >> 5)] = bits;
                    }
                    if constexpr (C::kResidTmem) {
                        if (resid_tm) {
                            const uint32_t t_res = tmem_base + (static_cast<uint32_t>(lane_grp * 32) << 16) +
                                                   C::kResidCol + half * (BN / kSlices) + c * 32;
                            tc::tmem_ld_32x32(t_res, v);
                            tc::tmem_ld_wait();
#pragma unroll
                            for (int j = 0; j < 32; ++j) f[j] += __uint_as_float(v[j]);
                        }
                    }
                    if constexpr (CN > 1) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) xs[c][j] = f[j];
                    }
                    uint8_t* buf;
                    if (wide) {
                        buf = smem_a + ((warp - kEpiWarp0) * kChunks + c) * kEpiBufBytes;
                    } else {
                        buf = bufs + nbuf * kEpiBufBytes;
                        if (lane == 0) tc::bulk_wait_read<C::kEpiBufs - 1>();  // the store that last read `buf` is done
                        __syncwarp();
                    }
                    stage_row(buf, lane, f, out_bf16);
                    tc::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0 && !(MM_GEMM_DEBUG & 2)) {
                        if (reduce) tc::tma_reduce_add_2d(&P.td, buf, col0, row0);
                        else tc::tma_store_2d(&P.td, buf, col0, row0);
                        tc::bulk_commit();
                    }
                    if (!wide && ++nbuf == C::kEpiBufs) nbuf = 0;
                }
            }
            // accumulator drained: one arrive per warp on the MMA CTA's barrier
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if constexpr (CG == 2) tc::mbar_arrive_cluster(&tempty_bar[acc], lead);
                else tc::mbar_arrive(&tempty_bar[acc]);
            }
            if constexpr (CN > 1 && !(MM_GEMM_DEBUG & 16)) {
                // ---- fused LayerNorm of the rows just written (x = resid + acc
                // + bias).  Each CTA of the cluster holds 128 of the row's
                // N = CN * 128 columns: per-row partial sums go through
                // distributed shared memory, summed in cluster-rank order so
                // every CTA normalises with identical statistics.
                const int rloc = lane_grp * 32 + lane;  // row within the tile
                // one exchange per tile: (sum x, sum x^2) per row; var =
                // E[x^2] - mean^2 in fp32 (the residual stream's |mean| is a
                // few sigma at most, so the cancellation costs < 1e-5 relative)
                auto row_totals = [&](float v1, float v2) -> float2 {
                    if constexpr (MM_GEMM_DEBUG & 8) return make_float2(v1 * CN, v2 * CN);  // no exchange
                    float2* part2 = reinterpret_cast<float2*>(ln_part);  // [2][BM]
                    float2* xch2 = reinterpret_cast<float2*>(ln_xch);    // [2][BM]
                    part2[half * BM + rloc] = make_float2(v1, v2);
                    tc::named_barrier_sync(1, kEpiWarps * 32);
                    const int par = ln_round & 1;
                    if (half == 0) {
                        const float2 a0 = part2[rloc], a1 = part2[BM + rloc];
                        xch2[par * BM + rloc] = make_float2(a0.x + a1.x, a0.y + a1.y);
                    }
                    tc::named_barrier_sync(1, kEpiWarps * 32);
                    if (threadIdx.x == kEpiWarp0 * 32) {
#pragma unroll
                        for (int r = 0; r < CN; ++r) tc::mbar_arrive_cluster(&xch_bar[par], r);
                    }
                    tc::mbar_spin_cluster(&xch_bar[par], (ln_round >> 1) & 1);
                    ++ln_round;
                    const uint32_t slot = tc::smem_u32(&xch2[par * BM + rloc]);
                    float2 t = make_float2(0.f, 0.f);
#pragma unroll
                    for (int r = 0; r < CN; ++r) {
                        const float2 q = tc::ld_shared_cluster_f32x2(tc::mapa_u32(slot, r));
                        t.x += q.x;
                        t.y += q.y;
                    }
                    return t;
                };
                float s1 = 0.f, s2 = 0.f;
#pragma unroll
                for (int c = 0; c < kChunks; ++c)
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        s1 += xs[c][j];
                        s2 = fmaf(xs[c][j], xs[c][j], s2);
                    }
                const float inv_n = 1.f / static_cast<float>(P.n);
                const float2 tot = row_totals(s1, s2);
                const float mu = tot.x * inv_n;
                const float var = fmaxf(tot.y * inv_n - mu * mu, 0.f);
                const float rs = rsqrtf(var + g.ln.eps);
#pragma unroll
                for (int c = 0; c < kChunks; ++c) {
                    const int col0 = cbase + c * 32;
                    float hv[32];
                    const float4* g4 = reinterpret_cast<const float4*>(g.ln.gamma + col0);
                    const float4* b4 = reinterpret_cast<const float4*>(g.ln.beta + col0);
#pragma unroll
                    for (int q = 0; q < 8; ++q) {  // warp-uniform addresses: broadcast loads
                        const float4 gg = __ldg(g4 + q), bb = __ldg(b4 + q);
                        hv[4 * q + 0] = (xs[c][4 * q + 0] - mu) * rs * gg.x + bb.x;
                        hv[4 * q + 1] = (xs[c][4 * q + 1] - mu) * rs * gg.y + bb.y;
                        hv[4 * q + 2] = (xs[c][4 * q + 2] - mu) * rs * gg.z + bb.z;
                        hv[4 * q + 3] = (xs[c][4 * q + 3] - mu) * rs * gg.w + bb.w;
                    }
                    uint8_t* buf = bufs + nbuf * kEpiBufBytes;
                    if (lane == 0) tc::bulk_wait_read<C::kEpiBufs - 1>();
                    __syncwarp();
                    stage_row(buf, lane, hv, true);
                    tc::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        tc::tma_store_2d(&g.ln.th, buf, col0, row0);
                        tc::bulk_commit();
                    }
                    if (++nbuf == C::kEpiBufs) nbuf = 0;
                }
                if (crank == 0 && half == 0 && row < P.m) {
                    g.ln.mean[row] = mu;
                    g.ln.rstd[row] = rs;
                }
            }
        }
        if (warp == kEpiWarp0 && lane == 0) MM_TRACE(5);
        // the CTA may exit once its staging boxes have been READ: the global
        // writes themselves complete with the grid (what griddepcontrol.wait
        // of the next kernel and stream order wait for), as in CUTLASS's
        // tma_store_wait
        if (lane == 0) tc::bulk_wait_read<0>();
        if (warp == kEpiWarp0 && lane == 0) MM_TRACE(6);
    }
    pdl_trigger();
    tc::tc_fence_before();
    // pair: both CTAs done with the pair's TMEM / barriers; LN cluster: no peer
    // still reads this CTA's exchange slots
    if constexpr (CG == 2 || CN > 1) tc::cluster_sync();
    else __syncthreads();
    if (warp == 1) {
        tc::tc_fence_after();
        if constexpr (CG == 2) tc::tmem_dealloc_pair(tmem_base, C::kTmemCols);
        else tc::tmem_dealloc(tmem_base, C::kTmemCols);
    }
    if (threadIdx.x == 0) MM_TRACE(7);
    if (threadIdx.x == 0 && g.span_hi) atomicMax(g.span_hi, gtime());
}

// ----------------------------------------------------------------------------
// host side

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* ptr = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    });
    return fn;
}

// 2D tensor map over a row-major [outer, inner] matrix with row stride `ld`
// elements, box {box_inner, box_outer}; OOB loads read 0, OOB stores clip.
int make_map(CUtensorMap* map, const void* base, int64_t inner, int64_t outer, int64_t ld,
             int box_outer, int box_inner = 64, bool fp32 = false,
             CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
    auto enc = get_encode();
    if (!enc) {
        mm::set_error("cuTensorMapEncodeTiled unavailable");
        return mm::kCuda;
    }
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * (fp32 ? 4 : 2))};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(box_inner), static_cast<cuuint32_t>(box_outer)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, fp32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                     2, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        mm::set_error("cuTensorMapEncodeTiled failed (%d): inner=%lld outer=%lld ld=%lld box=%d",
                      (int)r, (long long)inner, (long long)outer, (long long)ld, box_outer);
        return mm::kCuda;
    }
    return 0;
}

template <int BN, int A_MN, int B_MN, int NP, int CG, int CN = 1, int RT = 0, int MC = 1, int EK = -1>
int launch(const Group<NP>& g, cudaStream_t s) {
    using C = Cfg<BN, CG, CN, RT>;
    auto kern = gemm_tcgen05_kernel<BN, A_MN, B_MN, NP, CG, CN, RT, MC, EK>;
    static bool attr_set = false;  // per instantiation
    if (!attr_set) {
        MM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::kSmem));
        attr_set = true;
    }
    // persistent: one CTA (pair / cluster) per SM (pair / cluster of SMs);
    // clusters wider than a pair fit only as often as the GPCs allow
    const int per = CG * CN * MC;
    static int max_clusters = 0;  // per instantiation
    if (max_clusters == 0) {
        max_clusters = mm::num_sms() / per;
        if (per > 2) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(static_cast<unsigned>(per * max_clusters));
            cfg.blockDim = dim3(kThreads);
            cfg.dynamicSmemBytes = C::kSmem;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = static_cast<unsigned>(per);
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            int n = 0;
            if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) == cudaSuccess && n > 0)
                max_clusters = std::min(max_clusters, n);
            (void)cudaGetLastError();
        }
    }
    const int ctas = std::min(g.units, max_clusters) * per;
    MM_CUDA_TRY(mm::launch_pdl_cluster(kern, dim3(ctas), dim3(kThreads), C::kSmem, s,
                                       static_cast<unsigned>(per), g));
    MM_LAUNCH_CHECK("gemm_tcgen05_kernel");
    return 0;
}

template <int BN, int NP, int CG>
int dispatch(int a_mn, int b_mn, const Group<NP>& g, cudaStream_t s) {
    if (!a_mn && !b_mn) return launch<BN, 0, 0, NP, CG>(g, s);
    if (!a_mn && b_mn) return launch<BN, 0, 1, NP, CG>(g, s);
    if (a_mn && !b_mn) return launch<BN, 1, 0, NP, CG>(g, s);
    return launch<BN, 1, 1, NP, CG>(g, s);
}
// single-problem 128-wide single-CTA launches, one instantiation per
// epilogue of the step's hot shapes (forward: K-major A and B; dgrad:
// MN-major B); kNotSpecialised: use the generic instantiation
constexpr int kNotSpecialised = 1;  // (library status codes are <= 0)
template <int NP>
int dispatch_epi(int a_mn, int b_mn, int epi, const Group<NP>& g, cudaStream_t s) {
    if constexpr (NP == 1) {
        if (!a_mn && !b_mn) {
            if (epi == MM_EPI_BF16) return launch<128, 0, 0, 1, 1, 1, 0, 1, MM_EPI_BF16>(g, s);
            if (epi == MM_EPI_BF16_RELU) return launch<128, 0, 0, 1, 1, 1, 0, 1, MM_EPI_BF16_RELU>(g, s);
            if (epi == MM_EPI_F32) return launch<128, 0, 0, 1, 1, 1, 0, 1, MM_EPI_F32>(g, s);
        } else if (!a_mn && b_mn) {
            if (epi == MM_EPI_BF16) return launch<128, 0, 1, 1, 1, 1, 0, 1, MM_EPI_BF16>(g, s);
            if (epi == MM_EPI_BF16_DRELU) return launch<128, 0, 1, 1, 1, 1, 0, 1, MM_EPI_BF16_DRELU>(g, s);
            if (epi == MM_EPI_F32) return launch<128, 0, 1, 1, 1, 1, 0, 1, MM_EPI_F32>(g, s);
            if (epi == MM_EPI_F32_ACCUM) return launch<128, 0, 1, 1, 1, 1, 0, 1, MM_EPI_F32_ACCUM>(g, s);
        }
    }
    return kNotSpecialised;
}
// the same for 256-wide tiles: single CTAs (MC = 1) and clustered CTA pairs
// (MC = 2) -- the config-5 shapes and the generator
template <int NP, int CG, int MC>
int dispatch_epi256(int a_mn, int b_mn, int epi, const Group<NP>& g, cudaStream_t s) {
    if constexpr (NP == 1) {
        if (!a_mn && !b_mn) {
            if (epi == MM_EPI_BF16) return launch<256, 0, 0, 1, CG, 1, 0, MC, MM_EPI_BF16>(g, s);
            if (epi == MM_EPI_BF16_RELU) return launch<256, 0, 0, 1, CG, 1, 0, MC, MM_EPI_BF16_RELU>(g, s);
            if (epi == MM_EPI_F32_RESID) return launch<256, 0, 0, 1, CG, 1, 0, MC, MM_EPI_F32_RESID>(g, s);
        } else if (!a_mn && b_mn) {
            if (epi == MM_EPI_BF16) return launch<256, 0, 1, 1, CG, 1, 0, MC, MM_EPI_BF16>(g, s);
            if (epi == MM_EPI_BF16_DRELU) return launch<256, 0, 1, 1, CG, 1, 0, MC, MM_EPI_BF16_DRELU>(g, s);
            if (epi == MM_EPI_F32) return launch<256, 0, 1, 1, CG, 1, 0, MC, MM_EPI_F32>(g, s);
        }
    }
    return kNotSpecialised;
}
// CTA pairs in clusters of two pairs with multicast A halves (MC = 2)
template <int BN, int NP>
int dispatch_mc(int a_mn, int b_mn, const Group<NP>& g, cudaStream_t s) {
    if (!a_mn && !b_mn) return launch<BN, 0, 0, NP, 2, 1, 0, 2>(g, s);
    if (!a_mn && b_mn) return launch<BN, 0, 1, NP, 2, 1, 0, 2>(g, s);
    if (a_mn && !b_mn) return launch<BN, 1, 0, NP, 2, 1, 0, 2>(g, s);
    return launch<BN, 1, 1, NP, 2, 1, 0, 2>(g, s);
}

unsigned long long* g_trace_buf = nullptr;  // set by mm_gemm_trace (diagnostics)

// optional per-launch timing (roofline evidence inside bench.py): every
// launch records its own span on the device (%globaltimer: first CTA past
// griddepcontrol.wait -> last CTA exit), so no event or host call sits
// between kernels and programmatic dependent launch stays as in the
// untimed step
struct GemmTiming {
    bool on = false;
    unsigned long long* buf = nullptr;  // [cap] span starts, then [cap] span ends
    size_t cap = 0;
    std::vector<double> flops;
    std::vector<int> shape;  // m, n, k, problems per launch (first problem's shape)
    size_t used = 0;
} g_timing;

bool out_bf16_epi(int e) {
    return e == MM_EPI_BF16 || e == MM_EPI_BF16_RELU || e == MM_EPI_BF16_DRELU;
}

int check_args(const mm_gemm_args* a) {
    MM_CHECK_ARG(a != nullptr, "args is NULL");
    MM_CHECK_ARG(a->m > 0 && a->n > 0 && a->k > 0, "empty GEMM %lldx%lldx%lld", (long long)a->m,
                 (long long)a->n, (long long)a->k);
    MM_CHECK_ARG(a->epilogue >= MM_EPI_BF16 && a->epilogue <= MM_EPI_F32_RESID_LN, "bad epilogue");
    if (a->epilogue == MM_EPI_F32_RESID_LN) {
        MM_CHECK_ARG(a->n == 512 || a->n == 1024, "fused LayerNorm needs N in {512, 1024} (got %lld)",
                     (long long)a->n);
        MM_CHECK_ARG(a->a_kmajor && a->b_kmajor, "fused LayerNorm needs K-major A and B");
        MM_CHECK_ARG(a->ln_gamma && a->ln_beta && a->ln_out && a->ln_mean && a->ln_rstd,
                     "fused LayerNorm needs gamma, beta, out, mean and rstd");
        MM_CHECK_ARG((reinterpret_cast<uintptr_t>(a->ln_out) & 15) == 0 &&
                         (reinterpret_cast<uintptr_t>(a->ln_gamma) & 15) == 0 &&
                         (reinterpret_cast<uintptr_t>(a->ln_beta) & 15) == 0,
                     "LayerNorm tensors must be 16-byte aligned");
    }
    MM_CHECK_ARG(a->a && a->b && a->d, "NULL operand");
    const bool out_bf16 = out_bf16_epi(a->epilogue);
    MM_CHECK_ARG((a->lda % 8) == 0 && (a->ldb % 8) == 0, "lda/ldb must be multiples of 8");
    MM_CHECK_ARG((reinterpret_cast<uintptr_t>(a->a) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(a->b) & 15) == 0,
                 "A/B must be 16-byte aligned");
    MM_CHECK_ARG((reinterpret_cast<uintptr_t>(a->d) & 15) == 0 && (a->ldd % (out_bf16 ? 8 : 4)) == 0,
                 "D must be 16-byte aligned with 16-byte row stride");
    MM_CHECK_ARG((a->epilogue != MM_EPI_F32_RESID && a->epilogue != MM_EPI_F32_RESID_LN) || a->resid,
                 "RESID epilogue needs resid");
    MM_CHECK_ARG(a->epilogue != MM_EPI_BF16_DRELU || a->aux || a->relu_mask, "DRELU epilogue needs aux or relu_mask");
    MM_CHECK_ARG(!a->relu_mask || a->epilogue == MM_EPI_BF16_RELU || a->epilogue == MM_EPI_BF16_DRELU,
                 "relu_mask is for the RELU / DRELU epilogues");
    MM_CHECK_ARG(a->dbias == nullptr || !a->a_kmajor, "dbias needs an MN-major A operand");
    MM_CHECK_ARG(a->m < (int64_t(1) << 31) && a->n < (int64_t(1) << 31) && a->k < (int64_t(1) << 31),
                 "GEMM dimension >= 2^31");
    return 0;
}

// Tile shape for a launch: (BN, CG) minimising a per-SM time model fitted to
// tools/gemm_micro.py sweeps on the B200 (config-3 shapes, N = 512..32000):
//   t = c0 + waves * kb * x
// c0 = fixed cost of a launch (prologue, first-load latency, last tile's
// epilogue and drain) and x = time per 64-deep k-block of one unit, which is
// MMA-issue bound (~80 cycles per tcgen05.mma) for 128-wide tiles and
// tensor-pipe bound for 256-wide ones; wide tiles then cost little more per
// k-block but quantise into fewer, longer waves.  A pair (CG = 2) computes a
// 256-row tile on two SMs for the same per-k-block time as a single CTA's
// 128-row tile, at a larger fixed cost.
struct TileChoice {
    int bn, cg;
};
struct TileCost {
    double c0_us, x_us;
};
TileCost tile_cost(int bn, int cg) {
    if (cg == 2) return bn == 256 ? TileCost{5.97, 0.301} : TileCost{5.44, 0.194};
    return bn == 256 ? TileCost{5.27, 0.305} : bn == 192 ? TileCost{4.64, 0.248} : TileCost{4.16, 0.179};
}
constexpr double kAccumWaveUs = 0.9;  // extra per wave of fp32 reduce-add (split-K / wgrad) epilogues

int split_cap(const mm_gemm_args* const* probs, int n, int bn, int cg, int sms);

// an fp32 weight-gradient problem: reduce-add (MM_EPI_F32_ACCUM) or the store
// of a module's first micro-batch (MM_EPI_F32 with both operands MN-major)
bool f32_wgrad(const mm_gemm_args* a) {
    return a->epilogue == MM_EPI_F32_ACCUM ||
           (a->epilogue == MM_EPI_F32 && !a->a_kmajor && !a->b_kmajor);
}

TileChoice choose_tile(const mm_gemm_args* const* probs, int n, int sms) {
    // MM_GEMM_RULES=0 (diagnostics): the bare fitted model, without the two
    // measured corrections for CTA pairs below
    static const bool rules = [] {
        const char* e = std::getenv("MM_GEMM_RULES");
        return !(e && e[0] == '0');
    }();
    TileChoice best{128, 1};
    double best_cost = 1e300;
    for (int cg : {1, 2}) {
        for (int cand : {128, 192, 256}) {
            if (cg == 2 && cand == 192) continue;
            bool fits = true, accum = true;
            for (int i = 0; i < n; ++i) {
                if (cand > 128 && probs[i]->n <= cand - 64) fits = false;
                // fp32 weight-gradient launches (reduce-add, or the store of a
                // module's first micro-batch) share one cost model
                accum = accum && f32_wgrad(probs[i]);
            }
            if (!fits) continue;
            const int cap = split_cap(probs, n, cand, cg, sms);
            int64_t units = 0;
            double kb_sum = 0;
            for (int i = 0; i < n; ++i) {
                const int64_t t = ((probs[i]->m + BM * cg - 1) / (BM * cg)) * ((probs[i]->n + cand - 1) / cand);
                const int num_kb = static_cast<int>((probs[i]->k + BK - 1) / BK);
                int splits = probs[i]->epilogue == MM_EPI_F32_ACCUM ? std::max(1, std::min(cap, num_kb / 2)) : 1;
                const int kb_per = (num_kb + splits - 1) / splits;
                splits = (num_kb + kb_per - 1) / kb_per;
                units += t * splits;
                kb_sum += double(t * splits) * kb_per;
            }
            const int slots = sms / cg;
            const double waves = double((units + slots - 1) / slots);
            const TileCost tc = tile_cost(cand, cg);
            const double kb_unit = kb_sum / double(units);
            double x_us = tc.x_us;
            double wave_us = accum ? kAccumWaveUs : 0.0;
            if (cg == 2 && rules) {
                // measured in the config-3 step (MM_GEMM_OVERRIDE A/B, r02ai):
                // a pair's per-unit handshakes (cluster-scope accumulator
                // barriers, multicast commits) do not amortise over 8 k-blocks
                // -- the generator forward (4096 x 32000 x 512) runs 12 us
                // faster on single-CTA 256-wide tiles -- while over hundreds of
                // k-blocks the pair's halved B traffic per SM wins -- the
                // generator dgrad (4096 x 512 x 32000) runs 7 us faster on
                // 256 x 128 pair tiles
                if (kb_unit <= 8.0) wave_us += 0.35;
                if (cand == 128 && kb_unit >= 256.0) x_us *= 0.9;
            }
            double cost = tc.c0_us + waves * (kb_unit * x_us + wave_us);
            // a launch that keeps every SM busy is L2->SM bandwidth bound
            // (~32 KB per k-block per CTA at every shape): only the pair's
            // 128 x 256 per-SM tile does enough MMA work per byte (measured on
            // the grouped weight-gradient launches, tools/wgrad_micro.py)
            if (accum && waves >= 2.0 && !(cg == 2 && cand == 256)) cost *= 1.15;
            if (cost < best_cost - 1e-9) { best_cost = cost; best = {cand, cg}; }
        }
    }
    // diagnostics: per-shape overrides "N,K,Bmn=CG:BN;..." (single-problem
    // launches; Bmn = 1 when B is MN-major), for step-level A/B of choices
    static const char* ovr = std::getenv("MM_GEMM_OVERRIDE");
    if (ovr && n == 1) {
        const char* q = ovr;
        while (*q) {
            long on = 0, ok = 0, ob = 0, ocg = 0, obn = 0;
            if (std::sscanf(q, "%ld,%ld,%ld=%ld:%ld", &on, &ok, &ob, &ocg, &obn) == 5 &&
                on == probs[0]->n && ok == probs[0]->k && ob == (probs[0]->b_kmajor ? 0 : 1) &&
                (ocg == 1 || ocg == 2) && (obn == 128 || obn == 192 || obn == 256 ||
                                           (MM_GEMM_BN64 && obn == 64 && ocg == 1))) {
                best = {static_cast<int>(obn), static_cast<int>(ocg)};
                break;
            }
            const char* semi = std::strchr(q, ';');
            if (!semi) break;
            q = semi + 1;
        }
    }
    if (const char* force = std::getenv("MM_GEMM_BN")) {  // diagnostics
        const int f = std::atoi(force);
        if (f == 128 || f == 192 || f == 256) best.bn = f;
    }
    if (const char* force = std::getenv("MM_GEMM_CG")) {  // diagnostics
        const int f = std::atoi(force);
        if (f == 1 || f == 2) best.cg = f;
    }
    if (best.cg == 2 && best.bn == 192) best.bn = 256;
    return best;
}

// Fill one problem of a launch (tensor maps + tiling); splits K for fp32
// accumulation when the launch has fewer tiles than two waves.
int setup_prob(Prob& P, const mm_gemm_args* a, int bn, int cg, int splits_cap, int mc = 1) {
    const bool out_bf16 = out_bf16_epi(a->epilogue);
    const int a_mn = a->a_kmajor ? 0 : 1;
    const int b_mn = a->b_kmajor ? 0 : 1;
    const int64_t tiles_m = (a->m + BM * cg - 1) / (BM * cg);
    // mc = 2: units are pairs of adjacent N-tiles (one per pair of the cluster)
    const int64_t tiles_n = ((a->n + bn - 1) / bn + mc - 1) / mc;
    const int num_kb = static_cast<int>((a->k + BK - 1) / BK);
    int splits = a->epilogue == MM_EPI_F32_ACCUM ? std::max(1, std::min(splits_cap, num_kb / 2)) : 1;
    const int kb_per = (num_kb + splits - 1) / splits;
    splits = (num_kb + kb_per - 1) / kb_per;  // no empty splits
    MM_CHECK_ARG(tiles_m * tiles_n * splits < (int64_t(1) << 31), "GEMM too large");
    int st;
    // A: K-major [M, K] rows of lda; MN-major [K, M] rows of lda
    st = a_mn ? make_map(&P.ta, a->a, a->m, a->k, a->lda, BK)
              : make_map(&P.ta, a->a, a->k, a->m, a->lda, mc == 2 ? 64 : BM);  // mc = 2: 64-row halves
    if (st) return st;
    st = b_mn ? make_map(&P.tb, a->b, a->n, a->k, a->ldb, BK)
              : make_map(&P.tb, a->b, a->k, a->n, a->ldb, bn / cg);  // a pair CTA stages BN/2 rows
    if (st) return st;
    // D: 32 x 32 boxes, swizzle matching the staging layout
    st = make_map(&P.td, a->d, a->n, a->m, a->ldd, 32, 32, !out_bf16,
                  out_bf16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B);
    if (st) return st;
    P.m = a->m; P.n = a->n; P.k = a->k; P.ldd = a->ldd;
    P.d = a->d; P.bias = a->bias; P.resid = a->resid;
    P.aux = reinterpret_cast<const __nv_bfloat16*>(a->aux);
    P.relu_mask = a->relu_mask;
    P.mask_ld = (a->n + 31) / 32;
    P.dbias = a->dbias;
    P.epilogue = a->epilogue;
    P.tiles_m = static_cast<int>(tiles_m);
    P.tiles_n = static_cast<int>(tiles_n);
    P.resid_early = a->resid_early != 0;
    P.splits = splits;
    P.kb_per_split = kb_per;
    P.num_kb = num_kb;
    // Consecutive units run at the same time on the persistent CTAs.  Walking
    // M first over every M-tile re-streams A from HBM for each N-tile once A
    // outgrows the L2 (8192^3: 2.3x cuBLAS's DRAM traffic, lower clocks under
    // the power cap); group the M-tiles so one group's A slices stay resident.
    const char* env_budget = std::getenv("MM_GEMM_L2_GROUP_MB");  // diagnostics / tests (0: off)
    const double budget = (env_budget ? std::atof(env_budget) : 48.0) * 1e6;
    const double a_slice = double(BM * cg) * double(a->k) * 2.0;  // bytes of A per M-tile
    P.group_m = static_cast<int>(tiles_m);
    if (budget > 0 && a_slice * double(tiles_m) > budget)
        P.group_m = std::max(1, static_cast<int>(budget / a_slice));
    return 0;
}

// K-split for fp32-accumulating launches: double while the launch stays
// within two waves
int split_cap(const mm_gemm_args* const* probs, int n, int bn, int cg, int sms) {
    int64_t tiles = 0;
    int min_kb = 1 << 30;
    bool all_accum = true;
    sms /= cg;
    for (int i = 0; i < n; ++i) {
        tiles += ((probs[i]->m + BM * cg - 1) / (BM * cg)) * ((probs[i]->n + bn - 1) / bn);
        min_kb = std::min<int>(min_kb, static_cast<int>((probs[i]->k + BK - 1) / BK));
        all_accum = all_accum && f32_wgrad(probs[i]);
    }
    int splits = 1;
    if (all_accum)
        while (tiles * splits * 2 <= 2 * sms && splits * 2 <= min_kb / 2) splits *= 2;
    return splits;
}

template <int NP>
int run_group(const mm_gemm_args* const* probs_in, int n, cudaStream_t s) {
    const int sms = mm::num_sms();
    const bool ln = probs_in[0]->epilogue == MM_EPI_F32_RESID_LN;
    const TileChoice tc = ln ? TileChoice{128, 1} : choose_tile(probs_in, n, sms);
    const int bn = tc.bn, cg = tc.cg;
    const int cap = ln ? 1 : split_cap(probs_in, n, bn, cg, sms);
    // a launch that splits K: store-mode weight gradients become zero + the
    // split reduce-add, so the result never depends on which micro-batch
    // stored (bit-identical to memset + MM_EPI_F32_ACCUM)
    static mm_gemm_args conv[kMaxProbs];
    static const mm_gemm_args* conv_ptr[kMaxProbs];
    const mm_gemm_args* const* probs = probs_in;
    if (cap > 1) {
        for (int i = 0; i < n; ++i) {
            conv[i] = *probs_in[i];
            if (conv[i].epilogue == MM_EPI_F32 && f32_wgrad(&conv[i])) {
                MM_CUDA_TRY(cudaMemset2DAsync(conv[i].d, size_t(conv[i].ldd) * 4, 0, size_t(conv[i].n) * 4,
                                              size_t(conv[i].m), s));
                conv[i].epilogue = MM_EPI_F32_ACCUM;
            }
            conv_ptr[i] = &conv[i];
        }
        probs = conv_ptr;
    }
    static Group<NP> g;  // host staging of the kernel parameter (large: tensor maps)
    std::memset(&g, 0, sizeof(g));
    int64_t units = 0;
    double flops = 0;
    static const bool log = std::getenv("MM_GEMM_LOG") != nullptr;  // diagnostics
    // CTA pairs run in clusters of two pairs with multicast A halves
    // (MM_GEMM_MC=0 for A/B): fewer L2 requests per SM, so less power at the
    // same work -- config 5 26.60 -> 26.42 ms at 1620 -> 1700+ MHz under the
    // power cap, config 3 3.418 -> 3.412 ms.  Not with the bias-gradient
    // warps (they read the stages the pair alone releases).
    bool dbias = false;
    for (int i = 0; i < n; ++i) dbias = dbias || probs[i]->dbias != nullptr;
    const char* mc_env = std::getenv("MM_GEMM_MC");
    const int mc = (cg == 2 && !ln && !dbias && !(mc_env && mc_env[0] == '0')) ? 2 : 1;
    for (int i = 0; i < n; ++i) {
        Prob& P = g.prob[i];
        if (int st = setup_prob(P, probs[i], bn, cg, cap, mc)) return st;
        P.unit_begin = static_cast<int>(units);
        units += int64_t(P.tiles_m) * P.tiles_n * P.splits;
        MM_CHECK_ARG(units < (int64_t(1) << 31), "GEMM launch too large");
        flops += 2.0 * double(probs[i]->m) * double(probs[i]->n) * double(probs[i]->k);
        if (log)
            std::fprintf(stderr, "mm_gemm m=%lld n=%lld k=%lld a_mn=%d b_mn=%d epi=%d bn=%d cg=%d mc=%d splits=%d units=%d group=%d/%d\n",
                         (long long)probs[i]->m, (long long)probs[i]->n, (long long)probs[i]->k,
                         probs[i]->a_kmajor ? 0 : 1, probs[i]->b_kmajor ? 0 : 1, probs[i]->epilogue,
                         bn, cg, mc, P.splits, P.tiles_m * P.tiles_n * P.splits, i, n);
    }
    g.n_probs = n;
    g.units = static_cast<int>(units);
    g.trace = g_trace_buf;
    g.b_prefetch = 1;
    g.any_dbias = 0;
    for (int i = 0; i < n; ++i) {
        g.b_prefetch &= probs[i]->b_prefetch ? 1 : 0;
        if (probs[i]->dbias) g.any_dbias = 1;
    }
    g.span_lo = g.span_hi = nullptr;
    if (g_timing.on && g_timing.used < g_timing.cap) {
        g.span_lo = g_timing.buf + g_timing.used;
        g.span_hi = g_timing.buf + g_timing.cap + g_timing.used;
        g_timing.flops.push_back(flops);
        g_timing.shape.insert(g_timing.shape.end(), {int(probs[0]->m), int(probs[0]->n), int(probs[0]->k), n});
        ++g_timing.used;
    }
    const int a_mn = probs[0]->a_kmajor ? 0 : 1;
    const int b_mn = probs[0]->b_kmajor ? 0 : 1;
    const char* spec_env = std::getenv("MM_GEMM_SPECIALIZE");  // read per call: tests toggle it
    const bool specialize = !(spec_env && spec_env[0] == '0');
    int rc;
    if (ln) {
        // units are 128-row blocks; a cluster of N / 128 CTAs shares each one
        const mm_gemm_args* a = probs[0];
        if (int st = make_map(&g.ln.th, a->ln_out, a->n, a->m, a->n, 32, 32, false,
                              CU_TENSOR_MAP_SWIZZLE_64B))
            return st;
        g.ln.gamma = a->ln_gamma; g.ln.beta = a->ln_beta;
        g.ln.mean = a->ln_mean; g.ln.rstd = a->ln_rstd; g.ln.eps = a->ln_eps;
        g.units = g.prob[0].tiles_m;
        if constexpr (NP == 1) {
            rc = g.prob[0].tiles_n == 4 ? launch<128, 0, 0, 1, 1, 4>(g, s) : launch<128, 0, 0, 1, 1, 8>(g, s);
        } else {
            rc = mm::kArg;
        }
    } else if (mc == 2) {
        if (NP == 1 && specialize && bn == 128 && !a_mn && b_mn && probs[0]->epilogue == MM_EPI_F32)
            rc = launch<128, 0, 1, NP, 2, 1, 0, 2, MM_EPI_F32>(g, s);  // the generator dgrad
        else if (NP == 1 && specialize && bn == 256 &&
                 (rc = dispatch_epi256<NP, 2, 2>(a_mn, b_mn, probs[0]->epilogue, g, s)) != kNotSpecialised) {
        } else if (bn == 256) rc = dispatch_mc<256, NP>(a_mn, b_mn, g, s);
        else rc = dispatch_mc<128, NP>(a_mn, b_mn, g, s);
    } else if (cg == 2) {
        if (bn == 256) rc = dispatch<256, NP, 2>(a_mn, b_mn, g, s);
        else rc = dispatch<128, NP, 2>(a_mn, b_mn, g, s);
    } else if (NP == 1 && bn == 128 && !a_mn && !b_mn && probs[0]->epilogue == MM_EPI_F32_RESID) {
        // residual parked in TMEM; the RESID epilogue alone
        if (specialize) rc = launch<128, 0, 0, NP, 1, 1, 1, 1, MM_EPI_F32_RESID>(g, s);
        else rc = launch<128, 0, 0, NP, 1, 1, 1>(g, s);
    } else if (NP == 1 && bn == 128 && specialize &&
               (rc = dispatch_epi<NP>(a_mn, b_mn, probs[0]->epilogue, g, s)) != kNotSpecialised) {
        // one epilogue's instantiation (MM_GEMM_SPECIALIZE=0 for A/B)
    } else if (NP == 1 && bn == 256 && cg == 1 && specialize &&
               (rc = dispatch_epi256<NP, 1, 1>(a_mn, b_mn, probs[0]->epilogue, g, s)) != kNotSpecialised) {
        // the generator forward, config 5's 256-wide single-CTA launches
    } else {
        if (bn == 256) rc = dispatch<256, NP, 1>(a_mn, b_mn, g, s);
        else if (bn == 192) rc = dispatch<192, NP, 1>(a_mn, b_mn, g, s);
#if MM_GEMM_BN64
        else if (bn == 64 && NP == 1) rc = dispatch<64, NP, 1>(a_mn, b_mn, g, s);
#endif
        else rc = dispatch<128, NP, 1>(a_mn, b_mn, g, s);
    }
    return rc;
}

}  // namespace

// diagnostics: device buffer of >= 8 * num_SMs u64 for per-CTA phase stamps of
// subsequent mm_gemm launches (NULL disables)
extern "C" int mm_gemm_trace(unsigned long long* dev_buf) {
    g_trace_buf = dev_buf;
    return 0;
}

extern "C" int mm_gemm_timing(int mode, double* flops, float* ms, int* launches) {
    if (mode == 1) {
        if (!g_timing.buf) {
            g_timing.cap = 1 << 14;
            MM_CUDA_TRY(cudaMalloc(&g_timing.buf, 2 * g_timing.cap * sizeof(unsigned long long)));
        }
        MM_CUDA_TRY(cudaMemset(g_timing.buf, 0xff, g_timing.cap * sizeof(unsigned long long)));
        MM_CUDA_TRY(cudaMemset(g_timing.buf + g_timing.cap, 0, g_timing.cap * sizeof(unsigned long long)));
        g_timing.on = true;
        g_timing.used = 0;
        g_timing.flops.clear();
        g_timing.shape.clear();
        return 0;
    }
    // mode 0: stop; the caller has synchronised the launches' stream
    g_timing.on = false;
    double f = 0, t_ns = 0;
    if (g_timing.used) {
        std::vector<unsigned long long> h(2 * g_timing.cap);
        MM_CUDA_TRY(cudaMemcpy(h.data(), g_timing.buf, h.size() * sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < g_timing.used; ++i) {
            const unsigned long long lo = h[i], hi = h[g_timing.cap + i];
            if (hi > lo) t_ns += double(hi - lo);
            f += g_timing.flops[i];
        }
    }
    if (flops) *flops = f;
    if (ms) *ms = static_cast<float>(t_ns * 1e-6);
    if (launches) *launches = static_cast<int>(g_timing.used);
    return 0;
}

// diagnostics: the spans (ns, %globaltimer) of the launches recorded since the
// last mm_gemm_timing(1), after mm_gemm_timing(0): lo[i], hi[i], flops[i] and
// shape[4 i .. 4 i + 3] = m, n, k of the first problem, problems in the launch
extern "C" int mm_gemm_spans(int max, unsigned long long* lo, unsigned long long* hi, double* flops,
                             int* shape, int* count) {
    const int n = static_cast<int>(std::min<size_t>(g_timing.used, static_cast<size_t>(max)));
    if (n > 0) {
        MM_CUDA_TRY(cudaMemcpy(lo, g_timing.buf, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
        MM_CUDA_TRY(cudaMemcpy(hi, g_timing.buf + g_timing.cap, n * sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost));
        for (int i = 0; i < n; ++i) {
            flops[i] = g_timing.flops[i];
            for (int j = 0; j < 4; ++j) shape[4 * i + j] = g_timing.shape[4 * i + j];
        }
    }
    *count = n;
    return 0;
}

extern "C" int mm_gemm(const mm_gemm_args* a, void* stream) {
    if (int st = check_args(a)) return st;
    return run_group<1>(&a, 1, mm::as_stream(stream));
}

extern "C" int mm_gemm_grouped(const mm_gemm_args* probs, int n, void* stream) {
    MM_CHECK_ARG(probs != nullptr && n >= 0, "bad problem list");
    if (n == 0) return 0;
    for (int i = 0; i < n; ++i) {
        if (int st = check_args(&probs[i])) return st;
        MM_CHECK_ARG(probs[i].epilogue != MM_EPI_F32_RESID_LN, "fused LayerNorm GEMMs are not grouped");
        MM_CHECK_ARG(probs[i].a_kmajor == probs[0].a_kmajor && probs[i].b_kmajor == probs[0].b_kmajor,
                     "grouped GEMM: problem %d operand majorness differs from problem 0", i);
    }
    const mm_gemm_args* ptrs[kMaxProbs];
    for (int i0 = 0; i0 < n; i0 += kMaxProbs) {
        const int cnt = std::min(kMaxProbs, n - i0);
        for (int i = 0; i < cnt; ++i) ptrs[i] = &probs[i0 + i];
        if (int st = cnt == 1 ? run_group<1>(ptrs, 1, mm::as_stream(stream))
                              : run_group<kMaxProbs>(ptrs, cnt, mm::as_stream(stream)))
            return st;
    }
    return 0;
}
