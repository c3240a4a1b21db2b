// Option B of the module exchange: K2 + K3 + the parameter
// all-gather fused into one HBM/NVLink streaming kernel over peer memory,
// plus the flag barrier that orders it against the other ranks and the CUDA
// IPC plumbing that maps the peers' buckets.
//
// Algorithm 1 (syncsim.py:121-153) per module of group
// size g: member r owns the contiguous shard r, sums the READY members'
// gradients over it (masked peer loads, ascending member order -- the exact
// fp32 sequence of `total += dev.buffers[key]`), divides by n, runs Adam on
// its own master/moment shard and stores the new bf16 weights into every
// member's weight bucket.  Per element that is n*4 B of (mostly NVLink)
// reads, 24 B of local optimizer state traffic and g*2 B of weight stores --
// versus 2(g-1)/g*4 B on the wire plus 30 B locally for each of the g
// members with NCCL all-reduce + a replicated update.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "adam.cuh"
#include "mm_common.h"

namespace {

constexpr int kThreads = 256;
constexpr int kUnroll = 1;  // float4s per thread per member: 1 + 4 CTAs/SM beat 2 + 2 (r01: 3.92 vs 4.46 ms)
constexpr int64_t kChunk = int64_t(kThreads) * kUnroll * 4 * 8;  // 8192 elements per CTA
constexpr int kPeerMaxShards = 112;  // 112 * (248 + 8 + 1) B < 32 KB of kernel parameters

struct PeerTable {
    mm_peer_shard sh[kPeerMaxShards];
    int64_t chunk_begin[kPeerMaxShards + 1];
    mm_adam_hyper hp;
    int n;
    uint8_t vec[kPeerMaxShards];
};

__device__ __forceinline__ int find_shard(const int64_t* begin, int n, int64_t chunk) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (begin[mid] <= chunk) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ void add4(float4& a, const float4& x) {
    a.x += x.x; a.y += x.y; a.z += x.z; a.w += x.w;
}

__global__ void __launch_bounds__(kThreads, 4) peer_update_kernel(const __grid_constant__ PeerTable t) {
    pdl_wait();
    const int64_t n_chunks = t.chunk_begin[t.n];
    const float unscale = t.hp.inv_loss_scale;
    const bool zero_grad = t.hp.zero_grad != 0;
    for (int64_t chunk = blockIdx.x; chunk < n_chunks; chunk += gridDim.x) {
        const int si = find_shard(t.chunk_begin, t.n, chunk);
        const mm_peer_shard& sh = t.sh[si];
        const int g = sh.group_size;
        const uint32_t mask = sh.ready_mask;
        const float fn = (float)__popc(mask);
        const float ss = sh.step_size, isb = sh.inv_sqrt_bc2;
        const int64_t base = sh.begin + (chunk - t.chunk_begin[si]) * kChunk;
        const int64_t end = min(base + kChunk, sh.end);
        if (t.vec[si]) {
            const int64_t v0 = base >> 2, v1 = end >> 2;
            float4* P = reinterpret_cast<float4*>(sh.master);
            float4* M = reinterpret_cast<float4*>(sh.exp_avg);
            float4* V = reinterpret_cast<float4*>(sh.exp_avg_sq);
            for (int64_t v = v0 + threadIdx.x; v < v1; v += kThreads * kUnroll) {
                // issue every ready member's loads before the first add: up to
                // 8 members x 2 float4 of peer reads in flight per thread
                float4 x[MM_MAX_GROUP][kUnroll];
#pragma unroll
                for (int r = 0; r < MM_MAX_GROUP; ++r) {
                    if (r >= g || !((mask >> r) & 1u)) continue;
                    const float4* src = reinterpret_cast<const float4*>(sh.grad[r]);
#pragma unroll
                    for (int u = 0; u < kUnroll; ++u) {
                        const int64_t vi = v + int64_t(u) * kThreads;
                        if (vi < v1) x[r][u] = __ldcs(src + vi);
                    }
                }
                float4 p[kUnroll], m[kUnroll], s[kUnroll];
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    const int64_t vi = v + int64_t(u) * kThreads;
                    if (vi < v1) { p[u] = __ldcs(P + vi); m[u] = __ldcs(M + vi); s[u] = __ldcs(V + vi); }
                }
                if (zero_grad) {
#pragma unroll
                    for (int r = 0; r < MM_MAX_GROUP; ++r) {
                        if (r >= g || !((mask >> r) & 1u)) continue;
                        float4* dst = reinterpret_cast<float4*>(sh.grad[r]);
#pragma unroll
                        for (int u = 0; u < kUnroll; ++u) {
                            const int64_t vi = v + int64_t(u) * kThreads;
                            if (vi < v1) __stcs(dst + vi, make_float4(0.f, 0.f, 0.f, 0.f));
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    const int64_t vi = v + int64_t(u) * kThreads;
                    if (vi >= v1) continue;
                    // ascending member order from +0 (syncsim.py:146-148)
                    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                    for (int r = 0; r < MM_MAX_GROUP; ++r)
                        if (r < g && ((mask >> r) & 1u)) add4(acc, x[r][u]);
                    // total / n * inv_loss_scale: the rounding sequence of
                    // sync_emulated + fused_update(n_ready = 1) (x / 1 is exact)
                    adam_elem(adam_grad(acc.x, fn, unscale), p[u].x, m[u].x, s[u].x, ss, isb, t.hp);
                    adam_elem(adam_grad(acc.y, fn, unscale), p[u].y, m[u].y, s[u].y, ss, isb, t.hp);
                    adam_elem(adam_grad(acc.z, fn, unscale), p[u].z, m[u].z, s[u].z, ss, isb, t.hp);
                    adam_elem(adam_grad(acc.w, fn, unscale), p[u].w, m[u].w, s[u].w, ss, isb, t.hp);
                    __stcs(P + vi, p[u]); __stcs(M + vi, m[u]); __stcs(V + vi, s[u]);
                    uint2 b;
                    b.x = pack_bf16x2(p[u].x, p[u].y);
                    b.y = pack_bf16x2(p[u].z, p[u].w);
#pragma unroll
                    for (int r = 0; r < MM_MAX_GROUP; ++r) {
                        if (r >= g) continue;
                        if (sh.param[r]) __stcs(reinterpret_cast<uint2*>(sh.param[r]) + vi, b);
                        if (sh.master_copy[r]) __stcs(reinterpret_cast<float4*>(sh.master_copy[r]) + vi, p[u]);
                    }
                }
            }
        } else {
            for (int64_t i = base + threadIdx.x; i < end; i += kThreads) {
                float acc = 0.f;
                for (int r = 0; r < g; ++r) {
                    if (!((mask >> r) & 1u)) continue;
                    acc += sh.grad[r][i];
                    if (zero_grad) sh.grad[r][i] = 0.f;
                }
                float p = sh.master[i], m = sh.exp_avg[i], s = sh.exp_avg_sq[i];
                adam_elem(adam_grad(acc, fn, unscale), p, m, s, ss, isb, t.hp);
                sh.master[i] = p; sh.exp_avg[i] = m; sh.exp_avg_sq[i] = s;
                __nv_bfloat16 h = __float2bfloat16_rn(p);
                const uint16_t hb = *reinterpret_cast<uint16_t*>(&h);
                for (int r = 0; r < g; ++r) {
                    if (sh.param[r]) sh.param[r][i] = hb;
                    if (sh.master_copy[r]) sh.master_copy[r][i] = p;
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// flag barrier over peer memory

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void __launch_bounds__(32) peer_barrier_kernel(const __grid_constant__ mm_peer_signal s) {
    pdl_wait();  // every earlier kernel of this stream has completed and flushed
    const int i = threadIdx.x;
    if (i < s.n_peers) {
        // order this rank's earlier writes (previous kernels, stream order)
        // before the signal at system scope, then publish the epoch
        __threadfence_system();
        st_release_sys(s.peer_flags[i] + s.my_rank, s.epoch);
        const uint32_t* f = s.local_flags + s.peer_rank[i];
        const uint64_t t0 = globaltimer_ns();
        while ((int32_t)(ld_acquire_sys(f) - s.epoch) < 0) {
            __nanosleep(128);
            if (s.timeout_ms > 0 && globaltimer_ns() - t0 > uint64_t(s.timeout_ms) * 1000000ull) {
                printf("mm_peer_barrier: rank %d timed out waiting for rank %d (epoch %u)\n",
                       s.my_rank, s.peer_rank[i], s.epoch);
                __trap();
            }
        }
    }
    __syncthreads();
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ---------------------------------------------------------------------------
// CUDA IPC mappings, refcounted per exported allocation

struct IpcMap {
    std::mutex mu;
    std::map<std::string, std::pair<void*, int>> by_handle;  // handle -> (base, refs)
    std::map<void*, std::pair<std::string, int>> handle_of;  // returned ptr -> (handle, count)
};
IpcMap& ipc() {
    static IpcMap m;
    return m;
}

using AddrRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
AddrRangeFn addr_range_fn() {
    static AddrRangeFn fn = [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess && q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<AddrRangeFn>(ptr);
        return AddrRangeFn(nullptr);
    }();
    return fn;
}

}  // namespace

extern "C" int64_t mm_peer_shard_begin(int64_t n_elems, int group_size, int member) {
    if (group_size < 1 || member < 0 || n_elems < 0) return -1;
    int64_t s = (n_elems + group_size - 1) / group_size;
    s = (s + 3) & ~int64_t(3);
    return std::min<int64_t>(n_elems, s * member);
}

extern "C" int mm_peer_update(const mm_peer_shard* shards, int n, const mm_adam_hyper* hyper,
                              void* stream) {
    MM_CHECK_ARG(hyper != nullptr, "hyper is NULL");
    MM_CHECK_ARG(n >= 0 && (n == 0 || shards), "bad shard table");
    for (int base = 0; base < n; base += kPeerMaxShards) {
        PeerTable t{};
        t.hp = *hyper;
        int used = 0;
        int64_t chunks = 0;
        for (int i = base; i < std::min(n, base + kPeerMaxShards); ++i) {
            const mm_peer_shard& sh = shards[i];
            MM_CHECK_ARG(sh.group_size >= 1 && sh.group_size <= MM_MAX_GROUP,
                         "shard %d: group size %d outside [1,%d]", i, sh.group_size, MM_MAX_GROUP);
            MM_CHECK_ARG((sh.ready_mask >> sh.group_size) == 0, "shard %d: ready bit beyond group", i);
            MM_CHECK_ARG(0 <= sh.begin && sh.begin <= sh.end, "shard %d: bad range", i);
            MM_CHECK_ARG(sh.master && sh.exp_avg && sh.exp_avg_sq, "shard %d: NULL optimizer state", i);
            if (sh.ready_mask == 0 || sh.end == sh.begin) continue;  // n = 0: no step at all
            bool vec = (sh.begin & 3) == 0 && (sh.end & 3) == 0 && aligned16(sh.master) &&
                       aligned16(sh.exp_avg) && aligned16(sh.exp_avg_sq);
            for (int r = 0; r < sh.group_size; ++r) {
                const bool ready = (sh.ready_mask >> r) & 1u;
                MM_CHECK_ARG(!ready || sh.grad[r], "shard %d: NULL gradient of ready member %d", i, r);
                if (ready) vec = vec && aligned16(sh.grad[r]);
                if (sh.param[r]) vec = vec && ((reinterpret_cast<uintptr_t>(sh.param[r]) & 7u) == 0);
                if (sh.master_copy[r]) vec = vec && aligned16(sh.master_copy[r]);
            }
            t.sh[used] = sh;
            t.vec[used] = vec ? 1 : 0;
            t.chunk_begin[used] = chunks;
            chunks += (sh.end - sh.begin + kChunk - 1) / kChunk;
            ++used;
        }
        t.n = used;
        t.chunk_begin[used] = chunks;
        if (chunks == 0) continue;
        const int64_t grid = hyper->max_ctas > 0 ? std::min<int64_t>(chunks, hyper->max_ctas) : chunks;
        MM_CUDA_TRY(mm::launch_pdl(peer_update_kernel, dim3((unsigned)grid), dim3(kThreads), 0,
                                   mm::as_stream(stream), t));
        MM_LAUNCH_CHECK("peer_update_kernel");
    }
    return 0;
}

extern "C" int mm_peer_barrier(const mm_peer_signal* sig, void* stream) {
    MM_CHECK_ARG(sig != nullptr, "signal is NULL");
    MM_CHECK_ARG(sig->n_peers >= 0 && sig->n_peers <= MM_PEER_MAX_RANKS, "n_peers %d outside [0,%d]",
                 sig->n_peers, MM_PEER_MAX_RANKS);
    MM_CHECK_ARG(sig->my_rank >= 0 && sig->my_rank < MM_PEER_MAX_RANKS, "my_rank %d", sig->my_rank);
    if (sig->n_peers == 0) return 0;
    MM_CHECK_ARG(sig->local_flags != nullptr, "local_flags is NULL");
    for (int i = 0; i < sig->n_peers; ++i) {
        MM_CHECK_ARG(sig->peer_flags[i] != nullptr, "peer %d: NULL flag array", i);
        MM_CHECK_ARG(sig->peer_rank[i] >= 0 && sig->peer_rank[i] < MM_PEER_MAX_RANKS &&
                         sig->peer_rank[i] != sig->my_rank,
                     "peer %d: bad rank %d", i, sig->peer_rank[i]);
    }
    MM_CUDA_TRY(mm::launch_pdl(peer_barrier_kernel, dim3(1), dim3(32), 0, mm::as_stream(stream),
                               *sig));
    MM_LAUNCH_CHECK("peer_barrier_kernel");
    return 0;
}

extern "C" int mm_ipc_export(const void* ptr, uint8_t handle[64], uint64_t* offset) {
    MM_CHECK_ARG(ptr && handle && offset, "NULL argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    AddrRangeFn fn = addr_range_fn();
    if (!fn) {
        mm::set_error("cuMemGetAddressRange unavailable");
        return mm::kUnsupported;
    }
    CUdeviceptr base = 0;
    size_t size = 0;
    if (fn(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS) {
        mm::set_error("cuMemGetAddressRange failed for %p", ptr);
        return mm::kCuda;
    }
    cudaIpcMemHandle_t h;
    MM_CUDA_TRY(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
    std::memcpy(handle, &h, 64);
    *offset = reinterpret_cast<uintptr_t>(ptr) - base;
    return 0;
}

extern "C" int mm_ipc_import(const uint8_t handle[64], uint64_t offset, void** ptr) {
    MM_CHECK_ARG(handle && ptr, "NULL argument");
    IpcMap& m = ipc();
    std::lock_guard<std::mutex> lk(m.mu);
    std::string key(reinterpret_cast<const char*>(handle), 64);
    auto it = m.by_handle.find(key);
    if (it == m.by_handle.end()) {
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, 64);
        void* base = nullptr;
        MM_CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
        it = m.by_handle.emplace(key, std::make_pair(base, 0)).first;
    }
    it->second.second += 1;
    *ptr = static_cast<char*>(it->second.first) + offset;
    auto& ho = m.handle_of[*ptr];
    ho.first = key;
    ho.second += 1;
    return 0;
}

extern "C" int mm_ipc_release(void* ptr) {
    IpcMap& m = ipc();
    std::lock_guard<std::mutex> lk(m.mu);
    auto h = m.handle_of.find(ptr);
    MM_CHECK_ARG(h != m.handle_of.end(), "%p was not returned by mm_ipc_import", ptr);
    auto it = m.by_handle.find(h->second.first);
    if (--h->second.second == 0) m.handle_of.erase(h);
    if (it != m.by_handle.end() && --it->second.second == 0) {
        void* base = it->second.first;
        m.by_handle.erase(it);
        MM_CUDA_TRY(cudaIpcCloseMemHandle(base));
    }
    return 0;
}
