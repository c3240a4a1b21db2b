// Algorithm 1 on the device: the emulated multi-device sync (the literal
// sync_step of syncsim.py:121-153 with every "device" resident in this GPU's
// HBM) and K3, the fused masked-rescale + loss-unscale + Adam + bf16 cast.
//
// Both are HBM-bound streaming kernels over flat per-module fp32 buckets:
// 128-bit loads/stores (float4), several independent vectors in flight per
// thread, one CTA per fixed-size chunk of a module, descriptor tables passed
// by value in the kernel parameter space (no H2D copy, CUDA-graph friendly).
#include <cuda_bf16.h>

#include <vector>

#include "mm_common.h"
#include "adam.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kVecPerThread = 4;                               // float4s in flight
constexpr int64_t kChunk = int64_t(kThreads) * kVecPerThread * 4 * 4;  // 16384 elems

// ---------------------------------------------------------------------------
// emulated sync

constexpr int kSyncMaxMods = 32;  // kernel-parameter table: 32 x 296 B

struct SyncTable {
    mm_sync_module mod[kSyncMaxMods];
    int64_t chunk_begin[kSyncMaxMods + 1];  // prefix of chunk counts
    int n_mods;
    int only_ready;
};

__device__ __forceinline__ int find_module(const int64_t* begin, int n, int64_t chunk) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {  // last m with begin[m] <= chunk
        int mid = (lo + hi + 1) >> 1;
        if (begin[mid] <= chunk) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__global__ void __launch_bounds__(kThreads) sync_emulated_kernel(const __grid_constant__ SyncTable t) {
    pdl_wait();
    const int64_t chunk = blockIdx.x;
    const int m = find_module(t.chunk_begin, t.n_mods, chunk);
    MM_DCHECK(m >= 0 && m < t.n_mods && chunk < t.chunk_begin[m + 1]);
    const mm_sync_module& md = t.mod[m];
    const int g = md.group_size;
    const int n = __popc(md.used_mask);
    const int64_t base = (chunk - t.chunk_begin[m]) * kChunk;
    const int64_t end = min(base + kChunk, md.n_elems);
    if (n == 0) {  // untouched buffers, zero synced copy (syncsim.py:143-145)
        if (md.out) for (int64_t i = base + threadIdx.x; i < end; i += kThreads) md.out[i] = 0.f;
        return;
    }
    uint32_t take = t.only_ready ? md.used_mask : ((g >= 32) ? 0xffffffffu : ((1u << g) - 1u));
    const float fn = (float)n;
    const bool vec_ok = ((md.n_elems & 3) == 0);
    if (vec_ok) {
        const int64_t v0 = base >> 2, v1 = end >> 2;
        for (int64_t v = v0 + threadIdx.x; v < v1; v += kThreads * kVecPerThread) {
            float4 acc[kVecPerThread];
#pragma unroll
            for (int u = 0; u < kVecPerThread; ++u) acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
            // ascending member order, fp32 adds starting from +0: the exact
            // sequence numpy performs in `total += dev.buffers[key]`
            for (int r = 0; r < g; ++r) {
                if (!((take >> r) & 1u)) continue;
                const float4* src = reinterpret_cast<const float4*>(md.bufs[r]);
#pragma unroll
                for (int u = 0; u < kVecPerThread; ++u) {
                    const int64_t vi = v + int64_t(u) * kThreads;
                    if (vi < v1) {
                        float4 x = __ldcs(src + vi);
                        acc[u].x += x.x; acc[u].y += x.y; acc[u].z += x.z; acc[u].w += x.w;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < kVecPerThread; ++u) {
                const int64_t vi = v + int64_t(u) * kThreads;
                if (vi >= v1) continue;
                float4 y;
                y.x = __fdiv_rn(acc[u].x, fn); y.y = __fdiv_rn(acc[u].y, fn);
                y.z = __fdiv_rn(acc[u].z, fn); y.w = __fdiv_rn(acc[u].w, fn);
                for (int r = 0; r < g; ++r) __stcs(reinterpret_cast<float4*>(md.bufs[r]) + vi, y);
                if (md.out) __stcs(reinterpret_cast<float4*>(md.out) + vi, y);
            }
        }
    } else {
        for (int64_t i = base + threadIdx.x; i < end; i += kThreads) {
            float acc = 0.f;
            for (int r = 0; r < g; ++r)
                if ((take >> r) & 1u) acc += md.bufs[r][i];
            const float y = __fdiv_rn(acc, fn);
            for (int r = 0; r < g; ++r) md.bufs[r][i] = y;
            if (md.out) md.out[i] = y;
        }
    }
}

// fp64 buffers (the reference's default DeviceState dtype, syncsim.py:103-106):
// the same chunk table, member pointers addressing doubles; 16-byte double2
// accesses, IEEE double adds in ascending member order and __ddiv_rn
__global__ void __launch_bounds__(kThreads) sync_emulated_f64_kernel(const __grid_constant__ SyncTable t) {
    pdl_wait();
    const int64_t chunk = blockIdx.x;
    const int m = find_module(t.chunk_begin, t.n_mods, chunk);
    const mm_sync_module& md = t.mod[m];
    double* const* bufs = reinterpret_cast<double* const*>(md.bufs);
    double* out = reinterpret_cast<double*>(md.out);
    const int g = md.group_size;
    const int n = __popc(md.used_mask);
    const int64_t base = (chunk - t.chunk_begin[m]) * kChunk;
    const int64_t end = min(base + kChunk, md.n_elems);
    if (n == 0) {
        if (out) for (int64_t i = base + threadIdx.x; i < end; i += kThreads) out[i] = 0.0;
        return;
    }
    const uint32_t take = t.only_ready ? md.used_mask : ((g >= 32) ? 0xffffffffu : ((1u << g) - 1u));
    const double fn = static_cast<double>(n);
    if ((md.n_elems & 1) == 0) {
        const int64_t v0 = base >> 1, v1 = end >> 1;
        for (int64_t v = v0 + threadIdx.x; v < v1; v += kThreads) {
            double2 acc = make_double2(0.0, 0.0);
            for (int r = 0; r < g; ++r) {
                if (!((take >> r) & 1u)) continue;
                const double2 x = __ldcs(reinterpret_cast<const double2*>(bufs[r]) + v);
                acc.x = __dadd_rn(acc.x, x.x);
                acc.y = __dadd_rn(acc.y, x.y);
            }
            const double2 y = make_double2(__ddiv_rn(acc.x, fn), __ddiv_rn(acc.y, fn));
            for (int r = 0; r < g; ++r) __stcs(reinterpret_cast<double2*>(bufs[r]) + v, y);
            if (out) __stcs(reinterpret_cast<double2*>(out) + v, y);
        }
    } else {
        for (int64_t i = base + threadIdx.x; i < end; i += kThreads) {
            double acc = 0.0;
            for (int r = 0; r < g; ++r)
                if ((take >> r) & 1u) acc = __dadd_rn(acc, bufs[r][i]);
            const double y = __ddiv_rn(acc, fn);
            for (int r = 0; r < g; ++r) bufs[r][i] = y;
            if (out) out[i] = y;
        }
    }
}

// ---------------------------------------------------------------------------
// K3 fused update

constexpr int kAdamMaxMods = 96;

struct AdamTable {
    mm_adam_module mod[kAdamMaxMods];
    int64_t chunk_begin[kAdamMaxMods + 1];
    mm_adam_hyper hp;
    const int32_t* ready_dev;
    int n_mods;
};

__global__ void __launch_bounds__(kThreads) fused_update_kernel(const __grid_constant__ AdamTable t) {
    pdl_wait();
    const int64_t n_chunks = t.chunk_begin[t.n_mods];
    for (int64_t chunk = blockIdx.x; chunk < n_chunks; chunk += gridDim.x) {
    const int mi = find_module(t.chunk_begin, t.n_mods, chunk);
    const mm_adam_module& md = t.mod[mi];
    int n = md.n_ready;
    if (t.ready_dev != nullptr && md.ready_index >= 0) n = t.ready_dev[md.ready_index];
    if (n <= 0) continue;  // unused everywhere: no reduction, no optimizer step
    // g = sum / n * inv_loss_scale, the rescale of Algorithm 1 fused here
    const float fn = (float)n;
    const float unscale = t.hp.inv_loss_scale;
    const bool zero_grad = t.hp.zero_grad != 0;
    const int64_t base = (chunk - t.chunk_begin[mi]) * kChunk;
    const int64_t end = min(base + kChunk, md.n_elems);
    const float ss = md.step_size, isb = md.inv_sqrt_bc2;
    if ((md.n_elems & 3) == 0) {
        const int64_t v0 = base >> 2, v1 = end >> 2;
        const float4* G = reinterpret_cast<const float4*>(md.grad);
        float4* G0 = reinterpret_cast<float4*>(md.grad);
        float4* P = reinterpret_cast<float4*>(md.master);
        float4* M = reinterpret_cast<float4*>(md.exp_avg);
        float4* V = reinterpret_cast<float4*>(md.exp_avg_sq);
        uint2* B = reinterpret_cast<uint2*>(md.param_bf16);
        for (int64_t v = v0 + threadIdx.x; v < v1; v += kThreads * 2) {
            float4 g[2], p[2], m[2], s[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int64_t vi = v + int64_t(u) * kThreads;
                if (vi < v1) {
                    g[u] = __ldcs(G + vi); p[u] = __ldcs(P + vi);
                    m[u] = __ldcs(M + vi); s[u] = __ldcs(V + vi);
                }
            }

#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int64_t vi = v + int64_t(u) * kThreads;
                if (vi >= v1) continue;
                adam_elem(adam_grad(g[u].x, fn, unscale), p[u].x, m[u].x, s[u].x, ss, isb, t.hp);
                adam_elem(adam_grad(g[u].y, fn, unscale), p[u].y, m[u].y, s[u].y, ss, isb, t.hp);
                adam_elem(adam_grad(g[u].z, fn, unscale), p[u].z, m[u].z, s[u].z, ss, isb, t.hp);
                adam_elem(adam_grad(g[u].w, fn, unscale), p[u].w, m[u].w, s[u].w, ss, isb, t.hp);
                __stcs(P + vi, p[u]); __stcs(M + vi, m[u]); __stcs(V + vi, s[u]);
                if (zero_grad) __stcs(G0 + vi, make_float4(0.f, 0.f, 0.f, 0.f));  // lazy zeroing
                if (B) {
                    uint2 b;
                    b.x = pack_bf16x2(p[u].x, p[u].y);
                    b.y = pack_bf16x2(p[u].z, p[u].w);
                    B[vi] = b;
                }
            }
        }
    } else {
        for (int64_t i = base + threadIdx.x; i < end; i += kThreads) {
            float p = md.master[i], m = md.exp_avg[i], s = md.exp_avg_sq[i];
            const float gi = md.grad[i];
            if (zero_grad) md.grad[i] = 0.f;
            adam_elem(adam_grad(gi, fn, unscale), p, m, s, ss, isb, t.hp);
            md.master[i] = p; md.exp_avg[i] = m; md.exp_avg_sq[i] = s;
            if (md.param_bf16) {
                __nv_bfloat16 h = __float2bfloat16_rn(p);
                md.param_bf16[i] = *reinterpret_cast<uint16_t*>(&h);
            }
        }
    }
}  // chunk loop
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

__global__ void axpy_kernel(float* __restrict__ y, const float* __restrict__ x, float alpha,
                            int64_t n) {
    pdl_wait();
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        y[i] = fmaf(alpha, x[i], y[i]);
}

__global__ void axpy_f64_kernel(double* __restrict__ y, const double* __restrict__ x, double alpha,
                                int64_t n) {
    pdl_wait();
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        y[i] = fma(alpha, x[i], y[i]);
}

}  // namespace

static int sync_emulated(const mm_sync_module* mods, int n_mods, int only_ready, bool f64,
                         void* stream) {
    MM_CHECK_ARG(n_mods >= 0 && (n_mods == 0 || mods), "bad module table");
    for (int base = 0; base < n_mods; base += kSyncMaxMods) {
        SyncTable t{};
        t.n_mods = std::min(kSyncMaxMods, n_mods - base);
        t.only_ready = only_ready;
        int64_t chunks = 0;
        for (int i = 0; i < t.n_mods; ++i) {
            const mm_sync_module& md = mods[base + i];
            MM_CHECK_ARG(md.group_size >= 1 && md.group_size <= MM_MAX_SYNC_GROUP,
                         "module %d: group size %d outside [1,%d]", base + i, md.group_size,
                         MM_MAX_SYNC_GROUP);
            MM_CHECK_ARG(md.n_elems >= 0, "module %d: negative size", base + i);
            MM_CHECK_ARG(md.group_size == 32 || (md.used_mask >> md.group_size) == 0, "module %d: used bit beyond group",
                         base + i);
            mm_sync_module c = md;
            const int64_t vmask = f64 ? 1 : 3;  // elements per 16-byte vector - 1
            bool vec = (md.n_elems & vmask) == 0 && (md.out == nullptr || aligned16(md.out));
            for (int r = 0; r < md.group_size; ++r) {
                MM_CHECK_ARG(md.bufs[r] != nullptr, "module %d: NULL member buffer", base + i);
                vec = vec && aligned16(md.bufs[r]);
            }
            // the kernel takes the float4 path iff n_elems % 4 == 0, which needs
            // 16-byte aligned buffers (torch allocations are 256-byte aligned)
            MM_CHECK_ARG(vec || (md.n_elems & vmask) != 0,
                         "module %d: buffers must be 16-byte aligned", base + i);
            t.mod[i] = c;
            t.chunk_begin[i] = chunks;
            chunks += (md.n_elems + kChunk - 1) / kChunk;
        }
        t.chunk_begin[t.n_mods] = chunks;
        if (chunks == 0) continue;
        MM_CUDA_TRY(mm::launch_pdl(f64 ? sync_emulated_f64_kernel : sync_emulated_kernel,
                                   dim3((unsigned)chunks), dim3(kThreads), 0, mm::as_stream(stream), t));
        MM_LAUNCH_CHECK(f64 ? "sync_emulated_f64_kernel" : "sync_emulated_kernel");
    }
    return 0;
}

extern "C" int mm_sync_emulated(const mm_sync_module* mods, int n_mods, int only_ready,
                                void* stream) {
    return sync_emulated(mods, n_mods, only_ready, false, stream);
}

extern "C" int mm_sync_emulated_f64(const mm_sync_module* mods, int n_mods, int only_ready,
                                    void* stream) {
    return sync_emulated(mods, n_mods, only_ready, true, stream);
}

extern "C" int mm_fused_update(const mm_adam_module* mods, int n_mods, const mm_adam_hyper* hyper,
                               const int32_t* ready_dev, void* stream) {
    MM_CHECK_ARG(hyper != nullptr, "hyper is NULL");
    MM_CHECK_ARG(n_mods >= 0 && (n_mods == 0 || mods), "bad module table");
    for (int base = 0; base < n_mods; base += kAdamMaxMods) {
        AdamTable t{};
        t.hp = *hyper;
        t.ready_dev = ready_dev;
        int used = 0;
        int64_t chunks = 0;
        for (int i = base; i < std::min(n_mods, base + kAdamMaxMods); ++i) {
            const mm_adam_module& md = mods[i];
            MM_CHECK_ARG(md.grad && md.master && md.exp_avg && md.exp_avg_sq,
                         "module %d: NULL state pointer", i);
            const bool vec = aligned16(md.grad) && aligned16(md.master) &&
                             aligned16(md.exp_avg) && aligned16(md.exp_avg_sq) &&
                             (md.param_bf16 == nullptr ||
                              (reinterpret_cast<uintptr_t>(md.param_bf16) & 7u) == 0);
            MM_CHECK_ARG(vec || (md.n_elems & 3) != 0, "module %d: misaligned buckets", i);
            // host-known n == 0 modules cost nothing: drop them from the table
            if ((ready_dev == nullptr || md.ready_index < 0) && md.n_ready <= 0) continue;
            if (md.n_elems <= 0) continue;
            t.mod[used] = md;
            t.chunk_begin[used] = chunks;
            chunks += (md.n_elems + kChunk - 1) / kChunk;
            ++used;
        }
        t.n_mods = used;
        t.chunk_begin[used] = chunks;
        if (chunks == 0) continue;
        const int64_t grid = hyper->max_ctas > 0 ? std::min<int64_t>(chunks, hyper->max_ctas) : chunks;
        MM_CUDA_TRY(mm::launch_pdl(fused_update_kernel, dim3((unsigned)grid), dim3(kThreads), 0,
                                   mm::as_stream(stream), t));
        MM_LAUNCH_CHECK("fused_update_kernel");
    }
    return 0;
}

extern "C" int mm_flush_l2(void* scratch, size_t bytes, void* stream) {
    MM_CUDA_TRY(cudaMemsetAsync(scratch, (int)(bytes & 0xff) ^ 0x5a, bytes, mm::as_stream(stream)));
    return 0;
}

extern "C" int mm_axpy_f32(float* y, const float* x, float alpha, int64_t n, void* stream) {
    MM_CHECK_ARG((y && x) || n == 0, "NULL pointer");
    if (n == 0) return 0;
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 8 * mm::num_sms()));
    MM_CUDA_TRY(mm::launch_pdl(axpy_kernel, dim3(grid), dim3(256), 0, mm::as_stream(stream), y, x,
                               alpha, n));
    MM_LAUNCH_CHECK("axpy_kernel");
    return 0;
}

extern "C" int mm_axpy_f64(double* y, const double* x, double alpha, int64_t n, void* stream) {
    MM_CHECK_ARG((y && x) || n == 0, "NULL pointer");
    if (n == 0) return 0;
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 8 * mm::num_sms()));
    MM_CUDA_TRY(mm::launch_pdl(axpy_f64_kernel, dim3(grid), dim3(256), 0, mm::as_stream(stream), y, x,
                               alpha, n));
    MM_LAUNCH_CHECK("axpy_f64_kernel");
    return 0;
}

extern "C" int mm_memset(void* ptr, int value, size_t bytes, void* stream) {
    MM_CHECK_ARG(ptr != nullptr || bytes == 0, "NULL pointer");
    if (bytes == 0) return 0;
    MM_CUDA_TRY(cudaMemsetAsync(ptr, value, bytes, mm::as_stream(stream)));
    return 0;
}
