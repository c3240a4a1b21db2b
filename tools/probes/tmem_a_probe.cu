// Probe: tcgen05.mma with the A operand in TMEM (kind::f16, bf16).  A[128x16]
// is written to TMEM with tcgen05.st (lane m = row m, 32-bit column j = the
// bf16 pair (A[m][2j], A[m][2j+1]), low half first), B[32x16] sits in shared
// memory (K-major, SWIZZLE_128B), D[128x32] = A B^T is read back and checked
// on the host.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -o tmem_a_probe tmem_a_probe.cu
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3FFF);
    d |= uint64_t((16 >> 4) & 0x3FFF) << 16;
    d |= uint64_t((1024 >> 4) & 0x3FFF) << 32;
    d |= uint64_t(1) << 46;
    d |= uint64_t(2) << 61;
    return d;
}
__host__ __device__ constexpr uint32_t idesc(int m, int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}

__global__ void probe(const uint16_t* A, const uint16_t* B, float* D, int swap_halves) {
    __shared__ alignas(1024) uint8_t sB[32 * 128];
    __shared__ uint32_t slot;
    __shared__ alignas(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 32 * 8; i += 128) {  // 32 rows x 8 16-byte chunks
        const int n = i >> 3, c = i & 7;
        uint16_t v[8];
        for (int e = 0; e < 8; ++e) {
            const int k = c * 8 + e;
            v[e] = k < 16 ? B[n * 16 + k] : 0;
        }
        *reinterpret_cast<uint4*>(sB + n * 128 + ((c ^ (n & 7)) * 16)) = *reinterpret_cast<uint4*>(v);
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = slot;
    const int m = tid;
    uint32_t w[8];
    for (int j = 0; j < 8; ++j) {
        const uint32_t lo = A[m * 16 + 2 * j], hi = A[m * 16 + 2 * j + 1];
        w[j] = swap_halves ? (hi | (lo << 16)) : (lo | (hi << 16));
    }
    const uint32_t ta = tmem + (uint32_t(warp * 32) << 16);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta),
                 "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) {
        const uint32_t td = tmem + 32;
        const uint64_t bd = desc_sw128(smem_u32(sB));
        asm volatile(
            "{\n\t.reg .pred e;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 0;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%4];\n\t}" ::"r"(td),
            "r"(tmem), "l"(bd), "r"(idesc(128, 32)), "r"(smem_u32(&bar))
            : "memory");
    }
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
        "@!p bra WAIT;\n\t}" ::"r"(smem_u32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t v[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
          "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(tmem + 32 + (uint32_t(warp * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 32; ++j) D[m * 32 + j] = __uint_as_float(v[j]);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

static uint16_t f2bf(float f) {
    uint32_t u; memcpy(&u, &f, 4);
    return uint16_t((u + 0x7FFF + ((u >> 16) & 1)) >> 16);
}
static float bf2f(uint16_t h) { uint32_t u = uint32_t(h) << 16; float f; memcpy(&f, &u, 4); return f; }

int main() {
    std::vector<uint16_t> A(128 * 16), B(32 * 16);
    for (int i = 0; i < 128 * 16; ++i) A[i] = f2bf(std::sin(0.37f * i) );
    for (int i = 0; i < 32 * 16; ++i) B[i] = f2bf(std::cos(0.11f * i));
    uint16_t *dA, *dB; float* dD;
    cudaMalloc(&dA, A.size() * 2); cudaMalloc(&dB, B.size() * 2); cudaMalloc(&dD, 128 * 32 * 4);
    cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
    for (int swap = 0; swap < 2; ++swap) {
        cudaMemset(dD, 0, 128 * 32 * 4);
        probe<<<1, 128>>>(dA, dB, dD, swap);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        std::vector<float> D(128 * 32);
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        double maxerr = 0, maxref = 0;
        for (int m = 0; m < 128; ++m)
            for (int n = 0; n < 32; ++n) {
                double r = 0;
                for (int k = 0; k < 16; ++k) r += double(bf2f(A[m * 16 + k])) * bf2f(B[n * 16 + k]);
                maxerr = std::fmax(maxerr, std::fabs(r - D[m * 32 + n]));
                maxref = std::fmax(maxref, std::fabs(r));
            }
        printf("swap_halves=%d max|err| %.3e (max|ref| %.3e) -> %s\n", swap, maxerr, maxref,
               maxerr < 1e-3 * maxref ? "MATCH" : "mismatch");
    }
    return 0;
}
