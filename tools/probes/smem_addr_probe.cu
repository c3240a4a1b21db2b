// Probe: numeric form of shared::cta (cvta) and shared::cluster (mapa)
// addresses in a 4-CTA cluster.  nvcc -gencode arch=compute_100a,code=sm_100a -o p smem_addr_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __cluster_dims__(4, 1, 1) probe(unsigned* out) {
    __shared__ unsigned long long bar[4];
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    const unsigned local = static_cast<unsigned>(__cvta_generic_to_shared(&bar[1]));
    if (threadIdx.x == 0) {
        out[r * 8 + 0] = r;
        out[r * 8 + 1] = local;
        for (unsigned t = 0; t < 4; ++t) {
            unsigned m;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(m) : "r"(local), "r"(t));
            out[r * 8 + 2 + t] = m;
        }
    }
}
int main() {
    unsigned* d; cudaMalloc(&d, 4 * 8 * sizeof(unsigned));
    cudaMemset(d, 0, 4 * 8 * sizeof(unsigned));
    probe<<<4, 32>>>(d);
    unsigned h[32]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    for (int r = 0; r < 4; ++r)
        printf("rank %u local %08x mapa0 %08x mapa1 %08x mapa2 %08x mapa3 %08x\n", h[r*8], h[r*8+1], h[r*8+2], h[r*8+3], h[r*8+4], h[r*8+5]);
}
