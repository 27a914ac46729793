#include <cstdio>
#include <cuda_runtime.h>
__global__ void __cluster_dims__(4,1,1) k(unsigned long long *out) {
    extern __shared__ unsigned sm[];
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    if (threadIdx.x == 0) {
        for (unsigned q = 0; q < 4; ++q) {
            void *p;
            asm volatile("mapa.u64 %0, %1, %2;" : "=l"(p) : "l"((void*)sm), "r"(q));
            out[blockIdx.x * 8 + q] = (unsigned long long)p;
            unsigned sa;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(sa) : "r"((unsigned)__cvta_generic_to_shared(sm)), "r"(q));
            out[blockIdx.x * 8 + 4 + q] = sa;
        }
    }
}
int main() {
    unsigned long long *d, h[64];
    cudaMalloc(&d, sizeof(h));
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    k<<<8, 32, 200000>>>(d);
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    for (int b = 0; b < 8; ++b) { printf("blk %d:", b); for (int q = 0; q < 8; ++q) printf(" %llx", h[b*8+q]); printf("\n"); }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
