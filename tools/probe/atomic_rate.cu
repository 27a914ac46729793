// Same-address global atomicAdd (with return) throughput from every warp of the chip: one lane per warp,
// K dependent atomics each (the team path's list-counter pattern), against per-warp addresses.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ar tools/probe/atomic_rate.cu && /tmp/ar
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(512, 1) k(int *ctr, int iters, int spread, long long *out) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int *a = ctr + (spread ? warp * 32 : 0);
    long long t0 = clock64();
    int acc = 0;
    if ((threadIdx.x & 31) == 0)
        for (int i = 0; i < iters; ++i) acc += atomicAdd(a, 1 + (acc & 1));
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
    if (acc == -1) out[1] = acc;
}
int main() {
    int *ctr; long long *out;
    cudaMalloc(&ctr, 148 * 16 * 32 * 4); cudaMalloc(&out, 64);
    const int iters = 2000;
    for (int G : {1, 8, 37, 148})
        for (int spread : {0, 1}) {
            cudaMemset(ctr, 0, 148 * 16 * 32 * 4);
            k<<<G, 512>>>(ctr, iters, spread, out);
            cudaDeviceSynchronize();
            long long h = 0; cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
            const double total = (double)G * 16 * iters;
            printf("G=%3d %s: %.0f cycles per atomic per warp (latency), %.2f cycles per atomic chip-wide\n", G,
                   spread ? "per-warp addresses" : "one address      ", (double)h / iters, (double)h / total);
        }
    return 0;
}
