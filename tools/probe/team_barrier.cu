// Latency probe of the team barrier used by the cooperative (large-image) path:
// G CTAs x 512 threads, N back-to-back barriers (red.release arrive + ld.acquire poll).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tb tools/probe/team_barrier.cu && /tmp/tb
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512, 1) k(unsigned *bar, int *data, int n, int mode, long long *out) {
    __shared__ unsigned epoch;
    if (threadIdx.x == 0) epoch = 0;
    __syncthreads();
    const unsigned G = gridDim.x;
    long long t0 = clock64();
    int acc = 0;
    for (int i = 0; i < n; ++i) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned target = (epoch += 1u) * G;
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
            while (true) {
                unsigned c;
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(c) : "l"(bar) : "memory");
                if ((int)(c - target) >= 0) break;
            }
        }
        __syncthreads();
        if (mode == 1) acc += *reinterpret_cast<volatile int *>(data + (i & 3));   // the post-barrier count read
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
    if (acc == 12345) out[1] = acc;
}

int main() {
    unsigned *bar; int *data; long long *out;
    cudaMalloc(&bar, 256); cudaMalloc(&data, 256); cudaMalloc(&out, 64);
    const int n = 2000;
    for (int G : {2, 4, 8, 37, 74, 148}) {
        for (int mode : {0, 1}) {
            cudaMemset(bar, 0, 256); cudaMemset(data, 0, 256);
            void *args[] = {&bar, &data, (void *)&n, &mode, &out};
            cudaError_t e = cudaLaunchCooperativeKernel((void *)k, dim3(G), dim3(512), args, 0, 0);
            cudaDeviceSynchronize();
            long long h[2] = {0, 0};
            cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
            printf("G=%3d mode %d: %.0f cycles / barrier (%s)\n", G, mode, (double)h[0] / n, cudaGetErrorString(e));
        }
    }
    return 0;
}
