// Host-side dispatch over the fused HASF kernel variants (kernel body in
// ts_hasf_impl.cuh; one translation unit per <adjacency, placement, threads>
// variant).
#include <cuda_runtime.h>
#include <mutex>
#include "ts_internal.h"

namespace ts {

#define TS_DECLARE_HASF_VARIANT(SUFFIX)                                                                   \
    cudaError_t launch_hasf_##SUFFIX(const KParams &p, int grid, size_t smem_bytes, cudaStream_t stream); \
    cudaError_t occupancy_hasf_##SUFFIX(size_t smem_bytes, int *blocks);                                  \
    cudaError_t clusters_hasf_##SUFFIX(size_t smem_bytes, int team, int *clusters);
TS_DECLARE_HASF_VARIANT(8h)
TS_DECLARE_HASF_VARIANT(8g)
TS_DECLARE_HASF_VARIANT(4h)
TS_DECLARE_HASF_VARIANT(4g)
TS_DECLARE_HASF_VARIANT(8h256)
TS_DECLARE_HASF_VARIANT(4h256)
TS_DECLARE_HASF_VARIANT(8g1024)
TS_DECLARE_HASF_VARIANT(4g1024)

cudaError_t raise_smem_limit_once(const void *fn, std::mutex &mu, bool (&done)[64]) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lk(mu);
    if (done[dev]) return cudaSuccess;
    int optin = 0;
    cudaFuncAttributes fa{};
    if ((e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev)) != cudaSuccess) return e;
    if ((e = cudaFuncGetAttributes(&fa, fn)) != cudaSuccess) return e;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes);
    if (e == cudaSuccess) done[dev] = true;
    return e;
}

// threads: 512 (any placement), 256 (hot placement only, two CTAs per SM) or
// 1024 (global placement only: cluster teams)
cudaError_t launch_hasf(const KParams &p, int fg, int grid, size_t smem_bytes, cudaStream_t stream) {
    if (p.threads == kWideThreads && !p.hot) {
        return fg == 8 ? launch_hasf_8g1024(p, grid, smem_bytes, stream) : launch_hasf_4g1024(p, grid, smem_bytes, stream);
    }
    if (p.threads == 256 && p.hot) {
        return fg == 8 ? launch_hasf_8h256(p, grid, smem_bytes, stream) : launch_hasf_4h256(p, grid, smem_bytes, stream);
    }
    if (fg == 8) return p.hot ? launch_hasf_8h(p, grid, smem_bytes, stream) : launch_hasf_8g(p, grid, smem_bytes, stream);
    return p.hot ? launch_hasf_4h(p, grid, smem_bytes, stream) : launch_hasf_4g(p, grid, smem_bytes, stream);
}

// co-resident clusters of `team` CTAs of the global-placement variant
cudaError_t hasf_cluster_occupancy(int fg, int threads, size_t smem_bytes, int team, int *clusters) {
    if (threads == kWideThreads)
        return fg == 8 ? clusters_hasf_8g1024(smem_bytes, team, clusters) : clusters_hasf_4g1024(smem_bytes, team, clusters);
    return fg == 8 ? clusters_hasf_8g(smem_bytes, team, clusters) : clusters_hasf_4g(smem_bytes, team, clusters);
}

cudaError_t hasf_occupancy(int fg, bool hot, int threads, size_t smem_bytes, int *blocks_per_sm) {
    if (threads == kWideThreads) {
        if (hot) return cudaErrorInvalidValue;
        return fg == 8 ? occupancy_hasf_8g1024(smem_bytes, blocks_per_sm) : occupancy_hasf_4g1024(smem_bytes, blocks_per_sm);
    }
    if (threads == 256) {
        if (!hot) return cudaErrorInvalidValue;
        return fg == 8 ? occupancy_hasf_8h256(smem_bytes, blocks_per_sm) : occupancy_hasf_4h256(smem_bytes, blocks_per_sm);
    }
    if (fg == 8) return hot ? occupancy_hasf_8h(smem_bytes, blocks_per_sm) : occupancy_hasf_8g(smem_bytes, blocks_per_sm);
    return hot ? occupancy_hasf_4h(smem_bytes, blocks_per_sm) : occupancy_hasf_4g(smem_bytes, blocks_per_sm);
}

}  // namespace ts
