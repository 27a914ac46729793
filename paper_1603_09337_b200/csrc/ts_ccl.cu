// Connected-component counting on the device (the topology verifier of the
// reference, grid.py:93-128: component_count / background_component_count).
//
// Lock-free union-find over the pixels of the selected set (object pixels, or
// background pixels), batched over images:
//   init   parent[p] = p for pixels in the set
//   union  every pixel with its raster-earlier neighbours in the set
//          (W, N for 4-adjacency; W, NW, N, NE for 8-adjacency); for the
//          background "with exterior" count, window-border pixels are also
//          united with a virtual exterior node (index h*w), which stands for the
//          reference's one-pixel background ring (grid.py:124-128)
//   count  roots = pixels p in the set with parent[p] == p, plus the exterior
//          node when it is a root itself (no border pixel in the set)
// Hooking always points the larger root at the smaller one (atomicCAS), so the
// forest stays acyclic; finds use path halving.
#include <cuda_runtime.h>
#include <cstdint>

namespace ts {

__device__ __forceinline__ int find_root(int *parent, int a) {
    int pa = parent[a];
    while (pa != a) {
        const int gp = parent[pa];
        if (gp != pa) atomicCAS(&parent[a], pa, gp);   // path halving (benign race)
        a = pa;
        pa = parent[a];
    }
    return a;
}

__device__ __forceinline__ void unite(int *parent, int a, int b) {
    while (true) {
        a = find_root(parent, a);
        b = find_root(parent, b);
        if (a == b) return;
        if (a < b) {
            const int t = a;
            a = b;
            b = t;
        }
        const int old = atomicCAS(&parent[a], a, b);   // hook the larger root under the smaller
        if (old == a) return;
        a = old;
    }
}

struct CclArgs {
    const uint8_t *img;
    int *parent;        // [n][h*w + 1]
    long long *counts;  // [n]
    int n, h, w;
    int conn;           // 4 or 8
    int target;         // pixel value of the set (1: object, 0: background)
    int exterior;       // attach the window exterior (background count)
};

__global__ void ccl_init(CclArgs a) {
    const size_t per = (size_t)a.h * a.w + 1;
    const size_t total = per * a.n;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const size_t b = i / per, q = i - b * per;
        int v;
        if (q == per - 1)
            v = (int)q;   // exterior node
        else
            v = a.img[b * (per - 1) + q] == a.target ? (int)q : -1;
        a.parent[i] = v;
    }
}

__global__ void ccl_union(CclArgs a) {
    const size_t hw = (size_t)a.h * a.w, per = hw + 1;
    const size_t total = hw * a.n;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const size_t b = i / hw, q = i - b * hw;
        const uint8_t *img = a.img + b * hw;
        if (img[q] != a.target) continue;
        int *parent = a.parent + b * per;
        const int r = (int)(q / a.w), c = (int)(q - (size_t)r * a.w);
        const int p = (int)q;
        const bool W = c > 0 && img[q - 1] == a.target;
        const bool N = r > 0 && img[q - a.w] == a.target;
        if (W) unite(parent, p, p - 1);
        if (a.conn == 8) {
            // edges implied by others are skipped (8-adjacency): W-N, NW-W, NW-N
            // and N-NE are themselves neighbour pairs, so one union per
            // connected group of earlier neighbours suffices
            const bool NW = r > 0 && c > 0 && img[q - a.w - 1] == a.target;
            const bool NE = r > 0 && c + 1 < a.w && img[q - a.w + 1] == a.target;
            if (N && !W) unite(parent, p, p - a.w);
            if (NW && !W && !N) unite(parent, p, p - a.w - 1);
            if (NE && !N) unite(parent, p, p - a.w + 1);
        } else if (N) {
            unite(parent, p, p - a.w);
        }
        // pixels on the window border touch the exterior ring (the ring pixels
        // are 4- and 8-adjacent to every border pixel)
        if (a.exterior && (r == 0 || c == 0 || r == a.h - 1 || c == a.w - 1)) unite(parent, p, (int)hw);
    }
}

__global__ void ccl_count(CclArgs a) {
    const size_t hw = (size_t)a.h * a.w, per = hw + 1;
    const size_t total = per * a.n;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const size_t b = i / per, q = i - b * per;
        const int v = a.parent[i];
        const bool ext = q == hw;
        // roots only: when border pixels attached the exterior node it hangs under
        // the smallest pixel index of that component
        const bool root = v == (int)q && (!ext || a.exterior);
        // one atomic per image run of the warp (lanes of a warp mostly share b)
        const unsigned act = __activemask();
        const unsigned same = __match_any_sync(act, (unsigned long long)b);
        const unsigned cnt = __popc(__ballot_sync(act, root) & same);
        if (cnt && (threadIdx.x & 31) == __ffs(same) - 1) atomicAdd((unsigned long long *)&a.counts[b], (unsigned long long)cnt);
    }
}

cudaError_t launch_ccl(const uint8_t *img, int *parent, long long *counts, int n, int h, int w, int conn,
                       int target, int exterior, cudaStream_t st) {
    CclArgs a{img, parent, counts, n, h, w, conn, target, exterior};
    const int blocks = 148 * 8;
    ccl_init<<<blocks, 256, 0, st>>>(a);
    ccl_union<<<blocks, 256, 0, st>>>(a);
    ccl_count<<<blocks, 256, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace ts
