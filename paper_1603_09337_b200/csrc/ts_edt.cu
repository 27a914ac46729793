// Exact squared EDT (int64 output, INF sentinel) and the per-pixel classifier
// kernels for sm_100a.  These back the stage-level parity API (edt_squared,
// edt_phase1_columns, edt_phase2_rows, background_distances, dilate, erode,
// neighborhood_codes, simple_point_mask); the fused HASF kernel uses its own
// radius-clamped bit-parallel EDT (ts_hasf.cu).
//
// Phase 1 (edt.py:45-71): one thread per column, down then up sweep; adjacent
// threads touch adjacent columns, so every row step is one coalesced access.
// Phase 2 (edt.py:74-119): one thread per row builds the lower envelope of the
// parabolas (x-u)^2 + g(u)^2; its stacks s,t live in a column-major scratch
// ([W][rows]) so that the 32 rows of a warp hit consecutive addresses.
#include <cuda_runtime.h>
#include <cstdint>
#include "ts_common.cuh"

namespace ts {

// floor division for a positive divisor (Python //, edt.py:106)
__device__ __forceinline__ long long floordiv_pos(long long a, long long b) {
    long long q = a / b;
    if ((a % b) != 0 && (a < 0)) q -= 1;
    return q;
}

__global__ void edt_phase1_kernel(const uint8_t *__restrict__ pix, long long *__restrict__ g, int n, int H, int W,
                                  int invert, long long inf) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int b = blockIdx.y;
    if (c >= W || b >= n) return;
    const uint8_t *p = pix + (size_t)b * H * W + c;
    long long *gg = g + (size_t)b * H * W + c;
    long long prev = (p[0] != invert) ? 0 : inf;
    gg[0] = prev;
    for (int r = 1; r < H; ++r) {
        long long v;
        if (p[(size_t)r * W] != invert)
            v = 0;
        else
            v = prev < inf ? prev + 1 : inf;
        gg[(size_t)r * W] = v;
        prev = v;
    }
    for (int r = H - 2; r >= 0; --r) {
        const long long cur = gg[(size_t)r * W];
        if (prev < cur) {
            const long long v = prev + 1;
            gg[(size_t)r * W] = v;
            prev = v;
        } else {
            prev = cur;
        }
    }
}

// out_mode: 0 -> int64 distance; 1 -> int64 min(distance, border^2)
//           2 -> uint8 (distance <= thr)      3 -> uint8 (min(distance, border^2) > thr)
__global__ void edt_phase2_kernel(const long long *__restrict__ g, void *__restrict__ out, long long *__restrict__ stk,
                                  int n, int H, int W, long long inf, int out_mode, long long thr) {
    const int row = blockIdx.x * blockDim.x + threadIdx.x;
    const int b = blockIdx.y;
    if (row >= H || b >= n) return;
    const long long *gr = g + ((size_t)b * H + row) * W;
    const size_t rows_total = (size_t)n * H;
    const size_t myrow = (size_t)b * H + row;
    // column-major stacks: s at stk[u * rows_total + myrow], t after W*rows_total
    long long *S = stk + myrow;
    long long *T = stk + (size_t)W * rows_total + myrow;
    auto s_at = [&](long long q) -> long long & { return S[(size_t)q * rows_total]; };
    auto t_at = [&](long long q) -> long long & { return T[(size_t)q * rows_total]; };
    long long q = -1;
    for (long long u = 0; u < W; ++u) {
        const long long gu = gr[u];
        if (gu >= inf) continue;
        if (q < 0) {
            q = 0;
            s_at(0) = u;
            t_at(0) = 0;
            continue;
        }
        while (q >= 0) {
            const long long tq = t_at(q), sq = s_at(q);
            const long long gs = gr[sq];
            const long long f_old = (tq - sq) * (tq - sq) + gs * gs;
            const long long f_new = (tq - u) * (tq - u) + gu * gu;
            if (f_old > f_new)
                q -= 1;
            else
                break;
        }
        if (q < 0) {
            q = 0;
            s_at(0) = u;
            t_at(0) = 0;
        } else {
            const long long sq = s_at(q);
            const long long gs = gr[sq];
            const long long wv = 1 + floordiv_pos(u * u - sq * sq + gu * gu - gs * gs, 2 * (u - sq));
            if (wv < W) {
                q += 1;
                s_at(q) = u;
                t_at(q) = wv;
            }
        }
    }
    const size_t obase = ((size_t)b * H + row) * W;
    const long long rb = min(row + 1, H - row);
    for (long long u = W - 1; u >= 0; --u) {
        long long d;
        if (q < 0) {
            d = inf;
        } else {
            const long long sq = s_at(q);
            const long long dd = u - sq;
            const long long gs = gr[sq];
            d = dd * dd + gs * gs;
            if (u == t_at(q)) q -= 1;
        }
        if (out_mode == 1 || out_mode == 3) {   // morph.py:25-31 border term
            const long long cb = min(u + 1, (long long)W - u);
            const long long bb = min(rb, cb);
            d = min(d, bb * bb);
        }
        if (out_mode <= 1)
            reinterpret_cast<long long *>(out)[obase + u] = d;
        else if (out_mode == 2)
            reinterpret_cast<uint8_t *>(out)[obase + u] = d <= thr ? 1 : 0;
        else
            reinterpret_cast<uint8_t *>(out)[obase + u] = d > thr ? 1 : 0;
    }
}

// 8-bit neighbour code per pixel (topo.py:97-106); optional simple mask via a
// 256-entry LUT staged in shared memory (topo.py:144-148)
__global__ void classify_kernel(const uint8_t *__restrict__ pix, uint8_t *__restrict__ out, int n, int H, int W,
                                const uint8_t *__restrict__ lut) {
    __shared__ uint8_t s_lut[256];
    if (lut) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) s_lut[i] = lut[i];
        __syncthreads();
    }
    const size_t total = (size_t)n * H * W;
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
        const size_t b = idx / ((size_t)H * W);
        const int rem = (int)(idx - b * (size_t)H * W);
        const int r = rem / W, c = rem - r * W;
        const uint8_t *p = pix + b * (size_t)H * W;
        const int dr[8] = {-1, -1, -1, 0, 0, 1, 1, 1};
        const int dc[8] = {-1, 0, 1, -1, 1, -1, 0, 1};
        uint32_t code = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int rr = r + dr[k], cc = c + dc[k];
            if (rr >= 0 && rr < H && cc >= 0 && cc < W && p[(size_t)rr * W + cc]) code |= 1u << k;
        }
        out[idx] = lut ? (uint8_t)(p[(size_t)r * W + c] == 1 && s_lut[code] == 1) : (uint8_t)code;
    }
}

// the bit-sliced simple-point circuit of the engine, evaluated on all 256 codes
__global__ void selftest_circuit_kernel(uint8_t *out84, uint8_t *out48) {
    const int j = threadIdx.x;   // 8 threads, 32 codes each
    if (j >= 8) return;
    uint32_t nb[8];
    for (int k = 0; k < 8; ++k) {
        uint32_t v = 0;
        for (int i = 0; i < 32; ++i) v |= (uint32_t)(((32 * j + i) >> k) & 1) << i;
        nb[k] = v;
    }
    const uint32_t s84 = simple_bits<8>(nb[0], nb[1], nb[2], nb[3], nb[4], nb[5], nb[6], nb[7]);
    const uint32_t s48 = simple_bits<4>(nb[0], nb[1], nb[2], nb[3], nb[4], nb[5], nb[6], nb[7]);
    for (int i = 0; i < 32; ++i) {
        out84[32 * j + i] = (s84 >> i) & 1;
        out48[32 * j + i] = (s48 >> i) & 1;
    }
}

cudaError_t launch_edt_phase1(const uint8_t *pix, long long *g, int n, int H, int W, int invert, long long inf,
                              cudaStream_t st) {
    dim3 grid((W + 127) / 128, n);
    edt_phase1_kernel<<<grid, 128, 0, st>>>(pix, g, n, H, W, invert, inf);
    return cudaGetLastError();
}

cudaError_t launch_edt_phase2(const long long *g, void *out, long long *stk, int n, int H, int W, long long inf,
                              int out_mode, long long thr, cudaStream_t st) {
    dim3 grid((H + 63) / 64, n);
    edt_phase2_kernel<<<grid, 64, 0, st>>>(g, out, stk, n, H, W, inf, out_mode, thr);
    return cudaGetLastError();
}

cudaError_t launch_classify(const uint8_t *pix, uint8_t *out, int n, int H, int W, const uint8_t *lut,
                            cudaStream_t st) {
    const size_t total = (size_t)n * H * W;
    size_t nb = (total + 255) / 256;
    int blocks = (int)(nb < 148 * 16 ? nb : 148 * 16);
    if (blocks < 1) blocks = 1;
    classify_kernel<<<blocks, 256, 0, st>>>(pix, out, n, H, W, lut);
    return cudaGetLastError();
}

cudaError_t launch_selftest_circuit(uint8_t *out84, uint8_t *out48, cudaStream_t st) {
    selftest_circuit_kernel<<<1, 32, 0, st>>>(out84, out48);
    return cudaGetLastError();
}

}  // namespace ts
