// Exact squared EDT (int64 output, INF sentinel) and the per-pixel classifier
// kernels for sm_100a.  These back the stage-level parity API (edt_squared,
// edt_phase1_columns, edt_phase2_rows, background_distances, dilate, erode,
// neighborhood_codes, simple_point_mask); the fused HASF kernel uses its own
// radius-clamped bit-parallel EDT (ts_hasf_impl.cuh).
//
// All arithmetic is int32 (g^2 + u^2 <= 2 * 32767^2 < 2^31, and
// INF = h^2 + w^2 + 1 fits); int64 appears only at the API (the reference's
// dtype).  Every global access is coalesced:
//   phase 1 (edt.py:45-71): one thread per column, down then up sweep; a
//     warp's 32 columns are adjacent, so each row step is one transaction;
//   transpose: 32x32 shared-memory tiles, g [H][W] -> gT [W][H];
//   phase 2 (edt.py:74-119): one thread per ROW on the transposed map -- the
//     32 rows of a warp read gT[u][row..row+31] together, and the lower-
//     envelope stacks s, t live as [q][row] for the same reason; the result
//     goes out transposed (outT [W][H]);
//   transpose back, fused with the output conversion (int64 distance, border
//     term of morph.py:25-31, dilate / erode thresholds).
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

template <class T>
__global__ void edt_phase1_kernel(const uint8_t *__restrict__ pix, T *__restrict__ g, int n, int H, int W, int invert,
                                  int inf) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int b = blockIdx.y;
    if (c >= W || b >= n) return;
    const uint8_t *p = pix + (size_t)b * H * W + c;
    T *gg = g + (size_t)b * H * W + c;
    int prev = (p[0] != invert) ? 0 : inf;
    gg[0] = prev;
    for (int r = 1; r < H; ++r) {
        const int v = p[(size_t)r * W] != invert ? 0 : (prev < inf ? prev + 1 : inf);
        gg[(size_t)r * W] = v;
        prev = v;
    }
    for (int r = H - 2; r >= 0; --r) {
        const int cur = (int)gg[(size_t)r * W];
        if (prev < cur) {
            gg[(size_t)r * W] = ++prev;
        } else {
            prev = cur;
        }
    }
}

// [n][H][W] (TI) -> [n][W][H] int32, 32x32 tiles through shared memory
template <class TI>
__global__ void transpose_in_kernel(const TI *__restrict__ src, int *__restrict__ dst, int H, int W) {
    __shared__ int tile[32][33];
    const size_t img = (size_t)blockIdx.z * H * W;
    const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const int y = y0 + j, x = x0 + threadIdx.x;
        if (y < H && x < W) tile[j][threadIdx.x] = (int)src[img + (size_t)y * W + x];
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const int x = x0 + j, y = y0 + threadIdx.x;
        if (y < H && x < W) dst[img + (size_t)x * H + y] = tile[threadIdx.x][j];
    }
}

// lower envelope of the parabolas (x-u)^2 + g(u)^2 of one row (edt.py:74-119),
// on the transposed map: gT[u * H + row], stacks s/t at [q * H + row]
__global__ void edt_phase2T_kernel(const int *__restrict__ gT, int *__restrict__ outT, int *__restrict__ stk, int n,
                                   int H, int W, int inf) {
    const int row = blockIdx.x * blockDim.x + threadIdx.x;
    const int b = blockIdx.y;
    if (row >= H || b >= n) return;
    const size_t img = (size_t)b * H * W;
    const int *gr = gT + img + row;                   // g(u) = gr[u * H]
    int *S = stk + 2 * img + row, *T = S + (size_t)W * H;
    auto at = [&](int *base, int q) -> int & { return base[(size_t)q * H]; };
    int q = -1;
    for (int u = 0; u < W; ++u) {
        const int gu = gr[(size_t)u * H];
        if (gu >= inf) continue;
        while (q >= 0) {
            const int tq = at(T, q), sq = at(S, q);
            const int gs = gr[(size_t)sq * H];
            const int f_old = (tq - sq) * (tq - sq) + gs * gs;
            const int f_new = (tq - u) * (tq - u) + gu * gu;
            if (f_old > f_new)
                --q;
            else
                break;
        }
        if (q < 0) {
            q = 0;
            at(S, 0) = u;
            at(T, 0) = 0;
        } else {
            const int sq = at(S, q), gs = gr[(size_t)sq * H];
            const long long num = (long long)u * u - (long long)sq * sq + (long long)gu * gu - (long long)gs * gs;
            const long long wv = 1 + floordiv_pos(num, 2LL * (u - sq));
            if (wv < W) {
                ++q;
                at(S, q) = u;
                at(T, q) = (int)wv;
            }
        }
    }
    int *o = outT + img + row;
    for (int u = W - 1; u >= 0; --u) {
        int d = inf;
        if (q >= 0) {
            const int sq = at(S, q), dd = u - sq, gs = gr[(size_t)sq * H];
            d = dd * dd + gs * gs;
            if (u == at(T, q)) --q;
        }
        o[(size_t)u * H] = d;
    }
}

// [n][W][H] int32 -> [n][H][W] output.  out_mode: 0 int64 distance;
// 1 int64 min(distance, border^2) (morph.py:25-31); 2 uint8 distance <= thr
// (dilate); 3 uint8 min(distance, border^2) > thr (erode)
__global__ void transpose_out_kernel(const int *__restrict__ srcT, void *__restrict__ out, int H, int W, int out_mode,
                                     long long thr) {
    __shared__ int tile[32][33];
    const size_t img = (size_t)blockIdx.z * H * W;
    const int y0 = blockIdx.x * 32, x0 = blockIdx.y * 32;   // tile: rows y0.., columns x0..
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const int x = x0 + j, y = y0 + threadIdx.x;
        if (y < H && x < W) tile[j][threadIdx.x] = srcT[img + (size_t)x * H + y];
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const int y = y0 + j, x = x0 + threadIdx.x;
        if (y >= H || x >= W) continue;
        long long d = tile[threadIdx.x][j];
        if (out_mode == 1 || out_mode == 3) {
            const long long bb = min(min(y + 1, H - y), min(x + 1, W - x));
            d = min(d, bb * bb);
        }
        const size_t o = img + (size_t)y * W + x;
        if (out_mode <= 1)
            reinterpret_cast<long long *>(out)[o] = d;
        else if (out_mode == 2)
            reinterpret_cast<uint8_t *>(out)[o] = d <= thr ? 1 : 0;
        else
            reinterpret_cast<uint8_t *>(out)[o] = d > thr ? 1 : 0;
    }
}

// Stage masks of the multi-launch HASF path (radii above the fused kernel's
// kMaxR, smoothing.py:107-146): mode 0 F = (dist > thr) | a (thinning floor,
// a = keep or the filling's input, may be null); mode 1 V = (dist <= thr) & a
// (cutting's regrowth cap, a = X); mode 2 V = (dist <= thr) & ~b (filling's
// cap, b = avoid, may be null).
__global__ void stage_mask_kernel(const long long *__restrict__ dist, const uint8_t *__restrict__ a,
                                  const uint8_t *__restrict__ b, uint8_t *__restrict__ out, size_t px, long long thr,
                                  int mode) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < px; i += (size_t)gridDim.x * blockDim.x) {
        const long long d = dist[i];
        uint8_t v;
        if (mode == 0)
            v = (d > thr) | (a ? a[i] : 0);
        else if (mode == 1)
            v = (d <= thr) & a[i];
        else
            v = (d <= thr) & (b ? (uint8_t)(b[i] ^ 1) : (uint8_t)1);
        out[i] = v;
    }
}

cudaError_t launch_stage_mask(const long long *dist, const uint8_t *a, const uint8_t *b, uint8_t *out, size_t px,
                              long long thr, int mode, cudaStream_t st) {
    size_t nb = (px + 255) / 256;
    const int blocks = (int)(nb < 148 * 16 ? (nb < 1 ? 1 : nb) : 148 * 16);
    stage_mask_kernel<<<blocks, 256, 0, st>>>(dist, a, b, out, px, thr, mode);
    return cudaGetLastError();
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

// phase 1 alone (ts_edt_phase1_batch): int64 column distances, row-major
cudaError_t launch_edt_phase1(const uint8_t *pix, long long *g, int n, int H, int W, int invert, long long inf,
                              cudaStream_t st) {
    dim3 grid((W + 127) / 128, n);
    edt_phase1_kernel<long long><<<grid, 128, 0, st>>>(pix, g, n, H, W, invert, (int)inf);
    return cudaGetLastError();
}

// the exact EDT pipeline: phase 1 (or a caller's int64 g), transpose, phase 2
// on rows, transpose back into the output.  scratch: 5 int32 per pixel.
cudaError_t launch_edt(const uint8_t *pix, const long long *g64, void *out, int *scratch, int n, int H, int W,
                       int invert, long long inf, int out_mode, long long thr, cudaStream_t st) {
    const size_t px = (size_t)n * H * W;
    int *g = scratch, *gT = scratch + px, *outT = g, *stk = scratch + 2 * px;   // outT reuses g
    const dim3 tb(32, 8), tgrid((W + 31) / 32, (H + 31) / 32, n);
    if (g64) {
        transpose_in_kernel<long long><<<tgrid, tb, 0, st>>>(g64, gT, H, W);
    } else {
        edt_phase1_kernel<int><<<dim3((W + 127) / 128, n), 128, 0, st>>>(pix, g, n, H, W, invert, (int)inf);
        transpose_in_kernel<int><<<tgrid, tb, 0, st>>>(g, gT, H, W);
    }
    edt_phase2T_kernel<<<dim3((H + 127) / 128, n), 128, 0, st>>>(gT, outT, stk, n, H, W, (int)inf);
    transpose_out_kernel<<<dim3((H + 31) / 32, (W + 31) / 32, n), tb, 0, st>>>(outT, out, H, W, out_mode, thr);
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
