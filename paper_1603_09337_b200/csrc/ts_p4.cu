// netpbm P4 rasters <-> the device bit-row layout.
//
// P4 (reference netpbm.py:68-129): one bit per pixel, MSB first, rows padded
// to a whole byte, padding bits ignored on read and zero on write; value 1 =
// black = object.  The fused kernel's host-packed input/output format
// (KParams::packed_io) is [n][H][WW] uint32 words, word x of a row holding
// pixels 32x .. 32x+31 with the LEFTMOST pixel in bit 0, padding bits zero.
// Word x of a row is therefore P4 bytes 4x .. 4x+3 with the bits of every byte
// reversed: brev(byteswap(w)) when the four bytes are read little-endian.
// Both directions are one thread per word: reads of 4 consecutive bytes per
// thread (row_bytes need not be a multiple of 4, so byte loads, coalesced
// across the warp), one 32-bit store.  HBM-bound (1/8 B/px each way).
#include <cuda_runtime.h>
#include <cstdint>

namespace ts {

__global__ void p4_to_rows_kernel(const uint8_t *__restrict__ p4, uint32_t *__restrict__ rows, long long nrows, int w,
                                  int row_bytes, int ww) {
    const long long total = nrows * ww;
    const uint32_t lastmask = (w & 31) ? ((1u << (w & 31)) - 1u) : ~0u;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / ww;
        const int x = (int)(i - r * ww);
        const uint8_t *s = p4 + r * row_bytes + 4 * x;
        const int nb = min(4, row_bytes - 4 * x);
        uint32_t v = 0;
        for (int b = 0; b < nb; ++b) v |= (uint32_t)s[b] << (8 * b);
        uint32_t word = __brev(__byte_perm(v, 0, 0x0123));
        if (x == ww - 1) word &= lastmask;   // P4 padding bits are ignored on read
        rows[i] = word;
    }
}

__global__ void rows_to_p4_kernel(const uint32_t *__restrict__ rows, uint8_t *__restrict__ p4, long long nrows, int w,
                                  int row_bytes, int ww) {
    const long long total = nrows * ww;
    const uint32_t lastmask = (w & 31) ? ((1u << (w & 31)) - 1u) : ~0u;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / ww;
        const int x = (int)(i - r * ww);
        uint32_t word = rows[i];
        if (x == ww - 1) word &= lastmask;   // padding bits written as zero
        const uint32_t v = __byte_perm(__brev(word), 0, 0x0123);
        uint8_t *d = p4 + r * row_bytes + 4 * x;
        const int nb = min(4, row_bytes - 4 * x);
        for (int b = 0; b < nb; ++b) d[b] = (uint8_t)(v >> (8 * b));
    }
}

// P4 raster <-> uint8 {0,1} planes (the stage path for radii above kMaxR works on bytes)
__global__ void p4_to_u8_kernel(const uint8_t *__restrict__ p4, uint8_t *__restrict__ out, long long nrows, int w,
                                int row_bytes) {
    const long long total = nrows * w;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / w;
        const int c = (int)(i - r * w);
        out[i] = (p4[r * row_bytes + (c >> 3)] >> (7 - (c & 7))) & 1u;
    }
}

__global__ void u8_to_p4_kernel(const uint8_t *__restrict__ in, uint8_t *__restrict__ p4, long long nrows, int w,
                                int row_bytes) {
    const long long total = nrows * row_bytes;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / row_bytes;
        const int c0 = (int)(i - r * row_bytes) * 8;
        uint32_t v = 0;
        for (int k = 0; k < 8; ++k)
            if (c0 + k < w) v |= (uint32_t)(in[r * w + c0 + k] & 1u) << (7 - k);
        p4[i] = (uint8_t)v;
    }
}

static int grid_for(long long work) {
    long long g = (work + 255) / 256;
    return (int)(g < 1 ? 1 : (g > 148 * 32 ? 148 * 32 : g));
}

cudaError_t launch_p4_to_rows(const uint8_t *p4, uint32_t *rows, long long nrows, int w, cudaStream_t st) {
    const int ww = (w + 31) / 32, rb = (w + 7) / 8;
    p4_to_rows_kernel<<<grid_for(nrows * ww), 256, 0, st>>>(p4, rows, nrows, w, rb, ww);
    return cudaGetLastError();
}

cudaError_t launch_rows_to_p4(const uint32_t *rows, uint8_t *p4, long long nrows, int w, cudaStream_t st) {
    const int ww = (w + 31) / 32, rb = (w + 7) / 8;
    rows_to_p4_kernel<<<grid_for(nrows * ww), 256, 0, st>>>(rows, p4, nrows, w, rb, ww);
    return cudaGetLastError();
}

cudaError_t launch_p4_to_u8(const uint8_t *p4, uint8_t *out, long long nrows, int w, cudaStream_t st) {
    p4_to_u8_kernel<<<grid_for(nrows * w), 256, 0, st>>>(p4, out, nrows, w, (w + 7) / 8);
    return cudaGetLastError();
}

cudaError_t launch_u8_to_p4(const uint8_t *in, uint8_t *p4, long long nrows, int w, cudaStream_t st) {
    u8_to_p4_kernel<<<grid_for(nrows * ((w + 7) / 8)), 256, 0, st>>>(in, p4, nrows, w, (w + 7) / 8);
    return cudaGetLastError();
}

}  // namespace ts
