// Host-side bit packing for the streamed host entry (ts_hasf_batch_host).
//
// The host API takes and returns uint8 {0,1} images (grid.py:48-62); the
// device works on 1-bit planes.  Packing on the host before the copy moves 8x
// fewer bytes over the host link -- the link, not the GPU, decides how fast
// the first wave of images can start.  Layout: image i, row y, word x holds
// pixels 32x .. 32x+31 of the row, LSB = leftmost (the device bit-plane
// layout, ts_common.cuh).  AVX2 (movemask of the bytes' bit 0) with a scalar
// fallback; rows are split over the OpenMP threads.
#include <cstdint>
#include <cstring>

#if defined(__x86_64__)
#include <immintrin.h>
#endif

#include "ts_hostpack.h"

namespace ts {
namespace {

#if defined(__x86_64__)
__attribute__((target("avx2"))) bool pack_row_avx2(const uint8_t *s, uint32_t *d, int w, int ww) {
    __m256i bad = _mm256_setzero_si256();
    const __m256i hi = _mm256_set1_epi8((char)0xFE);
    int x = 0;
    for (; (x + 1) * 32 <= w; ++x) {
        const __m256i v = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(s + 32 * x));
        bad = _mm256_or_si256(bad, _mm256_and_si256(v, hi));
        d[x] = (uint32_t)_mm256_movemask_epi8(_mm256_slli_epi16(v, 7));
    }
    uint32_t tailbad = 0;
    if (x < ww) {
        uint32_t bits = 0;
        for (int c = 32 * x; c < w; ++c) {
            bits |= (uint32_t)(s[c] & 1u) << (c - 32 * x);
            tailbad |= s[c] & 0xFEu;
        }
        d[x] = bits;
    }
    return _mm256_testz_si256(bad, bad) && tailbad == 0;
}

__attribute__((target("avx2"))) void unpack_row_avx2(const uint32_t *s, uint8_t *d, int w, int ww) {
    // byte j of the 32 output bytes takes bit j of the word: broadcast the
    // word, route byte j / 8 of it to lane j, test bit j % 8
    const __m256i route = _mm256_setr_epi8(0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 1, 1, 1, 1, 2, 2, 2, 2, 2, 2, 2, 2, 3, 3,
                                           3, 3, 3, 3, 3, 3);
    const __m256i sel = _mm256_set1_epi64x((long long)0x8040201008040201ULL);
    const __m256i one = _mm256_set1_epi8(1);
    int x = 0;
    // the output (8x the input) is written once and not read back here:
    // non-temporal stores skip the read-for-ownership of every line
    const bool aligned = (reinterpret_cast<uintptr_t>(d) & 31) == 0;
    for (; (x + 1) * 32 <= w; ++x) {
        const __m256i b = _mm256_shuffle_epi8(_mm256_set1_epi32((int)s[x]), route);
        const __m256i m = _mm256_cmpeq_epi8(_mm256_and_si256(b, sel), sel);
        if (aligned)
            _mm256_stream_si256(reinterpret_cast<__m256i *>(d + 32 * x), _mm256_and_si256(m, one));
        else
            _mm256_storeu_si256(reinterpret_cast<__m256i *>(d + 32 * x), _mm256_and_si256(m, one));
    }
    if (x < ww)
        for (int c = 32 * x; c < w; ++c) d[c] = (uint8_t)((s[x] >> (c - 32 * x)) & 1u);
}
#endif

bool pack_row_scalar(const uint8_t *s, uint32_t *d, int w, int ww) {
    uint32_t bad = 0;
    for (int x = 0; x < ww; ++x) {
        uint32_t bits = 0;
        const int c1 = w < 32 * x + 32 ? w : 32 * x + 32;
        for (int c = 32 * x; c < c1; ++c) {
            bits |= (uint32_t)(s[c] & 1u) << (c - 32 * x);
            bad |= s[c] & 0xFEu;
        }
        d[x] = bits;
    }
    return bad == 0;
}

void unpack_row_scalar(const uint32_t *s, uint8_t *d, int w, int) {
    for (int c = 0; c < w; ++c) d[c] = (uint8_t)((s[c >> 5] >> (c & 31)) & 1u);
}

bool have_avx2() {
#if defined(__x86_64__)
    static const bool a = __builtin_cpu_supports("avx2");
    return a;
#else
    return false;
#endif
}

}  // namespace

bool pack_images(const uint8_t *in, uint32_t *out, int64_t n, int h, int w, int ww) {
    const int64_t rows = n * h;
    const bool avx = have_avx2();
    int ok = 1;
#pragma omp parallel for schedule(static) reduction(& : ok) if (rows >= 256)
    for (int64_t r = 0; r < rows; ++r) {
        const uint8_t *s = in + r * (int64_t)w;
        uint32_t *d = out + r * (int64_t)ww;
#if defined(__x86_64__)
        const bool good = avx ? pack_row_avx2(s, d, w, ww) : pack_row_scalar(s, d, w, ww);
#else
        const bool good = pack_row_scalar(s, d, w, ww);
#endif
        ok &= good ? 1 : 0;
    }
    return ok != 0;
}

// the same for up to 3 planes (image, keep, avoid) in ONE parallel region: a
// chunk of the constrained streamed entry pays one fork / join instead of three
bool pack_planes(const uint8_t *const *in, uint32_t *const *out, int planes, int64_t n, int h, int w, int ww) {
    const int64_t rows = n * h, total = rows * planes;
    const bool avx = have_avx2();
    int ok = 1;
#pragma omp parallel for schedule(static) reduction(& : ok) if (total >= 256)
    for (int64_t t = 0; t < total; ++t) {
        const int pl = (int)(t / rows);
        const int64_t r = t - pl * rows;
        const uint8_t *s = in[pl] + r * (int64_t)w;
        uint32_t *d = out[pl] + r * (int64_t)ww;
#if defined(__x86_64__)
        const bool good = avx ? pack_row_avx2(s, d, w, ww) : pack_row_scalar(s, d, w, ww);
#else
        const bool good = pack_row_scalar(s, d, w, ww);
#endif
        ok &= good ? 1 : 0;
    }
    return ok != 0;
}

void unpack_images(const uint32_t *in, uint8_t *out, int64_t n, int h, int w, int ww) {
    const int64_t rows = n * h;
    const bool avx = have_avx2();
#pragma omp parallel for schedule(static) if (rows >= 256)
    for (int64_t r = 0; r < rows; ++r) {
        const uint32_t *s = in + r * (int64_t)ww;
        uint8_t *d = out + r * (int64_t)w;
#if defined(__x86_64__)
        if (avx)
            unpack_row_avx2(s, d, w, ww);
        else
            unpack_row_scalar(s, d, w, ww);
#else
        unpack_row_scalar(s, d, w, ww);
#endif
    }
#if defined(__x86_64__)
    _mm_sfence();   // the streamed stores are globally visible before the caller returns
#endif
}

}  // namespace ts
