// Shared device helpers for the B200 HASF path (sm_100a).
//
// Bit-plane layout: an H x W binary image is H rows of WW = ceil(W/32) uint32
// words; bit i of word x is pixel column 32*x + i (LSB = leftmost).  Bits at
// columns >= W are padding and always 0 in image planes.
#pragma once
#include <cstdint>
#include <utility>
#include <type_traits>

namespace ts {

// ---- compile-time loops -------------------------------------------------
template <typename F, int... Is>
__device__ __forceinline__ void static_for_impl(F &&f, std::integer_sequence<int, Is...>) {
    (f(std::integral_constant<int, Is>{}), ...);
}
template <int N, typename F>
__device__ __forceinline__ void static_for(F &&f) {
    static_for_impl(f, std::make_integer_sequence<int, N>{});
}

// ---- squared-distance levels of a radius-R disc ---------------------------
// level values = distinct a^2 + b^2 <= R^2 (0 <= a,b <= R), ascending.  A clamped
// squared distance d <= R^2 is always one of them, so comparing ranks equals
// comparing distances (values above r^2 are never observed).
__host__ __device__ constexpr bool is_level(int v, int R) {
    for (int a = 0; a <= R; ++a)
        for (int b = 0; b <= a; ++b)
            if (a * a + b * b == v) return true;
    return false;
}
__host__ __device__ constexpr int level_count(int R) {
    int c = 0;
    for (int v = 0; v <= R * R; ++v) c += is_level(v, R) ? 1 : 0;
    return c;
}
__host__ __device__ constexpr int level_value(int R, int i) {
    int c = 0;
    for (int v = 0; v <= R * R; ++v)
        if (is_level(v, R)) {
            if (c == i) return v;
            ++c;
        }
    return -1;
}
__host__ __device__ constexpr int isqrt_c(int x) {
    int k = 0;
    while ((k + 1) * (k + 1) <= x) ++k;
    return k;
}
// largest |dy| with dx^2 + dy^2 <= level_value(R, i); -1 if |dx| is too far
__host__ __device__ constexpr int k_at(int R, int i, int dx) {
    int rem = level_value(R, i) - dx * dx;
    return rem < 0 ? -1 : isqrt_c(rem);
}
__host__ __device__ constexpr int bits_for(int n) {   // bits to hold 0..n-1 (>= 1)
    int b = 1;
    while ((1 << b) < n) ++b;
    return b;
}
__host__ __device__ constexpr int rank_slices(int R) { return bits_for(level_count(R)); }

constexpr int kMaxR = 16;                          // radii 1..kMaxR are instantiated
constexpr int kMaxSlices = rank_slices(kMaxR);      // 7

// ---- word shifts (neighbour access inside a row) ----------------------------
// value of pixel (col + d) placed at bit position of col, from words (l, c, r)
__device__ __forceinline__ uint32_t from_west(uint32_t l, uint32_t c) { return __funnelshift_l(l, c, 1); }
__device__ __forceinline__ uint32_t from_east(uint32_t c, uint32_t r) { return __funnelshift_r(c, r, 1); }

// ---- simple-point test, bit-sliced ----------------------------------------
// 32 pixels at once from the 8 neighbour bit-words (reference code bit order
// NW,N,NE,W,E,SW,S,SE, topo.py:35).  Yokoi connectivity number == 1:
//   (8,4): sum_{k odd} ~a_k & (a_{k+1} | a_{k+2})          == 1
//   (4,8): sum_{k odd}  a_k & ~(a_{k+1} & a_{k+2})         == 1
// with the circular order a1..a8 = E,NE,N,NW,W,SW,S,SE.  Equal to SIMPLE_84 /
// SIMPLE_48 (topo.py:82-84) on all 256 codes (checked by ts_selftest_circuit).
template <int FG>
__device__ __forceinline__ uint32_t simple_bits(uint32_t nw, uint32_t n, uint32_t ne, uint32_t w,
                                                uint32_t e, uint32_t sw, uint32_t s, uint32_t se) {
    uint32_t t1, t3, t5, t7;
    if constexpr (FG == 8) {
        t1 = ~e & (ne | n);
        t3 = ~n & (nw | w);
        t5 = ~w & (sw | s);
        t7 = ~s & (se | e);
    } else {
        t1 = e & ~(ne & n);
        t3 = n & ~(nw & w);
        t5 = w & ~(sw & s);
        t7 = s & ~(se & e);
    }
    uint32_t x1 = t1 ^ t3, c1 = t1 & t3;
    uint32_t x2 = t5 ^ t7, c2 = t5 & t7;
    return (x1 ^ x2) & ~(c1 | c2);    // exactly one of t1,t3,t5,t7
}

// segmented scheduler (KParams::nseg): segment `seg` of an image's `total`
// stages is [k0, k1): segments of `len` stages, the last `fine` stages one each
__host__ __device__ __forceinline__ int seg_count(int total, int len, int fine) {
    const int body = total > fine ? total - fine : 0;
    return (body + len - 1) / len + (total - body);
}
__host__ __device__ __forceinline__ void seg_range(int total, int len, int fine, int seg, int &k0, int &k1) {
    const int body = total > fine ? total - fine : 0;
    const int nbody = (body + len - 1) / len;
    if (seg < nbody) {
        k0 = seg * len;
        k1 = k0 + len < body ? k0 + len : body;
    } else {
        k0 = body + (seg - nbody);
        k1 = k0 + 1;
    }
}

}  // namespace ts
