// Fused per-image HASF kernel for sm_100a.
//
// One persistent CTA owns one image at a time (images are pulled from an
// atomic queue, so uneven per-image work balances across SMs) and runs the
// whole filter on the bit-packed image without leaving the CTA:
//
//   for r in r_first..r_last                       smoothing.py:209-211
//     cutting  (smoothing.py:127-135)              filling (smoothing.py:138-146)
//       S1 prep  P = min(EDT(~X), B), F            S5 prep  D = EDT(X'), V
//       S2 FLIP  thin   (target 1)                 S6 FLIP  thicken (target 0)
//       S3 prep  D = EDT(Y), V = D<=r^2 & X        S7 prep  P = min(EDT(~Z), B), F
//       S4 FLIP  thicken (target 0)                S8 FLIP  thin   (target 1)
//
// "prep" is the radius-r clamped squared EDT computed bit-parallel (32 px per
// thread op): vertical OR-dilations V_k (k <= r) then the disc as an OR of
// shifted V_k, level by level, giving the rank of each pixel's clamped
// distance as bit-slices (values > r^2 are never observed) and
// the blocked plane (the reference's _thin_prepare_kernel / _cap_kernel,
// smoothing.py:51-100).
//
// "FLIP" is the reference engine (topo.py:211-258, restated in SURVEY A.1):
// per sweep, C = simple unblocked target pixels; visit C in (priority,
// raster) order, flipping each still-simple pixel.  It is reproduced exactly
// by a chaotic fixpoint over the sweep's candidates: pixel p
// flips iff SIMPLE(code of p with every candidate neighbour q that precedes p
// in key order toggled iff q flips).  The precedence masks ("E" planes) are
// computed once per engine call from the rank slices; a pass with no change
// certifies the unique solution.  Later sweeps only re-examine the 3x3 word
// neighbourhood of the previous sweep's flips (the reference's re-queue,
// topo.py:245-257).
#include <cuda_runtime.h>
#include "ts_common.cuh"
#include "ts_internal.h"

namespace ts {

constexpr int kThreads = 512;

struct Img {
    uint32_t *I, *D, *C, *B, *XS, *R, *K, *A, *list, *E;
    uint8_t *dirty;
    int H, W, WW, nwords;
    uint32_t lastmask;   // valid bits of the last word of a row
};

__device__ __forceinline__ void set_err(int *err, int code) { atomicCAS(err, 0, code); }

__device__ __forceinline__ uint32_t valid_bits(const Img &g, int x) { return x == g.WW - 1 ? g.lastmask : ~0u; }

__device__ __forceinline__ uint32_t ldw(const uint32_t *P, const Img &g, int y, int x) {
    return (y < 0 || y >= g.H || x < 0 || x >= g.WW) ? 0u : P[y * g.WW + x];
}

struct Nb {
    uint32_t nw, n, ne, w, e, sw, s, se;
};

// neighbour bit-words of the 32 pixels of word (y, x); outside the window = 0
__device__ __forceinline__ Nb nbrs(const uint32_t *P, const Img &g, int y, int x) {
    const uint32_t u0 = ldw(P, g, y - 1, x - 1), u1 = ldw(P, g, y - 1, x), u2 = ldw(P, g, y - 1, x + 1);
    const uint32_t m0 = ldw(P, g, y, x - 1), m2 = ldw(P, g, y, x + 1), m1 = ldw(P, g, y, x);
    const uint32_t d0 = ldw(P, g, y + 1, x - 1), d1 = ldw(P, g, y + 1, x), d2 = ldw(P, g, y + 1, x + 1);
    Nb r;
    r.nw = from_west(u0, u1);
    r.n = u1;
    r.ne = from_east(u1, u2);
    r.w = from_west(m0, m1);
    r.e = from_east(m1, m2);
    r.sw = from_west(d0, d1);
    r.s = d1;
    r.se = from_east(d1, d2);
    return r;
}

// ---- bit packing of uint8 {0,1} images ---------------------------------
__device__ __forceinline__ uint32_t pack4(uint32_t v) {
    v &= 0x01010101u;
    v |= v >> 7;
    v |= v >> 14;
    return v & 0xFu;
}
__device__ __forceinline__ uint32_t pack16(uint4 a) {
    return pack4(a.x) | (pack4(a.y) << 4) | (pack4(a.z) << 8) | (pack4(a.w) << 12);
}
__device__ __forceinline__ uint32_t spread4(uint32_t nib) {
    return (nib & 1u) | ((nib & 2u) << 7) | ((nib & 4u) << 14) | ((nib & 8u) << 21);
}

// pack one [H,W] uint8 image into a bit-plane; flags bytes > 1
__device__ void pack_plane(const uint8_t *src, uint32_t *dst, const Img &g, int *err, int code) {
    for (int w = threadIdx.x; w < g.nwords; w += kThreads) {
        const int y = w / g.WW, x = w - y * g.WW;
        const int c0 = x * 32;
        const int cnt = min(32, g.W - c0);
        const uint8_t *p = src + (size_t)y * g.W + c0;
        uint32_t bits = 0, bad = 0;
        if (cnt == 32 && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
            const uint4 a = __ldg(reinterpret_cast<const uint4 *>(p));
            const uint4 b = __ldg(reinterpret_cast<const uint4 *>(p + 16));
            bits = pack16(a) | (pack16(b) << 16);
            bad = (a.x | a.y | a.z | a.w | b.x | b.y | b.z | b.w) & 0xFEFEFEFEu;
        } else {
            for (int i = 0; i < cnt; ++i) {
                const uint32_t v = p[i];
                bits |= (v & 1u) << i;
                bad |= v & ~1u;
            }
        }
        if (bad) set_err(err, code);
        dst[w] = bits;
    }
}

__device__ void unpack_plane(const uint32_t *src, uint8_t *dst, const Img &g) {
    for (int w = threadIdx.x; w < g.nwords; w += kThreads) {
        const int y = w / g.WW, x = w - y * g.WW;
        const int c0 = x * 32;
        const int cnt = min(32, g.W - c0);
        uint8_t *p = dst + (size_t)y * g.W + c0;
        const uint32_t bits = src[w];
        if (cnt == 32 && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
            uint4 a, b;
            a.x = spread4(bits);
            a.y = spread4(bits >> 4);
            a.z = spread4(bits >> 8);
            a.w = spread4(bits >> 12);
            b.x = spread4(bits >> 16);
            b.y = spread4(bits >> 20);
            b.z = spread4(bits >> 24);
            b.w = spread4(bits >> 28);
            reinterpret_cast<uint4 *>(p)[0] = a;
            reinterpret_cast<uint4 *>(p)[1] = b;
        } else {
            for (int i = 0; i < cnt; ++i) p[i] = (bits >> i) & 1u;
        }
    }
}

// warp-aggregated append to the active-word list (all 32 lanes must call)
__device__ __forceinline__ void append(bool has, uint32_t entry, uint32_t *list, int *counter) {
    const unsigned m = __ballot_sync(0xffffffffu, has);
    if (m == 0) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(m) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(counter, __popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (has) list[base + __popc(m & ((1u << lane) - 1u))] = entry;
}

// candidates of word (y,x): target-valued, unblocked, simple (topo.py:186-208,
// smoothing.py:83-86); t = 1 thins, t = 0 thickens
template <int FG>
__device__ __forceinline__ uint32_t cand_word(const Img &g, int y, int x, int t) {
    const int w = y * g.WW + x;
    const uint32_t me = g.I[w];
    const uint32_t pre = valid_bits(g, x) & (t ? me : ~me) & ~g.B[w];
    if (!pre) return 0;
    const Nb i = nbrs(g.I, g, y, x);
    return pre & simple_bits<FG>(i.nw, i.n, i.ne, i.w, i.e, i.sw, i.s, i.se);
}

// ---- stage prep: clamped EDT -> rank slices + blocked plane ----------------
template <int R>
struct Lev {
    static constexpr int L = level_count(R);
    static constexpr int S = rank_slices(R);
    struct Arr {
        int v[level_count(R)];
    };
    static constexpr Arr make() {
        Arr a{};
        int c = 0;
        for (int v = 0; v <= R * R; ++v)
            if (is_level(v, R)) a.v[c++] = v;
        return a;
    }
    static constexpr Arr vals = make();
    static constexpr int kat(int i, int dx) {
        return vals.v[i] - dx * dx < 0 ? -1 : isqrt_c(vals.v[i] - dx * dx);
    }
};

// thin = true : seeds = background + window exterior  (P for thinning, S1/S7)
// thin = false: seeds = object pixels                  (D for thickening, S3/S5)
// xmode (thin) : 0 -> F = P > r^2 ; 1 -> | keep ; 2 -> | XS
// xmode (thick): 0 -> V = D <= r^2 ; 1 -> & ~avoid ; 2 -> & XS
template <int R>
__device__ int prep_rank(const Img &g, bool thin, int xmode, bool save_xs) {
    using LV = Lev<R>;
    constexpr int L = LV::L;
    constexpr int S = LV::S;
    const uint32_t inv = thin ? ~0u : 0u;
    for (int w = threadIdx.x; w < g.nwords; w += kThreads) {
        const int y = w / g.WW, x = w - y * g.WW;
        auto seed = [&](int yy, int xx) -> uint32_t {
            if (yy < 0 || yy >= g.H || xx < 0 || xx >= g.WW) return inv;
            uint32_t v = g.I[yy * g.WW + xx] ^ inv;
            if (thin && xx == g.WW - 1) v |= ~g.lastmask;
            return v;
        };
        uint32_t V[R + 1][3];
#pragma unroll
        for (int j = 0; j < 3; ++j) V[0][j] = seed(y, x - 1 + j);
#pragma unroll
        for (int k = 1; k <= R; ++k)
#pragma unroll
            for (int j = 0; j < 3; ++j) V[k][j] = V[k - 1][j] | seed(y - k, x - 1 + j) | seed(y + k, x - 1 + j);

        uint32_t dil = 0, prev = 0;
        uint32_t rs[S];
#pragma unroll
        for (int s = 0; s < S; ++s) rs[s] = 0;
        static_for<L>([&](auto ic) {
            constexpr int i = decltype(ic)::value;
            static_for<2 * R + 1>([&](auto jc) {
                constexpr int dx = decltype(jc)::value - R;
                constexpr int k = LV::kat(i, dx);
                constexpr int kp = (i == 0) ? -1 : LV::kat(i - 1, dx);
                if constexpr (k >= 0 && k != kp) {
                    if constexpr (dx == 0)
                        dil |= V[k][1];
                    else if constexpr (dx > 0)
                        dil |= __funnelshift_r(V[k][1], V[k][2], dx);
                    else
                        dil |= __funnelshift_l(V[k][0], V[k][1], -dx);
                }
            });
            const uint32_t newly = dil & ~prev;
            static_for<S>([&](auto sc) {
                constexpr int s = decltype(sc)::value;
                if constexpr (((i >> s) & 1) != 0) rs[s] |= newly;
            });
            prev = dil;
        });
        // dil = pixels whose clamped distance is <= r^2
        uint32_t blocked;
        if (thin) {
            const uint32_t extra = xmode == 1 ? g.K[w] : (xmode == 2 ? g.XS[w] : 0u);
            blocked = ~dil | extra;
        } else {
            const uint32_t m = xmode == 1 ? ~g.A[w] : (xmode == 2 ? g.XS[w] : ~0u);
            blocked = ~(dil & m);
        }
        g.B[w] = blocked | ~valid_bits(g, x);
#pragma unroll
        for (int s = 0; s < S; ++s) g.R[(size_t)s * g.nwords + w] = rs[s];
        if (save_xs) g.XS[w] = g.I[w];
    }
    return S;
}

__device__ int prep_dispatch(int r, const Img &g, bool thin, int xmode, bool save_xs) {
    switch (r) {
#define TS_PREP_CASE(RR) \
    case RR:             \
        return prep_rank<RR>(g, thin, xmode, save_xs);
        TS_PREP_CASE(1) TS_PREP_CASE(2) TS_PREP_CASE(3) TS_PREP_CASE(4)
        TS_PREP_CASE(5) TS_PREP_CASE(6) TS_PREP_CASE(7) TS_PREP_CASE(8)
        TS_PREP_CASE(9) TS_PREP_CASE(10) TS_PREP_CASE(11) TS_PREP_CASE(12)
        TS_PREP_CASE(13) TS_PREP_CASE(14) TS_PREP_CASE(15) TS_PREP_CASE(16)
#undef TS_PREP_CASE
        default:
            return -1;
    }
}
static_assert(kMaxR == 16, "prep_dispatch covers radii 1..16");

__device__ __forceinline__ void cmp_step(uint32_t &lt, uint32_t &eq, uint32_t nb, uint32_t own) {
    lt |= eq & ~nb & own;   // neighbour < own at the first differing slice
    eq &= ~(nb ^ own);
}

// E planes from rank slices + initial candidate list.  E_k(p) = key(q) < key(p)
// for q = neighbour k, key = (rank, raster index) (topo.py:225,256): ties go to
// the raster-earlier neighbours NW,N,NE,W.
template <int FG>
__device__ void epass_ranks(const Img &g, int S, int t, int *counter) {
    for (int base = 0; base < g.nwords; base += kThreads) {
        const int w = base + threadIdx.x;
        uint32_t c = 0, entry = 0;
        if (w < g.nwords) {
            const int y = w / g.WW, x = w - y * g.WW;
            const uint32_t bw = g.B[w];
            if (~bw & valid_bits(g, x)) {
                uint32_t lt[8], eq[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    lt[k] = 0;
                    eq[k] = ~0u;
                }
                for (int s = S - 1; s >= 0; --s) {
                    const uint32_t *P = g.R + (size_t)s * g.nwords;
                    const Nb nb = nbrs(P, g, y, x);
                    const uint32_t own = P[w];
                    cmp_step(lt[0], eq[0], nb.nw, own);
                    cmp_step(lt[1], eq[1], nb.n, own);
                    cmp_step(lt[2], eq[2], nb.ne, own);
                    cmp_step(lt[3], eq[3], nb.w, own);
                    cmp_step(lt[4], eq[4], nb.e, own);
                    cmp_step(lt[5], eq[5], nb.sw, own);
                    cmp_step(lt[6], eq[6], nb.s, own);
                    cmp_step(lt[7], eq[7], nb.se, own);
                }
                uint4 *ep = reinterpret_cast<uint4 *>(g.E + (size_t)w * 8);
                ep[0] = make_uint4(lt[0] | eq[0], lt[1] | eq[1], lt[2] | eq[2], lt[3] | eq[3]);
                ep[1] = make_uint4(lt[4], lt[5], lt[6], lt[7]);
                c = cand_word<FG>(g, y, x, t);
            }
            g.C[w] = c;
            g.D[w] = c;
            entry = ((uint32_t)y << 16) | (uint32_t)x;
        }
        append(c != 0, entry, g.list, counter);
    }
}

// E planes straight from an int64 priority map (public homotopic_thin /
// homotopic_thicken: arbitrary priorities, topo.py:303-342)
template <int FG>
__device__ void epass_prio(const Img &g, const int64_t *prio, int t, int *counter) {
    const int dy[8] = {-1, -1, -1, 0, 0, 1, 1, 1};
    const int dx[8] = {-1, 0, 1, -1, 1, -1, 0, 1};
    for (int base = 0; base < g.nwords; base += kThreads) {
        const int w = base + threadIdx.x;
        uint32_t c = 0, entry = 0;
        if (w < g.nwords) {
            const int y = w / g.WW, x = w - y * g.WW;
            const uint32_t bw = g.B[w];
            if (~bw & valid_bits(g, x)) {
                uint32_t e[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                const int cnt = min(32, g.W - x * 32);
                for (int i = 0; i < cnt; ++i) {
                    const int col = x * 32 + i;
                    const int64_t pv = prio[(size_t)y * g.W + col];
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const int ny = y + dy[k], nc = col + dx[k];
                        if (ny < 0 || ny >= g.H || nc < 0 || nc >= g.W) continue;
                        const int64_t q = prio[(size_t)ny * g.W + nc];
                        if (q < pv || (q == pv && k < 4)) e[k] |= 1u << i;
                    }
                }
                uint4 *ep = reinterpret_cast<uint4 *>(g.E + (size_t)w * 8);
                ep[0] = make_uint4(e[0], e[1], e[2], e[3]);
                ep[1] = make_uint4(e[4], e[5], e[6], e[7]);
                c = cand_word<FG>(g, y, x, t);
            }
            g.C[w] = c;
            g.D[w] = c;
            entry = ((uint32_t)y << 16) | (uint32_t)x;
        }
        append(c != 0, entry, g.list, counter);
    }
}

// one chaotic-fixpoint update of the decisions of listed word `entry`
template <int FG>
__device__ __forceinline__ bool jacobi_slot(const Img &g, uint32_t entry) {
    const int y = (int)(entry >> 16), x = (int)(entry & 0xFFFFu);
    const int w = y * g.WW + x;
    const Nb i = nbrs(g.I, g, y, x);
    const Nb d = nbrs(g.D, g, y, x);
    const uint4 *ep = reinterpret_cast<const uint4 *>(g.E + (size_t)w * 8);
    const uint4 e0 = ep[0], e1 = ep[1];
    const uint32_t nd =
        g.C[w] & simple_bits<FG>(i.nw ^ (d.nw & e0.x), i.n ^ (d.n & e0.y), i.ne ^ (d.ne & e0.z), i.w ^ (d.w & e0.w),
                                 i.e ^ (d.e & e1.x), i.sw ^ (d.sw & e1.y), i.s ^ (d.s & e1.z), i.se ^ (d.se & e1.w));
    if (nd != g.D[w]) {
        g.D[w] = nd;
        return true;
    }
    return false;
}

// re-examine every dirty word: new candidates -> C, D (= tentative flip), list
template <int FG>
__device__ void rebuild(const Img &g, int t, int *counter) {
    const int n16 = (g.nwords + 15) >> 4;
    uint4 *d4 = reinterpret_cast<uint4 *>(g.dirty);
    for (int q = threadIdx.x; q < n16; q += kThreads) {
        const uint4 v = d4[q];
        if ((v.x | v.y | v.z | v.w) == 0) continue;
        d4[q] = make_uint4(0, 0, 0, 0);
        const uint32_t f[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            if (((f[j >> 2] >> ((j & 3) * 8)) & 0xFFu) == 0) continue;
            const int w = q * 16 + j;
            const int y = w / g.WW, x = w - y * g.WW;
            const uint32_t c = cand_word<FG>(g, y, x, t);
            g.C[w] = c;
            g.D[w] = c;
            if (c) g.list[atomicAdd(counter, 1)] = ((uint32_t)y << 16) | (uint32_t)x;
        }
    }
}

struct Stats {
    long long sweeps, passes, calls;
    long long cyc_prep, cyc_jacobi, cyc_update;   // thread-0 clock64 deltas (stats mode only)
    bool timing;
};

// the priority-ordered flip engine (topo.py:211-258), see file header.
// Precondition (after a __syncthreads): list/C/D built, counters[cur] = size,
// dirty all zero, D zero outside listed words.
template <int FG>
__device__ void engine(const Img &g, int t, long long max_sweeps, int *counters, int &cur, int *err,
                       Stats &st, unsigned long long *s_flips) {
    long long sweeps = 0;
    const long long sweep_cap = (long long)g.H * g.W + 2;   // >= 1 flip per sweep, <= 1 flip per pixel
    while (true) {
        const int n = counters[cur];
        if (n == 0) break;
        if ((max_sweeps >= 0 && sweeps >= max_sweeps) || sweeps >= sweep_cap) {
            if (sweeps >= sweep_cap && (max_sweeps < 0 || sweeps < max_sweeps)) {
                if (threadIdx.x == 0) set_err(err, ERR_SWEEP_CAP);
            }
            for (int s = threadIdx.x; s < n; s += kThreads) {
                const uint32_t e = g.list[s];
                g.D[(int)(e >> 16) * g.WW + (int)(e & 0xFFFFu)] = 0;
            }
            __syncthreads();
            break;
        }
        // chaotic fixpoint over this sweep's candidates
        const long long tj0 = st.timing ? clock64() : 0;
        long long passes = 0;
        const long long cap = 32LL * n + 4;   // DAG depth <= #candidates
        bool bad = false;
        while (true) {
            bool ch = false;
            for (int s = threadIdx.x; s < n; s += kThreads) ch |= jacobi_slot<FG>(g, g.list[s]);
            ++passes;
            if (!__syncthreads_or(ch)) break;
            if (passes > cap) {
                bad = true;
                break;
            }
        }
        if (bad) {
            if (threadIdx.x == 0) set_err(err, ERR_JACOBI_CAP);
            break;
        }
        const long long tj1 = st.timing ? clock64() : 0;
        // apply the sweep's flips, mark the 3x3 word neighbourhoods dirty
        if (threadIdx.x == 0) counters[cur ^ 1] = 0;
        unsigned flips = 0;
        for (int s = threadIdx.x; s < n; s += kThreads) {
            const uint32_t e = g.list[s];
            const int y = (int)(e >> 16), x = (int)(e & 0xFFFFu);
            const int w = y * g.WW + x;
            const uint32_t dw = g.D[w];
            g.dirty[w] = 1;
            if (dw) {
                g.I[w] ^= dw;
                g.D[w] = 0;
                flips += __popc(dw);
                const bool lft = (dw & 1u) && x > 0, rgt = (dw >> 31) && x + 1 < g.WW;
#pragma unroll
                for (int yy = y - 1; yy <= y + 1; ++yy) {
                    if (yy < 0 || yy >= g.H) continue;
                    const int b = yy * g.WW + x;
                    g.dirty[b] = 1;
                    if (lft) g.dirty[b - 1] = 1;
                    if (rgt) g.dirty[b + 1] = 1;
                }
            }
        }
        if (s_flips && flips) atomicAdd(s_flips, (unsigned long long)flips);
        __syncthreads();
        cur ^= 1;
        rebuild<FG>(g, t, &counters[cur]);
        __syncthreads();
        ++sweeps;
        st.passes += passes;
        if (st.timing) {
            const long long tj2 = clock64();
            st.cyc_jacobi += tj1 - tj0;
            st.cyc_update += tj2 - tj1;
        }
    }
    st.sweeps += sweeps;
    st.calls += 1;
}

template <int FG>
__device__ void run_stage(const Img &g, int r, bool thin, int xmode, bool save_xs, int *counters, int &cur,
                          int *err, Stats &st, unsigned long long *s_flips) {
    if (threadIdx.x == 0) counters[cur] = 0;
    const long long tp0 = st.timing ? clock64() : 0;
    const int S = prep_dispatch(r, g, thin, xmode, save_xs);
    __syncthreads();
    epass_ranks<FG>(g, S, thin ? 1 : 0, &counters[cur]);
    __syncthreads();
    if (st.timing) st.cyc_prep += clock64() - tp0;
    engine<FG>(g, thin ? 1 : 0, -1, counters, cur, err, st, s_flips);
}

template <int FG>
__global__ void __launch_bounds__(kThreads, 1) hasf_kernel(const KParams p) {
    extern __shared__ __align__(16) uint32_t smem[];
    __shared__ int s_img;
    __shared__ int s_counters[2];
    __shared__ unsigned long long s_flips;

    uint32_t *cta = p.gws + (size_t)blockIdx.x * (size_t)p.gws_stride;
    auto buf = [&](int b) -> uint32_t * { return ((p.smem_mask >> b) & 1u) ? smem + p.off[b] : cta + p.off[b]; };
    Img g;
    g.I = buf(B_I);
    g.D = buf(B_D);
    g.C = buf(B_C);
    g.dirty = reinterpret_cast<uint8_t *>(buf(B_DIRTY));
    g.list = buf(B_LIST);
    g.E = buf(B_E);
    g.B = buf(B_B);
    g.XS = buf(B_XS);
    g.R = buf(B_R);
    g.K = buf(B_K);
    g.A = buf(B_A);
    g.H = p.H;
    g.W = p.W;
    g.WW = p.WW;
    g.nwords = p.nwords;
    g.lastmask = (p.W & 31) ? ((1u << (p.W & 31)) - 1u) : ~0u;
    const bool has_k = p.keep != nullptr, has_a = p.avoid != nullptr;

    for (;;) {
        if (threadIdx.x == 0) s_img = atomicAdd(p.counter, 1);
        __syncthreads();
        const int img = s_img;
        if (img >= p.n) break;
        const size_t pix = (size_t)img * p.H * p.W;

        // ---- load + validate -------------------------------------------------
        pack_plane(p.in + pix, g.I, g, p.err, ERR_NOT_BINARY);
        if (p.mode == MODE_THIN) {
            pack_plane(p.keep + pix, g.B, g, p.err, ERR_CONSTRAINT_NOT_BINARY);
        } else if (p.mode == MODE_THICKEN) {
            pack_plane(p.keep + pix, g.B, g, p.err, ERR_CONSTRAINT_NOT_BINARY);
        } else {
            if (has_k) pack_plane(p.keep + pix, g.K, g, p.err, ERR_CONSTRAINT_NOT_BINARY);
            if (has_a) pack_plane(p.avoid + pix, g.A, g, p.err, ERR_CONSTRAINT_NOT_BINARY);
        }
        for (int w = threadIdx.x; w < g.nwords; w += kThreads) g.D[w] = 0;
        {
            const int n16 = (g.nwords + 15) >> 4;
            uint4 *d4 = reinterpret_cast<uint4 *>(g.dirty);
            for (int q = threadIdx.x; q < n16; q += kThreads) d4[q] = make_uint4(0, 0, 0, 0);
        }
        if (threadIdx.x == 0) {
            s_counters[0] = 0;
            s_flips = 0;
        }
        __syncthreads();
        for (int w = threadIdx.x; w < g.nwords; w += kThreads) {
            const uint32_t X = g.I[w];
            if (p.mode == MODE_THIN) {
                if (g.B[w] & ~X) set_err(p.err, ERR_KEEP_NOT_OBJECT);          // topo.py:264-265
            } else if (p.mode == MODE_THICKEN) {
                const uint32_t allowed = g.B[w];
                if (X & ~allowed) set_err(p.err, ERR_ALLOWED_NOT_SUPERSET);    // topo.py:332-333
                g.B[w] = ~allowed;   // blocked = not allowed; padding bits blocked
            } else {
                const uint32_t K = has_k ? g.K[w] : 0u, A = has_a ? g.A[w] : 0u;
                if (K & A) set_err(p.err, ERR_KEEP_AVOID);                     // smoothing.py:201-202
                if (K & ~X) set_err(p.err, ERR_KEEP_NOT_OBJECT);               // smoothing.py:203-204
                if (A & X) set_err(p.err, ERR_AVOID_ON_OBJECT);                // smoothing.py:205-206
            }
        }
        __syncthreads();

        Stats st{0, 0, 0, 0, 0, 0, p.stats != nullptr};
        const long long t_img0 = st.timing ? clock64() : 0;
        int cur = 0;
        unsigned long long *fl = p.stats ? &s_flips : nullptr;
        if (p.mode == MODE_HASF) {
            for (int r = p.r_first; r <= p.r_last; ++r) {
                if (p.do_cut) {   // smoothing.py:127-135
                    run_stage<FG>(g, r, true, has_k ? 1 : 0, true, s_counters, cur, p.err, st, fl);
                    run_stage<FG>(g, r, false, 2, false, s_counters, cur, p.err, st, fl);
                }
                if (p.do_fill) {  // smoothing.py:138-146
                    run_stage<FG>(g, r, false, has_a ? 1 : 0, true, s_counters, cur, p.err, st, fl);
                    run_stage<FG>(g, r, true, 2, false, s_counters, cur, p.err, st, fl);
                }
            }
        } else {
            const int t = p.mode == MODE_THIN ? 1 : 0;
            epass_prio<FG>(g, p.prio + pix, t, &s_counters[cur]);
            __syncthreads();
            engine<FG>(g, t, p.max_sweeps, s_counters, cur, p.err, st, fl);
        }

        unpack_plane(g.I, p.out + pix, g);
        if (threadIdx.x == 0 && p.stats) {
            long long *sp = p.stats + (size_t)img * kStatFields;
            sp[0] = st.sweeps;
            sp[1] = st.passes;
            sp[2] = st.calls;
            sp[3] = (long long)s_flips;
            sp[4] = st.cyc_prep;
            sp[5] = st.cyc_jacobi;
            sp[6] = st.cyc_update;
            sp[7] = clock64() - t_img0;
        }
        __syncthreads();
    }
}

template __global__ void hasf_kernel<8>(const KParams);
template __global__ void hasf_kernel<4>(const KParams);

// ---- launch helper (host) ------------------------------------------------
cudaError_t launch_hasf(const KParams &p, int fg, int grid, size_t smem_bytes, cudaStream_t stream) {
    const void *fn = fg == 8 ? (const void *)hasf_kernel<8> : (const void *)hasf_kernel<4>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes);
    if (e != cudaSuccess) return e;
    void *args[] = {(void *)&p};
    return cudaLaunchKernel(fn, dim3(grid), dim3(kThreads), args, smem_bytes, stream);
}

int hasf_threads() { return kThreads; }

cudaError_t hasf_occupancy(int fg, size_t smem_bytes, int *blocks_per_sm) {
    const void *fn = fg == 8 ? (const void *)hasf_kernel<8> : (const void *)hasf_kernel<4>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, fn, kThreads, smem_bytes);
}

}  // namespace ts
