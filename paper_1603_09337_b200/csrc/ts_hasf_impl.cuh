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
// topo.py:245-257), found through a 1-bit-per-word dirty bitmap.
//
// Memory: the hot planes (image I, decisions D, candidates C, blocked B, the
// dirty bitmap and the active-word list) live in shared memory whenever they
// fit (the HOT variant; accessed as true LDS/STS); the E planes, rank slices
// and saved image go to shared memory if space remains, else to the CTA's
// slice of an L2-resident global workspace.  Thread <-> word mappings are
// always lane-consecutive, so neighbour-word loads are bank-conflict free.
#pragma once
#include <cuda_runtime.h>
#include "ts_common.cuh"
#include "ts_internal.h"

namespace ts {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
#ifndef TS_MIN_BLOCKS
#define TS_MIN_BLOCKS 1
#endif
constexpr int kMinBlocks = TS_MIN_BLOCKS;   // resident images per SM the register budget targets

struct Img {
    uint32_t *I, *D, *B, *dirty;              // hot planes
    uint8_t *mark;                            // hot: fixpoint worklist stamps
    uint32_t *list, *E, *XS, *R, *K, *A;      // smem or global
    int H, W, WW, nwords;
    uint32_t lastmask;   // valid bits of the last word of a row
    int ww_shift;        // log2(WW) if WW is a power of two, else -1
};

__device__ __forceinline__ void set_err(int *err, int code) { atomicCAS(err, 0, code); }

__device__ __forceinline__ uint32_t valid_bits(const Img &g, int x) { return x == g.WW - 1 ? g.lastmask : ~0u; }

__device__ __forceinline__ void word_yx(const Img &g, int w, int &y, int &x) {
    if (g.ww_shift >= 0) {
        y = w >> g.ww_shift;
        x = w & (g.WW - 1);
    } else {
        y = w / g.WW;
        x = w - y * g.WW;
    }
}

__device__ __forceinline__ uint32_t ldw(const uint32_t *P, const Img &g, int y, int x) {
    return (y < 0 || y >= g.H || x < 0 || x >= g.WW) ? 0u : P[y * g.WW + x];
}

struct Nb {
    uint32_t nw, n, ne, w, e, sw, s, se;
    uint32_t m;   // the centre word itself
};

__device__ __forceinline__ Nb shifts(uint32_t u0, uint32_t u1, uint32_t u2, uint32_t m0, uint32_t m1, uint32_t m2,
                                     uint32_t d0, uint32_t d1, uint32_t d2) {
    Nb r;
    r.nw = from_west(u0, u1);
    r.n = u1;
    r.ne = from_east(u1, u2);
    r.w = from_west(m0, m1);
    r.e = from_east(m1, m2);
    r.sw = from_west(d0, d1);
    r.s = d1;
    r.se = from_east(d1, d2);
    r.m = m1;
    return r;
}

// neighbour bit-words of the 32 pixels of word (y, x); outside the window = 0
__device__ __forceinline__ Nb nbrs(const uint32_t *P, const Img &g, int y, int x) {
    const bool up = y > 0, dn = y + 1 < g.H, lf = x > 0, rt = x + 1 < g.WW;
    const uint32_t *row = P + y * g.WW + x;
    const uint32_t u1 = up ? row[-g.WW] : 0u, d1 = dn ? row[g.WW] : 0u, m1 = row[0];
    const uint32_t u0 = (up && lf) ? row[-g.WW - 1] : 0u, u2 = (up && rt) ? row[-g.WW + 1] : 0u;
    const uint32_t m0 = lf ? row[-1] : 0u, m2 = rt ? row[1] : 0u;
    const uint32_t d0 = (dn && lf) ? row[g.WW - 1] : 0u, d2 = (dn && rt) ? row[g.WW + 1] : 0u;
    return shifts(u0, u1, u2, m0, m1, m2, d0, d1, d2);
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
__device__ __forceinline__ void pack_plane(const uint8_t *src, uint32_t *dst, const Img &g, int *err, int code) {
    for (int w = threadIdx.x; w < g.nwords; w += kThreads) {
        int y, x;
        word_yx(g, w, y, x);
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

__device__ __forceinline__ void unpack_plane(const uint32_t *src, uint8_t *dst, const Img &g) {
    for (int w = threadIdx.x; w < g.nwords; w += kThreads) {
        int y, x;
        word_yx(g, w, y, x);
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

// warp-aggregated append to the active-word list (all 32 lanes must call);
// entries keep lane order, so a warp's entries are consecutive words
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
__device__ __forceinline__ int prep_rank(const Img &g, bool thin, int xmode, bool save_xs) {
    using LV = Lev<R>;
    constexpr int L = LV::L;
    constexpr int S = LV::S;
    const uint32_t inv = thin ? ~0u : 0u;
    for (int w = threadIdx.x; w < g.nwords; w += kThreads) {
        int y, x;
        word_yx(g, w, y, x);
        const bool lf = x > 0, rt = x + 1 < g.WW;
        const uint32_t padl = inv, padr = (thin && x + 2 == g.WW) ? ~g.lastmask : 0u;
        const uint32_t padc = (thin && x + 1 == g.WW) ? ~g.lastmask : 0u;
        auto seed3 = [&](int yy, uint32_t &a, uint32_t &b, uint32_t &c) {
            if (yy < 0 || yy >= g.H) {
                a = b = c = inv;
                return;
            }
            const uint32_t *row = g.I + yy * g.WW + x;
            a = lf ? (row[-1] ^ inv) : padl;
            b = (row[0] ^ inv) | padc;
            c = rt ? ((row[1] ^ inv) | padr) : inv;
        };
        uint32_t V[R + 1][3];
        seed3(y, V[0][0], V[0][1], V[0][2]);
#pragma unroll
        for (int k = 1; k <= R; ++k) {
            uint32_t a0, a1, a2, b0, b1, b2;
            seed3(y - k, a0, a1, a2);
            seed3(y + k, b0, b1, b2);
            V[k][0] = V[k - 1][0] | a0 | b0;
            V[k][1] = V[k - 1][1] | a1 | b1;
            V[k][2] = V[k - 1][2] | a2 | b2;
        }
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

__device__ __forceinline__ int prep_dispatch(int r, const Img &g, bool thin, int xmode, bool save_xs) {
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
__device__ __forceinline__ void epass_ranks(const Img &g, int S, int t, int *counter) {
    for (int base = 0; base < g.nwords; base += kThreads) {
        const int w = base + threadIdx.x;
        uint32_t c = 0, entry = 0;
        if (w < g.nwords) {
            int y, x;
            word_yx(g, w, y, x);
            const uint32_t bw = g.B[w];
            if (~bw & valid_bits(g, x)) {
                c = cand_word<FG>(g, y, x, t);
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
            }
            g.D[w] = c;
            entry = ((uint32_t)y << 16) | (uint32_t)x;
        }
        append(c != 0, entry, g.list, counter);
    }
}

// E planes straight from an int64 priority map (public homotopic_thin /
// homotopic_thicken: arbitrary priorities, topo.py:303-342)
template <int FG>
__device__ __forceinline__ void epass_prio(const Img &g, const int64_t *prio, int t, int *counter) {
    const int dy[8] = {-1, -1, -1, 0, 0, 1, 1, 1};
    const int dx[8] = {-1, 0, 1, -1, 1, -1, 0, 1};
    for (int base = 0; base < g.nwords; base += kThreads) {
        const int w = base + threadIdx.x;
        uint32_t c = 0, entry = 0;
        if (w < g.nwords) {
            int y, x;
            word_yx(g, w, y, x);
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
            g.D[w] = c;
            entry = ((uint32_t)y << 16) | (uint32_t)x;
        }
        append(c != 0, entry, g.list, counter);
    }
}

// sweep-constant data of one listed word: neighbour image words, precedence
// masks and candidates (cached in registers for the thread's first slot)
struct Slot {
    int w, y, x;
    bool up, dn, lf, rt;
    Nb in;          // image neighbours at the sweep start
    uint4 e0, e1;   // E masks
    uint32_t c;     // candidates
    uint32_t d;     // current decision (only this thread writes D[w])
};

template <int FG>
__device__ __forceinline__ void load_slot(const Img &g, uint32_t entry, Slot &s, int t) {
    s.y = (int)(entry >> 16);
    s.x = (int)(entry & 0xFFFFu);
    s.w = s.y * g.WW + s.x;
    s.up = s.y > 0;
    s.dn = s.y + 1 < g.H;
    s.lf = s.x > 0;
    s.rt = s.x + 1 < g.WW;
    s.in = nbrs(g.I, g, s.y, s.x);
    const uint4 *ep = reinterpret_cast<const uint4 *>(g.E + (size_t)s.w * 8);
    s.e0 = ep[0];
    s.e1 = ep[1];
    // the sweep's candidates, recomputed from the sweep-start image
    const uint32_t pre = valid_bits(g, s.x) & (t ? s.in.m : ~s.in.m) & ~g.B[s.w];
    const Nb &i = s.in;
    s.c = pre & simple_bits<FG>(i.nw, i.n, i.ne, i.w, i.e, i.sw, i.s, i.se);
    s.d = g.D[s.w];
}

// position + current decision only (apply phase: must not read the image,
// which other threads are updating)
__device__ __forceinline__ void load_slot_pos(const Img &g, uint32_t entry, Slot &s) {
    s.y = (int)(entry >> 16);
    s.x = (int)(entry & 0xFFFFu);
    s.w = s.y * g.WW + s.x;
    s.up = s.y > 0;
    s.dn = s.y + 1 < g.H;
    s.lf = s.x > 0;
    s.rt = s.x + 1 < g.WW;
    s.d = g.D[s.w];
}

// stamp the word neighbourhood affected by changed decision bits `chg` of a
// slot for re-evaluation in the next pass (byte stores, races benign)
__device__ __forceinline__ void stamp_slot(const Img &g, const Slot &s, uint32_t chg, uint8_t v) {
    const int xa = ((chg & 1u) && s.lf) ? s.x - 1 : s.x;
    const int xb = ((chg >> 31) && s.rt) ? s.x + 1 : s.x;
    const int ya = s.up ? s.y - 1 : s.y, yb = s.dn ? s.y + 1 : s.y;
    for (int yy = ya; yy <= yb; ++yy)
        for (int xx = xa; xx <= xb; ++xx) g.mark[yy * g.WW + xx] = v;
}

// one chaotic-fixpoint update of a slot's decisions; with STAMP, words whose
// inputs changed are stamped for the next pass of the worklist
template <int FG, bool STAMP>
__device__ __forceinline__ bool update_slot(const Img &g, Slot &s, uint8_t stamp = 0) {
    const uint32_t *row = g.D + s.w;
    const int WW = g.WW;
    const uint32_t u1 = s.up ? row[-WW] : 0u, d1 = s.dn ? row[WW] : 0u;
    const uint32_t u0 = (s.up && s.lf) ? row[-WW - 1] : 0u, u2 = (s.up && s.rt) ? row[-WW + 1] : 0u;
    const uint32_t m0 = s.lf ? row[-1] : 0u, m2 = s.rt ? row[1] : 0u;
    const uint32_t d0 = (s.dn && s.lf) ? row[WW - 1] : 0u, d2 = (s.dn && s.rt) ? row[WW + 1] : 0u;
    const Nb d = shifts(u0, u1, u2, m0, s.d, m2, d0, d1, d2);   // W/E inside the word: own decisions
    const Nb &i = s.in;
    const uint32_t nd =
        s.c & simple_bits<FG>(i.nw ^ (d.nw & s.e0.x), i.n ^ (d.n & s.e0.y), i.ne ^ (d.ne & s.e0.z),
                              i.w ^ (d.w & s.e0.w), i.e ^ (d.e & s.e1.x), i.sw ^ (d.sw & s.e1.y),
                              i.s ^ (d.s & s.e1.z), i.se ^ (d.se & s.e1.w));
    if (nd != s.d) {
        if constexpr (STAMP) stamp_slot(g, s, nd ^ s.d, stamp);
        s.d = nd;
        g.D[s.w] = nd;
        return true;
    }
    return false;
}

// mark the bitmap bits of words [w0, w1] (consecutive, at most 3)
__device__ __forceinline__ void mark_words(const Img &g, int w0, int w1) {
    const int q0 = w0 >> 5, q1 = w1 >> 5;
    if (q0 == q1) {
        atomicOr(&g.dirty[q0], (0xFFFFFFFFu >> (31 - (w1 - w0))) << (w0 & 31));
    } else {
        atomicOr(&g.dirty[q0], 0xFFFFFFFFu << (w0 & 31));
        atomicOr(&g.dirty[q1], 0xFFFFFFFFu >> (31 - (w1 & 31)));
    }
}

// flips of one slot: I ^= d, D = 0, dirty 3x3 word neighbourhood
__device__ __forceinline__ unsigned apply_slot(const Img &g, const Slot &s) {
    const uint32_t dw = s.d;
    if (!dw) return 0;
    g.I[s.w] ^= dw;
    g.D[s.w] = 0;
    const int xa = ((dw & 1u) && s.lf) ? s.x - 1 : s.x;
    const int xb = ((dw >> 31) && s.rt) ? s.x + 1 : s.x;
    const int ya = s.up ? s.y - 1 : s.y, yb = s.dn ? s.y + 1 : s.y;
    for (int yy = ya; yy <= yb; ++yy) mark_words(g, yy * g.WW + xa, yy * g.WW + xb);
    return __popc(dw);
}

// re-examine every dirty word (warp per 32-word bitmap group, lane = word):
// new candidates -> C, D (= tentative flip), list
template <int FG>
__device__ __forceinline__ void rebuild(const Img &g, int t, int *counter) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nq = (g.nwords + 31) >> 5;
    for (int q = warp; q < nq; q += kWarps) {
        const uint32_t bits = g.dirty[q];
        if (bits == 0) continue;   // warp-uniform
        __syncwarp();
        if (lane == 0) g.dirty[q] = 0;
        const int w = q * 32 + lane;
        uint32_t c = 0, entry = 0;
        if ((bits >> lane) & 1u) {
            int y, x;
            word_yx(g, w, y, x);
            c = cand_word<FG>(g, y, x, t);
            g.D[w] = c;
            entry = ((uint32_t)y << 16) | (uint32_t)x;
        }
        append(c != 0, entry, g.list, counter);
    }
}

struct Stats {
    long long sweeps, passes, calls;
    long long cyc_prep, cyc_jacobi, cyc_update;   // thread-0 clock64 deltas (stats mode only)
    long long cyc_tiny, n_tiny, pass_tiny;        // sweeps with <= 32 listed words
    long long cyc_dense, n_dense, pass_dense;     // sweeps with > kThreads listed words
    long long cyc_rank;                           // clamped-EDT part of prep
    long long evals;                              // slot evaluations in worklist passes
    bool timing;
};

// the priority-ordered flip engine (topo.py:211-258), see file header.
// Precondition (after a __syncthreads): list/C/D built, counters[cur] = size,
// dirty all zero, D zero outside listed words.
template <int FG>
__device__ __forceinline__ void engine(const Img &g, int t, long long max_sweeps, int *counters, int &cur, int *err,
                                       Stats &st, unsigned long long *s_flips, int *s_bad, int &pc,
                                       unsigned long long *s_evals) {
    const int tid = threadIdx.x, warp = tid >> 5;
    long long sweeps = 0;
    const long long sweep_cap = (long long)g.H * g.W + 2;   // >= 1 flip per sweep, <= 1 flip per pixel
    while (true) {
        const int n = counters[cur];
        if (n == 0) break;
        if ((max_sweeps >= 0 && sweeps >= max_sweeps) || sweeps >= sweep_cap) {
            if (sweeps >= sweep_cap && (max_sweeps < 0 || sweeps < max_sweeps)) {
                if (tid == 0) set_err(err, ERR_SWEEP_CAP);
            }
            for (int s = tid; s < n; s += kThreads) {
                const uint32_t e = g.list[s];
                g.D[(int)(e >> 16) * g.WW + (int)(e & 0xFFFFu)] = 0;
            }
            __syncthreads();
            break;
        }
        const long long tj0 = st.timing ? clock64() : 0;
        const long long cap = 32LL * n + 4;   // DAG depth <= #candidates
        long long passes = 0;
        unsigned flips = 0;
        Slot s0;
        const bool has0 = tid < n;
        if (has0) load_slot<FG>(g, g.list[tid], s0, t);
        if (n <= 32) {
            // tiny sweep: one warp iterates to the fixpoint with warp syncs only
            if (warp == 0) {
                bool bad = false;
                while (true) {
                    const bool ch = has0 && update_slot<FG, false>(g, s0);
                    ++passes;
                    __syncwarp();
                    if (!__any_sync(0xffffffffu, ch)) break;
                    if (passes > cap) {
                        bad = true;
                        break;
                    }
                }
                if (tid == 0) {
                    *s_bad = bad ? 1 : 0;
                    counters[cur ^ 1] = 0;
                }
                if (has0) flips += apply_slot(g, s0);
            }
            __syncthreads();
        } else {
            // worklist passes: pass 1 evaluates every slot; later passes only the
            // words stamped (by a changed neighbour decision) with the current
            // pass number.  A pass without change is a fixpoint: every slot was
            // last evaluated after its last input change.
            bool bad = false;
            while (true) {
                const uint8_t cur_stamp = (uint8_t)pc, next_stamp = (uint8_t)(pc + 1);
                const bool full = passes == 0;
                bool ch = false;
                int ev = 0;
                if (has0 && (full || (uint8_t)(g.mark[s0.w] - cur_stamp) <= 1)) {
                    ch = update_slot<FG, true>(g, s0, next_stamp);
                    ++ev;
                }
                for (int sl = tid + kThreads; sl < n; sl += kThreads) {
                    const uint32_t e = g.list[sl];
                    if (!full) {
                        const int w = (int)(e >> 16) * g.WW + (int)(e & 0xFFFFu);
                        if ((uint8_t)(g.mark[w] - cur_stamp) > 1) continue;
                    }
                    Slot s;
                    load_slot<FG>(g, e, s, t);
                    ch |= update_slot<FG, true>(g, s, next_stamp);
                    ++ev;
                }
                if (st.timing) {
                    ev = __reduce_add_sync(0xffffffffu, ev);
                    if ((tid & 31) == 0 && ev) atomicAdd(s_evals, (unsigned long long)ev);
                }
                ++passes;
                ++pc;
                if (!__syncthreads_or(ch)) break;
                if (passes > cap) {
                    bad = true;
                    break;
                }
            }
            if (tid == 0) {
                *s_bad = bad ? 1 : 0;
                counters[cur ^ 1] = 0;
            }
            if (has0) flips += apply_slot(g, s0);
            for (int sl = tid + kThreads; sl < n; sl += kThreads) {
                Slot s;
                load_slot_pos(g, g.list[sl], s);
                flips += apply_slot(g, s);
            }
            __syncthreads();
        }
        if (*s_bad) {
            if (tid == 0) set_err(err, ERR_JACOBI_CAP);
            break;
        }
        if (s_flips && flips) atomicAdd(s_flips, (unsigned long long)flips);
        const long long tj1 = st.timing ? clock64() : 0;
        cur ^= 1;
        rebuild<FG>(g, t, &counters[cur]);
        __syncthreads();
        ++sweeps;
        st.passes += passes;
        if (st.timing) {
            const long long tj2 = clock64();
            st.cyc_jacobi += tj1 - tj0;
            st.cyc_update += tj2 - tj1;
            if (n <= 32) {
                st.cyc_tiny += tj1 - tj0;
                st.n_tiny += 1;
                st.pass_tiny += passes;
            } else if (n > kThreads) {
                st.cyc_dense += tj1 - tj0;
                st.n_dense += 1;
                st.pass_dense += passes;
            }
        }
    }
    st.sweeps += sweeps;
    st.calls += 1;
}

template <int FG>
__device__ __forceinline__ void run_stage(const Img &g, int r, bool thin, int xmode, bool save_xs, int *counters,
                                          int &cur, int *err, Stats &st, unsigned long long *s_flips, int *s_bad,
                                          int &pc, unsigned long long *s_evals) {
    if (threadIdx.x == 0) counters[cur] = 0;
    const long long tp0 = st.timing ? clock64() : 0;
    const int S = prep_dispatch(r, g, thin, xmode, save_xs);
    __syncthreads();
    if (st.timing) st.cyc_rank += clock64() - tp0;
    epass_ranks<FG>(g, S, thin ? 1 : 0, &counters[cur]);
    __syncthreads();
    if (st.timing) st.cyc_prep += clock64() - tp0;
    engine<FG>(g, thin ? 1 : 0, -1, counters, cur, err, st, s_flips, s_bad, pc, s_evals);
}

template <int FG, bool HOT>
__global__ void __launch_bounds__(kThreads, kMinBlocks) hasf_kernel(const KParams p) {
    extern __shared__ __align__(16) uint32_t smem[];
    __shared__ int s_img;
    __shared__ int s_counters[2];
    __shared__ int s_bad;
    __shared__ unsigned long long s_flips;
    __shared__ unsigned long long s_evals;

    uint32_t *cta = p.gws + (size_t)blockIdx.x * (size_t)p.gws_stride;
    auto buf = [&](int b) -> uint32_t * { return ((p.smem_mask >> b) & 1u) ? smem + p.off[b] : cta + p.off[b]; };
    Img g;
    if constexpr (HOT) {   // derived from the shared array: compiled to LDS/STS
        g.I = smem + p.off[B_I];
        g.D = smem + p.off[B_D];
        g.B = smem + p.off[B_B];
        g.dirty = smem + p.off[B_DIRTY];
        g.mark = reinterpret_cast<uint8_t *>(smem + p.off[B_MARK]);
    } else {
        g.I = buf(B_I);
        g.D = buf(B_D);
        g.B = buf(B_B);
        g.dirty = buf(B_DIRTY);
        g.mark = reinterpret_cast<uint8_t *>(buf(B_MARK));
    }
    g.list = buf(B_LIST);
    g.E = buf(B_E);
    g.XS = buf(B_XS);
    g.R = buf(B_R);
    g.K = buf(B_K);
    g.A = buf(B_A);
    g.H = p.H;
    g.W = p.W;
    g.WW = p.WW;
    g.nwords = p.nwords;
    g.lastmask = (p.W & 31) ? ((1u << (p.W & 31)) - 1u) : ~0u;
    g.ww_shift = (p.WW & (p.WW - 1)) == 0 ? __ffs(p.WW) - 1 : -1;
    const bool has_k = p.keep != nullptr, has_a = p.avoid != nullptr;
    const int nq = (g.nwords + 31) >> 5;

    for (;;) {
        if (threadIdx.x == 0) s_img = atomicAdd(p.counter, 1);
        __syncthreads();
        const int img = s_img;
        if (img >= p.n) break;
        const size_t pix = (size_t)img * p.H * p.W;

        // ---- load + validate -------------------------------------------------
        pack_plane(p.in + pix, g.I, g, p.err, ERR_NOT_BINARY);
        if (p.mode == MODE_THIN || p.mode == MODE_THICKEN) {
            pack_plane(p.keep + pix, g.B, g, p.err, ERR_CONSTRAINT_NOT_BINARY);
        } else {
            if (has_k) pack_plane(p.keep + pix, g.K, g, p.err, ERR_CONSTRAINT_NOT_BINARY);
            if (has_a) pack_plane(p.avoid + pix, g.A, g, p.err, ERR_CONSTRAINT_NOT_BINARY);
        }
        for (int w = threadIdx.x; w < g.nwords; w += kThreads) g.D[w] = 0;
        for (int q = threadIdx.x; q < nq; q += kThreads) g.dirty[q] = 0;
        for (int q = threadIdx.x; q < (g.nwords + 15) >> 4; q += kThreads)
            reinterpret_cast<uint4 *>(g.mark)[q] = make_uint4(0, 0, 0, 0);
        if (threadIdx.x == 0) {
            s_counters[0] = 0;
            s_flips = 0;
            s_evals = 0;
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

        Stats st{};
        st.timing = p.stats != nullptr;
        const long long t_img0 = st.timing ? clock64() : 0;
        int cur = 0;
        int pc = 2;   // worklist pass counter (stamps are its low byte; marks start at 0)
        unsigned long long *fl = p.stats ? &s_flips : nullptr;
        if (p.mode == MODE_HASF) {
            // stage table: (thin, xmode, save_xs) for S1/S3 (cutting) and S5/S7 (filling)
            const int first = p.do_cut ? 0 : 2, last = p.do_fill ? 3 : 1;
            for (int r = p.r_first; r <= p.r_last; ++r) {
                for (int stg = first; stg <= last; ++stg) {
                    const bool thin = stg == 0 || stg == 3;
                    const int xmode = (stg == 1 || stg == 3) ? 2 : ((stg == 0 ? has_k : has_a) ? 1 : 0);
                    const bool save = stg == 0 || stg == 2;
                    run_stage<FG>(g, r, thin, xmode, save, s_counters, cur, p.err, st, fl, &s_bad, pc, &s_evals);
                }
            }
        } else {
            const int t = p.mode == MODE_THIN ? 1 : 0;
            epass_prio<FG>(g, p.prio + pix, t, &s_counters[cur]);
            __syncthreads();
            engine<FG>(g, t, p.max_sweeps, s_counters, cur, p.err, st, fl, &s_bad, pc, &s_evals);
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
            sp[8] = st.cyc_tiny;
            sp[9] = st.n_tiny;
            sp[10] = st.pass_tiny;
            sp[11] = st.cyc_dense;
            sp[12] = st.n_dense;
            sp[13] = st.pass_dense;
            sp[14] = st.cyc_rank;
            sp[15] = (long long)s_evals;
        }
        __syncthreads();
    }
}

// per-variant host entry points, one translation unit each (ts_hasf_<fg><h|g>.cu)
#define TS_DEFINE_HASF_VARIANT(FG, HOT, SUFFIX)                                                              \
    cudaError_t launch_hasf_##SUFFIX(const KParams &p, int grid, size_t smem_bytes, cudaStream_t stream) {    \
        const void *fn = (const void *)hasf_kernel<FG, HOT>;                                                  \
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes); \
        if (e != cudaSuccess) return e;                                                                       \
        void *args[] = {(void *)&p};                                                                          \
        return cudaLaunchKernel(fn, dim3(grid), dim3(kThreads), args, smem_bytes, stream);                   \
    }                                                                                                         \
    cudaError_t occupancy_hasf_##SUFFIX(size_t smem_bytes, int *blocks) {                                     \
        const void *fn = (const void *)hasf_kernel<FG, HOT>;                                                  \
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes); \
        if (e != cudaSuccess) return e;                                                                       \
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, fn, kThreads, smem_bytes);              \
    }

}  // namespace ts
