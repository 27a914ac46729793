// Fused per-image HASF kernel for sm_100a (body; instantiated per variant in
// ts_hasf_<fg><h|g>.cu).
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
// computed once per engine call from the rank slices.  Any evaluation order
// reaches the unique solution.  A pixel reads only the decisions of the
// neighbours that precede it, so when a word's decisions change only the
// neighbour words named by its own E masks can be affected: those are
// re-evaluated, and a pass that affects no candidate word certifies the
// fixpoint.  Sweep modes:
//   dense  (many candidates): one strip-walk pass -- every thread walks its
//          vertical strip of words with a sliding 3-row register window
//          (updates propagate down the strip), byte-stamping the affected
//          words; a scan lists them; then claim passes: one listed word per
//          thread, changed words claim their affected candidate words into
//          the next pass's list (claim bitmap: first claimant appends);
//   list   (fewer candidates): claim passes from the sweep's word list, then
//          the 3x3 word neighbourhoods of the flips (the reference's
//          re-queue, topo.py:245-257) are re-examined through a dirty bitmap
//          compacted into a word list;
//   tiny   (<= 32 words): warp 0 runs whole sweeps alone, warp syncs only.
//
// Layout: every plane is padded with one zero row above and below and
// one zero word between rows (row stride S >= WW + 1, chosen on the host so
// the 32 lanes of a warp touch 32 distinct banks), so neighbour and disc
// accesses need no bounds checks.  The hot planes (I, D, C, B, the dirty /
// claim bitmaps and the stamps) live in shared memory when they fit (HOT
// variant, accessed as LDS/STS); lists, saved image, E and rank slices follow
// in shared memory while they fit, the rest in the CTA's slice of an
// L2-resident global workspace.  The phase functions take the per-CTA View by
// reference from shared memory (a by-value View cost 15% in ABI copies).
#pragma once
#include <cuda_runtime.h>
#include <mutex>
#include "ts_common.cuh"
#include "ts_internal.h"

// The body is compiled once per (threads per CTA, CTAs per SM) flavour, each in
// its own namespace: 512 x 1 (default) and 256 x 2 (small images, two per SM).
#ifndef TS_IMPL_THREADS
#define TS_IMPL_THREADS 512
#define TS_IMPL_MINB 1
#define TS_IMPL_NS v512
#endif

namespace ts {
namespace TS_IMPL_NS {

constexpr int kThreads = TS_IMPL_THREADS;
// E4: only the 4 precedence masks towards the raster-earlier neighbours
// (NW, N, NE, W) are stored, for EVERY word; the other 4 follow by
// antisymmetry of the (unique) keys from the neighbours' masks (load_e).
// Half the E footprint: fits shared memory for small images (256-thread
// variant) and keeps large images' L2 working set down (team variant).
#ifndef TS_IMPL_E4
#define TS_IMPL_E4 0
#endif
constexpr bool kE4 = TS_IMPL_E4 != 0;
constexpr int kEWords = kE4 ? 4 : 8;   // E words per bit-plane word
#ifndef TS_PREP_U4
#define TS_PREP_U4 1   // fused prep: 4 comparators per word, lower masks by antisymmetry (E8 variants)
#endif
constexpr int kWarps = kThreads / 32;
constexpr int kMinBlocks = TS_IMPL_MINB;   // resident images per SM the register budget targets

struct Img {
    uint32_t *I, *D, *C, *dirty;          // hot planes
    uint8_t *mark;                        // hot: worklist pass stamps, one byte per word
    uint32_t *B, *list, *E, *XS, *R, *K, *A;  // smem or global (generic pointers)
    uint32_t *claim;                      // 2 claim bitmaps of the compacted passes, mw words each
    int mw;
    int H, W, WW;
    int S;          // padded row stride (words)
    int plen;       // padded plane length (words)
    int org;        // index of word (0, 0)
    uint32_t lastmask;   // valid bits of the last word of a row
    int nblk, hb;        // strip mapping: row blocks per column, rows per block
    int nstrips;         // nblk * WW strips; thread walks strips tid, tid + nthr, ...
    int dense_min;       // sweeps with more listed words run in dense mode
    int scan_min;        // teams: scan passes while more words than this change per pass (< 0: none)
    int scan_first;      // the first pass of a dense sweep as a scan over the candidate plane too
    // team of CTAs working on this image (G == 1: this CTA alone)
    int G, tid, nthr;    // CTAs, team thread id, team thread count
    int cs;              // thread-block cluster size of the team's launch (1: none; G: the team is one cluster)
    unsigned *bar;       // team barrier: monotonic arrival counter (G > 1, cs < G)
    unsigned *epoch;     // this CTA's count of team barriers (shared memory)
    int *err;
    struct Shared *sh;   // control block: shared memory (G == 1) or global (G > 1)
};

__device__ __forceinline__ int pidx(const Img &g, int y, int x) { return g.org + y * g.S + x; }

__device__ __forceinline__ void set_err(int *err, int code) { atomicCAS(err, 0, code); }

// generic address of the same shared-memory variable in CTA `rank` of this
// thread-block cluster (mapa: distributed shared memory)
__device__ __forceinline__ void *dsmem_map(void *p, unsigned rank) {
    void *r;
    asm volatile("mapa.u64 %0, %1, %2;" : "=l"(r) : "l"(p), "r"(rank));
    return r;
}

#ifdef TS_BAR_TRACE
// debug build (tools/bar_trace.py): %globaltimer at arrival and release of every
// cooperative team barrier, per CTA, into the ts_set_trace buffer
// [barrier][rank][2]
__shared__ long long *g_bt;
__shared__ long long g_bt_cap;
__device__ __forceinline__ void bt_rec(const Img &g, unsigned epoch1, int k) {
    const long long idx = (long long)(epoch1 - 1u);
    if (g_bt && idx < g_bt_cap) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_bt[(idx * g.G + g.tid / kThreads) * 2 + k] = (long long)t;
    }
}
#define TS_BT(e, k) bt_rec(g, (e), (k))
#else
#define TS_BT(e, k)
#endif

// Barrier over the G CTAs of a team (co-resident: cooperative launch).  One
// monotonic arrival counter per team: barrier number k (counted per CTA in
// *g.epoch; every CTA of a team executes the same barriers) completes when the
// counter reaches k * arrivals.  Thread 0 of each CTA arrives with a
// fire-and-forget red.release (the CTA's writes, ordered by the __syncthreads
// before it, are visible at gpu scope first) and polls with ld.acquire (which
// drops this SM's stale L1 lines, so plane data written by other CTAs is read
// from L2): one L2 round trip on the critical path instead of four (generation
// read, arrival atomic with return, counter reset, generation bump).  A spin
// bound turns a lost CTA into an error instead of a hang.
__device__ __forceinline__ void team_sync(const Img &g) {
    if (g.G == 1) {
        __syncthreads();
        return;
    }
    if (g.cs == g.G) {
        // the team is a thread-block cluster: the hardware cluster barrier,
        // release / acquire at cluster scope (planes written by one CTA of the
        // team are read by the others after it)
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        return;
    }
    // hierarchical (team of several clusters): cluster barrier, then one CTA
    // per cluster on the global counter (G / cs arrivals instead of G), then
    // the cluster barrier releases the rest; otherwise every CTA arrives
    const bool hier = g.cs > 1;
    if (hier)
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    else
        __syncthreads();
    const unsigned parts = hier ? (unsigned)(g.G / g.cs) : (unsigned)g.G;
    const bool leader = threadIdx.x == 0 && (!hier || (g.tid / kThreads) % g.cs == 0);
    if (threadIdx.x == 0) {
        const unsigned target = (*g.epoch += 1u) * parts;   // every CTA counts, leaders arrive
        if (leader) {
            TS_BT(*g.epoch, 0);
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(g.bar) : "memory");
            long long spins = 0;
            while (true) {
                unsigned c;
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(c) : "l"(g.bar) : "memory");
                if ((int)(c - target) >= 0) break;
                if (++spins > (1LL << 27)) {   // ~ seconds
                    set_err(g.err, ERR_TEAM_TIMEOUT);
                    break;
                }
            }
            TS_BT(*g.epoch, 1);
        }
    }
    if (hier)
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    else
        __syncthreads();
}

// team barrier + the value of a team counter as of the barrier.  Cooperative
// teams: read by the CTA's polling thread right after its acquire and handed
// to the CTA through shared memory -- 148 loads of the word instead of one per
// warp of the chip (2 368), which alone cost ~1 000 cycles per barrier
// (tools/probe/team_barrier.cu: 2 518 -> 3 577 cycles with the read).
__device__ __forceinline__ int team_sync_get(const Img &g, const int *ctr) {
    if (g.G == 1 || g.cs > 1) {   // one CTA, or clusters (the counter is a DSMEM / cluster-local read)
        team_sync(g);
        return *reinterpret_cast<const volatile int *>(ctr);
    }
    __shared__ int s_val;
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned target = (*g.epoch += 1u) * (unsigned)g.G;
        TS_BT(*g.epoch, 0);
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(g.bar) : "memory");
        long long spins = 0;
        while (true) {
            unsigned c;
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(c) : "l"(g.bar) : "memory");
            if ((int)(c - target) >= 0) break;
            if (++spins > (1LL << 27)) {   // ~ seconds
                set_err(g.err, ERR_TEAM_TIMEOUT);
                break;
            }
        }
        s_val = *reinterpret_cast<const volatile int *>(ctr);
        TS_BT(*g.epoch, 1);
    }
    __syncthreads();
    return s_val;
}

struct Nb {
    uint32_t nw, n, ne, w, e, sw, s, se;
    uint32_t m;   // the centre word itself
};

// neighbour bit-words of the 32 pixels of padded word p (pads read as 0)
__device__ __forceinline__ Nb nbrs(const uint32_t *P, const Img &g, int p) {
    const uint32_t *u = P + p - g.S, *m = P + p, *d = P + p + g.S;
    Nb r;
    r.nw = from_west(u[-1], u[0]);
    r.n = u[0];
    r.ne = from_east(u[0], u[1]);
    r.w = from_west(m[-1], m[0]);
    r.e = from_east(m[0], m[1]);
    r.sw = from_west(d[-1], d[0]);
    r.s = d[0];
    r.se = from_east(d[0], d[1]);
    r.m = m[0];
    return r;
}

struct Row3 {   // raw words x-1, x, x+1 of one row
    uint32_t l, c, r;
};
__device__ __forceinline__ Row3 row3(const uint32_t *P, int p) { return Row3{P[p - 1], P[p], P[p + 1]}; }

// runs strip(x, y0, y1, sid) for this thread's strips: strip s = blk * WW + x
// covers column x, rows [blk * hb, blk * hb + hb); thread t walks s = t,
// t + nthr, ...  (the host picks nblk / hb / stride so that the strips a warp
// walks together hit distinct shared-memory banks)
template <class F>
__device__ __forceinline__ void walk_strips(const Img &g, F &&strip) {
    // one call site: the strip body is inlined once
    for (int s = g.tid; s < g.nstrips; s += g.nthr) {
        const int blk = s / g.WW, x = s - blk * g.WW;
        const int y0 = blk * g.hb;
        strip(x, y0, min(g.H, y0 + g.hb), s);
    }
}

// calls f(y, x, p) for the words of this thread's strips, top to bottom
template <class F>
__device__ __forceinline__ void for_strip(const Img &g, F &&f) {
    walk_strips(g, [&](int x, int y0, int y1, int) {
        for (int y = y0; y < y1; ++y) f(y, x, pidx(g, y, x));
    });
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

// pack one [H,W] uint8 image into a bit-plane; flags bytes > 1.  The source
// may be page-locked host memory read over the bus (zero-copy host entry), so
// the loads of kPackBatch strip rows are issued before any is consumed.
constexpr int kPackBatch = 8;

__device__ __forceinline__ void pack_plane(const uint8_t *src, uint32_t *dst, const Img &g, int *err, int code) {
    const bool fast = (g.W % 32) == 0 && ((reinterpret_cast<uintptr_t>(src) & 15) == 0);
    if (fast) {
        uint32_t bad = 0;
        walk_strips(g, [&](int x, int y0, int y1, int) {
            for (int yb = y0; yb < y1; yb += kPackBatch) {
                uint4 a[kPackBatch], b[kPackBatch];
#pragma unroll
                for (int j = 0; j < kPackBatch; ++j) {
                    if (yb + j < y1) {
                        const uint4 *q = reinterpret_cast<const uint4 *>(src + (size_t)(yb + j) * g.W + x * 32);
                        a[j] = __ldg(q);
                        b[j] = __ldg(q + 1);
                    }
                }
#pragma unroll
                for (int j = 0; j < kPackBatch; ++j) {
                    if (yb + j < y1) {
                        dst[pidx(g, yb + j, x)] = pack16(a[j]) | (pack16(b[j]) << 16);
                        bad |= (a[j].x | a[j].y | a[j].z | a[j].w | b[j].x | b[j].y | b[j].z | b[j].w) & 0xFEFEFEFEu;
                    }
                }
            }
        });
        if (bad) set_err(err, code);
        return;
    }
    for_strip(g, [&](int y, int x, int p) {
        const int c0 = x * 32;
        const int cnt = min(32, g.W - c0);
        const uint8_t *s = src + (size_t)y * g.W + c0;
        uint32_t bits = 0, bad = 0;
        for (int i = 0; i < cnt; ++i) {
            const uint32_t v = s[i];
            bits |= (v & 1u) << i;
            bad |= v & ~1u;
        }
        if (bad) set_err(err, code);
        dst[p] = bits;
    });
}

__device__ __forceinline__ void unpack_plane(const uint32_t *src, uint8_t *dst, const Img &g) {
    for_strip(g, [&](int y, int x, int p) {
        const int c0 = x * 32;
        const int cnt = min(32, g.W - c0);
        uint8_t *d = dst + (size_t)y * g.W + c0;
        const uint32_t bits = src[p];
        if (cnt == 32 && ((reinterpret_cast<uintptr_t>(d) & 15) == 0)) {
            uint4 a, b;
            a.x = spread4(bits);
            a.y = spread4(bits >> 4);
            a.z = spread4(bits >> 8);
            a.w = spread4(bits >> 12);
            b.x = spread4(bits >> 16);
            b.y = spread4(bits >> 20);
            b.z = spread4(bits >> 24);
            b.w = spread4(bits >> 28);
            reinterpret_cast<uint4 *>(d)[0] = a;
            reinterpret_cast<uint4 *>(d)[1] = b;
        } else {
            for (int i = 0; i < cnt; ++i) d[i] = (bits >> i) & 1u;
        }
    });
}

// warp-aggregated append to the active-word list among the currently active
// lanes (entries of one aggregate are consecutive in the list)
__device__ __forceinline__ void append(bool has, uint32_t entry, uint32_t *list, int *counter) {
    const unsigned act = __activemask();
    const unsigned m = __ballot_sync(act, has);
    if (m == 0) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(m) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(counter, __popc(m));
    base = __shfl_sync(act, base, leader);
    if (has) list[base + __popc(m & ((1u << lane) - 1u))] = entry;
}

// adds per-thread counts to a counter; the warp may have diverged before
__device__ __forceinline__ void add_count_partial(int cnt, int *counter) {
    __syncwarp();
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(counter, cnt);
}

// adds per-thread counts to a shared/global counter (all threads call)
__device__ __forceinline__ void add_count(int cnt, int *counter) {
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(counter, cnt);
}

// candidates of padded word p: target-valued, unblocked, simple
// (topo.py:186-208, smoothing.py:83-86); t = 1 thins, t = 0 thickens (SURVEY
// A.2.2).  Padding bits and pad words are blocked in B.
template <int FG>
__device__ __forceinline__ uint32_t cand_word(const Img &g, int p, int t) {
    const uint32_t me = g.I[p];
    const uint32_t pre = (t ? me : ~me) & ~g.B[p];
    if (!pre) return 0;
    const Nb i = nbrs(g.I, g, p);
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
// (the zero pads and padding bits make ~I the exterior seed automatically)
// xmode (thin) : 0 -> F = P > r^2 ; 1 -> | keep ; 2 -> | XS
// xmode (thick): 0 -> V = D <= r^2 ; 1 -> & ~avoid ; 2 -> & XS
// rank slices rs[] and blocked bits of word (y, x) (padded index p)
// THIN: -1 = runtime `thin`, 0 / 1 = compile-time (folds the seed inversion)
template <int R, int THIN = -1>
__device__ __forceinline__ uint32_t rank_word(const Img &g, int y, int x, int p, bool thin_rt, int xmode,
                                              uint32_t (&rs)[Lev<R>::S]) {
    const bool thin = THIN < 0 ? thin_rt : THIN != 0;
    using LV = Lev<R>;
    constexpr int L = LV::L;
    constexpr int S = LV::S;
    const uint32_t inv = thin ? ~0u : 0u;
    const int SS = g.S;
    const uint32_t *c = g.I + p;
    // constraint plane read first: it may live in L2
    const uint32_t xw = xmode == 1 ? (thin ? g.K[p] : g.A[p]) : (xmode == 2 ? g.XS[p] : 0u);
    // rows beyond the frame read the single zero pad row (-1 or H): all
    // exterior rows are equal, so the disc needs no deeper padding
    const int up = y + 1, dn = g.H - y;
    uint32_t V[R + 1][3];
    V[0][0] = c[-1] ^ inv;
    V[0][1] = c[0] ^ inv;
    V[0][2] = c[1] ^ inv;
#pragma unroll
    for (int k = 1; k <= R; ++k) {
        const uint32_t *a = c - min(k, up) * SS, *b = c + min(k, dn) * SS;
        V[k][0] = V[k - 1][0] | (a[-1] ^ inv) | (b[-1] ^ inv);
        V[k][1] = V[k - 1][1] | (a[0] ^ inv) | (b[0] ^ inv);
        V[k][2] = V[k - 1][2] | (a[1] ^ inv) | (b[1] ^ inv);
    }
    uint32_t dil = 0, prev = 0;
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
        blocked = ~dil | xw;   // xw: keep (xmode 1) or XS (xmode 2)
    } else {
        const uint32_t m = xmode == 1 ? ~xw : (xmode == 2 ? xw : ~0u);
        blocked = ~(dil & m);
    }
    return blocked | (x == g.WW - 1 ? ~g.lastmask : 0u);
}

template <int R>
__device__ __forceinline__ int prep_rank(const Img &g, bool thin, int xmode, bool save_xs) {
    constexpr int S = Lev<R>::S;
    for_strip(g, [&](int y, int x, int p) {
        uint32_t rs[S];
        const uint32_t xs = g.I[p];
        g.B[p] = rank_word<R>(g, y, x, p, thin, xmode, rs);
#pragma unroll
        for (int s = 0; s < S; ++s) g.R[(size_t)s * g.plen + p] = rs[s];
        if (save_xs) g.XS[p] = xs;
    });
    return S;
}

static_assert(kMaxR == 16, "prep_dispatch covers radii 1..16");

__device__ __forceinline__ void cmp_step(uint32_t &lt, uint32_t &eq, uint32_t nb, uint32_t own) {
    lt |= eq & ~nb & own;   // neighbour < own at the first differing slice
    eq &= ~(nb ^ own);
}

// E masks of word p from the rank slices of its 3x3 word neighbourhood
// (bit-sliced comparator, most significant slice first), stored interleaved
template <int S>
__device__ __forceinline__ void store_e(const Img &g, int p, const Row3 (&ru)[S], const Row3 (&rm)[S],
                                        const Row3 (&rd)[S]) {
    uint32_t lt[8], eq[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        lt[k] = 0;
        eq[k] = ~0u;
    }
#pragma unroll
    for (int s = S - 1; s >= 0; --s) {
        const uint32_t own = rm[s].c;
        cmp_step(lt[0], eq[0], from_west(ru[s].l, ru[s].c), own);
        cmp_step(lt[1], eq[1], ru[s].c, own);
        cmp_step(lt[2], eq[2], from_east(ru[s].c, ru[s].r), own);
        cmp_step(lt[3], eq[3], from_west(rm[s].l, rm[s].c), own);
        if constexpr (!kE4) {
            cmp_step(lt[4], eq[4], from_east(rm[s].c, rm[s].r), own);
            cmp_step(lt[5], eq[5], from_west(rd[s].l, rd[s].c), own);
            cmp_step(lt[6], eq[6], rd[s].c, own);
            cmp_step(lt[7], eq[7], from_east(rd[s].c, rd[s].r), own);
        }
    }
    uint4 *ep = reinterpret_cast<uint4 *>(g.E + (size_t)p * kEWords);
    ep[0] = make_uint4(lt[0] | eq[0], lt[1] | eq[1], lt[2] | eq[2], lt[3] | eq[3]);
    if constexpr (!kE4) ep[1] = make_uint4(lt[4], lt[5], lt[6], lt[7]);
}

// the 8 precedence masks of word p: stored (E8), or (E4) the stored NW, N,
// NE, W and, by antisymmetry of the unique keys, E(p) = ~W of pixel+1,
// SW = ~NE of the pixel below-left, S = ~N below, SE = ~NW below-right
__device__ __forceinline__ void load_e(const Img &g, int p, uint4 &e0, uint4 &e1) {
    const uint4 *ep = reinterpret_cast<const uint4 *>(g.E + (size_t)p * kEWords);
    if constexpr (!kE4) {
        e0 = ep[0];
        e1 = ep[1];
    } else {
        const int S = g.S;
        e0 = ep[0];
        const uint4 b = ep[S];                 // word below
        const uint32_t w_r = g.E[(size_t)(p + 1) * 4 + 3];        // W of the word to the right
        const uint32_t ne_bl = g.E[(size_t)(p + S - 1) * 4 + 2];  // NE of the word below-left
        const uint32_t nw_br = g.E[(size_t)(p + S + 1) * 4 + 0];  // NW of the word below-right
        e1 = make_uint4(~from_east(e0.w, w_r), ~from_west(ne_bl, b.z), ~b.y, ~from_east(b.x, nw_br));
    }
}

// E planes from rank slices + the sweep-1 candidates (C, D = C, list).
// E_k(p) = key(q) < key(p) for q = neighbour k, key = (rank, raster index)
// (topo.py:225,256): ties go to the raster-earlier neighbours NW,N,NE,W.
template <int FG, int S>
__device__ __forceinline__ void epass_ranks(const Img &g, int t, int *counter) {
    int cnt = 0;   // words with candidates (the list is built lazily, see build_list)
    auto strip = [&](int x, int y0, int y1) {
        int p = pidx(g, y0, x);
        Row3 iu = row3(g.I, p - g.S), im = row3(g.I, p);
        Row3 ru[S], rm[S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            ru[s] = row3(g.R + (size_t)s * g.plen, p - g.S);
            rm[s] = row3(g.R + (size_t)s * g.plen, p);
        }
        for (int y = y0; y < y1; ++y, p += g.S) {
            Row3 rd[S];
#pragma unroll
            for (int s = 0; s < S; ++s) rd[s] = row3(g.R + (size_t)s * g.plen, p + g.S);
            const Row3 id = row3(g.I, p + g.S);
            // E is read only for words holding candidates in some sweep of this
            // engine call, and those lie inside the unblocked target pixels
            // (flips never create target pixels): skip the rest
            const uint32_t pre = (t ? im.c : ~im.c) & ~g.B[p];
            uint32_t c = 0;
            if (pre) {
                c = pre & simple_bits<FG>(from_west(iu.l, iu.c), iu.c, from_east(iu.c, iu.r), from_west(im.l, im.c),
                                          from_east(im.c, im.r), from_west(id.l, id.c), id.c, from_east(id.c, id.r));
                if constexpr (!kE4) store_e<S>(g, p, ru, rm, rd);
            }
            if constexpr (kE4) store_e<S>(g, p, ru, rm, rd);   // neighbours' masks are read too
            g.C[p] = c;
            g.D[p] = c;
            cnt += c != 0;
            iu = im;
            im = id;
#pragma unroll
            for (int s = 0; s < S; ++s) {
                ru[s] = rm[s];
                rm[s] = rd[s];
            }
        }
    };
    walk_strips(g, [&](int x, int y0, int y1, int) { strip(x, y0, y1); });
    add_count(cnt, counter);
}

// Fused prep + E-pass for images whose rows fit in a warp (WW divides 32 and
// every thread walks one strip): each thread computes the rank slices of its
// own word row by row and keeps a 3-row window; the slices of the left / right
// words (the neighbouring lanes, same row, same step) come by warp shuffles,
// so the slices never touch memory and the two phases need no barrier between.
template <int FG, int R, bool THIN>
__device__ __forceinline__ void prep_fused(const Img &g, int xmode, bool save_xs, int *counter) {
    constexpr bool thin = THIN;
    constexpr int t = THIN ? 1 : 0;
    constexpr int S = Lev<R>::S;
    const int lane = threadIdx.x & 31;
    const int x = g.tid % g.WW, blk = g.tid / g.WW;
    const bool act = blk < g.nblk;
    const int y0 = act ? blk * g.hb : 0, y1 = act ? min(g.H, y0 + g.hb) : 0;
    const bool hasl = x > 0, hasr = x < g.WW - 1;
    int cnt = 0;
    // rank slices of row y of this column (with the left / right words' by
    // shuffle; all lanes take part in every step)
    auto row = [&](int y, Row3 (&r)[S], uint32_t &bl) {
        const bool in = act && y >= 0 && y < g.H;
        uint32_t rs[S];
        bl = ~0u;
        if (in) {
            const int p = pidx(g, y, x);
            const uint32_t xs = g.I[p];
            bl = rank_word<R, THIN ? 1 : 0>(g, y, x, p, thin, xmode, rs);
            if (y >= y0 && y < y1) {
                g.B[p] = bl;
                if (save_xs) g.XS[p] = xs;
            }
        } else {
#pragma unroll
            for (int s = 0; s < S; ++s) rs[s] = 0;
        }
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const uint32_t l = __shfl_up_sync(0xffffffffu, rs[s], 1);
            const uint32_t rr = __shfl_down_sync(0xffffffffu, rs[s], 1);
            r[s] = Row3{hasl ? l : 0u, rs[s], hasr ? rr : 0u};
        }
    };
    Row3 ru[S], rm[S], rd[S];
    uint32_t bu, bm, bd;
    row(y0 - 1, ru, bu);
    row(y0, rm, bm);
    const int steps = g.hb;   // warp-uniform trip count (shorter strips idle)
    int p = pidx(g, y0, x);
    Row3 iu = row3(g.I, p - g.S), im = row3(g.I, p);
#if TS_PREP_U4
    // E8 storage from 4 comparators per word: at row y the masks towards the
    // upper neighbours U(y) = {NW, N, NE, W} (every word, all lanes); row
    // y-1's lower four follow by antisymmetry of the unique keys and are
    // stored one step late: S = ~N(y), SW = ~NE(y) of pixel-1 (lane-1 at bit
    // 0), SE = ~NW(y) of pixel+1, E = ~W of pixel+1 (lane+1 at bit 31; pads
    // at row ends: those neighbours' decisions are 0)
    if constexpr (!kE4) {
        auto upper = [&]() -> uint4 {
            uint32_t lt[4], eq[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                lt[k] = 0;
                eq[k] = ~0u;
            }
#pragma unroll
            for (int s = S - 1; s >= 0; --s) {
                const uint32_t own = rm[s].c;
                cmp_step(lt[0], eq[0], from_west(ru[s].l, ru[s].c), own);
                cmp_step(lt[1], eq[1], ru[s].c, own);
                cmp_step(lt[2], eq[2], from_east(ru[s].c, ru[s].r), own);
                cmp_step(lt[3], eq[3], from_west(rm[s].l, rm[s].c), own);
            }
            return make_uint4(lt[0] | eq[0], lt[1] | eq[1], lt[2] | eq[2], lt[3] | eq[3]);
        };
        uint4 uprev = make_uint4(0, 0, 0, 0);
        uint32_t eprev = 0, cprev = 0;
        int pprev = 0;
        auto finish = [&](const uint4 &u) {   // row y-1's masks, given U(y); returns E of row y
            const uint32_t w_r = __shfl_down_sync(0xffffffffu, u.w, 1);
            const uint32_t ne_l = __shfl_up_sync(0xffffffffu, u.z, 1);
            const uint32_t nw_r = __shfl_down_sync(0xffffffffu, u.x, 1);
            if (cprev) {   // (E is read only for words with unblocked target pixels, see below)
                uint4 *ep = reinterpret_cast<uint4 *>(g.E + (size_t)pprev * 8);
                ep[0] = uprev;
                ep[1] = make_uint4(eprev, ~from_west(ne_l, u.z), ~u.y, ~from_east(u.x, nw_r));
            }
            return ~from_east(u.w, w_r);
        };
        for (int j = 0; j < steps; ++j, p += g.S) {
            const int y = y0 + j;
            row(y + 1, rd, bd);
            const uint4 u = upper();
            const uint32_t e_here = finish(u);
            cprev = 0;
            if (y < y1) {
                const Row3 id = row3(g.I, p + g.S);
                const uint32_t pre = (t ? im.c : ~im.c) & ~bm;
                uint32_t c = 0;
                if (pre)
                    c = pre & simple_bits<FG>(from_west(iu.l, iu.c), iu.c, from_east(iu.c, iu.r),
                                              from_west(im.l, im.c), from_east(im.c, im.r), from_west(id.l, id.c),
                                              id.c, from_east(id.c, id.r));
                g.C[p] = c;
                g.D[p] = c;
                cnt += c != 0;
                cprev = pre;   // any later sweep's candidates lie inside pre
                pprev = p;
                iu = im;
                im = id;
            }
            uprev = u;
            eprev = e_here;
#pragma unroll
            for (int s = 0; s < S; ++s) {
                ru[s] = rm[s];
                rm[s] = rd[s];
            }
            bu = bm;
            bm = bd;
        }
        finish(upper());   // the strip's last row, from the row below it
        (void)lane;
        (void)bu;
        add_count(cnt, counter);
        return;
    }
#endif
    for (int j = 0; j < steps; ++j, p += g.S) {
        const int y = y0 + j;
        row(y + 1, rd, bd);
        if (y < y1) {
            const Row3 id = row3(g.I, p + g.S);
            // E is read only for words holding candidates in some sweep of this
            // engine call, and those lie inside the unblocked target pixels
            const uint32_t pre = (t ? im.c : ~im.c) & ~bm;
            uint32_t c = 0;
            if (pre) {
                c = pre & simple_bits<FG>(from_west(iu.l, iu.c), iu.c, from_east(iu.c, iu.r), from_west(im.l, im.c),
                                          from_east(im.c, im.r), from_west(id.l, id.c), id.c, from_east(id.c, id.r));
                if constexpr (!kE4) store_e<S>(g, p, ru, rm, rd);
            }
            if constexpr (kE4) store_e<S>(g, p, ru, rm, rd);   // neighbours' masks are read too
            g.C[p] = c;
            g.D[p] = c;
            cnt += c != 0;
            iu = im;
            im = id;
        }
#pragma unroll
        for (int s = 0; s < S; ++s) {
            ru[s] = rm[s];
            rm[s] = rd[s];
        }
        bu = bm;
        bm = bd;
    }
    (void)lane;
    (void)bu;
    add_count(cnt, counter);
}

// E planes straight from an int64 priority map (public homotopic_thin /
// homotopic_thicken: arbitrary priorities, topo.py:303-342)
template <int FG>
__device__ __forceinline__ void epass_prio(const Img &g, const int64_t *prio, int t, int *counter) {
    int cnt = 0;
    const int dy[8] = {-1, -1, -1, 0, 0, 1, 1, 1};
    const int dx[8] = {-1, 0, 1, -1, 1, -1, 0, 1};
    for_strip(g, [&](int y, int x, int p) {
        uint32_t c = 0;
        if (kE4 || ~g.B[p]) {   // E4: every word's masks (neighbours read them)
            uint32_t e[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            const int cnt = min(32, g.W - x * 32);
            for (int i = 0; i < cnt; ++i) {
                const int col = x * 32 + i;
                const int64_t pv = prio[(size_t)y * g.W + col];
#pragma unroll
                for (int k = 0; k < (kE4 ? 4 : 8); ++k) {
                    const int ny = y + dy[k], nc = col + dx[k];
                    if (ny < 0 || ny >= g.H || nc < 0 || nc >= g.W) continue;
                    const int64_t q = prio[(size_t)ny * g.W + nc];
                    if (q < pv || (q == pv && k < 4)) e[k] |= 1u << i;
                }
            }
            uint4 *ep = reinterpret_cast<uint4 *>(g.E + (size_t)p * kEWords);
            ep[0] = make_uint4(e[0], e[1], e[2], e[3]);
            if constexpr (!kE4) ep[1] = make_uint4(e[4], e[5], e[6], e[7]);
            if (~g.B[p]) c = cand_word<FG>(g, p, t);
        }
        g.C[p] = c;
        g.D[p] = c;
        cnt += c != 0;
    });
    add_count(cnt, counter);
}

// ---- strip-walk pass stamps -------------------------------------------------
// The strip-walk pass of a dense sweep (counter k) stamps the words it must
// have re-evaluated with k + 1 (the counter's low byte; byte stores -- all
// writers of a word store the same value, so no atomics); a scan then lists
// them (collect_stamped).  A stale stamp only costs an extra evaluation (any
// evaluation order reaches the same fixpoint).

// stamp, for re-evaluation in the next pass, the words whose inputs changed
// when decision bits `chg` of word p flipped.  A pixel's decision reads the
// decision of neighbour q only when q precedes it in key order, i.e. (keys
// are unique) exactly the neighbours in the directions k with E_k(q) == 0; so
// the E masks of the changed word itself (e0: NW,N,NE,W; e1: E,SW,S,SE) name
// the neighbour words that can be affected.  `self`: also stamp word p (its
// own W/E in-word neighbours, when the caller did not resolve them).
__device__ __forceinline__ void stamp_chg(const Img &g, int p, uint32_t chg, uint4 e0, uint4 e1, uint8_t v,
                                          bool self) {
    uint8_t *m = g.mark + p;
    const int S = g.S;
    const uint32_t lNW = ~e0.x, lN = ~e0.y, lNE = ~e0.z, lW = ~e0.w;   // "that neighbour is later"
    const uint32_t lE = ~e1.x, lSW = ~e1.y, lS = ~e1.z, lSE = ~e1.w;
    if (chg & (lN | (lNW & ~1u) | (lNE & 0x7FFFFFFFu))) m[-S] = v;
    if (chg & (lS | (lSW & ~1u) | (lSE & 0x7FFFFFFFu))) m[S] = v;
    if (self) m[0] = v;
    if (chg & 1u) {
        if (lNW & 1u) m[-S - 1] = v;
        if (lW & 1u) m[-1] = v;
        if (lSW & 1u) m[S - 1] = v;
    }
    if (chg >> 31) {
        if (lNE >> 31) m[-S + 1] = v;
        if (lE >> 31) m[1] = v;
        if (lSE >> 31) m[S + 1] = v;
    }
}

template <int FG>
__device__ __forceinline__ uint32_t decide(uint32_t c, const Nb &i, const Nb &d, uint4 e0, uint4 e1) {
    return c & simple_bits<FG>(i.nw ^ (d.nw & e0.x), i.n ^ (d.n & e0.y), i.ne ^ (d.ne & e0.z), i.w ^ (d.w & e0.w),
                               i.e ^ (d.e & e1.x), i.sw ^ (d.sw & e1.y), i.s ^ (d.s & e1.z), i.se ^ (d.se & e1.w));
}

// ---- dense sweeps: strip walk with a sliding 3-row window ------------------

// one worklist pass over the strip; returns whether any decision changed.
// Rows are processed in groups of kDenseBatch: the group's candidate / stamp
// checks and E loads (from L2 when E does not fit in shared memory) are issued
// together, then the rows are evaluated in order with the sliding window.
#ifndef TS_DENSE_BATCH
#define TS_DENSE_BATCH 2
#endif
constexpr int kDenseBatch = TS_DENSE_BATCH;
#ifndef TS_DENSE_PREFETCH
#define TS_DENSE_PREFETCH 0
#endif
constexpr int kDensePrefetch = TS_DENSE_PREFETCH;   // rows of E prefetch in the shared-memory strip walk (0: batches)
#ifndef TS_DENSE_BATCH_L2
#define TS_DENSE_BATCH_L2 2
#endif
#ifndef TS_DENSE_PIPE
#define TS_DENSE_PIPE 1
#endif
constexpr bool kDensePipe = TS_DENSE_PIPE != 0;   // software-pipelined strip walk over L2 planes
constexpr int kDenseBatchL2 = TS_DENSE_BATCH_L2;
#ifndef TS_STREAM_BATCH
#define TS_STREAM_BATCH 4
#endif
constexpr int kStreamBatch = TS_STREAM_BATCH;   // rows per load batch of the streaming passes over L2 / DRAM planes   // rows whose C / E loads are in flight together (L2 planes)


template <int FG>
__device__ __forceinline__ bool dense_pass(const Img &g, int pc, int &evals) {
    bool ch = false;
    const uint8_t next = (uint8_t)(pc + 1);
    auto strip = [&](int x, int y0, int y1, int) {
        if (y0 >= y1) return;
        int p = pidx(g, y0, x);
        Row3 iu = row3(g.I, p - g.S), im = row3(g.I, p);
        Row3 du = row3(g.D, p - g.S), dm = row3(g.D, p);
        // one row: evaluate word p (candidates c, masks e0 / e1), slide the window
        auto row = [&](uint32_t c, const uint4 &e0, const uint4 &e1) {
            const Row3 id = row3(g.I, p + g.S), dd = row3(g.D, p + g.S);
            if (c) {
                Nb in, dn;
                in.nw = from_west(iu.l, iu.c);
                in.n = iu.c;
                in.ne = from_east(iu.c, iu.r);
                in.w = from_west(im.l, im.c);
                in.e = from_east(im.c, im.r);
                in.sw = from_west(id.l, id.c);
                in.s = id.c;
                in.se = from_east(id.c, id.r);
                dn.nw = from_west(du.l, du.c);
                dn.n = du.c;
                dn.ne = from_east(du.c, du.r);
                dn.w = from_west(dm.l, dm.c);
                dn.e = from_east(dm.c, dm.r);
                dn.sw = from_west(dd.l, dd.c);
                dn.s = dd.c;
                dn.se = from_east(dd.c, dd.r);
                uint32_t nd = decide<FG>(c, in, dn, e0, e1);
                // resolve chains inside the word now: re-decide with the
                // word's own new decisions as its W/E neighbours
                for (uint32_t pd = dm.c; nd != pd;) {
                    pd = nd;
                    dn.w = from_west(dm.l, nd);
                    dn.e = from_east(nd, dm.r);
                    nd = decide<FG>(c, in, dn, e0, e1);
                }
                ++evals;
                if (nd != dm.c) {
                    const uint32_t chg = nd ^ dm.c;
                    g.D[p] = nd;
                    dm.c = nd;   // the next row sees this update (Gauss-Seidel down the strip)
                    stamp_chg(g, p, chg, e0, e1, next, false);
                    ch = true;
                }
            }
            iu = im;
            im = id;
            du = dm;
            dm = dd;
            p += g.S;
        };
        if constexpr (kDensePrefetch > 0) {
            // E masks live in L2 (they do not fit shared memory beside the hot
            // planes): the masks of the row kDensePrefetch rows below are
            // requested before the current row is evaluated, so their latency
            // overlaps the evaluation (c1: 3.28 -> 3.21 ms)
            constexpr int PF = kDensePrefetch > 0 ? kDensePrefetch : 1;
            uint32_t cq[PF];
            uint4 e0q[PF], e1q[PF];
#pragma unroll
            for (int j = 0; j < PF; ++j) {
                cq[j] = y0 + j < y1 ? g.C[p + j * g.S] : 0u;
                if (cq[j]) load_e(g, p + j * g.S, e0q[j], e1q[j]);
            }
            for (int y = y0; y < y1; ++y) {
                const uint32_t c = cq[0];
                const uint4 e0 = e0q[0], e1 = e1q[0];
#pragma unroll
                for (int j = 0; j + 1 < PF; ++j) {
                    cq[j] = cq[j + 1];
                    e0q[j] = e0q[j + 1];
                    e1q[j] = e1q[j + 1];
                }
                cq[PF - 1] = y + PF < y1 ? g.C[p + PF * g.S] : 0u;
                if (cq[PF - 1]) load_e(g, p + PF * g.S, e0q[PF - 1], e1q[PF - 1]);
                row(c, e0, e1);
            }
        } else {
            for (int yb = y0; yb < y1; yb += kDenseBatch) {
                // the batch's candidates and E masks (L2) are requested together
                uint32_t cb[kDenseBatch];
                uint4 e0b[kDenseBatch], e1b[kDenseBatch];
#pragma unroll
                for (int j = 0; j < kDenseBatch; ++j) {
                    const int q = p + j * g.S;
                    cb[j] = yb + j < y1 ? g.C[q] : 0u;
                    if (cb[j]) load_e(g, q, e0b[j], e1b[j]);
                }
#pragma unroll
                for (int j = 0; j < kDenseBatch; ++j) {
                    if (yb + j >= y1) break;
                    row(cb[j], e0b[j], e1b[j]);
                }
            }
        }
    };
    walk_strips(g, strip);
    return ch;
}

// L2-resident planes, plain batches (the 1024-thread variant: 64 registers
// per thread leave no room for the pipelined walk's prefetched rows)
template <int FG>
__device__ __forceinline__ bool dense_pass_l2_plain(const Img &g, int pc, int &evals) {
    bool ch = false;
    const uint8_t next = (uint8_t)(pc + 1);
    auto strip = [&](int x, int y0, int y1, int) {
        if (y0 >= y1) return;
        int p = pidx(g, y0, x);
        int y = y0;
        Row3 iu = row3(g.I, p - g.S), im = row3(g.I, p);
        Row3 du = row3(g.D, p - g.S), dm = row3(g.D, p);
        auto step = [&](uint32_t c, uint4 e0, uint4 e1) {
            const Row3 id = row3(g.I, p + g.S), dd = row3(g.D, p + g.S);
            if (c) {
                Nb in, dn;
                in.nw = from_west(iu.l, iu.c);
                in.n = iu.c;
                in.ne = from_east(iu.c, iu.r);
                in.w = from_west(im.l, im.c);
                in.e = from_east(im.c, im.r);
                in.sw = from_west(id.l, id.c);
                in.s = id.c;
                in.se = from_east(id.c, id.r);
                dn.nw = from_west(du.l, du.c);
                dn.n = du.c;
                dn.ne = from_east(du.c, du.r);
                dn.w = from_west(dm.l, dm.c);
                dn.e = from_east(dm.c, dm.r);
                dn.sw = from_west(dd.l, dd.c);
                dn.s = dd.c;
                dn.se = from_east(dd.c, dd.r);
                const uint32_t nd = decide<FG>(c, in, dn, e0, e1);
                ++evals;
                if (nd != dm.c) {
                    const uint32_t chg = nd ^ dm.c;
                    g.D[p] = nd;
                    dm.c = nd;
                    stamp_chg(g, p, chg, e0, e1, next, true);
                    ch = true;
                }
            }
            iu = im;
            im = id;
            du = dm;
            dm = dd;
            p += g.S;
            ++y;
        };
        auto fetch = [&](int q, uint32_t &c, uint4 &e0, uint4 &e1) {
            c = g.C[q];
            if (c) load_e(g, q, e0, e1);
        };
        while (y + 2 <= y1) {
            uint32_t cb[2];
            uint4 e0b[2], e1b[2];
#pragma unroll
            for (int j = 0; j < 2; ++j) fetch(p + j * g.S, cb[j], e0b[j], e1b[j]);
#pragma unroll
            for (int j = 0; j < 2; ++j) step(cb[j], e0b[j], e1b[j]);
        }
        while (y < y1) {
            uint32_t c;
            uint4 e0, e1;
            fetch(p, c, e0, e1);
            step(c, e0, e1);
        }
    };
    walk_strips(g, strip);
    return ch;
}

// variant for the L2-resident planes (generic / team kernel).  Software
// pipelined over batches of kDenseBatchL2 rows: a batch's candidate words are
// requested one batch ahead, so its E masks (needed only where candidates
// exist), the image / decision rows below it and the next batch's candidates
// are all in flight together -- one L2 / DRAM latency per batch instead of
// three dependent ones per row.  Prefetched decisions of the neighbouring
// columns may be stale: any evaluation order reaches the fixpoint, and every
// later change stamps the words it affects.
template <int FG>
__device__ __forceinline__ bool dense_pass_l2(const Img &g, int pc, int &evals) {
    bool ch = false;
    const uint8_t next = (uint8_t)(pc + 1);
    constexpr int KB = kDenseBatchL2;
    auto strip = [&](int x, int y0, int y1, int) {
        if (y0 >= y1) return;
        int p = pidx(g, y0, x);
        const int S = g.S;
        Row3 iu = row3(g.I, p - S), im = row3(g.I, p);
        Row3 du = row3(g.D, p - S), dm = row3(g.D, p);
        uint32_t cn[KB];
#pragma unroll
        for (int j = 0; j < KB; ++j) cn[j] = y0 + j < y1 ? g.C[p + j * S] : 0u;
        for (int yb = y0; yb < y1; yb += KB) {
            uint32_t cb[KB];
            uint4 e0b[KB], e1b[KB];
            Row3 idb[KB], ddb[KB];
#pragma unroll
            for (int j = 0; j < KB; ++j) {
                cb[j] = cn[j];
                if (cb[j]) load_e(g, p + j * S, e0b[j], e1b[j]);
            }
#pragma unroll
            for (int j = 0; j < KB; ++j) {
                if (yb + j < y1) {
                    idb[j] = row3(g.I, p + (j + 1) * S);
                    ddb[j] = row3(g.D, p + (j + 1) * S);
                }
            }
#pragma unroll
            for (int j = 0; j < KB; ++j) cn[j] = yb + KB + j < y1 ? g.C[p + (KB + j) * S] : 0u;
#pragma unroll
            for (int j = 0; j < KB; ++j) {
                if (yb + j >= y1) break;
                const Row3 id = idb[j], dd = ddb[j];
                const uint32_t c = cb[j];
                if (c) {
                    const uint4 e0 = e0b[j], e1 = e1b[j];
                    Nb in, dn;
                    in.nw = from_west(iu.l, iu.c);
                    in.n = iu.c;
                    in.ne = from_east(iu.c, iu.r);
                    in.w = from_west(im.l, im.c);
                    in.e = from_east(im.c, im.r);
                    in.sw = from_west(id.l, id.c);
                    in.s = id.c;
                    in.se = from_east(id.c, id.r);
                    dn.nw = from_west(du.l, du.c);
                    dn.n = du.c;
                    dn.ne = from_east(du.c, du.r);
                    dn.w = from_west(dm.l, dm.c);
                    dn.e = from_east(dm.c, dm.r);
                    dn.sw = from_west(dd.l, dd.c);
                    dn.s = dd.c;
                    dn.se = from_east(dd.c, dd.r);
                    const uint32_t nd = decide<FG>(c, in, dn, e0, e1);
                    ++evals;
                    if (nd != dm.c) {
                        const uint32_t chg = nd ^ dm.c;
                        g.D[p] = nd;
                        dm.c = nd;
                        stamp_chg(g, p, chg, e0, e1, next, true);
                        ch = true;
                    }
                }
                iu = im;
                im = id;
                du = dm;
                dm = dd;
                p += S;
            }
        }
    };
    walk_strips(g, strip);
    return ch;
}

// ---- sparse sweeps: list of words ------------------------------------------
struct Slot {
    int p;
    Nb in;          // image neighbours at the sweep start
    uint4 e0, e1;   // E masks
    uint32_t c;     // candidates
    uint32_t d;     // current decision (only this thread writes D[p])
};

template <int FG>
__device__ __forceinline__ void load_slot(const Img &g, uint32_t p, Slot &s) {
    s.p = (int)p;
    s.in = nbrs(g.I, g, s.p);
    load_e(g, s.p, s.e0, s.e1);
    s.c = g.C[s.p];
    s.d = g.D[s.p];
}

template <int FG, bool STAMP>
__device__ __forceinline__ bool update_slot(const Img &g, Slot &s, uint8_t M = 0) {
    const uint32_t *u = g.D + s.p - g.S, *m = g.D + s.p, *d = g.D + s.p + g.S;
    Nb dn;
    dn.nw = from_west(u[-1], u[0]);
    dn.n = u[0];
    dn.ne = from_east(u[0], u[1]);
    dn.w = from_west(m[-1], s.d);   // W/E inside the word: own decisions
    dn.e = from_east(s.d, m[1]);
    dn.sw = from_west(d[-1], d[0]);
    dn.s = d[0];
    dn.se = from_east(d[0], d[1]);
    const uint32_t nd = decide<FG>(s.c, s.in, dn, s.e0, s.e1);
    if (nd != s.d) {
        if constexpr (STAMP) stamp_chg(g, s.p, nd ^ s.d, s.e0, s.e1, M, true);
        s.d = nd;
        g.D[s.p] = nd;
        return true;
    }
    return false;
}

// mark the dirty bits of padded words [p0, p1] (consecutive, at most 3)
__device__ __forceinline__ void mark_words(const Img &g, int p0, int p1) {
    const int q0 = p0 >> 5, q1 = p1 >> 5;
    if (q0 == q1) {
        atomicOr(&g.dirty[q0], (0xFFFFFFFFu >> (31 - (p1 - p0))) << (p0 & 31));
    } else {
        atomicOr(&g.dirty[q0], 0xFFFFFFFFu << (p0 & 31));
        atomicOr(&g.dirty[q1], 0xFFFFFFFFu >> (31 - (p1 & 31)));
    }
}

// flips of one listed word: I ^= d, D = 0, dirty 3x3 word neighbourhood
__device__ __forceinline__ unsigned apply_word(const Img &g, int p, uint32_t dw) {
    if (!dw) return 0;
    g.I[p] ^= dw;
    g.D[p] = 0;
    const int a = (dw & 1u) ? -1 : 0, b = (dw >> 31) ? 1 : 0;
    mark_words(g, p - g.S + a, p - g.S + b);
    mark_words(g, p + a, p + b);
    mark_words(g, p + g.S + a, p + g.S + b);
    return __popc(dw);
}

// re-examination after a list sweep: the dirty bitmap is compacted into a
// word list (thread per bitmap word, warp prefix sums), then every listed word
// is re-examined by one thread -- full lanes instead of a warp per bitmap word
template <int FG, bool GET = false>
__device__ __forceinline__ void rebuild_compact(const Img &g, int t, uint32_t *dl, int *dcount, int *counter) {
    const int lane = threadIdx.x & 31;
    const int nq = (g.plen + 31) >> 5;
    for (int q0 = g.tid - lane; q0 < nq; q0 += g.nthr) {   // warp-uniform trip count
        const int q = q0 + lane;
        uint32_t bits = 0;
        if (q < nq) {
            bits = g.dirty[q];
            if (bits) g.dirty[q] = 0;
        }
        const int cnt = __popc(bits);
        int incl = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int o = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += o;
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 31);
        if (tot == 0) continue;
        int base = 0;
        if (lane == 31) base = atomicAdd(dcount, tot);
        base = __shfl_sync(0xffffffffu, base, 31) + incl - cnt;
        for (; bits; bits &= bits - 1) dl[base++] = (uint32_t)(q * 32 + __ffs(bits) - 1);
    }
    int nd;
    if constexpr (GET) {
        nd = team_sync_get(g, dcount);
    } else {
        team_sync(g);
        nd = *reinterpret_cast<volatile int *>(dcount);
    }
    for (int s0 = g.tid - lane; s0 < nd; s0 += g.nthr) {   // warp-uniform trip count
        const int sl = s0 + lane;
        uint32_t c = 0;
        int p = 0;
        if (sl < nd) {
            p = (int)dl[sl];
            c = cand_word<FG>(g, p, t);
            g.C[p] = c;
            g.D[p] = c;
        }
        append(c != 0, (uint32_t)p, g.list, counter);
    }
}

// recompute the candidates of every word (after a dense sweep).  KB rows'
// loads (I rows, B) are issued together: one memory latency per batch when the
// planes live in L2 / DRAM (KB = 1 in shared memory)
template <int FG, int KB>
__device__ __forceinline__ void rebuild_dense(const Img &g, int t, int *counter) {
    int cnt = 0;
    auto strip = [&](int x, int y0, int y1) {
        int p = pidx(g, y0, x);
        Row3 iu = row3(g.I, p - g.S), im = row3(g.I, p);
        for (int yb = y0; yb < y1; yb += KB) {
            Row3 idb[KB];
            uint32_t bb[KB];
#pragma unroll
            for (int j = 0; j < KB; ++j) {
                if (yb + j < y1) {
                    idb[j] = row3(g.I, p + (j + 1) * g.S);
                    bb[j] = g.B[p + j * g.S];
                }
            }
#pragma unroll
            for (int j = 0; j < KB; ++j) {
                if (yb + j >= y1) break;
                const Row3 id = idb[j];
                const uint32_t pre = (t ? im.c : ~im.c) & ~bb[j];
                uint32_t c = 0;
                if (pre)
                    c = pre & simple_bits<FG>(from_west(iu.l, iu.c), iu.c, from_east(iu.c, iu.r),
                                              from_west(im.l, im.c), from_east(im.c, im.r), from_west(id.l, id.c),
                                              id.c, from_east(id.c, id.r));
                g.C[p] = c;
                g.D[p] = c;
                cnt += c != 0;
                iu = im;
                im = id;
                p += g.S;
            }
        }
    };
    walk_strips(g, [&](int x, int y0, int y1, int) { strip(x, y0, y1); });
    add_count(cnt, counter);
}

// active-word list from the C plane (needed when a sparse sweep follows a
// dense one or the E-pass, which only count).  Planes outside shared memory
// (BATCH): the C words of up to 32 rows of a strip are loaded in batches of 8,
// then ONE warp-aggregated append (a single counter atomic) lists them --
// a load and an atomic round trip per row otherwise.
template <bool BATCH>
__device__ __forceinline__ void build_list(const Img &g, int *counter) {
    if constexpr (!BATCH) {
        for_strip(g, [&](int y, int x, int p) { append(g.C[p] != 0, (uint32_t)p, g.list, counter); });
    } else {
        const int lane = threadIdx.x & 31;
        for (int s0 = g.tid - lane; s0 < g.nstrips; s0 += g.nthr) {   // warp-uniform trip counts
            const int s = s0 + lane;
            const bool valid = s < g.nstrips;
            const int blk = valid ? s / g.WW : 0, x = valid ? s - blk * g.WW : 0;
            const int y0 = blk * g.hb, y1 = valid ? min(g.H, y0 + g.hb) : y0;
            for (int yc = 0; yc < g.hb; yc += 32) {
                const int pb = pidx(g, y0 + yc, x);
                uint32_t nz = 0;
                for (int jb = 0; jb < 32 && yc + jb < g.hb; jb += 8) {
                    uint32_t c[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) c[j] = (y0 + yc + jb + j < y1) ? g.C[pb + (jb + j) * g.S] : 0u;
#pragma unroll
                    for (int j = 0; j < 8; ++j) nz |= (c[j] != 0u ? 1u : 0u) << (jb + j);
                }
                const int cnt = __popc(nz);
                int incl = cnt;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const int o = __shfl_up_sync(0xffffffffu, incl, d);
                    if (lane >= d) incl += o;
                }
                const int tot = __shfl_sync(0xffffffffu, incl, 31);
                if (tot == 0) continue;
                int base = 0;
                if (lane == 31) base = atomicAdd(counter, tot);
                base = __shfl_sync(0xffffffffu, base, 31) + incl - cnt;
                for (; nz; nz &= nz - 1) g.list[base++] = (uint32_t)(pb + (__ffs(nz) - 1) * g.S);
            }
        }
    }
}

struct Stats {
    long long sweeps, passes, calls;
    long long cyc_prep, cyc_jacobi, cyc_update;   // thread-0 clock64 deltas (stats mode only)
    long long cyc_tiny, n_tiny, pass_tiny;        // sweeps with <= 32 listed words
    long long cyc_dense, n_dense, pass_dense;     // dense-mode sweeps
    long long cyc_rank;                           // clamped-EDT part of prep
    bool timing;
};

struct EngineIO {   // engine statistics of the current image, accumulated by team thread 0
    long long sweeps, passes, calls;
    long long cyc_jacobi, cyc_update, cyc_tiny, n_tiny, pass_tiny, cyc_dense, n_dense, pass_dense;
};

struct Shared {
    int img;
    int counters[2];
    int bad;
    unsigned long long flips, evals;
    long long tiny[2];   // tiny-sweep regime results (warp 0 -> CTA): sweeps, passes
    int lcount[6];       // [0..2] lengths of the compacted re-evaluation lists (rotating, see claim_passes);
                         // [3..5] words changed by the scan passes (rotating, see dense_sweep)
    int dcount;          // dirty words listed for re-examination after a list sweep
    long long dtime[4];  // stats: dense pass-1 / collect / list-pass cycles, listed words
    long long sstat[4];  // stats: list sweeps (33..512 words) count / cycles, (> 512) count / cycles
    long long bstat[4];  // stats, list sweeps > 512 words: list-build / sweep / re-examination cycles, list builds
    long long xstat[4];  // stats: tiny regimes (incl. list build and barriers) cycles / count; engine; stage
    long long ystat[4];  // stats: engine prologue, loop tops, epilogue cycles; sweeps-loop iterations
    EngineIO eio;        // engine statistics (returned through here, not by value: no local-memory copies)
};

// per-team control block in global memory (teams of G > 1 CTAs)
struct TeamCtl {
    Shared sh;
    unsigned bar[2];
};
static_assert(sizeof(TeamCtl) <= kTeamCtlBytes, "kTeamCtlBytes too small");

// ---- phase functions ----------------------------------------------------------
// Each phase is a separate (non-inlined) function so that its register
// allocation is independent of the others.  They receive the image as a View:
// hot planes as 32-bit shared-window addresses (HOT) re-materialised with
// cvta inside the callee (so accesses compile to LDS/STS), others as pointers.
struct View {
    unsigned long long I, D, C, dirty, mark;   // shared address (HOT) or pointer bits
    uint32_t *list, *E, *XS, *R, *K, *A;
    unsigned long long B, claim;   // shared address (HOT) or pointer bits
    int H, W, WW, S, plen, org, nblk, hb, nstrips, dense_min, scan_min, scan_first, fused, mw;
    uint32_t lastmask;
    unsigned long long sh;   // Shared block: shared address (G == 1) or global pointer (team)
    int G, rank, cs;
    unsigned *bar;
    unsigned *epoch;
    int *err;
};

template <bool HOT>
__device__ __forceinline__ uint32_t *hot_ptr(unsigned long long h) {
    if constexpr (HOT)
        return reinterpret_cast<uint32_t *>(__cvta_shared_to_generic((size_t)h));
    else
        return reinterpret_cast<uint32_t *>(h);
}

template <bool HOT>
__device__ __forceinline__ Img make_img(const View &v) {
    Img g;
    g.I = hot_ptr<HOT>(v.I);
    g.D = hot_ptr<HOT>(v.D);
    g.C = hot_ptr<HOT>(v.C);
    g.dirty = hot_ptr<HOT>(v.dirty);
    g.mark = reinterpret_cast<uint8_t *>(hot_ptr<HOT>(v.mark));
    g.B = hot_ptr<HOT>(v.B);
    g.claim = hot_ptr<HOT>(v.claim);
    g.mw = v.mw;
    g.list = v.list;
    g.E = v.E;
    g.XS = v.XS;
    g.R = v.R;
    g.K = v.K;
    g.A = v.A;
    g.H = v.H;
    g.W = v.W;
    g.WW = v.WW;
    g.S = v.S;
    g.plen = v.plen;
    g.org = v.org;
    g.nblk = v.nblk;
    g.hb = v.hb;
    g.nstrips = v.nstrips;
    g.dense_min = v.dense_min;
    g.scan_min = v.scan_min;
    g.scan_first = v.scan_first;
    g.lastmask = v.lastmask;
    // HOT implies a single CTA per image: constants, so team code folds away
    g.G = HOT ? 1 : v.G;
    g.cs = HOT ? 1 : v.cs;
    g.tid = HOT ? (int)threadIdx.x : v.rank * kThreads + (int)threadIdx.x;
    g.nthr = HOT ? kThreads : v.G * kThreads;
    g.bar = v.bar;
    g.epoch = v.epoch;
    g.err = v.err;
    g.sh = g.G == 1 ? reinterpret_cast<Shared *>(__cvta_shared_to_generic((size_t)v.sh))
                    : reinterpret_cast<Shared *>(v.sh);
    return g;
}

template <bool HOT, int R>
__device__ __noinline__ int prep_nl(const View &v, bool thin, int xmode, bool save_xs) {
    const Img g = make_img<HOT>(v);
    return prep_rank<R>(g, thin, xmode, save_xs);
}

template <bool HOT>
__device__ __forceinline__ int prep_dispatch_v(int r, const View &v, bool thin, int xmode, bool save_xs) {
    switch (r) {
#define TS_PREP_CASE(RR) \
    case RR:             \
        return prep_nl<HOT, RR>(v, thin, xmode, save_xs);
        TS_PREP_CASE(1) TS_PREP_CASE(2) TS_PREP_CASE(3) TS_PREP_CASE(4)
        TS_PREP_CASE(5) TS_PREP_CASE(6) TS_PREP_CASE(7) TS_PREP_CASE(8)
        TS_PREP_CASE(9) TS_PREP_CASE(10) TS_PREP_CASE(11) TS_PREP_CASE(12)
        TS_PREP_CASE(13) TS_PREP_CASE(14) TS_PREP_CASE(15) TS_PREP_CASE(16)
#undef TS_PREP_CASE
        default:
            return -1;
    }
}

template <int FG, bool HOT, int S>
__device__ __noinline__ void epass_nl(const View &v, int t, int cur) {
    const Img g = make_img<HOT>(v);
    epass_ranks<FG, S>(g, t, &g.sh->counters[cur]);
}

template <int FG, bool HOT>
__device__ __forceinline__ void epass_dispatch_v(const View &v, int S, int t, int cur) {
    switch (S) {
        case 1: epass_nl<FG, HOT, 1>(v, t, cur); break;
        case 2: epass_nl<FG, HOT, 2>(v, t, cur); break;
        case 3: epass_nl<FG, HOT, 3>(v, t, cur); break;
        case 4: epass_nl<FG, HOT, 4>(v, t, cur); break;
        case 5: epass_nl<FG, HOT, 5>(v, t, cur); break;
        case 6: epass_nl<FG, HOT, 6>(v, t, cur); break;
        default: epass_nl<FG, HOT, 7>(v, t, cur); break;
    }
}
static_assert(kMaxSlices <= 7, "epass_dispatch covers up to 7 rank slices");

template <int FG, bool HOT, int R>
__device__ __noinline__ void prep_fused_nl(const View &v, bool thin, int xmode, bool save_xs, int t, int cur) {
    const Img g = make_img<HOT>(v);
    (void)t;   // == thin
    if (thin)
        prep_fused<FG, R, true>(g, xmode, save_xs, &g.sh->counters[cur]);
    else
        prep_fused<FG, R, false>(g, xmode, save_xs, &g.sh->counters[cur]);
}

// fused prep + E-pass (see prep_fused); false when not eligible
template <int FG, bool HOT>
__device__ __forceinline__ bool prep_fused_dispatch_v(int r, const View &v, bool thin, int xmode, bool save_xs, int t,
                                                      int cur) {
    // the host planner decided (make_plan_fixed: no R planes then)
    if (!HOT || !v.fused) return false;
    switch (r) {
#define TS_FUSED_CASE(RR)                                            \
    case RR:                                                          \
        prep_fused_nl<FG, HOT, RR>(v, thin, xmode, save_xs, t, cur); \
        return true;
        TS_FUSED_CASE(1) TS_FUSED_CASE(2) TS_FUSED_CASE(3) TS_FUSED_CASE(4)
        TS_FUSED_CASE(5) TS_FUSED_CASE(6) TS_FUSED_CASE(7) TS_FUSED_CASE(8)
#undef TS_FUSED_CASE
        default:
            return false;
    }
}
static_assert(kFusedMaxR == 8, "prep_fused_dispatch_v covers radii 1..8");

template <int FG, bool HOT>
__device__ __noinline__ void epass_prio_nl(const View &v, const int64_t *prio, int t, int cur) {
    const Img g = make_img<HOT>(v);
    epass_prio<FG>(g, prio, t, &g.sh->counters[cur]);
}

struct SweepOut {
    long long passes;
    unsigned flips;
    int evals;
    bool bad;
};

// Tiny-sweep regime (single-CTA images): while the list holds <= 32 words,
// warp 0 runs whole sweeps alone -- fixpoint passes, apply, and re-examination
// of the 3x3 word neighbourhoods of the flipped words (the words a scan of the
// dirty bitmap would find; the bitmap only deduplicates them here and
// is left zero) -- with warp syncs only, no CTA barrier per sweep.  The new
// list keeps the engine precondition; the pass counter is not advanced (tiny
// sweeps use no stamps).  The new list length is left in counters[cur].
struct TinyOut {
    long long sweeps, passes, cycles;
    long long ph[3];   // TS_TINY_PROF: load+passes, apply+claim, re-examination cycles
    unsigned flips;
    bool bad;
};

template <int FG, bool HOT>
__device__ __noinline__ TinyOut tiny_sweeps(const View &v, int t, int cur, long long budget, bool timing) {
    const Img g = make_img<HOT>(v);
    const int lane = threadIdx.x & 31;
    Shared &sh = *g.sh;
    TinyOut o{0, 0, 0, {0, 0, 0}, 0, false};
    const long long c0 = timing ? clock64() : 0;
    int n = *reinterpret_cast<volatile int *>(&sh.counters[cur]);
    const unsigned lt = (1u << lane) - 1u;
    while (n > 0 && n <= 32 && o.sweeps < budget) {
#ifdef TS_TINY_PROF
        long long tq = clock64();
#endif
        Slot s;
        const bool has = lane < n;
        if (has) load_slot<FG>(g, g.list[lane], s);
        const long long cap = 32LL * n + 4;
        long long np = 0;
        while (true) {
            const bool ch = has && update_slot<FG, false>(g, s);
            ++np;
            __syncwarp();
            if (!__any_sync(0xffffffffu, ch)) break;
            if (np > cap) {
                o.bad = true;
                break;
            }
        }
        o.passes += np;
        if (o.bad) break;
#ifdef TS_TINY_PROF
        { const long long t1 = clock64(); o.ph[0] += t1 - tq; tq = t1; }
#endif
        const uint32_t dw = has ? s.d : 0u;
        if (dw) {
            g.I[s.p] ^= dw;
            g.D[s.p] = 0;
            o.flips += __popc(dw);
        }
        __syncwarp();
        // 3x3 word neighbourhoods of the flipped words: the first claimant
        // (dirty bit; all claims in flight together) queues the word at the
        // list head, then the queue is re-examined 32 words at a time and
        // compacted in place into the new list (writes trail the reads)
        const int a = (dw & 1u) ? -1 : 0, b = (dw >> 31) ? 1 : 0;
        const int p0 = has ? s.p : 0;
        unsigned firsts = 0;
        if (dw) {
            uint32_t bit[9], old[9];
#pragma unroll
            for (int k = 0; k < 9; ++k) {   // branch-free: the 9 atomics issue back to back
                const int dx = k % 3 - 1;
                const int q = p0 + (k / 3 - 1) * g.S + dx;
                bit[k] = (dx >= a && dx <= b) ? 1u << (q & 31) : 0u;
                old[k] = atomicOr(&g.dirty[q >> 5], bit[k]);
            }
#pragma unroll
            for (int k = 0; k < 9; ++k)
                if (bit[k] & ~old[k]) firsts |= 1u << k;
        }
        const unsigned any_first = __reduce_or_sync(0xffffffffu, firsts);
        int m = 0;
#pragma unroll
        for (int k = 0; k < 9; ++k) {
            if (!((any_first >> k) & 1u)) continue;   // warp-uniform
            const bool first = (firsts >> k) & 1u;
            const unsigned fm = __ballot_sync(0xffffffffu, first);
            if (first) g.list[m + __popc(fm & lt)] = (uint32_t)(p0 + (k / 3 - 1) * g.S + k % 3 - 1);
            m += __popc(fm);
        }
        __syncwarp();
#ifdef TS_TINY_PROF
        { const long long t1 = clock64(); o.ph[1] += t1 - tq; tq = t1; }
#endif
        int cnt = 0;
        for (int base = 0; base < m; base += 32) {
            const bool in = base + lane < m;
            const int q = in ? (int)g.list[base + lane] : 0;
            __syncwarp();
            uint32_t c = 0;
            if (in) {
                g.dirty[q >> 5] = 0;
                c = cand_word<FG>(g, q, t);
                g.C[q] = c;
                g.D[q] = c;
            }
            const unsigned cm = __ballot_sync(0xffffffffu, c != 0);
            if (c) {
                g.list[cnt + __popc(cm & lt)] = (uint32_t)q;
                asm volatile("prefetch.global.L1 [%0];" ::"l"(g.E + (size_t)q * kEWords));
            }
            cnt += __popc(cm);
            __syncwarp();
        }
        n = cnt;
        __syncwarp();
        ++o.sweeps;
#ifdef TS_TINY_PROF
        o.ph[2] += clock64() - tq;
#endif
    }
    if (lane == 0) sh.counters[cur] = n;
    __syncwarp();
    o.flips = __reduce_add_sync(0xffffffffu, o.flips);
    if (timing) o.cycles = clock64() - c0;
    return o;
}

// ---- compacted re-evaluation passes (dense sweeps after their first pass) --
// After the strip-walk pass only the words stamped by a changed neighbour
// decision need evaluating -- a few percent of the image, scattered, so a
// strip walk would run its warps mostly idle.  Instead the stamped candidate
// words are gathered into a list and evaluated one word per thread.  A pass
// whose changes stamp no candidate word reached the fixpoint (every
// candidate's inputs are unchanged), so an empty list ends the sweep.

// words stamped `v` holding candidates -> list (all team threads; *counter
// zeroed by the caller before a barrier)
__device__ __forceinline__ void collect_stamped(const Img &g, uint8_t v, uint32_t *list, int *counter) {
    const int nchunk = (g.plen + 15) >> 4;   // 16 stamps per uint4
    const uint32_t vv = 0x01010101u * v;
    const int lane = threadIdx.x & 31;
    for (int c0 = g.tid - lane; c0 < nchunk; c0 += g.nthr) {   // warp-uniform trip count
        const int ch = c0 + lane;
        uint32_t h = 0;
        if (ch < nchunk) {
            const uint4 m = reinterpret_cast<const uint4 *>(g.mark)[ch];
            // one bit per matching stamp byte: byte b of word k -> bit 4k + b
            h = ((__vcmpeq4(m.x, vv) & 0x01010101u) * 0x10204080u) >> 28 |
                (((__vcmpeq4(m.y, vv) & 0x01010101u) * 0x10204080u) >> 28) << 4 |
                (((__vcmpeq4(m.z, vv) & 0x01010101u) * 0x10204080u) >> 28) << 8 |
                (((__vcmpeq4(m.w, vv) & 0x01010101u) * 0x10204080u) >> 28) << 12;
        }
        if (!__any_sync(0xffffffffu, h != 0u)) continue;
        // which of the warp's 512 words hold candidates: a lane checking its own
        // 16 consecutive words reads at a 16-word stride (16-way bank conflicts
        // in shared memory, and a dependent load per stamp: a third of c1's
        // excess wavefronts); instead the warp reads the 512 words row-wise
        // (lane l: words 32 j + l, conflict-free, independent) and 16 ballots
        // hand every lane the bits of its own 16 words
        uint32_t mine = 0;   // lane j keeps ballot j (words 32 j .. 32 j + 31)
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int q = c0 * 16 + j * 32 + lane;
            const uint32_t cw = q < g.plen ? g.C[q] : 0u;
            const uint32_t bm = __ballot_sync(0xffffffffu, cw != 0u);
            if (lane == j) mine = bm;
        }
        const uint32_t sel = __shfl_sync(0xffffffffu, mine, lane >> 1);   // words 16 lane .. 16 lane + 15
        const uint32_t valid = h & ((sel >> (16 * (lane & 1))) & 0xFFFFu);
        const int cnt = __popc(valid);
        int incl = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int o = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += o;
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 31);
        if (tot == 0) continue;
        int base = 0;
        if (lane == 31) base = atomicAdd(counter, tot);
        base = __shfl_sync(0xffffffffu, base, 31) + incl - cnt;
        for (uint32_t t = valid; t; t &= t - 1) list[base++] = (uint32_t)(ch * 16 + __ffs(t) - 1);
    }
}

// one listed word's evaluation: inputs, then the word-fix solve, then commit
struct WordEval {
    int p;
    Nb in, dn;       // image neighbours; decision neighbours (W/E from the word itself)
    uint4 e0, e1;    // E masks
    uint32_t c, ml, mr, old;
};

__device__ __forceinline__ void load_eval(const Img &g, int p, WordEval &w) {
    w.p = p;
    w.in = nbrs(g.I, g, p);
    load_e(g, p, w.e0, w.e1);
    w.c = g.C[p];
    const uint32_t *u = g.D + p - g.S, *m = g.D + p, *d = g.D + p + g.S;
    w.dn.nw = from_west(u[-1], u[0]);
    w.dn.n = u[0];
    w.dn.ne = from_east(u[0], u[1]);
    w.dn.sw = from_west(d[-1], d[0]);
    w.dn.s = d[0];
    w.dn.se = from_east(d[0], d[1]);
    w.ml = m[-1];
    w.mr = m[1];
    w.old = m[0];
}

// decisions of the word with its in-word chains resolved (word fix)
template <int FG>
__device__ __forceinline__ uint32_t solve_eval(WordEval &w) {
    uint32_t nd = w.old;
    for (uint32_t pd = ~w.old; nd != pd;) {
        pd = nd;
        w.dn.w = from_west(w.ml, nd);
        w.dn.e = from_east(nd, w.mr);
        nd = decide<FG>(w.c, w.in, w.dn, w.e0, w.e1);
    }
    return nd;
}

__device__ __forceinline__ bool commit_eval(const Img &g, const WordEval &w, uint32_t nd, uint8_t next) {
    if (nd == w.old) return false;
    g.D[w.p] = nd;
    stamp_chg(g, w.p, nd ^ w.old, w.e0, w.e1, next, false);
    return true;
}

// Compacted passes with claims: when a word's decisions change, each affected
// neighbour word (E-directed, as in stamp_chg) that holds candidates is
// claimed in the pass's claim bitmap; its first claimant appends it to the next
// pass's list.  A pass that claims nothing ends the sweep (every candidate's
// inputs are unchanged since its last evaluation).
__device__ __forceinline__ void claim_chg(const Img &g, int p, uint32_t chg, uint4 e0, uint4 e1, uint32_t *Q,
                                          uint32_t *next, int *ncount) {
    const int S = g.S;
    auto claim = [&](int q) {
        if (g.C[q] == 0u) return;
        const uint32_t bit = 1u << (q & 31);
        if (atomicOr(&Q[q >> 5], bit) & bit) return;
        next[atomicAdd(ncount, 1)] = (uint32_t)q;
    };
    const uint32_t lNW = ~e0.x, lN = ~e0.y, lNE = ~e0.z, lW = ~e0.w;   // "that neighbour is later"
    const uint32_t lE = ~e1.x, lSW = ~e1.y, lS = ~e1.z, lSE = ~e1.w;
    if (chg & (lN | (lNW & ~1u) | (lNE & 0x7FFFFFFFu))) claim(p - S);
    if (chg & (lS | (lSW & ~1u) | (lSE & 0x7FFFFFFFu))) claim(p + S);
    if (chg & 1u) {
        if (lNW & 1u) claim(p - S - 1);
        if (lW & 1u) claim(p - 1);
        if (lSW & 1u) claim(p + S - 1);
    }
    if (chg >> 31) {
        if (lNE >> 31) claim(p - S + 1);
        if (lE >> 31) claim(p + 1);
        if (lSE >> 31) claim(p + S + 1);
    }
}

// the same claims, returning the newly claimed words as a mask over qs[]
// (the caller appends them, aggregated per warp)
__device__ __forceinline__ uint32_t claim_chg_mask(const Img &g, int p, uint32_t chg, uint4 e0, uint4 e1, uint32_t *Q,
                                                   int (&qs)[8]) {
    const int S = g.S;
    uint32_t firsts = 0;   // bit k: qs[k] newly claimed here
    auto claim = [&](int k, int q) {
        qs[k] = q;
        if (g.C[q] == 0u) return;
        const uint32_t bit = 1u << (q & 31);
        if (!(atomicOr(&Q[q >> 5], bit) & bit)) firsts |= 1u << k;
    };
    const uint32_t lNW = ~e0.x, lN = ~e0.y, lNE = ~e0.z, lW = ~e0.w;   // "that neighbour is later"
    const uint32_t lE = ~e1.x, lSW = ~e1.y, lS = ~e1.z, lSE = ~e1.w;
    if (chg & (lN | (lNW & ~1u) | (lNE & 0x7FFFFFFFu))) claim(0, p - S);
    if (chg & (lS | (lSW & ~1u) | (lSE & 0x7FFFFFFFu))) claim(1, p + S);
    if (chg & 1u) {
        if (lNW & 1u) claim(2, p - S - 1);
        if (lW & 1u) claim(3, p - 1);
        if (lSW & 1u) claim(4, p + S - 1);
    }
    if (chg >> 31) {
        if (lNE >> 31) claim(5, p - S + 1);
        if (lE >> 31) claim(6, p + 1);
        if (lSE >> 31) claim(7, p + S + 1);
    }
    return firsts;
}

// pass j of a sweep's compacted phase: evaluate list (n words, in-word chains
// resolved at once), claims into bitmap Q -> next; Qclear (the next pass's
// bitmap, idle now) is cleared on the way.  Single-CTA images append per
// claim (shared-memory counter); teams aggregate the appends per warp (one
// atomic on the team's global counter per warp and step: per-claim global
// atomics on one address serialised c3 by 25%).
template <int FG>
__device__ __forceinline__ void claim_pass(const Img &g, const uint32_t *list, int n, uint32_t *Q, uint32_t *Qclear,
                                           uint32_t *next, int *ncount, int &evals) {
    for (int q = g.tid; q < g.mw; q += g.nthr) Qclear[q] = 0u;
    if (g.G == 1) {
        for (int sl = g.tid; sl < n; sl += g.nthr) {
            WordEval a;
            load_eval(g, (int)list[sl], a);
            const uint32_t nd = solve_eval<FG>(a);
            ++evals;
            if (nd != a.old) {
                g.D[a.p] = nd;
                claim_chg(g, a.p, nd ^ a.old, a.e0, a.e1, Q, next, ncount);
            }
        }
        return;
    }
    const int lane = threadIdx.x & 31;
    for (int s0 = g.tid - lane; s0 < n; s0 += g.nthr) {   // warp-uniform trip count
        const int sl = s0 + lane;
        uint32_t firsts = 0;
        int qs[8];
        if (sl < n) {
            WordEval a;
            load_eval(g, (int)list[sl], a);
            const uint32_t nd = solve_eval<FG>(a);
            ++evals;
            if (nd != a.old) {
                g.D[a.p] = nd;
                firsts = claim_chg_mask(g, a.p, nd ^ a.old, a.e0, a.e1, Q, qs);
            }
        }
        const int cnt = __popc(firsts);
        int incl = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int o = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += o;
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 31);
        if (tot == 0) continue;
        int base = 0;
        if (lane == 31) base = atomicAdd(ncount, tot);
        base = __shfl_sync(0xffffffffu, base, 31) + incl - cnt;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if ((firsts >> k) & 1u) next[base++] = (uint32_t)qs[k];
    }
}

// ---- global-plane kernels: every phase of a sweep as its own function ------
// With the planes in L2 the per-thread state of a phase is mostly 64-bit plane
// pointers; inlined together the phases of a sweep exceeded the register
// budget (64 registers at 1024 threads) and 15% of the executed instructions
// of the c2 dense sweeps were local-memory spill traffic (ncu: 5.7 G L2
// sectors of local traffic against 7.2 G of global).  As separate functions
// each phase materialises only the pointers it uses.
#ifndef TS_SPLIT
#define TS_SPLIT 1
#endif

template <int FG>
__device__ __noinline__ int dpass_nl(const View &v, int pc) {
    const Img g = make_img<false>(v);
    int evals = 0;
    if constexpr (kDensePipe)
        dense_pass_l2<FG>(g, pc, evals);
    else
        dense_pass_l2_plain<FG>(g, pc, evals);
    return evals;
}

static __device__ __noinline__ void collect_nl(const View &v, int stamp, uint32_t *list, int *counter) {
    const Img g = make_img<false>(v);
    collect_stamped(g, (uint8_t)stamp, list, counter);
}

template <int FG>
__device__ __noinline__ int claim_pass_nl(const View &v, const uint32_t *list, int n, int jq, uint32_t *next,
                                          int *ncount) {
    const Img g = make_img<false>(v);
    int evals = 0;
    claim_pass<FG>(g, list, n, g.claim + (jq & 1) * g.mw, g.claim + ((jq + 1) & 1) * g.mw, next, ncount, evals);
    return evals;
}

// apply after a dense sweep: the decisions of 8 rows, then the image words of
// the flipping ones, are requested together
static __device__ __noinline__ unsigned apply_dense_nl(const View &v) {
    const Img g = make_img<false>(v);
    unsigned flips = 0;
    walk_strips(g, [&](int x, int y0, int y1, int) {
        constexpr int kB = 8;
        int p = pidx(g, y0, x);
        for (int yb = y0; yb < y1; yb += kB, p += kB * g.S) {
            uint32_t dw[kB], iw[kB];
#pragma unroll
            for (int j = 0; j < kB; ++j) dw[j] = yb + j < y1 ? g.D[p + j * g.S] : 0u;
#pragma unroll
            for (int j = 0; j < kB; ++j)
                if (dw[j]) iw[j] = g.I[p + j * g.S];
#pragma unroll
            for (int j = 0; j < kB; ++j) {
                if (dw[j]) {
                    g.I[p + j * g.S] = iw[j] ^ dw[j];
                    g.D[p + j * g.S] = 0;
                    flips += __popc(dw[j]);
                }
            }
        }
    });
    return flips;
}

static __device__ __noinline__ unsigned apply_list_nl(const View &v, int n) {
    const Img g = make_img<false>(v);
    unsigned flips = 0;
    for (int sl = g.tid; sl < n; sl += g.nthr) {
        const int p = (int)g.list[sl];
        flips += apply_word(g, p, g.D[p]);
    }
    return flips;
}

// Scan pass (teams, planes in L2): every thread scans 16 stamps, evaluates the
// candidate words stamped `cur` (word fix) and stamps `next` on the words a
// change affects -- no list, no claim bitmap, no counter atomics.  A listed
// evaluation over L2 is a chain of five dependent round trips (list entry,
// planes, neighbours' candidates, claim atomic, list counter: ~10 K cycles per
// word and thread on c3); here it is two (stamps, planes), the stamps are
// fire-and-forget byte stores, and a thread's words are neighbours (L1 hits).
// Measured on c3 (148-CTA cooperative team): all compacted passes of the dense
// sweeps as scan passes 19.5 -> 18.3 ms; stopping at a change threshold and
// finishing with claim passes was in between; two words in flight per thread
// were slower (20.2 ms).  On c2 (cluster teams of 4: 43 words per thread) the
// scan itself costs more than the lists save (35.1 -> 36.7 ms), so only the
// cooperative teams use it (KParams::scan_min).  Returns through *counter the
// number of words changed (0: fixpoint).
__shared__ uint16_t g_scan_queue[kWarps][512];   // scan_pass: per-warp queue of stamped words (offsets in the warp's 512)

template <int FG, bool FIRST>
__device__ __forceinline__ void scan_pass(const Img &g, uint8_t cur, uint8_t next, int *counter, int &evals) {
    // Stamped words cluster (changes spread locally): a thread evaluating its
    // own 16 stamps would serialise up to 16 evaluations while its warp idles.
    // So the warp compacts the stamped words of its 512 stamps into a queue in
    // shared memory (ballot-free prefix sums, no atomics) and the lanes take
    // queue entries round-robin.
    uint16_t(&wq)[kWarps][512] = g_scan_queue;
    const int nchunk = (g.plen + 15) >> 4;   // 16 stamps per uint4
    const uint32_t vv = 0x01010101u * cur;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int changed = 0;
    for (int c0 = g.tid - lane; c0 < nchunk; c0 += g.nthr) {   // warp-uniform trip count
        const int ch = c0 + lane;
        uint32_t h = 0;
        if (ch < nchunk) {
            if constexpr (FIRST) {
                // a sweep's first pass: every word holding candidates (instead of
                // the strip walk, whose warps pay an evaluation for every row in
                // which any lane has candidates)
                const uint4 *cp = reinterpret_cast<const uint4 *>(g.C) + (size_t)ch * 4;
                uint4 c4[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) c4[j] = (ch * 16 + j * 4 < g.plen) ? cp[j] : make_uint4(0, 0, 0, 0);
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    h |= ((c4[j].x != 0u ? 1u : 0u) | (c4[j].y != 0u ? 2u : 0u) | (c4[j].z != 0u ? 4u : 0u) |
                          (c4[j].w != 0u ? 8u : 0u))
                         << (4 * j);
            } else {
                const uint4 m = reinterpret_cast<const uint4 *>(g.mark)[ch];
                h = ((__vcmpeq4(m.x, vv) & 0x01010101u) * 0x10204080u) >> 28 |
                    (((__vcmpeq4(m.y, vv) & 0x01010101u) * 0x10204080u) >> 28) << 4 |
                    (((__vcmpeq4(m.z, vv) & 0x01010101u) * 0x10204080u) >> 28) << 8 |
                    (((__vcmpeq4(m.w, vv) & 0x01010101u) * 0x10204080u) >> 28) << 12;
            }
        }
        const int cnt = __popc(h);
        int incl = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int o = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += o;
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 31);
        if (tot == 0) continue;
        int at = incl - cnt;
        for (uint32_t t = h; t; t &= t - 1) wq[warp][at++] = (uint16_t)(lane * 16 + __ffs(t) - 1);
        __syncwarp();
        for (int i = lane; i < tot; i += 32) {
            const int p = c0 * 16 + (int)wq[warp][i];
            if (p >= g.plen || g.C[p] == 0u) continue;
            WordEval a;
            load_eval(g, p, a);
            const uint32_t nd = solve_eval<FG>(a);
            ++evals;
            if (commit_eval(g, a, nd, next)) ++changed;
        }
        __syncwarp();
    }
    add_count_partial(changed, counter);
}

template <int FG, bool FIRST>
__device__ __noinline__ int scan_pass_nl(const View &v, int cur, int next, int *counter) {
    const Img g = make_img<false>(v);
    int evals = 0;
    scan_pass<FG, FIRST>(g, (uint8_t)cur, (uint8_t)next, counter, evals);
    return evals;
}

// Passes j, j+1, ... until one claims nothing.  Pass j reads lists[j & 1]
// (n words), claims into bitmap j & 1 and list (j + 1) & 1 counted in
// lcount[(j + 1) % 3], clears bitmap (j + 1) & 1 and zeroes lcount[(j + 2) % 3]
// (last read before the previous barrier).  Between sweeps both bitmaps are
// zero and lcount[] is reset by the engine after the post-sweep barrier.
template <int FG, bool SPLIT>
__device__ __forceinline__ void claim_passes(const View &v, const Img &g, uint32_t *const (&lists)[2], int j, int n,
                                             long long cap, SweepOut &o) {
    Shared &sh = *g.sh;
    while (n > 0) {
        if (o.passes > cap) {
            o.bad = true;
            break;
        }
        if (g.tid == 0) sh.lcount[(j + 2) % 3] = 0;
        if constexpr (SPLIT)
            o.evals += claim_pass_nl<FG>(v, lists[j & 1], n, j, lists[(j + 1) & 1], &sh.lcount[(j + 1) % 3]);
        else
            claim_pass<FG>(g, lists[j & 1], n, g.claim + (j & 1) * g.mw, g.claim + ((j + 1) & 1) * g.mw,
                           lists[(j + 1) & 1], &sh.lcount[(j + 1) % 3], o.evals);
        ++o.passes;
        if constexpr (SPLIT) {
            n = team_sync_get(g, &sh.lcount[(j + 1) % 3]);
        } else {
            team_sync(g);
            n = *reinterpret_cast<volatile int *>(&sh.lcount[(j + 1) % 3]);
        }
        ++j;
    }
}

// list sweep (> 32 listed words): a claim pass over the sweep list, then
// claim passes until none claims; then apply
template <int FG, bool SPLIT>
__device__ __forceinline__ SweepOut list_sweep(const View &v, const Img &g, int n, long long cap) {
    SweepOut o{0, 0, 0, false};
    Shared &sh = *g.sh;
    uint32_t *const lists[2] = {g.list + g.plen, g.list + g.plen + g.plen / 2};   // each >= nwords / 2 >= n
    if (g.tid == 0) sh.dcount = 0;
    // pass 1 (j = 1): the sweep list; its claims become lists[0] (lcount[2])
    if constexpr (SPLIT)
        o.evals += claim_pass_nl<FG>(v, g.list, n, 1, lists[0], &sh.lcount[2]);
    else
        claim_pass<FG>(g, g.list, n, g.claim + g.mw, g.claim, lists[0], &sh.lcount[2], o.evals);
    ++o.passes;
    team_sync(g);
    claim_passes<FG, SPLIT>(v, g, lists, 2, *reinterpret_cast<volatile int *>(&sh.lcount[2]), cap, o);
    if constexpr (SPLIT) {
        o.flips += apply_list_nl(v, n);
    } else {
        for (int sl = g.tid; sl < n; sl += g.nthr) {
            const int p = (int)g.list[sl];
            o.flips += apply_word(g, p, g.D[p]);
        }
    }
    return o;
}

// dense sweep: one strip-walk pass, then compacted passes until no candidate
// word is stamped; then apply (all threads)
template <int FG, bool HOT>
__device__ __forceinline__ SweepOut dense_sweep(const View &v, const Img &g, long long cap, int pc0, bool timing) {
    constexpr bool SPLIT = !HOT && TS_SPLIT;
    SweepOut o{0, 0, 0, false};
    int pc = pc0;
    Shared &sh = *g.sh;
    uint32_t *const lists[2] = {g.list, g.list + g.plen};
    const bool tm = timing && g.tid == 0;
    long long t0 = tm ? clock64() : 0;
    if constexpr (HOT)
        dense_pass<FG>(g, pc, o.evals);
    else if constexpr (SPLIT) {
        if (g.scan_min >= 0 && g.scan_first)   // (its change count is not needed: the scan passes follow)
            o.evals += scan_pass_nl<FG, true>(v, pc, pc + 1, &sh.dcount);
        else
            o.evals += dpass_nl<FG>(v, pc);
    }
    else if constexpr (kDensePipe)
        dense_pass_l2<FG>(g, pc, o.evals);
    else
        dense_pass_l2_plain<FG>(g, pc, o.evals);
    ++o.passes;
    ++pc;
    team_sync(g);   // stamps of the strip-walk pass complete
    if (tm) {
        const long long t1 = clock64();
        sh.dtime[0] += t1 - t0;
        t0 = t1;
    }
    bool fixpoint = false;   // a scan pass changed nothing: no stamps left, skip the compacted passes
    if constexpr (SPLIT) {
        // scan passes while many words change (see scan_pass); pass k counts
        // its changes in lcount[3 + k % 3] and zeroes the counter of pass k + 1
        // (lcount[0..2], the compacted passes' counters, stay zero meanwhile)
        if (g.scan_min >= 0) {
            for (int k = 0;; ++k) {
                if (o.passes > cap) {
                    o.bad = true;
                    break;
                }
                if (g.tid == 0) sh.lcount[3 + (k + 1) % 3] = 0;   // last read before the previous barrier
                o.evals += scan_pass_nl<FG, false>(v, pc, pc + 1, &sh.lcount[3 + k % 3]);
                ++o.passes;
                ++pc;
                const int nchg = team_sync_get(g, &sh.lcount[3 + k % 3]);
                if (nchg == 0) fixpoint = true;
                if (nchg <= g.scan_min) break;   // few changes: the words stamped `pc` -> compacted passes
            }
        }
    }
    if (!fixpoint) {
    // the strip walk stamped densely: gather the stamped candidate words by a
    // scan (j = 2's list, lcount[2]); later passes build their lists by claims
    if constexpr (SPLIT)
        collect_nl(v, pc, lists[0], &sh.lcount[2]);
    else
        collect_stamped(g, (uint8_t)pc, lists[0], &sh.lcount[2]);
    int n2;
    if constexpr (SPLIT) {
        n2 = team_sync_get(g, &sh.lcount[2]);
    } else {
        team_sync(g);
        n2 = *reinterpret_cast<volatile int *>(&sh.lcount[2]);
    }
    if (tm) {
        const long long t1 = clock64();
        sh.dtime[1] += t1 - t0;
        sh.dtime[3] += n2;
        t0 = t1;
    }
    claim_passes<FG, SPLIT>(v, g, lists, 2, n2, cap, o);
    if (tm) sh.dtime[2] += clock64() - t0;
    }
    if constexpr (SPLIT) {
        o.flips += apply_dense_nl(v);
    } else {
        for_strip(g, [&](int y, int x, int p) {
            const uint32_t dw = g.D[p];
            if (dw) {
                g.I[p] ^= dw;
                g.D[p] = 0;
                o.flips += __popc(dw);
            }
        });
    }
    return o;
}

// the sweeps as separate functions: each gets its own register allocation
// (sweeps of <= 32 words run in the tiny regime, tiny_sweeps)
template <int FG, bool HOT>
__device__ __noinline__ SweepOut dense_sweep_nl(const View &v, long long cap, int pc, bool timing) {
    const Img g = make_img<HOT>(v);
    return dense_sweep<FG, HOT>(v, g, cap, pc, timing);
}

template <int FG, bool HOT>
__device__ __noinline__ SweepOut sparse_sweep_nl(const View &v, int n, long long cap, int pc) {
    const Img g = make_img<HOT>(v);
    (void)pc;
    return list_sweep<FG, !HOT && TS_SPLIT>(v, g, n, cap);
}

// re-examination after a sweep: all words (dense) or the compacted dirty words
// (list sweeps; the compacted lists' space is free again)
template <int FG, bool HOT>
__device__ __forceinline__ void rebuild_any(const Img &g, bool dense, int t, int *counter) {
    if (dense)
        rebuild_dense<FG, HOT ? 1 : kStreamBatch>(g, t, counter);
    else
        rebuild_compact<FG, !HOT>(g, t, g.list + g.plen, &g.sh->dcount, counter);
}

template <int FG>
__device__ __noinline__ void rebuild_nl(const View &v, bool dense, int t, int *counter) {
    const Img g = make_img<false>(v);
    rebuild_any<FG, false>(g, dense, t, counter);
}

static __device__ __noinline__ void build_list_nl(const View &v, int *counter) {
    const Img g = make_img<false>(v);
    build_list<true>(g, counter);
}

// discard a prepared sweep (max_iter reached): D and C back to zero
__device__ __forceinline__ void discard_sweep(const Img &g, int n, bool list_ok) {
    if (!list_ok) {
        for_strip(g, [&](int y, int x, int p) {
            g.D[p] = 0;
            g.C[p] = 0;
        });
        return;
    }
    for (int s = g.tid; s < n; s += g.nthr) {
        const int p = (int)g.list[s];
        g.D[p] = 0;
        g.C[p] = 0;
    }
}

// the priority-ordered flip engine (topo.py:211-258), see file header.
// Precondition (after a __syncthreads): C = candidates of every word, D = C,
// list = words with C != 0, counters[cur] = its size, dirty bitmap zero.
#ifndef TS_ENGINE_INLINE
#define TS_ENGINE_INLINE __noinline__
#endif

template <int FG, bool HOT>
__device__ TS_ENGINE_INLINE int2 engine_nl(const View &v, int t, long long max_sweeps, int *err, bool timing, int cur0,
                                           int pc0) {
    (void)err;
    const long long ty0 = timing ? clock64() : 0;
    const Img g = make_img<HOT>(v);
    Shared &sh = *g.sh;
    const int tid = g.tid;
    volatile int *vcount = sh.counters;
    long long tyl = timing ? clock64() : 0;   // start of the current loop top
    if (timing && tid == 0) sh.ystat[0] += tyl - ty0;
    int cur = cur0, pc = pc0;
    Stats st{};
    st.timing = timing;
    long long sweeps = 0;
    const long long sweep_cap = (long long)g.H * g.W + 2;   // >= 1 flip per sweep, <= 1 flip per pixel
    bool list_ok = false;   // the E-pass and dense re-examination only count candidates
    int n_next = vcount[cur];   // global planes: handed over by the barrier that ends a sweep
    while (true) {
        const int n = HOT ? vcount[cur] : n_next;
        if (n == 0) break;
        if ((max_sweeps >= 0 && sweeps >= max_sweeps) || sweeps >= sweep_cap) {
            if (sweeps >= sweep_cap && (max_sweeps < 0 || sweeps < max_sweeps)) {
                if (tid == 0) set_err(g.err, ERR_SWEEP_CAP);
            }
            discard_sweep(g, n, list_ok);
            team_sync(g);
            break;
        }
        const long long tj0 = st.timing ? clock64() : 0;
        if (st.timing && tid == 0) {
            sh.ystat[1] += tj0 - tyl;
            sh.ystat[3] += 1;
        }
        const long long cap = 32LL * n + 4;   // DAG depth <= #candidates
        // warp-resident regime (needs the list).  Teams too: warp 0 of the
        // team's rank-0 CTA runs the sweeps alone (its own writes are coherent
        // in its L1, write-through to L2); the team barriers around it publish
        // the planes in both directions -- 2 team barriers per regime instead
        // of ~5 per sweep plus a scan of the whole dirty bitmap
        const bool tiny = n <= 32;
        const bool dense = n > g.dense_min && !tiny;
        if (!dense && !list_ok) {   // sparse sweep after a counting pass: build the list
            if (tid == 0) sh.counters[cur ^ 1] = 0;
            team_sync(g);
            if constexpr (!HOT && TS_SPLIT)
                build_list_nl(v, &sh.counters[cur ^ 1]);
            else
                build_list<!HOT>(g, &sh.counters[cur ^ 1]);
            team_sync(g);
            list_ok = true;
            if (st.timing && tid == 0 && n > 512) {
                sh.bstat[0] += clock64() - tj0;
                sh.bstat[3] += 1;
            }
        }
        const long long tjb = st.timing ? clock64() : 0;
        if (tiny) {
            long long budget = sweep_cap - sweeps;
            if (max_sweeps >= 0) budget = min(budget, max_sweeps - sweeps);
            if (tid < 32) {   // (tid is the team thread id)
                const TinyOut to = tiny_sweeps<FG, HOT>(v, t, cur, budget, st.timing);
                if (tid == 0) {
                    sh.bad = to.bad ? 1 : 0;
                    sh.tiny[0] = to.sweeps;
                    sh.tiny[1] = to.passes;
                    if (st.timing) {
                        st.cyc_tiny += to.cycles;
                        st.cyc_jacobi += to.cycles;
                        st.n_tiny += to.sweeps;
                        st.pass_tiny += to.passes;
#ifdef TS_TINY_PROF
                        st.cyc_dense += to.ph[0];
                        st.pass_dense += to.ph[1];
                        st.cyc_update += to.ph[2];
#endif
                        atomicAdd(&sh.flips, (unsigned long long)to.flips);
                    }
                }
            }
            team_sync(g);
            sweeps += *reinterpret_cast<volatile long long *>(&sh.tiny[0]);
            st.passes += *reinterpret_cast<volatile long long *>(&sh.tiny[1]);
            const bool tbad = *reinterpret_cast<volatile int *>(&sh.bad) != 0;
            team_sync(g);   // shared results read before they can be rewritten
            if (st.timing && tid == 0) {
                sh.xstat[0] += clock64() - tj0;
                sh.xstat[1] += 1;
            }
            if (tbad) {
                if (tid == 0) set_err(g.err, ERR_JACOBI_CAP);
                break;
            }
            if (st.timing) tyl = clock64();
            if constexpr (!HOT) n_next = vcount[cur];   // left by the tiny regime
            continue;
        }
        SweepOut o;
        if (dense)
            o = dense_sweep_nl<FG, HOT>(v, cap, pc, st.timing);
        else
            o = sparse_sweep_nl<FG, HOT>(v, n, cap, pc);
        if (tid == 0) {
            sh.bad = o.bad ? 1 : 0;
            sh.counters[cur ^ 1] = 0;
        }
        int sweep_bad;
        if constexpr (HOT) {
            team_sync(g);
            sweep_bad = 0;
        } else {
            sweep_bad = team_sync_get(g, &sh.bad);
        }
        if (tid == 0)   // all read before that barrier
            sh.lcount[0] = sh.lcount[1] = sh.lcount[2] = sh.lcount[3] = sh.lcount[4] = sh.lcount[5] = 0;
        if (HOT ? *reinterpret_cast<volatile int *>(&sh.bad) : sweep_bad) {
            if (tid == 0) set_err(g.err, ERR_JACOBI_CAP);
            break;
        }
        // pass counter stays team-uniform: dense and list sweeps count passes
        // uniformly (the tiny regime, one warp and no stamps, does not advance it)
        pc += (int)o.passes;
        if (st.timing) {
            const int ev = __reduce_add_sync(0xffffffffu, o.evals);
            const unsigned fl = __reduce_add_sync(0xffffffffu, o.flips);
            if ((tid & 31) == 0) {
                if (ev) atomicAdd(&sh.evals, (unsigned long long)ev);
                if (fl) atomicAdd(&sh.flips, (unsigned long long)fl);
            }
        }
        const long long tj1 = st.timing ? clock64() : 0;
        cur ^= 1;
        if constexpr (!HOT && TS_SPLIT)
            rebuild_nl<FG>(v, dense, t, &sh.counters[cur]);
        else
            rebuild_any<FG, HOT>(g, dense, t, &sh.counters[cur]);
        list_ok = !dense;
        if constexpr (HOT)
            team_sync(g);
        else
            n_next = team_sync_get(g, &sh.counters[cur]);
        ++sweeps;
        st.passes += o.passes;
        if (st.timing) {
            const long long tj2 = clock64();
            st.cyc_jacobi += tj1 - tj0;
            st.cyc_update += tj2 - tj1;
            if (dense) {
                st.cyc_dense += tj1 - tj0;
                st.n_dense += 1;
                st.pass_dense += o.passes;
            } else if (n <= 32) {
                st.cyc_tiny += tj1 - tj0;
                st.n_tiny += 1;
                st.pass_tiny += o.passes;
            } else if (tid == 0) {
#ifndef TS_SSTAT_SPLIT
#define TS_SSTAT_SPLIT 512   // stats: boundary between the two list-sweep buckets
#endif
                const int b = n <= TS_SSTAT_SPLIT ? 0 : 2;
                sh.sstat[b] += 1;
                sh.sstat[b + 1] += tj2 - tj0;
                if (n > 512) {
                    sh.bstat[1] += tj1 - tjb;
                    sh.bstat[2] += tj2 - tj1;
                }
            }
            tyl = clock64();
        }
    }
    const long long tye = timing ? clock64() : 0;
    if (tid == 0) {
        EngineIO &io = sh.eio;
        io.sweeps += sweeps;
        io.passes += st.passes;
        io.calls += 1;
        io.cyc_jacobi += st.cyc_jacobi;
        io.cyc_update += st.cyc_update;
        io.cyc_tiny += st.cyc_tiny;
        io.n_tiny += st.n_tiny;
        io.pass_tiny += st.pass_tiny;
        io.cyc_dense += st.cyc_dense;
        io.n_dense += st.n_dense;
        io.pass_dense += st.pass_dense;
        if (timing) sh.ystat[2] += clock64() - tye;
    }
    return make_int2(cur, pc);
}

template <int FG, bool HOT>
__device__ __forceinline__ void engine(const View &v, int t, long long max_sweeps, Shared &sh, int &cur, int *err,
                                       Stats &st, int &pc) {
    (void)sh;
    (void)st;
    const int2 r = engine_nl<FG, HOT>(v, t, max_sweeps, err, st.timing, cur, pc);
    cur = r.x;
    pc = r.y;
}

template <int FG, bool HOT>
__device__ __forceinline__ void run_stage(const View &v, const Img &gt, int r, bool thin, int xmode, bool save_xs,
                                          Shared &sh, int &cur, int *err, Stats &st, int &pc) {
    if (gt.tid == 0) sh.counters[cur] = 0;
    const long long tp0 = st.timing ? clock64() : 0;
#ifndef TS_FUSED
#define TS_FUSED 1
#endif
    if (!(TS_FUSED && prep_fused_dispatch_v<FG, HOT>(r, v, thin, xmode, save_xs, thin ? 1 : 0, cur))) {
        // the counter reset above must land before the E-pass counts
        const int S = prep_dispatch_v<HOT>(r, v, thin, xmode, save_xs);
        team_sync(gt);
        if (st.timing) st.cyc_rank += clock64() - tp0;
        epass_dispatch_v<FG, HOT>(v, S, thin ? 1 : 0, cur);
    }
    team_sync(gt);
    if (st.timing) st.cyc_prep += clock64() - tp0;
    const long long te0 = st.timing ? clock64() : 0;
    engine<FG, HOT>(v, thin ? 1 : 0, -1, sh, cur, err, st, pc);
    if (st.timing && gt.tid == 0) {
        const long long te1 = clock64();
        sh.xstat[2] += te1 - te0;   // whole engine call
        sh.xstat[3] += te1 - tp0;   // whole stage
    }
}

// bit rows [H][WW] (host- or P4-packed, or a segment's saved state) into a
// plane; the strip's words are requested together (one latency per batch).
// Plain (L1-cached) loads: a segment's state written on another SM is read
// only after the lead's ld.acquire.gpu (which invalidates this SM's L1,
// CCTL.IVALL) and a CTA barrier.
__device__ __forceinline__ void load_rows(const Img &g, const uint32_t *from, uint32_t *to) {
    walk_strips(g, [&](int x, int y0, int y1, int) {
        constexpr int kB = 16;
        for (int yb = y0; yb < y1; yb += kB) {
            uint32_t w[kB];
#pragma unroll
            for (int j = 0; j < kB; ++j)
                if (yb + j < y1) w[j] = from[(size_t)(yb + j) * g.WW + x];
#pragma unroll
            for (int j = 0; j < kB; ++j)
                if (yb + j < y1) to[pidx(g, yb + j, x)] = w[j];
        }
    });
}

// image prologue: clear planes, pack inputs, validate (all team threads)
template <bool HOT>
__device__ __noinline__ void load_image_nl(const View &v, const KParams *pp, size_t pix, int img) {
    const KParams &p = *pp;
    const Img g = make_img<HOT>(v);
    const int tid = g.tid, nthr = g.nthr;
    const bool has_k = p.keep != nullptr, has_a = p.avoid != nullptr;
    for (int q = tid; q < g.plen; q += nthr) {
        g.I[q] = 0;
        g.D[q] = 0;
        g.C[q] = 0;
        g.B[q] = ~0u;   // pads blocked
    }
    for (int q = tid; q < (g.plen + 31) >> 5; q += nthr) g.dirty[q] = 0;
    for (int q = tid; q < 2 * g.mw; q += nthr) g.claim[q] = 0;
    for (int q = tid; q < (g.plen + 15) >> 4; q += nthr)
        reinterpret_cast<uint4 *>(g.mark)[q] = make_uint4(0, 0, 0, 0);
    team_sync(g);
    const size_t wimg = (size_t)img * g.H * g.WW;
    if (p.packed_io) {   // bit rows (host- or P4-packed: always binary), constraints too
        load_rows(g, reinterpret_cast<const uint32_t *>(p.in) + wimg, g.I);
    } else {
        pack_plane(p.in + pix, g.I, g, p.err, ERR_NOT_BINARY);
    }
    if (p.mode == MODE_THIN || p.mode == MODE_THICKEN) {
        pack_plane(p.keep + pix, g.B, g, p.err, ERR_CONSTRAINT_NOT_BINARY);
    } else if (p.packed_io) {
        if (has_k) load_rows(g, reinterpret_cast<const uint32_t *>(p.keep) + wimg, g.K);
        if (has_a) load_rows(g, reinterpret_cast<const uint32_t *>(p.avoid) + wimg, g.A);
    } else {
        if (has_k) pack_plane(p.keep + pix, g.K, g, p.err, ERR_CONSTRAINT_NOT_BINARY);
        if (has_a) pack_plane(p.avoid + pix, g.A, g, p.err, ERR_CONSTRAINT_NOT_BINARY);
    }
    team_sync(g);
    for_strip(g, [&](int y, int x, int q) {
        const uint32_t X = g.I[q];
        if (p.mode == MODE_THIN) {
            if (g.B[q] & ~X) set_err(p.err, ERR_KEEP_NOT_OBJECT);          // topo.py:264-265
        } else if (p.mode == MODE_THICKEN) {
            const uint32_t allowed = g.B[q];
            if (X & ~allowed) set_err(p.err, ERR_ALLOWED_NOT_SUPERSET);    // topo.py:332-333
            g.B[q] = ~allowed;   // blocked = not allowed; padding bits blocked
        } else {
            const uint32_t K = has_k ? g.K[q] : 0u, A = has_a ? g.A[q] : 0u;
            if (K & A) set_err(p.err, ERR_KEEP_AVOID);                     // smoothing.py:201-202
            if (K & ~X) set_err(p.err, ERR_KEEP_NOT_OBJECT);               // smoothing.py:203-204
            if (A & X) set_err(p.err, ERR_AVOID_ON_OBJECT);                // smoothing.py:205-206
        }
    });
}

// segment prologue (segmented scheduling, see KParams::nseg): the image's
// bit-plane from xbuf (written by the predecessor segment, possibly on another
// SM: L2 loads, never a stale L1 line), the constraint planes re-packed.  The
// other planes carry no image state between stages (each prep rewrites B, C, D,
// XS, E; the bitmaps are zero between engine calls); `clear` initialises them
// (pads included) when this CTA has not run an image yet.
template <bool HOT>
__device__ __noinline__ void load_state_nl(const View &v, const KParams *pp, size_t pix, int img, bool clear,
                                           bool with_xs) {
    const KParams &p = *pp;
    const Img g = make_img<HOT>(v);
    const int tid = g.tid, nthr = g.nthr;
    if (clear) {
        for (int q = tid; q < g.plen; q += nthr) {
            g.I[q] = 0;
            g.D[q] = 0;
            g.C[q] = 0;
            g.B[q] = ~0u;
        }
        for (int q = tid; q < (g.plen + 31) >> 5; q += nthr) g.dirty[q] = 0;
        for (int q = tid; q < 2 * g.mw; q += nthr) g.claim[q] = 0;
    }
    for (int q = tid; q < (g.plen + 15) >> 4; q += nthr)
        reinterpret_cast<uint4 *>(g.mark)[q] = make_uint4(0, 0, 0, 0);
    if (clear) team_sync(g);
    const size_t wimg = (size_t)g.H * g.WW;
    const uint32_t *src = p.xbuf + (size_t)img * 4 * wimg;
    load_rows(g, src, g.I);
    if (with_xs) load_rows(g, src + wimg, g.XS);
    (void)pix;
    if (p.packed_io) {
        if (p.keep) load_rows(g, reinterpret_cast<const uint32_t *>(p.keep) + (size_t)img * wimg, g.K);
        if (p.avoid) load_rows(g, reinterpret_cast<const uint32_t *>(p.avoid) + (size_t)img * wimg, g.A);
    } else {   // packed by the image's first segment (store_state_nl)
        if (p.keep) load_rows(g, src + 2 * wimg, g.K);
        if (p.avoid) load_rows(g, src + 3 * wimg, g.A);
    }
}

// segment epilogue: the bit-plane to xbuf for the next segment (L2)
template <bool HOT>
__device__ __noinline__ void store_state_nl(const View &v, uint32_t *dst, bool with_xs, bool with_k, bool with_a) {
    const Img g = make_img<HOT>(v);
    const size_t wimg = (size_t)g.H * g.WW;
    // slots: 0 the image, 1 XS, 2 / 3 keep / avoid packed once (first segment)
    // plain stores (L1 is write-through): ordered before the lead's release
    // by the CTA barrier and its __threadfence; planes that may live in L2
    // are read in batches (one latency per batch)
    auto out = [&](const uint32_t *plane, uint32_t *to) {
        walk_strips(g, [&](int x, int y0, int y1, int) {
            constexpr int kB = 16;
            for (int yb = y0; yb < y1; yb += kB) {
                uint32_t w[kB];
#pragma unroll
                for (int j = 0; j < kB; ++j)
                    if (yb + j < y1) w[j] = plane[pidx(g, yb + j, x)];
#pragma unroll
                for (int j = 0; j < kB; ++j)
                    if (yb + j < y1) to[(size_t)(yb + j) * g.WW + x] = w[j];
            }
        });
    };
    out(g.I, dst);
    if (with_xs) out(g.XS, dst + wimg);
    if (with_k) out(g.K, dst + 2 * wimg);
    if (with_a) out(g.A, dst + 3 * wimg);
}

template <bool HOT>
__device__ __noinline__ void store_image_nl(const View &v, uint8_t *out, uint32_t *out_bits) {
    const Img g = make_img<HOT>(v);
    if (out_bits)   // packed output: bit rows, copied back and unpacked by the host
        for_strip(g, [&](int y, int x, int q) { out_bits[(size_t)y * g.WW + x] = g.I[q]; });
    else
        unpack_plane(g.I, out, g);
}

// stages S3 / S7 (stg 1 / 3) read the plane XS saved by the stage before them
__device__ __forceinline__ bool reads_xs(int stg) { return stg == 1 || stg == 3; }

// HOT: one CTA per image, hot planes in shared memory.  !HOT: a team of
// p.team CTAs per image (consecutive blockIdx), planes in the team's slice of
// the global workspace, launched cooperatively when p.team > 1.
template <int FG, bool HOT>
__global__ void __launch_bounds__(kThreads, kMinBlocks) hasf_kernel(const KParams p) {
    extern __shared__ __align__(16) uint32_t smem[];
    __shared__ Shared sh_local;

    const int G = HOT ? 1 : p.team;
    const int team = (int)blockIdx.x / G, rank = (int)blockIdx.x - team * G;
    uint32_t *cta = p.gws + (size_t)(G == 1 ? blockIdx.x : team) * (size_t)p.gws_stride;
    auto buf = [&](int b) -> uint32_t * { return ((p.smem_mask >> b) & 1u) ? smem + p.off[b] : cta + p.off[b]; };
    // teams: a global control block (cooperative launch), or -- when the team
    // is a thread-block cluster -- the control block of the team's rank-0 CTA,
    // shared with the others over distributed shared memory (DSMEM)
    const bool one_cluster = !HOT && G > 1 && p.cluster == G;
    TeamCtl *tc = (G == 1 || one_cluster) ? nullptr : reinterpret_cast<TeamCtl *>(p.tctl) + team;
    Shared *shp = G == 1 ? &sh_local : (one_cluster ? reinterpret_cast<Shared *>(dsmem_map(&sh_local, 0)) : &tc->sh);
    View vl;   // built by every thread, published in shared memory: the noinline
               // phases take it by reference (no per-call copy to local memory)
    if constexpr (HOT) {
        const unsigned long long base = (unsigned long long)__cvta_generic_to_shared(smem);
        vl.I = base + 4ull * p.off[B_I];
        vl.D = base + 4ull * p.off[B_D];
        vl.C = base + 4ull * p.off[B_C];
        vl.dirty = base + 4ull * p.off[B_DIRTY];
        vl.mark = base + 4ull * p.off[B_MARK];
    } else {
        vl.I = (unsigned long long)buf(B_I);
        vl.D = (unsigned long long)buf(B_D);
        vl.C = (unsigned long long)buf(B_C);
        vl.dirty = (unsigned long long)buf(B_DIRTY);
        vl.mark = (unsigned long long)buf(B_MARK);
    }
    vl.B = HOT ? (unsigned long long)__cvta_generic_to_shared(smem) + 4ull * p.off[B_B]
               : (unsigned long long)buf(B_B);
    vl.claim = HOT ? (unsigned long long)__cvta_generic_to_shared(smem) + 4ull * p.off[B_CLAIM]
                   : (unsigned long long)buf(B_CLAIM);
    vl.mw = p.mwords;
    vl.list = buf(B_LIST);
    vl.E = buf(B_E);
    vl.XS = buf(B_XS);
    vl.R = buf(B_R);
    vl.K = buf(B_K);
    vl.A = buf(B_A);
    vl.H = p.H;
    vl.W = p.W;
    vl.WW = p.WW;
    vl.S = p.stride;
    vl.plen = p.plen;
    vl.org = p.pad * p.stride + 1;
    vl.nblk = p.nblk;
    vl.hb = p.hb;
    vl.nstrips = p.nstrips;
    vl.fused = p.fused;
    vl.dense_min = p.dense_min;
    vl.scan_min = p.scan_min;
    vl.scan_first = p.scan_first;
    vl.lastmask = (p.W & 31) ? ((1u << (p.W & 31)) - 1u) : ~0u;
    vl.sh = G == 1 ? (unsigned long long)__cvta_generic_to_shared(&sh_local) : (unsigned long long)shp;
    vl.G = G;
    vl.cs = G > 1 && p.cluster > 1 ? p.cluster : 1;
    vl.rank = rank;
    vl.bar = tc ? tc->bar : nullptr;
    __shared__ unsigned epoch_local;
    vl.epoch = &epoch_local;
    vl.err = p.err;
    __shared__ View v_shared;
    static_assert(sizeof(Shared) + sizeof(View) + 16 <= kStaticSmemReserve, "kStaticSmemReserve too small");
    if (threadIdx.x == 0) {
        v_shared = vl;
        epoch_local = 0;
#ifdef TS_BAR_TRACE
        g_bt = (!HOT && G > 1 && p.cluster <= 1) ? p.trace : nullptr;
        g_bt_cap = p.trace_cap;
        if (g_bt) {   // one extra row: the SM each rank runs on
            unsigned long long smid;
            asm volatile("{ .reg .u32 s; mov.u32 s, %%smid; cvt.u64.u32 %0, s; }" : "=l"(smid));
            g_bt[(g_bt_cap * G + rank) * 2] = (long long)smid;
        }
#endif
    }
    __syncthreads();
    if (one_cluster) {   // rank 0's control block: zeroed, and every CTA of the cluster running
        if (rank == 0 && threadIdx.x == 0) sh_local = Shared{};
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    const View &v = v_shared;
    const Img gk = make_img<HOT>(v);   // team / sync view for this function
    Shared &sh = *shp;
    const bool has_k = p.keep != nullptr, has_a = p.avoid != nullptr;
    const bool lead = gk.tid == 0;

    // stage list of one image: k = (r - r_first) * nst + (stg - first)
    const int first = p.do_cut ? 0 : 2, last = p.do_fill ? 3 : 1;
    const int nst = last - first + 1;
    const int total_stages = p.mode == MODE_HASF ? (p.r_last - p.r_first + 1) * nst : 0;
    const int nseg = p.nseg;
    bool inited = false;   // this CTA's planes initialised (pads) by a first image load
    for (;;) {
        if (lead) sh.img = atomicAdd(p.counter, 1);
        team_sync(gk);
        const int task = *reinterpret_cast<volatile int *>(&sh.img);
        if (task >= p.n * nseg) break;
        const int seg = task / p.n, img = task - seg * p.n;
        unsigned long long tr0 = 0;
        if (p.trace && lead) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr0));
        int k0 = 0, k1 = total_stages;
        if (nseg > 1) seg_range(total_stages, p.seg_stages, p.seg_fine, seg, k0, k1);
        if (seg > 0) {   // segmented: wait until the predecessor segment published the image
            if (lead) {
                const unsigned *f = p.progress + img;
                long long spins = 0;
                unsigned v;
                while (true) {
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
                    if ((int)v >= seg) break;
                    __nanosleep(128);
                    if (++spins > (1LL << 25)) {   // seconds: the predecessor was lost
                        set_err(p.err, ERR_TEAM_TIMEOUT);
                        break;
                    }
                }
            }
            team_sync(gk);
        } else if (p.ready) {   // streamed host entry: wait for the image's input chunk
            if (lead) {
                const unsigned *f = p.ready + img / p.chunk;
                long long spins = 0;
                unsigned v;
                while (true) {
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
                    if (v) break;
                    __nanosleep(256);
                    if (++spins > (1LL << 24)) {   // seconds: the copy never came
                        set_err(p.err, ERR_INPUT_TIMEOUT);
                        break;
                    }
                }
            }
            team_sync(gk);
        }
        const size_t pix = (size_t)img * p.H * p.W;
        if (lead) {
            sh.counters[0] = 0;
            sh.lcount[0] = sh.lcount[1] = sh.lcount[2] = sh.lcount[3] = sh.lcount[4] = sh.lcount[5] = 0;
            sh.flips = 0;
            sh.evals = 0;
            sh.dtime[0] = sh.dtime[1] = sh.dtime[2] = sh.dtime[3] = 0;
            sh.sstat[0] = sh.sstat[1] = sh.sstat[2] = sh.sstat[3] = 0;
            sh.bstat[0] = sh.bstat[1] = sh.bstat[2] = sh.bstat[3] = 0;
            sh.xstat[0] = sh.xstat[1] = sh.xstat[2] = sh.xstat[3] = 0;
            sh.ystat[0] = sh.ystat[1] = sh.ystat[2] = sh.ystat[3] = 0;
            sh.eio = EngineIO{};
        }
        // debug trace: [smid, grabbed, ready, loaded, stages done, stored, end] (%globaltimer ns)
#ifdef TS_BAR_TRACE
        const bool tracing = false;   // the buffer holds the barrier trace
#else
        const bool tracing = p.trace && lead && task < p.trace_cap;
#endif
        auto stamp = [&](int k) {
            if (!tracing) return;
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            p.trace[(size_t)task * kTraceFields + k] = (long long)t;
        };
        if (tracing) {
            unsigned long long smid;
            asm volatile("{ .reg .u32 s; mov.u32 s, %%smid; cvt.u64.u32 %0, s; }" : "=l"(smid));
            p.trace[(size_t)task * kTraceFields + 0] = (long long)smid;
            p.trace[(size_t)task * kTraceFields + 1] = (long long)tr0;
        }
        stamp(2);
        if (seg == 0)
            load_image_nl<HOT>(v, &p, pix, img);
        else
            load_state_nl<HOT>(v, &p, pix, img, !inited, reads_xs(first + k0 % nst));
        inited = true;
        team_sync(gk);
        stamp(3);

        Stats st{};
        st.timing = p.stats != nullptr;
        const long long t_img0 = st.timing ? clock64() : 0;
        int cur = 0;
        int pc = 2;   // worklist pass counter (stamps are its low byte; marks start at 0)
        if (p.mode == MODE_HASF) {
            // stage table: (thin, xmode, save_xs) for S1/S3 (cutting) and S5/S7 (filling)
            for (int k = k0; k < k1; ++k) {
                const int r = p.r_first + k / nst, stg = first + k % nst;
                const bool thin = stg == 0 || stg == 3;
                const int xmode = (stg == 1 || stg == 3) ? 2 : ((stg == 0 ? has_k : has_a) ? 1 : 0);
                const bool save = stg == 0 || stg == 2;
                run_stage<FG, HOT>(v, gk, r, thin, xmode, save, sh, cur, p.err, st, pc);
            }
        } else {
            const int t = p.mode == MODE_THIN ? 1 : 0;
            epass_prio_nl<FG, HOT>(v, p.prio + pix, t, cur);
            team_sync(gk);
            engine<FG, HOT>(v, t, p.max_sweeps, sh, cur, p.err, st, pc);
        }

        stamp(4);
        const bool final_seg = seg == nseg - 1;
        if (final_seg)
            store_image_nl<HOT>(v, p.out + pix,
                                p.packed_io ? reinterpret_cast<uint32_t *>(p.out) + (size_t)img * p.H * p.WW : nullptr);
        else
            store_state_nl<HOT>(v, p.xbuf + (size_t)img * 4 * p.H * p.WW, reads_xs(first + k1 % nst),
                                seg == 0 && has_k && !p.packed_io, seg == 0 && has_a && !p.packed_io);
        stamp(5);
        if (lead && p.stats) {   // accumulated over the image's segments (zeroed buffer)
            unsigned long long *sp = reinterpret_cast<unsigned long long *>(p.stats + (size_t)img * kStatFields);
            const EngineIO eio = *const_cast<const EngineIO *>(&sh.eio);
            auto add = [&](int k, long long x) { atomicAdd(sp + k, (unsigned long long)x); };
            add(0, eio.sweeps);
            add(1, eio.passes);
            add(2, eio.calls);
            add(3, (long long)*reinterpret_cast<volatile unsigned long long *>(&sh.flips));
            add(4, st.cyc_prep);
            add(5, eio.cyc_jacobi);
            add(6, eio.cyc_update);
            add(7, clock64() - t_img0);
            add(8, eio.cyc_tiny);
            add(9, eio.n_tiny);
            add(10, eio.pass_tiny);
            add(11, eio.cyc_dense);
            add(12, eio.n_dense);
            add(13, eio.pass_dense);
            add(14, st.cyc_rank);
            add(15, (long long)*reinterpret_cast<volatile unsigned long long *>(&sh.evals));
            for (int k = 0; k < 4; ++k) {
                add(16 + k, *reinterpret_cast<volatile long long *>(&sh.sstat[k]));
                add(20 + k, *reinterpret_cast<volatile long long *>(&sh.dtime[k]));
                add(24 + k, *reinterpret_cast<volatile long long *>(&sh.bstat[k]));
                add(28 + k, *reinterpret_cast<volatile long long *>(&sh.xstat[k]));
                add(32 + k, *reinterpret_cast<volatile long long *>(&sh.ystat[k]));
            }
        }
        team_sync(gk);
        stamp(6);
        if (!final_seg && lead) {   // image state stored by the whole CTA (barrier above): publish it
            __threadfence();
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p.progress + img), "r"((unsigned)(seg + 1))
                         : "memory");
        }
        if (final_seg && p.done && lead) {   // all the image's output stored: publish it to the copy-out stream
            __threadfence_system();
            atomicAdd(p.done + img / p.chunk, 1u);
        }
    }
    // cluster teams: no CTA leaves while another may still read rank 0's control block
    if (one_cluster)
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// per-variant host entry points, one translation unit each (ts_hasf_<fg><h|g>.cu)
}  // namespace TS_IMPL_NS

// The kernel's dynamic shared-memory limit is a process-wide function
// attribute: it is raised ONCE per device to the opt-in maximum (never changed
// per call, so concurrent host threads planning different images cannot race
// a launch against a smaller limit).
cudaError_t raise_smem_limit_once(const void *fn, std::mutex &mu, bool (&done)[64]);

#define TS_DEFINE_HASF_VARIANT(FG, HOT, SUFFIX)                                                                \
    static std::mutex g_attr_mu_##SUFFIX;                                                                      \
    static bool g_attr_done_##SUFFIX[64];                                                                      \
    cudaError_t launch_hasf_##SUFFIX(const KParams &p, int grid, size_t smem_bytes, cudaStream_t stream) {      \
        using namespace TS_IMPL_NS;                                                                             \
        const void *fn = (const void *)hasf_kernel<FG, HOT>;                                                    \
        cudaError_t e = raise_smem_limit_once(fn, g_attr_mu_##SUFFIX, g_attr_done_##SUFFIX);                   \
        if (e != cudaSuccess) return e;                                                                         \
        void *args[] = {(void *)&p};                                                                            \
        if (p.team > 1 && p.cluster > 1) {   /* clusters of p.cluster CTAs; several per team: cooperative */   \
            cudaLaunchConfig_t cfg{};                                                                           \
            cudaLaunchAttribute at[2];                                                                          \
            at[0].id = cudaLaunchAttributeClusterDimension;                                                     \
            at[0].val.clusterDim.x = (unsigned)p.cluster;                                                       \
            at[0].val.clusterDim.y = 1;                                                                         \
            at[0].val.clusterDim.z = 1;                                                                         \
            at[1].id = cudaLaunchAttributeCooperative;                                                          \
            at[1].val.cooperative = 1;                                                                          \
            cfg.gridDim = dim3(grid);                                                                           \
            cfg.blockDim = dim3(kThreads);                                                                      \
            cfg.dynamicSmemBytes = smem_bytes;                                                                  \
            cfg.stream = stream;                                                                                \
            cfg.attrs = at;                                                                                     \
            cfg.numAttrs = p.cluster < p.team ? 2 : 1;                                                          \
            return cudaLaunchKernelExC(&cfg, fn, args);                                                         \
        }                                                                                                       \
        if (p.team > 1)                                                                                         \
            return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kThreads), args, smem_bytes, stream);      \
        return cudaLaunchKernel(fn, dim3(grid), dim3(kThreads), args, smem_bytes, stream);                     \
    }                                                                                                           \
    cudaError_t clusters_hasf_##SUFFIX(size_t smem_bytes, int team, int *clusters) {                            \
        using namespace TS_IMPL_NS;                                                                             \
        const void *fn = (const void *)hasf_kernel<FG, HOT>;                                                    \
        cudaError_t e = raise_smem_limit_once(fn, g_attr_mu_##SUFFIX, g_attr_done_##SUFFIX);                   \
        if (e != cudaSuccess) return e;                                                                         \
        cudaLaunchConfig_t cfg{};                                                                               \
        cudaLaunchAttribute at[1];                                                                              \
        at[0].id = cudaLaunchAttributeClusterDimension;                                                         \
        at[0].val.clusterDim.x = (unsigned)team;                                                                \
        at[0].val.clusterDim.y = 1;                                                                             \
        at[0].val.clusterDim.z = 1;                                                                             \
        cfg.gridDim = dim3(team * 64);                                                                          \
        cfg.blockDim = dim3(kThreads);                                                                          \
        cfg.dynamicSmemBytes = smem_bytes;                                                                      \
        cfg.attrs = at;                                                                                         \
        cfg.numAttrs = 1;                                                                                       \
        return cudaOccupancyMaxActiveClusters(clusters, fn, &cfg);                                              \
    }                                                                                                           \
    cudaError_t occupancy_hasf_##SUFFIX(size_t smem_bytes, int *blocks) {                                       \
        using namespace TS_IMPL_NS;                                                                             \
        const void *fn = (const void *)hasf_kernel<FG, HOT>;                                                    \
        cudaError_t e = raise_smem_limit_once(fn, g_attr_mu_##SUFFIX, g_attr_done_##SUFFIX);                   \
        if (e != cudaSuccess) return e;                                                                         \
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, fn, kThreads, smem_bytes);                \
    }

}  // namespace ts
