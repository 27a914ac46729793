// C ABI of the B200 HASF path (see include/toposmooth_b200.h).
//
// Host-side responsibilities: argument checks, per-call workspace planning
// (which per-image buffers of the fused kernel live in shared memory and
// which in the CTA's slice of an L2-resident global workspace), launches on
// the caller's stream, and surfacing device-side error flags as status codes
// (nothing is ever returned silently wrong).  No global mutable state besides
// the thread-local error string and the shared-memory budget knob.
#include <cuda_runtime.h>
#include <algorithm>
#include <atomic>
#include <chrono>
#include <mutex>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/toposmooth_b200.h"
#include "ts_common.cuh"
#include "ts_internal.h"
#include "ts_hostpack.h"

namespace ts {
cudaError_t launch_hasf(const KParams &p, int fg, int grid, size_t smem_bytes, cudaStream_t stream);
cudaError_t hasf_occupancy(int fg, bool hot, int threads, size_t smem_bytes, int *blocks_per_sm);
cudaError_t hasf_cluster_occupancy(int fg, int threads, size_t smem_bytes, int team, int *clusters);
cudaError_t launch_edt_phase1(const uint8_t *pix, long long *g, int n, int H, int W, int invert, long long inf,
                              cudaStream_t st);
cudaError_t launch_edt(const uint8_t *pix, const long long *g64, void *out, int *scratch, int n, int H, int W,
                       int invert, long long inf, int out_mode, long long thr, cudaStream_t st);
cudaError_t launch_stage_mask(const long long *dist, const uint8_t *a, const uint8_t *b, uint8_t *out, size_t px,
                              long long thr, int mode, cudaStream_t st);
cudaError_t launch_classify(const uint8_t *pix, uint8_t *out, int n, int H, int W, const uint8_t *lut,
                            cudaStream_t st);
cudaError_t launch_selftest_circuit(uint8_t *out84, uint8_t *out48, cudaStream_t st);
cudaError_t launch_p4_to_rows(const uint8_t *p4, uint32_t *rows, long long nrows, int w, cudaStream_t st);
cudaError_t launch_rows_to_p4(const uint32_t *rows, uint8_t *p4, long long nrows, int w, cudaStream_t st);
cudaError_t launch_p4_to_u8(const uint8_t *p4, uint8_t *out, long long nrows, int w, cudaStream_t st);
cudaError_t launch_u8_to_p4(const uint8_t *in, uint8_t *p4, long long nrows, int w, cudaStream_t st);
cudaError_t launch_ccl(const uint8_t *img, int *parent, long long *counts, int n, int h, int w, int conn,
                       int target, int exterior, cudaStream_t st);
}  // namespace ts

using namespace ts;

namespace {

thread_local std::string g_err;
std::atomic<long long> g_smem_budget{0};

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}
int ok() {
    g_err.clear();
    return TS_OK;
}
int cuda_fail(cudaError_t e, const char *where) {
    return fail(TS_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define TS_CUDA(call)                                   \
    do {                                                \
        cudaError_t e_ = (call);                        \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
    } while (0)

// ---- connectivity tables, restated from their definition -----------------
// T_conn(code) = number of conn-components of the set neighbours of the 3x3
// window's centre that are conn-adjacent to the centre (topo.py:44-84).
const int kOffR[8] = {-1, -1, -1, 0, 0, 1, 1, 1};
const int kOffC[8] = {-1, 0, 1, -1, 1, -1, 0, 1};

int comp_count(int mask, int conn) {
    int parent[8];
    for (int i = 0; i < 8; ++i) parent[i] = i;
    auto find = [&](int a) {
        while (parent[a] != a) a = parent[a] = parent[parent[a]];
        return a;
    };
    auto adjacent = [&](int a, int b) {
        int dr = kOffR[a] - kOffR[b], dc = kOffC[a] - kOffC[b];
        dr = dr < 0 ? -dr : dr;
        dc = dc < 0 ? -dc : dc;
        return conn == 4 ? (dr + dc == 1) : (dr <= 1 && dc <= 1 && (dr | dc));
    };
    for (int a = 0; a < 8; ++a)
        for (int b = a + 1; b < 8; ++b)
            if (((mask >> a) & 1) && ((mask >> b) & 1) && adjacent(a, b)) parent[find(a)] = find(b);
    int roots = 0;   // bitmask of component roots touching the centre
    for (int a = 0; a < 8; ++a) {
        if (!((mask >> a) & 1)) continue;
        const bool touches = conn == 8 || (kOffR[a] == 0 || kOffC[a] == 0);
        if (touches) roots |= 1 << find(a);
    }
    return __builtin_popcount(roots);
}

struct Tables {
    uint8_t t8[256], t4[256], s84[256], s48[256];
    Tables() {
        for (int m = 0; m < 256; ++m) {
            t8[m] = (uint8_t)comp_count(m, 8);
            t4[m] = (uint8_t)comp_count(m, 4);
        }
        for (int m = 0; m < 256; ++m) {
            s84[m] = (t8[m] == 1 && t4[m ^ 0xFF] == 1);
            s48[m] = (t4[m] == 1 && t8[m ^ 0xFF] == 1);
        }
    }
};
const Tables &tables() {
    static const Tables t;
    return t;
}

// ---- fused-kernel planning ------------------------------------------------
struct Plan {
    int WW = 0, nwords = 0, slices = 0;
    int stride = 0, plen = 0, nblk = 1, hb = 1, nstrips = 1, dense_min = 0;
    int pad = kPadRows;
    int mwords = 0;
    bool fused = false;   // fused prep + E-pass (no R planes)
    int per_sm = 0, per_wave = 0;
    size_t smem_bytes = 0;
    uint32_t mask = 0;
    bool hot = false;
    int team = 1, threads = 512;
    long long off[B_COUNT] = {};
    long long stride_ws = 0;   // global workspace words per CTA
};

std::atomic<int> g_fused{1};      // fused prep + E-pass where eligible
std::atomic<long long *> g_trace_buf{nullptr};   // debug task trace (ts_set_trace)
std::atomic<long long> g_trace_cap{0};
// stages per segment of the segmented scheduler (0: whole images); 2 = half a
// radius (one cutting or one filling), the image state between them is one plane
std::atomic<int> g_seg_stages{[] {
    const char *e = getenv("TS_SEG_STAGES");
    return e ? atoi(e) : 8;
}()};
std::atomic<int> g_seg_force{0};   // tests: segment batches of any size
// the streamed host entry's segmentation (env TS_SEG_STAGES_HOST / TS_SEG_FINE_HOST)
std::atomic<int> g_seg_stages_host{[] {
    const char *e = getenv("TS_SEG_STAGES_HOST");
    return e ? atoi(e) : 8;
}()};
std::atomic<int> g_seg_fine_host{[] {
    const char *e = getenv("TS_SEG_FINE_HOST");
    return e ? atoi(e) : 0;
}()};
// the last g_seg_fine stages run as one-stage segments (env TS_SEG_FINE)
std::atomic<int> g_seg_fine{[] {
    const char *e = getenv("TS_SEG_FINE");
    return e ? atoi(e) : 2;
}()};
// The fine tail is tuned per problem unless the caller fixed it (TS_SEG_FINE,
// ts_set_segment_fine, TS_SEG_TUNE=0).  Which tail wins depends on how the
// batch's (segment, image) tasks tile the resident CTAs -- c1 (256 x 512^2 on
// 148 CTAs) runs 1.7% faster with a tail of 1 than of 2, c4 (1024 x 256^2 on
// 296) 3.5% slower -- and no closed form predicted it over the measured
// settings.  The blocking device entry therefore times its own first three
// launches of a problem (tail 2, tail 1, tail 2: the first launch of a process
// also pays one-time costs) and keeps the faster tail for that problem; results
// are identical under every segmentation (tests force every boundary).
std::atomic<int> g_seg_fine_fixed{[] {
    const char *t = getenv("TS_SEG_TUNE");
    return (getenv("TS_SEG_FINE") != nullptr || (t && atoi(t) == 0)) ? 1 : 0;
}()};
thread_local int tl_seg_fine = -1;   // >= 0: the fine tail of this thread's next fused launches
using TuneKey = std::tuple<int, int, long long, int, int, int, int, int, int, int>;
struct TuneState {
    int trials = 0;
    float best[2] = {1e30f, 1e30f};   // candidate 0: tail 2, candidate 1: tail 1
    int choice = -1;
};
constexpr int kTuneFine[2] = {2, 1};
std::mutex g_tune_mu;
std::map<TuneKey, TuneState> g_tune;
std::atomic<int> g_scan_div{[] {
    const char *e = getenv("TS_SCAN_DIV");
    return e ? atoi(e) : -1;
}()};   // global planes: scan passes (< 0: until the fixpoint, 0: off, d: while > threads / d words change)
std::atomic<int> g_dense_div{4};   // measured: 4 beats 2 by ~1.5% on c1, neutral on c4

// strip mapping (thread t -> word column t % WW, row block t / WW) and the
// padded row stride that puts the 32 lanes of every warp on distinct banks
// returns the worst bank multiplicity of a warp's first-row accesses
int plan_strips(int H, int WW, int threads, Plan &pl) {
    if (WW > threads) {
        pl.nblk = 1;
        pl.hb = H;
        pl.stride = WW + 1;
        pl.nstrips = WW;
        return 1;
    }
    int nblk = std::min(threads / WW, H);
    const int hb = (H + nblk - 1) / nblk;
    nblk = (H + hb - 1) / hb;
    pl.nblk = nblk;
    pl.hb = hb;
    const int active = nblk * WW;
    int best_s = WW + 1, best_cost = 1 << 30;
    for (int S = WW + 1; S <= WW + 64; ++S) {
        int cost = 0;
        for (int w0 = 0; w0 < active; w0 += 32) {
            int cnt[32] = {0};
            int worst = 0;
            for (int t = w0; t < std::min(active, w0 + 32); ++t) {
                const long long a = (long long)(t / WW) * hb * S + (t % WW);
                worst = std::max(worst, ++cnt[a & 31]);
            }
            cost = std::max(cost, worst);
        }
        if (cost < best_cost) {
            best_cost = cost;
            best_s = S;
        }
        if (best_cost == 1) break;
    }
    pl.stride = best_s;
    pl.nstrips = nblk * WW;
    return best_cost;
}

// Workspace comes from a PRIVATE stream-ordered memory pool per device whose
// release threshold keeps freed blocks cached across calls (the default
// threshold of 0 would return them to the OS at every synchronize and
// re-map tens of MB per call).  The device's default pool -- shared with
// the rest of the process -- is left untouched.
std::mutex g_pool_mu;
cudaMemPool_t g_pool[64] = {};

cudaError_t ws_malloc(void **ptr, size_t bytes, cudaStream_t st) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    cudaMemPool_t pool;
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        if (!g_pool[dev]) {
            cudaMemPoolProps props{};
            props.allocType = cudaMemAllocationTypePinned;
            props.handleTypes = cudaMemHandleTypeNone;
            props.location.type = cudaMemLocationTypeDevice;
            props.location.id = dev;
            if ((e = cudaMemPoolCreate(&g_pool[dev], &props)) != cudaSuccess) return e;
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(g_pool[dev], cudaMemPoolAttrReleaseThreshold, &thr);
        }
        pool = g_pool[dev];
    }
    return cudaMallocFromPoolAsync(ptr, bytes, pool, st);
}

int device_props(int *sms, int *smem_optin, int *smem_per_sm) {
    int dev = 0;
    TS_CUDA(cudaGetDevice(&dev));
    TS_CUDA(cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, dev));
    TS_CUDA(cudaDeviceGetAttribute(smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    TS_CUDA(cudaDeviceGetAttribute(smem_per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
    return TS_OK;
}

std::atomic<int> g_team_knob{0};   // 0 = automatic team size
std::atomic<int> g_cluster_knob{1};   // teams of 2..8 CTAs as thread-block clusters

// team = CTAs per image (> 1 only with every plane in global memory)
std::atomic<int> g_threads_knob{0};   // 0 = automatic kernel flavour
#ifndef TS_BIG_THREADS
#define TS_BIG_THREADS 512
#endif
constexpr int kBigThreads = TS_BIG_THREADS;   // threads per CTA of the one-CTA-per-SM flavour

// one fixed flavour: `threads` per CTA, `team` CTAs per image, shared-memory
// budget `budget_cap` bytes per CTA (<= 0: device maximum)
int make_plan_fixed(int H, int W, int r_last, int mode, bool has_k, bool has_a, int fg, Plan &pl, int team,
                    int threads, long long budget_cap, bool skip_fused = false, bool e4 = false) {
    if (threads == 256) e4 = true;
#ifdef TS_IMPL_E4_HOT
    e4 = true;
#endif
    pl.WW = (W + 31) / 32;
    if (H >= (1 << 20) || pl.WW >= (1 << 16))
        return fail(TS_ERR_UNSUPPORTED, "image too large for the fused kernel");
    pl.threads = threads;
    // strips: one per thread, or two when that leaves a warp's strips on
    // conflicting banks (e.g. 256 threads on 16-word rows: 32-row blocks)
    if (plan_strips(H, pl.WW, threads * team, pl) > 1 && team == 1 && !getenv("TS_ONE_STRIP")) {
        Plan p2 = pl;
        if (plan_strips(H, pl.WW, 2 * threads, p2) == 1) pl = p2;
    }
    pl.pad = kPadRows;
    const long long plen = (((long long)H + 2 * pl.pad) * pl.stride + 4 + 3) & ~3LL;
    if (plen * 8 >= (long long)INT_MAX)
        return fail(TS_ERR_UNSUPPORTED, "image too large for the fused kernel (padded plane * 8 >= 2^31 words)");
    pl.plen = (int)plen;
    pl.nwords = H * pl.WW;
    pl.dense_min = pl.nwords / std::max(1, g_dense_div.load());
    pl.fused = false;
    pl.slices = (mode == MODE_HASF && r_last >= 1) ? rank_slices(r_last) : 0;
    auto r4 = [](long long x) { return (x + 3) & ~3LL; };
    long long size[B_COUNT];
    size[B_I] = plen;
    size[B_D] = plen;
    size[B_C] = plen;
    size[B_B] = plen;
    size[B_DIRTY] = r4((plen + 31) / 32);
    size[B_CLAIM] = 2 * size[B_DIRTY];
    pl.mwords = (int)size[B_DIRTY];
    size[B_MARK] = r4(((plen + 15) / 16) * 4);
    size[B_LIST] = 2 * plen;   // two compacted re-evaluation lists in dense sweeps
    // E: 8 precedence planes, or 4 (antisymmetry) in the 256-thread and the
    // generic / team variants (ts_hasf_{8,4}{h256,g}.cu define TS_IMPL_E4)
    size[B_E] = (e4 ? 4 : 8) * plen;
    size[B_XS] = mode == MODE_HASF ? plen : 0;
    // the fused prep + E-pass (one strip per thread, rows of <= 32 words that
    // tile a warp, r <= 8) keeps the rank slices in registers: no R planes
    const bool fused = mode == MODE_HASF && team == 1 && pl.nstrips <= threads && 32 % pl.WW == 0 &&
                       r_last <= kFusedMaxR && !skip_fused && g_fused.load();
    size[B_R] = fused ? 0 : (long long)pl.slices * plen;
    pl.fused = fused;
    size[B_K] = (mode == MODE_HASF && has_k) ? plen : 0;
    size[B_A] = (mode == MODE_HASF && has_a) ? plen : 0;

    int sms = 0, optin = 0, per_sm = 0;
    int rc = device_props(&sms, &optin, &per_sm);
    if (rc) return rc;
    long long budget = optin - kStaticSmemReserve;   // static Shared block, View, epoch of the kernel
    if (budget_cap > 0 && budget_cap < budget) budget = budget_cap;
    const long long knob = g_smem_budget.load();
    if (knob > 0 && knob < budget) budget = knob;
    if (team > 1) budget = 0;   // teams share planes through L2
    long long used = 0, gused = 0;
    pl.mask = 0;
    for (int i = 0; i < B_COUNT; ++i) {
        const int b = kPlaceOrder[i];
        if (size[b] == 0) {
            pl.off[b] = 0;
            continue;
        }
        if ((used + size[b]) * 4 <= budget) {
            pl.mask |= 1u << b;
            pl.off[b] = used;
            used += size[b];
        } else {
            pl.off[b] = gused;
            gused += size[b];
        }
    }
    pl.smem_bytes = (size_t)(used * 4);
    pl.stride_ws = gused;
    const uint32_t hot_mask =
        (1u << B_I) | (1u << B_D) | (1u << B_C) | (1u << B_DIRTY) | (1u << B_MARK) | (1u << B_CLAIM) | (1u << B_B);
    pl.hot = (pl.mask & hot_mask) == hot_mask;
    if (fused && !pl.hot)   // the fused path runs only with the hot placement: plan the R planes
        return make_plan_fixed(H, W, r_last, mode, has_k, has_a, fg, pl, team, threads, budget_cap, true, e4);
    if (!pl.hot && !e4)     // the generic variant keeps 4 precedence planes: re-plan with them
        return make_plan_fixed(H, W, r_last, mode, has_k, has_a, fg, pl, team, threads, budget_cap, skip_fused, true);
    pl.team = team;
    int blocks = 0;
    if (threads == 256 && !pl.hot) return fail(TS_ERR_UNSUPPORTED, "256-thread flavour needs the hot placement");
    TS_CUDA(hasf_occupancy(fg, pl.hot, threads, pl.smem_bytes, &blocks));
    if (blocks < 1) return fail(TS_ERR_CUDA, "fused kernel does not fit on an SM");
    pl.per_sm = blocks;
    pl.per_wave = blocks * sms;
    return TS_OK;
}

// chooses the kernel flavour: two 256-thread CTAs per SM when the hot planes
// fit half an SM's shared memory (small images), else one 512-thread CTA
int make_plan(int H, int W, int r_last, int mode, bool has_k, bool has_a, int fg, Plan &pl, int team = 1) {
    const int knob = g_threads_knob.load();
    if (team == 1 && knob != kBigThreads) {
        int sms = 0, optin = 0, per_sm = 0;
        int rc = device_props(&sms, &optin, &per_sm);
        if (rc) return rc;
        Plan p2;
        const long long half = per_sm / 2 - 1024 - kStaticSmemReserve;
        rc = make_plan_fixed(H, W, r_last, mode, has_k, has_a, fg, p2, 1, 256, half);
        // (measured: two images per SM pay off only when each thread walks a
        // single strip; with two strips per thread c1 ran 10% slower)
        if (rc == TS_OK && p2.hot && ((p2.per_sm >= 2 && p2.nstrips <= 256) || knob == 256 || getenv("TS_ONE_STRIP"))) {
            pl = p2;
            return TS_OK;
        }
        if (knob == 256) return rc ? rc : fail(TS_ERR_UNSUPPORTED, "256-thread flavour does not fit");
    }
    // cluster teams (2..8 CTAs, planes in L2) are latency bound: 1024 threads
    // per CTA (64 registers) hide more of it; the cooperative teams of very
    // large images are barrier bound and keep 512
    int threads = kBigThreads;
    if (team >= 2 && ((team <= 8 && g_cluster_knob.load() && knob != kBigThreads) || knob == kWideThreads)) threads = kWideThreads;
    return make_plan_fixed(H, W, r_last, mode, has_k, has_a, fg, pl, team, threads, 0);
}

const char *err_message(int code, int mode) {
    switch (code) {
        case ERR_NOT_BINARY:
        case ERR_CONSTRAINT_NOT_BINARY:
            return "binary image pixels must be 0 or 1";                               // grid.py:60-61
        case ERR_KEEP_NOT_OBJECT:
            return mode == MODE_THIN ? "constraint pixels must be a subset of the object pixels"   // topo.py:265
                                     : "keep-constraint pixels must be object pixels";              // smoothing.py:204
        case ERR_AVOID_ON_OBJECT:
            return "avoid-constraint pixels must be background pixels";                 // smoothing.py:206
        case ERR_KEEP_AVOID:
            return "keep and avoid constraints overlap";                                // smoothing.py:202
        case ERR_ALLOWED_NOT_SUPERSET:
            return "object pixels must be a subset of the allowed set";                 // topo.py:333
        case ERR_JACOBI_CAP:
            return "internal: fixpoint iteration exceeded its bound";
        case ERR_SWEEP_CAP:
            return "internal: engine exceeded its sweep bound";
        case ERR_TEAM_TIMEOUT:
            return "internal: team barrier timed out";
        case ERR_INPUT_TIMEOUT:
            return "internal: streamed input chunk never arrived";
        default:
            return "internal: unknown device error";
    }
}

int check_shape(int64_t n, int32_t h, int32_t w) {
    if (n < 0) return fail(TS_ERR_VALUE, "batch size must be >= 0");
    if (h < 1 || w < 1)
        return fail(TS_ERR_VALUE, "expected a 2D image with positive dimensions, got shape (" + std::to_string(h) +
                                      ", " + std::to_string(w) + ")");
    if (n > INT_MAX) return fail(TS_ERR_UNSUPPORTED, "batch too large");
    return TS_OK;
}

int check_fg(int32_t fg) {
    if (fg != 8 && fg != 4) return fail(TS_ERR_VALUE, "foreground adjacency must be 4 or 8, got " + std::to_string(fg));
    return TS_OK;
}

// Enqueues one fused-kernel launch on `st` (workspace alloc/free stream-ordered);
// device-side errors go to *err_dev (zeroed by the caller).  With team_out
// non-null it receives the team size chosen.
int fused_launch(int mode, const uint8_t *in, uint8_t *out, int64_t n, int32_t h, int32_t w, int r_first, int r_last,
                 int do_cut, int do_fill, int fg, const uint8_t *keep, const uint8_t *avoid, const int64_t *prio,
                 long long max_sweeps, cudaStream_t st, int64_t *stats_host, int *err_dev, int *team_out,
                 const unsigned *ready = nullptr, unsigned *done = nullptr, int chunk = 1, int packed_io = 0) {
    int rc;
    if ((rc = check_shape(n, h, w)) || (rc = check_fg(fg))) return rc;
    if (mode == MODE_HASF && r_last > kMaxR)
        return fail(TS_ERR_UNSUPPORTED, "radius " + std::to_string(r_last) + " exceeds the fused kernel's maximum " +
                                            std::to_string(kMaxR) + " (use the stage path)");
    if (n == 0) return ok();
    Plan pl;
    if ((rc = make_plan(h, w, r_last, mode, keep != nullptr, avoid != nullptr, fg, pl))) return rc;
    // large images (hot planes do not fit one SM) and too few of them to fill
    // the chip: a team of CTAs per image (rows split across the team)
    int team = 1;
    const int knob = g_team_knob.load();
    if (knob > 0) {
        team = knob;
    } else if (!pl.hot && n < pl.per_wave) {
        team = (int)std::min<long long>(pl.per_wave / n, std::max(1, h / 16));
    }
    if (team > 1) {
        Plan pt;
        if ((rc = make_plan(h, w, r_last, mode, keep != nullptr, avoid != nullptr, fg, pt, team))) return rc;
        if (team > pt.per_wave) return fail(TS_ERR_UNSUPPORTED, "team larger than the co-resident CTA count");
        pl = pt;
    }
    // teams of 2..8 CTAs run as thread-block clusters (hardware barriers, the
    // control block in DSMEM); larger teams (c3: one image over every SM) use
    // the cooperative launch with a global barrier
    int cluster = 0;   // cluster size of the launch
    int max_teams = pl.per_wave / team;
    if (team >= 2 && team <= 8 && g_cluster_knob.load()) {
        int nc = 0;
        if (hasf_cluster_occupancy(fg, pl.threads, pl.smem_bytes, team, &nc) == cudaSuccess && nc >= 1) {
            cluster = team;
            max_teams = std::min(max_teams, nc);
        } else {
            cudaGetLastError();
        }
    } else if (team > 8 && g_cluster_knob.load() >= 2 &&
               team * 1LL * std::min<long long>(n, max_teams) <= pl.per_wave) {
        // larger teams (c3: one image over all SMs), opt-in: hierarchical barrier
        // over clusters of 4 (or 2) CTAs when every cluster of the grid fits at
        // once (measured slower on c3 than the flat barrier: 26.6 vs 25.0 ms)
        for (int cs : {4, 2}) {
            if (team % cs) continue;
            const int teams_ = (int)std::min<long long>(n, max_teams);
            int nc = 0;
            if (hasf_cluster_occupancy(fg, pl.threads, pl.smem_bytes, cs, &nc) == cudaSuccess && nc * cs >= teams_ * team) {
                cluster = cs;
                break;
            }
            cudaGetLastError();
        }
    }
    const int teams = (int)std::min<long long>(n, max_teams);
    const int grid = teams * team;
    // segmented scheduling: a batch larger than one wave of single-CTA images
    // is handed out as (segment, image) tasks, so the last wave's idle SMs are
    // bounded by one segment instead of one whole image (KParams::nseg)
    const int nst = (do_cut ? 2 : 0) + (do_fill ? 2 : 0);
    const int total_stages = mode == MODE_HASF ? (r_last - r_first + 1) * nst : 0;
    // segments of seg_stages stages, the last `fine` stages one per segment
    // (the tail when the queue drains is then at most one short stage)
    // (the streamed host entry prefers coarser segments: its copy-back and host
    // unpacking overlap the kernel only while images keep completing)
    const int seg_stages = ready ? g_seg_stages_host.load() : g_seg_stages.load();
    const int fine = std::max(0, ready ? g_seg_fine_host.load() : (tl_seg_fine >= 0 ? tl_seg_fine : g_seg_fine.load()));
    int nseg = 1;
    if (mode == MODE_HASF && team == 1 && seg_stages > 0 && (n > pl.per_wave || g_seg_force.load()) &&
        total_stages > 1)
        nseg = seg_count(total_stages, seg_stages, fine);
    const size_t ws_words = (size_t)pl.stride_ws * (team > 1 ? teams : grid);
    const size_t xbuf_words = nseg > 1 ? (size_t)n * 4 * h * pl.WW : 0;   // image, XS, keep, avoid
    const size_t tctl_bytes = team > 1 && cluster != team ? (size_t)teams * kTeamCtlBytes : 0;
    const size_t stats_bytes = stats_host ? (size_t)n * kStatFields * sizeof(long long) : 0;
    const size_t prog_bytes = nseg > 1 ? (((size_t)n * sizeof(unsigned) + 63) & ~(size_t)63) : 0;
    const size_t ctrl_bytes = 64 + stats_bytes + prog_bytes + tctl_bytes;
    if (team_out) *team_out = team;
    char *ctrl = nullptr;
    uint32_t *gws = nullptr;
    TS_CUDA(ws_malloc((void **)&ctrl, ctrl_bytes, st));
    if (ws_words + xbuf_words) {
        cudaError_t e = ws_malloc((void **)&gws, (ws_words + xbuf_words) * 4, st);
        if (e != cudaSuccess) {
            cudaFreeAsync(ctrl, st);
            return cuda_fail(e, "ws_malloc(workspace)");
        }
    }
    TS_CUDA(cudaMemsetAsync(ctrl, 0, ctrl_bytes, st));
    KParams p{};
    p.in = in;
    p.out = out;
    p.keep = keep;
    p.avoid = avoid;
    p.prio = prio;
    p.n = (int)n;
    p.H = h;
    p.W = w;
    p.WW = pl.WW;
    p.nwords = pl.nwords;
    p.r_first = r_first;
    p.r_last = r_last;
    p.do_cut = do_cut;
    p.do_fill = do_fill;
    p.mode = mode;
    p.max_sweeps = max_sweeps;
    p.slices = pl.slices;
    p.gws = gws;
    p.gws_stride = pl.stride_ws;
    p.stride = pl.stride;
    p.plen = pl.plen;
    p.nblk = pl.nblk;
    p.hb = pl.hb;
    p.nstrips = pl.nstrips;
    p.pad = pl.pad;
    p.mwords = pl.mwords;
    p.dense_min = pl.dense_min;
    {   // global planes: the dense sweeps run as scan passes (scan_pass) -- a scan over the candidate
        // plane, then scans over the stamps until the fixpoint -- and with them a sweep is dense down
        // to 1/12 of the words holding candidates (c2: divisor 6 -> 29.7, 10 -> 29.4, 32 -> 30.1 ms).
        // Environment (A/B): TS_SCAN_DIV = 0 disables them, d > 0 hands over to the claim passes once
        // <= threads / d words change; TS_SCAN_FIRST = 0 keeps the strip walk as the first pass;
        // TS_SCAN_DENSE_DIV sets the divisor; TS_SCAN_SINGLE = 0 excludes single-CTA launches.
        static const int sfirst = getenv("TS_SCAN_FIRST") ? atoi(getenv("TS_SCAN_FIRST")) : 1;
        static const int sdd = getenv("TS_SCAN_DENSE_DIV") ? atoi(getenv("TS_SCAN_DENSE_DIV")) : 12;
        static const int ssingle = getenv("TS_SCAN_SINGLE") ? atoi(getenv("TS_SCAN_SINGLE")) : 1;
        const int div = g_scan_div.load();
        p.scan_min = -1;
        p.scan_first = sfirst;
        if (!pl.hot && (team > 1 || ssingle) && div != 0)
            p.scan_min = div < 0 ? 0 : (int)std::min<long long>(INT_MAX, (long long)pl.threads * team / div);
        if (p.scan_min >= 0) p.dense_min = pl.nwords / std::max(1, sdd);
    }
    p.smem_mask = pl.mask;
    p.hot = pl.hot ? 1 : 0;
    for (int b = 0; b < B_COUNT; ++b) p.off[b] = pl.off[b];
    p.counter = reinterpret_cast<int *>(ctrl);
    p.err = err_dev;
    p.stats = stats_host ? reinterpret_cast<long long *>(ctrl + 64) : nullptr;
    p.team = team;
    p.threads = pl.threads;
    p.tctl = tctl_bytes ? (void *)(ctrl + ctrl_bytes - tctl_bytes) : nullptr;
    p.cluster = cluster;
    p.fused = pl.fused ? 1 : 0;
    p.packed_io = packed_io;
    p.ready = ready;
    p.done = done;
    p.chunk = chunk;
    p.trace = g_trace_buf.load();
    p.trace_cap = g_trace_cap.load();
    p.nseg = nseg;
    p.seg_stages = seg_stages;
    p.seg_fine = fine;
    p.xbuf = nseg > 1 ? gws + ws_words : nullptr;
    p.progress = nseg > 1 ? reinterpret_cast<unsigned *>(ctrl + 64 + stats_bytes) : nullptr;
    cudaError_t le = launch_hasf(p, fg, grid, pl.smem_bytes, st);
    cudaError_t ce = cudaSuccess;
    if (le == cudaSuccess && stats_host)
        ce = cudaMemcpyAsync(stats_host, ctrl + 64, (size_t)n * kStatFields * sizeof(long long), cudaMemcpyDeviceToHost, st);
    if (gws) cudaFreeAsync(gws, st);
    cudaFreeAsync(ctrl, st);
    if (le != cudaSuccess) return cuda_fail(le, "launch hasf_kernel");
    if (ce != cudaSuccess) return cuda_fail(ce, "cudaMemcpyAsync(stats)");
    return TS_OK;
}

int device_error(int herr, int mode) {
    const bool internal = herr == ERR_JACOBI_CAP || herr == ERR_SWEEP_CAP || herr == ERR_TEAM_TIMEOUT ||
                          herr == ERR_INPUT_TIMEOUT;
    return fail(internal ? TS_ERR_INTERNAL : TS_ERR_VALUE, err_message(herr, mode));
}

// runs the fused kernel over a batch; waits for completion and checks the
// device error flag
int run_fused(int mode, const uint8_t *in, uint8_t *out, int64_t n, int32_t h, int32_t w, int r_first, int r_last,
              int do_cut, int do_fill, int fg, const uint8_t *keep, const uint8_t *avoid, const int64_t *prio,
              long long max_sweeps, cudaStream_t st, int64_t *stats_host) {
    if (n <= 0) return fused_launch(mode, in, out, n, h, w, r_first, r_last, do_cut, do_fill, fg, keep, avoid, prio,
                                    max_sweeps, st, stats_host, nullptr, nullptr) ?: ok();
    int *err = nullptr;
    TS_CUDA(ws_malloc((void **)&err, sizeof(int), st));
    cudaError_t me = cudaMemsetAsync(err, 0, sizeof(int), st);
    // fine-tail tuning (see g_seg_fine_fixed): this call is a trial, or uses the problem's choice
    const bool tunable = mode == MODE_HASF && !stats_host && !g_seg_fine_fixed.load();
    const TuneKey key{h, w, (long long)n, r_first, r_last, do_cut, do_fill, fg, keep ? 1 : 0, avoid ? 1 : 0};
    int trial = -1;
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    tl_seg_fine = -1;
    if (tunable) {
        std::lock_guard<std::mutex> lk(g_tune_mu);
        auto it = g_tune.find(key);
        if (it == g_tune.end() && g_tune.size() < 256) it = g_tune.emplace(key, TuneState{}).first;
        if (it != g_tune.end()) {
            TuneState &ts = it->second;
            if (ts.choice >= 0) {
                tl_seg_fine = kTuneFine[ts.choice];
            } else if (cudaEventCreate(&t0) == cudaSuccess && cudaEventCreate(&t1) == cudaSuccess) {
                trial = ts.trials & 1;   // 0, 1, 0
                tl_seg_fine = kTuneFine[trial];
            }
        }
    }
    if (trial >= 0) cudaEventRecord(t0, st);
    int rc = me == cudaSuccess ? fused_launch(mode, in, out, n, h, w, r_first, r_last, do_cut, do_fill, fg, keep,
                                              avoid, prio, max_sweeps, st, stats_host, err, nullptr)
                               : cuda_fail(me, "cudaMemsetAsync");
    if (trial >= 0) cudaEventRecord(t1, st);
    tl_seg_fine = -1;
    int herr = 0;
    cudaError_t ce = cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(err, st);
    cudaError_t se = cudaStreamSynchronize(st);
    if (trial >= 0) {
        float ms = 0.f;
        const bool timed = rc == TS_OK && se == cudaSuccess && cudaEventElapsedTime(&ms, t0, t1) == cudaSuccess;
        std::lock_guard<std::mutex> lk(g_tune_mu);
        auto it = g_tune.find(key);
        if (it != g_tune.end() && it->second.choice < 0) {
            TuneState &ts = it->second;
            if (timed) ts.best[trial] = std::min(ts.best[trial], ms);
            if (++ts.trials >= 3) ts.choice = ts.best[1] < ts.best[0] ? 1 : 0;
        }
    }
    if (t0) cudaEventDestroy(t0);
    if (t1) cudaEventDestroy(t1);
    if (rc) return rc;
    if (ce != cudaSuccess) return cuda_fail(ce, "cudaMemcpyAsync(error flag)");
    if (se != cudaSuccess) return cuda_fail(se, "hasf_kernel");
    if (herr) return device_error(herr, mode);
    return ok();
}

// ---- radii above the fused kernel's kMaxR: one launch sequence per stage ----
// The fused kernel instantiates its clamped bit-parallel EDT for r <= kMaxR.
// Larger radii (the reference accepts any r >= 0, morph.py:18-22) run each
// stage of smoothing.py:107-146 as: exact EDT (int64, border term for the
// thinning priority) -> stage mask (F or V) -> the same engine in its int64-
// priority mode (MODE_THIN / MODE_THICKEN, the homotopic_thin / _thicken
// parity surfaces).  X is updated in place in `x` (device [n,h,w] uint8).
int hasf_stages(uint8_t *x, int64_t n, int32_t h, int32_t w, int r_first, int r_last, int do_cut, int do_fill, int fg,
                const uint8_t *keep, const uint8_t *avoid, cudaStream_t st) {
    if (r_first > r_last) return ok();
    if (h > 32767 || w > 32767) return fail(TS_ERR_UNSUPPORTED, "radius above the fused path needs h, w <= 32767");
    const size_t px = (size_t)n * h * w;
    const long long inf = (long long)h * h + (long long)w * w + 1;
    char *ws = nullptr;
    // dist int64 | EDT scratch 4 x int32 | mask | saved plane | engine output
    TS_CUDA(ws_malloc((void **)&ws, px * (8 + 16 + 3), st));
    long long *dist = reinterpret_cast<long long *>(ws);
    int *scratch = reinterpret_cast<int *>(ws + 8 * px);
    uint8_t *mask = reinterpret_cast<uint8_t *>(ws + 24 * px), *saved = mask + px, *y = saved + px;
    int rc = TS_OK;
    cudaError_t e = cudaSuccess;
    auto edt = [&](const uint8_t *img, int background) {   // background: P = min(EDT(~img), B); else D = EDT(img)
        if (e == cudaSuccess) e = launch_edt(img, nullptr, dist, scratch, (int)n, h, w, background, inf, background, 0, st);
    };
    auto mk = [&](const uint8_t *a, const uint8_t *b, long long thr, int mode) {
        if (e == cudaSuccess) e = launch_stage_mask(dist, a, b, mask, px, thr, mode, st);
    };
    auto engine = [&](int emode, const uint8_t *img) {   // y = FLIP(img), then img <- y
        if (e != cudaSuccess || rc) return;
        rc = run_fused(emode, img, y, n, h, w, 1, 0, 0, 0, fg, mask, nullptr, reinterpret_cast<const int64_t *>(dist),
                       -1, st, nullptr);
        if (!rc) e = cudaMemcpyAsync(const_cast<uint8_t *>(img), y, px, cudaMemcpyDeviceToDevice, st);
    };
    for (int r = r_first; r <= r_last && e == cudaSuccess && rc == TS_OK; ++r) {
        const long long r2 = (long long)r * r;
        if (do_cut) {   // smoothing.py:127-135
            if (e == cudaSuccess) e = cudaMemcpyAsync(saved, x, px, cudaMemcpyDeviceToDevice, st);
            edt(x, 1);
            mk(keep, nullptr, r2, 0);        // F = (P > r^2) | keep
            engine(MODE_THIN, x);            // Y
            edt(x, 0);
            mk(saved, nullptr, r2, 1);       // V = (D <= r^2) & X
            engine(MODE_THICKEN, x);
        }
        if (do_fill) {   // smoothing.py:138-146
            if (e == cudaSuccess) e = cudaMemcpyAsync(saved, x, px, cudaMemcpyDeviceToDevice, st);
            edt(x, 0);
            mk(nullptr, avoid, r2, 2);       // V = (D <= r^2) & ~avoid
            engine(MODE_THICKEN, x);         // Z
            edt(x, 1);
            mk(saved, nullptr, r2, 0);       // F = (P > r^2) | X
            engine(MODE_THIN, x);
        }
    }
    const std::string keep_msg = g_err;
    cudaFreeAsync(ws, st);
    cudaError_t se = cudaStreamSynchronize(st);
    if (rc) {
        g_err = keep_msg;
        return rc;
    }
    if (e != cudaSuccess) return cuda_fail(e, "stage path");
    if (se != cudaSuccess) return cuda_fail(se, "stage path");
    return ok();
}

// HASF over radii r_first..r_last: the fused kernel up to kMaxR, the stage
// path beyond (validation happens in the first launch)
int run_hasf_any(const uint8_t *in, uint8_t *out, int64_t n, int32_t h, int32_t w, int r_first, int r_last, int do_cut,
                 int do_fill, int fg, const uint8_t *keep, const uint8_t *avoid, cudaStream_t st,
                 int64_t *stats_host) {
    if (r_last <= kMaxR)
        return run_fused(MODE_HASF, in, out, n, h, w, r_first, r_last, do_cut, do_fill, fg, keep, avoid, nullptr, -1,
                         st, stats_host);
    int rc;
    if ((rc = check_shape(n, h, w)) || (rc = check_fg(fg))) return rc;
    if (n == 0) return ok();
    // radii up to kMaxR fused (also validates input and constraints); with
    // r_first > kMaxR a zero-radius pass only validates and copies
    const int fl = std::min(r_last, kMaxR);
    rc = run_fused(MODE_HASF, in, out, n, h, w, r_first <= kMaxR ? r_first : 1, r_first <= kMaxR ? fl : 0, do_cut,
                   do_fill, fg, keep, avoid, nullptr, -1, st, stats_host);
    if (rc) return rc;
    return hasf_stages(out, n, h, w, std::max(r_first, kMaxR + 1), r_last, do_cut, do_fill, fg, keep, avoid, st);
}

}  // namespace

extern "C" {

int ts_version(void) { return 100; }

const char *ts_last_error(void) { return g_err.c_str(); }

int ts_max_radius(void) { return kMaxR; }

int64_t ts_set_smem_budget(int64_t bytes) { return g_smem_budget.exchange(bytes < 0 ? 0 : bytes); }

// >= 2: list sweeps then hold at most nwords / 2 words, which the two
// compacted lists (half a plane each) rely on
int32_t ts_set_dense_divisor(int32_t div) { return g_dense_div.exchange(div < 2 ? 2 : div); }

int32_t ts_set_team_size(int32_t ctas) { return g_team_knob.exchange(ctas < 0 ? 0 : ctas); }

int32_t ts_set_cta_threads(int32_t threads) {
    if (threads == 1024) threads = kWideThreads;   // "the wide flavour"
    return g_threads_knob.exchange(threads == 256 || threads == kBigThreads || threads == kWideThreads ? threads : 0);
}

int ts_hasf_plan(int32_t h, int32_t w, int32_t r_max, int32_t has_keep, int32_t has_avoid, int64_t *info5) {
    int rc;
    if ((rc = check_shape(1, h, w))) return rc;
    Plan pl;
    if ((rc = make_plan(h, w, r_max, MODE_HASF, has_keep != 0, has_avoid != 0, 8, pl))) return rc;
    info5[0] = pl.per_wave;
    info5[1] = pl.per_sm;
    info5[2] = (int64_t)pl.smem_bytes;
    info5[3] = pl.mask;
    info5[4] = pl.stride_ws * 4;
    info5[5] = pl.threads;
    return ok();
}

int ts_hasf_batch(const uint8_t *in_dev, uint8_t *out_dev, int64_t n, int32_t h, int32_t w, int32_t r_max,
                  int32_t fg, const uint8_t *keep_dev, const uint8_t *avoid_dev, void *stream,
                  int64_t *stats_host) {
    if (r_max < 0) return fail(TS_ERR_VALUE, "ball radius must be >= 0");   // morph.py:18-22
    return run_hasf_any(in_dev, out_dev, n, h, w, 1, r_max, 1, 1, fg, keep_dev, avoid_dev, (cudaStream_t)stream,
                        stats_host);
}

// Non-blocking variant for callers whose buffers already live on the device:
// everything is stream-ordered, nothing synchronizes; the device error code
// (0 = none) lands in *err_dev in stream order -- read it whenever convenient
// and map it with ts_check_device_error.
int ts_hasf_batch_async(const uint8_t *in_dev, uint8_t *out_dev, int64_t n, int32_t h, int32_t w, int32_t r_max,
                        int32_t fg, const uint8_t *keep_dev, const uint8_t *avoid_dev, void *stream,
                        int32_t *err_dev) {
    if (r_max < 0) return fail(TS_ERR_VALUE, "ball radius must be >= 0");   // morph.py:18-22
    if (!err_dev) return fail(TS_ERR_VALUE, "err_dev is required");
    if (r_max > kMaxR) return fail(TS_ERR_UNSUPPORTED, "the non-blocking entry runs radii <= 16 (fused kernel)");
    cudaStream_t st = (cudaStream_t)stream;
    TS_CUDA(cudaMemsetAsync(err_dev, 0, sizeof(int32_t), st));
    tl_seg_fine = -1;   // the fine tail the blocking entry tuned for this problem, if it has
    if (!g_seg_fine_fixed.load()) {
        std::lock_guard<std::mutex> lk(g_tune_mu);
        auto it = g_tune.find(TuneKey{h, w, (long long)n, 1, r_max, 1, 1, fg, keep_dev ? 1 : 0, avoid_dev ? 1 : 0});
        if (it != g_tune.end() && it->second.choice >= 0) tl_seg_fine = kTuneFine[it->second.choice];
    }
    const int rc = fused_launch(MODE_HASF, in_dev, out_dev, n, h, w, 1, r_max, 1, 1, fg, keep_dev, avoid_dev, nullptr,
                                -1, st, nullptr, reinterpret_cast<int *>(err_dev), nullptr);
    tl_seg_fine = -1;
    return rc ?: ok();
}

int ts_check_device_error(int32_t code) {
    if (code == 0) return ok();
    return device_error(code, MODE_HASF);
}

// ---- streamed host entry ---------------------------------------------------
// One fused launch over the whole batch while the inputs are still arriving:
// the copy-in stream copies chunk k and then writes ready[k] = 1 (a stream
// memory operation, executed in stream order after the copy); CTAs wait for
// their image's chunk flag; each finished image counts itself in done[k]; the
// copy-out stream waits (stream memory operation) until done[k] reaches the
// chunk's size and copies the chunk back.  The GPU therefore fills as soon as
// the first chunk lands and no chunk boundary idles SMs.  The driver entry
// points are resolved at run time (no link-time libcuda dependency).
typedef int (*StreamWriteValue32Fn)(void *, unsigned long long, unsigned int, unsigned int);
typedef int (*StreamWaitValue32Fn)(void *, unsigned long long, unsigned int, unsigned int);
constexpr unsigned kWaitGeq = 0x0;        // CU_STREAM_WAIT_VALUE_GEQ
constexpr unsigned kWriteDefault = 0x0;   // CU_STREAM_WRITE_VALUE_DEFAULT (fence before the write)

struct MemOps {
    StreamWriteValue32Fn write = nullptr;
    StreamWaitValue32Fn wait = nullptr;
};
const MemOps &memops() {
    static const MemOps m = [] {
        MemOps r;
        void *fw = nullptr, *fv = nullptr;
        cudaDriverEntryPointQueryResult q1 = cudaDriverEntryPointSymbolNotFound, q2 = cudaDriverEntryPointSymbolNotFound;
        // the CUDA 12 (v2) memory operations, which need no device opt-in
        if (cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", &fw, 12000, cudaEnableDefault, &q1) ==
                cudaSuccess &&
            cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &fv, 12000, cudaEnableDefault, &q2) ==
                cudaSuccess &&
            q1 == cudaDriverEntryPointSuccess && q2 == cudaDriverEntryPointSuccess) {
            r.write = (StreamWriteValue32Fn)fw;
            r.wait = (StreamWaitValue32Fn)fv;
        }
        return r;
    }();
    return m;
}
std::atomic<int> g_streamed{1};

// uint8 bytes per streamed chunk (TS_CHUNK_BYTES overrides, for measurements)
size_t chunk_bytes() {
    static const size_t b = [] {
        const char *e = getenv("TS_CHUNK_BYTES");
        const long long v = e ? atoll(e) : 0;
        return v > 0 ? (size_t)v : (size_t)(4u << 20);
    }();
    return b;
}

// chunk flag buffers for the streamed entry: plain cudaMalloc allocations
// (stream memory operations target them), recycled, never freed
constexpr int kMaxChunks = 64;
std::mutex g_flag_mu;
std::vector<std::pair<int, unsigned *>> g_flag_free;   // (device, buffer of 2 * kMaxChunks)

unsigned *take_flags(int dev) {
    {
        std::lock_guard<std::mutex> lk(g_flag_mu);
        for (size_t i = 0; i < g_flag_free.size(); ++i)
            if (g_flag_free[i].first == dev) {
                unsigned *b = g_flag_free[i].second;
                g_flag_free.erase(g_flag_free.begin() + (long)i);
                return b;
            }
    }
    unsigned *b = nullptr;
    if (cudaMalloc((void **)&b, 2 * kMaxChunks * sizeof(unsigned)) != cudaSuccess) return nullptr;
    return b;
}
void give_flags(int dev, unsigned *b) {
    std::lock_guard<std::mutex> lk(g_flag_mu);
    g_flag_free.emplace_back(dev, b);
}

int hasf_host_streamed(const uint8_t *in_host, uint8_t *out_host, int64_t n, int32_t h, int32_t w, int32_t r_max,
                       int32_t fg, const uint8_t *keep_host, const uint8_t *avoid_host, cudaStream_t user,
                       const MemOps &mo) {
    const size_t img = (size_t)h * w, bytes = (size_t)n * img;
    // chunks of ~4 MB (16 images at 512^2), at most 64 of them
    int64_t chunk = std::max<int64_t>(1, (int64_t)(chunk_bytes() / std::max<size_t>(img, 1)));
    chunk = std::max<int64_t>(chunk, (n + kMaxChunks - 1) / kMaxChunks);
    const int nchunks = (int)((n + chunk - 1) / chunk);
    const int nbuf = 2 + (keep_host ? 1 : 0) + (avoid_host ? 1 : 0);
    uint8_t *d = nullptr;
    int *err = nullptr;
    unsigned *flags = nullptr;   // ready[nchunks], done[nchunks]
    TS_CUDA(ws_malloc((void **)&d, bytes * nbuf, user));
    TS_CUDA(ws_malloc((void **)&err, sizeof(int), user));
    int dev = 0;
    TS_CUDA(cudaGetDevice(&dev));
    flags = take_flags(dev);
    if (!flags) return fail(TS_ERR_CUDA, "cudaMalloc(chunk flags)");
    TS_CUDA(cudaMemsetAsync(err, 0, sizeof(int), user));
    TS_CUDA(cudaMemsetAsync(flags, 0, 2 * nchunks * sizeof(unsigned), user));
    uint8_t *din = d, *dout = d + bytes;
    uint8_t *dk = keep_host ? d + 2 * bytes : nullptr;
    uint8_t *da = avoid_host ? d + (2 + (keep_host ? 1 : 0)) * bytes : nullptr;
    unsigned *ready = flags, *done = flags + nchunks;
    cudaStream_t sin = nullptr, sout = nullptr, sc = nullptr;
    cudaEvent_t ev0 = nullptr, ec = nullptr, eo = nullptr;
    cudaError_t e = cudaStreamCreateWithFlags(&sin, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&sout, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&sc, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev0, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ec, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&eo, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(ev0, user);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sin, ev0, 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sc, ev0, 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sout, ev0, 0);
    int rc = TS_OK, mrc = 0;
    for (int k = 0; k < nchunks && e == cudaSuccess && mrc == 0; ++k) {
        const int64_t i0 = k * chunk, cnt = std::min<int64_t>(chunk, n - i0);
        const size_t off = (size_t)i0 * img, sz = (size_t)cnt * img;
        e = cudaMemcpyAsync(din + off, in_host + off, sz, cudaMemcpyHostToDevice, sin);
        if (e == cudaSuccess && dk) e = cudaMemcpyAsync(dk + off, keep_host + off, sz, cudaMemcpyHostToDevice, sin);
        if (e == cudaSuccess && da) e = cudaMemcpyAsync(da + off, avoid_host + off, sz, cudaMemcpyHostToDevice, sin);
        if (e == cudaSuccess) mrc = mo.write(sin, (unsigned long long)(uintptr_t)(ready + k), 1u, kWriteDefault);
    }
    if (e == cudaSuccess && mrc == 0)
        rc = fused_launch(MODE_HASF, din, dout, n, h, w, 1, r_max, 1, 1, fg, dk, da, nullptr, -1, sc, nullptr, err,
                          nullptr, ready, done, (int)chunk);
    if (e == cudaSuccess && mrc == 0 && rc == TS_OK) {
        for (int k = 0; k < nchunks && e == cudaSuccess && mrc == 0; ++k) {
            const int64_t i0 = k * chunk, cnt = std::min<int64_t>(chunk, n - i0);
            const size_t off = (size_t)i0 * img, sz = (size_t)cnt * img;
            mrc = mo.wait(sout, (unsigned long long)(uintptr_t)(done + k), (unsigned)cnt, kWaitGeq);
            if (mrc == 0) e = cudaMemcpyAsync(out_host + off, dout + off, sz, cudaMemcpyDeviceToHost, sout);
        }
    }
    cudaEventRecord(ec, sc);
    cudaEventRecord(eo, sout);
    cudaStreamWaitEvent(user, ec, 0);
    cudaStreamWaitEvent(user, eo, 0);
    cudaEventRecord(ev0, sin);   // ev0 reused: the copy-in stream drained too (also on error paths)
    cudaStreamWaitEvent(user, ev0, 0);
    int herr = 0;
    cudaError_t ce = cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, user);
    const std::string keep_msg = g_err;
    cudaFreeAsync(d, user);
    cudaFreeAsync(err, user);
    cudaError_t se = cudaStreamSynchronize(user);
    give_flags(dev, flags);   // idle again once the stream drained
    cudaEventDestroy(ev0);
    cudaEventDestroy(ec);
    cudaEventDestroy(eo);
    cudaStreamDestroy(sin);
    cudaStreamDestroy(sout);
    cudaStreamDestroy(sc);
    if (rc) {
        g_err = keep_msg;
        return rc;
    }
    if (mrc) return fail(TS_ERR_CUDA, "stream memory operation failed (code " + std::to_string(mrc) + ")");
    if (e != cudaSuccess) return cuda_fail(e, "streamed host path");
    if (ce != cudaSuccess) return cuda_fail(ce, "cudaMemcpyAsync(error flag)");
    if (se != cudaSuccess) return cuda_fail(se, "hasf_kernel");
    if (herr) return device_error(herr, MODE_HASF);
    return ok();
}

// Streamed host entry with host-side bit packing (no keep / avoid planes):
// chunk k is packed on the host threads (8x fewer bytes over the link),
// copied, flagged; the fused launch (packed_io) starts after chunk 0; every
// chunk's packed result is copied back when its images are done and unpacked
// on the host while the GPU finishes the later chunks.  Pinned staging
// buffers are cached per process (one streamed call at a time holds them).
std::mutex g_stage_mu;
struct Stage {
    uint32_t *in = nullptr, *out = nullptr;   // in: image, keep, avoid planes (words each)
    size_t words = 0;
} g_stage;

// streams and events of the streamed entry, created once per device (held
// under g_stage_mu for a call; creating them per call cost ~0.1 ms)
struct HostCtx {
    bool made = false;
    cudaStream_t sin = nullptr, sout = nullptr, sc = nullptr;
    cudaEvent_t ev0 = nullptr, ec = nullptr, ein = nullptr;
    cudaEvent_t eo[kMaxChunks] = {};
};
HostCtx g_ctx[64];

int host_ctx(int dev, HostCtx *&c) {
    if (dev < 0 || dev >= 64) return fail(TS_ERR_UNSUPPORTED, "device index >= 64");
    c = &g_ctx[dev];
    if (c->made) return TS_OK;
    TS_CUDA(cudaStreamCreateWithFlags(&c->sin, cudaStreamNonBlocking));
    TS_CUDA(cudaStreamCreateWithFlags(&c->sout, cudaStreamNonBlocking));
    TS_CUDA(cudaStreamCreateWithFlags(&c->sc, cudaStreamNonBlocking));
    TS_CUDA(cudaEventCreateWithFlags(&c->ev0, cudaEventDisableTiming));
    TS_CUDA(cudaEventCreateWithFlags(&c->ec, cudaEventDisableTiming));
    TS_CUDA(cudaEventCreateWithFlags(&c->ein, cudaEventDisableTiming));
    for (int k = 0; k < kMaxChunks; ++k) TS_CUDA(cudaEventCreateWithFlags(&c->eo[k], cudaEventDisableTiming));
    c->made = true;
    return TS_OK;
}

int stage_reserve(size_t words) {
    if (g_stage.words >= words) return TS_OK;
    if (g_stage.in) cudaFreeHost(g_stage.in);
    if (g_stage.out) cudaFreeHost(g_stage.out);
    g_stage = Stage{};
    TS_CUDA(cudaHostAlloc((void **)&g_stage.in, 3 * words * 4, cudaHostAllocDefault));
    TS_CUDA(cudaHostAlloc((void **)&g_stage.out, words * 4, cudaHostAllocDefault));
    g_stage.words = words;
    return TS_OK;
}

int hasf_host_streamed_packed(const uint8_t *in_host, uint8_t *out_host, int64_t n, int32_t h, int32_t w,
                              int32_t r_max, int32_t fg, const uint8_t *keep_host, const uint8_t *avoid_host,
                              cudaStream_t user, const MemOps &mo) {
    const int ww = (w + 31) / 32;
    const size_t img = (size_t)h * w, wimg = (size_t)h * ww, words = (size_t)n * wimg;
    int64_t chunk = std::max<int64_t>(1, (int64_t)(chunk_bytes() / std::max<size_t>(img, 1)));
    chunk = std::max<int64_t>(chunk, (n + kMaxChunks - 1) / kMaxChunks);
    const int nchunks = (int)((n + chunk - 1) / chunk);
    std::lock_guard<std::mutex> lk(g_stage_mu);
    int rc = stage_reserve(words);
    if (rc) return rc;
    uint32_t *hin = g_stage.in, *hout = g_stage.out;
    uint32_t *hk = keep_host ? g_stage.in + g_stage.words : nullptr;
    uint32_t *ha = avoid_host ? g_stage.in + 2 * g_stage.words : nullptr;
    // pack (and validate) chunk k of the image and the constraint planes
    auto pack_chunk = [&](int64_t i0, int64_t cnt) {
        if (!hk && !ha) return pack_images(in_host + i0 * img, hin + i0 * wimg, cnt, h, w, ww);
        const uint8_t *src[3] = {in_host + i0 * img, nullptr, nullptr};   // one parallel region for all planes
        uint32_t *dst[3] = {hin + i0 * wimg, nullptr, nullptr};
        int np = 1;
        if (hk) src[np] = keep_host + i0 * img, dst[np++] = hk + i0 * wimg;
        if (ha) src[np] = avoid_host + i0 * img, dst[np++] = ha + i0 * wimg;
        return pack_planes(src, dst, np, cnt, h, w, ww);
    };
    static const bool htrace = getenv("TS_HOST_TRACE") != nullptr;   // debug: host timeline of the call on stderr
    const auto ht0 = std::chrono::steady_clock::now();
    auto hnow = [&]() { return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - ht0).count(); };
    std::vector<double> tr_send(nchunks, 0.0), tr_back(nchunks, 0.0), tr_unp(nchunks, 0.0);
    // chunk 0 packed (and validated) before anything is enqueued
    if (!pack_chunk(0, std::min<int64_t>(chunk, n)))
        return fail(TS_ERR_VALUE, "binary image pixels must be 0 or 1");   // grid.py:60-61
    int dev = 0;
    TS_CUDA(cudaGetDevice(&dev));
    HostCtx *hc = nullptr;
    if ((rc = host_ctx(dev, hc))) return rc;
    uint32_t *d = nullptr;
    int *err = nullptr;
    TS_CUDA(ws_malloc((void **)&d, words * 4 * 4, user));
    TS_CUDA(ws_malloc((void **)&err, sizeof(int), user));
    TS_CUDA(cudaMemsetAsync(err, 0, sizeof(int), user));
    unsigned *flags = take_flags(dev);
    if (!flags) return fail(TS_ERR_CUDA, "cudaMalloc(chunk flags)");
    TS_CUDA(cudaMemsetAsync(flags, 0, 2 * nchunks * sizeof(unsigned), user));
    uint32_t *din = d, *dout = d + words;
    uint32_t *dk = keep_host ? d + 2 * words : nullptr, *da = avoid_host ? d + 3 * words : nullptr;
    unsigned *ready = flags, *done = flags + nchunks;
    cudaStream_t sin = hc->sin, sout = hc->sout, sc = hc->sc;
    cudaEvent_t ev0 = hc->ev0, ec = hc->ec;
    cudaEvent_t *eo = hc->eo;
    cudaError_t e = cudaEventRecord(ev0, user);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sin, ev0, 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sc, ev0, 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sout, ev0, 0);
    int mrc = 0;
    bool bad = false;
    auto send = [&](int k) {   // chunk k (already packed): copy, then flag
        const int64_t i0 = k * chunk, cnt = std::min<int64_t>(chunk, n - i0);
        if (!bad) e = cudaMemcpyAsync(din + i0 * wimg, hin + i0 * wimg, cnt * wimg * 4, cudaMemcpyHostToDevice, sin);
        if (!bad && dk && e == cudaSuccess)
            e = cudaMemcpyAsync(dk + i0 * wimg, hk + i0 * wimg, cnt * wimg * 4, cudaMemcpyHostToDevice, sin);
        if (!bad && da && e == cudaSuccess)
            e = cudaMemcpyAsync(da + i0 * wimg, ha + i0 * wimg, cnt * wimg * 4, cudaMemcpyHostToDevice, sin);
        if (e == cudaSuccess) mrc = mo.write(sin, (unsigned long long)(uintptr_t)(ready + k), 1u, kWriteDefault);
        if (htrace) tr_send[k] = hnow();
    };
    if (e == cudaSuccess) send(0);
    if (e == cudaSuccess && mrc == 0)
        rc = fused_launch(MODE_HASF, reinterpret_cast<const uint8_t *>(din), reinterpret_cast<uint8_t *>(dout), n, h,
                          w, 1, r_max, 1, 1, fg, reinterpret_cast<const uint8_t *>(dk),
                          reinterpret_cast<const uint8_t *>(da), nullptr, -1, sc, nullptr, err, nullptr, ready, done,
                          (int)chunk, 1);
    const bool launched = e == cudaSuccess && mrc == 0 && rc == TS_OK;
    if (launched) {
        // the rest of the input: pack chunk k while chunk k-1 is on the link
        // (after a bad chunk the flags are still raised so the launch drains).
        // Every send is enqueued before any copy-back wait: were the streams'
        // work funnelled into one hardware queue, a wait ahead of a send
        // would block the copy the kernel is waiting for.
        for (int k = 1; k < nchunks && e == cudaSuccess && mrc == 0; ++k) {
            const int64_t i0 = k * chunk, cnt = std::min<int64_t>(chunk, n - i0);
            if (!bad && !pack_chunk(i0, cnt)) bad = true;
            send(k);
        }
        for (int k = 0; k < nchunks && e == cudaSuccess && mrc == 0; ++k) {
            const int64_t i0 = k * chunk, cnt = std::min<int64_t>(chunk, n - i0);
            mrc = mo.wait(sout, (unsigned long long)(uintptr_t)(done + k), (unsigned)cnt, kWaitGeq);
            if (mrc == 0)
                e = cudaMemcpyAsync(hout + i0 * wimg, dout + i0 * wimg, cnt * wimg * 4, cudaMemcpyDeviceToHost, sout);
            if (e == cudaSuccess) e = cudaEventRecord(eo[k], sout);
        }
        // results: unpack chunk k as soon as its copy-back finished
        for (int k = 0; k < nchunks && e == cudaSuccess && mrc == 0 && !bad; ++k) {
            const int64_t i0 = k * chunk, cnt = std::min<int64_t>(chunk, n - i0);
            e = cudaEventSynchronize(eo[k]);
            if (htrace) tr_back[k] = hnow();
            if (e == cudaSuccess) unpack_images(hout + i0 * wimg, out_host + i0 * img, cnt, h, w, ww);
            if (htrace) tr_unp[k] = hnow();
        }
    }
    // the user stream (which frees the buffers) waits for all three streams,
    // on every exit path -- also the copy-in stream, whose copies may still
    // target the buffers when the launch failed
    cudaEventRecord(ec, sc);
    cudaStreamWaitEvent(user, ec, 0);
    cudaEventRecord(hc->ein, sin);
    cudaStreamWaitEvent(user, hc->ein, 0);
    if (launched) {
        cudaEvent_t el = eo[nchunks - 1];
        if (el) cudaStreamWaitEvent(user, el, 0);
    }
    int herr = 0;
    cudaError_t ce = cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, user);
    const std::string keep_msg = g_err;
    cudaFreeAsync(d, user);
    cudaFreeAsync(err, user);
    cudaError_t se = cudaStreamSynchronize(user);
    give_flags(dev, flags);
    if (htrace) {   // TS_HOST_TRACE: when each chunk was sent, copied back and unpacked (tools/e2e_trace.py)
        fprintf(stderr, "[ts host trace] n=%lld chunks=%d end=%.0f us\n  k: sent / copied back / unpacked (us)\n", (long long)n,
                nchunks, hnow());
        for (int k = 0; k < nchunks; ++k) fprintf(stderr, "  %2d: %6.0f %6.0f %6.0f\n", k, tr_send[k], tr_back[k], tr_unp[k]);
    }
    if (rc) {
        g_err = keep_msg;
        return rc;
    }
    if (mrc) return fail(TS_ERR_CUDA, "stream memory operation failed (code " + std::to_string(mrc) + ")");
    if (e != cudaSuccess) return cuda_fail(e, "streamed host path");
    if (ce != cudaSuccess) return cuda_fail(ce, "cudaMemcpyAsync(error flag)");
    if (se != cudaSuccess) return cuda_fail(se, "hasf_kernel");
    if (bad) return fail(TS_ERR_VALUE, "binary image pixels must be 0 or 1");   // grid.py:60-61
    if (herr) return device_error(herr, MODE_HASF);
    return ok();
}

int32_t ts_set_host_streaming(int32_t on) { return g_streamed.exchange(on < 0 ? 0 : (on > 2 ? 2 : on)); }

int32_t ts_set_fused_prep(int32_t on) { return g_fused.exchange(on ? 1 : 0); }

int32_t ts_set_segment_stages(int32_t stages) { return g_seg_stages.exchange(stages < 0 ? 0 : stages); }

int32_t ts_set_segment_fine(int32_t stages) {
    if (stages < 0) {   // back to per-problem tuning (the stored tail stays the untuned default)
        g_seg_fine_fixed.store(0);
        return g_seg_fine.load();
    }
    g_seg_fine_fixed.store(1);   // the caller's choice: no tuning
    return g_seg_fine.exchange(stages);
}

int32_t ts_set_cluster_teams(int32_t on) { return g_cluster_knob.exchange(on < 0 ? 0 : (on > 2 ? 2 : on)); }

int32_t ts_set_host_segments(int32_t stages, int32_t fine) {
    g_seg_fine_host.store(fine < 0 ? 0 : fine);
    return g_seg_stages_host.exchange(stages < 0 ? 0 : stages);
}

int32_t ts_set_segment_force(int32_t on) { return g_seg_force.exchange(on ? 1 : 0); }

void ts_set_trace(int64_t *trace_dev, int64_t tasks) {
    g_trace_cap.store(trace_dev ? tasks : 0);
    g_trace_buf.store(reinterpret_cast<long long *>(trace_dev));
}

int ts_hasf_batch_host(const uint8_t *in_host, uint8_t *out_host, int64_t n, int32_t h, int32_t w, int32_t r_max,
                       int32_t fg, const uint8_t *keep_host, const uint8_t *avoid_host, void *stream) {
    // Pipelined: the batch is cut into chunks; chunk k's H2D copy (copy-in
    // stream), fused kernel (compute streams, round-robin so a chunk's kernel
    // back-fills SMs freed by the previous one) and D2H copy (copy-out stream)
    // overlap the neighbouring chunks' work.  Page-locked buffers copy
    // asynchronously; pageable ones are staged by the CUDA runtime.
    int rc;
    if ((rc = check_shape(n, h, w)) || (rc = check_fg(fg))) return rc;
    if (r_max < 0) return fail(TS_ERR_VALUE, "ball radius must be >= 0");
    if (n == 0) return ok();
    cudaStream_t user = (cudaStream_t)stream;
    const size_t img = (size_t)h * w, bytes = (size_t)n * img;
    if (r_max > kMaxR) {   // radii above the fused kernel: copy in, the stage path, copy out
        const int nb = 2 + (keep_host ? 1 : 0) + (avoid_host ? 1 : 0);
        uint8_t *d = nullptr;
        TS_CUDA(ws_malloc((void **)&d, bytes * nb, user));
        uint8_t *di = d, *dout = d + bytes, *dk = keep_host ? d + 2 * bytes : nullptr;
        uint8_t *da = avoid_host ? d + (2 + (keep_host ? 1 : 0)) * bytes : nullptr;
        cudaError_t e = cudaMemcpyAsync(di, in_host, bytes, cudaMemcpyHostToDevice, user);
        if (e == cudaSuccess && dk) e = cudaMemcpyAsync(dk, keep_host, bytes, cudaMemcpyHostToDevice, user);
        if (e == cudaSuccess && da) e = cudaMemcpyAsync(da, avoid_host, bytes, cudaMemcpyHostToDevice, user);
        rc = e == cudaSuccess ? run_hasf_any(di, dout, n, h, w, 1, r_max, 1, 1, fg, dk, da, user, nullptr) : TS_OK;
        if (e == cudaSuccess && rc == TS_OK) e = cudaMemcpyAsync(out_host, dout, bytes, cudaMemcpyDeviceToHost, user);
        const std::string keep_msg = g_err;
        cudaFreeAsync(d, user);
        cudaError_t se = cudaStreamSynchronize(user);
        if (rc) {
            g_err = keep_msg;
            return rc;
        }
        if (e != cudaSuccess) return cuda_fail(e, "host entry (stage path)");
        if (se != cudaSuccess) return cuda_fail(se, "host entry (stage path)");
        return ok();
    }
    const bool big = (long long)h * w > 1024LL * 1024;   // team-sized images: one chunk
    const MemOps &mo = memops();
    // the streamed entry needs the copy engine to run while the kernel waits
    // for it: not under a serialising profiler / injection library (ncu,
    // nsys) or CUDA_LAUNCH_BLOCKING, where it would only time out
    static const bool serialised = [] {
        const char *lb = getenv("CUDA_LAUNCH_BLOCKING");
        // fewer hardware queues than the entry's three streams (copy-in,
        // kernel, copy-out) may serialise a copy behind the kernel that waits for it
        const char *mc = getenv("CUDA_DEVICE_MAX_CONNECTIONS");
        const bool few_queues = mc && atoi(mc) > 0 && atoi(mc) < 3;
        return getenv("CUDA_INJECTION64_PATH") != nullptr || getenv("NV_TPS_LAUNCH_TOKEN") != nullptr ||
               getenv("NV_COMPUTE_PROFILER_PERFWORKS_DIR") != nullptr ||
               getenv("NV_NSIGHT_INJECTION_TRANSPORT_TYPE") != nullptr || (lb && lb[0] == '1') || few_queues;
    }();
    // TS_STREAM_BIG=0: team-sized images through the chunked uint8 pipeline below instead
    static const bool stream_big = !(getenv("TS_STREAM_BIG") && atoi(getenv("TS_STREAM_BIG")) == 0);
    if ((!big || (stream_big && g_streamed.load() == 1)) && !serialised && g_streamed.load() && mo.write && mo.wait &&
        r_max <= kMaxR) {
        if (g_streamed.load() == 1)
            return hasf_host_streamed_packed(in_host, out_host, n, h, w, r_max, fg, keep_host, avoid_host, user, mo);
        return hasf_host_streamed(in_host, out_host, n, h, w, r_max, fg, keep_host, avoid_host, user, mo);
    }
    const int nchunks = big ? 1 : (int)std::min<int64_t>(n, 4);
    const int ncs = 3;   // compute streams
    const int64_t per = (n + nchunks - 1) / nchunks;
    uint8_t *d = nullptr;
    int *err = nullptr;
    const int nbuf = 2 + (keep_host ? 1 : 0) + (avoid_host ? 1 : 0);
    TS_CUDA(ws_malloc((void **)&d, bytes * nbuf, user));
    TS_CUDA(ws_malloc((void **)&err, sizeof(int), user));
    TS_CUDA(cudaMemsetAsync(err, 0, sizeof(int), user));
    uint8_t *din = d, *dout = d + bytes;
    uint8_t *dk = keep_host ? d + 2 * bytes : nullptr;
    uint8_t *da = avoid_host ? d + (2 + (keep_host ? 1 : 0)) * bytes : nullptr;
    cudaStream_t sin = nullptr, sout = nullptr, sc[ncs] = {};
    std::vector<cudaEvent_t> evs;
    auto ev = [&]() {
        cudaEvent_t e = nullptr;
        cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        evs.push_back(e);
        return e;
    };
    cudaError_t e = cudaStreamCreateWithFlags(&sin, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&sout, cudaStreamNonBlocking);
    for (int i = 0; i < ncs && e == cudaSuccess; ++i) e = cudaStreamCreateWithFlags(&sc[i], cudaStreamNonBlocking);
    cudaEvent_t ev0 = ev();
    if (e == cudaSuccess) e = cudaEventRecord(ev0, user);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sin, ev0, 0);
    for (int i = 0; i < ncs && e == cudaSuccess; ++i) e = cudaStreamWaitEvent(sc[i], ev0, 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sout, ev0, 0);
    rc = TS_OK;
    for (int k = 0; k < nchunks && e == cudaSuccess && rc == TS_OK; ++k) {
        const int64_t i0 = k * per, cnt = std::min<int64_t>(per, n - i0);
        if (cnt <= 0) break;
        const size_t off = (size_t)i0 * img, sz = (size_t)cnt * img;
        e = cudaMemcpyAsync(din + off, in_host + off, sz, cudaMemcpyHostToDevice, sin);
        if (e == cudaSuccess && dk) e = cudaMemcpyAsync(dk + off, keep_host + off, sz, cudaMemcpyHostToDevice, sin);
        if (e == cudaSuccess && da) e = cudaMemcpyAsync(da + off, avoid_host + off, sz, cudaMemcpyHostToDevice, sin);
        cudaEvent_t ein = ev(), eout = ev();
        cudaStream_t cs = sc[k % ncs];
        if (e == cudaSuccess) e = cudaEventRecord(ein, sin);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, ein, 0);
        if (e != cudaSuccess) break;
        rc = fused_launch(MODE_HASF, din + off, dout + off, cnt, h, w, 1, r_max, 1, 1, fg, dk ? dk + off : nullptr,
                          da ? da + off : nullptr, nullptr, -1, cs, nullptr, err, nullptr);
        if (rc) break;
        e = cudaEventRecord(eout, cs);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(sout, eout, 0);
        if (e == cudaSuccess) e = cudaMemcpyAsync(out_host + off, dout + off, sz, cudaMemcpyDeviceToHost, sout);
    }
    cudaEvent_t edone = ev();
    cudaEventRecord(edone, sout);
    cudaStreamWaitEvent(user, edone, 0);
    int herr = 0;
    cudaError_t ce = cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, user);
    const std::string keep_msg = g_err;
    cudaFreeAsync(d, user);
    cudaFreeAsync(err, user);
    cudaError_t se = cudaStreamSynchronize(user);
    for (cudaEvent_t x : evs) cudaEventDestroy(x);
    cudaStreamDestroy(sin);
    cudaStreamDestroy(sout);
    for (int i = 0; i < ncs; ++i)
        if (sc[i]) cudaStreamDestroy(sc[i]);
    if (rc) {
        g_err = keep_msg;
        return rc;
    }
    if (e != cudaSuccess) return cuda_fail(e, "pipelined host path");
    if (ce != cudaSuccess) return cuda_fail(ce, "cudaMemcpyAsync(error flag)");
    if (se != cudaSuccess) return cuda_fail(se, "hasf_kernel");
    if (herr) return device_error(herr, MODE_HASF);
    return ok();
}

int ts_cutting_batch(const uint8_t *in_dev, uint8_t *out_dev, int64_t n, int32_t h, int32_t w, int32_t r, int32_t fg,
                     const uint8_t *keep_dev, void *stream) {
    if (r < 0) return fail(TS_ERR_VALUE, "ball radius must be >= 0");
    return run_hasf_any(in_dev, out_dev, n, h, w, r == 0 ? 1 : r, r, 1, 0, fg, keep_dev, nullptr,
                        (cudaStream_t)stream, nullptr);
}

int ts_filling_batch(const uint8_t *in_dev, uint8_t *out_dev, int64_t n, int32_t h, int32_t w, int32_t r, int32_t fg,
                     const uint8_t *avoid_dev, void *stream) {
    if (r < 0) return fail(TS_ERR_VALUE, "ball radius must be >= 0");
    return run_hasf_any(in_dev, out_dev, n, h, w, r == 0 ? 1 : r, r, 0, 1, fg, nullptr, avoid_dev,
                        (cudaStream_t)stream, nullptr);
}

int ts_thin_batch(const uint8_t *img_dev, const uint8_t *keep_dev, const int64_t *prio_dev, uint8_t *out_dev,
                  int64_t n, int32_t h, int32_t w, int32_t fg, int64_t max_iter, void *stream) {
    if (!keep_dev || !prio_dev) return fail(TS_ERR_VALUE, "keep and priority are required");
    return run_fused(MODE_THIN, img_dev, out_dev, n, h, w, 1, 0, 0, 0, fg, keep_dev, nullptr, prio_dev,
                     max_iter < 0 ? -1 : max_iter, (cudaStream_t)stream, nullptr);
}

int ts_thicken_batch(const uint8_t *img_dev, const uint8_t *allowed_dev, const int64_t *prio_dev, uint8_t *out_dev,
                     int64_t n, int32_t h, int32_t w, int32_t fg, int64_t max_iter, void *stream) {
    if (!allowed_dev || !prio_dev) return fail(TS_ERR_VALUE, "allowed and priority are required");
    return run_fused(MODE_THICKEN, img_dev, out_dev, n, h, w, 1, 0, 0, 0, fg, allowed_dev, nullptr, prio_dev,
                     max_iter < 0 ? -1 : max_iter, (cudaStream_t)stream, nullptr);
}

static int run_edt(const uint8_t *in, const int64_t *g_in, void *out, int64_t n, int32_t h, int32_t w, int invert,
                   int out_mode, long long thr, bool phase1_only, cudaStream_t st) {
    int rc;
    if ((rc = check_shape(n, h, w))) return rc;
    if (h > 32767 || w > 32767) return fail(TS_ERR_UNSUPPORTED, "exact EDT supports h, w <= 32767");
    if (n == 0) return ok();
    const long long inf = (long long)h * h + (long long)w * w + 1;   // edt.py:25-28
    const size_t px = (size_t)n * h * w;
    if (phase1_only) {
        TS_CUDA(launch_edt_phase1(in, reinterpret_cast<long long *>(out), (int)n, h, w, invert, inf, st));
        TS_CUDA(cudaStreamSynchronize(st));
        return ok();
    }
    int *scratch = nullptr;
    TS_CUDA(ws_malloc((void **)&scratch, sizeof(int) * px * 4, st));
    cudaError_t e = launch_edt(in, reinterpret_cast<const long long *>(g_in), out, scratch, (int)n, h, w, invert, inf,
                               out_mode, thr, st);
    cudaFreeAsync(scratch, st);
    cudaError_t se = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "edt launch");
    if (se != cudaSuccess) return cuda_fail(se, "edt kernels");
    return ok();
}

int ts_edt_sq_batch(const uint8_t *in_dev, int64_t *out_dev, int64_t n, int32_t h, int32_t w, int32_t mode,
                    void *stream) {
    if (mode != 0 && mode != 1) return fail(TS_ERR_VALUE, "mode must be 0 (object) or 1 (background)");
    return run_edt(in_dev, nullptr, out_dev, n, h, w, mode, mode, 0, false, (cudaStream_t)stream);
}

int ts_edt_phase1_batch(const uint8_t *in_dev, int64_t *g_dev, int64_t n, int32_t h, int32_t w, void *stream) {
    return run_edt(in_dev, nullptr, g_dev, n, h, w, 0, 0, 0, true, (cudaStream_t)stream);
}

int ts_edt_phase2_batch(const int64_t *g_dev, int64_t *out_dev, int64_t n, int32_t h, int32_t w, void *stream) {
    return run_edt(nullptr, g_dev, out_dev, n, h, w, 0, 0, 0, false, (cudaStream_t)stream);
}

int ts_dilate_batch(const uint8_t *in_dev, uint8_t *out_dev, int64_t n, int32_t h, int32_t w, int32_t r,
                    void *stream) {
    if (r < 0) return fail(TS_ERR_VALUE, "ball radius must be >= 0");
    return run_edt(in_dev, nullptr, out_dev, n, h, w, 0, 2, (long long)r * r, false, (cudaStream_t)stream);
}

int ts_erode_batch(const uint8_t *in_dev, uint8_t *out_dev, int64_t n, int32_t h, int32_t w, int32_t r,
                   void *stream) {
    if (r < 0) return fail(TS_ERR_VALUE, "ball radius must be >= 0");
    return run_edt(in_dev, nullptr, out_dev, n, h, w, 1, 3, (long long)r * r, false, (cudaStream_t)stream);
}

int ts_neighborhood_codes_batch(const uint8_t *in_dev, uint8_t *out_dev, int64_t n, int32_t h, int32_t w,
                                void *stream) {
    int rc;
    if ((rc = check_shape(n, h, w))) return rc;
    if (n == 0) return ok();
    cudaStream_t st = (cudaStream_t)stream;
    TS_CUDA(launch_classify(in_dev, out_dev, (int)n, h, w, nullptr, st));
    TS_CUDA(cudaStreamSynchronize(st));
    return ok();
}

int ts_simple_point_mask_batch(const uint8_t *in_dev, uint8_t *out_dev, int64_t n, int32_t h, int32_t w, int32_t fg,
                               void *stream) {
    int rc;
    if ((rc = check_shape(n, h, w)) || (rc = check_fg(fg))) return rc;
    if (n == 0) return ok();
    cudaStream_t st = (cudaStream_t)stream;
    uint8_t *dlut = nullptr;
    TS_CUDA(ws_malloc((void **)&dlut, 256, st));
    const uint8_t *src = fg == 8 ? tables().s84 : tables().s48;
    cudaError_t e = cudaMemcpyAsync(dlut, src, 256, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = launch_classify(in_dev, out_dev, (int)n, h, w, dlut, st);
    cudaFreeAsync(dlut, st);
    cudaError_t se = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "simple_point_mask");
    if (se != cudaSuccess) return cuda_fail(se, "simple_point_mask");
    return ok();
}

int ts_component_counts_batch(const uint8_t *in_dev, int64_t *counts_host, int64_t n, int32_t h, int32_t w,
                              int32_t conn, int32_t foreground, int32_t exterior, void *stream) {
    int rc;
    if ((rc = check_shape(n, h, w))) return rc;
    if (conn != 4 && conn != 8) return fail(TS_ERR_VALUE, "adjacency must be 4 or 8, got " + std::to_string(conn));
    if ((long long)h * w + 1 >= (long long)INT_MAX) return fail(TS_ERR_UNSUPPORTED, "image too large for int32 labels");
    if (n == 0) return ok();
    cudaStream_t st = (cudaStream_t)stream;
    int *parent = nullptr;
    long long *cnt = nullptr;
    TS_CUDA(ws_malloc((void **)&parent, sizeof(int) * (size_t)n * ((size_t)h * w + 1), st));
    TS_CUDA(ws_malloc((void **)&cnt, sizeof(long long) * (size_t)n, st));
    cudaError_t e = cudaMemsetAsync(cnt, 0, sizeof(long long) * (size_t)n, st);
    if (e == cudaSuccess)
        e = launch_ccl(in_dev, parent, cnt, (int)n, h, w, conn, foreground ? 1 : 0, exterior ? 1 : 0, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(counts_host, cnt, sizeof(long long) * (size_t)n, cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(parent, st);
    cudaFreeAsync(cnt, st);
    cudaError_t se = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "component counts");
    if (se != cudaSuccess) return cuda_fail(se, "component counts");
    return ok();
}

// ---- netpbm P4 straight into the device bit-row layout (row f2) --------------
int ts_p4_to_rows(const uint8_t *p4_dev, uint32_t *rows_dev, int64_t n, int32_t h, int32_t w, void *stream) {
    int rc;
    if ((rc = check_shape(n, h, w))) return rc;
    if (n == 0) return ok();
    cudaStream_t st = (cudaStream_t)stream;
    TS_CUDA(launch_p4_to_rows(p4_dev, rows_dev, n * h, w, st));
    TS_CUDA(cudaStreamSynchronize(st));
    return ok();
}

int ts_rows_to_p4(const uint32_t *rows_dev, uint8_t *p4_dev, int64_t n, int32_t h, int32_t w, void *stream) {
    int rc;
    if ((rc = check_shape(n, h, w))) return rc;
    if (n == 0) return ok();
    cudaStream_t st = (cudaStream_t)stream;
    TS_CUDA(launch_rows_to_p4(rows_dev, p4_dev, n * h, w, st));
    TS_CUDA(cudaStreamSynchronize(st));
    return ok();
}

int ts_hasf_batch_p4(const uint8_t *p4_in_dev, uint8_t *p4_out_dev, int64_t n, int32_t h, int32_t w, int32_t r_max,
                     int32_t fg, const uint8_t *keep_p4_dev, const uint8_t *avoid_p4_dev, void *stream) {
    int rc;
    if ((rc = check_shape(n, h, w)) || (rc = check_fg(fg))) return rc;
    if (r_max < 0) return fail(TS_ERR_VALUE, "ball radius must be >= 0");   // morph.py:18-22
    if (n == 0) return ok();
    cudaStream_t st = (cudaStream_t)stream;
    if (r_max > kMaxR) {   // stage path (bytes): P4 -> uint8 planes -> HASF -> P4
        const size_t px = (size_t)n * h * w;
        uint8_t *b = nullptr;
        TS_CUDA(ws_malloc((void **)&b, px * 4, st));
        uint8_t *bi = b, *bo = b + px, *bk = keep_p4_dev ? b + 2 * px : nullptr, *ba = avoid_p4_dev ? b + 3 * px : nullptr;
        cudaError_t e = launch_p4_to_u8(p4_in_dev, bi, n * h, w, st);
        if (e == cudaSuccess && bk) e = launch_p4_to_u8(keep_p4_dev, bk, n * h, w, st);
        if (e == cudaSuccess && ba) e = launch_p4_to_u8(avoid_p4_dev, ba, n * h, w, st);
        rc = e == cudaSuccess ? run_hasf_any(bi, bo, n, h, w, 1, r_max, 1, 1, fg, bk, ba, st, nullptr) : TS_OK;
        if (e == cudaSuccess && rc == TS_OK) e = launch_u8_to_p4(bo, p4_out_dev, n * h, w, st);
        const std::string keep_msg = g_err;
        cudaFreeAsync(b, st);
        cudaError_t se = cudaStreamSynchronize(st);
        if (rc) {
            g_err = keep_msg;
            return rc;
        }
        if (e != cudaSuccess) return cuda_fail(e, "P4 path");
        if (se != cudaSuccess) return cuda_fail(se, "P4 path");
        return ok();
    }
    const int ww = (w + 31) / 32;
    const size_t words = (size_t)n * h * ww;
    char *ws = nullptr;
    TS_CUDA(ws_malloc((void **)&ws, 4 * words * 4 + 64, st));
    uint32_t *rin = reinterpret_cast<uint32_t *>(ws), *rout = rin + words, *rk = rout + words, *ra = rk + words;
    int *err = reinterpret_cast<int *>(ra + words);
    cudaError_t e = cudaMemsetAsync(err, 0, sizeof(int), st);
    if (e == cudaSuccess) e = launch_p4_to_rows(p4_in_dev, rin, n * h, w, st);
    if (e == cudaSuccess && keep_p4_dev) e = launch_p4_to_rows(keep_p4_dev, rk, n * h, w, st);
    if (e == cudaSuccess && avoid_p4_dev) e = launch_p4_to_rows(avoid_p4_dev, ra, n * h, w, st);
    rc = TS_OK;
    if (e == cudaSuccess)   // packed_io: image and constraints as bit rows
        rc = fused_launch(MODE_HASF, reinterpret_cast<const uint8_t *>(rin), reinterpret_cast<uint8_t *>(rout), n, h, w,
                          1, r_max, 1, 1, fg, keep_p4_dev ? reinterpret_cast<const uint8_t *>(rk) : nullptr,
                          avoid_p4_dev ? reinterpret_cast<const uint8_t *>(ra) : nullptr, nullptr, -1, st, nullptr, err,
                          nullptr, nullptr, nullptr, 1, 1);
    if (e == cudaSuccess && rc == TS_OK) e = launch_rows_to_p4(rout, p4_out_dev, n * h, w, st);
    int herr = 0;
    cudaError_t ce = cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, st);
    const std::string keep_msg = g_err;
    cudaFreeAsync(ws, st);
    cudaError_t se = cudaStreamSynchronize(st);
    if (rc) {
        g_err = keep_msg;
        return rc;
    }
    if (e != cudaSuccess) return cuda_fail(e, "P4 path");
    if (ce != cudaSuccess) return cuda_fail(ce, "cudaMemcpyAsync(error flag)");
    if (se != cudaSuccess) return cuda_fail(se, "hasf_kernel");
    if (herr) return device_error(herr, MODE_HASF);
    return ok();
}

int ts_connectivity_tables(uint8_t *t8, uint8_t *t4, uint8_t *s84, uint8_t *s48) {
    const Tables &t = tables();
    if (t8) std::memcpy(t8, t.t8, 256);
    if (t4) std::memcpy(t4, t.t4, 256);
    if (s84) std::memcpy(s84, t.s84, 256);
    if (s48) std::memcpy(s48, t.s48, 256);
    return ok();
}

int ts_selftest_circuit(uint8_t *s84, uint8_t *s48) {
    uint8_t *d = nullptr;
    TS_CUDA(cudaMalloc((void **)&d, 512));
    cudaError_t e = launch_selftest_circuit(d, d + 256, 0);
    if (e == cudaSuccess) e = cudaMemcpy(s84, d, 256, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(s48, d + 256, 256, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return cuda_fail(e, "selftest_circuit");
    return ok();
}

}  // extern "C"
