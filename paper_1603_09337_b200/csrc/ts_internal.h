// Host/device shared parameter blocks (internal; not part of the C ABI).
#pragma once
#include <cstdint>

// threads per CTA of the "wide" flavour of the global-plane kernel (cluster
// teams of large images; ts_hasf_{8,4}g1024.cu).  Measured on c2 (32 x 2048^2,
// teams of 4): 512 threads (128 registers) 37.2 ms, 768 (80) 35.1 ms, 1024 (64,
// spill-bound strip walk) 38.3 ms.
#ifndef TS_WIDE_THREADS
#define TS_WIDE_THREADS 768
#endif
namespace ts {
constexpr int kWideThreads = TS_WIDE_THREADS;

// Per-image working buffers of the fused HASF kernel.  Each lives either in
// the CTA's shared memory or in its private slice of a global workspace
// (L2-resident); the host places them greedily in kPlaceOrder.
// All planes use the padded layout: `pad` zero rows above and below the image
// (reads beyond them are clamped to the pad row), one zero word between rows
// (row stride `stride` >= WW + 1); word (y, x) is at (pad + y) * stride + x + 1;
// plane length `plen` words.
constexpr int kPadRows = 1;

// largest radius of the fused prep + E-pass (rank slices kept in registers)
constexpr int kFusedMaxR = 8;

// threads per CTA of the fused kernel (host planning must agree)
#ifndef TS_THREADS
#define TS_THREADS 512
#endif
constexpr int kHasfThreads = TS_THREADS;

// most segments per image of the segmented scheduler (4 stages per radius, r <= 16)
constexpr int kMaxSegs = 64;

// debug task trace: SM id, then %globaltimer ns when the task was taken, its
// input ready, loaded, its stages done, its result stored, finished
constexpr int kTraceFields = 7;

// static shared memory of the fused kernel (control block, View, barrier
// epoch) that the host planner leaves out of the dynamic budget
constexpr int kStaticSmemReserve = 768;

// bytes reserved per team control block (teams of > 1 CTA per image)
constexpr int kTeamCtlBytes = 8192;

enum Buf : int {
    B_I = 0,     // current image, bit-packed                          plen
    B_D,         // fixpoint decisions of the current sweep            plen
    B_C,         // candidates of the current sweep                    plen
    B_B,         // blocked (floor) plane; pads blocked                plen
    B_DIRTY,     // "re-examine" bitmap, 1 bit per word                plen / 32
    B_MARK,      // per-word pass stamps of the fixpoint worklist      plen bytes
    B_LIST,      // active-word list (padded word indices)             plen
    B_E,         // 8 "earlier neighbour" masks per word, interleaved  8 * plen
    B_XS,        // saved image (cutting input X / filling input X')   plen
    B_R,         // rank bit-slices of the clamped distance map        S * plen
    B_K,         // keep constraint plane (optional)                   plen
    B_A,         // avoid constraint plane (optional)                  plen
    B_CLAIM,     // 2 claim bitmaps of the compacted passes             2 * plen / 32
    B_COUNT
};

// shared-memory placement priority: the planes every fixpoint evaluation reads
// with neighbours (I, D), the candidates, the bitmaps; then the rest
constexpr int kPlaceOrder[B_COUNT] = {B_I, B_D, B_C, B_DIRTY, B_MARK, B_CLAIM, B_B, B_LIST, B_XS, B_E, B_R, B_K, B_A};

// per-image stats: 0 sweeps, 1 fixpoint passes, 2 engine calls, 3 flips, then
// thread-0 clock64 cycles: 4 prep (EDT/rank + E passes), 5 fixpoint passes,
// 6 apply+rebuild, 7 whole image (incl. pack/unpack); 8-10 cycles / sweeps /
// passes of tiny sweeps (<= 32 words), 11-13 the same for dense sweeps
// (> one word per thread), 14 cycles of the clamped-EDT part of prep
// 16-19 list sweeps of 33..512 words: count, cycles (incl. re-examination),
// of > 512 words: count, cycles; 20-23 dense sweeps: cycles of the strip-walk pass, of the list collection
// (incl. barriers), of the compacted passes; listed words; 24-27 list sweeps
// of > 512 words: list-build, sweep, re-examination cycles, list builds;
// 28-29 tiny regimes: cycles (incl. list build and barriers), count; 30 whole
// engine calls, 31 whole stages (cycles); 32-35 engine prologue, loop tops,
// epilogue cycles, sweep-loop iterations
constexpr int kStatFields = 36;

enum Mode : int { MODE_HASF = 0, MODE_THIN = 1, MODE_THICKEN = 2 };

enum Err : int {
    ERR_NONE = 0,
    ERR_NOT_BINARY = 1,        // input pixel not in {0,1}
    ERR_JACOBI_CAP = 2,        // fixpoint iteration exceeded its proven bound
    ERR_SWEEP_CAP = 3,         // engine exceeded its proven sweep bound
    ERR_KEEP_NOT_OBJECT = 4,   // keep constraint outside the object
    ERR_AVOID_ON_OBJECT = 5,   // avoid constraint on object pixels
    ERR_KEEP_AVOID = 6,        // keep and avoid overlap
    ERR_CONSTRAINT_NOT_BINARY = 7,
    ERR_ALLOWED_NOT_SUPERSET = 8,  // thicken: object outside allowed
    ERR_TEAM_TIMEOUT = 9,      // a team barrier did not complete (CTA not co-resident)
    ERR_INPUT_TIMEOUT = 10,    // streamed host entry: an input chunk never arrived
};

struct KParams {
    const uint8_t *in;
    uint8_t *out;
    const uint8_t *keep;    // [n,h,w] or null  (MODE_THIN: keep; MODE_THICKEN: allowed)
    const uint8_t *avoid;   // [n,h,w] or null
    const int64_t *prio;    // [n,h,w] (engine modes only)
    int n, H, W, WW, nwords;
    int stride, plen;       // padded layout (see kPadRows)
    int pad;                // zero rows above / below the image (kPadRows)
    int mwords;             // words of one 1-bit-per-word bitmap (dirty, each claim bitmap)
    int nstrips;            // strips = nblk * WW (a thread walks strips tid, tid + nthr, ...)
    int nblk, hb;           // strip mapping: row blocks per word column, rows per block
    int dense_min;          // sweeps with more listed words run in dense (strip) mode
    int scan_min;           // global planes: scan passes while more words than this change per pass (< 0: off)
    int scan_first;         // dense sweeps start with a scan over the candidate plane instead of the strip walk
    int team;               // CTAs per image (1, or > 1 for the generic variant; cooperative launch)
    int threads;            // threads per CTA of the variant (512, or 256 = two CTAs per SM)
    void *tctl;             // team control blocks, kTeamCtlBytes each, zeroed (team > 1, not a cluster)
    int cluster;            // thread-block cluster size of the launch (0/1 none); == team: each team is one
                            // cluster (control block in rank 0's smem, cluster barriers); < team: hierarchical
                            // team barrier (cluster barrier + one global arrival per cluster)
    int r_first, r_last, do_cut, do_fill;
    int mode;
    long long max_sweeps;   // < 0: unbounded
    int slices;             // rank slices allocated (for r_last)
    uint32_t *gws;          // global workspace, gws_stride words per CTA
    long long gws_stride;
    uint32_t smem_mask;     // bit b set: buffer b lives in shared memory
    int hot;                // I, D, C, B, DIRTY, MARK, CLAIM all in shared memory (fast variant)
    long long off[B_COUNT]; // word offset of each buffer (smem or CTA slice)
    int *counter;           // image queue head
    // streamed host entry (or null): image i waits for ready[i / chunk] != 0
    // (written by the copy-in stream after the chunk's H2D copy) and, once
    // stored, counts itself in done[i / chunk] (awaited by the copy-out stream)
    const unsigned *ready;
    unsigned *done;
    int chunk;
    int fused;              // 1: fused prep + E-pass allowed (the planner left out the R planes)
    int packed_io;          // 1: in / out (and keep / avoid) are [n][H][WW] uint32 bit rows (binary by construction)
    // segmented scheduling (batches larger than one wave, single-CTA images):
    // an image's stage list is cut into nseg segments (see seg_range);
    // the queue hands out (segment, image) tasks segment-major, the image's
    // bit-plane passes between segments through xbuf ([n][H][WW] words), and
    // progress[i] counts image i's completed segments (a task waits for its
    // predecessor).  nseg == 1: whole images.
    int nseg;
    int seg_stages, seg_fine;   // segments of seg_stages stages, the last seg_fine stages one each
    uint32_t *xbuf;         // [n][4][H][WW]: the image, XS when the next stage reads it, keep, avoid
    unsigned *progress;
    long long *trace;       // debug: per task kTraceFields int64 (see hasf_kernel) or null
    long long trace_cap;    // tasks recorded
    int *err;               // first error code (atomicCAS from 0)
    long long *stats;       // [n][kStatFields] (or null), see kStatFields
};

}  // namespace ts
