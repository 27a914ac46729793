/*
 * toposmooth_b200 -- C ABI of the B200-native HASF path (sm_100a).
 *
 * Drop-in boundary for the reference's public Python API (toposmooth, which
 * has no native FFI of its own: its kernels are numba functions taking numpy
 * arrays by reference and writing preallocated outputs, e.g.
 * _phase1_kernel(pix, g, cols, inf, invert), edt.py:46).  Each entry point
 * below names the reference function it replaces
 * (paths relative to /root/reference/pkg/src/toposmooth/).
 *
 * Conventions
 *  - Images are uint8 {0,1}, row-major [n][h][w] batches of independent
 *    images (the reference handles one 2-D image per call; n = 1 is that).
 *  - "_dev" pointers are CUDA device pointers owned by the caller; nothing is
 *    retained after return.  "_host" entry points take host pointers and do
 *    the host<->device copies inside the call.
 *  - stream: a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Every call is stream-ordered and returns after the stream has drained
 *    the call's work (errors are device-checked before returning).
 *  - fg: foreground adjacency, 8 -> the (8,4) pair (ADJ_84), 4 -> (4,8)
 *    (ADJ_48), grid.py:22-45.
 *  - Return value: TS_OK or an error class; ts_last_error() gives the
 *    message (thread-local).  TS_ERR_VALUE corresponds to the reference's
 *    ValueError conditions (same messages).
 */
#ifndef TOPOSMOOTH_B200_H
#define TOPOSMOOTH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TS_OK 0
#define TS_ERR_VALUE 1        /* invalid argument / input (reference ValueError) */
#define TS_ERR_CUDA 2         /* CUDA runtime failure */
#define TS_ERR_INTERNAL 3     /* device-side invariant violated (never silently truncates) */
#define TS_ERR_UNSUPPORTED 4  /* outside the device path's limits (e.g. h, w > 32767 for r > 16) */

/* Library version, e.g. 100 for 0.1.0. */
int ts_version(void);

/* Message of the last failing call on this thread ("" if none). */
const char *ts_last_error(void);

/* Largest radius the fused single-launch HASF kernel is instantiated for
 * (16).  Every radius is supported: above it, each stage runs as exact EDT ->
 * stage mask -> the int64-priority engine (several launches per radius;
 * images up to 32767 x 32767; ts_hasf_batch_async rejects r > 16). */
int ts_max_radius(void);

/* HASF: alternate homotopic cutting and filling at radii 1..r_max.
 * Replaces hasf(img, SmoothingConfig(r_max, adj, keep, avoid)) and smooth(img, r_max)
 * (smoothing.py:187-217).  keep_dev / avoid_dev: [n][h][w] constraint images or
 * NULL.  stats_host: NULL or int64[n*36] receiving per image: sweeps, fixpoint
 * passes, engine calls, flips, then SM clock cycles spent in prep (clamped
 * EDT + precedence masks), fixpoint passes, apply+re-examination, in total,
 * and a breakdown by sweep size (fields 8-14; 15 reserved). */
int ts_hasf_batch(const uint8_t *in_dev, uint8_t *out_dev, int64_t n, int32_t h, int32_t w,
                  int32_t r_max, int32_t fg, const uint8_t *keep_dev, const uint8_t *avoid_dev,
                  void *stream, int64_t *stats_host);

/* Same, from host buffers: the batch is pipelined in chunks (H2D copy, fused
 * kernel and D2H copy of neighbouring chunks overlap on separate streams);
 * page-locked buffers give asynchronous copies, pageable ones are staged. */
int ts_hasf_batch_host(const uint8_t *in_host, uint8_t *out_host, int64_t n, int32_t h, int32_t w,
                       int32_t r_max, int32_t fg, const uint8_t *keep_host, const uint8_t *avoid_host,
                       void *stream);

/* One homotopic cutting at radius r (smoothing.py:127-135, 149-165). keep_dev may be NULL. */
int ts_cutting_batch(const uint8_t *in_dev, uint8_t *out_dev, int64_t n, int32_t h, int32_t w,
                     int32_t r, int32_t fg, const uint8_t *keep_dev, void *stream);

/* One homotopic filling at radius r (smoothing.py:138-146, 168-184). avoid_dev may be NULL. */
int ts_filling_batch(const uint8_t *in_dev, uint8_t *out_dev, int64_t n, int32_t h, int32_t w,
                     int32_t r, int32_t fg, const uint8_t *avoid_dev, void *stream);

/* Priority-ordered homotopic thinning (topo.py:279-314): removes simple object
 * points outside keep in (priority, raster) order; max_iter < 0 = unbounded. */
int ts_thin_batch(const uint8_t *img_dev, const uint8_t *keep_dev, const int64_t *prio_dev,
                  uint8_t *out_dev, int64_t n, int32_t h, int32_t w, int32_t fg, int64_t max_iter,
                  void *stream);

/* Priority-ordered homotopic thickening inside allowed (topo.py:317-354). */
int ts_thicken_batch(const uint8_t *img_dev, const uint8_t *allowed_dev, const int64_t *prio_dev,
                     uint8_t *out_dev, int64_t n, int32_t h, int32_t w, int32_t fg, int64_t max_iter,
                     void *stream);

/* Exact squared EDT, int64 out, INF = h^2 + w^2 + 1 where no seed.
 * mode 0: distance to object pixels (edt_squared, edt.py:173-187);
 * mode 1: distance to background incl. the window exterior
 *         (background_distances, morph.py:34-42). */
int ts_edt_sq_batch(const uint8_t *in_dev, int64_t *out_dev, int64_t n, int32_t h, int32_t w,
                    int32_t mode, void *stream);

/* Phase 1 alone: vertical distances G (edt_phase1_columns, edt.py:122-136). */
int ts_edt_phase1_batch(const uint8_t *in_dev, int64_t *g_dev, int64_t n, int32_t h, int32_t w,
                        void *stream);

/* Phase 2 alone: row lower envelopes from G (edt_phase2_rows, edt.py:139-149). */
int ts_edt_phase2_batch(const int64_t *g_dev, int64_t *out_dev, int64_t n, int32_t h, int32_t w,
                        void *stream);

/* Ball dilation / erosion by EDT thresholding (dilate / erode, morph.py:45-59). */
int ts_dilate_batch(const uint8_t *in_dev, uint8_t *out_dev, int64_t n, int32_t h, int32_t w,
                    int32_t r, void *stream);
int ts_erode_batch(const uint8_t *in_dev, uint8_t *out_dev, int64_t n, int32_t h, int32_t w,
                   int32_t r, void *stream);

/* 8-bit neighbour codes (neighborhood_codes, topo.py:97-106). */
int ts_neighborhood_codes_batch(const uint8_t *in_dev, uint8_t *out_dev, int64_t n, int32_t h,
                                int32_t w, void *stream);

/* Simple object points, LUT staged in shared memory (simple_point_mask, topo.py:144-148). */
int ts_simple_point_mask_batch(const uint8_t *in_dev, uint8_t *out_dev, int64_t n, int32_t h,
                               int32_t w, int32_t fg, void *stream);

/* Topology verifier: number of conn-connected components (conn 4 or 8) of the
 * object pixels (foreground = 1) or background pixels (foreground = 0) of each
 * image; exterior = 1 attaches the window exterior to the background as one
 * extra component (component_count / background_component_count,
 * grid.py:93-128).  counts_host: int64[n]. */
int ts_component_counts_batch(const uint8_t *in_dev, int64_t *counts_host, int64_t n, int32_t h, int32_t w,
                              int32_t conn, int32_t foreground, int32_t exterior, void *stream);

/* Host tables: component counts T8/T4 of every 8-bit code and the simple-point
 * LUTs (T8_TABLE, T4_TABLE, SIMPLE_84, SIMPLE_48, topo.py:79-84). */
int ts_connectivity_tables(uint8_t *t8_256, uint8_t *t4_256, uint8_t *s84_256, uint8_t *s48_256);

/* Evaluates the engine's bit-sliced simple-point circuit on all 256 codes on
 * the device (must equal SIMPLE_84 / SIMPLE_48). */
int ts_selftest_circuit(uint8_t *s84_256_host, uint8_t *s48_256_host);

/* Tuning: shared-memory budget (bytes) for the fused kernel's per-image
 * buffers; 0 = device maximum.  Returns the previous value. */
int64_t ts_set_smem_budget(int64_t bytes);

/* Tuning: a sweep runs in dense (strip-walk) mode when more than
 * (words / div) words hold candidates (default 4, minimum 2).  Returns the
 * previous value. */
int32_t ts_set_dense_divisor(int32_t div);

/* Non-blocking ts_hasf_batch for device-resident callers: stream-ordered, no
 * synchronization inside; the device-side error code (0 = none) is written to
 * the caller's device int *err_dev in stream order (zeroed by the call).
 * Returns host-side argument / launch errors only.  Map a code read back
 * later with ts_check_device_error (status + ts_last_error message). */
int ts_hasf_batch_async(const uint8_t *in_dev, uint8_t *out_dev, int64_t n, int32_t h, int32_t w, int32_t r_max,
                        int32_t fg, const uint8_t *keep_dev, const uint8_t *avoid_dev, void *stream,
                        int32_t *err_dev);
int ts_check_device_error(int32_t code);

/* ---- netpbm P4 straight to / from the device bit-row layout -------------
 * P4 rasters (reference netpbm.py:68-129, the raster bytes after the header):
 * [n][h][(w + 7) / 8] bytes, 1 bit per pixel, MSB first, rows padded to a
 * byte, 1 = object; padding bits ignored on read, written as zero.
 * "rows" = the fused kernel's packed format: [n][h][(w + 31) / 32] uint32,
 * leftmost pixel in bit 0, padding bits zero. */
int ts_p4_to_rows(const uint8_t *p4_dev, uint32_t *rows_dev, int64_t n, int32_t h, int32_t w, void *stream);
int ts_rows_to_p4(const uint32_t *rows_dev, uint8_t *p4_dev, int64_t n, int32_t h, int32_t w, void *stream);

/* HASF on P4 rasters without ever unpacking to bytes: P4 -> bit rows on the
 * device, the fused kernel reading / writing bit rows, bit rows -> P4.
 * Replaces read_pbm -> hasf -> write_pbm of cli.run_smooth_command
 * (cli.py:109-143) for P4 files.  keep/avoid: P4 rasters or NULL. */
int ts_hasf_batch_p4(const uint8_t *p4_in_dev, uint8_t *p4_out_dev, int64_t n, int32_t h, int32_t w, int32_t r_max,
                     int32_t fg, const uint8_t *keep_p4_dev, const uint8_t *avoid_p4_dev, void *stream);

/* Tuning/testing: CTAs cooperating on one image (0 = automatic: teams only for
 * images whose hot planes exceed one SM's shared memory and when there are
 * fewer images than co-resident CTAs).  Returns the previous value. */
int32_t ts_set_team_size(int32_t ctas);

/* Tuning / A-B: 1 (default) = teams of 2..8 CTAs (large images, e.g. c2's
 * 2048^2 with 4 CTAs each) run as thread-block clusters: hardware cluster
 * barriers instead of the global-atomic team barrier, and the team's control
 * block (queues' counters, list lengths) in the rank-0 CTA's shared memory,
 * reached by the others over distributed shared memory; 2 = also teams of
 * more than 8 CTAs as several clusters with a hierarchical barrier (cluster
 * barrier + one global arrival per cluster; measured slower on c3); 0 =
 * cooperative launch with the global control block.  Returns the previous value. */
int32_t ts_set_cluster_teams(int32_t on);

/* Tuning/testing: force the kernel flavour, 512 threads x 1 CTA/SM or 256 x 2
 * (0 = automatic: 256 x 2 when the hot planes fit half an SM; 1024 threads per
 * CTA for the cluster teams of large images); 1024 forces 1024-thread CTAs for
 * every team, 512 forces 512-thread teams.  Returns the previous value. */
int32_t ts_set_cta_threads(int32_t threads);

/* Tuning / A-B of ts_hasf_batch_host: 1 (default) = the images are bit-packed
 * on host threads (8x fewer bytes over the host link) and ONE fused launch
 * starts while the packed chunks are still being copied (stream memory
 * operations gate each image on its chunk and each chunk's copy-back on its
 * images); the results are unpacked on the host chunk by chunk; keep /
 * avoid planes are bit-packed and streamed the same way; 2 = streamed uint8
 * chunks, no host packing; 0 = the chunked pipeline of separate launches
 * (always used under a serialising profiler -- ncu / nsys injection --
 * or CUDA_LAUNCH_BLOCKING=1).  Returns the previous value. */
int32_t ts_set_host_streaming(int32_t on);

/* Tuning / A-B: 1 (default) = where eligible (one strip per thread, rows of
 * <= 32 words tiling a warp, r <= 8) the rank slices of the clamped EDT stay in
 * registers (fused prep + E-pass); 0 = always the two-phase prep / E-pass
 * through the rank planes.  Returns the previous value. */
int32_t ts_set_fused_prep(int32_t on);

/* Tuning / A-B of the segmented scheduler: batches with more single-CTA
 * images than one wave of CTAs are handed out as (segment, image) tasks of
 * `stages` consecutive stages (4 stages = one radius: S1/S3 cutting, S5/S7
 * filling, each a prep + engine call), segment-major, so the SMs left idle
 * when the queue drains wait for at most one segment instead of one whole
 * image.  The image's bit-plane passes between segments through global
 * memory; results are identical.  0 = whole images; default 8 (two radii;
 * env TS_SEG_STAGES overrides at load).  Returns the previous value. */
int32_t ts_set_segment_stages(int32_t stages);

/* Tuning / A-B: the last `stages` stages of an image run as one-stage
 * segments (the queue's drain then waits for at most one short stage).
 * Unless this is called (or env TS_SEG_FINE is set, or TS_SEG_TUNE=0), the
 * blocking device entry picks 2 or 1 per problem (shape, batch, radii,
 * adjacency, constraints) by timing its own first three launches of it;
 * the outputs do not depend on the segmentation.  A negative value returns
 * to that per-problem tuning.  Returns the previous value. */
int32_t ts_set_segment_fine(int32_t stages);

/* Tuning / A-B: the segmentation used by the streamed host entry
 * (ts_hasf_batch_host), whose copy-back and host unpacking overlap the
 * kernel only while images keep completing, so it prefers coarser segments;
 * default 8 stages, fine 0 (env TS_SEG_STAGES_HOST / TS_SEG_FINE_HOST).
 * Returns the previous stage count. */
int32_t ts_set_host_segments(int32_t stages, int32_t fine);

/* Testing: 1 = segment batches of any size (tasks then often wait for their
 * predecessor segment on another SM).  Returns the previous value. */
int32_t ts_set_segment_force(int32_t on);

/* Debug: record, for the first `tasks` tasks of every later fused launch, 7
 * int64 per task into the device buffer trace_dev: SM id, then %globaltimer
 * (ns) when the task was taken from the queue, when its input was ready (after
 * any wait for the predecessor segment / input chunk), loaded into the CTA,
 * its stages were done, its result stored, and the task finished.  Task t =
 * segment * n + image (segmented) or image.  NULL disables. */
void ts_set_trace(int64_t *trace_dev, int64_t tasks);

/* Placement/occupancy the fused kernel would use for an image shape:
 * info[0] = grid CTAs per wave, info[1] = CTAs per SM, info[2] = smem bytes,
 * info[3] = smem buffer mask, info[4] = global workspace bytes per CTA,
 * info[5] = threads per CTA (info must hold 6 values). */
int ts_hasf_plan(int32_t h, int32_t w, int32_t r_max, int32_t has_keep, int32_t has_avoid,
                 int64_t *info5);

#ifdef __cplusplus
}
#endif

#endif /* TOPOSMOOTH_B200_H */
