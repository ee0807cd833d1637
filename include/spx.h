/*
 * spx.h -- C ABI of the B200-native SLIC superpixel library (libspx.so).
 *
 * This is the drop-in boundary.  The reference selects its kernel set through
 * the plugin protocol of pkg/src/superpix/kernels/__init__.py:12-44 and the
 * engine calls each kernel as fn(*args, lo, hi) (engine.py:38-39, 56-63).
 * The nine per-stage entry points below replace, one for one, the nine
 * functions of pkg/src/superpix/kernels/_core.pyx (same argument meaning,
 * same half-open band / cluster-range semantics, same in-place outputs), but
 * take DEVICE pointers plus a CUDA stream.  The engine entry points replace
 * SegEngine.perform_segmentation (engine.py:125-230) for whole frames and for
 * batches of frames.
 *
 * Conventions
 *   - All arrays are C-contiguous with the reference layouts:
 *       rgb    uint8  [h][w][3]        img/out float32 [h][w][3]
 *       labels int32  [h][w]           cxy float64 [K][2] (x, y)
 *       clab   float64 [K][3]          counts int64 [K]
 *       slab   float64 [K][n_bl][6]   (sum_l, sum_a, sum_b, sum_x, sum_y, count)
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *   - Every call returns an spx_status; on error spx_last_error() describes it.
 *   - Work is enqueued asynchronously on `stream` unless stated otherwise.
 *   - There is no CPU fallback: without a usable sm_100 device every entry
 *     point returns SPX_ERR_CUDA.
 */
#ifndef SPX_H
#define SPX_H

#include <stdint.h>

#if defined(__GNUC__)
#define SPX_API __attribute__((visibility("default")))
#else
#define SPX_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum spx_status {
  SPX_OK = 0,
  SPX_ERR_INVALID_SETTINGS = 1, /* -> errors.InvalidSettingsError (errors.py:12) */
  SPX_ERR_DIMENSION = 2,        /* -> errors.DimensionMismatchError (errors.py:16) */
  SPX_ERR_CUDA = 3,             /* CUDA runtime failure                            */
  SPX_ERR_NOMEM = 4,            /* -> MemoryError (_core.pyx:380-394)             */
  SPX_ERR_VALUE = 5             /* -> ValueError (bad argument)                   */
} spx_status;

/* Thread-local description of the last failing call on this thread. */
SPX_API const char *spx_last_error(void);
/* Implementation name, the analogue of _core.pyx:16 `NAME = "compiled"`. */
SPX_API const char *spx_name(void);
SPX_API int32_t spx_abi_version(void);
/* Test hook: the host-side colour tables (tables.py:14-54) the kernels use. */
SPX_API int32_t spx_debug_tables(double *lut, double *mat, double *white);
/* Test hook: max relative error of the association filter's fp32 sqrt over
 * all floats in [1,4) (the error bound assumes <= 2^-21).  Synchronous. */
SPX_API int32_t spx_debug_sqrt_error(double *out_host);
/* Test hook: the update's branch-free division vs the IEEE division on n
 * random operand pairs; out2_host = {mismatches, pairs that took the fast path}. */
SPX_API int32_t spx_debug_ddiv_check(int64_t n, uint64_t seed, int64_t *out2_host);

/* ---- kernel protocol: replaces pkg/src/superpix/kernels/_core.pyx ---------- */

/* _core.pyx:45-83 convert_band: rows [y0,y1) of rgb -> out in `space`
 * (0 RGB /255, 1 XYZ, 2 CIELAB; tables.py:10-12), bit-exact. */
SPX_API int32_t spx_convert_band(const uint8_t *rgb, float *out, int64_t h, int64_t w,
                         int32_t space, int64_t y0, int64_t y1, void *stream);

/* _core.pyx:86-107 init_centers_range: clusters [k0,k1). */
SPX_API int32_t spx_init_centers_range(const float *img, int64_t h, int64_t w, int64_t s,
                               int64_t ns_c, double *cxy, double *clab, int64_t k0,
                               int64_t k1, void *stream);

/* _core.pyx:123-156 perturb_range: clusters [k0,k1), in place. */
SPX_API int32_t spx_perturb_range(const float *img, int64_t h, int64_t w, double *cxy,
                          double *clab, int64_t k0, int64_t k1, void *stream);

/* _core.pyx:172-197 associate_band: rows [y0,y1).  n_clusters = rows of
 * cxy/clab (must be >= ns_r*ns_c; the reference reads them unchecked). */
SPX_API int32_t spx_associate_band(const float *img, int64_t h, int64_t w, const double *cxy,
                           const double *clab, int64_t n_clusters, int32_t *labels,
                           int64_t s, int64_t ns_r, int64_t ns_c, double xy_weight,
                           int64_t y0, int64_t y1, void *stream);

/* _core.pyx:200-255 accumulate_range: per-strip sums of clusters [k0,k1). */
SPX_API int32_t spx_accumulate_range(const float *img, const int32_t *labels, int64_t h,
                             int64_t w, double *slab, int64_t n_bl, int64_t s,
                             int64_t ns_c, int64_t tile_len, int64_t k0, int64_t k1,
                             void *stream);

/* _core.pyx:258-285 accumulate_spill.  n_clusters = rows of slab.  Writes the
 * spill count to *spills_host; SYNCHRONISES `stream` (the count is a host
 * return value in the reference). */
SPX_API int32_t spx_accumulate_spill(const float *img, const int32_t *labels, int64_t h,
                             int64_t w, double *slab, int64_t n_clusters, int64_t n_bl,
                             int64_t s, int64_t ns_c, int64_t *spills_host, void *stream);

/* _core.pyx:288-325 reduce_range: destroys slab rows [k0,k1). */
SPX_API int32_t spx_reduce_range(double *slab, int64_t n_bl, const double *prev_xy,
                         const double *prev_lab, double *out_xy, double *out_lab,
                         int64_t *out_counts, int64_t k0, int64_t k1, void *stream);

/* _core.pyx:328-356 weak_band: rows [y0,y1) of dst from frozen src. */
SPX_API int32_t spx_weak_band(const int32_t *src, int32_t *dst, int64_t h, int64_t w,
                      int64_t y0, int64_t y1, void *stream);

/* _core.pyx:359-461 strict_fill, computed in parallel (connected components +
 * ordered absorption) with results identical to the sequential scan.
 * SYNCHRONISES `stream` (needs the label range). */
SPX_API int32_t spx_strict_fill(const int32_t *src, int32_t *dst, int64_t h, int64_t w,
                        int64_t min_size, void *stream);

/* L1 centre shift exactly as engine.py:196 / slic_core.py:384-390 evaluate
 * it (numpy pairwise summation order).  Device inputs, device output. */
SPX_API int32_t spx_center_shift(const double *new_xy, const double *old_xy, int64_t k,
                         double *out_dev, void *stream);
/* numpy's pairwise summation (np.add.reduce over a contiguous float64
 * array, the tree the shift above uses) of n device doubles into out_dev[0];
 * the row strips' early-stop shift over the gathered per-cluster |delta|. */
SPX_API int32_t spx_pairwise_sum(const double *x, int64_t n, double *out_dev, void *stream);

/* ---- engine: replaces SegEngine (engine.py:86-230) ------------------------- */

typedef struct spx_settings {
  int64_t width, height;  /* Settings.img_width / img_height              */
  int64_t s, ns_r, ns_c;  /* compute_grid() result (slic_core.py:228-249)  */
  double compactness;     /* Settings.compactness (xy_weight = m / s)     */
  int32_t no_iters;       /* Settings.no_iters                            */
  int32_t color_space;    /* 0 RGB, 1 XYZ, 2 LAB                          */
  int32_t connectivity;   /* 0 off, 1 weak, 2 strict                      */
  int32_t perturb;        /* Settings.enable_perturbation                 */
  int64_t tile_len;       /* Settings.tile_len                            */
  int64_t min_size;       /* resolved strict min_size                     */
  double early_stop;      /* < 0 means None                               */
} spx_settings;

typedef struct spx_engine spx_engine;

/* Per-stage device times (ms) of the last segment call, batch-wide.
 * associate/update hold one entry per pass actually run (max over frames). */
typedef struct spx_timing {
  float convert, init, perturb, connectivity, total;
  float associate[1024];
  float update[1024];
  int32_t n_associate, n_update;
} spx_timing;

SPX_API int32_t spx_engine_create(const spx_settings *st, int64_t max_batch, int32_t device,
                          spx_engine **out);
SPX_API int32_t spx_engine_destroy(spx_engine *eng);

/* Segment `batch` frames already resident in device memory.  Outputs:
 * labels [batch][h][w], cxy [batch][K][2], clab [batch][K][3],
 * counts [batch][K], passes [batch] (updates run per frame; may be NULL).
 * Asynchronous on `stream`. */
SPX_API int32_t spx_engine_segment(spx_engine *eng, const uint8_t *rgb_dev, int64_t batch,
                           int32_t *labels_dev, double *cxy_dev, double *clab_dev,
                           int64_t *counts_dev, int32_t *passes_dev, void *stream);

/* Same with HOST buffers (any batch size): frames are processed in chunks of
 * up to 64 (spx_engine_set_host_chunk) through three device staging slots on
 * three streams (H2D, compute, D2H), so the H2D copy of the next chunk and the
 * D2H copy of the previous one overlap the compute of the current one.  Pinned host buffers make the copies
 * asynchronous (pageable ones are correct but serialised).  Synchronous. */
SPX_API int32_t spx_engine_segment_host(spx_engine *eng, const uint8_t *rgb_host, int64_t batch,
                                int32_t *labels_host, double *cxy_host, double *clab_host,
                                int64_t *counts_host, int32_t *passes_host);

/* Byte offsets of the five outputs of `batch` frames laid out in ONE host
 * block: out6 = {labels, cxy, clab, counts, passes, total bytes}.  Host
 * outputs placed at these offsets from labels_host (pinned) are copied back
 * with a single D2H per call (batch <= the host chunk). */
SPX_API int32_t spx_engine_output_layout(spx_engine *eng, int64_t batch, int64_t *out6);

/* Asynchronous form of spx_engine_segment_host for streams of batches: enqueues
 * the batch's H2D / compute / D2H chunks and returns.  Consecutive submits
 * continue one pipeline, so the copies of batch i overlap the compute of
 * batch i+1.  Host buffers must stay valid (and the outputs unread) until
 * spx_engine_wait returns.  Input buffers should be pinned. */
SPX_API int32_t spx_engine_submit_host(spx_engine *eng, const uint8_t *rgb_host, int64_t batch,
                               int32_t *labels_host, double *cxy_host, double *clab_host,
                               int64_t *counts_host, int32_t *passes_host);
SPX_API int32_t spx_engine_wait(spx_engine *eng);
/* Ticket of the work submitted so far (read it after a submit) and a wait for
 * that submission only, so a caller can consume batch i while i+1 runs. */
SPX_API int64_t spx_engine_ticket(spx_engine *eng);
SPX_API int32_t spx_engine_wait_ticket(spx_engine *eng, int64_t ticket);
/* Device time (ms, compute stream) of the submission that returned `ticket`
 * (kept for the last 8 submissions); waits for that submission's compute
 * only -- unlike spx_engine_timing, which describes the newest call. */
SPX_API int32_t spx_engine_ticket_time(spx_engine *eng, int64_t ticket, float *ms);
/* Frames per host-pipeline chunk (default 64, capped at max_batch); waits for
 * submitted work and re-allocates the staging buffers. */
SPX_API int32_t spx_engine_set_host_chunk(spx_engine *eng, int64_t frames);

/* Lanes: a segment call of two or more frames may be split into `lanes`
 * sub-batches on concurrent streams, each on a child engine created on first
 * use (so the per-frame buffers exist twice); the convert of one lane
 * overlaps the association of another.  Calls of <= 64 frames replay a
 * CUDA graph that forks the lanes.  0 (default) = automatic: none below 4
 * frames, three for calls of more than 64 frames under 24 Mpx, otherwise
 * four.  Results do not depend on the split.  With more
 * than one lane, spx_engine_timing reports lane 0's stage times (measured
 * while the other lanes ran) and the whole call's total. */
SPX_API int32_t spx_engine_set_lanes(spx_engine *eng, int32_t lanes);
/* Lanes the last spx_engine_segment* call used. */
SPX_API int32_t spx_engine_last_lanes(spx_engine *eng);

/* Stage timings of the last spx_engine_segment* call (synchronises). */
SPX_API int32_t spx_engine_timing(spx_engine *eng, spx_timing *out);

/* ---- row strips: one large image across ranks --------
 * A strip owns grid cell rows [row_lo, row_hi) of the global settings `st`.
 * Its input is the RGB window rows [y0, y0 + hl) reported by
 * spx_strip_geometry (own rows plus one halo cell row on each side that
 * exists).  Per iteration the host moves three kinds of buffers between
 * vertical neighbours (NCCL send/recv between ranks, or device copies):
 *   centres  ns_c * 5 doubles   (pack after begin/update, unpack before associate)
 *   sums     ns_c * 48 bytes    (pack after associate-with-update, unpack before update)
 *   labels   S * W int32        (pack after associate, unpack before update/finish)
 * Sequence: begin, xchg centres, { associate(1), xchg sums+labels, update,
 * xchg centres } x no_iters, associate(0), xchg labels, finish.
 * Results equal the single-GPU engine bit for bit.  Fused-cell geometry
 * (4 <= S <= 255); early stop through spx_strip_shift_local +
 * spx_pairwise_sum over the gathered shifts.  With strict connectivity
 * (a whole-image scan-order pass) finish returns the raw labels and the
 * caller runs spx_strict_fill over the gathered image. */
typedef struct spx_strip spx_strip;
SPX_API int32_t spx_strip_create(const spx_settings *st, int64_t row_lo, int64_t row_hi,
                                 int32_t device, spx_strip **out);
SPX_API int32_t spx_strip_destroy(spx_strip *s);
/* out6 = {y0, hl, own_y0, own_y1, row_lo, row_hi} (global pixel / cell rows). */
SPX_API int32_t spx_strip_geometry(spx_strip *s, int64_t *out6);
SPX_API int32_t spx_strip_begin(spx_strip *s, const uint8_t *rgb_window, void *stream);
SPX_API int32_t spx_strip_associate(spx_strip *s, int32_t with_update, void *stream);
SPX_API int32_t spx_strip_update(spx_strip *s, void *stream);
/* The same steps split so the exchanges overlap compute: part 1 = interior
 * own cell rows / clusters (need nothing from the neighbours), part 2 =
 * boundary rows / clusters (after the neighbours' centres, respectively
 * partial sums and labels, are unpacked), part 0 = all.  Per iteration:
 * associate(1, interior), unpack centres, associate(1, boundary), start the
 * sums + labels exchange, update(interior), unpack sums + labels,
 * update(boundary) [which runs the exact fallback], start the centres
 * exchange. */
SPX_API int32_t spx_strip_associate_part(spx_strip *s, int32_t with_update, int32_t part,
                                         void *stream);
SPX_API int32_t spx_strip_update_part(spx_strip *s, int32_t part, void *stream);
/* Early stop: |new - old| of the own clusters' centres after an update
 * ((row_hi - row_lo) * ns_c * 2 doubles, cluster order); the ranks' arrays
 * concatenated in rank order are the whole image's, whose spx_pairwise_sum
 * is the reference's shift (engine.py:196). */
SPX_API int32_t spx_strip_shift_local(spx_strip *s, double *out, void *stream);
SPX_API int32_t spx_strip_pack_centres(spx_strip *s, double *up, double *down, void *stream);
SPX_API int32_t spx_strip_unpack_centres(spx_strip *s, const double *from_up,
                                         const double *from_down, void *stream);
SPX_API int32_t spx_strip_pack_sums(spx_strip *s, void *up, void *down, void *stream);
SPX_API int32_t spx_strip_unpack_sums(spx_strip *s, const void *from_up, const void *from_down,
                                      void *stream);
SPX_API int32_t spx_strip_pack_labels(spx_strip *s, int32_t *up, int32_t *down, void *stream);
SPX_API int32_t spx_strip_unpack_labels(spx_strip *s, const int32_t *from_up,
                                        const int32_t *from_down, void *stream);
/* Own rows' labels (global ids) and own clusters' centres / counts. */
SPX_API int32_t spx_strip_finish(spx_strip *s, int32_t *labels, double *cxy, double *clab,
                                 int64_t *counts, void *stream);

/* Number of kernel launches the last segment call enqueued. */
SPX_API int64_t spx_engine_last_launches(spx_engine *eng);

/* 1 when the engine runs the fused cell kernels (4 <= S <= 255 and
 * ceil(3S / tile_len) <= 64 strips), 0 for the generic per-stage kernels. */
SPX_API int32_t spx_engine_fused_path(spx_engine *eng);

#ifdef __cplusplus
}
#endif

#endif /* SPX_H */
