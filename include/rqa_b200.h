/*
 * rqa_b200.h -- C-ABI of the B200-native RQA engine (librqa_b200.so).
 *
 * This boundary replaces the reference's tiled engine entry point
 *     tiledrqa.engine.run_analysis(embedded, settings, tile_size, workers)
 *     (/root/reference/pkg/src/tiledrqa/engine.py:215-280)
 * which the reference's API calls from analyze() (__init__.py:31-39) and the
 * CLI (cli.py:129-131).  The Python mirror paper_2402_16853_b200.engine
 * .run_analysis binds these symbols with ctypes.
 *
 * Conventions: plain pointers and sizes only; series are float64 samples of
 * the scalar time series (the embedding is implicit, embedding.py:32-69);
 * histograms are int64[n+1] with index = line length (index 0 unused), like
 * LineHistograms (histograms.py:16-67).  metric: 0 = L1 (manhattan),
 * 1 = L2 (euclidean), 2 = Linf (maximum) (settings.py:9-23).  theiler: 0 keeps
 * the main diagonal (reference default), 1 = include_main_diagonal=False
 * (embedding.py:158-171), w > 1 zeroes every cell with |i-j| < w (extension).
 *
 * Return codes: 0 ok; RQA_EINVAL (-1) -> InvalidArgument;
 * RQA_ESHORT (-2) -> SeriesTooShort (embedding.py:64-68); RQA_EDEVICE (-3)
 * -> DeviceError (CUDA failure); RQA_ENOMEM (-4) -> DeviceError (allocation).
 * A message is written to err (NUL-terminated, at most errlen bytes).
 * There is no CPU fallback: without a usable CUDA device every compute entry
 * point returns RQA_EDEVICE.
 */
#ifndef RQA_B200_H
#define RQA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RQA_OK 0
#define RQA_EINVAL (-1)
#define RQA_ESHORT (-2)
#define RQA_EDEVICE (-3)
#define RQA_ENOMEM (-4)
#define RQA_EUNSUPPORTED (-5) /* rqa_read_column: input the native reader does not handle */
#define RQA_EIO (-6)          /* rqa_read_column: FileNotReadable */
#define RQA_ECOLUMN (-7)      /* rqa_read_column: ColumnOutOfRange */
#define RQA_EPARSE (-8)       /* rqa_read_column: ParseError (token in err) */
#define RQA_EEMPTY (-9)       /* rqa_read_column: EmptySeries */

/* Number of timing slots written by rqa_run (seconds):
 * [0] h2d, [1] band kernel, [2] fold kernel, [3] d2h, [4] total device span,
 * [5] cells per second over the band+fold kernels, [6] band height,
 * [7] number of bands, [8] evaluation path (-1 float64 kernels, 0 f32 filter
 * with float64 re-evaluation (exact), 1 fp32 mode, 2 float64 sparse
 * prefilter (exact)), [9] certified band half-width of the f32 filter,
 * [10] sampled fraction of prefilter candidate cells (-1 if not sampled).  Very large n is split into row stripes
 * processed one after the other on the device when the band summaries would
 * not fit. */
#define RQA_TIMING_SLOTS 11

/* rqa_run_prec flags */
#define RQA_FLAG_OUT_ZEROED 1

/* Library version as MAJOR*10000 + MINOR*100 + PATCH. */
int rqa_version(void);

/* Number of visible CUDA devices (0 when none / no driver). */
int rqa_device_count(void);

/* Total kernel launches issued by this library since load (for evidence of
 * GPU execution in benchmarks). */
int64_t rqa_launch_counter(void);

/* Exact threshold used by the kernels: T* = max{x : RN(sqrt(x)) <= radius}
 * for L2 with m > 1 (replaces sqrt, embedding.py:154-156), radius otherwise. */
int rqa_threshold(int32_t metric, int32_t m, double radius, double *thr);

/* Band height (rows per CTA) and kernel variant chosen for (metric, m, tau)
 * and n embedded vectors (mid-size n uses shorter bands to balance the SMs). */
int rqa_band_rows(int32_t metric, int32_t m, int32_t tau, int64_t n, int64_t *band_rows,
                  int32_t *reuse_kernel);

/*
 * Host-only diagnostic: the work-unit plan of the band kernel for n vectors,
 * rows [row_lo, row_hi), bands of band_rows = r * slot_rows rows and `slots`
 * resident CTAs (no device needed).  Writes up to cap units as (band, xa, xb)
 * triples in band order (iteration ranges of each band's diagonal sweep) and
 * *count (the full number, also when > cap).  The plan replaces the
 * reference's tile partition (engine.py:86-126) as the unit of scheduling.
 */
int rqa_plan_units(int64_t n, int64_t row_lo, int64_t row_hi, int32_t slot_rows, int32_t r,
                   int32_t slots, int32_t *units, int64_t cap, int64_t *count);

/*
 * Full analysis of a host series on one device: replaces run_analysis
 * (engine.py:215-280).  Writes the three histograms (int64[n+1] each, n =
 * len - (m-1)*tau), the recurrence point count and RQA_TIMING_SLOTS timings.
 */
int rqa_run(const double *series, int64_t len, int32_t m, int32_t tau, int32_t metric,
            double radius, int64_t theiler, int32_t device, int64_t *diag, int64_t *vert,
            int64_t *white, int64_t *points, double *timing, char *err, size_t errlen);

/*
 * rqa_run with a precision (the reference's run_analysis plus the
 * `precision=` keyword of SURVEY.md 8b):
 *   64: results bit-exact against the float64 reference.  Cells may be
 *       evaluated in float32 inside a certified band test (the "f32
 *       filter"); every word with a cell near the threshold is re-evaluated
 *       in float64, so the histograms are identical either way.
 *   32: fp32 mode -- samples, arithmetic and threshold in float32 (numpy
 *       float32 semantics); *mismatches (may be NULL) receives the number of
 *       cells of the full n x n matrix whose fp32 decision differs from the
 *       float64 one.
 * flags: RQA_FLAG_OUT_ZEROED -- diag/vert/white are already zero-filled; only
 *       the nonzero bins are copied back (compacted on the device).
 */
int rqa_run_prec(const double *series, int64_t len, int32_t m, int32_t tau, int32_t metric,
                 double radius, int64_t theiler, int32_t precision, int32_t device,
                 int32_t flags, int64_t *diag, int64_t *vert, int64_t *white, int64_t *points,
                 int64_t *mismatches, double *timing, char *err, size_t errlen);

/*
 * Single-process multi-GPU analysis (run_analysis(devices=[...])): the rows
 * are split into n_devices equal-area stripes of the upper triangle, one host
 * thread per stripe runs it on devices[g] (a device may appear more than
 * once), the stripe summaries are gathered on devices[0] by peer copies
 * (NVLink) and stitched there (rqa_stitch_device semantics); the stripes'
 * histograms and counts are summed on devices[0] as well (peer copies plus a
 * reduction kernel), so one (sparse, with RQA_FLAG_OUT_ZEROED) copy-back
 * crosses PCIe.  Results are identical to rqa_run_prec for every device
 * list.  n_devices == 1 is rqa_run_prec.  Timing: [1] slowest stripe's
 * kernels, [2] gather + reduction + stitch, [4] wall, [5] cells/s over the
 * wall, [6] band rows, [7] stripes, [8..10] as rqa_run_prec.
 * Replaces the merge of per-worker partials, engine.py:271-276.
 */
int rqa_run_multi(const double *series, int64_t len, int32_t m, int32_t tau, int32_t metric,
                  double radius, int64_t theiler, int32_t precision, const int32_t *devices,
                  int32_t n_devices, int32_t flags, int64_t *diag, int64_t *vert, int64_t *white,
                  int64_t *points, int64_t *mismatches, double *timing, char *err,
                  size_t errlen);

/*
 * Device-resident variant for callers that own device memory and a stream
 * (torch tensors): rows [row_lo, row_hi) of the recurrence matrix.
 *   mode 0 (final): rows must be [0, n); d_hist (int64[3*(n+1)], rows diag,
 *     vert, white) and d_points are ACCUMULATED into (zero them first).
 *   mode 1 (stripe): one row stripe of a multi-GPU run.  Lines that cross
 *     the stripe's edges are not counted; instead the stripe reports
 *       d_stripe_prefix / d_stripe_suffix (int32[n]): per diagonal k >= 0 the
 *         1-run starting at the stripe's top / ending at its bottom edge;
 *       d_stripe_col (uint32[2n]): per column c the first and last run
 *         ((len << 1) | bit) of the column's part inside the stripe above the
 *         main diagonal;
 *       d_rowpart (uint32[2n], zero-initialised by the caller): for the
 *         stripe's rows i, the first and last run of row i from the diagonal
 *         to column n-1.
 *     All four go to rqa_stitch_device (after an all-gather / sum-reduce).
 * Only the upper triangle k >= 0 is evaluated: R = R^T exactly, so diagonal
 * -k equals diagonal k and column c equals the "hook" (upper column c above
 * the diagonal, then upper row c) -- see DESIGN.md.
 * stream is a cudaStream_t (NULL = legacy default stream); the call is
 * asynchronous with respect to the host except for workspace growth.
 */
int rqa_run_device(const double *d_series, int64_t len, int32_t m, int32_t tau, int32_t metric,
                   double radius, int64_t theiler, int64_t row_lo, int64_t row_hi, int32_t mode,
                   int64_t *d_hist, int64_t *d_points, int32_t *d_stripe_prefix,
                   int32_t *d_stripe_suffix, uint32_t *d_stripe_col, uint32_t *d_rowpart,
                   void *stream, char *err, size_t errlen);

/* rqa_run_device with a precision (64 or 32, see rqa_run_prec); in fp32 mode
 * the mismatch count is ACCUMULATED into *d_mismatches (int64, device). */
int rqa_run_device_prec(const double *d_series, int64_t len, int32_t m, int32_t tau,
                        int32_t metric, double radius, int64_t theiler, int32_t precision,
                        int64_t row_lo, int64_t row_hi, int32_t mode, int64_t *d_hist,
                        int64_t *d_points, int64_t *d_mismatches, int32_t *d_stripe_prefix,
                        int32_t *d_stripe_suffix, uint32_t *d_stripe_col, uint32_t *d_rowpart,
                        void *stream, char *err, size_t errlen);

/*
 * Cross-stripe stitch (engine.py:287-319 carry contract + flush :195-212):
 * d_prefix / d_suffix (int32[nstripes][n]) and d_col (uint32[nstripes][2n])
 * gathered from every stripe in row order, d_rowpart (uint32[2n]) summed over
 * the stripes, bounds (host) the nstripes+1 stripe row boundaries.  Adds the
 * diagonal, vertical and white-vertical lines that cross stripe edges into
 * d_hist.
 */
int rqa_stitch_device(const int32_t *d_prefix, const int32_t *d_suffix, const uint32_t *d_col,
                      const uint32_t *d_rowpart, const int64_t *bounds, int32_t nstripes,
                      int64_t n, int64_t *d_hist, void *stream, char *err, size_t errlen);

/*
 * Recurrence-matrix block / recurrence plot (reference recurrence_block,
 * embedding.py:115-171, and compute_plot/_or_reduce, plotting.py:48-109):
 * rows [row0, row1) x columns [col0, col1) of the n x n matrix, OR-reduced in
 * factor x factor blocks aligned to row0/col0, written row by row (row0 first)
 * packed MSB-first and padded to whole bytes: ceil((row1-row0)/factor) rows of
 * ceil(ceil((col1-col0)/factor)/8) bytes (numpy.packbits(axis=1) layout).
 */
int rqa_block(const double *series, int64_t len, int32_t m, int32_t tau, int32_t metric,
              double radius, int64_t theiler, int64_t row0, int64_t row1, int64_t col0,
              int64_t col1, int32_t factor, int32_t device, uint8_t *out, char *err,
              size_t errlen);

/*
 * Per-tile line detectors of the reference's operator API on the GPU
 * (detect_diagonal_lines / detect_vertical_lines, engine.py:167-192 and the
 * scans of :322-433, carry contract :287-319).  tile_bits: height x width
 * bits, row-major, MSB first (np.packbits of the flattened tile).
 *   kind 0: diagonals; carry_a = the tile's height+width-1 diagonal carries
 *     (CarryoverBuffers.diagonal[(col0-row0) - (height-1) + n-1 ...]),
 *     hist_a = LineHistograms.diagonal (n+1, accumulated into).
 *   kind 1: columns; carry_a / carry_b = the width vertical / white-vertical
 *     carries, hist_a / hist_b = vertical / white_vertical histograms.
 * Carries are updated in place.  Dependency checks stay with the caller.
 */
int rqa_tile_scan(const uint8_t *tile_bits, int64_t height, int64_t width, int64_t n,
                  int32_t kind, int64_t *carry_a, int64_t *carry_b, int64_t *hist_a,
                  int64_t *hist_b, int32_t device, char *err, size_t errlen);

/* FP64 pipe microbenchmark on `device`: sustained DADD and DMUL operations
 * per second (the roofline denominator of the FP64-bound band kernel). */
int rqa_fp64_peak(int32_t device, double *dadd_per_s, double *dmul_per_s, char *err,
                  size_t errlen);

/*
 * Native, multi-threaded read_column (ingest.py:53-129) for ASCII files:
 * universal newlines, blank lines ignored, `offset` non-empty rows skipped
 * unparsed, the token str.strip()ped and parsed like Python float()
 * (underscores, inf/nan spellings), non-finite values rejected.  On success
 * *values is a malloc'ed array of *count doubles (free with rqa_free) and
 * *skipped the rows dropped by skip_invalid.  Errors: RQA_EIO, RQA_ECOLUMN
 * (*err_line, *err_fields), RQA_EPARSE (*err_line, the token's bytes in err and
 * their count in *err_fields), RQA_EEMPTY;
 * RQA_EUNSUPPORTED for non-ASCII content or delimiters (use the Python
 * reader).  threads <= 0: all hardware threads.
 */
int rqa_read_column(const char *path, char delimiter, int64_t column, int64_t offset,
                    int32_t skip_invalid, int32_t threads, double **values, int64_t *count,
                    int64_t *skipped, int64_t *err_line, int64_t *err_fields, char *err,
                    size_t errlen);
void rqa_free(void *p);

/* Release cached device workspaces of this process. */
int rqa_release(void);

#ifdef __cplusplus
}
#endif

#endif /* RQA_B200_H */
