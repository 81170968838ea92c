/*
 * trigbf_b200.h -- C ABI of the B200-native constant-time trigonometric
 * bilateral filter (arXiv 1105.4204 hot path).
 *
 * All pointers named d_* / f / out / num / den / workspace are DEVICE
 * pointers (CUDA global memory on the current device); h_* are host
 * pointers; `stream` is a cudaStream_t passed as void*.  Every entry point
 * is asynchronous on `stream` and returns a status code for errors
 * detectable at launch time.  No torch / C++ types cross this boundary.
 *
 * What each entry replaces in the reference package (/root/reference/pkg):
 *
 *   tbf_bilateral_trig_host
 *                        engines.py:228-306  bilateral_trig(img, spatial, kernel)
 *                        end to end on host arrays (the NumPy-level call)
 *   tbf_bilateral_trig   engines.py:228-306  bilateral_trig(img, spatial, kernel)
 *                        (term loop + smooth_plane + demodulate + _guarded_ratio)
 *                        on device buffers
 *   tbf_trig_partial     engines.py:249-300  the term loop restricted to the
 *                        pairs [term_begin, term_end): accumulates num/den only
 *                        (term-sharded multi-GPU path; NCCL reduce sits between
 *                        this and tbf_finalize)
 *   tbf_trig_partial_rows the same restricted to a band of output rows (balanced
 *                        term sharding: leftover terms split by rows)
 *   tbf_finalize         engines.py:109-117  _guarded_ratio(num, den, f)
 *   tbf_range_check      engines.py:218-225  _check_range(plane, T)
 *   tbf_recursive_smooth_f64
 *                        _core.pyx:56-96     recursive_smooth(a, scale, c1..c4, pad)
 *                        (the L1 plugin entry _backend.recursive_smooth,
 *                        _backend.py:38-39)
 *   tbf_box_pass_f64     _core.pyx:28-53     box_pass(a, radius)
 *                        (_backend.box_pass, _backend.py:38)
 *   tbf_bilateral_direct engines.py:120-151  bilateral_direct(img, spatial, range_fn)
 *                        (fp64 brute force; Gaussian kernels.py:174-182 or
 *                        raised cosine kernels.py:161-171 range kernel)
 *   tbf_workspace_bytes, tbf_layout_info, tbf_set_option, tbf_profile_*, tbf_last_error,
 *   tbf_abi_version      (new: sizing, tuning, per-kernel timing, errors)
 */
#ifndef TRIGBF_B200_H
#define TRIGBF_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define TBF_API __attribute__((visibility("default")))
#else
#define TBF_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes (the Python wrapper maps them to the reference's exception
 * classes, errors.py:4-24). */
#define TBF_OK 0
#define TBF_ERR_RANGE 1     /* ParameterError: samples outside [0, T]      */
#define TBF_ERR_PARAM 2     /* ParameterError: bad filter / kernel params   */
#define TBF_ERR_DIM 3       /* DimensionError: bad shape                    */
#define TBF_ERR_CUDA 4      /* CUDA launch / runtime error                  */
#define TBF_ERR_WORKSPACE 5 /* workspace too small                          */

#define TBF_SPATIAL_RECURSIVE 0 /* SpatialKind.GAUSSIAN_RECURSIVE, spatial.py:31-34 */
#define TBF_SPATIAL_BOX 1       /* SpatialKind.BOX                                   */

/* Spatial smoother (SpatialSpec, spatial.py:41-74), already reduced to the
 * numbers the device needs.  Recursive Gaussian: the reference's 4th-order
 * recursion (spatial.py:124-144) factored into its two pole pairs, i.e. two
 * second-order sections y = g*x + a1*y[-1] + a2*y[-2] (g1,a1,a2) then
 * (g2,b1,b2).  ext_y / ext_x: mirror warm-up length per axis, min(K, n-1)
 * where K is the decay length of the recursion (the reference uses n-1,
 * spatial.py:163-172; beyond K the difference is below 1e-7 relative). */
typedef struct tbf_spatial {
    int32_t kind;
    int32_t radius; /* box radius (>= 0) */
    double g1, a1, a2;
    double g2, b1, b2;
    int32_t ext_y;
    int32_t ext_x;
} tbf_spatial;

/* Raised-cosine range kernel expansion (make_trig_kernel, kernels.py:125-158,
 * folded into frequency/weight pairs as in engines.py:249-253).  Host arrays,
 * ascending frequency; nu[j] = nu[0] + j*dnu must hold (true for the
 * reference's pairs, including a leading zero frequency for even N). */
typedef struct tbf_terms {
    int32_t n_terms;      /* number of pairs (P + [N even]) */
    const double* nu;     /* [n_terms] frequencies */
    const double* weight; /* [n_terms] pair weights */
    double dnu;           /* 2*omega */
    double T;             /* declared intensity range */
} tbf_terms;

/* Launch layout a call would use (no GPU needed; for tests and tuning).
 * host_entry != 0: the layout of tbf_bilateral_trig_host.  Fills
 * info[TBF_LAYOUT_INFO_N]: term batches, terms per batch, pass-1 y-chunks,
 * planned unequal y-chunks (0/1), first two y-chunk ends (rows; H when absent),
 * largest y-chunk (rows), pass-2 x-chunks of the first batch, planned unequal
 * x-chunks (0/1), first two x-chunk ends (column tiles), equal-chunk width
 * (tiles), dispatch order of planned x-chunks (2 bits per rank), column tiles.
 * Returns TBF_OK or an error code. */
#define TBF_LAYOUT_INFO_N 14
TBF_API int tbf_layout_info(int32_t B, int32_t H, int32_t W, const tbf_spatial* sp, int32_t term_begin,
                            int32_t term_end, int32_t batch_terms, int32_t host_entry, int32_t* info,
                            int32_t n_info);

/* Device workspace needed by tbf_bilateral_trig / tbf_trig_partial for the
 * given shape and term range.  batch_terms <= 0 selects all terms at once. */
TBF_API size_t tbf_workspace_bytes(int32_t B, int32_t H, int32_t W, const tbf_spatial* sp,
                           int32_t term_begin, int32_t term_end, int32_t batch_terms);

/* Full filter: out[b][y][x] for B frames of H x W fp32 samples (row-major,
 * frame-major).  d_counters (device, 2 x uint64, zeroed by the caller):
 * [0] += number of samples outside [-1e-9, T+1e-9] (or non-finite),
 * [1] += number of guarded pixels (den < 1e-12, engines.py:109-117). */
TBF_API int tbf_bilateral_trig(const float* f, float* out, int32_t B, int32_t H, int32_t W,
                       const tbf_spatial* sp, const tbf_terms* terms, int32_t batch_terms,
                       void* workspace, size_t workspace_bytes,
                       unsigned long long* d_counters, void* stream);

/* Host-buffer form of tbf_bilateral_trig: what a reference-side FFI binds
 * with NumPy arrays (replaces engines.py:228-306 end to end, host in, host
 * out).  h_f / h_out are host [B][H][W] fp32 arrays (pinned memory lets the
 * copies overlap the filter; pageable memory works).  d_io is a device
 * buffer of 2*B*H*W floats (input copy, then output); the workspace is sized
 * by tbf_workspace_bytes as for tbf_bilateral_trig.  Column strips of h_f
 * are copied on an internal stream and pass 1 starts on each strip as it
 * lands; the output returns in row bands while later bands filter.  The
 * range check runs on the device copy (d_counters[0], as tbf_range_check).
 * Stream-ordered: h_out is complete and d_counters valid once `stream`
 * reaches this point; h_f and h_out must stay valid until then. */
TBF_API int tbf_bilateral_trig_host(const float* h_f, float* h_out, int32_t B, int32_t H, int32_t W,
                            const tbf_spatial* sp, const tbf_terms* terms, int32_t batch_terms,
                            float* d_io, void* workspace, size_t workspace_bytes,
                            unsigned long long* d_counters, void* stream);

/* Term-sharded piece: num/den[b][y][x] (+)= the contribution of pairs
 * [term_begin, term_end).  accumulate=0 overwrites num/den. */
TBF_API int tbf_trig_partial(const float* f, float* num, float* den, int32_t B, int32_t H, int32_t W,
                     const tbf_spatial* sp, const tbf_terms* terms, int32_t term_begin,
                     int32_t term_end, int32_t batch_terms, int32_t accumulate,
                     void* workspace, size_t workspace_bytes, void* stream);

/* Row-band form of tbf_trig_partial (recursive Gaussian only): the pairs'
 * contribution to rows [row_begin, row_end) of num/den only (other rows are
 * not touched).  row_begin is a multiple of 128, row_end a multiple of 128 or
 * H.  Pass 1 starts its y sweeps a warm-up length outside the band, so the
 * band equals the same rows of a full-image call to the warm-up truncation
 * level (1e-7 relative).  The term-sharded path gives the terms left over
 * after an even split to every rank as one band each (balanced work).
 * Workspace: tbf_workspace_bytes of the whole image. */
TBF_API int tbf_trig_partial_rows(const float* f, float* num, float* den, int32_t B, int32_t H, int32_t W,
                                  const tbf_spatial* sp, const tbf_terms* terms, int32_t term_begin,
                                  int32_t term_end, int32_t row_begin, int32_t row_end, int32_t batch_terms,
                                  int32_t accumulate, void* workspace, size_t workspace_bytes, void* stream);

/* out = num/den where den >= 1e-12, else f; d_counters[1] += guarded count. */
TBF_API int tbf_finalize(const float* num, const float* den, const float* f, float* out, int64_t count,
                 unsigned long long* d_counters, void* stream);

/* d_counters[0] += number of samples outside [-1e-9, T+1e-9] or non-finite. */
TBF_API int tbf_range_check(const float* f, int64_t count, double T, unsigned long long* d_counters,
                    void* stream);

/* Brute-force bilateral filter in fp64 (engines.py:120-151 bilateral_direct):
 * the reference's validation engine, used here to report the trig filter's
 * error against brute-force Gaussian bilateral on every config.  f is
 * [B][H][W] fp32 on the device; taps (device, 2*radius+1 doubles) are the
 * separable window (engines.py:96-106: uniform for box, truncated Gaussian
 * FIR otherwise).  range_kind 0: Gaussian exp(-s^2 / 2 range_param^2);
 * 1: raised cosine cos(range_param * s)^degree (= trig_eval).  samples:
 * NULL for every pixel (out[B*H*W]), else n (b, y, x) int32 triples
 * (out[n]).  Borders reflect as np.pad(mode="reflect"); den < 1e-12 gives
 * the centre sample and counts d_counters[1] (if non-NULL). */
TBF_API int tbf_bilateral_direct(const float* f, int32_t B, int32_t H, int32_t W, const int32_t* samples,
                         int64_t n, const double* taps, int32_t radius, int32_t range_kind,
                         double range_param, int32_t degree, double* out, unsigned long long* d_counters,
                         void* stream);
/* tbf_bilateral_direct on fp64 samples (the reference's Image planes are
 * float64: no quantisation to fp32 before the fp64 brute force). */
TBF_API int tbf_bilateral_direct_f64(const double* f, int32_t B, int32_t H, int32_t W, const int32_t* samples,
                                     int64_t n, const double* taps, int32_t radius, int32_t range_kind,
                                     double range_param, int32_t degree, double* out,
                                     unsigned long long* d_counters, void* stream);

/* Plugin-level twins of the reference's compiled core, fp64 like the
 * reference.  recursive_smooth filters along axis 0 of a[h][w] with `pad`
 * mirrored rows per side and replicate start-up; scratch holds
 * (h + 2*pad + 8) * w doubles.  box_pass filters along the last axis. */
TBF_API int tbf_recursive_smooth_f64(const double* a, double* out, int32_t h, int32_t w, double scale,
                             double c1, double c2, double c3, double c4, int32_t pad,
                             double* scratch, void* stream);
TBF_API int tbf_box_pass_f64(const double* a, double* out, int32_t h, int32_t w, int32_t radius,
                     void* stream);

/* Per-kernel timing for measurement: when enabled, CUDA events are recorded
 * on the launch stream around every kernel; collect synchronizes them and
 * returns summed milliseconds and launch counts per kernel kind (arrays of
 * tbf_profile_kinds() entries, names from tbf_kernel_name), then resets. */
TBF_API int tbf_profile_enable(int32_t on);
TBF_API int32_t tbf_profile_kinds(void);
TBF_API const char* tbf_kernel_name(int32_t kind);
TBF_API int tbf_profile_collect(double* ms, long long* launches, int32_t n);
/* Alternative to collect: the recorded launches in order, start offsets
 * relative to the first one (ms), durations and kinds; returns the count
 * (at most cap) and clears the records.  Host-entry copies are recorded as
 * kinds "h2d" / "d2h". */
TBF_API int32_t tbf_profile_timeline(double* start_ms, double* dur_ms, int32_t* kind, int32_t cap);

/* Process-wide tuning options.
 *   TBF_OPT_PIPELINE (default 0): with several term batches, run pass 1 of
 *     batch k+1 on the caller's stream while the rest of batch k runs on an
 *     internal stream (double-buffered batch workspace, event dependencies).
 *   TBF_OPT_BATCHES (default 2): batches when batch_terms <= 0 and pipelining is on.
 * Options change tbf_workspace_bytes; set them before sizing. */
#define TBF_OPT_PIPELINE 0
#define TBF_OPT_BATCHES 1
#define TBF_OPT_P2_CHUNKS 3 /* default 0 = automatic x-chunks per pass-2 row */
#define TBF_OPT_P1_OCC 4    /* default 3 pass-1 blocks/SM; 2 leaves room for a pass-2 block */
#define TBF_OPT_P1_YCHUNKS 5 /* default 0 = automatic row chunks per pass-1 column */
/* (2 and 10, the round-1 pass-2 variant and pass-1 block-order options, were
 * removed: pass 2 has one variant and pass 1 one block order; tbf_set_option
 * rejects them) */
#define TBF_OPT_HOST_STRIPS 7 /* column strips of tbf_bilateral_trig_host's input copy (0 = auto) */
#define TBF_OPT_HOST_BANDS 8  /* row bands of tbf_bilateral_trig_host's output copy (0 = auto) */
#define TBF_OPT_LPT_SPLIT 11 /* default 1: for launches of a few waves, pass-1 y-chunks and pass-2
                                x-chunks of unequal size, dispatched costliest first, planned by a
                                list-scheduling model; 0 = equal chunks */
#define TBF_OPT_P2_ORDER 9  /* block order of the block-summed pass 2: 0 (default) row fastest, 1 x-chunk fastest, 2/3 reversed */
#define TBF_OPT_ZERO_UNIT 12 /* 1: the zero frequency (even N) as one packed unit whose four lanes
                                are f at four row quarters (a quarter of a term's work and bytes;
                                engines.py:265-271 filters f alone there), on a side stream;
                                default 0 (a full term): measured 1-20% slower end to end */
#define TBF_OPT_P1_CLUSTER 13 /* stripes per pass-1 thread-block cluster (default 1 = none; else the
                                 largest of it, 2, 1 that divides the stripe count): the x hand-off
                                 between a cluster's stripes goes through distributed shared memory
                                 and mbarriers (bit-identical; measured 2-6% slower) */
#define TBF_OPT_P1_FOLD 6   /* default 1: folds the y-sweep gain into the pass-2 weights
                               (skips 4 multiplies per pixel-term in pass 1 when T/g^4 is safe); 0 scales in pass 1 */
TBF_API int tbf_set_option(int32_t option, int64_t value);

/* Last error message of the calling thread (static storage). */
TBF_API const char* tbf_last_error(void);
/* ABI version (bumped on any signature change). */
TBF_API int32_t tbf_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* TRIGBF_B200_H */
