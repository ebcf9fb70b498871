/*
 * hos.h — C-ABI of the B200 direct-method HOS estimator (libhos_b200.so).
 *
 * Plain pointers and sizes only; no torch or CUDA types in the signatures
 * (streams travel as void*, i.e. a cudaStream_t; NULL = legacy stream).
 *
 * The reference (hospectra 0.1.0) is pure Python, so "the interface each
 * entry point replaces" is the Python function named beside it
 * (paths relative to /root/reference/pkg/src/hospectra/):
 *
 *   hos_estimate               estimate_spectrum            spectra.py:434-439
 *                              (segment_and_demean series.py:159-165,
 *                               dft_segments dft.py:36-41,
 *                               _compute_values spectra.py:391-416)
 *   hos_estimate_from_spectra  estimate_from_spectra        spectra.py:419-431
 *   hos_segment_spectra        dft_segments∘segment_and_demean
 *                                                           dft.py:36-41, series.py:159-165
 *   hos_domain_size/indices    principal_domain / domain_slice
 *                                                           spectra.py:133-196
 *   hos_partial_raw +          parallel_estimate's worker split
 *   hos_smooth_raw               (_worker_run + _compute_values on a slice)
 *                                                           parallel.py:94-162
 *   hos_last_error             the ParameterError / DataError messages
 *                                                           errors.py:4-9
 *
 * Error convention: every int-returning call returns HOS_OK (0) or one of
 * HOS_EPARAM (-> ParameterError), HOS_EDATA (-> DataError), HOS_ECUDA /
 * HOS_ENOMEM (-> RuntimeError); hos_last_error() returns the thread-local
 * message of the last failure, keeping the reference's message fragments
 * ("m3 < m/2", "k*m = ... exceeds series length n = ...").
 *
 * Numerics: precision 32 computes FFT + products in fp32 (FFMA2), combines
 * segment-chunk partial sums and smooths in fp64, and writes complex64;
 * precision 64 is fp64 end to end and writes complex128.
 *
 * Ownership: the caller owns every input/output buffer; a plan owns its
 * cuFFT plan, scratch and geometry tables, all allocated at create time so
 * hos_estimate* never allocate (stream-ordered, CUDA-graph capturable).
 * Calls on one plan are serialised by a per-plan lock and run on the
 * plan's device whatever device the calling thread has selected.
 */
#ifndef HOS_B200_H
#define HOS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HOS_OK 0
#define HOS_EPARAM 1
#define HOS_EDATA 2
#define HOS_ECUDA 3
#define HOS_ENOMEM 4

/* element types */
#define HOS_F32 0
#define HOS_F64 1
#define HOS_C64 2
#define HOS_C128 3

/* tapers */
#define HOS_TAPER_NONE 0
#define HOS_TAPER_HANN 1 /* periodic Hann 0.5-0.5cos(2 pi u/M), applied after demeaning */

typedef struct hos_plan hos_plan;

/* Library identification, e.g. "hos_b200 0.1.0 sm_100a". */
const char* hos_version(void);

/* Thread-local message of the last failed call ("" if none). */
const char* hos_last_error(void);

/* ---- principal domain (host-side, no GPU) -------------------------------
 * spectra.py:133-196.  Order 3: 0<=k2<=k1, k1+k2<m/2.  Order 4:
 * 0<=k3<=k2<=k1, k1+k2+k3<m/2.  Lexicographic order. */
int64_t hos_domain_size(int order, int m);
/* out: (stop-start) x (order-1) int32, the rows [start, stop) of the domain. */
int hos_domain_indices(int order, int m, int64_t start, int64_t stop, int32_t* out);

/* ---- plans ----------------------------------------------------------------
 * order 3|4; segment length m >= 2; segments k >= 1; window m3 >= 1 with
 * 2*m3 < m (spectra.py:70-79); conjugate_last 0|1; precision 32|64;
 * taper HOS_TAPER_*; batch = independent series per call (>= 1);
 * device = CUDA ordinal the plan's memory lives on. */
int hos_plan_create(hos_plan** plan, int order, int m, int k, int m3, int conjugate_last,
                    int precision, int taper, int batch, int device);
void hos_plan_destroy(hos_plan* plan);

/* Principal-domain points per series (= hos_domain_size(order, m)). */
int64_t hos_plan_npoints(const hos_plan* plan);
/* Raw cells of the dilated domain D_h per series (the smoothing support). */
int64_t hos_plan_cells(const hos_plan* plan);
/* Metric units per series: K * |D_h| segment.bin products. */
int64_t hos_plan_units(const hos_plan* plan);
/* Triple-product work per series actually issued by the kernel (cells incl.
 * tile padding) times K; units/issued is the tiling efficiency. */
int64_t hos_plan_issued(const hos_plan* plan);
/* Elements per row of the staged segment spectra E (the frequency window
 * [f_lo, f_hi] the triple product reads): the front end writes K rows of
 * this many complex values per series. */
int64_t hos_plan_row_len(const hos_plan* plan);
/* Device bytes the plan holds. */
size_t hos_plan_device_bytes(const hos_plan* plan);
/* Number of this library's kernels one hos_estimate launches: 4 with the fused
 * front end (power-of-two m), else 5 plus cuFFT's own kernels. */
int hos_plan_launches(const hos_plan* plan);

/* ---- the hot path -----------------------------------------------------------
 * x_dev: batch series, series b starting at x_dev + b*x_stride elements,
 *   each with at least k*m samples (extra samples are ignored, as in
 *   series.py:163); x_dtype HOS_F32 | HOS_F64.
 * out_dev: batch x npoints complex values (HOS_C64 for precision 32,
 *   HOS_C128 for precision 64), lexicographic principal-domain order. */
int hos_estimate(hos_plan* plan, const void* x_dev, int x_dtype, int64_t x_stride,
                 void* out_dev, void* stream);

/* spec_dev: batch x k x m full complex spectra (spec_dtype HOS_C64|HOS_C128),
 * arbitrary complex values (not required to be conjugate-symmetric). */
int hos_estimate_from_spectra(hos_plan* plan, const void* spec_dev, int spec_dtype,
                              void* out_dev, void* stream);

/* Segment, demean (, taper) and transform: spec_dev receives batch x k x m
 * full complex spectra (HOS_C64 for precision 32, HOS_C128 for 64). */
int hos_segment_spectra(hos_plan* plan, const void* x_dev, int x_dtype, int64_t x_stride,
                        void* spec_dev, void* stream);

/* Plain batched DFT of `rows` real rows of length m (no demeaning): the
 * reference's dft_segments on an already-demeaned SegmentSet (dft.py:36-41).
 * spec_dev receives rows x m full complex spectra (HOS_C64 for precision 32,
 * HOS_C128 for 64).  cuFFT plans are cached per (m, rows, precision). */
int hos_dft_rows(const void* x_dev, int x_dtype, int rows, int m, int precision, void* spec_dev,
                 void* stream);

/* End to end with HOST buffers, synchronous.  Page-locked buffers: the
 * values are written in place over PCIe by the smoothing kernel, and the
 * series is read in place by the front end (zero-copy; the default) or, with
 * HOS_CHUNKS=n set at plan creation (single-series plans whose k splits into
 * n chunks), copied chunk by chunk by the copy engine while the previous
 * chunk's front end and triple product run; replayed as one CUDA graph per
 * buffer binding -- the buffers must stay
 * allocated and page-locked while the plan may reuse the binding.  Pageable
 * buffers are staged with copies.  stream NULL = the plan's private stream. */
int hos_estimate_host(hos_plan* plan, const void* x_host, int x_dtype, int64_t x_stride,
                      void* out_host, void* stream);

/* ---- multi-GPU building blocks (segment sharding) -------------------------
 * Raw sums live in a CSR "line" layout over D_h: order 3 one line per raw
 * row a = lo..; order 4 one line per raw pair (a,b).  line_start has
 * nlines+1 entries (cells), point_line gives, for each output row k1
 * (order 3) or pair (k1,k2) (order 4), the first line its window touches. */
int64_t hos_plan_lines(const hos_plan* plan);
int hos_plan_line_starts(const hos_plan* plan, int64_t* line_start /* nlines+1 */);

/* Unscaled raw sums over segments [seg_begin, seg_end) of the (single)
 * series: raw_dev receives cells values (c64 for precision 32, c128 for 64). */
int hos_partial_raw(hos_plan* plan, const void* x_dev, int x_dtype, int seg_begin, int seg_end,
                    void* raw_dev, void* stream);

/* Smooth output rows [row_begin, row_end) (order 3: k1 rows; order 4: k1
 * planes) from raw sums summed over ALL k segments.  raw_dev holds the
 * cells of lines [line_begin, ...) (line_begin = the first line those rows
 * need, i.e. row_begin for order 3), out_dev receives the lexicographic
 * points of those rows (first point = domain offset of row_begin). */
int hos_smooth_raw(hos_plan* plan, const void* raw_dev, int64_t line_begin, int row_begin,
                   int row_end, void* out_dev, void* stream);
/* Lexicographic offset of the first point of output row (k1) `row`. */
int64_t hos_row_point_offset(const hos_plan* plan, int row);
/* First line (inclusive) and last line (exclusive) needed by rows [r0,r1). */
int hos_rows_line_range(const hos_plan* plan, int row_begin, int row_end, int64_t* line_begin,
                        int64_t* line_end);

/* ---- measurement helpers ----------------------------------------------------
 * FP32 pipe peak (FFMA2 outer-product microbenchmark, flops counted as 2 per
 * lane FMA) and the SM clock seen meanwhile, on the current device. */
int hos_peak_fp32(double* tflops, double* sm_mhz, void* stream);
/* FP64 pipe peak (DFMA chains, 2 flops per FMA) and the SM clock seen meanwhile. */
int hos_peak_fp64(double* tflops, double* sm_mhz, void* stream);
/* Mean duration (ms) of the triple-product kernel launches of the last
 * hos_estimate* call on this plan when timing was enabled (events recorded on
 * the launching stream). */
int hos_plan_set_timing(hos_plan* plan, int enable);
/* In-step kernel timing: stamps_dev = a zeroed device buffer of 16 x 192
 * uint64 (NULL: off) on the plan's device.  While set, every pipeline kernel
 * of every plan on that device records, per SM, ~(globaltimer at its first
 * CTA's start on that SM, after its PDL wait) into [2 kind][sm] and the
 * globaltimer of its last warp's end there into [2 kind + 1][sm] (atomicMax);
 * kind = 0 front end, 1 prep, 2 extend, 3 triple product, 4 line scan, 5 box,
 * 6 per-series smoothing, 7 slot reduction.  The caller zeroes the buffer
 * between calls and reduces over SMs.  Works under graph replay. */
int hos_plan_set_stamps(hos_plan* plan, void* stamps_dev);
/* ---- multi-GPU ----------------------------------------------
 * One process (or thread) per GPU.  The caller creates an NCCL communicator
 * (ncclCommInitRank; libnccl.so.2 is resolved at attach time, no link-time
 * dependency) and attaches it to a batch-1 plan on that rank's device.
 * hos_estimate_distributed then runs the segment-sharded estimate of ONE
 * series: every rank passes the full series (device memory, it reads only its
 * own segments), computes partial raw sums over D_h for its segment shard,
 * the partials are reduce-scattered by line blocks (ncclReduceScatter), the
 * halo lines are exchanged (ncclAllGather), each rank smooths its own output
 * rows and the lexicographic slices are all-gathered: out_dev receives the
 * full grid on every rank.  Replaces the reference's process fan-out
 * (hospectra/parallel.py:120-162) with a GPU-per-rank split of the K-sum. */
int hos_comm_attach(hos_plan* plan, void* nccl_comm, int rank, int nranks);
int hos_estimate_distributed(hos_plan* plan, const void* x_dev, int x_dtype, void* out_dev, void* stream);
/* The sharded layout (host only, no device): per rank {seg0, seg1, row0,
 * row1, own_l0, own_l1, need_l0, need_l1, own_c0, own_c1, need_c0, need_c1,
 * p0, p1}, then {block, halo, halo_in_next}: 14 * nranks + 3 int64. */
int hos_shard_layout(int order, int m, int k, int m3, int nranks, int64_t* out);

/* Host-only check of the k_triple_cta schedule a plan of this shape would
 * use on a GPU with `sms` SMs (interleave != 0: the streaming host path's
 * schedule): every (series, region group, segment) covered exactly once,
 * stages inside their block's series, warp roles within the CTA, partial
 * slot bases consecutive and counted.  No device needed.  stats (12 int64):
 * {ctas, stages, max stages per CTA, min, max slots, tile step, ring depth,
 * groups, regions, blocks, segments per stage, slot bytes}; ctas = 0: the plan would not
 * use k_triple_cta.  Returns HOS_EDATA with the failed property. */
int hos_cta_schedule_check(int order, int m, int k, int m3, int precision, int batch, int sms, int interleave,
                           int64_t* stats);
/* Diagnostics: K2 CTAs per series (4 warps each) of the per-warp staged kernel. */
int hos_plan_nctas(const hos_plan* plan);
/* Diagnostics: which K2 the plan's full estimate launches: 1 = k_triple_cta
 * (CTA-shared bulk-copied rows, one CTA per SM), 0 = k_triple_w (per-warp
 * cp.async staging; also every segment-range launch of hos_partial_raw). */
int hos_plan_k2_kind(const hos_plan* plan);
/* Diagnostics: a device buffer of 4 x (4 nctas) x batch uint64 that K2 fills
 * per warp with {start, first staged data, end (globaltimer ns), smid};
 * NULL disables.  Traced calls run without graph replay. */
int hos_plan_set_trace(hos_plan* plan, void* trace_dev);
/* Diagnostics: mean per-launch device time (ms) of each stage {prep, fft,
 * extend, triple, scan, box}: `reps` launches of the stage captured into one
 * CUDA graph, replayed between two events on `stream` after one full estimate
 * of x_dev (same arguments as hos_estimate).  Resolves sub-microsecond changes
 * that single event pairs (~1 us granularity) cannot; with the fused front
 * end (power-of-two m) "prep" is the fused kernel and fft/extend read 0. */
int hos_plan_time_stages(hos_plan* plan, const void* x_dev, int x_dtype, int64_t x_stride, void* out_dev, int reps,
                         double* ms6, void* stream);
int hos_plan_kernel_ms(const hos_plan* plan, double* triple_ms, double* total_ms);
/* Per-stage durations (ms) of the last timed call: prep, FFT, extend,
 * triple product, line scan, box (6 values; the triple product includes
 * the PDL-overlapped prologue). */
int hos_plan_stage_ms(const hos_plan* plan, double* ms6);

#ifdef __cplusplus
}
#endif
#endif /* HOS_B200_H */
