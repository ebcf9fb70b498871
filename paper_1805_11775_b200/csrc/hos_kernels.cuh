// sm_100a kernels of the direct-method HOS hot path.
//
//   K0 prep     segment + demean (+ Hann) + cast        hospectra/series.py:159-165
//   (cuFFT)     batched R2C / D2Z per segment            hospectra/dft.py:36-41
//   K0+1 front  fused segment + demean + taper + shared-memory FFT + extension (power-of-two m)
//   K1 extend   conjugate-symmetric extension of the half spectrum onto the
//               frequency window [f_lo, f_hi] the triple product reads
//   K2 triple   R(line, c) = sum_i F_i(row) F_i(c) G_i(row + c [+ a])  over D_h,
//               per segment chunk (hospectra/spectra.py:227-263)
//   K4a scan    per-line prefix sums of the chunk-summed raw cells (fp64,
//               warp shuffles)                           hospectra/tiled.py:36-47
//   K4b box     window sums as prefix differences, scale 1/(M K w^(d)), write
//               lexicographic principal-domain values   hospectra/spectra.py:405-415
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <vector>

#include "hos_geometry.h"

namespace hos {

// ---------------------------------------------------------------------------
// packed fp32x2 arithmetic (sm_100a FFMA2 / FMUL2).  Non-volatile asm so
// ptxas can interleave independent cells; broadcast (make_float2(s, s)) and
// swapped (make_float2(v.y, v.x)) operands compile to operand swizzles.

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long ra = *reinterpret_cast<unsigned long long*>(&a);
  unsigned long long rb = *reinterpret_cast<unsigned long long*>(&b);
  unsigned long long rc = *reinterpret_cast<unsigned long long*>(&c);
  unsigned long long rd;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rd) : "l"(ra), "l"(rb), "l"(rc));
  return *reinterpret_cast<float2*>(&rd);
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  unsigned long long ra = *reinterpret_cast<unsigned long long*>(&a);
  unsigned long long rb = *reinterpret_cast<unsigned long long*>(&b);
  unsigned long long rd;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(rd) : "l"(ra), "l"(rb));
  return *reinterpret_cast<float2*>(&rd);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// ---------------------------------------------------------------------------
// launch wrappers (hos_kernels.cu)

// K2's static split of W (region, segment) units over Nw warps: the first H
// warps weigh wa, the rest wb (wa == wb: equal contiguous ranges).  The
// hardware favours the older of the two CTAs on an SM (measured: 25.9 vs
// 35.1 us for equal work, tools/k2_trace.py), so giving the first wave of
// CTAs more units makes both finish together.  Fixed by the launch shape, so
// partial-slot numbering and results stay deterministic.
struct WarpSplit {
  int64_t W, Nw, H;
  int wa, wb;
  HOS_HD int64_t cum(int64_t g) const { return wa * (g < H ? g : H) + wb * (g > H ? g - H : 0); }
  HOS_HD int64_t begin(int64_t g) const { return W * cum(g) / cum(Nw); }
  // the warp whose range holds unit u (the last one when ranges coincide)
  HOS_HD int64_t warp_of(int64_t u) const {
    const int64_t X = ((u + 1) * cum(Nw) - 1) / W;
    const int64_t g = X < wa * H ? X / wa : H + (X - wa * H) / wb;
    return g < Nw - 1 ? g : Nw - 1;
  }
  // partial slots of region r (warps whose range touches it)
  HOS_HD int region_slots(int r, int nseg) const {
    return (int)(warp_of((int64_t)(r + 1) * nseg - 1) - warp_of((int64_t)r * nseg) + 1);
  }
};

struct TripleArgs {
  const void* E;              // [series][K][Lp] float2 (fp32) / double2 (fp64) spectrum elements
  int Lp;                     // row pitch in elements (even: rows stay 16-byte aligned)
  int f_lo;                   // frequency of element 0
  int K;                      // segments per series (E rows per series)
  int seg_begin, seg_end;     // segment range reduced by this launch
  const Tile* tiles;          // [nregions][tiles_per_region] D_h tiles (4S lines x 8S columns)
  int nregions;
  int tile_step;              // lane step S (2 or 4): tiles_per_region = 32 / S^2
  int64_t nwarps;             // warps splitting the region x segment work (<= units)
  int split_wa, split_wb;     // WarpSplit weights (first half / second half of the warps)
  const int32_t* line_cmax;
  const int64_t* line_start;
  int lo;
  void* part;                 // [series][maxslots][ncells] float2 / double2
  int64_t ncells;
  int maxslots;
  int order;
  int conj;
  int batch;
  int accumulate;             // add into the partial slots (chunked launches after the first)
  unsigned long long* trace;  // diagnostics (nullptr: off): per warp {start, first data, end, smid} globaltimer ns
};

#ifndef HOS_K2_WARPS
#define HOS_K2_WARPS 4
#endif
constexpr int kTripleWarps = HOS_K2_WARPS;  // warps per CTA of the triple-product kernel

// Where the partial slots of a K2 launch are (for the K4a / reduce readers).
struct SlotInfo {
  const int32_t* line_tile0;    // nullptr: plain buffer with `nparts` parts
  int nseg;
  int nregions;
  int tile_cols, tiles_per_region;  // Geometry tile shape (tile -> region map)
  int64_t nwarps;
  int split_wa, split_wb;
  const int32_t* region_slots;  // optional host-precomputed slots per region (same values), nullptr: compute
  int64_t rs_stride;            // region_slots entries per series (0: one table for every series)
};

// K2 (CTA-staged, k_triple_cta): host-built schedule.  A GROUP is up to
// kCtaWarps consecutive regions; with n < kCtaWarps regions each region gets
// `halves` x `phases` warps: with halves = 2 each warp computes one of the
// region's two tiles, and each warp takes every phases-th stage.  A BLOCK is one CTA's
// segment range of one (series, group); its warps write partial slots
// slot_base + phase.  A STAGE is up to 4 consecutive E rows of one block.
constexpr int kCtaWarps = 8;    // float2 / double2 rows, ~252-register cells
constexpr int kCtaWarpsQ = 16;  // fp32 quad rows (HOS_K2_QUAD=1), <= 128-register cells
inline int cta_warps(int quad) { return quad ? kCtaWarpsQ : kCtaWarps; }
constexpr int kCtaMaxDepth = 8;
constexpr size_t kCtaMaxSmem = 220 * 1024;    // the staging ring
constexpr size_t kCtaSmemLimit = 226 * 1024;  // ring + the CTA's stage / block tables (+ static smem <= 227 KB)
struct CtaGroup {
  int32_t r0, n, phases;
  int32_t halves;     // 2: a region's two tiles go to different warps (n <= kCtaWarps / 2)
};
struct CtaBlock {
  int32_t row0;       // E row of the block's first segment (series * K + seg)
  int32_t series;
  int32_t group;
  int32_t slot_base;
};
struct CtaStage {
  int32_t row;        // E row of the stage's first segment
  int32_t nseg;       // 1..4
  int32_t block;
  int32_t pad;
};
struct CtaTripleArgs {
  const void* E;
  int Lp, f_lo;
  const Tile* tiles;
  int tile_step;
  const CtaGroup* groups;
  const CtaBlock* blocks;
  const CtaStage* stages;
  const int32_t* cta_stage0;  // nctas + 1
  int nctas;
  int depth;                  // ring slots
  int stage_segs;             // segments per full stage (block stages start every stage_segs segments)
  int slot_bytes;             // per ring slot (copy A, copy B)
  int copy_b;                 // byte offset of copy B in a slot (== 64 mod 128)
  const int32_t* line_cmax;
  const int64_t* line_start;
  int lo;
  void* part;
  int64_t ncells;
  int maxslots;
  int order, conj;
  unsigned long long* trace;  // diagnostics (nullptr: off): per warp {start, first data, end, smid}
  int trace_cta;              // diagnostics: CTA whose per-stage times are traced
  int quad;                   // fp32: E rows hold quads {re, im, im, im} (cells_q, 16 warps)
  int refill_last;            // 1: the warp completing a stage's count refills it; 0: warp 0 waits on empty[]
  int skew_cycles;            // > 0: the second warp of every SM sub-partition starts its first stage this much later
  const int4* cta_head;       // per CTA {first stage, stages, first block, blocks} (one load)
  int tab_stages;             // stage-table entries reserved in shared memory (>= stages of any CTA)
  int tab_blocks;             // block-table entries reserved in shared memory (>= blocks of any CTA)
  const int* ready;           // nullptr, or per E row: 1 once a concurrently running front end wrote it
  int* err;                   // streaming: set to 1 (host-mapped word) when a ready wait timed out
  int row_shift;              // added to every stage's E row (chunked host path: the chunk's first segment)
  int accumulate;             // 1: add the block sums into the partial slots (later chunks), 0: store them
};
// in-step kernel timing slots (hos_plan_set_stamps): [kind][~first start | last end][SM]
enum StampKind { kStampFront = 0, kStampPrep, kStampExtend, kStampTriple, kStampScan, kStampBox, kStampSeries,
                 kStampReduce, kStampKinds };
constexpr unsigned kStampSms = 192;  // SM slots per (kind, start|end)
cudaError_t set_stamp_buffer(unsigned long long* dev_buf);  // on the current device; nullptr: off

cudaError_t launch_triple_cta(const CtaTripleArgs& a, int precision, cudaStream_t st);

// occupancy (CTAs / SM) of the triple-product kernel
int triple_occupancy(int precision, int tile_step);

cudaError_t launch_prep(const void* x, int x_dtype, int64_t x_stride, int m, int seg_begin, int nseg,
                        int batch, int taper, const double* taper_tab, int precision, void* seg_out,
                        cudaStream_t st);
// fused K0 + FFT + K1 for power-of-two m <= kFrontMaxM (tw: m twiddles exp(-2 pi i t/m) in the
// compute precision); returns cudaErrorInvalidValue for other m
constexpr int kFrontMaxM = 4096;
// x: first segment of series 0 (series b at x + b*x_stride); segment s of series b -> E row b*krows + s
// ready != nullptr: streaming launch (a PDL dependent of the consuming K2), publishing
// ready[b*krows + s] = 1 with release semantics once E row s is written
constexpr int kStreamFrontCtas = 20;  // SMs left to the streaming front end (K2 runs on the rest)
// quad != 0 (fp32 only): E elements are quads {re, im, im, im} (16 bytes) for k_triple_cta
cudaError_t launch_front(const void* x, int x_dtype, int64_t x_stride, int m, int nseg, int krows, int batch,
                         int taper, const double* taper_tab, const void* tw, int precision, int f_lo, int L, int Lp,
                         void* E, cudaStream_t st, int quad, int* ready = nullptr);
cudaError_t launch_extend_half(const void* H, int m, int hstride, int rows, const void* /*unused*/,
                               int f_lo, int L, int Lp, int precision, void* E, cudaStream_t st, int quad);
cudaError_t launch_extend_full(const void* S, int spec_dtype, int m, int rows, int f_lo, int L, int Lp,
                               int precision, void* E, cudaStream_t st, int quad);
cudaError_t launch_expand_full(const void* H, int m, int hstride, int rows, int precision, void* out,
                               cudaStream_t st);
cudaError_t launch_triple(const TripleArgs& a, int precision, cudaStream_t st);
// max_line: longest line (cells) of the range -- short lines get one warp per line
cudaError_t launch_line_scan(const void* part, int nparts, int64_t part_stride, const SlotInfo& si, int precision,
                             const int64_t* line_start, int64_t line_begin, int64_t nlines,
                             int64_t ncells_series, int batch, double* S, cudaStream_t st, int max_line);
struct BoxArgs {
  const double* S;          // prefix sums [series][ncells] (cells of lines from line_base)
  int64_t s_series_stride;
  int64_t line_base;        // line index of S's first line
  const int64_t* line_start;
  int64_t cell_base;        // line_start[line_base]
  const int64_t* row_off;   // order 3: lexicographic offset per k1 row (rows+1)
  int rows;
  const int32_t* pair_k1;   // order 4 pair table
  const int32_t* pair_k2;
  const int64_t* pair_base;
  int npairs;
  const int32_t* line_of_ab;
  int b_count;
  int lo, hi, m3, order, m;
  int row_begin, row_end;   // order 3: output rows k1 written
  int pair_begin, pair_end; // order 4: pairs written
  int64_t p_begin, p_end;   // lexicographic point range written (out[0] = point p_begin)
  double scale;
  void* out;                // [series][..] values for points [p_begin, p_end)
  int64_t out_series_stride;
  int precision;
  int batch;
};
cudaError_t launch_box(const BoxArgs& a, cudaStream_t st);
// K4a + K4b for a small order-3 grid, one CTA per series with the whole grid
// in shared memory (smooth_series3_smem bytes; the caller checks it fits)
size_t smooth_series3_smem(int64_t ncells, int64_t nlines, int rows, int nregions, int64_t npoints);
cudaError_t launch_smooth_series3(const void* part, int nparts, int64_t part_stride, const SlotInfo& si, int precision,
                                  const BoxArgs& a, int64_t nlines, cudaStream_t st);
// separable variant (default for small order-3 grids, W in 3/5/7/9): vertical
// then horizontal direct window sums in the compute precision
size_t smooth_series_sep_smem(int64_t ncells, int64_t nlines, int rows, int nregions, int64_t npoints, int w,
                              int64_t nvitems, int64_t nhitems, int precision);
void smooth_series_sep_items(const int64_t* row_off, int rows, int w, int64_t* nvitems, int64_t* nhitems);
bool smooth_series_sep_supports(int w);
cudaError_t launch_smooth_series_sep(const void* part, int nparts, int64_t part_stride, const SlotInfo& si,
                                     int precision, const BoxArgs& a, int64_t nlines, int64_t nvitems,
                                     int64_t nhitems, const int* series_slots, cudaStream_t st);
// pipelined separable variant (default when its shared memory fits): the
// series' raw cells land by one bulk copy while the previous series' outputs
// are formed
struct PipeLayout {  // shared-memory layout (byte offsets) and item counts
  size_t R, V, tabs, rowrec, vb, vrow, hrow, rsl, bar, total;
  int table_bytes;  // [tabs, tabs + table_bytes): the host-built table image
  int ltab;         // ints per vertical block record
  int vtot, nvitems, nhitems;
};
struct PipePlan {
  PipeLayout L;
  std::vector<unsigned char> tables;
};
// L.total == ~0: the grid does not qualify
PipePlan smooth_series_pipe_plan(const int64_t* row_off, int rows, const int64_t* line_start, int64_t nlines,
                                 int64_t ncells, int nregions, int w, int precision);
cudaError_t launch_smooth_series_pipe(const void* part, int nparts, int64_t part_stride, const SlotInfo& si,
                                      int precision, const BoxArgs& a, const PipeLayout& L, const void* tables,
                                      const unsigned short* cell_region, const int* series_slots, cudaStream_t st);
// separable K4 for order-3 grids that do not fit one CTA (cfg2, cfg3): slot sums
// into R (compute precision), then kTR x kTC output tiles of direct window sums
bool box_tiles_supports(int w);
std::vector<int32_t> box_tile_list(const int64_t* row_off, int rows);
// region of every cell (the K2 region whose slots hold it), for k_raw_cells
std::vector<uint16_t> cell_region_table(const int32_t* line_tile0, const int64_t* line_start, int64_t nlines,
                                        int tile_cols, int tiles_per_region);
cudaError_t launch_raw_cells(const void* part, int nparts, int64_t part_stride, const int32_t* region_slots,
                             int64_t rs_stride, const unsigned short* cell_region, int64_t ncells, int batch,
                             int precision, void* R, cudaStream_t st);
cudaError_t launch_box_tiles(const void* R, int64_t ncells, int precision, const BoxArgs& a, int nlines,
                             const int* tiles, int ntiles, cudaStream_t st);
// raw[c] = sum_p part[p][c] (fp64 sum, stored in the compute precision)
// dst_line (optional): per line, the output index of its first cell (else raw[c]);
// dst_addr (optional, wins): per line, the address (possibly a peer GPU's) of its first cell
cudaError_t launch_reduce_parts(const void* part, int64_t part_stride, const SlotInfo& si, const int64_t* line_start,
                                int64_t nlines, int lo, int precision, void* raw, cudaStream_t st,
                                const int64_t* dst_line = nullptr, const unsigned long long* dst_addr = nullptr);
// out[i] = sum_{r < nranks} land[r * block + i], i < count (fp64, rank order)
cudaError_t launch_sum_land(const void* land, int nranks, int64_t block, int64_t count, int precision, void* out,
                            cudaStream_t st);
cudaError_t launch_cast(const void* x, int x_dtype, int64_t n, int precision, void* out, cudaStream_t st);
cudaError_t launch_peak_fp32(float2* buf, int blocks, int iters, cudaStream_t st);
cudaError_t launch_peak_fp64(double* buf, int blocks, int iters, cudaStream_t st);
cudaError_t launch_clock_probe(unsigned long long* out, long long spin, cudaStream_t st);

}  // namespace hos
