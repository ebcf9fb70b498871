// C-ABI of libhos_b200 (include/hos.h): plan lifetime, orchestration of
// K0 -> cuFFT -> K1 -> K2 -> K4a -> K4b on one stream, error mapping.
#include <cuda_runtime.h>
#include <cufft.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <string>
#include <vector>

#include "../../include/hos.h"
#include "hos_geometry.h"
#include "hos_kernels.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(expr)                                                                           \
  do {                                                                                           \
    cudaError_t e_ = (expr);                                                                     \
    if (e_ != cudaSuccess)                                                                       \
      return fail(e_ == cudaErrorMemoryAllocation ? HOS_ENOMEM : HOS_ECUDA,                      \
                  std::string("CUDA error in ") + #expr + ": " + cudaGetErrorString(e_));        \
  } while (0)

#define CUFFT_TRY(expr)                                                                         \
  do {                                                                                          \
    cufftResult r_ = (expr);                                                                    \
    if (r_ != CUFFT_SUCCESS) return fail(HOS_ECUDA, std::string("cuFFT error ") +              \
                                                        std::to_string((int)r_) + " in " + #expr); \
  } while (0)

}  // namespace

struct hos_plan {
  int order = 3, m = 0, k = 0, m3 = 1, conj = 1, precision = 32, taper = 0, batch = 1, device = 0;
  hos::Geometry geo;
  int nctas = 1;      // K2 CTAs per series (full-K launch); warps = 4 x nctas
  int maxslots = 1;   // partial slots allocated per series
  int occupancy = 1;  // K2 CTAs per SM
  int sms = 148;
  int max_line = 0;  // longest D_h line (cells)
  bool series_k4 = false;  // K4 as one CTA per series with the grid in shared memory
  bool sep_k4 = false;     // ... as separable direct window sums (k_smooth_series_sep; else prefix sums)
  int64_t sep_vitems = 0, sep_hitems = 0;  // k_smooth_series_sep work items
  bool pipe_k4 = false;    // ... pipelined (k_smooth_series_pipe: bulk-copied raw cells, conflict-free passes)
  hos::PipeLayout pipe_layout{};
  unsigned char* d_pipe_tables = nullptr;
  // separable K4 of order-3 grids (k_raw_cells + k_box_tiles) instead of line scans + prefix differences
  bool tiles_k4 = false;
  int box_ntiles = 0;
  int32_t* d_box_tiles = nullptr;
  uint16_t* d_cell_region = nullptr;  // region of every cell (k_raw_cells' slot counts)
  int32_t* d_series_slots = nullptr;    // per series: most partial slots of any region (main launch)
  int32_t* d_s_series_slots = nullptr;  // ... of the streaming schedule
  int split_wa = 1, split_wb = 1;  // K2 WarpSplit weights for two-CTA-per-SM launches
  // K2 as k_triple_cta (CTA-staged full rows, host schedule) for the plan's main launch
  bool cta = false;
  bool quad = false;  // fp32 k_triple_cta plan: E rows hold quads {re, im, im, im} (16 bytes)
  int cta_warps = 8;  // warps per k_triple_cta CTA (16 for fp32, 8 for fp64)
  int cta_nctas = 0, cta_depth = 0, cta_stage_segs = 4, cta_slot_bytes = 0, cta_copy_b = 0;
  int cta_tab_stages = 0, cta_tab_blocks = 0, s_tab_stages = 0, s_tab_blocks = 0;
  hos::CtaGroup* d_groups = nullptr;
  hos::CtaBlock* d_blocks = nullptr;
  hos::CtaStage* d_stages = nullptr;
  int32_t* d_cta_stage0 = nullptr;
  int4* d_cta_head = nullptr;    // per CTA {first stage, stages, first block, blocks}
  int4* d_s_cta_head = nullptr;  // ... of the streaming schedule
  int64_t rs_stride = 0;  // d_region_slots entries per series
  // streaming host path (hos_estimate_host, zero-copy): the front end runs on
  // kStreamFrontCtas SMs reading the series over PCIe while k_triple_cta (an
  // interleaved schedule on the other SMs) consumes rows as they are published
  bool stream_ok = false;
  int s_nctas = 0, s_maxslots = 1;
  hos::CtaBlock* d_s_blocks = nullptr;
  hos::CtaStage* d_s_stages = nullptr;
  int32_t* d_s_cta_stage0 = nullptr;
  int32_t* d_s_region_slots = nullptr;
  int* d_ready = nullptr;
  cudaStream_t side = nullptr;
  cudaEvent_t e_fork = nullptr, e_join = nullptr;
  // chunked host path (hos_estimate_host, page-locked buffers): the series
  // crosses PCIe in `chunks` copy-engine transfers of chunk_k segments on
  // c_copy while the front end and a k_triple_cta launch per chunk (one
  // schedule of chunk_k segments, its E rows shifted per chunk) add each
  // chunk's products into the same partial slots
  int chunks = 0, chunk_k = 0;
  int c_nctas = 0, c_tab_stages = 0, c_tab_blocks = 0;
  hos::CtaBlock* d_c_blocks = nullptr;
  hos::CtaStage* d_c_stages = nullptr;
  int32_t* d_c_cta_stage0 = nullptr;
  int4* d_c_cta_head = nullptr;
  int32_t* d_c_region_slots = nullptr;
  cudaStream_t c_copy = nullptr;
  std::vector<cudaEvent_t> c_ev;  // chunk i landed (c_ev[chunks]: fork)
  int hstride = 0;   // complex elements per half-spectrum row
  int L = 0, Lp = 0; // extended-spectrum length / pitch (complex elements)
  // device tables
  hos::Tile* d_tiles = nullptr;
  int32_t* d_line_tile0 = nullptr;
  int32_t* d_region_slots = nullptr;  // slots per region of the full-K launch (K4 lookups)
  int32_t* d_line_cmax = nullptr;
  int64_t* d_line_start = nullptr;
  int64_t* d_row_off = nullptr;
  int32_t* d_pair_k1 = nullptr;
  int32_t* d_pair_k2 = nullptr;
  int64_t* d_pair_base = nullptr;
  int32_t* d_line_of_ab = nullptr;
  double* d_taper = nullptr;
  void* d_tw = nullptr;     // fused front end: m twiddles exp(-2 pi i t/m), compute precision
  bool fused = false;       // K0+FFT+K1 as one kernel (power-of-two m <= hos::kFrontMaxM)
  // work buffers
  void* d_seg = nullptr;   // batch*k*m real
  void* d_half = nullptr;  // batch*k*hstride complex
  void* d_E = nullptr;     // batch*k*Lp complex elements
  void* d_part = nullptr;  // batch*maxslots*ncells complex
  double* d_S = nullptr;   // batch*ncells double2
  void* d_xin = nullptr;   // host path staging (batch*k*m*8 bytes)
  void* d_out = nullptr;   // host path staging
  size_t bytes = 0;
  unsigned long long* trace = nullptr;  // K2 per-warp trace (diagnostics; 4 x nwarps x batch)
  // multi-GPU (hos_comm_attach): NCCL communicator and the segment-sharded layout's buffers
  void* comm = nullptr;
  int rank = 0, nranks = 1;
  std::vector<int64_t> layout;  // hos_shard_layout record of (order, m, k, m3, nranks)
  void* d_raw = nullptr;        // ncells partial raw sums of this rank's segments
  void* d_send = nullptr;       // nranks x block reduce-scatter input
  void* d_mine = nullptr;       // block: this rank's reduced lines
  void* d_local = nullptr;      // lines this rank smooths (own block + halo)
  void* d_heads = nullptr;      // nranks x halo (or nranks x block when the halo spans ranks)
  void* d_vals = nullptr;       // pmax: this rank's values
  void* d_parts = nullptr;      // nranks x pmax gathered values
  int64_t* d_send_line = nullptr;  // per line: index of its first cell in the padded send buffer
  // fused reduce-scatter over peer memory (HOS_DIST_P2P != 0): every rank's
  // slot reduction stores its partial sums straight into the owner rank's
  // landing buffer (nranks x block, one slot per source rank) through CUDA IPC
  // mappings; the owner adds the slots in rank order after a barrier
  bool p2p = false;
  void* d_land = nullptr;
  std::vector<void*> peer_land;               // per rank (this rank's own: d_land), IPC-opened
  unsigned long long* d_p2p_line = nullptr;   // per line: address of its first cell in the owner's slot
  void* d_bar = nullptr;                      // barrier all-gather scratch (nranks floats)
  std::map<int, cufftHandle> ffts;  // rows -> plan
  // CUDA graphs of the whole stream-ordered pipeline, one per buffer binding
  struct GraphKey {
    int kind;  // 0 estimate, 1 from_spectra, 2 host (pinned)
    const void* in;
    int dtype;
    int64_t stride;
    void* out;
    bool operator<(const GraphKey& o) const {
      return std::tie(kind, in, dtype, stride, out) < std::tie(o.kind, o.in, o.dtype, o.stride, o.out);
    }
  };
  std::map<GraphKey, cudaGraphExec_t> graphs;
  cudaStream_t cap = nullptr;   // capture stream
  bool use_graphs = true;
  // timing
  int timing = 0;
  // stage events: 0 start | 1 prep | 2 fft | 3 extend | 4 triple | 5 scan | 6 box
  cudaEvent_t ev[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  bool timed = false;
  // one caller at a time per plan: graph cache, capture stream and scratch
  // buffers are shared (recursive: entry points call each other)
  std::recursive_mutex mu;
  // streaming host path: host-mapped error word K2 sets when a ready-flag wait timed out
  int* h_err = nullptr;
  int* d_err = nullptr;
};

namespace {

size_t csize(int precision) { return precision == 32 ? 8 : 16; }

// Serialises callers of one plan and runs the call on the plan's device
// (restoring the caller's current device afterwards), so a plan built for
// cuda:1 works whatever device the calling thread has selected.
struct PlanGuard {
  std::lock_guard<std::recursive_mutex> lock;
  int prev = -1, dev;
  explicit PlanGuard(hos_plan* p) : lock(p->mu), dev(p->device) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~PlanGuard() {
    if (prev >= 0 && prev != dev) cudaSetDevice(prev);
  }
};
size_t rsize(int precision) { return precision == 32 ? 4 : 8; }

template <typename T>
int upload(hos_plan* p, T** dst, const std::vector<T>& src) {
  if (src.empty()) return HOS_OK;
  CUDA_TRY(cudaMalloc((void**)dst, src.size() * sizeof(T)));
  p->bytes += src.size() * sizeof(T);
  CUDA_TRY(cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice));
  return HOS_OK;
}

int alloc(hos_plan* p, void** dst, size_t n) {
  if (n == 0) n = 16;
  CUDA_TRY(cudaMalloc(dst, n));
  p->bytes += n;
  return HOS_OK;
}

int get_fft(hos_plan* p, int rows, cufftHandle* out) {
  auto it = p->ffts.find(rows);
  if (it != p->ffts.end()) {
    *out = it->second;
    return HOS_OK;
  }
  cufftHandle h;
  int n[1] = {p->m};
  int inembed[1] = {p->m};
  int onembed[1] = {p->hstride};
  CUFFT_TRY(cufftPlanMany(&h, 1, n, inembed, 1, p->m, onembed, 1, p->hstride,
                          p->precision == 32 ? CUFFT_R2C : CUFFT_D2Z, rows));
  p->ffts[rows] = h;
  *out = h;
  return HOS_OK;
}

int run_fft(hos_plan* p, int rows, const void* in, void* out, cudaStream_t st) {
  cufftHandle h;
  int rc = get_fft(p, rows, &h);
  if (rc) return rc;
  CUFFT_TRY(cufftSetStream(h, st));
  if (p->precision == 32)
    CUFFT_TRY(cufftExecR2C(h, (cufftReal*)in, (cufftComplex*)out));
  else
    CUFFT_TRY(cufftExecD2Z(h, (cufftDoubleReal*)in, (cufftDoubleComplex*)out));
  return HOS_OK;
}

// k_triple_cta stages 4 whole E rows per ring slot, twice (two bank
// offsets), in a ring of 3 slots: it is used when that fits in shared memory
// (fp32: pitch <= 1152 elements, i.e. M up to ~2048; larger M keeps the
// per-warp staged k_triple_w, which copies only the windows a tile reads).
bool cta_allowed() {
  const char* env = std::getenv("HOS_K2");  // "warp": per-warp staged k_triple_w for every launch
  return !(env && std::string(env) == "warp");
}
int pitch_of(const hos::Geometry& g) { return (g.f_hi - g.f_lo + 1 + 4 + 15) & ~15; }
// fp32 quad E rows for k_triple_cta (opt-in, HOS_K2_QUAD=1): 16 warps of <= 128
// registers with one float2 accumulator per cell and no operand-building
// instructions, but twice the staged bytes; measured slower than the float2
// kernel on cfg2/cfg4/cfg5, so off by default
bool want_quad(int precision) {
  const char* env = std::getenv("HOS_K2_QUAD");
  return precision == 32 && env && env[0] == '1';
}
size_t e_bytes(int precision) { return want_quad(precision) ? 16 : csize(precision); }
bool cta_fits(const hos::Geometry& g, int precision) {
  const int64_t A = (4 * (int64_t)pitch_of(g) * (int64_t)e_bytes(precision) + 127) / 128 * 128;
  return 3 * (2 * A + 128) <= (int64_t)hos::kCtaMaxSmem;
}

// D_h geometry with the K2 tile shape for this M: 8 x 16 tiles (lane step 2)
// when they issue enough fewer cells than 16 x 32 tiles, else 16 x 32.  With
// k_triple_cta an 8 x 16 region's eight tiles share two bank offsets (the
// staged rows' copies A and B), so its loads conflict: it pays from 1.25x
// fewer cells (cfg4 at 1.54x: 70 vs 117 us; cfg5 at 1.29x: 1012 vs 1407 us;
// cfg2 at 1.08x: 42 vs 34 us).  With
// k_triple_w an 8 x 16 region stages 2.5x the chunks of a 16 x 32 one and
// measured 1.79x slower per issued cell, so it needs 1.8x.  HOS_K2_TILE=2|4
// forces the step.
// For order 3 the first band's height (1..tile rows) shifts every later band
// across D_h's staircase edges: the tiling with the fewest regions is kept
// (ties: full first band).  E.g. M = 2048, w = 11: 289 instead of 297
// regions; cfg2 and cfg5 are already minimal.
std::string build_best_band(hos::Geometry& g, int order, int m, int m3, int step) {
  std::string err = g.build(order, m, m3, step);
  if (!err.empty() || order != 3) return err;
  for (int fb = 1; fb < 4 * step; fb++) {
    hos::Geometry t;
    if (t.build(order, m, m3, step, fb).empty() && t.nregions < g.nregions) g = std::move(t);
  }
  return "";
}

std::string build_geometry(hos::Geometry& g, int order, int m, int m3, int precision) {
  int forced = 0;
  if (const char* env = std::getenv("HOS_K2_TILE")) forced = std::atoi(env);
  if (forced == 2 || forced == 4) return build_best_band(g, order, m, m3, forced);
  std::string err = build_best_band(g, order, m, m3, 4);
  if (!err.empty()) return err;
  hos::Geometry g2;
  if (!build_best_band(g2, order, m, m3, 2).empty()) return "";
  const bool cta = cta_allowed() && cta_fits(g2, precision);
  if ((double)g.issued_cells >= (cta ? 1.25 : 1.8) * (double)g2.issued_cells) g = std::move(g2);
  return "";
}

int check_plan(const hos_plan* p) {
  if (!p) return fail(HOS_EPARAM, "null plan");
  return HOS_OK;
}

// CTAs splitting a launch over nseg segments of `batch` series: one wave of
// SMs x occupancy CTAs in total, at least 16 work units per CTA (and never
// more CTAs than units, so every CTA's range is non-empty).
int64_t work_items(const hos_plan* p) { return (int64_t)p->geo.nregions; }

int nctas_for(const hos_plan* p, int nseg, int batch) {
  const int64_t work = work_items(p) * nseg;
  int64_t n = 0;
  if (const char* env = std::getenv("HOS_NCTAS")) n = std::atoll(env);
  if (n <= 0) {
    const int64_t slots = (int64_t)p->sms * p->occupancy;
    n = (slots + batch - 1) / batch;
    n = std::min<int64_t>(n, std::max<int64_t>(1, work / 16));
  }
  n = std::min<int64_t>(n, std::max<int64_t>(1, work));
  return (int)std::max<int64_t>(1, n);
}

// warps splitting K2's work for an n-CTA launch (never more than units)
int64_t nwarps_for(const hos_plan* p, int nseg, int n) {
  return std::max<int64_t>(1, std::min<int64_t>((int64_t)n * hos::kTripleWarps, work_items(p) * nseg));
}

// WarpSplit weights for an n-CTA launch: skewed towards the first wave of
// CTAs only when every SM holds exactly two CTAs of one series and each warp
// keeps >= 16 units (so no range can be empty)
hos::WarpSplit warp_split(const hos_plan* p, int nseg, int n, int batch) {
  const int64_t W = work_items(p) * nseg, Nw = nwarps_for(p, nseg, n);
  hos::WarpSplit sp{W, Nw, Nw / 2, 1, 1};
  if (batch == 1 && n == 2 * p->sms && p->occupancy == 2 && W >= 16 * Nw) {
    sp.wa = p->split_wa;
    sp.wb = p->split_wb;
  }
  return sp;
}

int slots_needed(const hos_plan* p, int nseg, int n, int batch) {
  const int64_t T = work_items(p);
  if (T * nseg <= 0) return 1;
  // partial slots the worst region needs (same arithmetic as the kernel)
  const hos::WarpSplit sp = warp_split(p, nseg, n, batch);
  int best = 1;
  for (int64_t t = 0; t < T; t++) best = std::max(best, sp.region_slots((int)t, nseg));
  return best;
}

hos::SlotInfo slot_info(const hos_plan* p, int nseg, int n) {
  hos::SlotInfo si{};
  if (!p->cta && nseg == p->k && n == p->nctas) si.region_slots = p->d_region_slots;  // the plan's main launch
  si.line_tile0 = p->d_line_tile0;
  si.nseg = nseg;
  si.nregions = p->geo.nregions;
  si.tile_cols = p->geo.tile_cols;
  si.tiles_per_region = p->geo.tiles_per_region;
  si.nwarps = nwarps_for(p, nseg, n);
  const hos::WarpSplit sp = warp_split(p, nseg, n, p->batch);
  si.split_wa = sp.wa;
  si.split_wb = sp.wb;
  return si;
}

hos::TripleArgs triple_args(const hos_plan* p, int seg_begin, int seg_end, int n, int batch) {
  hos::TripleArgs x;
  std::memset(&x, 0, sizeof(x));
  x.f_lo = p->geo.f_lo;
  x.K = p->k;
  x.seg_begin = seg_begin;
  x.seg_end = seg_end;
  x.E = p->d_E;
  x.Lp = p->Lp;
  x.tiles = p->d_tiles;
  x.nregions = p->geo.nregions;
  x.tile_step = p->geo.tile_step;
  x.nwarps = nwarps_for(p, seg_end - seg_begin, n);
  {
    const hos::WarpSplit sp = warp_split(p, seg_end - seg_begin, n, batch);
    x.split_wa = sp.wa;
    x.split_wb = sp.wb;
  }
  x.line_cmax = p->d_line_cmax;
  x.line_start = p->d_line_start;
  x.lo = p->geo.win.lo;
  x.part = p->d_part;
  x.ncells = p->geo.ncells;
  x.maxslots = p->maxslots;
  x.order = p->order;
  x.conj = p->conj;
  x.batch = batch;
  x.accumulate = 0;
  x.trace = p->trace;
  return x;
}

// partial slots of the plan's main K2 launch (k_triple_cta or k_triple_w)
enum Sched { kMainSched = 0, kStreamSched = 1, kChunkSched = 2 };
hos::SlotInfo main_slot_info(const hos_plan* p, int sched = kMainSched) {
  hos::SlotInfo si = slot_info(p, p->k, p->nctas);
  si.region_slots = sched == kStreamSched ? p->d_s_region_slots
                    : sched == kChunkSched ? p->d_c_region_slots
                                           : p->d_region_slots;
  si.rs_stride = sched == kMainSched ? p->rs_stride : 0;
  return si;
}

hos::CtaTripleArgs cta_args(const hos_plan* p, bool streaming = false);
// K2 over chunk `c` of the chunked host path (rows shifted, slots accumulated after chunk 0)
hos::CtaTripleArgs chunk_args(const hos_plan* p, int c) {
  hos::CtaTripleArgs a = cta_args(p);
  a.blocks = p->d_c_blocks;
  a.stages = p->d_c_stages;
  a.cta_stage0 = p->d_c_cta_stage0;
  a.cta_head = p->d_c_cta_head;
  a.nctas = p->c_nctas;
  a.tab_stages = p->c_tab_stages;
  a.tab_blocks = p->c_tab_blocks;
  a.trace = nullptr;
  a.row_shift = c * p->chunk_k;
  a.accumulate = c > 0 ? 1 : 0;
  return a;
}

hos::CtaTripleArgs cta_args(const hos_plan* p, bool streaming) {
  hos::CtaTripleArgs a{};
  a.E = p->d_E;
  a.Lp = p->Lp;
  a.f_lo = p->geo.f_lo;
  a.tiles = p->d_tiles;
  a.tile_step = p->geo.tile_step;
  a.groups = p->d_groups;
  a.blocks = p->d_blocks;
  a.stages = p->d_stages;
  a.cta_stage0 = p->d_cta_stage0;
  a.cta_head = p->d_cta_head;
  a.nctas = p->cta_nctas;
  a.depth = p->cta_depth;
  a.stage_segs = p->cta_stage_segs;
  a.slot_bytes = p->cta_slot_bytes;
  a.copy_b = p->cta_copy_b;
  a.quad = p->quad ? 1 : 0;
  a.refill_last = p->m >= 512 ? 1 : 0;  // long stages (cfg2); short ones (cfg4, cfg5) wait on empty[]
  if (const char* env = std::getenv("HOS_K2_REFILL")) a.refill_last = env[0] == 'l';  // "last" | "empty"
  // warp-pair skew (see k_triple_cta): same-box A/B, K2 in-step -- cfg2 32.6 -> 31.7 us at 3000 cycles
  // (1000: 32.8, 5000: 32.9), cfg5 865 -> 846 us (1000-5000 alike); order 4 (cfg4) loses 3 %, so off there.
  // The gain is small because a warp alone on its sub-partition only reaches ~47 % of the pipe.
  a.skew_cycles = p->order == 3 && !p->quad ? 3000 : 0;
  if (const char* env = std::getenv("HOS_K2_SKEW")) a.skew_cycles = std::max(0, std::atoi(env));

  a.tab_stages = p->cta_tab_stages;
  a.tab_blocks = p->cta_tab_blocks;
  a.line_cmax = p->d_line_cmax;
  a.line_start = p->d_line_start;
  a.lo = p->geo.win.lo;
  a.part = p->d_part;
  a.ncells = p->geo.ncells;
  a.maxslots = p->maxslots;
  a.order = p->order;
  a.conj = p->conj;
  a.trace = p->trace;
  a.trace_cta = p->cta_nctas - 1;
  if (const char* env = std::getenv("HOS_TRACE_CTA")) a.trace_cta = std::atoi(env);
  if (streaming) {
    a.blocks = p->d_s_blocks;
    a.stages = p->d_s_stages;
    a.cta_stage0 = p->d_s_cta_stage0;
    a.cta_head = p->d_s_cta_head;
    a.nctas = p->s_nctas;
    a.tab_stages = p->s_tab_stages;
    a.tab_blocks = p->s_tab_blocks;
    a.ready = p->d_ready;
    a.err = p->d_err;
  }
  return a;
}

// K2 over all segments of every series of the plan
cudaError_t launch_main_triple(const hos_plan* p, cudaStream_t st) {
  if (p->cta) return hos::launch_triple_cta(cta_args(p), p->precision, st);
  return hos::launch_triple(triple_args(p, 0, p->k, p->nctas, p->batch), p->precision, st);
}

// Host schedule of k_triple_cta (see hos_kernels.cuh): regions in groups of
// kCtaWarps (+ one remainder group), the (series, group, segment) sequence
// split into one contiguous range per CTA (one CTA per SM) of balanced
// estimated time at segment granularity, ranges cut into blocks
// at (series, group) boundaries and blocks into stages of up to 4 segments.
// Partial slots per (series, region) are counted in CTA order.  Returns
// false when the plan is not eligible (ring too small for one segment).
struct CtaSchedule {
  std::vector<hos::CtaGroup> groups;
  std::vector<hos::CtaBlock> blocks;
  std::vector<hos::CtaStage> stages;
  std::vector<int32_t> cta_stage0;
  std::vector<int32_t> region_slots;  // batch x nregions
  int nctas = 0, depth = 0, stage_segs = 4, slot_bytes = 0, copy_b = 0, maxslots = 1;
  int tab_stages = 0, tab_blocks = 0;  // most stages / blocks of one CTA (shared-memory tables)
  std::vector<int4> heads() const {     // per CTA {first stage, stages, first block, blocks}
    std::vector<int4> h;
    for (int c = 0; c + 1 < (int)cta_stage0.size(); c++) {
      const int k0 = cta_stage0[c], n = cta_stage0[c + 1] - k0;
      const int b0 = n > 0 ? stages[k0].block : 0;
      h.push_back(make_int4(k0, n, b0, n > 0 ? stages[k0 + n - 1].block - b0 + 1 : 0));
    }
    return h;
  }
  // fills tab_* (0: ring + tables exceed the CTA's shared memory, the kernel reads them from global)
  bool size_tables() {
    tab_stages = tab_blocks = 0;
    for (int c = 0; c + 1 < (int)cta_stage0.size(); c++) {
      const int n = cta_stage0[c + 1] - cta_stage0[c];
      tab_stages = std::max(tab_stages, n);
      if (n > 0) tab_blocks = std::max(tab_blocks, stages[cta_stage0[c + 1] - 1].block - stages[cta_stage0[c]].block + 1);
    }
    if ((size_t)depth * slot_bytes + 16 * (size_t)(tab_stages + tab_blocks) > hos::kCtaSmemLimit)
      tab_stages = tab_blocks = 0;  // read from global memory
    return true;
  }
};

int stream_front_ctas() {
  if (const char* env = std::getenv("HOS_STREAM_CTAS")) return std::max(1, std::atoi(env));  // diagnostics
  return hos::kStreamFrontCtas;
}

bool build_cta_schedule(const hos_plan* p, CtaSchedule& cs, int interleave_ctas = 0, int k_override = 0) {
  const hos::Geometry& g = p->geo;
  const int R = g.nregions, K = k_override > 0 ? k_override : p->k, B = p->batch;
  if (R <= 0 || K <= 0) return false;
  const int64_t row_bytes = (int64_t)p->Lp * (int64_t)e_bytes(p->precision);
  if (!cta_fits(g, p->precision)) return false;
  int segs = 0;
  // Stage shape: the largest of 16 / 12 / 8 / 4 segments whose ring (staged
  // twice, two bank offsets) still holds 3 slots -- every stage hand-off
  // (mbarrier wait, refill bookkeeping) is paid once per stage, so longer
  // stages amortise it (same-box A/B, K2 in-step: cfg2 4 -> 8 segments 35.6
  // -> 32.5 us; cfg4 68.4 -> 63.3 -> 61.1 us at 8 / 16; cfg5 981 -> 888 ->
  // 865 us).  M up to ~2048 fits 4-segment stages only (with 3 slots).
  // HOS_K2_SEGS / HOS_K2_COPIES (diagnostics) force a stage size / one copy.
  int copies = 2;
  if (const char* env = std::getenv("HOS_K2_COPIES")) copies = std::atoi(env) == 1 ? 1 : 2;
  std::vector<int> tries = {16, 12, 8, 4};
  if (const char* env = std::getenv("HOS_K2_SEGS")) tries = {std::max(1, std::min(16, std::atoi(env)))};
  for (size_t ti = 0; ti < tries.size() && !segs; ti++) {
    const int s = tries[ti];
    const int64_t A = (s * row_bytes + 127) / 128 * 128;
    const int64_t slot = copies * A + 128;
    // 3 slots: a deeper ring lets the warp the scheduler favours run further
    // ahead of its sub-partition partner, which then runs alone (cfg2 K2 at
    // 4-segment stages: depth 3 33.6 us, 4 33.8, 5 34.4, 6 35.3); order 4
    // (short rows): 5 slots when they fit (at 16-segment stages 3 and 5 are even)
    int64_t depth = std::min<int64_t>({(int64_t)(p->order == 4 ? 5 : 3), (int64_t)hos::kCtaMaxDepth,
                                       (int64_t)hos::kCtaMaxSmem / slot});
    if (const char* env = std::getenv("HOS_CTA_DEPTH"))  // diagnostics
      depth = std::max<int64_t>(2, std::min<int64_t>({(int64_t)hos::kCtaMaxDepth, (int64_t)hos::kCtaMaxSmem / slot,
                                                       (int64_t)std::atoi(env)}));
    const bool last = ti + 1 == tries.size();
    if (depth >= 3 || (last && depth >= 2)) {
      segs = s;
      cs.depth = (int)depth;
      cs.slot_bytes = (int)slot;
      cs.copy_b = copies == 2 ? (int)(A + 64) : 0;
      cs.stage_segs = s;
    }
  }
  if (!segs) return false;
  // full groups of W regions, then the remainder r < W: its regions' tiles
  // split over two warps when r <= W/2 and its stages over `phases` warps.
  // A remainder stage takes about 1/phases of a full stage's compute but
  // still copies the whole stage (copy-bound at ~45% of a full stage, cfg2), so a segment weighs max(W / phases, 4)
  // where a full group's weighs W.
  const int W = hos::cta_warps(want_quad(p->precision));
  auto both_tiles = [&](int r0, int n) {  // every region of [r0, r0+n) has two real tiles
    if (g.tiles_per_region != 2) return false;
    for (int r = r0; r < r0 + n; r++)
      if (g.tiles[2 * r].nrows == 0 || g.tiles[2 * r + 1].nrows == 0) return false;
    return true;
  };
  for (int r0 = 0; r0 < R; r0 += W) {
    const int n = std::min(W, R - r0);
    const int halves = n <= W / 2 && both_tiles(r0, n) ? 2 : 1;
    const int ph = std::max(1, std::min({segs, W / (n * halves), cs.depth}));
    cs.groups.push_back({r0, n, ph, halves});
  }
  const int ng = (int)cs.groups.size();
  auto weight = [&](int gi) -> int64_t {
    const hos::CtaGroup& gr = cs.groups[gi];
    static const int64_t floor_w = [] { const char* e = std::getenv("HOS_K2_REMW"); return e ? (int64_t)std::atoi(e) : (int64_t)3; }();  // cfg2: 4 left the remainder group's CTAs idle from 23 of 33 us; 3: K2 31.9 -> 31.6 us; 2: 37.9
    return gr.n == W ? W : std::max<int64_t>(W / gr.phases, floor_w);
  };
  if (interleave_ctas > 0) {
    // Streaming schedule (host path, series arriving over PCIe while K2
    // runs): each group gets an integer number of CTAs in proportion to its
    // time, and CTA r of a group takes the group's stages j = r, r + n, ...
    // so every CTA works through the series in arrival order.  One block per
    // CTA (slot base r x phases).
    if (B != 1) return false;
    const int64_t N = interleave_ctas;
    const int nst = (K + segs - 1) / segs;
    std::vector<int64_t> n(ng);
    int64_t tot = 0, sum = 0;
    for (int gi = 0; gi < ng; gi++) tot += weight(gi);
    for (int gi = 0; gi < ng; gi++) {
      n[gi] = std::max<int64_t>(1, std::min<int64_t>(nst, (N * weight(gi) + tot / 2) / tot));
      sum += n[gi];
    }
    while (sum > N) {  // trim the groups with the most CTAs per unit of time
      int best = -1;
      for (int gi = 0; gi < ng; gi++)
        if (n[gi] > 1 && (best < 0 || n[gi] * weight(best) > n[best] * weight(gi))) best = gi;
      if (best < 0) return false;
      n[best]--;
      sum--;
    }
    cs.cta_stage0.push_back(0);
    std::vector<int32_t> slots(ng, 0);
    for (int gi = 0; gi < ng; gi++) {
      for (int64_t r = 0; r < n[gi]; r++) {
        const int blk = (int)cs.blocks.size();
        cs.blocks.push_back({0, 0, gi, slots[gi]});
        slots[gi] += cs.groups[gi].phases;
        for (int64_t j = r; j < nst; j += n[gi])
          cs.stages.push_back({(int)(j * segs), std::min(segs, K - (int)(j * segs)), blk, 0});
        cs.cta_stage0.push_back((int32_t)cs.stages.size());
      }
    }
    cs.nctas = (int)sum;
    cs.region_slots.assign(R, 0);
    cs.maxslots = 1;
    for (int gi = 0; gi < ng; gi++) {
      for (int r = cs.groups[gi].r0; r < cs.groups[gi].r0 + cs.groups[gi].n; r++) cs.region_slots[r] = slots[gi];
      cs.maxslots = std::max(cs.maxslots, slots[gi]);
    }
    return cs.size_tables();
  }
  // (series, group) chunks of K segments each.  The CTA ranges come from
  // the smallest per-CTA time budget T (bisection) for which a greedy fill
  // needs <= N CTAs; a CTA's time is its segments' weights plus kSwitch per
  // block after its first (the block switch -- partial-slot stores, the next
  // block's geometry loads -- stalls all of the CTA's warps, ~1 stage).
  const int64_t nchunks = (int64_t)B * ng;
  const int64_t N = std::max<int64_t>(1, std::min<int64_t>(p->sms, (int64_t)B * ng * K));
  const int64_t kSwitch = 3 * W;
  // greedy fill: cuts[c] = start (chunk, seg) of CTA c; returns CTAs used
  auto fill = [&](int64_t T, std::vector<std::pair<int64_t, int>>* cuts) -> int64_t {
    int64_t used = 0, ch = 0;
    int seg = 0;
    while (ch < nchunks) {
      if (cuts) cuts->push_back({ch, seg});
      used++;
      int64_t cost = 0;
      bool first = true;
      while (ch < nchunks) {
        const int64_t w = weight((int)(ch % ng));
        const int64_t sw = first ? 0 : kSwitch;
        const int64_t room = T - cost - sw;
        const int64_t take = room <= 0 ? 0 : std::min<int64_t>(K - seg, room / w);
        if (take <= 0) {
          if (first) {  // T below one segment: take one anyway
            if (++seg >= K) { ch++; seg = 0; }
          }
          break;
        }
        cost += sw + take * w;
        first = false;
        seg += (int)take;
        if (seg >= K) {
          ch++;
          seg = 0;
        } else {
          break;
        }
      }
    }
    return used;
  };
  int64_t lo_t = 1, hi_t = 1;
  for (int64_t c = 0; c < nchunks; c++) hi_t += weight((int)(c % ng)) * K + kSwitch;
  while (lo_t < hi_t) {
    const int64_t mid = lo_t + (hi_t - lo_t) / 2;
    if (fill(mid, nullptr) <= N) hi_t = mid;
    else lo_t = mid + 1;
  }
  std::vector<std::pair<int64_t, int>> cuts;
  const int64_t used = fill(lo_t, &cuts);
  cuts.push_back({nchunks, 0});
  std::vector<int32_t> slots(nchunks, 0);
  cs.cta_stage0.push_back(0);
  for (int64_t c = 0; c < used; c++) {
    const int64_t ch0 = cuts[c].first, ch1 = cuts[c + 1].first;
    const int sg0 = cuts[c].second, sg1 = cuts[c + 1].second;
    for (int64_t ch = ch0; ch <= ch1 && ch < nchunks; ch++) {
      const int sb = ch == ch0 ? sg0 : 0;
      const int se = ch == ch1 ? sg1 : K;
      if (se <= sb) continue;
      const int b = (int)(ch / ng), gi = (int)(ch % ng);
      const int blk = (int)cs.blocks.size();
      cs.blocks.push_back({b * K + sb, b, gi, slots[ch]});
      slots[ch] += cs.groups[gi].phases;
      for (int s = sb; s < se; s += segs) cs.stages.push_back({b * K + s, std::min(segs, se - s), blk, 0});
    }
    cs.cta_stage0.push_back((int32_t)cs.stages.size());
  }
  const int64_t N_used = used;
  cs.nctas = (int)N_used;
  cs.region_slots.assign((size_t)B * R, 0);
  cs.maxslots = 1;
  for (int64_t ch = 0; ch < nchunks; ch++) {
    const hos::CtaGroup& gr = cs.groups[ch % ng];
    for (int r = gr.r0; r < gr.r0 + gr.n; r++) cs.region_slots[(ch / ng) * R + r] = slots[ch];
    cs.maxslots = std::max(cs.maxslots, slots[ch]);
  }
  return cs.size_tables();
}

// K4b arguments for the whole grid of every series of the plan
hos::BoxArgs box_args(const hos_plan* p, void* out_dev) {
  hos::BoxArgs b{};
  b.S = p->d_S;
  b.s_series_stride = p->geo.ncells;
  b.line_base = 0;
  b.line_start = p->d_line_start;
  b.cell_base = 0;
  b.row_off = p->d_row_off;
  b.rows = p->geo.rows;
  b.pair_k1 = p->d_pair_k1;
  b.pair_k2 = p->d_pair_k2;
  b.pair_base = p->d_pair_base;
  b.npairs = (int)p->geo.pair_k1.size();
  b.line_of_ab = p->d_line_of_ab;
  b.b_count = p->geo.b_count;
  b.lo = p->geo.win.lo;
  b.hi = p->geo.win.hi;
  b.m3 = p->m3;
  b.order = p->order;
  b.m = p->m;
  b.row_begin = 0;
  b.row_end = p->geo.rows;
  b.pair_begin = 0;
  b.pair_end = (int)p->geo.pair_k1.size();
  b.p_begin = 0;
  b.p_end = p->geo.npoints;
  b.scale = 1.0 / ((double)p->m * (double)p->k * std::pow((double)p->m3, p->order - 1));
  b.out = out_dev;
  b.out_series_stride = p->geo.npoints;
  b.precision = p->precision;
  b.batch = p->batch;
  return b;
}

int run_box(hos_plan* p, void* out_dev, cudaStream_t st) {
  CUDA_TRY(hos::launch_box(box_args(p, out_dev), st));
  return HOS_OK;
}

// K4 of the whole grid: one CTA per series in shared memory when the grid is
// small (order 3), else line scans + box sums
int run_smooth(hos_plan* p, void* out_dev, cudaStream_t st, int stage = -1, int sched = kMainSched) {
  const hos::SlotInfo si = main_slot_info(p, sched);
  const bool streaming = sched == kStreamSched;
  if (p->series_k4) {
    if (stage != 5 && p->pipe_k4)
      CUDA_TRY(hos::launch_smooth_series_pipe(p->d_part, p->maxslots, p->geo.ncells, si, p->precision,
                                              box_args(p, out_dev), p->pipe_layout, p->d_pipe_tables,
                                              p->d_cell_region,
                                              streaming ? p->d_s_series_slots : p->d_series_slots, st));
    else if (stage != 5 && p->sep_k4)
      CUDA_TRY(hos::launch_smooth_series_sep(p->d_part, p->maxslots, p->geo.ncells, si, p->precision,
                                             box_args(p, out_dev), p->geo.nlines, p->sep_vitems, p->sep_hitems,
                                             streaming ? p->d_s_series_slots : p->d_series_slots, st));
    else if (stage != 5)
      CUDA_TRY(hos::launch_smooth_series3(p->d_part, p->maxslots, p->geo.ncells, si, p->precision,
                                          box_args(p, out_dev), p->geo.nlines, st));
    return HOS_OK;
  }
  if (p->tiles_k4) {  // R (compute precision) in p->d_S, then the separable box tiles
    if (stage != 5)
      CUDA_TRY(hos::launch_raw_cells(p->d_part, p->maxslots, p->geo.ncells, si.region_slots, si.rs_stride,
                                     p->d_cell_region, p->geo.ncells, p->batch, p->precision, p->d_S, st));
    if (p->timing && stage < 0) CUDA_TRY(cudaEventRecord(p->ev[5], st));
    if (stage != 4)
      CUDA_TRY(hos::launch_box_tiles(p->d_S, p->geo.ncells, p->precision, box_args(p, out_dev),
                                     (int)p->geo.nlines, p->d_box_tiles, p->box_ntiles, st));
    return HOS_OK;
  }
  if (stage != 5)
    CUDA_TRY(hos::launch_line_scan(p->d_part, p->maxslots, p->geo.ncells, si, p->precision, p->d_line_start, 0,
                                   p->geo.nlines, p->geo.ncells, p->batch, p->d_S, st, p->max_line));
  if (p->timing && stage < 0) CUDA_TRY(cudaEventRecord(p->ev[5], st));
  if (stage != 4) return run_box(p, out_dev, st);
  return HOS_OK;
}

// K2 + K4 over the extended spectra already in p->d_E.
int run_back(hos_plan* p, void* out_dev, cudaStream_t st) {
  CUDA_TRY(launch_main_triple(p, st));
  if (p->timing) CUDA_TRY(cudaEventRecord(p->ev[4], st));
  int rc = run_smooth(p, out_dev, st);
  if (rc) return rc;
  if (p->timing) {
    if (p->series_k4) CUDA_TRY(cudaEventRecord(p->ev[5], st));
    CUDA_TRY(cudaEventRecord(p->ev[6], st));
    p->timed = true;
  }
  return HOS_OK;
}

int check_dtype_x(int x_dtype) {
  if (x_dtype != HOS_F32 && x_dtype != HOS_F64)
    return fail(HOS_EPARAM, "series dtype must be HOS_F32 or HOS_F64, got " + std::to_string(x_dtype));
  return HOS_OK;
}

// Fused front end over segments [seg_begin, seg_begin+nseg) of `batch` series -> E rows.
// quad: E rows as quads for k_triple_cta (the plan's main launch); the
// segment-range launches of hos_partial_raw (k_triple_w) write plain rows.
int fused_front(hos_plan* p, const void* x_dev, int x_dtype, int64_t x_stride, int seg_begin, int nseg, int batch,
                cudaStream_t st, bool quad) {
  const char* xs = (const char*)x_dev + (size_t)seg_begin * p->m * (x_dtype == HOS_F32 ? 4 : 8);
  void* E = (char*)p->d_E + (size_t)seg_begin * p->Lp * (quad ? 16 : csize(p->precision));
  CUDA_TRY(hos::launch_front(xs, x_dtype, x_stride, p->m, nseg, p->k, batch, p->taper, p->d_taper, p->d_tw,
                             p->precision, p->geo.f_lo, p->L, p->Lp, E, st, quad ? 1 : 0));
  return HOS_OK;
}

// K0 + FFT + K1 for all batch*k segments.
int run_front(hos_plan* p, const void* x_dev, int x_dtype, int64_t x_stride, cudaStream_t st) {
  const int rows = p->batch * p->k;
  if (p->fused) {
    int rc = fused_front(p, x_dev, x_dtype, x_stride, 0, p->k, p->batch, st, p->quad);
    if (rc) return rc;
    if (p->timing)
      for (int i = 1; i <= 3; i++) CUDA_TRY(cudaEventRecord(p->ev[i], st));
    return HOS_OK;
  }
  CUDA_TRY(hos::launch_prep(x_dev, x_dtype, x_stride, p->m, 0, p->k, p->batch, p->taper, p->d_taper, p->precision,
                            p->d_seg, st));
  if (p->timing) CUDA_TRY(cudaEventRecord(p->ev[1], st));
  int rc = run_fft(p, rows, p->d_seg, p->d_half, st);
  if (rc) return rc;
  if (p->timing) CUDA_TRY(cudaEventRecord(p->ev[2], st));
  CUDA_TRY(hos::launch_extend_half(p->d_half, p->m, p->hstride, rows, nullptr, p->geo.f_lo, p->L, p->Lp,
                                   p->precision, p->d_E, st, p->quad));
  if (p->timing) CUDA_TRY(cudaEventRecord(p->ev[3], st));
  return HOS_OK;
}

// Run `body(stream)` through a cached CUDA graph keyed by the buffer binding
// (captured on the plan's private stream on first use, replayed on `st`).
template <typename F>
int run_graph(hos_plan* p, const hos_plan::GraphKey& key, cudaStream_t st, F body) {
  auto it = p->graphs.find(key);
  if (it == p->graphs.end()) {
    cudaGraph_t graph = nullptr;
    CUDA_TRY(cudaStreamBeginCapture(p->cap, cudaStreamCaptureModeThreadLocal));
    int rc = body(p->cap);
    cudaError_t e = cudaStreamEndCapture(p->cap, &graph);
    if (rc) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    CUDA_TRY(e);
    cudaGraphExec_t exec = nullptr;
    e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    CUDA_TRY(e);
    if (p->graphs.size() >= 16) {  // bound the cache
      cudaGraphExecDestroy(p->graphs.begin()->second);
      p->graphs.erase(p->graphs.begin());
    }
    it = p->graphs.emplace(key, exec).first;
  }
  CUDA_TRY(cudaGraphLaunch(it->second, st));
  return HOS_OK;
}

}  // namespace

// lines [lb, le) the output rows [r0, r1) read (order 3: rows r0 .. r1-1+w-1;
// order 4: the pair lines of planes a in [r0+lo, r1-1+hi])
void rows_lines(const hos::Geometry& g, int order, int m3, int r0, int r1, int64_t* lb, int64_t* le) {
  if (order == 3) {
    *lb = r0;
    *le = r1 == r0 ? r0 : r1 - 1 + (m3 - 1) + 1;
    return;
  }
  int64_t b = 0, e = 0;
  const int alo = r0 + g.win.lo, ahi = r1 - 1 + g.win.hi;
  while (b < g.nlines && g.line_a[b] < alo) b++;
  e = b;
  while (e < g.nlines && g.line_a[e] <= ahi) e++;
  *lb = b;
  *le = r1 == r0 ? b : e;
}

// Segment-sharded multi-GPU layout (the C++ twin of parallel.shard_layout):
// segments split evenly, output rows by whole-row point balance (the
// reference's row_blocks policy, hospectra/parallel.py:73-80), lines owned
// from each rank's first needed line, halo = lines past the owned block.
// Record: per rank {seg0, seg1, row0, row1, own_l0, own_l1, need_l0, need_l1,
// own_c0, own_c1, need_c0, need_c1, p0, p1}, then {block, halo, in_next}.
constexpr int kLayoutPerRank = 14;
std::vector<int64_t> shard_layout(const hos::Geometry& g, int order, int m3, int k, int n) {
  std::vector<int> rb(n + 1, 0);
  const int rows = g.rows;
  const int64_t total = g.row_off[rows];
  if (n == 1 || total == 0) {
    for (int r = 1; r <= n; r++) rb[r] = rows;
  } else {
    for (int r = 1; r < n; r++) {  // first row whose cumulative point count reaches r / n of the total
      const double t = (double)r * ((double)total / n);
      int i = 0;
      while (i < rows && (double)g.row_off[i + 1] < t) i++;
      rb[r] = std::min(rows, i + 1);
    }
    rb[n] = rows;
  }
  std::vector<int64_t> nl0(n), nl1(n), ol0(n), ol1(n);
  for (int r = 0; r < n; r++) rows_lines(g, order, m3, rb[r], rb[r + 1], &nl0[r], &nl1[r]);
  int64_t nxt = g.nlines;
  for (int r = n - 1; r >= 0; r--) {
    const int64_t l0 = rb[r] < rb[r + 1] ? nl0[r] : nxt;
    ol0[r] = l0;
    ol1[r] = nxt;
    nxt = l0;
  }
  ol0[0] = 0;
  for (int r = 0; r < n; r++)
    if (!(rb[r] < rb[r + 1])) nl0[r] = nl1[r] = ol0[r];
  std::vector<int64_t> rec;
  int64_t block = 1, halo = 1;
  bool in_next = true;
  std::vector<int64_t> oc0(n), oc1(n), nc0(n), nc1(n);
  for (int r = 0; r < n; r++) {
    oc0[r] = g.line_start[ol0[r]];
    oc1[r] = g.line_start[ol1[r]];
    nc0[r] = g.line_start[nl0[r]];
    nc1[r] = g.line_start[nl1[r]];
    block = std::max(block, oc1[r] - oc0[r]);
  }
  for (int r = 0; r < n; r++) {
    const int64_t h = std::max<int64_t>(0, nc1[r] - oc1[r]);
    halo = std::max(halo, h);
    if (h && !(r + 1 < n && h <= oc1[r + 1] - oc0[r + 1])) in_next = false;
  }
  for (int r = 0; r < n; r++) {
    const int64_t v[kLayoutPerRank] = {(int64_t)r * k / n, (int64_t)(r + 1) * k / n, rb[r], rb[r + 1], ol0[r], ol1[r],
                                       nl0[r], nl1[r], oc0[r], oc1[r], nc0[r], nc1[r], g.row_off[rb[r]],
                                       g.row_off[rb[r + 1]]};
    rec.insert(rec.end(), v, v + kLayoutPerRank);
  }
  rec.push_back(block);
  rec.push_back(halo);
  rec.push_back(in_next ? 1 : 0);
  return rec;
}

// NCCL, resolved at hos_comm_attach (no link-time dependency: the process may
// already hold another libnccl, e.g. the one PyTorch ships)
struct NcclApi {
  decltype(&ncclReduceScatter) reduce_scatter = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  decltype(&ncclCommCount) comm_count = nullptr;
  decltype(&ncclCommUserRank) comm_rank = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
};
const NcclApi* nccl_api(std::string* why) {
  static NcclApi api;
  static bool tried = false, ok = false;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);  // already in the process?
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.reduce_scatter = (decltype(api.reduce_scatter))dlsym(h, "ncclReduceScatter");
      api.all_gather = (decltype(api.all_gather))dlsym(h, "ncclAllGather");
      api.error_string = (decltype(api.error_string))dlsym(h, "ncclGetErrorString");
      api.comm_count = (decltype(api.comm_count))dlsym(h, "ncclCommCount");
      api.comm_rank = (decltype(api.comm_rank))dlsym(h, "ncclCommUserRank");
      api.send = (decltype(api.send))dlsym(h, "ncclSend");
      api.recv = (decltype(api.recv))dlsym(h, "ncclRecv");
      api.group_start = (decltype(api.group_start))dlsym(h, "ncclGroupStart");
      api.group_end = (decltype(api.group_end))dlsym(h, "ncclGroupEnd");
      ok = api.reduce_scatter && api.all_gather && api.error_string && api.comm_count && api.comm_rank &&
           api.send && api.recv && api.group_start && api.group_end;
    }
  }
  if (!ok && why) *why = "libnccl.so.2 (ncclReduceScatter, ncclAllGather) is not loadable";
  return ok ? &api : nullptr;
}

#define NCCL_TRY(api, expr)                                                                          \
  do {                                                                                               \
    ncclResult_t r_ = (expr);                                                                        \
    if (r_ != ncclSuccess) return fail(HOS_ECUDA, std::string("NCCL error in ") + #expr + ": " +     \
                                                       (api)->error_string(r_));                     \
  } while (0)

namespace {

void release_p2p(hos_plan* p) {
  for (size_t r = 0; r < p->peer_land.size(); r++)
    if (p->peer_land[r] && p->peer_land[r] != p->d_land) cudaIpcCloseMemHandle(p->peer_land[r]);
  p->peer_land.clear();
  for (void* b : {p->d_land, (void*)p->d_p2p_line, p->d_bar})
    if (b) cudaFree(b);
  p->d_land = nullptr;
  p->d_p2p_line = nullptr;
  p->d_bar = nullptr;
  p->p2p = false;
}

// Landing buffers + IPC handle exchange over the communicator (one
// all-gather of the 64-byte handles); any failure leaves the NCCL
// reduce-scatter path in place (p->p2p false)
int setup_p2p(hos_plan* p, const NcclApi* api, ncclComm_t comm, int me, int n) {
  release_p2p(p);
  // default: on with more than one rank (one rank has nothing to exchange and
  // the plain send-layout reduction is faster: 13.7 vs 22 us on cfg2);
  // HOS_DIST_P2P=1 forces it on (tests), =0 off
  const char* env = std::getenv("HOS_DIST_P2P");
  if (env ? env[0] == '0' : n == 1) return HOS_OK;
  const int64_t* L = p->layout.data();
  const int64_t block = L[kLayoutPerRank * n];
  const size_t cs = csize(p->precision);
  int rc = HOS_OK;
  if ((rc = alloc(p, &p->d_land, (size_t)n * block * cs)) || (rc = alloc(p, &p->d_bar, (size_t)n * 8))) return rc;
  p->peer_land.assign(n, nullptr);
  p->peer_land[me] = p->d_land;
  if (n > 1) {
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, p->d_land) != cudaSuccess) {
      cudaGetLastError();
      release_p2p(p);
      return HOS_OK;
    }
    void* dh = nullptr;
    CUDA_TRY(cudaMalloc(&dh, (size_t)(n + 1) * sizeof(h)));
    CUDA_TRY(cudaMemcpy((char*)dh + (size_t)n * sizeof(h), &h, sizeof(h), cudaMemcpyHostToDevice));
    NCCL_TRY(api, api->all_gather((char*)dh + (size_t)n * sizeof(h), dh, sizeof(h), ncclInt8, comm, nullptr));
    std::vector<cudaIpcMemHandle_t> all(n);
    const cudaError_t e = cudaMemcpy(all.data(), dh, (size_t)n * sizeof(h), cudaMemcpyDeviceToHost);
    cudaFree(dh);
    CUDA_TRY(e);
    for (int r = 0; r < n; r++) {
      if (r == me) continue;
      if (cudaIpcOpenMemHandle(&p->peer_land[r], all[r], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        p->peer_land[r] = nullptr;
        release_p2p(p);  // every rank must agree: fall back only if all do (checked below)
        break;
      }
    }
    // agree: all ranks use p2p only if every rank opened every peer
    float ok = p->peer_land.empty() ? 0.f : 1.f;
    std::vector<float> oks(n, 0.f);
    void* db = nullptr;
    CUDA_TRY(cudaMalloc(&db, (size_t)(n + 1) * sizeof(float)));
    CUDA_TRY(cudaMemcpy((float*)db + n, &ok, sizeof(float), cudaMemcpyHostToDevice));
    NCCL_TRY(api, api->all_gather((float*)db + n, db, 1, ncclFloat32, comm, nullptr));
    CUDA_TRY(cudaMemcpy(oks.data(), db, (size_t)n * sizeof(float), cudaMemcpyDeviceToHost));
    cudaFree(db);
    for (float v : oks)
      if (v != 1.f) {
        release_p2p(p);
        return HOS_OK;
      }
  }
  // per line: the address of its first cell in the owner's landing slot `me`
  std::vector<unsigned long long> da(p->geo.nlines);
  int r = 0;
  for (int64_t l = 0; l < p->geo.nlines; l++) {
    while (r + 1 < n && l >= L[kLayoutPerRank * r + 5]) r++;  // own_l1 of rank r
    const int64_t off = (int64_t)me * block + (p->geo.line_start[l] - L[kLayoutPerRank * r + 8]);
    da[l] = (unsigned long long)((char*)p->peer_land[r] + (size_t)off * cs);
  }
  if ((rc = upload(p, &p->d_p2p_line, da))) return rc;
  p->p2p = true;
  return HOS_OK;
}

}  // namespace

extern "C" {

const char* hos_version(void) { return "hos_b200 0.1.0 sm_100a"; }

const char* hos_last_error(void) { return g_err.c_str(); }

int64_t hos_domain_size(int order, int m) {
  if ((order != 3 && order != 4) || m < 2) return -1;
  return hos::domain_size(order, m);
}

int hos_domain_indices(int order, int m, int64_t start, int64_t stop, int32_t* out) {
  if (order != 3 && order != 4) return fail(HOS_EPARAM, "order must be 3 or 4, got " + std::to_string(order));
  if (m < 2) return fail(HOS_EPARAM, "segment length must be >= 2, got " + std::to_string(m));
  const int64_t total = hos::domain_size(order, m);
  if (stop <= start) return HOS_OK;
  if (!(0 <= start && start < stop && stop <= total))
    return fail(HOS_EPARAM, "slice [" + std::to_string(start) + ", " + std::to_string(stop) +
                                ") outside domain of size " + std::to_string(total));
  if (!out) return fail(HOS_EPARAM, "null output");
  hos::domain_rows(order, m, start, stop, out);
  return HOS_OK;
}

int hos_plan_create(hos_plan** out, int order, int m, int k, int m3, int conjugate_last, int precision, int taper,
                    int batch, int device) {
  if (!out) return fail(HOS_EPARAM, "null plan pointer");
  *out = nullptr;
  if (m < 1 || k < 1)
    return fail(HOS_EPARAM, "segment length and count must be positive, got m=" + std::to_string(m) +
                                ", k=" + std::to_string(k));
  if (precision != 32 && precision != 64)
    return fail(HOS_EPARAM, "precision must be 32 or 64, got " + std::to_string(precision));
  if (taper != HOS_TAPER_NONE && taper != HOS_TAPER_HANN)
    return fail(HOS_EPARAM, "unknown taper code " + std::to_string(taper));
  if (batch < 1) return fail(HOS_EPARAM, "batch must be >= 1, got " + std::to_string(batch));
  hos_plan* p = new hos_plan();
  p->order = order;
  p->m = m;
  p->k = k;
  p->m3 = m3;
  p->conj = conjugate_last ? 1 : 0;
  p->precision = precision;
  p->taper = taper;
  p->batch = batch;
  p->device = device;
  std::string err = build_geometry(p->geo, order, m, m3, precision);
  if (!err.empty()) {
    delete p;
    return fail(HOS_EPARAM, err);
  }
  int rc = HOS_OK;
  auto bail = [&](int code) {
    hos_plan_destroy(p);
    return code;
  };
  if (cudaSetDevice(device) != cudaSuccess) {
    delete p;
    return fail(HOS_ECUDA, "cannot select CUDA device " + std::to_string(device));
  }
  const hos::Geometry& g = p->geo;
  p->hstride = m / 2 + 1;
  p->L = g.f_hi - g.f_lo + 1;
  for (size_t l = 0; l + 1 < g.line_start.size(); l++)
    p->max_line = std::max<int>(p->max_line, (int)(g.line_start[l + 1] - g.line_start[l]));
  {
    const char* env = std::getenv("HOS_K4_SERIES");  // "0": always line scans + box sums
    p->series_k4 = order == 3 && hos::smooth_series3_smem(g.ncells, g.nlines, g.rows, g.nregions, g.npoints) <= 200 * 1024 &&
                   !(env && env[0] == '0');
    // separable direct window sums (default; HOS_K4_SEP=0: the prefix-sum kernel)
    const char* sep = std::getenv("HOS_K4_SEP");
    hos::smooth_series_sep_items(g.row_off.data(), g.rows, m3, &p->sep_vitems, &p->sep_hitems);
    // separable K4 for line grids (default; HOS_K4_TILES=0: line scans + prefix
    // differences): cfg2 scan + box 12.2 -> 7.3 us, step 60.3 -> 56.8 us;
    // cfg3 79.4 -> 52.3 us (same box)
    const char* tk = std::getenv("HOS_K4_TILES");
    p->tiles_k4 = order == 3 && !p->series_k4 && hos::box_tiles_supports(m3) && g.nregions < 65536 &&
                  !(tk && tk[0] == '0');
    p->sep_k4 = p->series_k4 && !(sep && sep[0] == '0') && hos::smooth_series_sep_supports(m3) &&
                hos::smooth_series_sep_smem(g.ncells, g.nlines, g.rows, g.nregions, g.npoints, m3, p->sep_vitems,
                                            p->sep_hitems, precision) <= 200 * 1024;
    // pipelined variant (default; HOS_K4_PIPE=0: k_smooth_series_sep)
    const char* pk = std::getenv("HOS_K4_PIPE");
    p->pipe_k4 = p->sep_k4 && !(pk && pk[0] == '0') && g.nregions < 65536;
  }
  // +4 elements: fp32 operands are staged from the 16-byte-aligned element at
  // or below their start, in whole 16-byte chunks (K2), so a copy may read up
  // to 3 elements past the last frequency; even pitch keeps rows 16-byte aligned
  // k_triple_cta bulk-copies whole rows: a pitch of 16 elements keeps every
  // row 128-byte aligned (TMA moves aligned rows at the full rate)
  p->Lp = pitch_of(g);
  cudaDeviceGetAttribute(&p->sms, cudaDevAttrMultiProcessorCount, device);
  p->occupancy = hos::triple_occupancy(precision, g.tile_step);
  if (const char* env = std::getenv("HOS_K2_SPLIT")) {  // "wa:wb"
    int wa = 0, wb = 0;
    if (std::sscanf(env, "%d:%d", &wa, &wb) == 2 && wa > 0 && wb > 0) {
      p->split_wa = wa;
      p->split_wb = wb;
    }
  }
  p->nctas = nctas_for(p, k, batch);
  p->maxslots = slots_needed(p, k, p->nctas, batch);
  CtaSchedule sched;
  p->cta = cta_allowed() && build_cta_schedule(p, sched);
  if (p->cta) {
    p->quad = want_quad(precision);
    p->cta_warps = hos::cta_warps(p->quad);
    p->cta_nctas = sched.nctas;
    p->cta_depth = sched.depth;
    p->cta_stage_segs = sched.stage_segs;
    p->cta_slot_bytes = sched.slot_bytes;
    p->cta_copy_b = sched.copy_b;
    p->cta_tab_stages = sched.tab_stages;
    p->cta_tab_blocks = sched.tab_blocks;
    // batch-1 plans keep room for the segment-range launches of k_triple_w (multi-GPU shards)
    p->maxslots = batch == 1 ? std::max(p->maxslots, sched.maxslots) : sched.maxslots;
    p->rs_stride = g.nregions;
  }
  CtaSchedule ssched;
  {
    // opt-in (HOS_STREAM=1): 1.3x faster host calls on most placements, but
    // some runs of some SM splits were 2.2x slower
    const char* env = std::getenv("HOS_STREAM");
    p->stream_ok = p->cta && batch == 1 && k >= 64 && (m & (m - 1)) == 0 && m <= hos::kFrontMaxM &&
                   (env && env[0] == '1') &&
                   build_cta_schedule(p, ssched, std::max(1, p->sms - stream_front_ctas()));
    if (p->stream_ok) {
      p->s_nctas = ssched.nctas;
      p->s_tab_stages = ssched.tab_stages;
      p->s_tab_blocks = ssched.tab_blocks;
      p->maxslots = std::max(p->maxslots, ssched.maxslots);
    }
  }


  std::vector<int32_t> cmax(g.line_cmax.begin(), g.line_cmax.end());
  if ((rc = upload(p, &p->d_tiles, g.tiles))) return bail(rc);
  if ((rc = upload(p, &p->d_line_tile0, g.line_tile0))) return bail(rc);
  if (p->stream_ok) {
    if ((rc = upload(p, &p->d_s_region_slots, ssched.region_slots))) return bail(rc);
    {
      int32_t mx = 1;
      for (int32_t v : ssched.region_slots) mx = std::max(mx, v);
      if ((rc = upload(p, &p->d_s_series_slots, std::vector<int32_t>(1, mx)))) return bail(rc);
    }
    if ((rc = upload(p, &p->d_s_blocks, ssched.blocks))) return bail(rc);
    if ((rc = upload(p, &p->d_s_stages, ssched.stages))) return bail(rc);
    if ((rc = upload(p, &p->d_s_cta_stage0, ssched.cta_stage0))) return bail(rc);
    if ((rc = upload(p, &p->d_s_cta_head, ssched.heads()))) return bail(rc);
    if ((rc = alloc(p, (void**)&p->d_ready, (size_t)k * sizeof(int)))) return bail(rc);
    if (cudaHostAlloc((void**)&p->h_err, sizeof(int), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer((void**)&p->d_err, p->h_err, 0) != cudaSuccess)
      return bail(fail(HOS_ECUDA, "cannot map the streaming path's error word"));
    *p->h_err = 0;
    if (cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&p->e_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&p->e_join, cudaEventDisableTiming) != cudaSuccess)
      return bail(fail(HOS_ECUDA, "cannot create the streaming path's stream/events"));
  }
  if (p->cta) {
    if ((rc = upload(p, &p->d_region_slots, sched.region_slots))) return bail(rc);
    std::vector<int32_t> ss(batch, 1);
    for (int b = 0; b < batch; b++)
      for (int r = 0; r < g.nregions; r++) ss[b] = std::max(ss[b], sched.region_slots[(size_t)b * g.nregions + r]);
    if ((rc = upload(p, &p->d_series_slots, ss))) return bail(rc);
    if ((rc = upload(p, &p->d_groups, sched.groups))) return bail(rc);
    if ((rc = upload(p, &p->d_blocks, sched.blocks))) return bail(rc);
    if ((rc = upload(p, &p->d_stages, sched.stages))) return bail(rc);
    if ((rc = upload(p, &p->d_cta_stage0, sched.cta_stage0))) return bail(rc);
    if ((rc = upload(p, &p->d_cta_head, sched.heads()))) return bail(rc);

  } else {
    const hos::WarpSplit sp = warp_split(p, k, p->nctas, batch);
    std::vector<int32_t> rs(g.nregions);
    for (size_t r = 0; r < rs.size(); r++) rs[r] = sp.region_slots((int)r, k);
    if ((rc = upload(p, &p->d_region_slots, rs))) return bail(rc);
    int32_t mx = 1;
    for (int32_t v : rs) mx = std::max(mx, v);
    if ((rc = upload(p, &p->d_series_slots, std::vector<int32_t>(batch, mx)))) return bail(rc);
  }
  if ((rc = upload(p, &p->d_line_cmax, cmax))) return bail(rc);
  if ((rc = upload(p, &p->d_line_start, g.line_start))) return bail(rc);
  if ((rc = upload(p, &p->d_row_off, g.row_off))) return bail(rc);
  if (order == 4) {
    if ((rc = upload(p, &p->d_pair_k1, g.pair_k1))) return bail(rc);
    if ((rc = upload(p, &p->d_pair_k2, g.pair_k2))) return bail(rc);
    if ((rc = upload(p, &p->d_pair_base, g.pair_base))) return bail(rc);
    if ((rc = upload(p, &p->d_line_of_ab, g.line_of_ab))) return bail(rc);
  }
  if (p->pipe_k4) {
    hos::PipePlan pp = hos::smooth_series_pipe_plan(g.row_off.data(), g.rows, g.line_start.data(), g.nlines, g.ncells,
                                                    g.nregions, m3, precision);
    if (pp.L.total <= 220 * 1024) {
      p->pipe_layout = pp.L;
      if ((rc = upload(p, &p->d_pipe_tables, pp.tables))) return bail(rc);
      const std::vector<uint16_t> cr = hos::cell_region_table(g.line_tile0.data(), g.line_start.data(), g.nlines,
                                                              g.tile_cols, g.tiles_per_region);
      if ((rc = upload(p, &p->d_cell_region, cr))) return bail(rc);
    } else {
      p->pipe_k4 = false;
    }
  }
  if (p->tiles_k4) {
    const std::vector<int32_t> bt = hos::box_tile_list(g.row_off.data(), g.rows);
    p->box_ntiles = (int)bt.size();
    if ((rc = upload(p, &p->d_box_tiles, bt))) return bail(rc);
    const std::vector<uint16_t> cr = hos::cell_region_table(g.line_tile0.data(), g.line_start.data(), g.nlines,
                                                            g.tile_cols, g.tiles_per_region);
    if ((rc = upload(p, &p->d_cell_region, cr))) return bail(rc);
  }
  {
    // m fp64 weights, then the same m weights rounded to fp32 (the fp32 front end)
    std::vector<double> tab(m + (m + 1) / 2, 0.0);
    for (int u = 0; u < m; u++) tab[u] = 0.5 - 0.5 * std::cos(2.0 * M_PI * u / m);
    float* t32 = reinterpret_cast<float*>(tab.data() + m);
    for (int u = 0; u < m; u++) t32[u] = (float)tab[u];
    if ((rc = upload(p, &p->d_taper, tab))) return bail(rc);
  }
  {
    const char* env = std::getenv("HOS_FRONT");  // "cufft": K0 -> cuFFT -> K1 even for power-of-two m
    p->fused = (m & (m - 1)) == 0 && m <= hos::kFrontMaxM && !(env && std::string(env) == "cufft");
    if (p->fused) {
      const int h = m;  // full circle: radix-4 stages read w^(j p s) for j <= 3
      if (precision == 32) {
        std::vector<float> tw(2 * h);
        for (int t = 0; t < h; t++) {
          tw[2 * t] = (float)std::cos(2.0 * M_PI * t / m);
          tw[2 * t + 1] = (float)-std::sin(2.0 * M_PI * t / m);
        }
        if ((rc = upload(p, (float**)&p->d_tw, tw))) return bail(rc);
      } else {
        std::vector<double> tw(2 * h);
        for (int t = 0; t < h; t++) {
          tw[2 * t] = std::cos(2.0 * M_PI * t / m);
          tw[2 * t + 1] = -std::sin(2.0 * M_PI * t / m);
        }
        if ((rc = upload(p, (double**)&p->d_tw, tw))) return bail(rc);
      }
    }
  }
  {
    // chunked host path (opt-in: HOS_CHUNKS=n >= 2): equal chunks of >= 32
    // segments cross PCIe on the copy engine while the previous chunk's front
    // end and K2 run.  Two chunks: cfg2 e2e 153.5 -> 148.7 us when the copy
    // engine is warm -- but a 4 MiB copy-engine H2D issued once per call runs
    // at 13-53 GB/s depending on what the link did in the preceding
    // milliseconds (tools/e2e_cliff.py: the same call takes 148 us or 350-490
    // us, and the default bench run hit the slow regime after 18 calls), while
    // the zero-copy front end (SM loads over PCIe) holds 153 us from the second
    // call on.  The default is therefore the zero-copy path.
    const char* env = std::getenv("HOS_CHUNKS");
    const int want = env ? std::atoi(env) : 0;
    CtaSchedule cs;
    if (p->cta && p->fused && batch == 1 && want > 1 && k % want == 0 && k / want >= 32 &&
        build_cta_schedule(p, cs, 0, k / want) && cs.groups.size() == sched.groups.size() &&
        cs.depth == p->cta_depth && cs.slot_bytes == p->cta_slot_bytes && cs.copy_b == p->cta_copy_b) {
      p->chunks = want;
      p->chunk_k = k / want;
      p->c_nctas = cs.nctas;
      p->c_tab_stages = cs.tab_stages;
      p->c_tab_blocks = cs.tab_blocks;
      p->maxslots = std::max(p->maxslots, cs.maxslots);
      if ((rc = upload(p, &p->d_c_blocks, cs.blocks))) return bail(rc);
      if ((rc = upload(p, &p->d_c_stages, cs.stages))) return bail(rc);
      if ((rc = upload(p, &p->d_c_cta_stage0, cs.cta_stage0))) return bail(rc);
      if ((rc = upload(p, &p->d_c_cta_head, cs.heads()))) return bail(rc);
      if ((rc = upload(p, &p->d_c_region_slots, cs.region_slots))) return bail(rc);
      p->c_ev.assign(want + 1, nullptr);
      for (auto& e : p->c_ev)
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
          return bail(fail(HOS_ECUDA, "cannot create the chunked host path's events"));
      if (cudaStreamCreateWithFlags(&p->c_copy, cudaStreamNonBlocking) != cudaSuccess)
        return bail(fail(HOS_ECUDA, "cannot create the chunked host path's copy stream"));
    }
  }
  const size_t rows = (size_t)batch * k;
  if ((rc = alloc(p, &p->d_seg, rows * m * rsize(precision)))) return bail(rc);
  if ((rc = alloc(p, &p->d_half, rows * p->hstride * csize(precision)))) return bail(rc);
  const size_t e_bytes = rows * p->Lp * (p->quad ? 16 : csize(precision));  // plain rows of partial_raw fit too
  if ((rc = alloc(p, &p->d_E, e_bytes))) return bail(rc);
  if (cudaMemset(p->d_E, 0, e_bytes) != cudaSuccess)  // pad elements stay defined
    return bail(fail(HOS_ECUDA, "cudaMemset failed"));
  // +64: k_smooth_series_pipe's bulk copy of a series rounds its size up to 16 bytes
  if ((rc = alloc(p, &p->d_part, (size_t)batch * p->maxslots * g.ncells * csize(precision) + 64))) return bail(rc);
  if ((rc = alloc(p, (void**)&p->d_S, (size_t)batch * g.ncells * 16))) return bail(rc);
  if ((rc = alloc(p, &p->d_xin, rows * m * 8))) return bail(rc);
  if ((rc = alloc(p, &p->d_out, (size_t)batch * g.npoints * csize(precision)))) return bail(rc);
  cufftHandle h;
  if ((rc = get_fft(p, (int)rows, &h))) return bail(rc);
  for (auto& e : p->ev)
    if (cudaEventCreate(&e) != cudaSuccess) return bail(fail(HOS_ECUDA, "cudaEventCreate failed"));
  if (cudaStreamCreateWithFlags(&p->cap, cudaStreamNonBlocking) != cudaSuccess)
    return bail(fail(HOS_ECUDA, "cudaStreamCreate failed"));
  if (const char* env = std::getenv("HOS_NO_GRAPH")) p->use_graphs = std::atoi(env) == 0;
  *out = p;
  return HOS_OK;
}

void hos_plan_destroy(hos_plan* p) {
  if (!p) return;
  for (auto& kv : p->graphs) cudaGraphExecDestroy(kv.second);
  if (p->cap) cudaStreamDestroy(p->cap);
  for (auto& kv : p->ffts) cufftDestroy(kv.second);
  if (p->side) cudaStreamDestroy(p->side);
  if (p->e_fork) cudaEventDestroy(p->e_fork);
  if (p->e_join) cudaEventDestroy(p->e_join);
  for (void* b : {(void*)p->d_s_blocks, (void*)p->d_s_stages, (void*)p->d_s_cta_stage0, (void*)p->d_s_region_slots,
                  (void*)p->d_ready})
    if (b) cudaFree(b);
  if (p->h_err) cudaFreeHost(p->h_err);
  for (void* b : {(void*)p->d_c_blocks, (void*)p->d_c_stages, (void*)p->d_c_cta_stage0, (void*)p->d_c_cta_head,
                  (void*)p->d_c_region_slots})
    if (b) cudaFree(b);
  for (cudaEvent_t e : p->c_ev)
    if (e) cudaEventDestroy(e);
  if (p->c_copy) cudaStreamDestroy(p->c_copy);
  release_p2p(p);
  for (void* b : {(void*)p->d_series_slots, (void*)p->d_s_series_slots, (void*)p->d_box_tiles,
                  (void*)p->d_cell_region, (void*)p->d_pipe_tables})
    if (b) cudaFree(b);
  for (void* b : {p->d_raw, p->d_send, p->d_mine, p->d_local, p->d_heads, p->d_vals, p->d_parts, (void*)p->d_send_line})
    if (b) cudaFree(b);
  void* bufs[] = {p->d_groups, p->d_blocks, p->d_stages, p->d_cta_stage0, p->d_cta_head, p->d_s_cta_head, p->d_tiles, p->d_line_tile0, p->d_region_slots, p->d_line_cmax, p->d_line_start, p->d_row_off, p->d_pair_k1, p->d_pair_k2,
                  p->d_pair_base, p->d_line_of_ab, p->d_taper, p->d_tw, p->d_seg, p->d_half, p->d_E, p->d_part,
                  p->d_S, p->d_xin, p->d_out};
  for (void* b : bufs)
    if (b) cudaFree(b);
  for (auto& e : p->ev)
    if (e) cudaEventDestroy(e);
  delete p;
}

int64_t hos_plan_npoints(const hos_plan* p) { return p ? p->geo.npoints : -1; }
int64_t hos_plan_cells(const hos_plan* p) { return p ? p->geo.ncells : -1; }
int64_t hos_plan_units(const hos_plan* p) { return p ? p->geo.ncells * (int64_t)p->k : -1; }
int64_t hos_plan_issued(const hos_plan* p) { return p ? p->geo.issued_cells * (int64_t)p->k : -1; }
int64_t hos_plan_row_len(const hos_plan* p) { return p ? p->L : -1; }
size_t hos_plan_device_bytes(const hos_plan* p) { return p ? p->bytes : 0; }
int hos_plan_launches(const hos_plan* p) {
  // kernels of this library per hos_estimate: [fused front | K0, K1 around
  // cuFFT's own kernels] + K2 + [per-series K4 | K4a, K4b]
  return p ? (p->fused ? 1 : 2) + 1 + (p->series_k4 ? 1 : 2) : -1;
}
int64_t hos_plan_lines(const hos_plan* p) { return p ? p->geo.nlines : -1; }

int hos_plan_line_starts(const hos_plan* p, int64_t* ls) {
  int rc = check_plan(p);
  if (rc) return rc;
  if (!ls) return fail(HOS_EPARAM, "null output");
  std::memcpy(ls, p->geo.line_start.data(), p->geo.line_start.size() * sizeof(int64_t));
  return HOS_OK;
}

int hos_estimate(hos_plan* p, const void* x_dev, int x_dtype, int64_t x_stride, void* out_dev, void* stream) {
  int rc = check_plan(p);
  if (rc) return rc;
  PlanGuard guard_(p);
  if ((rc = check_dtype_x(x_dtype))) return rc;
  if (!x_dev || !out_dev) return fail(HOS_EPARAM, "null buffer");
  if (p->batch > 1 && x_stride < (int64_t)p->k * p->m)
    return fail(HOS_EPARAM, "series stride " + std::to_string(x_stride) + " shorter than k*m = " +
                                std::to_string((int64_t)p->k * p->m));
  cudaStream_t st = (cudaStream_t)stream;
  if (p->timing || p->trace || !p->use_graphs) {
    if (p->timing) CUDA_TRY(cudaEventRecord(p->ev[0], st));
    if ((rc = run_front(p, x_dev, x_dtype, x_stride, st))) return rc;
    return run_back(p, out_dev, st);
  }
  const hos_plan::GraphKey key{0, x_dev, x_dtype, x_stride, out_dev};
  return run_graph(p, key, st, [&](cudaStream_t s) {
    int r = run_front(p, x_dev, x_dtype, x_stride, s);
    return r ? r : run_back(p, out_dev, s);
  });
}

int hos_estimate_from_spectra(hos_plan* p, const void* spec_dev, int spec_dtype, void* out_dev, void* stream) {
  int rc = check_plan(p);
  if (rc) return rc;
  PlanGuard guard_(p);
  if (spec_dtype != HOS_C64 && spec_dtype != HOS_C128)
    return fail(HOS_EPARAM, "spectra dtype must be HOS_C64 or HOS_C128");
  if (!spec_dev || !out_dev) return fail(HOS_EPARAM, "null buffer");
  cudaStream_t st = (cudaStream_t)stream;
  auto body = [&](cudaStream_t s) -> int {
    if (p->timing) CUDA_TRY(cudaEventRecord(p->ev[0], s));
    CUDA_TRY(hos::launch_extend_full(spec_dev, spec_dtype, p->m, p->batch * p->k, p->geo.f_lo, p->L, p->Lp,
                                     p->precision, p->d_E, s, p->quad));
    if (p->timing)
      for (int i = 1; i <= 3; i++) CUDA_TRY(cudaEventRecord(p->ev[i], s));
    return run_back(p, out_dev, s);
  };
  if (p->timing || p->trace || !p->use_graphs) return body(st);
  const hos_plan::GraphKey key{1, spec_dev, spec_dtype, 0, out_dev};
  return run_graph(p, key, st, body);
}

int hos_segment_spectra(hos_plan* p, const void* x_dev, int x_dtype, int64_t x_stride, void* spec_dev, void* stream) {
  int rc = check_plan(p);
  if (rc) return rc;
  PlanGuard guard_(p);
  if ((rc = check_dtype_x(x_dtype))) return rc;
  if (!x_dev || !spec_dev) return fail(HOS_EPARAM, "null buffer");
  cudaStream_t st = (cudaStream_t)stream;
  const int rows = p->batch * p->k;
  CUDA_TRY(hos::launch_prep(x_dev, x_dtype, x_stride, p->m, 0, p->k, p->batch, p->taper, p->d_taper, p->precision,
                            p->d_seg, st));
  if ((rc = run_fft(p, rows, p->d_seg, p->d_half, st))) return rc;
  CUDA_TRY(hos::launch_expand_full(p->d_half, p->m, p->hstride, rows, p->precision, spec_dev, st));
  return HOS_OK;
}

int hos_dft_rows(const void* x_dev, int x_dtype, int rows, int m, int precision, void* spec_dev, void* stream) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int, int>, std::pair<cufftHandle, void*>> cache;  // -> plan, scratch
  if ((x_dtype != HOS_F32 && x_dtype != HOS_F64) || (precision != 32 && precision != 64))
    return fail(HOS_EPARAM, "bad dtype/precision");
  if (rows < 1 || m < 1) return fail(HOS_EPARAM, "rows and m must be positive");
  if (!x_dev || !spec_dev) return fail(HOS_EPARAM, "null buffer");
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  cudaStream_t st = (cudaStream_t)stream;
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_tuple(dev, m, rows, precision);
  auto it = cache.find(key);
  const int hs = m / 2 + 1;
  const size_t rs = precision == 32 ? 4 : 8, cs = 2 * rs;
  if (it == cache.end()) {
    cufftHandle h;
    int n[1] = {m}, ine[1] = {m}, one[1] = {hs};
    CUFFT_TRY(cufftPlanMany(&h, 1, n, ine, 1, m, one, 1, hs, precision == 32 ? CUFFT_R2C : CUFFT_D2Z, rows));
    void* scratch = nullptr;  // cast input + half spectrum
    CUDA_TRY(cudaMalloc(&scratch, (size_t)rows * m * rs + (size_t)rows * hs * cs + 256));
    it = cache.emplace(key, std::make_pair(h, scratch)).first;
  }
  cufftHandle h = it->second.first;
  char* scratch = (char*)it->second.second;
  void* xin = scratch;
  void* half = scratch + (((size_t)rows * m * rs + 255) & ~(size_t)255);
  // cast only (rows are already demeaned): prep with taper off would demean again, so copy/cast here
  const bool same = (x_dtype == HOS_F32) == (precision == 32);
  if (same) {
    CUDA_TRY(cudaMemcpyAsync(xin, x_dev, (size_t)rows * m * rs, cudaMemcpyDeviceToDevice, st));
  } else {
    CUDA_TRY(hos::launch_cast(x_dev, x_dtype, (int64_t)rows * m, precision, xin, st));
  }
  CUFFT_TRY(cufftSetStream(h, st));
  if (precision == 32) CUFFT_TRY(cufftExecR2C(h, (cufftReal*)xin, (cufftComplex*)half));
  else CUFFT_TRY(cufftExecD2Z(h, (cufftDoubleReal*)xin, (cufftDoubleComplex*)half));
  CUDA_TRY(hos::launch_expand_full(half, m, hs, rows, precision, spec_dev, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return HOS_OK;
}

int hos_estimate_host(hos_plan* p, const void* x_host, int x_dtype, int64_t x_stride, void* out_host, void* stream) {
  int rc = check_plan(p);
  if (rc) return rc;
  PlanGuard guard_(p);
  if ((rc = check_dtype_x(x_dtype))) return rc;
  if (!x_host || !out_host) return fail(HOS_EPARAM, "null buffer");
  // synchronous host API: NULL stream = the plan's private stream
  cudaStream_t st = stream ? (cudaStream_t)stream : p->cap;
  const size_t es = x_dtype == HOS_F32 ? 4 : 8;
  const size_t km = (size_t)p->k * p->m;
  // copy path: H2D into the plan's staging buffer, the device pipeline, D2H
  auto body = [&](cudaStream_t s) -> int {
    if (p->batch == 1 || x_stride == (int64_t)km) {
      CUDA_TRY(cudaMemcpyAsync(p->d_xin, x_host, km * p->batch * es, cudaMemcpyHostToDevice, s));
    } else {
      CUDA_TRY(cudaMemcpy2DAsync(p->d_xin, km * es, x_host, (size_t)x_stride * es, km * es, p->batch,
                                 cudaMemcpyHostToDevice, s));
    }
    int r = run_front(p, p->d_xin, x_dtype, (int64_t)km, s);
    if (!r) r = run_back(p, p->d_out, s);
    if (r) return r;
    CUDA_TRY(cudaMemcpyAsync(out_host, p->d_out, (size_t)p->batch * p->geo.npoints * csize(p->precision),
                             cudaMemcpyDeviceToHost, s));
    return HOS_OK;
  };
  // page-locked host buffers are mapped into the device address space (UVA):
  // the fused front end then reads the series straight over PCIe and K4b
  // writes the values straight into host memory -- the transfers happen inside
  // the kernels that consume / produce them, with no copy-engine hop (a copy
  // overlapped with the kernels slows both, tools/dma_interference.py)
  cudaPointerAttributes ai{}, ao{};
  const bool pinned = cudaPointerGetAttributes(&ai, x_host) == cudaSuccess && ai.type == cudaMemoryTypeHost &&
                      cudaPointerGetAttributes(&ao, out_host) == cudaSuccess && ao.type == cudaMemoryTypeHost;
  cudaGetLastError();
  const char* zc_env = std::getenv("HOS_ZEROCOPY");  // "0": never, "1": always (with page-locked buffers)
  // Large batches go through the copy engines instead: the per-series
  // smoother writes its outputs as 8-byte pieces 32 bytes apart, which cross
  // PCIe as small writes (cfg5, 327 MB in + 136 MB out: 22.9 ms zero-copy,
  // 9.4 ms with one H2D and one D2H copy), and copies this long run at the
  // link rate (the cold-link behaviour of small copies does not matter).
  const size_t host_bytes = (size_t)p->batch * (km * es + (size_t)p->geo.npoints * csize(p->precision));
  const bool zc_size = p->batch == 1 || host_bytes <= ((size_t)16 << 20);
  const bool zero_copy = pinned && p->fused && ai.devicePointer && ao.devicePointer &&
                         (zc_env ? zc_env[0] != '0' : zc_size);
  // chunked: copy-engine transfers of the series in chunks on c_copy; per
  // chunk the front end (device-resident samples) and K2 (accumulating into
  // the partial slots) run while the next chunk crosses PCIe; the smoothing
  // writes the values straight into host memory
  const char* ch_env = std::getenv("HOS_CHUNKED");
  const bool chunked = zero_copy && p->chunks > 1 && !p->stream_ok && !p->timing && !p->trace &&
                       !(ch_env && ch_env[0] == '0');
  auto ch_body = [&](cudaStream_t s) -> int {
    const size_t cb = (size_t)p->chunk_k * p->m * es;
    CUDA_TRY(cudaEventRecord(p->c_ev[p->chunks], s));  // fork: the copies follow the caller's prior work
    CUDA_TRY(cudaStreamWaitEvent(p->c_copy, p->c_ev[p->chunks], 0));
    const bool nocopy = std::getenv("HOS_CHUNK_NOCOPY") != nullptr;  // diagnostics: compute chain alone
    for (int c = 0; c < p->chunks; c++) {
      if (!nocopy)
        CUDA_TRY(cudaMemcpyAsync((char*)p->d_xin + c * cb, (const char*)x_host + c * cb, cb,
                                 cudaMemcpyHostToDevice, p->c_copy));
      CUDA_TRY(cudaEventRecord(p->c_ev[c], p->c_copy));
    }
    for (int c = 0; c < p->chunks; c++) {
      CUDA_TRY(cudaStreamWaitEvent(s, p->c_ev[c], 0));
      int r = fused_front(p, p->d_xin, x_dtype, (int64_t)km, c * p->chunk_k, p->chunk_k, 1, s, p->quad);
      if (r) return r;
      CUDA_TRY(hos::launch_triple_cta(chunk_args(p, c), p->precision, s));
    }
    return run_smooth(p, ao.devicePointer, s, -1, kChunkSched);
  };
  auto zc_body = [&](cudaStream_t s) -> int {
    if (p->timing) CUDA_TRY(cudaEventRecord(p->ev[0], s));
    if (p->stream_ok && !p->timing) {
      // K2 first (its CTAs take one SM each and signal PDL dependents at
      // once), then the front end as its programmatic dependent: it fills the
      // SMs K2 left free, reads the series over PCIe and publishes each E row;
      // K2 consumes rows as their ready flags flip, so the PCIe read overlaps
      // the triple product.  The memset after them is a full barrier (K4 must
      // see K2's partial slots, and the front end ran ahead of K2's end).
      CUDA_TRY(cudaMemsetAsync(p->d_ready, 0, (size_t)p->k * sizeof(int), s));
      CUDA_TRY(hos::launch_triple_cta(cta_args(p, true), p->precision, s));
      CUDA_TRY(hos::launch_front(ai.devicePointer, x_dtype, x_stride, p->m, p->k, p->k, 1, p->taper, p->d_taper,
                                 p->d_tw, p->precision, p->geo.f_lo, p->L, p->Lp, p->d_E, s, p->quad ? 1 : 0,
                                 p->d_ready));
      CUDA_TRY(cudaMemsetAsync(p->d_ready, 0, sizeof(int), s));
      return run_smooth(p, ao.devicePointer, s, -1, kStreamSched);
    }
    int r = fused_front(p, ai.devicePointer, x_dtype, x_stride, 0, p->k, p->batch, s, p->quad);
    if (r) return r;
    if (p->timing)
      for (int i = 1; i <= 3; i++) CUDA_TRY(cudaEventRecord(p->ev[i], s));
    return run_back(p, ao.devicePointer, s);
  };
  if (chunked) {
    const hos_plan::GraphKey key{4, x_host, x_dtype, x_stride, out_host};
    if ((rc = p->use_graphs ? run_graph(p, key, st, ch_body) : ch_body(st))) return rc;
  } else if (pinned && p->use_graphs && !p->timing && !p->trace) {
    const hos_plan::GraphKey key{zero_copy ? 3 : 2, x_host, x_dtype, x_stride, out_host};
    if ((rc = zero_copy ? run_graph(p, key, st, zc_body) : run_graph(p, key, st, body))) return rc;
  } else if (zero_copy) {
    if ((rc = zc_body(st))) return rc;
  } else {
    if (p->timing) CUDA_TRY(cudaEventRecord(p->ev[0], st));
    if ((rc = body(st))) return rc;
  }
  // the call returns the values in host memory: wait by polling (a blocking
  // synchronize can add a scheduler wake-up to every call's latency)
  if (std::getenv("HOS_HOST_SYNC_BLOCK")) {
    CUDA_TRY(cudaStreamSynchronize(st));
  } else {
    cudaError_t q;
    while ((q = cudaStreamQuery(st)) == cudaErrorNotReady) {
    }
    CUDA_TRY(q);
  }
  if (p->h_err && *reinterpret_cast<volatile int*>(p->h_err)) {
    *p->h_err = 0;
    return fail(HOS_ECUDA, "streaming host path: the triple product waited > 200 ms for a spectrum row "
                           "(the front end found no free SM); unset HOS_STREAM");
  }
  return HOS_OK;
}

int partial_raw_impl(hos_plan* p, const void* x_dev, int x_dtype, int seg_begin, int seg_end, void* raw_dev,
                     cudaStream_t st, const int64_t* dst_line, size_t zero_bytes,
                     const unsigned long long* dst_addr = nullptr);

int hos_partial_raw(hos_plan* p, const void* x_dev, int x_dtype, int seg_begin, int seg_end, void* raw_dev,
                    void* stream) {
  int rc = check_plan(p);
  if (rc) return rc;
  PlanGuard guard_(p);
  if ((rc = check_dtype_x(x_dtype))) return rc;
  if (p->batch != 1) return fail(HOS_EPARAM, "hos_partial_raw needs a batch-1 plan");
  if (!(0 <= seg_begin && seg_begin <= seg_end && seg_end <= p->k))
    return fail(HOS_EPARAM, "segment range [" + std::to_string(seg_begin) + ", " + std::to_string(seg_end) +
                                ") outside [0, " + std::to_string(p->k) + ")");
  if (!raw_dev) return fail(HOS_EPARAM, "null buffer");
  return partial_raw_impl(p, x_dev, x_dtype, seg_begin, seg_end, raw_dev, (cudaStream_t)stream, nullptr,
                          p->geo.ncells * csize(p->precision));
}

// front end + K2 + slot reduction over segments [seg_begin, seg_end) of the
// single series; cell c of line l lands at raw[dst_line[l] + c - line_start[l]]
// (dst_line nullptr: raw[c]); an empty range zeroes zero_bytes of raw
int partial_raw_impl(hos_plan* p, const void* x_dev, int x_dtype, int seg_begin, int seg_end, void* raw_dev,
                     cudaStream_t st, const int64_t* dst_line, size_t zero_bytes,
                     const unsigned long long* dst_addr) {
  int rc = HOS_OK;
  const int nseg = seg_end - seg_begin;
  if (nseg == 0) {
    if (dst_addr) {  // zero this rank's slot in every owner's landing buffer
      const int64_t* L = p->layout.data();
      const int n = p->nranks;
      const int64_t block = L[kLayoutPerRank * n];
      for (int r = 0; r < n; r++)
        CUDA_TRY(cudaMemsetAsync((char*)p->peer_land[r] + (size_t)p->rank * block * csize(p->precision), 0,
                                 (size_t)block * csize(p->precision), st));
      return HOS_OK;
    }
    CUDA_TRY(cudaMemsetAsync(raw_dev, 0, zero_bytes, st));
    return HOS_OK;
  }
  // front end on the shard only, written at its own segment rows
  const size_t rs = rsize(p->precision);
  void* seg = (char*)p->d_seg + (size_t)seg_begin * p->m * rs;
  void* half = (char*)p->d_half + (size_t)seg_begin * p->hstride * csize(p->precision);
  void* E = (char*)p->d_E + (size_t)seg_begin * p->Lp * csize(p->precision);
  if (p->fused) {
    if ((rc = fused_front(p, x_dev, x_dtype, 0, seg_begin, nseg, 1, st, false))) return rc;
  } else {
    CUDA_TRY(hos::launch_prep(x_dev, x_dtype, 0, p->m, seg_begin, nseg, 1, p->taper, p->d_taper, p->precision, seg,
                              st));
    if ((rc = run_fft(p, nseg, seg, half, st))) return rc;
    CUDA_TRY(hos::launch_extend_half(half, p->m, p->hstride, nseg, nullptr, p->geo.f_lo, p->L, p->Lp, p->precision,
                                     E, st, 0));
  }
  int n = nctas_for(p, nseg, 1);
  while (n > 1 && slots_needed(p, nseg, n, 1) > p->maxslots) n--;
  const hos::TripleArgs ta = triple_args(p, seg_begin, seg_end, n, 1);
  CUDA_TRY(hos::launch_triple(ta, p->precision, st));
  CUDA_TRY(hos::launch_reduce_parts(p->d_part, p->geo.ncells, slot_info(p, nseg, n), p->d_line_start, p->geo.nlines,
                                    p->geo.win.lo, p->precision, raw_dev, st, dst_line, dst_addr));
  return HOS_OK;
}

int hos_smooth_raw(hos_plan* p, const void* raw_dev, int64_t line_begin, int row_begin, int row_end, void* out_dev,
                   void* stream) {
  int rc = check_plan(p);
  if (rc) return rc;
  PlanGuard guard_(p);
  if (p->batch != 1) return fail(HOS_EPARAM, "hos_smooth_raw needs a batch-1 plan");
  if (!raw_dev || !out_dev) return fail(HOS_EPARAM, "null buffer");
  int64_t lb = 0, le = 0;
  if ((rc = hos_rows_line_range(p, row_begin, row_end, &lb, &le))) return rc;
  if (row_end == row_begin) return HOS_OK;
  if (line_begin > lb)
    return fail(HOS_EPARAM, "raw buffer starts at line " + std::to_string(line_begin) + " but rows need line " +
                                std::to_string(lb));
  cudaStream_t st = (cudaStream_t)stream;
  const hos::Geometry& g = p->geo;
  // raw_dev holds cells of lines [line_begin, le); scan lines [lb, le)
  const int64_t cell0 = g.line_start[line_begin];
  const char* raw_lb = (const char*)raw_dev + (size_t)(g.line_start[lb] - cell0) * csize(p->precision);
  double* S = p->d_S;  // scratch: cells of lines [lb, le)
  hos::SlotInfo plain{};
  CUDA_TRY(hos::launch_line_scan(raw_lb, 1, 0, plain, p->precision, p->d_line_start, lb, le - lb, 0, 1, S, st,
                                 p->max_line));
  hos::BoxArgs b{};
  b.S = S;
  b.s_series_stride = 0;
  b.line_base = lb;
  b.line_start = p->d_line_start;
  b.cell_base = g.line_start[lb];
  b.row_off = p->d_row_off;
  b.rows = g.rows;
  b.pair_k1 = p->d_pair_k1;
  b.pair_k2 = p->d_pair_k2;
  b.pair_base = p->d_pair_base;
  b.npairs = (int)g.pair_k1.size();
  b.line_of_ab = p->d_line_of_ab;
  b.b_count = g.b_count;
  b.lo = g.win.lo;
  b.hi = g.win.hi;
  b.m3 = p->m3;
  b.order = p->order;
  b.m = p->m;
  b.row_begin = row_begin;
  b.row_end = row_end;
  b.pair_begin = p->order == 4 ? g.row_pair0[row_begin] : 0;
  b.pair_end = p->order == 4 ? g.row_pair0[row_end] : 0;
  b.p_begin = g.row_off[row_begin];
  b.p_end = g.row_off[row_end];
  b.scale = 1.0 / ((double)p->m * (double)p->k * std::pow((double)p->m3, p->order - 1));
  b.out = out_dev;
  b.out_series_stride = 0;
  b.precision = p->precision;
  b.batch = 1;
  CUDA_TRY(hos::launch_box(b, st));
  return HOS_OK;
}

int64_t hos_row_point_offset(const hos_plan* p, int row) {
  if (!p || row < 0 || row > p->geo.rows) return -1;
  return p->geo.row_off[row];
}

int hos_rows_line_range(const hos_plan* p, int row_begin, int row_end, int64_t* lb, int64_t* le) {
  int rc = check_plan(p);
  if (rc) return rc;
  if (!(0 <= row_begin && row_begin <= row_end && row_end <= p->geo.rows))
    return fail(HOS_EPARAM, "row range outside the domain");
  const hos::Geometry& g = p->geo;
  if (p->order == 3) {
    *lb = row_begin;
    *le = row_end == row_begin ? row_begin : row_end - 1 + (p->m3 - 1) + 1;
  } else {
    // lines are a-major: first line with a >= row_begin + lo, first line with a > row_end - 1 + hi
    int64_t b = 0, e = 0;
    const int alo = row_begin + g.win.lo, ahi = row_end - 1 + g.win.hi;
    while (b < g.nlines && g.line_a[b] < alo) b++;
    e = b;
    while (e < g.nlines && g.line_a[e] <= ahi) e++;
    *lb = b;
    *le = row_end == row_begin ? b : e;
  }
  return HOS_OK;
}

namespace {
// FMA-pipe peak microbenchmark on the current device: precision 32 = FFMA2
// (2 lane FMAs per instruction), 64 = DFMA; flops counted as 2 per FMA
int peak_probe(int precision, double* tflops, double* sm_mhz, void* stream) {
  if (!tflops || !sm_mhz) return fail(HOS_EPARAM, "null output");
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0, sms = 148;
  CUDA_TRY(cudaGetDevice(&dev));
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = sms * 4, iters = precision == 32 ? 4096 : 512;
  void* buf = nullptr;
  unsigned long long* clk = nullptr;
  CUDA_TRY(cudaMalloc(&buf, (size_t)blocks * 256 * 8));
  CUDA_TRY(cudaMalloc(&clk, 16));
  auto launch = [&]() {
    return precision == 32 ? hos::launch_peak_fp32((float2*)buf, blocks, iters, st)
                           : hos::launch_peak_fp64((double*)buf, blocks, iters, st);
  };
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  CUDA_TRY(launch());  // warm-up
  float best = 1e30f;
  for (int r = 0; r < 5; r++) {
    cudaEventRecord(a, st);
    CUDA_TRY(launch());
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  // SM clock while the probe kernel is resident alongside a loaded device
  CUDA_TRY(launch());
  CUDA_TRY(hos::launch_clock_probe(clk, 20000000, st));
  unsigned long long h[2] = {0, 0};
  CUDA_TRY(cudaMemcpyAsync(h, clk, 16, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  const double fmas_per_thread_iter = precision == 32 ? 32 * 2 : 32;
  const double flops = (double)blocks * 256 * iters * fmas_per_thread_iter * 2;
  *tflops = flops / (best * 1e-3) / 1e12;
  *sm_mhz = h[1] ? (double)h[0] / ((double)h[1] * 1e-3) : 0.0;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(buf);
  cudaFree(clk);
  return HOS_OK;
}
}  // namespace

int hos_peak_fp32(double* tflops, double* sm_mhz, void* stream) { return peak_probe(32, tflops, sm_mhz, stream); }
int hos_peak_fp64(double* tflops, double* sm_mhz, void* stream) { return peak_probe(64, tflops, sm_mhz, stream); }

int hos_plan_nctas(const hos_plan* p) { return p ? p->nctas : -1; }
int hos_plan_k2_kind(const hos_plan* p) { return p ? (p->cta ? 1 : 0) : -1; }

int hos_plan_set_trace(hos_plan* p, void* trace_dev) {
  int rc = check_plan(p);
  if (rc) return rc;
  p->trace = (unsigned long long*)trace_dev;
  return HOS_OK;
}

int hos_plan_set_stamps(hos_plan* p, void* stamps_dev) {
  int rc = check_plan(p);
  if (rc) return rc;
  PlanGuard guard_(p);
  CUDA_TRY(hos::set_stamp_buffer((unsigned long long*)stamps_dev));
  return HOS_OK;
}

int hos_plan_set_timing(hos_plan* p, int enable) {
  int rc = check_plan(p);
  if (rc) return rc;
  p->timing = enable ? 1 : 0;
  p->timed = false;
  return HOS_OK;
}

int hos_plan_kernel_ms(const hos_plan* p, double* triple_ms, double* total_ms) {
  int rc = check_plan(p);
  if (rc) return rc;
  if (!p->timed) return fail(HOS_EPARAM, "no timed call recorded (enable timing first)");
  float t1 = 0, t2 = 0;
  CUDA_TRY(cudaEventSynchronize(p->ev[6]));
  CUDA_TRY(cudaEventElapsedTime(&t1, p->ev[3], p->ev[4]));
  CUDA_TRY(cudaEventElapsedTime(&t2, p->ev[0], p->ev[6]));
  if (triple_ms) *triple_ms = t1;
  if (total_ms) *total_ms = t2;
  return HOS_OK;
}

int hos_plan_time_stages(hos_plan* p, const void* x_dev, int x_dtype, int64_t x_stride, void* out_dev, int reps,
                         double* ms6, void* stream) {
  int rc = check_plan(p);
  if (rc) return rc;
  PlanGuard guard_(p);
  if ((rc = check_dtype_x(x_dtype))) return rc;
  if (!ms6 || reps < 1) return fail(HOS_EPARAM, "null output or reps < 1");
  cudaStream_t st = (cudaStream_t)stream;
  const int saved = p->timing;
  p->timing = 0;
  rc = hos_estimate(p, x_dev, x_dtype, x_stride, out_dev, stream);  // fills every intermediate buffer
  p->timing = saved;
  if (rc) return rc;
  const int rows = p->batch * p->k;
  cudaEvent_t e0, e1;
  CUDA_TRY(cudaEventCreate(&e0));
  CUDA_TRY(cudaEventCreate(&e1));
  // each stage: `reps` launches captured into one CUDA graph (device-paced, as
  // in the estimate graph; back-to-back host launches would measure the
  // host's launch rate for the short stages), one warm replay, one timed replay
  auto launch_stage = [&](int s, cudaStream_t cs) -> int {
    cudaError_t e = cudaSuccess;
    int r2 = HOS_OK;
    switch (s) {
      case 0:
        if (p->fused)
          r2 = fused_front(p, x_dev, x_dtype, x_stride, 0, p->k, p->batch, cs, p->quad);
        else
          e = hos::launch_prep(x_dev, x_dtype, x_stride, p->m, 0, p->k, p->batch, p->taper, p->d_taper, p->precision,
                               p->d_seg, cs);
        break;
      case 1:
        if (!p->fused) r2 = run_fft(p, rows, p->d_seg, p->d_half, cs);
        break;
      case 2:
        if (!p->fused)
          e = hos::launch_extend_half(p->d_half, p->m, p->hstride, rows, nullptr, p->geo.f_lo, p->L, p->Lp,
                                      p->precision, p->d_E, cs, p->quad);
        break;
      case 3:
        e = launch_main_triple(p, cs);
        break;
      case 4:
        r2 = run_smooth(p, out_dev, cs, 4);
        break;
      default:
        r2 = run_smooth(p, out_dev, cs, 5);
    }
    if (e != cudaSuccess) return fail(HOS_ECUDA, std::string("CUDA error: ") + cudaGetErrorString(e));
    return r2;
  };
  for (int s = 0; s < 6 && !rc; s++) {
    if ((p->fused && (s == 1 || s == 2)) || (s == 5 && p->series_k4)) {
      ms6[s] = 0.0;
      continue;
    }
    cudaGraph_t graph = nullptr;
    CUDA_TRY(cudaStreamBeginCapture(p->cap, cudaStreamCaptureModeThreadLocal));
    for (int r = 0; r < reps && !rc; r++) rc = launch_stage(s, p->cap);
    cudaError_t ce = cudaStreamEndCapture(p->cap, &graph);
    if (rc) {
      if (graph) cudaGraphDestroy(graph);
      break;
    }
    CUDA_TRY(ce);
    cudaGraphExec_t exec = nullptr;
    ce = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    CUDA_TRY(ce);
    CUDA_TRY(cudaGraphLaunch(exec, st));
    CUDA_TRY(cudaEventRecord(e0, st));
    CUDA_TRY(cudaGraphLaunch(exec, st));
    CUDA_TRY(cudaEventRecord(e1, st));
    CUDA_TRY(cudaEventSynchronize(e1));
    cudaGraphExecDestroy(exec);
    float ms = 0;
    CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
    ms6[s] = ms / reps;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return rc;
}

int hos_plan_stage_ms(const hos_plan* p, double* ms6) {
  int rc = check_plan(p);
  if (rc) return rc;
  if (!p->timed) return fail(HOS_EPARAM, "no timed call recorded (enable timing first)");
  if (!ms6) return fail(HOS_EPARAM, "null output");
  CUDA_TRY(cudaEventSynchronize(p->ev[6]));
  for (int i = 0; i < 6; i++) {
    float t = 0;
    CUDA_TRY(cudaEventElapsedTime(&t, p->ev[i], p->ev[i + 1]));
    ms6[i] = t;
  }
  return HOS_OK;
}

int hos_shard_layout(int order, int m, int k, int m3, int nranks, int64_t* out) {
  if (!out) return fail(HOS_EPARAM, "null output");
  if (nranks < 1 || k < 1) return fail(HOS_EPARAM, "nranks and k must be positive");
  hos::Geometry g;
  const std::string err = g.build(order, m, m3);
  if (!err.empty()) return fail(HOS_EPARAM, err);
  const std::vector<int64_t> rec = shard_layout(g, order, m3, k, nranks);
  std::memcpy(out, rec.data(), rec.size() * sizeof(int64_t));
  return HOS_OK;
}

int hos_cta_schedule_check(int order, int m, int k, int m3, int precision, int batch, int sms, int interleave,
                           int64_t* stats) {
  if (!stats) return fail(HOS_EPARAM, "null output");
  if (m < 1 || k < 1 || batch < 1 || sms < 2 || (precision != 32 && precision != 64))
    return fail(HOS_EPARAM, "bad shape");
  hos_plan p;  // host fields only: no device resources
  p.order = order;
  p.m = m;
  p.k = k;
  p.m3 = m3;
  p.precision = precision;
  p.batch = batch;
  p.sms = sms;
  std::string err = build_geometry(p.geo, order, m, m3, precision);
  if (!err.empty()) return fail(HOS_EPARAM, err);
  p.Lp = pitch_of(p.geo);
  const hos::Geometry& g = p.geo;
  CtaSchedule cs;
  const int nf = interleave ? std::max(1, sms - stream_front_ctas()) : 0;
  for (int i = 0; i < 12; i++) stats[i] = 0;
  if (!build_cta_schedule(&p, cs, nf)) return HOS_OK;  // not eligible: stats[0] = 0
  const int R = g.nregions, W = hos::cta_warps(want_quad(precision));
  auto bad = [&](const std::string& why) { return fail(HOS_EDATA, "schedule check: " + why); };
  if ((int)cs.cta_stage0.size() != cs.nctas + 1 || cs.cta_stage0.front() != 0 ||
      cs.cta_stage0.back() != (int)cs.stages.size())
    return bad("CTA stage ranges");
  if (cs.nctas > sms) return bad("more CTAs than SMs");
  // every (series, group, segment) exactly once; stages inside their block's series
  const int ng = (int)cs.groups.size();
  std::vector<uint8_t> seen((size_t)batch * ng * k, 0);
  int64_t smax = 0, smin = INT64_MAX;
  std::vector<int> blk_cta(cs.blocks.size(), -1);
  for (int c = 0; c < cs.nctas; c++) {
    const int64_t n = cs.cta_stage0[c + 1] - cs.cta_stage0[c];
    smax = std::max(smax, n);
    smin = std::min(smin, n);
    for (int j = cs.cta_stage0[c]; j < cs.cta_stage0[c + 1]; j++) {
      const hos::CtaStage& st = cs.stages[j];
      if (st.block < 0 || st.block >= (int)cs.blocks.size()) return bad("stage block index");
      if (blk_cta[st.block] >= 0 && blk_cta[st.block] != c) return bad("block shared by two CTAs");
      blk_cta[st.block] = c;
      const hos::CtaBlock& b = cs.blocks[st.block];
      if (st.nseg < 1 || st.nseg > cs.stage_segs) return bad("stage size");
      for (int t = 0; t < st.nseg; t++) {
        const int row = st.row + t;
        if (row / k != b.series || b.series < 0 || b.series >= batch) return bad("stage outside its series");
        uint8_t& v = seen[((size_t)b.series * ng + b.group) * k + row % k];
        if (v) return bad("segment covered twice");
        v = 1;
      }
    }
  }
  for (uint8_t v : seen)
    if (!v) return bad("segment not covered");
  // roles: n x halves x phases warps; slot ranges of a (series, group) disjoint and counted
  std::vector<int> used((size_t)batch * ng, 0);
  for (const hos::CtaBlock& b : cs.blocks) {
    const hos::CtaGroup& gr = cs.groups[b.group];
    if (gr.n * gr.halves * gr.phases > W || gr.n < 1) return bad("group roles exceed the CTA's warps");
    if (gr.halves == 2 && g.tiles_per_region != 2) return bad("halves without tile pairs");
    int& u = used[(size_t)b.series * ng + b.group];
    if (b.slot_base != u) return bad("slot bases not consecutive");
    u += gr.phases;
  }
  for (int b = 0; b < batch; b++)
      for (int gi = 0; gi < ng; gi++)
        for (int r = cs.groups[gi].r0; r < cs.groups[gi].r0 + cs.groups[gi].n; r++) {
          const int want = used[(size_t)b * ng + gi];
          const int have = cs.region_slots[(size_t)(interleave ? 0 : b) * R + r];
          if (have != want || have > cs.maxslots) return bad("region slot counts");
        }
  stats[0] = cs.nctas;
  stats[1] = (int64_t)cs.stages.size();
  stats[2] = smax;
  stats[3] = smin;
  stats[4] = cs.maxslots;
  stats[5] = g.tile_step;
  stats[6] = cs.depth;
  stats[7] = ng;
  stats[8] = R;
  stats[9] = (int64_t)cs.blocks.size();
  stats[10] = cs.stage_segs;
  stats[11] = cs.slot_bytes;
  return HOS_OK;
}

int hos_comm_attach(hos_plan* p, void* nccl_comm, int rank, int nranks) {
  int rc = check_plan(p);
  if (rc) return rc;
  PlanGuard guard_(p);
  if (p->batch != 1) return fail(HOS_EPARAM, "multi-GPU estimates need a batch-1 plan");
  std::string why;
  const NcclApi* api = nccl_api(&why);
  if (!api) return fail(HOS_ECUDA, why);
  if (!nccl_comm || nranks < 1 || rank < 0 || rank >= nranks) return fail(HOS_EPARAM, "bad communicator/rank");
  int cnt = 0, me = 0;
  NCCL_TRY(api, api->comm_count((ncclComm_t)nccl_comm, &cnt));
  NCCL_TRY(api, api->comm_rank((ncclComm_t)nccl_comm, &me));
  if (cnt != nranks || me != rank)
    return fail(HOS_EPARAM, "communicator has rank " + std::to_string(me) + " of " + std::to_string(cnt) +
                                ", caller said " + std::to_string(rank) + " of " + std::to_string(nranks));
  if (cudaSetDevice(p->device) != cudaSuccess) return fail(HOS_ECUDA, "cannot select the plan's device");
  for (void* b : {p->d_raw, p->d_send, p->d_mine, p->d_local, p->d_heads, p->d_vals, p->d_parts})
    if (b) cudaFree(b);
  p->layout = shard_layout(p->geo, p->order, p->m3, p->k, nranks);
  const int64_t* L = p->layout.data();
  const int64_t block = L[kLayoutPerRank * nranks], halo = L[kLayoutPerRank * nranks + 1];
  const bool in_next = L[kLayoutPerRank * nranks + 2] != 0;
  int64_t pmax = 1, local = 1;
  for (int r = 0; r < nranks; r++) {
    const int64_t* R = L + kLayoutPerRank * r;
    pmax = std::max(pmax, R[13] - R[12]);
    local = std::max(local, std::max(R[11], R[9]) - R[8]);
    local = std::max(local, block + halo);  // the reduce-scatter lands a whole padded block at its head
  }
  const size_t cs = csize(p->precision);
  const int64_t heads = in_next ? halo : block;
  if ((rc = alloc(p, &p->d_raw, (size_t)p->geo.ncells * cs)) || (rc = alloc(p, &p->d_send, (size_t)nranks * block * cs)) ||
      (rc = alloc(p, &p->d_mine, (size_t)block * cs)) || (rc = alloc(p, &p->d_local, (size_t)local * cs)) ||
      (rc = alloc(p, &p->d_heads, (size_t)nranks * heads * cs)) || (rc = alloc(p, &p->d_vals, (size_t)pmax * cs)) ||
      (rc = alloc(p, &p->d_parts, (size_t)nranks * pmax * cs)))
    return rc;
  {  // line -> padded send-buffer position: owner r's cells start at r * block
    std::vector<int64_t> dl(p->geo.nlines);
    int r = 0;
    for (int64_t l = 0; l < p->geo.nlines; l++) {
      while (r + 1 < nranks && l >= L[kLayoutPerRank * r + 5]) r++;  // own_l1 of rank r
      dl[l] = (int64_t)r * block + (p->geo.line_start[l] - L[kLayoutPerRank * r + 8]);
    }
    if (p->d_send_line) cudaFree(p->d_send_line);
    p->d_send_line = nullptr;
    if ((rc = upload(p, &p->d_send_line, dl))) return rc;
  }
  if ((rc = setup_p2p(p, api, (ncclComm_t)nccl_comm, rank, nranks))) return rc;
  p->comm = nccl_comm;
  p->rank = rank;
  p->nranks = nranks;
  return HOS_OK;
}

int estimate_distributed_body(hos_plan* p, const void* x_dev, int x_dtype, void* out_dev, void* stream);

int hos_estimate_distributed(hos_plan* p, const void* x_dev, int x_dtype, void* out_dev, void* stream) {
  int rc = check_plan(p);
  if (rc) return rc;
  PlanGuard guard_(p);
  if (!p->comm) return fail(HOS_EPARAM, "no communicator attached (hos_comm_attach)");
  if (!x_dev || !out_dev) return fail(HOS_EPARAM, "null buffer");
  if ((rc = check_dtype_x(x_dtype))) return rc;
  // the ~20 small copies, kernels and NCCL collectives of a step replay as one
  // CUDA graph per buffer binding (NCCL operations are capturable)
  const char* env = std::getenv("HOS_DIST_GRAPH");
  if (p->use_graphs && !p->timing && !(env && env[0] == '0')) {
    const hos_plan::GraphKey key{4, x_dev, x_dtype, 0, out_dev};
    return run_graph(p, key, (cudaStream_t)stream,
                     [&](cudaStream_t s) { return estimate_distributed_body(p, x_dev, x_dtype, out_dev, s); });
  }
  return estimate_distributed_body(p, x_dev, x_dtype, out_dev, stream);
}

int estimate_distributed_body(hos_plan* p, const void* x_dev, int x_dtype, void* out_dev, void* stream) {
  int rc = HOS_OK;
  const NcclApi* api = nccl_api(nullptr);
  cudaStream_t st = (cudaStream_t)stream;
  ncclComm_t comm = (ncclComm_t)p->comm;
  const int n = p->nranks, me = p->rank;
  const int64_t* L = p->layout.data();
  const int64_t* R = L + kLayoutPerRank * me;
  const int64_t block = L[kLayoutPerRank * n], halo = L[kLayoutPerRank * n + 1];
  const bool in_next = L[kLayoutPerRank * n + 2] != 0;
  const size_t cs = csize(p->precision);
  const ncclDataType_t dt = p->precision == 32 ? ncclFloat32 : ncclFloat64;  // complex as 2 reals
  // 1. partial raw sums of this rank's segments over all of D_h, reduced from
  // K2's slots straight into the padded reduce-scatter send buffer (rank r's
  // owned cells at r * block; the padding is never written -- what NCCL sums
  // into the padded tail of the received block is never read)
  const int64_t oc0 = R[8], oc1 = R[9], nc1 = R[11];
  char* local = (char*)p->d_local;
  if (p->p2p) {
    // 1+2 fused: the slot reduction stores each owner's cells straight into
    // its landing slot `me` over NVLink (peer stores from the epilogue
    // kernel); a barrier (all-gather of one float per rank) orders them
    // before every owner adds its nranks slots in rank order
    if ((rc = partial_raw_impl(p, x_dev, x_dtype, (int)R[0], (int)R[1], nullptr, st, nullptr, 0, p->d_p2p_line)))
      return rc;
    NCCL_TRY(api, api->all_gather((char*)p->d_bar + (size_t)me * 4, p->d_bar, 1, ncclFloat32, comm, st));
    CUDA_TRY(hos::launch_sum_land(p->d_land, n, block, oc1 - oc0, p->precision, local, st));
  } else {
    if ((rc = partial_raw_impl(p, x_dev, x_dtype, (int)R[0], (int)R[1], p->d_send, st, p->d_send_line,
                               (size_t)n * block * cs)))
      return rc;
    // 2. reduce-scatter by owned line blocks, straight into the head of the
    // local lines (own block, then the halo past it)
    NCCL_TRY(api, api->reduce_scatter(p->d_send, local, (size_t)block * 2, dt, ncclSum, comm, st));
  }
  const int64_t need = std::max<int64_t>(0, nc1 - oc1);
  if (in_next) {
    // 3. halo: the w-1 lines past the own block are the head of rank me+1's
    // block -- one send/recv pair per neighbour
    const int64_t need_prev = me > 0 ? std::max<int64_t>(0, L[kLayoutPerRank * (me - 1) + 11] -
                                                                L[kLayoutPerRank * (me - 1) + 9])
                                     : 0;
    NCCL_TRY(api, api->group_start());
    if (need) NCCL_TRY(api, api->recv(local + (size_t)(oc1 - oc0) * cs, (size_t)need * 2, dt, me + 1, comm, st));
    if (need_prev) NCCL_TRY(api, api->send(local, (size_t)need_prev * 2, dt, me - 1, comm, st));
    NCCL_TRY(api, api->group_end());
  } else {  // halo spans several ranks' blocks: gather every block
    NCCL_TRY(api, api->all_gather(local, p->d_heads, (size_t)block * 2, dt, comm, st));
    for (int r = me + 1; r < n; r++) {
      const int64_t* Q = L + kLayoutPerRank * r;
      const int64_t lo = std::max(Q[8], oc1), hi = std::min(Q[9], nc1);
      if (lo < hi)
        CUDA_TRY(cudaMemcpyAsync(local + (size_t)(lo - oc0) * cs, (char*)p->d_heads + ((size_t)r * block + lo - Q[8]) * cs,
                                 (size_t)(hi - lo) * cs, cudaMemcpyDeviceToDevice, st));
    }
  }
  // 4. smooth this rank's output rows, 5. all-gather the lexicographic slices
  int64_t pmax = 1;
  for (int r = 0; r < n; r++) pmax = std::max(pmax, L[kLayoutPerRank * r + 13] - L[kLayoutPerRank * r + 12]);
  if (R[3] > R[2]) {
    if ((rc = hos_smooth_raw(p, local, R[4], (int)R[2], (int)R[3], p->d_vals, stream))) return rc;
  }
  NCCL_TRY(api, api->all_gather(p->d_vals, p->d_parts, (size_t)pmax * 2, dt, comm, st));
  for (int r = 0; r < n; r++) {
    const int64_t* Q = L + kLayoutPerRank * r;
    if (Q[13] > Q[12])
      CUDA_TRY(cudaMemcpyAsync((char*)out_dev + (size_t)Q[12] * cs, (char*)p->d_parts + (size_t)r * pmax * cs,
                               (size_t)(Q[13] - Q[12]) * cs, cudaMemcpyDeviceToDevice, st));
  }
  return HOS_OK;
}

}  // extern "C"
