// Host-side geometry of the direct-method estimator: the principal domain
// P (hospectra/spectra.py:133-168), its window dilation D_h (the raw cells
// the smoothing reads, SURVEY §8 notation) laid out as CSR "lines", and
// the 16 x 32 tiles (paired into K2 regions) that cover D_h.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#ifdef __CUDACC__
#define HOS_HD __host__ __device__
#else
#define HOS_HD
#endif

namespace hos {

// Window offsets per axis: [lo, hi] = [-m3/2, m3-1-m3/2]
// (hospectra/spectra.py:8-11,395).
struct Window {
  int m3, lo, hi;
  explicit Window(int w) : m3(w), lo(-(w / 2)), hi(w - 1 - w / 2) {}
};

// Output rows of the order-3 domain: k1 in [0, (m-1)/2], row length
// min(k1, (m-2k1-1)/2)+1 (hospectra/spectra.py:146-147).
HOS_HD inline int p3_rows(int m) { return (m - 1) / 2 + 1; }
HOS_HD inline int p3_len(int m, int k1) {
  int a = k1, b = (m - 2 * k1 - 1);
  b = b >= 0 ? b / 2 : -((-b + 1) / 2);  // floor division like Python
  return (a < b ? a : b) + 1;
}
// Order-4 k3 count for pair (k1,k2) (hospectra/spectra.py:155-158).
HOS_HD inline int p4_len(int m, int k1, int k2) {
  int b = m - 2 * k1 - 2 * k2 - 1;
  b = b >= 0 ? b / 2 : -((-b + 1) / 2);
  return (k2 < b ? k2 : b) + 1;
}

int64_t domain_size(int order, int m);
// rows [start, stop) of the lexicographic domain into out ((stop-start) x (order-1))
void domain_rows(int order, int m, int64_t start, int64_t stop, int32_t* out);

// K2 work decomposition.  D_h is cut into TILES of up to tile_rows
// consecutive lines (a "band" of one plane) x tile_cols columns, listed band
// after band; consecutive tiles are grouped into REGIONS of 1024 cells (a
// warp's unit of work, 32 cells per lane).  The tile shape follows the K2
// lane step S (hos_kernels.cu): tiles of 4S lines x 8S columns, 32/S^2 per
// region -- S = 4: 16 x 32 tiles in pairs (large M), S = 2: 8 x 16 tiles in
// groups of 8 (small M, where D_h's lines are short and large tiles are
// mostly empty).  The last region is completed with empty tiles (nrows 0)
// that mirror its last real tile, so their staged loads stay in range.
constexpr int kRegionCells = 1024;

struct Tile {
  int32_t line0;      // first line of the band
  int32_t nrows;      // lines in the band (<= tile_rows; 0: empty filler tile)
  int32_t row_freq0;  // frequency of line0's row factor (order 3: a, order 4: b)
  int32_t plane_freq; // order 4: a of the plane; order 3: 0
  int32_t col0;       // first column of the tile
};

struct Geometry {
  int order = 3, m = 0, m3 = 1;
  Window win{1};
  // principal domain
  int64_t npoints = 0;
  int rows = 0;                     // order 3: k1 rows; order 4: k1 planes
  std::vector<int64_t> row_off;     // rows+1: lexicographic offset of each k1
  // order 4 pair table (k1,k2) with k3 count and lexicographic base
  std::vector<int32_t> pair_k1, pair_k2, pair_n3;
  std::vector<int64_t> pair_base;
  std::vector<int32_t> row_pair0;   // order 4: first pair index of plane k1 (rows+1)
  // dilated domain D_h as lines (CSR)
  int64_t nlines = 0, ncells = 0;
  std::vector<int32_t> line_a, line_b;  // logical row / pair coordinates (b = 0 for order 3)
  std::vector<int32_t> line_cmax;       // last logical column; first column is win.lo
  std::vector<int64_t> line_start;      // nlines+1
  // order 4: dense (a,b) -> line lookup over [lo, amax] x [lo, bmax]
  int a_count = 0, b_count = 0;
  std::vector<int32_t> line_of_ab;
  // order 3: line index = a - lo; lines of output row k1 start at k1
  // frequencies any region reads (inclusive), for the extended spectrum
  int f_lo = 0, f_hi = 0;
  // K2 tiles and regions
  int tile_step = 4, tile_rows = 16, tile_cols = 32, tiles_per_region = 2;
  std::vector<Tile> tiles;            // band-major, padded to whole regions (region r = tiles r*NT ..)
  int ntiles = 0;                     // real tiles
  int nregions = 0;
  std::vector<int32_t> line_tile0;    // per line: index of the tile holding its first column
  int64_t issued_cells = 0;           // cells computed by K2 (regions x 1024)

  // first_band (order 3): lines in the first band (1..tile_rows; 0 = tile_rows) -- shifts every
  // later band, which changes how D_h's staircase edges fall into tiles
  std::string build(int order, int m, int m3, int tile_step = 4, int first_band = 0);  // "" or an error
};

}  // namespace hos
