// Geometry of P, D_h and the K2 regions (see hos_geometry.h).
#include "hos_geometry.h"

#include <algorithm>
#include <cstdio>

namespace hos {

int64_t domain_size(int order, int m) {
  int64_t n = 0;
  const int rows = p3_rows(m);
  for (int k1 = 0; k1 < rows; k1++) {
    const int n2 = p3_len(m, k1);
    if (order == 3) {
      n += n2 > 0 ? n2 : 0;
    } else {
      for (int k2 = 0; k2 < n2; k2++) {
        const int n3 = p4_len(m, k1, k2);
        n += n3 > 0 ? n3 : 0;
      }
    }
  }
  return n;
}

void domain_rows(int order, int m, int64_t start, int64_t stop, int32_t* out) {
  // walk the lexicographic enumeration, emitting [start, stop)
  int64_t t = 0;
  const int rows = p3_rows(m);
  const int d = order - 1;
  for (int k1 = 0; k1 < rows && t < stop; k1++) {
    const int n2 = p3_len(m, k1);
    if (order == 3) {
      if (n2 <= 0) continue;
      if (t + n2 <= start) { t += n2; continue; }
      for (int k2 = 0; k2 < n2 && t < stop; k2++, t++) {
        if (t < start) continue;
        out[(t - start) * d + 0] = k1;
        out[(t - start) * d + 1] = k2;
      }
    } else {
      for (int k2 = 0; k2 < n2 && t < stop; k2++) {
        const int n3 = p4_len(m, k1, k2);
        if (n3 <= 0) continue;
        if (t + n3 <= start) { t += n3; continue; }
        for (int k3 = 0; k3 < n3 && t < stop; k3++, t++) {
          if (t < start) continue;
          out[(t - start) * d + 0] = k1;
          out[(t - start) * d + 1] = k2;
          out[(t - start) * d + 2] = k3;
        }
      }
    }
  }
}

namespace {
struct RegionRec {
  int line0, nrows, row_freq0, plane_freq, col0;
};

void add_band_regions(std::vector<RegionRec>& regs, std::vector<int32_t>& line_tile0, int line0, int nrows,
                      int row_freq0, int plane_freq, int lo, int cmax_band, int tile_cols) {
  const int ncols = cmax_band - lo + 1;
  const int nr = (ncols + tile_cols - 1) / tile_cols;
  for (int l = line0; l < line0 + nrows; l++) line_tile0[l] = (int32_t)regs.size();
  for (int r = 0; r < nr; r++) regs.push_back({line0, nrows, row_freq0, plane_freq, lo + r * tile_cols});
}

}  // namespace

std::string Geometry::build(int order_, int m_, int m3_, int tile_step_, int first_band) {
  order = order_;
  m = m_;
  m3 = m3_;
  win = Window(m3);
  if (order != 3 && order != 4) return "order must be 3 or 4, got " + std::to_string(order);
  if (m < 2) return "segment length must be >= 2, got " + std::to_string(m);
  if (m3 < 1) return "smoothing window must be >= 1, got " + std::to_string(m3);
  if (tile_step_ != 2 && tile_step_ != 4) return "tile step must be 2 or 4";
  tile_step = tile_step_;
  tile_rows = 4 * tile_step;
  tile_cols = 8 * tile_step;
  tiles_per_region = 32 / (tile_step * tile_step);
  if (2 * m3 >= m)
    return "smoothing window " + std::to_string(m3) + " must satisfy m3 < m/2 (segment length m = " +
           std::to_string(m) + ")";
  const int lo = win.lo, hi = win.hi;
  rows = p3_rows(m);

  // ---- principal domain offsets
  row_off.assign(rows + 1, 0);
  pair_k1.clear(); pair_k2.clear(); pair_n3.clear(); pair_base.clear();
  row_pair0.assign(rows + 1, 0);
  int64_t t = 0;
  for (int k1 = 0; k1 < rows; k1++) {
    row_off[k1] = t;
    row_pair0[k1] = (int32_t)pair_k1.size();
    const int n2 = p3_len(m, k1);
    if (order == 3) {
      t += std::max(n2, 0);
    } else {
      for (int k2 = 0; k2 < n2; k2++) {
        const int n3 = p4_len(m, k1, k2);
        if (n3 <= 0) continue;
        pair_k1.push_back(k1);
        pair_k2.push_back(k2);
        pair_n3.push_back(n3);
        pair_base.push_back(t);
        t += n3;
      }
    }
  }
  row_off[rows] = t;
  row_pair0[rows] = (int32_t)pair_k1.size();
  npoints = t;

  // ---- order-3 dilation: raw rows a in [lo, rows-1+hi], cols [lo, cmax3(a)]
  const int n3lines = rows + m3 - 1;
  std::vector<int32_t> cmax3(n3lines);
  for (int l = 0; l < n3lines; l++) {
    const int a = lo + l;
    int best = -1;
    for (int k1 = std::max(0, a - hi); k1 <= std::min(rows - 1, a - lo); k1++)
      best = std::max(best, p3_len(m, k1) - 1);
    cmax3[l] = best + hi;
  }

  line_a.clear(); line_b.clear(); line_cmax.clear(); line_start.clear();
  line_tile0.clear();
  issued_cells = 0;
  std::vector<RegionRec> regs;
  if (order == 3) {
    nlines = n3lines;
    line_start.push_back(0);
    for (int l = 0; l < n3lines; l++) {
      line_a.push_back(lo + l);
      line_b.push_back(0);
      line_cmax.push_back(cmax3[l]);
      line_start.push_back(line_start.back() + (cmax3[l] - lo + 1));
    }
    ncells = line_start.back();
    line_tile0.assign(n3lines, 0);
    const int fb = first_band >= 1 && first_band <= tile_rows ? first_band : tile_rows;
    for (int l0 = 0; l0 < n3lines; l0 += (l0 == 0 ? fb : tile_rows)) {
      const int nr = std::min(l0 == 0 ? fb : tile_rows, n3lines - l0);
      int cb = lo;
      for (int l = l0; l < l0 + nr; l++) cb = std::max(cb, (int)cmax3[l]);
      add_band_regions(regs, line_tile0, l0, nr, lo + l0, 0, lo, cb, tile_cols);
    }
  } else {
    // lines = raw pairs (a,b) of the order-3 dilation; cols c in [lo, cmax4(a,b)]
    int bmax_all = lo;
    for (int l = 0; l < n3lines; l++) bmax_all = std::max(bmax_all, (int)cmax3[l]);
    a_count = n3lines;
    b_count = bmax_all - lo + 1;
    line_of_ab.assign((size_t)a_count * b_count, -1);
    line_start.push_back(0);
    for (int la = 0; la < n3lines; la++) {
      const int a = lo + la;
      const int first_line = (int)line_a.size();
      for (int b = lo; b <= cmax3[la]; b++) {
        int best = -1;
        for (int k1 = std::max(0, a - hi); k1 <= std::min(rows - 1, a - lo); k1++) {
          const int n2 = p3_len(m, k1);
          for (int k2 = std::max(0, b - hi); k2 <= std::min(n2 - 1, b - lo); k2++)
            best = std::max(best, p4_len(m, k1, k2) - 1);
        }
        if (best < 0) continue;  // cannot happen for b <= cmax3 (kept for safety)
        line_of_ab[(size_t)la * b_count + (b - lo)] = (int32_t)line_a.size();
        line_a.push_back(a);
        line_b.push_back(b);
        line_cmax.push_back(best + hi);
        line_start.push_back(line_start.back() + (best + hi - lo + 1));
      }
      const int nl = (int)line_a.size() - first_line;
      line_tile0.resize(line_a.size(), 0);
      for (int l0 = 0; l0 < nl; l0 += tile_rows) {
        const int nr = std::min(tile_rows, nl - l0);
        int cb = lo;
        for (int l = first_line + l0; l < first_line + l0 + nr; l++) cb = std::max(cb, (int)line_cmax[l]);
        add_band_regions(regs, line_tile0, first_line + l0, nr, line_b[first_line + l0], a, lo, cb, tile_cols);
      }
    }
    nlines = (int64_t)line_a.size();
    ncells = line_start.back();
  }

  // tiles, padded to whole regions with empty copies of the last real tile
  // (their staged loads stay in range; nrows 0 keeps them out of the results)
  ntiles = (int)regs.size();
  nregions = (ntiles + tiles_per_region - 1) / tiles_per_region;
  tiles.clear();
  f_lo = order == 3 ? 2 * lo : 3 * lo;
  f_hi = 0;
  for (int i = 0; i < nregions * tiles_per_region; i++) {
    const bool real = i < ntiles;
    const RegionRec& r = regs[real ? i : ntiles - 1];
    Tile t{};
    t.line0 = r.line0;
    t.nrows = real ? r.nrows : 0;
    t.row_freq0 = r.row_freq0;
    t.plane_freq = r.plane_freq;
    t.col0 = r.col0;
    tiles.push_back(t);
    // frequencies the tile's staged operands cover
    const int rmax = r.row_freq0 + tile_rows - 1, cmax = r.col0 + tile_cols - 1;
    f_hi = std::max({f_hi, r.plane_freq + rmax + cmax, rmax, cmax, r.plane_freq});
    f_lo = std::min({f_lo, r.plane_freq + r.row_freq0 + r.col0, r.row_freq0, r.col0, r.plane_freq});
  }
  issued_cells = (int64_t)nregions * kRegionCells;
  return "";
}

}  // namespace hos
