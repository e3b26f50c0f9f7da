// psg_grid.cuh — the cell grid over the first g projection keys, shared by
// the closest-pair and fixed-radius engines.
//
// Points are radix-sorted by cell id (stable, so a cell lists its points in
// original-index order) and keys are gathered into that order, so every cell
// is a contiguous window of sorted positions [cstart[c], cend[c]).  A pair
// whose key gaps are all <= w lies in the same or an adjacent cell; cell
// coordinates are clamped to [0, dims-1], which is monotone and contracting,
// so far-out points merge into border cells without breaking that property.
#pragma once

#include "psg_internal.cuh"

namespace psg {

struct GridDev {  // POD view passed to kernels
  const float* skeys = nullptr;   // n x nk keys, sorted by cell
  const uint32_t* sidx = nullptr; // sorted position -> original index
  const uint32_t* scell = nullptr;
  const uint32_t* cfirst = nullptr;  // cells+1: first sorted position with cell id >= c
  uint32_t n = 0;
  int g = 1;
  uint32_t dims[3] = {1, 1, 1};
  double lo[3] = {0, 0, 0};
  double inv_w = 1.0;
};

struct GridIndex {
  int nk = 4;
  double w = 0.0;
  uint64_t cells = 1;
  DevBuf<float> skeys;
  DevBuf<uint32_t> sidx, scell, cfirst;
  GridDev dev;
};

// The forward half of the 3^g stencil of sorted position p as at most five
// contiguous position ranges.  Cells of one "row" (all coordinates but the
// last fixed) are consecutive cell ids, hence consecutive positions:
//   own row  : [p+1, end of cell (.., c_last+1))   (own cell's later points + next cell)
//   g>=2     : row (c0, c1+1) and, for g=3, rows (c0+1, c1-1..c1+1); each row
//              spans cells c_last-1 .. c_last+1
// Each unordered pair within the stencil appears in exactly one range of
// exactly one of its two points.
__device__ __forceinline__ int grid_ranges(const GridDev& G, uint32_t p, uint32_t cell, uint32_t rb[5],
                                           uint32_t re[5]) {
  uint32_t cc[3] = {0, 0, 0};
  {
    uint32_t c = cell;
    for (int t = G.g - 1; t >= 0; --t) {
      cc[t] = c % G.dims[t];
      c /= G.dims[t];
    }
  }
  const int last = G.g - 1;
  const uint32_t D = G.dims[last];
  const uint32_t lo_last = cc[last] > 0 ? cc[last] - 1 : 0;
  const uint32_t hi_last = cc[last] + 1 < D ? cc[last] + 1 : D - 1;
  // own row
  int k = 0;
  rb[k] = p + 1;
  re[k] = G.cfirst[cell - cc[last] + hi_last + 1];
  ++k;
  if (G.g == 1) return k;
  // rows are identified by the prefix (c0[, c1]); row base id = prefix * D
  auto add_row = [&](int64_t a0, int64_t a1) {
    uint32_t prefix;
    if (G.g == 2) {
      if (a0 < 0 || a0 >= G.dims[0]) return;
      prefix = static_cast<uint32_t>(a0);
    } else {
      if (a0 < 0 || a0 >= G.dims[0] || a1 < 0 || a1 >= G.dims[1]) return;
      prefix = static_cast<uint32_t>(a0) * G.dims[1] + static_cast<uint32_t>(a1);
    }
    const uint32_t base = prefix * D;
    rb[k] = G.cfirst[base + lo_last];
    re[k] = G.cfirst[base + hi_last + 1];
    ++k;
  };
  if (G.g == 2) {
    add_row(static_cast<int64_t>(cc[0]) + 1, 0);
  } else {
    add_row(cc[0], static_cast<int64_t>(cc[1]) + 1);
    add_row(static_cast<int64_t>(cc[0]) + 1, static_cast<int64_t>(cc[1]) - 1);
    add_row(static_cast<int64_t>(cc[0]) + 1, cc[1]);
    add_row(static_cast<int64_t>(cc[0]) + 1, static_cast<int64_t>(cc[1]) + 1);
  }
  return k;
}

// The 0.1%..99.9% quantile box of the first g keys, from a deterministic
// strided sample (a tuning input only: clamping keeps any box exact).
void grid_sample_box(const float* keys, uint32_t n, int nk, int g, double lo[3], double span[3], cudaStream_t s);
// Cell width giving about `occupancy` points per cell over the box.
double grid_occupancy_width(uint32_t n, int g, const double span[3], double occupancy);
// (Re)build `gi` over `keys` (n x nk, original order) with cell width >= w
// (widened if the dense cell table would exceed 2^24 cells).
void build_grid(const float* keys, uint32_t n, int nk, int g, double w, const double lo[3], const double span[3],
                GridIndex& gi, cudaStream_t s);

// Decode a cell id, then the s-th cell of the 3^g stencil around it.
__device__ __forceinline__ void grid_coords(const GridDev& G, uint32_t c, uint32_t cc[3]) {
  for (int t = G.g - 1; t >= 0; --t) {
    cc[t] = c % G.dims[t];
    c /= G.dims[t];
  }
}
__device__ __forceinline__ bool grid_stencil(const GridDev& G, const uint32_t cc[3], int s, uint32_t* nc) {
  int off[3] = {0, 0, 0};
  for (int t = G.g - 1; t >= 0; --t) {
    off[t] = s % 3 - 1;
    s /= 3;
  }
  uint32_t c = 0;
  for (int t = 0; t < G.g; ++t) {
    const int64_t v = static_cast<int64_t>(cc[t]) + off[t];
    if (v < 0 || v >= static_cast<int64_t>(G.dims[t])) return false;
    c = c * G.dims[t] + static_cast<uint32_t>(v);
  }
  *nc = c;
  return true;
}
__host__ __device__ __forceinline__ int grid_stencil_size(int g) { return g == 1 ? 3 : (g == 2 ? 9 : 27); }

}  // namespace psg
