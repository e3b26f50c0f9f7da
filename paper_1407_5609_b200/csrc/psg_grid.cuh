// psg_grid.cuh — the cell grid over the first g projection keys, shared by
// the closest-pair and fixed-radius engines.
//
// Points are radix-sorted by cell id (stable, so a cell lists its points in
// original-index order) and keys are gathered into that order, so every cell
// is a contiguous window of sorted positions [cfirst[c], cfirst[c+1]).  A pair
// whose key gaps are all <= w lies in the same or an adjacent cell; cell
// coordinates are clamped to [0, dims-1], which is monotone and contracting,
// so far-out points merge into border cells without breaking that property.
//
// The grid parameters live in device memory (GridParams) so the whole build
// can be enqueued without a host round trip; kernels copy them to registers.
#pragma once

#include "psg_internal.cuh"

namespace psg {

constexpr uint64_t kMaxCells = 1ull << 24;
// the dense engine's radix-sorted grids over up to 8 keys (cfirst: 512 MiB)
constexpr uint64_t kMaxDenseCells = 1ull << 27;
constexpr uint32_t kGridSample = 4096;  // keys sampled (hashed positions) for the key box

// q = x / d for x < 2^31 by multiply-high (CUTLASS-style FastDivmod).
struct FastDiv {
  uint32_t d = 1, m = 0, s = 0;
  __host__ __device__ static FastDiv make(uint32_t divisor) {
    FastDiv f;
    f.d = divisor;
    if (divisor > 1) {
      int l = 0;
      while ((1u << l) < divisor) ++l;  // ceil(log2)
      const int p = 31 + l;
      // m = ceil(2^p / d) (< 2^32): from the FP64 quotient (53 bits) with an
      // exact 64-bit fix-up, not a 64-bit integer division (slow on device)
      const uint64_t two_p = 1ull << p;
      uint64_t m = static_cast<uint64_t>(static_cast<double>(two_p) / static_cast<double>(divisor));
      while (m * divisor < two_p) ++m;
      while (m > 0 && (m - 1) * divisor >= two_p) --m;
      f.m = static_cast<uint32_t>(m);
      f.s = static_cast<uint32_t>(p - 32);
    }
    return f;
  }
  __device__ __forceinline__ uint32_t div(uint32_t x) const { return d == 1 ? x : (__umulhi(x, m) >> s); }
};

constexpr int kMaxGridKeys = 8;  // sparse engine uses g <= 3; the dense engine up to 8

struct GridParams {
  int g = 1;
  uint32_t dims[kMaxGridKeys] = {1, 1, 1, 1, 1, 1, 1, 1};
  double lo[kMaxGridKeys] = {};
  double w = 1.0, inv_w = 1.0;
  uint64_t cells = 1;
  FastDiv fD, f1;  // division by the last dim and by dims[1] (g <= 3)
};

// Fill dims/cells/divisors for width >= w over the box (widened until the dense
// cell table fits max_cells).  Host and device.  lo/span have >= g entries.
__host__ __device__ inline void grid_params_for(GridParams& gp, int g, double w, const double* lo,
                                                const double* span, uint64_t max_cells = kMaxCells) {
  gp.g = g;
  for (;;) {
    double cells = 1.0;
    for (int t = 0; t < g; ++t) cells *= floor(span[t] / w) + 1.0;
    if (cells <= static_cast<double>(max_cells)) break;
    w *= 1.25;
  }
  gp.w = w;
  gp.inv_w = 1.0 / w;
  gp.cells = 1;
  for (int t = 0; t < kMaxGridKeys; ++t) {
    gp.lo[t] = t < g ? lo[t] : 0.0;
    gp.dims[t] = t < g ? static_cast<uint32_t>(floor(span[t] / w)) + 1 : 1;
    gp.cells *= gp.dims[t];
  }
  gp.fD = FastDiv::make(gp.dims[g - 1]);
  gp.f1 = FastDiv::make(gp.dims[1]);
}

#ifdef __CUDACC__
// Cell id of a key vector: cell coordinate floor((k_t - lo_t) / w) clamped to
// the grid, in FP64, row-major over the first g keys.  The ONE formula every
// builder uses (the projection's fused count, the counting and radix builds).
template <int NK>
__device__ __forceinline__ uint32_t cell_of(const float* k, const GridParams& P) {
  uint32_t c = 0;
#pragma unroll
  for (int t = 0; t < (NK < kMaxGridKeys ? NK : kMaxGridKeys); ++t) {
    if (t >= P.g) break;
    const uint32_t dim = P.dims[t];
    const double v = (static_cast<double>(k[t]) - P.lo[t]) * P.inv_w;
    const uint32_t ct = v <= 0.0 ? 0u : (v >= static_cast<double>(dim - 1) ? dim - 1 : static_cast<uint32_t>(v));
    c = c * dim + ct;
  }
  return c;
}
#endif

// The projection's fused counting pass (sparse grids, first build of a
// solve): the cell of every row and its arrival rank in the cell, exactly as
// k_cell_count would produce them (psg_grid.cu), so build_grid skips that
// kernel and its re-read of the keys.
struct CellCount {
  const GridParams* gp = nullptr;  // nullptr: no counting
  uint32_t* cnt = nullptr;
  uint32_t* cid = nullptr;
};

// The bootstrap folded into the counting build's per-position fix-up: every
// point's least key lower bound over the later points of its own cell and the
// next cell of its row (the sparse scan's own-row range), warp-reduced to one
// (lb, i, j) per warp of arrival positions; k_boot_select (psg_cpp.cu) then
// evaluates the best of them exactly.
struct BootLB {
  const float* keys = nullptr;  // original order, nk per row; nullptr: off
  float* wlb = nullptr;         // per warp: least lower bound (+inf: none)
  uint2* wpair = nullptr;       //           its (i, j), original indices
  uint64_t zone = 0;
};

#ifdef __CUDACC__
// The fused count of one row (CellCount): the k_cell_count step.
template <int NK>
__device__ __forceinline__ void count_cell(const float* k, uint32_t row, const CellCount& cc) {
  const uint32_t c = cell_of<NK>(k, *cc.gp);
  cc.cid[row] = c;
  atomicAdd(cc.cnt + c, 1u);  // result unused: a fire-and-forget reduction
}
#endif

struct GridDev {  // POD view passed to kernels
  const float* skeys = nullptr;   // n x nk keys, sorted by cell
  const uint32_t* sidx = nullptr; // sorted position -> original index
  const uint32_t* scell = nullptr;
  const uint32_t* cfirst = nullptr;  // cells+1: first sorted position with cell id >= c
  const GridParams* gp = nullptr;    // device
  uint32_t n = 0;
};

// Persistent buffers of one grid (reused across solves on the same point set).
struct GridIndex {
  int nk = 4;
  uint32_t n = 0;
  DevBuf<float> skeys;
  DevBuf<uint32_t> sidx, cid0, cid1, idx0, idx1, hist, cfirst;
  DevBuf<uint32_t> dcfirst;  // cfirst of a dense grid with more than kMaxCells cells
  // counting build: per-cell counters (kept all-zero between builds), the
  // scan's temp, the list of cells too big for the per-position fix-up, and
  // two device counters (big-cell count, cursor)
  DevBuf<uint32_t> cnt, ctmp, big, bctr;
  DevBuf<float> sample;
  DevBuf<GridParams> gp;
  DevBuf<float> wlb;   // BootLB outputs (one per warp of positions)
  DevBuf<uint2> wpair;
  GridDev dev;
  void ensure(uint32_t n_, int nk_, cudaStream_t s);
};

// Enqueue the build (no host synchronisation): cell ids from *G.gp, points
// ordered by (cell, original index), cfirst, keys gathered into that order.
// counting = true (sparse grids, a few points per cell): per-cell atomic
// counts, one scan (which IS cfirst), atomic placement, then a deterministic
// fix-up that ranks each point inside its cell by original index.
// counting = false (the dense engine's large cells): stable LSD radix sort on
// sort_bits, cfirst by search of the sorted ids.  Both give the same order.
// dense_cells (counting = false): the grid's cell count when the host knows
// it; above kMaxCells the table goes to gi.dcfirst and the sort covers its bits.
void build_grid(const float* keys, uint32_t n, int nk, GridIndex& gi, int sort_bits, cudaStream_t s,
                bool counting = true, uint64_t dense_cells = 0, bool counted = false, const BootLB* boot = nullptr);
// Strided sample of the first g keys into gi.sample (g x m floats); returns m.
uint32_t grid_sample(const float* keys, uint32_t n, int nk, int g, GridIndex& gi, cudaStream_t s);
// Host-side box from a host copy of the sample (mean +- 3 sd, clipped).
void grid_box_host(const float* sample, uint32_t m, int g, double lo[3], double span[3]);
// Cell width giving about `occupancy` points per cell over the box.
__host__ __device__ inline double grid_occupancy_width(uint32_t n, int g, const double span[3], double occupancy) {
  double vol = 1.0;
  for (int t = 0; t < g; ++t) vol *= span[t];
  const double x = vol * occupancy / (n > 0 ? static_cast<double>(n) : 1.0);
  return g == 1 ? x : g == 2 ? sqrt(x) : g == 3 ? cbrt(x) : pow(x, 1.0 / g);  // no pow for g <= 3
}

struct GridRanges {  // five ranges held in registers; empty ranges have b == e
  uint32_t b0, e0, b1, e1, b2, e2, b3, e3, b4, e4;
  __device__ __forceinline__ uint32_t b(int r) const {
    return r == 0 ? b0 : r == 1 ? b1 : r == 2 ? b2 : r == 3 ? b3 : b4;
  }
  __device__ __forceinline__ uint32_t e(int r) const {
    return r == 0 ? e0 : r == 1 ? e1 : r == 2 ? e2 : r == 3 ? e3 : e4;
  }
};

// The five ranges as one flattened candidate index space t in [0, total):
// lets a thread issue several candidates' loads before using any of them.
struct GridFlat {
  uint32_t b0, b1, b2, b3, b4;  // range starts
  uint32_t o1, o2, o3, o4;      // prefix offsets of ranges 1..4
  uint32_t total;
  __device__ __forceinline__ uint32_t at(uint32_t t) const {
    return t < o1 ? b0 + t : t < o2 ? b1 + (t - o1) : t < o3 ? b2 + (t - o2) : t < o4 ? b3 + (t - o3) : b4 + (t - o4);
  }
};

// Row (prefix) range of cells [lo_last, hi_last]; empty when the row is outside the grid.
__device__ __forceinline__ void grid_row(const uint32_t* __restrict__ cfirst, const GridParams& P, int a0, int a1,
                                         uint32_t D, uint32_t lo_last, uint32_t hi_last, uint32_t& b, uint32_t& e) {
  b = e = 0;
  uint32_t prefix;
  if (P.g == 2) {
    if (a0 < 0 || a0 >= static_cast<int>(P.dims[0])) return;
    prefix = static_cast<uint32_t>(a0);
  } else {
    if (a0 < 0 || a0 >= static_cast<int>(P.dims[0]) || a1 < 0 || a1 >= static_cast<int>(P.dims[1])) return;
    prefix = static_cast<uint32_t>(a0) * P.dims[1] + static_cast<uint32_t>(a1);
  }
  const uint32_t base = prefix * D;
  b = cfirst[base + lo_last];
  e = cfirst[base + hi_last + 1];
}

// The forward half of the 3^g stencil of sorted position p as at most five
// contiguous position ranges.  Cells of one "row" (all coordinates but the
// last fixed) are consecutive cell ids, hence consecutive positions:
//   own row  : [p+1, end of cell (.., c_last+1))   (own cell's later points + next cell)
//   g>=2     : row (c0, c1+1) and, for g=3, rows (c0+1, c1-1..c1+1); each row
//              spans cells c_last-1 .. c_last+1
// Each unordered pair within the stencil appears in exactly one range of
// exactly one of its two points.
__device__ __forceinline__ GridRanges grid_ranges(const uint32_t* __restrict__ cfirst, const GridParams& P,
                                                  uint32_t p, uint32_t cell) {
  GridRanges R{};
  const uint32_t D = P.g == 1 ? P.dims[0] : (P.g == 2 ? P.dims[1] : P.dims[2]);  // no dynamic indexing
  const uint32_t prefix = P.fD.div(cell);
  const uint32_t c_last = cell - prefix * D;
  const uint32_t lo_last = c_last > 0 ? c_last - 1 : 0;
  const uint32_t hi_last = c_last + 1 < D ? c_last + 1 : D - 1;
  R.b0 = p + 1;
  R.e0 = cfirst[cell - c_last + hi_last + 1];
  if (P.g == 2) {
    grid_row(cfirst, P, static_cast<int>(prefix) + 1, 0, D, lo_last, hi_last, R.b1, R.e1);
  } else if (P.g == 3) {
    const uint32_t q1 = P.f1.div(prefix);
    const int c0 = static_cast<int>(q1), c1 = static_cast<int>(prefix - q1 * P.dims[1]);
    grid_row(cfirst, P, c0, c1 + 1, D, lo_last, hi_last, R.b1, R.e1);
    grid_row(cfirst, P, c0 + 1, c1 - 1, D, lo_last, hi_last, R.b2, R.e2);
    grid_row(cfirst, P, c0 + 1, c1, D, lo_last, hi_last, R.b3, R.e3);
    grid_row(cfirst, P, c0 + 1, c1 + 1, D, lo_last, hi_last, R.b4, R.e4);
  }
  return R;
}

// grid_ranges restricted by the point's position inside its cell: a
// neighbour cell across a face the point is farther than `win` from holds no
// point within `win` in that key, so no pair passing the key test (every
// key gap <= sqrt(lb2) <= win).  Own row: the next cell only near the upper
// face of the last key; other rows only near the faces they lie across, and
// their last-key span only as wide as the point's nearness allows.
__device__ __forceinline__ GridRanges grid_ranges_pruned(const uint32_t* __restrict__ cfirst, const GridParams& P,
                                                         uint32_t p, uint32_t cell, const float* key, double win) {
  GridRanges R{};
  const uint32_t D = P.g == 1 ? P.dims[0] : (P.g == 2 ? P.dims[1] : P.dims[2]);
  const uint32_t prefix = P.fD.div(cell);
  const uint32_t c_last = cell - prefix * D;
  const int tl = P.g - 1;  // the last grid key (0, 1 or 2)
  const double lo_l = (tl == 0 ? P.lo[0] : tl == 1 ? P.lo[1] : P.lo[2]) + c_last * P.w;
  const double x_l = tl == 0 ? key[0] : tl == 1 ? key[1] : key[2];
  const bool lo_near = c_last > 0 && x_l - lo_l <= win;
  const bool hi_near = c_last + 1 < D && lo_l + P.w - x_l <= win;
  const uint32_t lo_last = lo_near ? c_last - 1 : c_last;
  const uint32_t hi_last = hi_near ? c_last + 1 : c_last;
  R.b0 = p + 1;
  R.e0 = cfirst[cell - c_last + hi_last + 1];
  if (P.g == 2) {
    const double lo0 = P.lo[0] + prefix * P.w;
    if (prefix + 1 < P.dims[0] && lo0 + P.w - key[0] <= win)
      grid_row(cfirst, P, static_cast<int>(prefix) + 1, 0, D, lo_last, hi_last, R.b1, R.e1);
  } else if (P.g == 3) {
    const uint32_t q1 = P.f1.div(prefix);
    const int c0 = static_cast<int>(q1), c1 = static_cast<int>(prefix - q1 * P.dims[1]);
    const double lo0 = P.lo[0] + c0 * P.w, lo1 = P.lo[1] + c1 * P.w;
    const bool hi0 = lo0 + P.w - key[0] <= win;
    const bool lo1n = key[1] - lo1 <= win, hi1 = lo1 + P.w - key[1] <= win;
    if (hi1) grid_row(cfirst, P, c0, c1 + 1, D, lo_last, hi_last, R.b1, R.e1);
    if (hi0) {
      if (lo1n) grid_row(cfirst, P, c0 + 1, c1 - 1, D, lo_last, hi_last, R.b2, R.e2);
      grid_row(cfirst, P, c0 + 1, c1, D, lo_last, hi_last, R.b3, R.e3);
      if (hi1) grid_row(cfirst, P, c0 + 1, c1 + 1, D, lo_last, hi_last, R.b4, R.e4);
    }
  }
  return R;
}

// Only the own row's forward range [p+1, end of cell (.., c_last+1)): one
// cfirst lookup (the bootstrap's cheap variant).
__device__ __forceinline__ GridRanges grid_own_row(const uint32_t* __restrict__ cfirst, const GridParams& P,
                                                   uint32_t p, uint32_t cell) {
  GridRanges R{};
  const uint32_t D = P.g == 1 ? P.dims[0] : (P.g == 2 ? P.dims[1] : P.dims[2]);
  const uint32_t prefix = P.fD.div(cell);
  const uint32_t c_last = cell - prefix * D;
  const uint32_t hi_last = c_last + 1 < D ? c_last + 1 : D - 1;
  R.b0 = p + 1;
  R.e0 = cfirst[cell - c_last + hi_last + 1];
  return R;
}

__device__ __forceinline__ GridFlat grid_flat(const GridRanges& R) {
  GridFlat F;
  F.b0 = R.b0;
  F.b1 = R.b1;
  F.b2 = R.b2;
  F.b3 = R.b3;
  F.b4 = R.b4;
  F.o1 = R.e0 > R.b0 ? R.e0 - R.b0 : 0;
  F.o2 = F.o1 + (R.e1 - R.b1);
  F.o3 = F.o2 + (R.e2 - R.b2);
  F.o4 = F.o3 + (R.e3 - R.b3);
  F.total = F.o4 + (R.e4 - R.b4);
  return F;
}

}  // namespace psg
