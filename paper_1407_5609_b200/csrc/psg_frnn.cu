// psg_frnn.cu — exact fixed-radius neighbours (refscan.cpp:159-209).
//
//   K1 project    keys = <U_k, X_i>                         (psg_cpp.cu / psg_project_tc.cu)
//   K2 grid       the closest-pair engine's cell grid (psg_grid.cuh) over the
//                 first g = min(3, q) keys with cell width >= the key window
//                 implied by R (+ rounding slack): every pair within R sits in
//                 the same or an adjacent cell; stable radix sort by cell, so a
//                 point's forward half-stencil is <= 5 contiguous position ranges
//   K4 scan       d <= 4 (k_frnn_cells): one warp per non-empty cell, lanes =
//                 32 stencil candidates at a time against the cell's points in
//                 shared memory; coordinates gathered into cell order (one
//                 float4 per point), the FP32 distance is the only filter.
//                 d > 4 (k_frnn_scan): one thread per sorted position, warps
//                 iterate in lockstep over their lanes' ranges; all nk keys
//                 prune (lower bound) before the distance.
//                 The FP32 distance decides outside the rounding band, the
//                 reference's FP64 arithmetic inside it (boundary inclusive,
//                 <= R; d <= 4: the rare band pairs go to k_frnn_band).  Pairs
//                 (min(i,j)<<32)|max(i,j) are appended through a per-warp
//                 shared-memory buffer (one global atomic per 32-128 pairs)
//                 and hashed in-kernel (order-independent sum)
//   lists         CSR without a global sort: per-row counts (atomics), scan,
//                 scatter, then each row sorted by one warp (bitonic in
//                 registers); the (i<j) pair list is the same with one direction
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <memory>

#include "psg_cpp.cuh"
#include "psg_engines.cuh"
#include "psg_grid.cuh"
#include "psg_scan.cuh"
#include "psg_sort.cuh"

namespace psg {

uint64_t brute_emit_pairs(psg_pointset* ps, double radius, uint64_t zone, DevBuf<uint64_t>& keys, uint64_t* hash,
                          cudaStream_t s);

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t x) {  // rng.cpp:46-51
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

unsigned blocks(uint64_t n, int per) { return static_cast<unsigned>((n + per - 1) / per); }

template <int NK>
__global__ void k_key_range(const float* __restrict__ keys, uint32_t n, int g, unsigned* __restrict__ mn,
                            unsigned* __restrict__ mx) {
  unsigned lo[3] = {0xffffffffu, 0xffffffffu, 0xffffffffu}, hi[3] = {0, 0, 0};
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    for (int t = 0; t < g; ++t) {
      const unsigned o = f32_order(keys[static_cast<size_t>(i) * NK + t]);
      lo[t] = min(lo[t], o);
      hi[t] = max(hi[t], o);
    }
  for (int t = 0; t < g; ++t) {
    const unsigned l = __reduce_min_sync(kFull, lo[t]), h = __reduce_max_sync(kFull, hi[t]);
    if ((threadIdx.x & 31) == 0) {
      atomicMin(mn + t, l);
      atomicMax(mx + t, h);
    }
  }
}

// d <= 4: the coordinates in cell order, one float4 per sorted position
__global__ void k_gather_rows4(Rows X, const uint32_t* __restrict__ sidx, uint32_t n, int d,
                               float4* __restrict__ sx) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint32_t i = sidx[p];
  float v[4] = {0.f, 0.f, 0.f, 0.f};
  for (int t = 0; t < d; ++t) v[t] = row_at(X, i, t);
  sx[p] = make_float4(v[0], v[1], v[2], v[3]);
}

struct FrnnArgs {
  Rows X;  // the working rows (materialised or virtual windows)
  const float* skeys;
  const float4* sx;  // d <= 4
  const uint32_t* sidx;
  GridDev grid;
  uint32_t n;
  int d;
  uint64_t zone;
  Thresholds th;
  float lo;  // s32 <= lo: inside R for certain
  double R;
  ExactSrc src;
  uint64_t* out;
  uint64_t cap;
  unsigned long long* acc;  // [0] count, [1] hash, [2] visited, [3] examined, [4] band pairs, [5] cell cursor,
                            // [6] / [7] the part's cell range (k_part_cells)
  uint64_t* band;           // k_frnn_cells: pairs inside the rounding band, decided by k_frnn_band
  uint64_t bcap;
  uint32_t plo, phi;        // the part's sorted positions [plo, phi) (pairs whose first position is there)
};

// The part's cells for k_frnn_cells: the cells whose first sorted position
// lies in [plo, phi) (cfirst is non-decreasing, so parts split the cells into
// consecutive ranges and every pair, visited from its earlier position's
// cell, has exactly one owner).  One thread; acc[6], acc[7].
__global__ void k_part_cells(FrnnArgs a) {
  const uint64_t cells = a.grid.gp->cells;
  auto first_at_or_after = [&](uint32_t pos) {  // least c with cfirst[c] >= pos
    uint64_t lo = 0, hi = cells;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (a.grid.cfirst[mid] < pos)
        lo = mid + 1;
      else
        hi = mid;
    }
    return lo;
  };
  a.acc[6] = a.plo == 0 ? 0 : first_at_or_after(a.plo);
  a.acc[7] = a.phi >= a.n ? cells : first_at_or_after(a.phi);
}

constexpr int kFrnnThreads = 256;

// d > 4: one thread per sorted position; the warp walks its lanes' ranges in
// lockstep (lane predicate t < total), so emission is warp-converged.
template <int NK>
__global__ void __launch_bounds__(kFrnnThreads) k_frnn_scan(FrnnArgs a) {
  __shared__ GridParams sP;
  __shared__ uint64_t wbuf[kFrnnThreads / 32][64];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) sP = *a.grid.gp;
  __syncthreads();
  const uint32_t p = a.plo + blockIdx.x * kFrnnThreads + tid;
  const bool valid = p < a.phi;
  uint64_t visited = 0, examined = 0, hsum = 0;
  GridRanges R{};
  float mk[NK];
  uint32_t mi = 0;
  if (valid) {
    R = grid_ranges(a.grid.cfirst, sP, p, a.grid.scell[p]);
    mi = a.sidx[p];
    load_keys<NK>(a.skeys + static_cast<size_t>(p) * NK, mk);
  }
  // walk the (at most five) ranges with a running position; the range
  // switch is the only place the five bounds are selected
  uint32_t j = R.b0, e = R.e0;
  int ri = 0;
  auto skip_empty = [&]() {
    while (j >= e && ri < 4) {
      ++ri;
      j = R.b(ri);
      e = R.e(ri);
    }
  };
  skip_empty();
  bool active = valid && j < e;

  const unsigned lt = (1u << lane) - 1u;
  const bool zoned = a.zone > 1;
  int c = 0;  // warp-uniform fill of wbuf[w]
  while (__any_sync(kFull, active)) {
    bool emit = false;
    uint64_t key = 0;
    if (active) {
      uint32_t mj = zoned ? a.sidx[j] : 0u;
      if (!zoned || admissible(mi, mj, a.zone)) {  // refscan.cpp:15-18
        ++visited;
        if (!zoned) mj = a.sidx[j];
        float kj[NK];
        load_keys<NK>(a.skeys + static_cast<size_t>(j) * NK, kj);
        const bool pass = lb2_full<NK>(mk, kj) <= a.th.lb2;
        const float s32 = pass ? thread_sqdist(a.X, mi, mj) : INFINITY;
        if (pass) {
          ++examined;
          if (s32 <= a.th.band) {
            if (s32 <= a.lo || exact_distance(a.src, mi, mj) <= a.R) {  // boundary inclusive
              emit = true;
              key = mi < mj ? (static_cast<uint64_t>(mi) << 32) | mj : (static_cast<uint64_t>(mj) << 32) | mi;
              hsum += mix64(key);
            }
          }
        }
      }
      ++j;
      if (j >= e) skip_empty();
      active = j < e;
    }
    const unsigned mask = __ballot_sync(kFull, emit);
    if (mask) {
      if (emit) wbuf[w][c + __popc(mask & lt)] = key;
      c += __popc(mask);
      if (c >= 32) {  // flush 32 with one atomic
        __syncwarp();
        unsigned long long g = 0;
        if (lane == 0) g = atomicAdd(a.acc, 32ull);
        g = __shfl_sync(kFull, g, 0);
        if (g + lane < a.cap) a.out[g + lane] = wbuf[w][lane];
        __syncwarp();
        if (lane < c - 32) wbuf[w][lane] = wbuf[w][32 + lane];
        c -= 32;
        __syncwarp();
      }
    }
  }
  if (c > 0) {
    __syncwarp();
    unsigned long long g = 0;
    if (lane == 0) g = atomicAdd(a.acc, static_cast<unsigned long long>(c));
    g = __shfl_sync(kFull, g, 0);
    if (lane < c && g + lane < a.cap) a.out[g + lane] = wbuf[w][lane];
  }
  for (int o = 16; o; o >>= 1) {
    hsum += __shfl_xor_sync(kFull, hsum, o);
    visited += __shfl_xor_sync(kFull, visited, o);
    examined += __shfl_xor_sync(kFull, examined, o);
  }
  if (lane == 0) {
    if (hsum) atomicAdd(a.acc + 1, static_cast<unsigned long long>(hsum));
    if (visited) atomicAdd(a.acc + 2, static_cast<unsigned long long>(visited));
    if (examined) atomicAdd(a.acc + 3, static_cast<unsigned long long>(examined));
  }
}

// d <= 4, cell-cooperative: one warp per non-empty cell.  Every point of a
// cell has the same stencil (the own row starts at the cell's first point;
// a pair needs sorted position j > i, which every later row satisfies), so
// the warp loads 32 stencil candidates at a time — lane = candidate, one
// coalesced float4 each — and runs them against the cell's points, which sit
// in shared memory and are read as broadcasts.  Compared with a thread per
// point this removes the per-candidate range decode and the lanes idling on
// their neighbours' longer stencils; the pair set, the FP32/FP64 decisions and
// the counters are the same.  A warp takes 32 consecutive cells at once and
// its lanes resolve those cells' ranges in parallel (one cfirst latency).
// kD4: the fourth coordinate is used (d = 4); for d <= 3 it is zero in both
// points and fmaf(0, 0, s) == s, so it is skipped without changing s32.
// Warps claim 32-cell chunks from a counter (acc[5]): cells differ widely in
// work (empty border cells vs full interior cells).
template <bool kEmit, bool kD4, bool kZoned>
__global__ void __launch_bounds__(kFrnnThreads, 4) k_frnn_cells(FrnnArgs a) {
  __shared__ GridParams sP;
  // accepted pairs are compacted into a per-warp buffer and hashed (and, in
  // list mode, written with one global atomic) kFlush at a time, lane-parallel:
  // hashing inside the divergent accept branch cost more than the distances
  constexpr int kW = kFrnnThreads / 32, kFlush = kEmit ? 512 : 64;  // list mode: one output-slot atomic per 512 pairs (a same-address atomic with return per 128 cost ~0.25 ms at C4)
  __shared__ float4 cp[kW][32];
  __shared__ uint32_t ci[kW][32];
  __shared__ uint64_t wbuf[kW][kFlush + 32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) sP = *a.grid.gp;
  __syncthreads();
  const uint64_t cell_lo = a.acc[6], cells = a.acc[7];  // this part's cells [cell_lo, cells)
  const uint32_t* __restrict__ cfirst = a.grid.cfirst;
  const unsigned lt = (1u << lane) - 1u;
  const float band = a.th.band, lo = a.lo;
  uint64_t visited = 0, hsum = 0, emitted = 0;  // emitted: warp-uniform (list mode: acc[0] counts)
  int c = 0;  // warp-uniform fill of wbuf[w]
  // hash (and write) the first `cnt` buffered pairs; warp-converged
  auto flush = [&](int cnt) {
    __syncwarp();
    unsigned long long gpos = 0;
    if (kEmit && lane == 0) gpos = atomicAdd(a.acc, static_cast<unsigned long long>(cnt));
    if constexpr (kEmit) gpos = __shfl_sync(kFull, gpos, 0);
    for (int t = lane; t < cnt; t += 32) {
      const uint64_t k = wbuf[w][t];
      hsum += mix64(k);
      if (kEmit && gpos + t < a.cap) a.out[gpos + t] = k;
    }
    emitted += cnt;
    __syncwarp();
  };
  for (;;) {
    unsigned long long claim = 0;
    if (lane == 0) claim = atomicAdd(a.acc + 5, 1ull);
    const uint64_t c0 = cell_lo + __shfl_sync(kFull, claim, 0) * 32ull;
    if (c0 >= cells) break;
    const uint64_t mycell = c0 + lane;
    uint32_t s = 0, e = 0;
    if (mycell < cells) {
      s = cfirst[mycell];
      e = cfirst[mycell + 1];
    }
    GridRanges mine{};
    if (e > s) mine = grid_ranges(cfirst, sP, s, static_cast<uint32_t>(mycell));
    unsigned todo = __ballot_sync(kFull, e > s);
    while (todo) {
      const int k = __ffs(todo) - 1;
      todo &= todo - 1;
      const uint32_t cs = __shfl_sync(kFull, s, k), ce = __shfl_sync(kFull, e, k);
      GridRanges R;
      R.e0 = __shfl_sync(kFull, mine.e0, k);
      R.b1 = __shfl_sync(kFull, mine.b1, k);
      R.e1 = __shfl_sync(kFull, mine.e1, k);
      R.b2 = __shfl_sync(kFull, mine.b2, k);
      R.e2 = __shfl_sync(kFull, mine.e2, k);
      R.b3 = __shfl_sync(kFull, mine.b3, k);
      R.e3 = __shfl_sync(kFull, mine.e3, k);
      R.b4 = __shfl_sync(kFull, mine.b4, k);
      R.e4 = __shfl_sync(kFull, mine.e4, k);
      for (uint32_t g0 = cs; g0 < ce; g0 += 32) {  // the cell's points, 32 at a time
        const int m = static_cast<int>(min(32u, ce - g0));
        R.b0 = g0 + 1;  // no candidate at or before the group's first point pairs with it
        const GridFlat F = grid_flat(R);
        // the group's points and the first candidate chunk are loaded together;
        // each chunk's loads are issued before the previous chunk's math
        float4 gx = make_float4(0.f, 0.f, 0.f, 0.f);
        uint32_t gi = 0;
        if (lane < m) {
          gx = a.sx[g0 + lane];
          gi = a.sidx[g0 + lane];
        }
        bool in = static_cast<uint32_t>(lane) < F.total;
        uint32_t j = in ? F.at(lane) : g0;
        float4 o = a.sx[j];
        uint32_t mj = a.sidx[j];
        __syncwarp();
        if (lane < m) {
          cp[w][lane] = gx;
          ci[w][lane] = gi;
        }
        __syncwarp();
        uint32_t vis = 0;
        for (uint32_t t0 = 0; t0 < F.total; t0 += 32) {
          const bool in2 = t0 + 32 + lane < F.total;
          const uint32_t j2 = in2 ? F.at(t0 + 32 + lane) : g0;
          float4 o2 = o;
          uint32_t mj2 = mj;
          if (t0 + 32 < F.total) {
            o2 = a.sx[j2];
            mj2 = a.sidx[j2];
          }
          for (int q = 0; q < m; ++q) {
            const float4 x = cp[w][q];
            const uint32_t pi = g0 + q;
            bool ok = in && j > pi;
            if constexpr (kZoned) ok = ok && admissible(ci[w][q], mj, a.zone);  // refscan.cpp:15-18
            float g = o.x - x.x;
            float s32 = g * g;
            g = o.y - x.y;
            s32 = fmaf(g, g, s32);
            g = o.z - x.z;
            s32 = fmaf(g, g, s32);
            if constexpr (kD4) {
              g = o.w - x.w;
              s32 = fmaf(g, g, s32);
            }
            vis += ok;
            const bool emit = ok && s32 <= lo;  // inside R for certain
            if (ok && s32 <= band && !emit) {  // the reference's FP64 decision, deferred to k_frnn_band (rare)
              const uint32_t mi = ci[w][q];
              const uint64_t key =
                  mi < mj ? (static_cast<uint64_t>(mi) << 32) | mj : (static_cast<uint64_t>(mj) << 32) | mi;
              const unsigned long long slot = atomicAdd(a.acc + 4, 1ull);
              if (slot < a.bcap) a.band[slot] = key;
            }
            const unsigned mask = __ballot_sync(kFull, emit);
            if (mask) {
              if (emit) {
                const uint32_t mi = ci[w][q];
                wbuf[w][c + __popc(mask & lt)] =
                    mi < mj ? (static_cast<uint64_t>(mi) << 32) | mj : (static_cast<uint64_t>(mj) << 32) | mi;
              }
              c += __popc(mask);
              if (c >= kFlush) {
                flush(kFlush);
                if (lane < c - kFlush) wbuf[w][lane] = wbuf[w][kFlush + lane];
                c -= kFlush;
                __syncwarp();
              }
            }
          }
          in = in2;
          j = j2;
          o = o2;
          mj = mj2;
        }
        visited += vis;
        __syncwarp();  // cp/ci are rewritten by the next group
      }
    }
  }
  if (c > 0) flush(c);
  for (int o = 16; o; o >>= 1) {
    hsum += __shfl_xor_sync(kFull, hsum, o);
    visited += __shfl_xor_sync(kFull, visited, o);
  }
  if (lane == 0) {
    if (!kEmit && emitted) atomicAdd(a.acc, static_cast<unsigned long long>(emitted));
    if (hsum) atomicAdd(a.acc + 1, static_cast<unsigned long long>(hsum));
    if (visited) {
      atomicAdd(a.acc + 2, static_cast<unsigned long long>(visited));
      atomicAdd(a.acc + 3, static_cast<unsigned long long>(visited));
    }
  }
}

// The rounding-band pairs of k_frnn_cells: the reference's FP64
// distance (metrics.cpp:16-24, symmetric in i, j), boundary inclusive (<= R)
__global__ void k_frnn_band(FrnnArgs a) {
  const unsigned long long m = min(static_cast<unsigned long long>(a.acc[4]), static_cast<unsigned long long>(a.bcap));
  for (unsigned long long t = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x; t < m;
       t += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
    const uint64_t k = a.band[t];
    if (exact_distance(a.src, k >> 32, k & 0xffffffffull) <= a.R) {
      const unsigned long long g = atomicAdd(a.acc, 1ull);
      if (g < a.cap) a.out[g] = k;  // cap = 0 when only the count is wanted
      atomicAdd(a.acc + 1, static_cast<unsigned long long>(mix64(k)));
    }
  }
}

// ---- CSR lists without a global sort ------------------------------------------
__global__ void k_row_counts(const uint64_t* __restrict__ pairs, uint64_t m, bool both, uint32_t* __restrict__ cnt) {
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < m;
       k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t v = pairs[k];
    atomicAdd(cnt + (v >> 32), 1u);
    if (both) atomicAdd(cnt + (v & 0xffffffffull), 1u);
  }
}

__global__ void k_row_scatter(const uint64_t* __restrict__ pairs, uint64_t m, bool both, uint32_t* __restrict__ cur,
                              uint32_t* __restrict__ cols) {
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < m;
       k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t v = pairs[k];
    const uint32_t i = static_cast<uint32_t>(v >> 32), j = static_cast<uint32_t>(v);
    cols[atomicAdd(cur + i, 1u)] = j;
    if (both) cols[atomicAdd(cur + j, 1u)] = i;
  }
}

// Warp bitonic sort of 32R values held as v[r] = element r*32 + lane.
template <int R>
__device__ __forceinline__ void warp_bitonic(uint32_t (&v)[R], int lane) {
#pragma unroll
  for (int k = 2; k <= 32 * R; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
        const int jr = j >> 5;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int pr = r ^ jr;
          if (pr > r) {
            const bool up = (((r << 5) | lane) & k) == 0;
            const uint32_t x = v[r], y = v[pr];
            if ((x > y) == up) {
              v[r] = y;
              v[pr] = x;
            }
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const uint32_t o = __shfl_xor_sync(kFull, v[r], j);
          const bool up = (((r << 5) | lane) & k) == 0;
          const bool lower = (lane & j) == 0;
          v[r] = (lower == up) ? min(v[r], o) : max(v[r], o);
        }
      }
    }
  }
}

template <int R>
__device__ __forceinline__ void sort_row(uint32_t* __restrict__ row, uint32_t len, int lane) {
  uint32_t v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const uint32_t e = r * 32 + lane;
    v[r] = e < len ? row[e] : 0xffffffffu;
  }
  warp_bitonic<R>(v, lane);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const uint32_t e = r * 32 + lane;
    if (e < len) row[e] = v[r];
  }
}

// One warp per row; rows longer than 1024 are flagged for the global fallback.
__global__ void k_sort_rows(const uint32_t* __restrict__ off, uint64_t n, uint32_t* __restrict__ cols,
                            unsigned* __restrict__ too_long) {
  const int lane = threadIdx.x & 31;
  const uint64_t nw = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t r = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5; r < n; r += nw) {
    const uint32_t b = off[r], len = off[r + 1] - b;
    uint32_t* row = cols + b;
    if (len <= 1) continue;
    if (len <= 32) sort_row<1>(row, len, lane);
    else if (len <= 64) sort_row<2>(row, len, lane);
    else if (len <= 128) sort_row<4>(row, len, lane);
    else if (len <= 256) sort_row<8>(row, len, lane);
    else if (len <= 512) sort_row<16>(row, len, lane);
    else if (len <= 1024) sort_row<32>(row, len, lane);
    else if (lane == 0) atomicOr(too_long, 1u);
  }
}

__global__ void k_widen_offsets(const uint32_t* __restrict__ in, uint64_t count, uint64_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = in[i];
}

// pairs[k] = (i<<32)|j for every row i and column j of the (i<j) CSR, in order
__global__ void k_csr_to_pairs(const uint32_t* __restrict__ off, uint64_t n, const uint32_t* __restrict__ cols,
                               uint64_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const uint64_t nw = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t r = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5; r < n; r += nw)
    for (uint32_t e = off[r] + lane; e < off[r + 1]; e += 32) out[e] = (r << 32) | cols[e];
}

__global__ void k_cols_to_u64(const uint32_t* __restrict__ in, uint64_t count, uint64_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = in[i];
}

// ---- fallback: global sort of the directed pairs (rows longer than 1024) ----
__global__ void k_directed(const uint64_t* __restrict__ pairs, uint64_t m, int b, uint64_t* __restrict__ out) {
  const uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (k >= m) return;
  const uint64_t i = pairs[k] >> 32, j = pairs[k] & 0xffffffffull;
  out[2 * k] = (i << b) | j;
  out[2 * k + 1] = (j << b) | i;
}

__global__ void k_pack(const uint64_t* __restrict__ pairs, uint64_t m, int b, uint64_t* __restrict__ out) {
  const uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (k >= m) return;
  out[k] = ((pairs[k] >> 32) << b) | (pairs[k] & 0xffffffffull);
}

__global__ void k_unpack(uint64_t* __restrict__ keys, uint64_t m, int b) {
  const uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (k >= m) return;
  const uint64_t v = keys[k];
  keys[k] = ((v >> b) << 32) | (v & ((1ull << b) - 1));
}

__global__ void k_offsets(const uint64_t* __restrict__ sorted, uint64_t m, uint64_t n, int b,
                          uint64_t* __restrict__ offsets) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i > n) return;
  const uint64_t target = i << b;
  uint64_t lo = 0, hi = m;
  while (lo < hi) {
    const uint64_t mid = lo + ((hi - lo) >> 1);
    if (sorted[mid] < target)
      lo = mid + 1;
    else
      hi = mid;
  }
  offsets[i] = i == n ? m : lo;
}

__global__ void k_low_bits(uint64_t* __restrict__ keys, uint64_t m, int b) {
  const uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (k < m) keys[k] &= (1ull << b) - 1;
}

// ---- the sorted list in i-range buckets (frnn_pairs, large outputs) ----------
// Bucket b holds the pairs with i in [n b / B, n (b + 1) / B): bucket order is
// i order, so sorting each bucket on its own gives the global order, and
// bucket b's copy to the host overlaps the sort of bucket b + 1.
constexpr int kListBuckets = 32;

__device__ __forceinline__ uint32_t bucket_of(uint64_t key, uint64_t n, int B) {
  return static_cast<uint32_t>(((key >> 32) * B) / n);
}

__global__ void k_bucket_count(const uint64_t* __restrict__ pairs, uint64_t m, uint64_t n, int B,
                               unsigned long long* __restrict__ cnt) {
  __shared__ unsigned sc[kListBuckets];
  for (int b = threadIdx.x; b < B; b += blockDim.x) sc[b] = 0;
  __syncthreads();
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < m;
       k += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    atomicAdd(&sc[bucket_of(pairs[k], n, B)], 1u);
  __syncthreads();
  for (int b = threadIdx.x; b < B; b += blockDim.x)
    if (sc[b]) atomicAdd(cnt + b, static_cast<unsigned long long>(sc[b]));
}

// Scatter into the buckets, packed for the per-bucket radix sort: the key
// becomes ((i - i0) << bj) | j.  A block reserves its slots with one global
// atomic per bucket.
__global__ void k_bucket_scatter(const uint64_t* __restrict__ pairs, uint64_t m, uint64_t n, int B, int bj,
                                 unsigned long long* __restrict__ cursor, uint64_t* __restrict__ out) {
  __shared__ unsigned sc[kListBuckets];
  __shared__ unsigned long long base[kListBuckets];
  const uint64_t per = (m + gridDim.x - 1) / gridDim.x;  // a contiguous slice per block
  const uint64_t k0 = blockIdx.x * per, k1 = min(m, k0 + per);
  for (int b = threadIdx.x; b < B; b += blockDim.x) sc[b] = 0;
  __syncthreads();
  for (uint64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) atomicAdd(&sc[bucket_of(pairs[k], n, B)], 1u);
  __syncthreads();
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    base[b] = sc[b] ? atomicAdd(cursor + b, static_cast<unsigned long long>(sc[b])) : 0ull;
    sc[b] = 0;
  }
  __syncthreads();
  for (uint64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
    const uint64_t v = pairs[k];
    const uint32_t b = bucket_of(v, n, B);
    const uint64_t i0 = (n * b + B - 1) / B;  // first i of bucket b
    const unsigned slot = atomicAdd(&sc[b], 1u);
    out[base[b] + slot] = (((v >> 32) - i0) << bj) | (v & 0xffffffffull);
  }
}

// Back from the bucket's packed keys to (i << 32) | j.
__global__ void k_bucket_unpack(uint64_t* __restrict__ keys, uint64_t m, int bj, uint64_t i0) {
  const uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (k >= m) return;
  const uint64_t v = keys[k];
  keys[k] = (((v >> bj) + i0) << 32) | (v & ((1ull << bj) - 1));
}

// A bucket's sorted packed keys as upper-triangular CSR: cols[k] = j, and
// offs[i] = the bucket's first slot plus the first k whose row is >= i, for
// every row i of the bucket's range [i0, i1) (each row written once, by the
// pair that starts it or by the bucket's last pair for trailing empty rows).
__global__ void k_bucket_csr(const uint64_t* __restrict__ keys, uint64_t len, int bj, uint64_t i0, uint64_t i1,
                             uint64_t slot0, uint32_t* __restrict__ cols, uint64_t* __restrict__ offs) {
  const uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (k >= len) return;
  const uint64_t v = keys[k];
  const uint64_t r = v >> bj;
  cols[k] = static_cast<uint32_t>(v & ((1ull << bj) - 1));
  const uint64_t first = k == 0 ? 0 : (keys[k - 1] >> bj) + 1;  // rows (prev, r] start here
  for (uint64_t rr = first; rr <= r; ++rr) offs[i0 + rr] = slot0 + k;
  if (k == len - 1)
    for (uint64_t rr = r + 1; rr < i1 - i0; ++rr) offs[i0 + rr] = slot0 + len;
}

__global__ void k_fill_u64(uint64_t* __restrict__ out, uint64_t count, uint64_t v) {
  const uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (k < count) out[k] = v;
}

// ---- the (i<j) lists as CSR by row groups (frnn_pairs_csr) -------------------
// Group g = rows [256 g, 256 g + 256).  One histogram pass and one scatter
// (both block-aggregated in shared memory: one global atomic per block and
// group) put every pair in its group's slice; then one CTA per group orders
// the slice in shared memory — rows counted, scanned and placed, each row's
// columns sorted by a warp — and writes its columns and row offsets
// coalesced.  No global sort: about three passes over the 8-byte pairs.
constexpr int kGroupShift = 8;
constexpr uint32_t kGroupRows = 1u << kGroupShift;
constexpr int kGroupHistThreads = 1024;
constexpr uint32_t kMaxGroups = 16384;  // shared-memory histogram (n <= 2^22 rows)
constexpr uint32_t kGroupCap = 16384;   // pairs a group CTA sorts in shared memory (64 KiB)

__global__ void __launch_bounds__(kGroupHistThreads) k_group_hist(const uint64_t* __restrict__ pairs, uint64_t m,
                                                                  uint32_t ng, unsigned* __restrict__ cnt) {
  extern __shared__ unsigned sh[];
  for (uint32_t g = threadIdx.x; g < ng; g += blockDim.x) sh[g] = 0;
  __syncthreads();
  const uint64_t per = (m + gridDim.x - 1) / gridDim.x;
  const uint64_t k0 = blockIdx.x * per, k1 = min(m, k0 + per);
  for (uint64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) atomicAdd(&sh[pairs[k] >> (32 + kGroupShift)], 1u);
  __syncthreads();
  for (uint32_t g = threadIdx.x; g < ng; g += blockDim.x)
    if (sh[g]) atomicAdd(cnt + g, sh[g]);
}

// Scatter by digit v >> (32 + shift) (nbins of them; cur[b] starts at bin
// b's first slot), block-aggregated: a block histograms its tile in shared
// memory, reserves each bin's run with one global atomic and writes the run.
// tile = 0: one contiguous slice per block (few bins: long runs); a pass
// over input already grouped by a coarser digit uses small tiles, so each
// tile touches few bins and its runs stay long.
__global__ void __launch_bounds__(kGroupHistThreads) k_group_scatter(const uint64_t* __restrict__ pairs, uint64_t m,
                                                                     int shift, uint32_t nbins, uint64_t tile,
                                                                     unsigned* __restrict__ cur,
                                                                     uint64_t* __restrict__ out) {
  extern __shared__ unsigned sh[];  // nbins counters, then nbins bases
  unsigned* base = sh + nbins;
  const uint64_t per = tile ? tile : (m + gridDim.x - 1) / gridDim.x;
  for (uint64_t k0 = blockIdx.x * per; k0 < m; k0 += gridDim.x * per) {
    const uint64_t k1 = min(m, k0 + per);
    __syncthreads();
    for (uint32_t g = threadIdx.x; g < nbins; g += blockDim.x) sh[g] = 0;
    __syncthreads();
    for (uint64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) atomicAdd(&sh[pairs[k] >> (32 + shift)], 1u);
    __syncthreads();
    for (uint32_t g = threadIdx.x; g < nbins; g += blockDim.x) {
      base[g] = sh[g] ? atomicAdd(cur + g, sh[g]) : 0u;
      sh[g] = 0;
    }
    __syncthreads();
    for (uint64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
      const uint64_t v = pairs[k];
      const uint32_t g = static_cast<uint32_t>(v >> (32 + shift));
      out[base[g] + atomicAdd(&sh[g], 1u)] = v;
    }
  }
}

// A row longer than 1024 (rare: a dense cluster), straight to its final
// place: each column's rank among the row's (distinct) columns.
__device__ void block_rank_row(const uint32_t* __restrict__ row, uint32_t len, uint32_t* __restrict__ out) {
  for (uint32_t k = threadIdx.x; k < len; k += blockDim.x) {
    const uint32_t v = row[k];
    uint32_t r = 0;
    for (uint32_t t = 0; t < len; ++t) r += row[t] < v;
    out[r] = v;
  }
}

// One CTA per group g0 + blockIdx.x (at most kGroupCap pairs): columns in
// row order, each row ascending, to cols[gstart[g] ..]; row offsets to offs.
constexpr int kGroupSortThreads = 512;
__global__ void __launch_bounds__(kGroupSortThreads) k_group_sort(const uint64_t* __restrict__ grouped,
                                                                  const uint32_t* __restrict__ gstart, uint32_t g0,
                                                                  uint64_t n, uint32_t* __restrict__ cols,
                                                                  uint64_t* __restrict__ offs) {
  __shared__ uint32_t rs[kGroupRows + 1];  // row counts, then row starts
  __shared__ uint32_t cur[kGroupRows];
  extern __shared__ uint32_t sc[];         // the group's columns, by row (kGroupCap)
  const uint32_t g = g0 + blockIdx.x;
  const uint32_t b = gstart[g], len = gstart[g + 1] - b;
  const uint64_t r0 = static_cast<uint64_t>(g) << kGroupShift;
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (uint32_t r = tid; r <= kGroupRows; r += blockDim.x) rs[r] = 0;
  __syncthreads();
  for (uint32_t k = tid; k < len; k += blockDim.x)
    atomicAdd(&rs[static_cast<uint32_t>(grouped[b + k] >> 32) & (kGroupRows - 1)], 1u);
  __syncthreads();
  if (warp == 0) {  // exclusive scan of 256 counts: 8 per lane
    uint32_t v[kGroupRows / 32], sum = 0;
#pragma unroll
    for (int t = 0; t < static_cast<int>(kGroupRows / 32); ++t) {
      v[t] = rs[lane * (kGroupRows / 32) + t];
      sum += v[t];
    }
    uint32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t x = __shfl_up_sync(kFull, inc, o);
      if (lane >= static_cast<uint32_t>(o)) inc += x;
    }
    uint32_t run = inc - sum;
#pragma unroll
    for (int t = 0; t < static_cast<int>(kGroupRows / 32); ++t) {
      rs[lane * (kGroupRows / 32) + t] = run;
      cur[lane * (kGroupRows / 32) + t] = run;
      run += v[t];
    }
    if (lane == 31) rs[kGroupRows] = run;
  }
  __syncthreads();
  for (uint32_t k = tid; k < len; k += blockDim.x) {
    const uint64_t v = grouped[b + k];
    sc[atomicAdd(&cur[static_cast<uint32_t>(v >> 32) & (kGroupRows - 1)], 1u)] = static_cast<uint32_t>(v);
  }
  __syncthreads();
  const uint32_t nw = blockDim.x >> 5;
  for (uint32_t r = warp; r < kGroupRows; r += nw) {
    const uint32_t a = rs[r], l = rs[r + 1] - a;
    if (l <= 1) continue;
    uint32_t* row = sc + a;
    if (l <= 32) sort_row<1>(row, l, lane);
    else if (l <= 64) sort_row<2>(row, l, lane);
    else if (l <= 128) sort_row<4>(row, l, lane);
    else if (l <= 256) sort_row<8>(row, l, lane);
    else if (l <= 512) sort_row<16>(row, l, lane);
    else if (l <= 1024) sort_row<32>(row, l, lane);
  }
  // rows over 1024 (rare; at most kGroupCap / 1025 of them) go straight to cols
  uint32_t big_lo[kGroupCap / 1025], big_hi[kGroupCap / 1025], nbig = 0;
  for (uint32_t r = 0; r < kGroupRows; ++r)
    if (rs[r + 1] - rs[r] > 1024) {
      block_rank_row(sc + rs[r], rs[r + 1] - rs[r], cols + b + rs[r]);
      big_lo[nbig] = rs[r];
      big_hi[nbig++] = rs[r + 1];
    }
  __syncthreads();
  for (uint32_t k = tid; k < len; k += blockDim.x) {
    bool in_big = false;
    for (uint32_t t = 0; t < nbig; ++t) in_big |= k >= big_lo[t] && k < big_hi[t];
    if (!in_big) cols[b + k] = sc[k];
  }
  for (uint32_t r = tid; r < kGroupRows; r += blockDim.x)
    if (r0 + r < n) offs[r0 + r] = static_cast<uint64_t>(b) + rs[r];
}

int bits_for(uint64_t n) {
  int b = 1;
  while ((1ull << b) < n) ++b;
  return b;
}

unsigned grid_cap(uint64_t work) { return static_cast<unsigned>(std::min<uint64_t>(blocks(work, 256), 148ull * 16)); }

// Sorts `count` u64 keys of `width` bits in buf (scratch allocated here); the
// sorted keys end in buf.
void sort_u64(DevBuf<uint64_t>& buf, uint64_t count, int width, cudaStream_t s) {
  if (count <= 1) return;
  DevBuf<uint64_t> tmp(count, s);
  DevBuf<uint32_t> hist(radix_hist_words(count), s);
  uint64_t* kk[2] = {buf.p, tmp.p};
  uint32_t* vv[2] = {nullptr, nullptr};
  const int passes = (width + 7) / 8;
  const int which = radix_sort<uint64_t>(kk, vv, count, 0, passes * 8, hist.p, s);
  g_launches += 1 + passes;
  if (which == 1) std::swap(buf, tmp);
}

// Rows of the (i<j) pairs (both = false) or of both directions: offsets (n+1,
// u32) and ascending columns.  Returns false when a row exceeds 1024 entries
// (the caller falls back to the global sort).
bool csr_rows(const DevBuf<uint64_t>& pairs, uint64_t m, uint64_t n, bool both, DevBuf<uint32_t>& off,
              DevBuf<uint32_t>& cols, cudaStream_t s) {
  const uint64_t entries = both ? 2 * m : m;
  if (entries >= 0xffffffffull) throw std::runtime_error("pairscan_b200: neighbour list exceeds 2^32 entries");
  DevBuf<uint32_t> cnt(n + 1, s), tmp(scan_temp_words(n + 1), s), flag(1, s);
  off.alloc(n + 1, s);
  cols.alloc(std::max<uint64_t>(entries, 1), s);
  PSG_CUDA(cudaMemsetAsync(cnt.p, 0, (n + 1) * 4, s));
  PSG_CUDA(cudaMemsetAsync(flag.p, 0, 4, s));
  if (m) {
    k_row_counts<<<grid_cap(m), 256, 0, s>>>(pairs.p, m, both, cnt.p);
    PSG_LAUNCHED();
  }
  exclusive_scan_u32(cnt.p, off.p, n + 1, tmp.p, s);
  PSG_CUDA(cudaMemcpyAsync(cnt.p, off.p, (n + 1) * 4, cudaMemcpyDeviceToDevice, s));  // cursors
  if (m) {
    k_row_scatter<<<grid_cap(m), 256, 0, s>>>(pairs.p, m, both, cnt.p, cols.p);
    PSG_LAUNCHED();
  }
  k_sort_rows<<<grid_cap(n * 32), 256, 0, s>>>(off.p, n, cols.p, flag.p);
  PSG_LAUNCHED();
  g_launches += 6;
  unsigned h = 0;
  PSG_CUDA(cudaMemcpyAsync(&h, flag.p, 4, cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaStreamSynchronize(s));
  return h == 0;
}

}  // namespace

// Emitted (i<<32|j) pairs on device -> CSR lists on the host (or counts only).
void finish_neighbors(DevBuf<uint64_t>& pairs, uint64_t m, uint64_t n, bool want_lists, psg_neighbor_result* out,
                      cudaStream_t s) {
  out->n = n;
  out->pair_count = m;
  out->offsets = nullptr;
  out->neighbors = nullptr;
  if (!want_lists) return;
  out->offsets = static_cast<uint64_t*>(std::malloc((n + 1) * sizeof(uint64_t)));
  out->neighbors = static_cast<uint64_t*>(std::malloc(std::max<uint64_t>(2 * m, 1) * sizeof(uint64_t)));
  if (!out->offsets || !out->neighbors) throw std::bad_alloc();
  DevBuf<uint32_t> off32, cols;
  if (csr_rows(pairs, m, n, true, off32, cols, s)) {
    DevBuf<uint64_t> off(n + 1, s), nb(std::max<uint64_t>(2 * m, 1), s);
    k_widen_offsets<<<grid_cap(n + 1), 256, 0, s>>>(off32.p, n + 1, off.p);
    PSG_LAUNCHED();
    if (m) {
      k_cols_to_u64<<<grid_cap(2 * m), 256, 0, s>>>(cols.p, 2 * m, nb.p);
      PSG_LAUNCHED();
    }
    g_launches += 2;
    PSG_CUDA(cudaMemcpyAsync(out->offsets, off.p, (n + 1) * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    if (m) PSG_CUDA(cudaMemcpyAsync(out->neighbors, nb.p, 2 * m * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  } else {  // a row longer than 1024: sort the directed pairs globally
    const int b = bits_for(n);
    DevBuf<uint64_t> dir(std::max<uint64_t>(2 * m, 1), s);
    k_directed<<<blocks(m, 256), 256, 0, s>>>(pairs.p, m, b, dir.p);
    PSG_LAUNCHED();
    sort_u64(dir, 2 * m, 2 * b, s);
    DevBuf<uint64_t> off(n + 1, s);
    k_offsets<<<blocks(n + 1, 256), 256, 0, s>>>(dir.p, 2 * m, n, b, off.p);
    PSG_LAUNCHED();
    k_low_bits<<<blocks(2 * m, 256), 256, 0, s>>>(dir.p, 2 * m, b);
    PSG_LAUNCHED();
    g_launches += 3;
    PSG_CUDA(cudaMemcpyAsync(out->offsets, off.p, (n + 1) * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    PSG_CUDA(cudaMemcpyAsync(out->neighbors, dir.p, 2 * m * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  }
  PSG_CUDA(cudaStreamSynchronize(s));
  g_prof.d2h_bytes += (n + 1 + 2 * m) * sizeof(uint64_t);
}

namespace {

struct FrnnRun {
  DevBuf<uint64_t> pairs;
  uint64_t count = 0, hash = 0, visited = 0, examined = 0;
};

}  // namespace

// Everything before the candidate scan, shared by every part of a sharded
// solve (identical on every rank): projection, the R-derived thresholds, the
// cell grid and (d <= 4) the coordinates in cell order.
struct FrnnPlan {
  psg_pointset* ps = nullptr;
  uint64_t zone = 0;
  double radius = 0;
  Thresholds th{};
  float lo = -1.f;
  uint64_t ncells = 1;
  int nk = 4;
  bool small_d = false;
  DevBuf<float> keys;
  GridIndex gi;
  DevBuf<float4> sx;
  DevBuf<unsigned long long> acc;
  DevBuf<uint64_t> band;
  uint64_t bcap = 1u << 16;
  FrnnRun run;  // the last part scanned
};

FrnnPlan* frnn_plan_create(psg_pointset* ps, double radius, uint64_t q, double f, uint64_t seed, uint64_t zone) {
  const uint64_t n = ps->n;
  if (n == 0) throw invalid_argument("empty input");  // refscan.cpp:162, before the radius check
  if (!(radius > 0.0) || !std::isfinite(radius)) throw invalid_argument("radius must be positive");
  check_reference_args(n, std::min(q, n), f);  // refscan.cpp:165 clamps q to n
  if (n >= 0xffffffffull) throw invalid_argument("point count exceeds 2^32-1");
  Ctx& c = ctx();
  cudaStream_t s = c.stream;
  StageTimer tm(s);
  auto plan = std::make_unique<FrnnPlan>();
  FrnnPlan& P = *plan;
  P.ps = ps;
  P.zone = zone;
  P.radius = radius;
  const Directions dir = make_directions(seed, ps->d, static_cast<int>(std::min<uint64_t>(std::min(q, n), 64)));
  const int nk = dir.nk;
  P.nk = nk;
  P.keys.alloc(n * nk, s);
  const float norm2 = project(*ps, dir, P.keys.p, s);
  tm.mark("project");
  const Budget bud = make_budget(*ps, dir, norm2);
  const double Rw = radius * ps->scale;
  const double dmax = (Rw * (1.0 + 4.0 * bud.gamma64) + 2.0 * bud.Rn) * (1.0 + 1e-12);
  P.th = budget_thresholds(bud, dmax);
  const double inner = Rw * (1.0 - 4.0 * bud.gamma64) - 2.0 * bud.Rn;
  P.lo = inner > 0 ? static_cast<float>(((inner * inner) * (1.0 - bud.e) - bud.a) * (1.0 - 1e-6)) : -1.0f;

  // grid over the first g keys, cell width >= the key window of R
  const int g = std::min(3, dir.q);
  GridIndex& gi = P.gi;
  gi.ensure(static_cast<uint32_t>(n), nk, s);
  {
    DevBuf<unsigned> mm(6, s);
    const unsigned init[6] = {~0u, ~0u, ~0u, 0u, 0u, 0u};
    PSG_CUDA(cudaMemcpyAsync(mm.p, init, 24, cudaMemcpyHostToDevice, s));
    const unsigned gb = std::min<unsigned>(blocks(n, 256), c.sm_count * 8);
    if (nk == 4)
      k_key_range<4><<<gb, 256, 0, s>>>(P.keys.p, static_cast<uint32_t>(n), g, mm.p, mm.p + 3);
    else
      k_key_range<8><<<gb, 256, 0, s>>>(P.keys.p, static_cast<uint32_t>(n), g, mm.p, mm.p + 3);
    PSG_LAUNCHED();
    ++g_launches;
    unsigned h[6];
    PSG_CUDA(cudaMemcpyAsync(h, mm.p, 24, cudaMemcpyDeviceToHost, s));
    PSG_CUDA(cudaStreamSynchronize(s));
    double lo3[kMaxGridKeys] = {}, span[kMaxGridKeys] = {};
    for (int t = 0; t < g; ++t) {
      lo3[t] = f32_unorder(h[t]);
      span[t] = std::max(static_cast<double>(f32_unorder(h[3 + t])) - lo3[t], 1e-30);
    }
    GridParams gp;
    grid_params_for(gp, std::max(g, 1), static_cast<double>(P.th.win) * (1.0 + 1e-6), lo3, span);
    P.ncells = gp.cells;
    PSG_CUDA(cudaMemcpyAsync(gi.gp.p, &gp, sizeof(GridParams), cudaMemcpyHostToDevice, s));
  }
  build_grid(P.keys.p, static_cast<uint32_t>(n), nk, gi, 24, s);
  P.small_d = ps->d <= 4;
  if (P.small_d) {
    P.sx.alloc(n, s);
    k_gather_rows4<<<blocks(n, 256), 256, 0, s>>>(ps->rows(), gi.sidx.p, static_cast<uint32_t>(n), ps->d, P.sx.p);
    PSG_LAUNCHED();
    ++g_launches;
  }
  P.acc.alloc(8, s);
  tm.mark("grid");
  PSG_CUDA(cudaStreamSynchronize(s));
  prof_stages(tm);
  return plan.release();
}

// The pairs of part `part` of `nparts` (sorted positions split evenly; a pair
// belongs to the part holding its earlier position).  emit = false: count +
// hash only (no pair list is materialised for d <= 4).
void frnn_plan_scan(FrnnPlan& P, uint64_t part, uint64_t nparts, bool emit) {
  psg_pointset* ps = P.ps;
  const uint64_t n = ps->n;
  Ctx& c = ctx();
  cudaStream_t s = c.stream;
  StageTimer tm(s);
  FrnnRun& run = P.run;
  run = FrnnRun{};
  FrnnArgs a{};
  a.X = ps->rows();
  a.skeys = P.gi.skeys.p;
  a.sx = P.sx.p;
  a.sidx = P.gi.sidx.p;
  a.grid = P.gi.dev;
  a.n = static_cast<uint32_t>(n);
  a.d = ps->d;
  a.zone = P.zone;
  a.th = P.th;
  a.lo = P.lo;
  a.R = P.radius;
  a.src = ps->exact();
  a.plo = static_cast<uint32_t>(n * part / nparts);
  a.phi = static_cast<uint32_t>(n * (part + 1) / nparts);
  const uint32_t rows = a.phi - a.plo;
  unsigned long long* acc = P.acc.p;
  // count-only runs of the small-d scan never write pairs
  const bool no_list = P.small_d && !emit;
  uint64_t cap = no_list ? 0 : std::max<uint64_t>(1u << 20, 24 * std::max<uint64_t>(rows, 1));
  for (;;) {
    run.pairs.alloc(std::max<uint64_t>(cap, 1), s);
    PSG_CUDA(cudaMemsetAsync(acc, 0, 64, s));
    a.out = run.pairs.p;
    a.cap = cap;
    a.acc = acc;
    if (P.small_d) {
      if (P.band.n < P.bcap) P.band.alloc(P.bcap, s);
      a.band = P.band.p;
      a.bcap = P.bcap;
      k_part_cells<<<1, 1, 0, s>>>(a);
      PSG_LAUNCHED();
      const uint64_t part_cells = (P.ncells + nparts - 1) / nparts + 1;  // launch size only (claims are dynamic)
      const unsigned cb = static_cast<unsigned>(std::min<uint64_t>(
          (part_cells + 32 * (kFrnnThreads / 32) - 1) / (32 * (kFrnnThreads / 32)), c.sm_count * 4ull));
      const int v = (no_list ? 0 : 4) + (ps->d == 4 ? 2 : 0) + (P.zone > 1 ? 1 : 0);
      switch (v) {
        case 0: k_frnn_cells<false, false, false><<<cb, kFrnnThreads, 0, s>>>(a); break;
        case 1: k_frnn_cells<false, false, true><<<cb, kFrnnThreads, 0, s>>>(a); break;
        case 2: k_frnn_cells<false, true, false><<<cb, kFrnnThreads, 0, s>>>(a); break;
        case 3: k_frnn_cells<false, true, true><<<cb, kFrnnThreads, 0, s>>>(a); break;
        case 4: k_frnn_cells<true, false, false><<<cb, kFrnnThreads, 0, s>>>(a); break;
        case 5: k_frnn_cells<true, false, true><<<cb, kFrnnThreads, 0, s>>>(a); break;
        case 6: k_frnn_cells<true, true, false><<<cb, kFrnnThreads, 0, s>>>(a); break;
        default: k_frnn_cells<true, true, true><<<cb, kFrnnThreads, 0, s>>>(a); break;
      }
      PSG_LAUNCHED();
      g_launches += 2;
      k_frnn_band<<<c.sm_count * 2, 256, 0, s>>>(a);
    } else if (rows) {
      if (P.nk == 4)
        k_frnn_scan<4><<<blocks(rows, kFrnnThreads), kFrnnThreads, 0, s>>>(a);
      else
        k_frnn_scan<8><<<blocks(rows, kFrnnThreads), kFrnnThreads, 0, s>>>(a);
    }
    PSG_LAUNCHED();
    ++g_launches;
    unsigned long long h[5];
    PSG_CUDA(cudaMemcpyAsync(h, acc, 40, cudaMemcpyDeviceToHost, s));
    PSG_CUDA(cudaStreamSynchronize(s));
    if (P.small_d && h[4] > P.bcap) {  // more rounding-band pairs than room: again with room for all
      P.bcap = h[4];
      continue;
    }
    if (no_list || h[0] <= cap) {
      run.count = h[0];
      run.hash = h[1];
      run.visited = h[2];
      run.examined = h[3];
      break;
    }
    cap = h[0];
  }
  tm.mark("scan");
  PSG_CUDA(cudaStreamSynchronize(s));
  prof_stages(tm);
  g_prof.window_pairs = run.visited;
  g_prof.lb_survivors = run.examined;
}

void frnn_plan_free(FrnnPlan* p) { delete p; }

// Part stats: examined = FP32-evaluated pairs, pruned = visited - examined;
// the caller adds the parts up and fills pairs_skipped_by_exit from the
// closed-form admissible count.
void frnn_plan_result(const FrnnPlan& P, uint64_t* count, uint64_t* hash, psg_scan_stats* stats) {
  *count = P.run.count;
  *hash = P.run.hash;
  stats->pairs_examined = P.run.examined;
  stats->pairs_pruned_by_reference = P.run.visited - P.run.examined;
  stats->pairs_skipped_by_exit = 0;
  stats->inner_loop_exits = 0;
}

namespace {

// The (i<j) pairs of a run, sorted ascending, into `sorted` (device).
void sort_pairs(const FrnnRun& run, uint64_t n, DevBuf<uint64_t>& sorted, cudaStream_t s) {
  sorted.alloc(std::max<uint64_t>(run.count, 1), s);
  if (run.count == 0) return;
  DevBuf<uint32_t> off, cols;
  if (csr_rows(run.pairs, run.count, n, false, off, cols, s)) {  // rows of i<j, ascending
    k_csr_to_pairs<<<grid_cap(n * 32), 256, 0, s>>>(off.p, n, cols.p, sorted.p);
    PSG_LAUNCHED();
    ++g_launches;
  } else {
    const int b = bits_for(n);
    k_pack<<<blocks(run.count, 256), 256, 0, s>>>(run.pairs.p, run.count, b, sorted.p);
    PSG_LAUNCHED();
    sort_u64(sorted, run.count, 2 * b, s);
    k_unpack<<<blocks(run.count, 256), 256, 0, s>>>(sorted.p, run.count, b);
    PSG_LAUNCHED();
    g_launches += 2;
  }
}

FrnnRun frnn_run(psg_pointset* ps, double radius, uint64_t q, double f, uint64_t seed, uint64_t zone,
                 bool emit = true) {
  trace("frnn: enter");
  std::unique_ptr<FrnnPlan> plan(frnn_plan_create(ps, radius, q, f, seed, zone));
  trace("frnn: plan");
  frnn_plan_scan(*plan, 0, 1, emit);
  trace("frnn: scan");
  return std::move(plan->run);
}

}  // namespace

void frnn_plan_pairs(FrnnPlan& P, uint64_t nbuckets, uint64_t* bucket_counts, uint64_t* out, uint64_t capacity) {
  cudaStream_t s = ctx().stream;
  const uint64_t n = P.ps->n, m = P.run.count;
  DevBuf<uint64_t> sorted;
  sort_pairs(P.run, n, sorted, s);
  std::vector<uint64_t> host;
  uint64_t* dst = out;
  if (m > capacity || !out) {  // bucket counts still need the keys: stage them
    host.resize(m);
    dst = host.data();
  }
  if (m) PSG_CUDA(cudaMemcpyAsync(dst, sorted.p, m * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaStreamSynchronize(s));
  if (dst == out) g_prof.d2h_bytes += m * sizeof(uint64_t);
  // bucket b holds the pairs with i in [n b / nb, n (b + 1) / nb): the sorted
  // list is already in bucket order
  uint64_t k = 0;
  for (uint64_t b = 0; b < nbuckets; ++b) {
    const uint64_t ihi = n * (b + 1) / nbuckets;
    const uint64_t* e = std::lower_bound(dst + k, dst + m, ihi << 32);
    bucket_counts[b] = static_cast<uint64_t>(e - (dst + k));
    k = static_cast<uint64_t>(e - dst);
  }
}

void frnn_solve(psg_pointset* ps, double radius, uint64_t q, double f, uint64_t seed, uint64_t zone,
                bool want_lists, psg_neighbor_result* out) {
  FrnnRun run = frnn_run(ps, radius, q, f, seed, zone, want_lists);
  cudaStream_t s = ctx().stream;
  finish_neighbors(run.pairs, run.count, ps->n, want_lists, out, s);
  out->pair_hash = run.hash;
  const uint64_t adm = admissible_pairs(ps->n, zone);
  out->stats.pairs_examined = run.examined;
  out->stats.pairs_pruned_by_reference = run.visited - run.examined;
  out->stats.pairs_skipped_by_exit = adm - run.visited;
  out->stats.inner_loop_exits = 0;
}

namespace {
// The sorted list to the host in i-range buckets: one scatter into packed
// buckets, then per bucket a radix sort on the library stream and its copy on
// the context's copy stream as soon as it is sorted (the D2H of one bucket
// overlaps the sort of the next; the copy engine stays busy).
void sorted_list_to_host(const FrnnRun& run, uint64_t n, uint64_t* host, uint64_t m, cudaStream_t s) {
  Ctx& c = ctx();
  const int B = kListBuckets;
  const int bj = bits_for(n);
  int bi = 1;
  while ((1ull << bi) < (n + B - 1) / B + 1) ++bi;
  DevBuf<unsigned long long> cnt(2 * B, s);
  PSG_CUDA(cudaMemsetAsync(cnt.p, 0, 2 * B * sizeof(unsigned long long), s));
  const unsigned g = grid_cap(run.count);
  k_bucket_count<<<g, 256, 0, s>>>(run.pairs.p, run.count, n, B, cnt.p);
  PSG_LAUNCHED();
  unsigned long long hc[kListBuckets];
  PSG_CUDA(cudaMemcpyAsync(hc, cnt.p, B * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaStreamSynchronize(s));
  unsigned long long off[kListBuckets + 1] = {0}, biggest = 0;
  for (int b = 0; b < B; ++b) {
    off[b + 1] = off[b] + hc[b];
    biggest = std::max(biggest, hc[b]);
  }
  PSG_CUDA(cudaMemcpyAsync(cnt.p + B, off, B * sizeof(unsigned long long), cudaMemcpyHostToDevice, s));
  DevBuf<uint64_t> a(run.count, s), tmp(std::max<uint64_t>(biggest, 1), s);
  DevBuf<uint32_t> hist(radix_hist_words(std::max<uint64_t>(biggest, 2)), s);
  k_bucket_scatter<<<g, 256, 0, s>>>(run.pairs.p, run.count, n, B, bj, cnt.p + B, a.p);
  PSG_LAUNCHED();
  g_launches += 2;
  if (!c.copy_stream) PSG_CUDA(cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking));
  std::vector<cudaEvent_t> ev(B);
  for (int b = 0; b < B; ++b) ev[b] = c.get_event();
  const int passes = (bi + bj + 7) / 8;
  for (int b = 0; b < B; ++b) {  // all sorts first (the copies below may block the host on pageable memory)
    const uint64_t len = hc[b];
    uint64_t* kk[2] = {a.p + off[b], tmp.p};
    uint32_t* vv[2] = {nullptr, nullptr};
    if (len > 1) {
      const int which = radix_sort<uint64_t>(kk, vv, len, 0, passes * 8, hist.p, s);
      if (which == 1) PSG_CUDA(cudaMemcpyAsync(kk[0], kk[1], len * 8, cudaMemcpyDeviceToDevice, s));
      g_launches += 1 + passes;
    }
    if (len) {
      k_bucket_unpack<<<blocks(len, 256), 256, 0, s>>>(a.p + off[b], len, bj, (n * b + B - 1) / B);
      PSG_LAUNCHED();
      ++g_launches;
    }
    PSG_CUDA(cudaEventRecord(ev[b], s));
  }
  for (int b = 0; b < B && off[b] < m; ++b) {
    PSG_CUDA(cudaStreamWaitEvent(c.copy_stream, ev[b], 0));
    const uint64_t len = std::min<uint64_t>(hc[b], m - off[b]);
    if (len)
      PSG_CUDA(cudaMemcpyAsync(host + off[b], a.p + off[b], len * 8, cudaMemcpyDeviceToHost, c.copy_stream));
  }
  PSG_CUDA(cudaStreamSynchronize(c.copy_stream));
  PSG_CUDA(cudaStreamSynchronize(s));
  for (int b = 0; b < B; ++b) c.put_event(ev[b]);
}

// The sorted (i<j) lists as upper-triangular CSR on the host: offs[n + 1]
// (u64) and cols (u32, the first `cap` of them), in i-range buckets like
// sorted_list_to_host — each bucket sorted on the library stream, turned into
// its columns and row offsets, and copied on the copy stream while the next
// bucket sorts.  12 bytes per pair less 4: the 530 MB of C4's packed pairs
// become 265 MB of columns + 32 MB of offsets.
// The (i<j) lists as CSR through the row-group kernels (k_group_*), the
// group sorts in chunks so the copies overlap them.  Returns false (nothing
// written) when the shape is outside their limits: more than kMaxGroups
// groups, a group over kGroupCap pairs, or 2^32 pairs.
bool sorted_csr_groups(const FrnnRun& run, uint64_t n, uint64_t* offs, uint32_t* cols, uint64_t cap,
                       cudaStream_t s) {
  Ctx& c = ctx();
  const uint64_t m = run.count;
  const uint32_t ng = static_cast<uint32_t>((n + kGroupRows - 1) >> kGroupShift);
  if (ng > kMaxGroups || m >= 0xffffffffull || m == 0) return false;
  set_max_dynamic_smem(reinterpret_cast<const void*>(k_group_hist), kMaxGroups * 4);
  set_max_dynamic_smem(reinterpret_cast<const void*>(k_group_scatter), kMaxGroups * 8);
  set_max_dynamic_smem(reinterpret_cast<const void*>(k_group_sort), kGroupCap * 4);
  DevBuf<unsigned> gcnt(ng + 1, s);
  PSG_CUDA(cudaMemsetAsync(gcnt.p, 0, (ng + 1) * 4, s));
  k_group_hist<<<c.sm_count, kGroupHistThreads, ng * 4, s>>>(run.pairs.p, m, ng, gcnt.p);
  PSG_LAUNCHED();
  std::vector<uint32_t> gs(ng + 1);
  PSG_CUDA(cudaMemcpyAsync(gs.data(), gcnt.p, ng * 4, cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaStreamSynchronize(s));
  uint32_t run_sum = 0, biggest = 0;
  for (uint32_t g = 0; g < ng; ++g) {
    const uint32_t v = gs[g];
    biggest = std::max(biggest, v);
    gs[g] = run_sum;
    run_sum += v;
  }
  gs[ng] = run_sum;
  trace("csr groups: histogram");
  if (biggest > kGroupCap) return false;
  DevBuf<uint32_t> gstart(ng + 1, s);
  DevBuf<uint64_t> grouped(m, s), doffs(n + 1, s);
  DevBuf<uint32_t> dcols(m, s);
  PSG_CUDA(cudaMemcpyAsync(gstart.p, gs.data(), (ng + 1) * 4, cudaMemcpyHostToDevice, s));
  PSG_CUDA(cudaMemcpyAsync(gcnt.p, gstart.p, ng * 4, cudaMemcpyDeviceToDevice, s));  // cursors
  // one pass by group, a contiguous slice per block (a coarse pass first to
  // lengthen the runs measured the same: ~0.57 ms per pass over C4's 66M pairs)
  k_group_scatter<<<c.sm_count, kGroupHistThreads, ng * 8, s>>>(run.pairs.p, m, kGroupShift, ng, 0, gcnt.p,
                                                                 grouped.p);
  PSG_LAUNCHED();
  g_launches += 2;
  if (!c.copy_stream) PSG_CUDA(cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking));
  const uint32_t chunks = std::min<uint32_t>(ng, 16);
  std::vector<cudaEvent_t> ev(chunks);
  for (auto& e : ev) e = c.get_event();
  for (uint32_t k = 0; k < chunks; ++k) {
    const uint32_t ga = static_cast<uint32_t>(static_cast<uint64_t>(ng) * k / chunks);
    const uint32_t gb = static_cast<uint32_t>(static_cast<uint64_t>(ng) * (k + 1) / chunks);
    if (gb > ga) {
      k_group_sort<<<gb - ga, kGroupSortThreads, kGroupCap * 4, s>>>(grouped.p, gstart.p, ga, n, dcols.p, doffs.p);
      PSG_LAUNCHED();
      ++g_launches;
    }
    PSG_CUDA(cudaEventRecord(ev[k], s));
  }
  trace("csr groups: enqueued");
  for (uint32_t k = 0; k < chunks; ++k) {
    const uint32_t ga = static_cast<uint32_t>(static_cast<uint64_t>(ng) * k / chunks);
    const uint32_t gb = static_cast<uint32_t>(static_cast<uint64_t>(ng) * (k + 1) / chunks);
    PSG_CUDA(cudaStreamWaitEvent(c.copy_stream, ev[k], 0));
    const uint64_t ra = static_cast<uint64_t>(ga) << kGroupShift, rb = std::min<uint64_t>(n, uint64_t(gb) << kGroupShift);
    if (rb > ra)
      PSG_CUDA(cudaMemcpyAsync(offs + ra, doffs.p + ra, (rb - ra) * 8, cudaMemcpyDeviceToHost, c.copy_stream));
    const uint64_t ca = gs[ga], cb = std::min<uint64_t>(gs[gb], cap);
    if (cb > ca)
      PSG_CUDA(cudaMemcpyAsync(cols + ca, dcols.p + ca, (cb - ca) * 4, cudaMemcpyDeviceToHost, c.copy_stream));
  }
  PSG_CUDA(cudaStreamSynchronize(s));
  trace("csr groups: sorted");
  PSG_CUDA(cudaStreamSynchronize(c.copy_stream));
  trace("csr groups: copied");
  offs[n] = m;
  for (auto& e : ev) c.put_event(e);
  return true;
}

void sorted_csr_to_host(const FrnnRun& run, uint64_t n, uint64_t* offs, uint32_t* cols, uint64_t cap,
                        cudaStream_t s) {
  Ctx& c = ctx();
  const uint64_t m = run.count;
  const int B = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(kListBuckets, m >> 17)));
  const int bj = bits_for(n);
  int bi = 1;
  while ((1ull << bi) < (n + B - 1) / B + 1) ++bi;
  DevBuf<unsigned long long> cnt(2 * kListBuckets, s);
  PSG_CUDA(cudaMemsetAsync(cnt.p, 0, 2 * kListBuckets * sizeof(unsigned long long), s));
  unsigned long long hc[kListBuckets] = {0};
  const unsigned g = grid_cap(std::max<uint64_t>(m, 1));
  if (m) {
    k_bucket_count<<<g, 256, 0, s>>>(run.pairs.p, m, n, B, cnt.p);
    PSG_LAUNCHED();
    PSG_CUDA(cudaMemcpyAsync(hc, cnt.p, B * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    PSG_CUDA(cudaStreamSynchronize(s));
  }
  unsigned long long off[kListBuckets + 1] = {0}, biggest = 0;
  for (int b = 0; b < B; ++b) {
    off[b + 1] = off[b] + hc[b];
    biggest = std::max(biggest, hc[b]);
  }
  PSG_CUDA(cudaMemcpyAsync(cnt.p + B, off, B * sizeof(unsigned long long), cudaMemcpyHostToDevice, s));
  DevBuf<uint64_t> a(std::max<uint64_t>(m, 1), s), tmp(std::max<uint64_t>(biggest, 1), s), doffs(n + 1, s);
  DevBuf<uint32_t> dcols(std::max<uint64_t>(m, 1), s);
  DevBuf<uint32_t> hist(radix_hist_words(std::max<uint64_t>(biggest, 2)), s);
  if (m) {
    k_bucket_scatter<<<g, 256, 0, s>>>(run.pairs.p, m, n, B, bj, cnt.p + B, a.p);
    PSG_LAUNCHED();
    g_launches += 2;
  }
  if (!c.copy_stream) PSG_CUDA(cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking));
  std::vector<cudaEvent_t> ev(B);
  for (int b = 0; b < B; ++b) ev[b] = c.get_event();
  const int passes = (bi + bj + 7) / 8;
  for (int b = 0; b < B; ++b) {
    const uint64_t len = hc[b], i0 = (n * b + B - 1) / B, i1 = (n * (b + 1) + B - 1) / B;
    uint64_t* kk[2] = {a.p + off[b], tmp.p};
    uint32_t* vv[2] = {nullptr, nullptr};
    if (len > 1) {
      const int which = radix_sort<uint64_t>(kk, vv, len, 0, passes * 8, hist.p, s);
      g_launches += 1 + passes;
      kk[0] = kk[which];
    }
    if (len) {
      k_bucket_csr<<<blocks(len, 256), 256, 0, s>>>(kk[0], len, bj, i0, i1, off[b], dcols.p + off[b], doffs.p);
    } else if (i1 > i0) {
      k_fill_u64<<<blocks(i1 - i0, 256), 256, 0, s>>>(doffs.p + i0, i1 - i0, off[b]);
    }
    PSG_LAUNCHED();
    ++g_launches;
    PSG_CUDA(cudaEventRecord(ev[b], s));
  }
  for (int b = 0; b < B; ++b) {
    PSG_CUDA(cudaStreamWaitEvent(c.copy_stream, ev[b], 0));
    const uint64_t i0 = (n * b + B - 1) / B, i1 = (n * (b + 1) + B - 1) / B;
    if (i1 > i0)
      PSG_CUDA(cudaMemcpyAsync(offs + i0, doffs.p + i0, (i1 - i0) * 8, cudaMemcpyDeviceToHost, c.copy_stream));
    if (off[b] < cap) {
      const uint64_t len = std::min<uint64_t>(hc[b], cap - off[b]);
      if (len)
        PSG_CUDA(cudaMemcpyAsync(cols + off[b], dcols.p + off[b], len * 4, cudaMemcpyDeviceToHost, c.copy_stream));
    }
  }
  PSG_CUDA(cudaStreamSynchronize(c.copy_stream));
  PSG_CUDA(cudaStreamSynchronize(s));
  offs[n] = m;
  for (int b = 0; b < B; ++b) c.put_event(ev[b]);
}
}  // namespace

void frnn_pairs(psg_pointset* ps, double radius, uint64_t q, double f, uint64_t seed, uint64_t zone,
                uint64_t* pairs, uint64_t capacity, uint64_t* count, uint64_t* hash) {
  FrnnRun run = frnn_run(ps, radius, q, f, seed, zone, pairs && capacity);
  cudaStream_t s = ctx().stream;
  *count = run.count;
  *hash = run.hash;
  if (!pairs || capacity == 0 || run.count == 0) return;
  const uint64_t m = std::min(capacity, run.count);
  static const bool no_buckets = std::getenv("PSG_LIST_CSR") != nullptr;  // A/B: the one-shot CSR + copy
  if (run.count >= (1u << 22) && ps->n >= 1024 && !no_buckets) {
    StageTimer tm(s);
    sorted_list_to_host(run, ps->n, pairs, m, s);
    tm.mark("sort+d2h");
    PSG_CUDA(cudaStreamSynchronize(s));
    prof_stages(tm);
    g_prof.d2h_bytes += m * sizeof(uint64_t);
    return;
  }
  StageTimer tm(s);
  DevBuf<uint64_t> sorted;
  sort_pairs(run, ps->n, sorted, s);
  tm.mark("sort");
  PSG_CUDA(cudaMemcpyAsync(pairs, sorted.p, m * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  tm.mark("d2h");
  PSG_CUDA(cudaStreamSynchronize(s));
  prof_stages(tm);
  g_prof.d2h_bytes += m * sizeof(uint64_t);
}

void frnn_pairs_csr(psg_pointset* ps, double radius, uint64_t q, double f, uint64_t seed, uint64_t zone,
                    uint64_t* offsets, uint32_t* cols, uint64_t capacity, uint64_t* count, uint64_t* hash) {
  FrnnRun run = frnn_run(ps, radius, q, f, seed, zone, true);
  cudaStream_t s = ctx().stream;
  *count = run.count;
  *hash = run.hash;
  if (!offsets) return;
  StageTimer tm(s);
  static const bool radix = std::getenv("PSG_CSR_RADIX") != nullptr;  // A/B: the i-range radix buckets
  if (radix || !sorted_csr_groups(run, ps->n, offsets, cols, cols ? capacity : 0, s))
    sorted_csr_to_host(run, ps->n, offsets, cols, cols ? capacity : 0, s);
  tm.mark("sort+d2h");
  trace("frnn: csr to host");
  PSG_CUDA(cudaStreamSynchronize(s));
  prof_stages(tm);
  g_prof.d2h_bytes += (ps->n + 1) * 8 + std::min(capacity, run.count) * 4;
}

void brute_neighbors(psg_pointset* ps, double radius, uint64_t zone, bool want_lists, psg_neighbor_result* out) {
  if (!(radius > 0.0) || !std::isfinite(radius)) throw invalid_argument("radius must be positive");
  if (ps->n >= 0xffffffffull) throw invalid_argument("point count exceeds 2^32-1");
  cudaStream_t s = ctx().stream;
  DevBuf<uint64_t> pairs;
  uint64_t hash = 0;
  const uint64_t m = ps->n >= 2 ? brute_emit_pairs(ps, radius, zone, pairs, &hash, s) : 0;
  if (!pairs.p) pairs.alloc(1, s);
  finish_neighbors(pairs, m, ps->n, want_lists, out, s);
  out->pair_hash = hash;
  out->stats = psg_scan_stats{admissible_pairs(ps->n, zone), 0, 0, 0};
}

}  // namespace psg
