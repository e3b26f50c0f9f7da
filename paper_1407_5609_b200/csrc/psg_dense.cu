// psg_dense.cu — dense cell-pair engine (psg_dense.cuh).
//
// When the grid's cells hold many points (clustered data: the closest pair
// sits at the scale of a cluster, so a key window of the bound spans whole
// clusters), per-point candidate lists degenerate: every point would walk
// ~10^4-10^5 candidates.  Here the unit of work is a pair of cells instead:
//   1. the non-empty cells (a list), per-cell boxes over all nk keys (warp
//      per non-empty cell)
//   2. keep a forward-stencil cell pair (A, B) only if the box gap lower
//      bound is within the threshold — pairs of points of different clusters
//      are dropped a whole cell pair at a time (warp per A, lanes over the
//      3^g/2 stencil offsets)
//   3. kept cell pairs are cut into 128x128 tiles; a persistent kernel takes
//      tiles from an atomic cursor and evaluates every pair as a canonical
//      FP32 distance (16-wide coordinate slabs in shared memory, 8x8 pairs per
//      thread — the all-pairs kernel's arithmetic and order) from rows
//      gathered into grid order, recording the band into the candidate list.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <cmath>

#include "psg_cpp.cuh"
#include "psg_dense.cuh"
#include "psg_points.cuh"
#include "psg_sort.cuh"
#include "psg_tc.cuh"

namespace psg {
namespace {

constexpr int kT = 128;   // tile edge (points)
constexpr int kDK = 16;   // coordinate slab
constexpr int kPad = 132;

unsigned blocks(uint64_t n, int per) { return static_cast<unsigned>((n + per - 1) / per); }

__device__ __forceinline__ int pow3(int g) {
  int r = 1;
  for (int t = 0; t < g; ++t) r *= 3;
  return r;
}

// Cell coordinates (dim 0 most significant), g <= kMaxGridKeys.
__device__ __forceinline__ void cell_decode(const GridParams& P, uint32_t c, int (&cc)[kMaxGridKeys]) {
#pragma unroll
  for (int t = kMaxGridKeys - 1; t >= 0; --t) {
    if (t >= P.g) {
      cc[t] = 0;
      continue;
    }
    cc[t] = static_cast<int>(c % P.dims[t]);
    c /= P.dims[t];
  }
}

// The s-th forward neighbour (s = 1..(3^g-1)/2): offsets lexicographically
// after (0,..,0) in the 3^g stencil.  false when outside the grid.
__device__ __forceinline__ bool cell_forward(const GridParams& P, const int (&cc)[kMaxGridKeys], int s,
                                             uint32_t* out) {
  int code = pow3(P.g) / 2 + s;
  int off[kMaxGridKeys];
#pragma unroll
  for (int t = kMaxGridKeys - 1; t >= 0; --t) {
    if (t >= P.g) {
      off[t] = 0;
      continue;
    }
    off[t] = code % 3 - 1;
    code /= 3;
  }
  uint32_t c = 0;
#pragma unroll
  for (int t = 0; t < kMaxGridKeys; ++t) {
    if (t >= P.g) break;
    const int v = cc[t] + off[t];
    if (v < 0 || v >= static_cast<int>(P.dims[t])) return false;
    c = c * P.dims[t] + static_cast<uint32_t>(v);
  }
  *out = c;
  return true;
}

__device__ __forceinline__ int forward_count(int g) { return (pow3(g) - 1) / 2; }

// Estimate of the stencil pairs the sparse scan would visit (the dense /
// sparse decision, a heuristic against 512 n): every kEstStride-th cell,
// scaled back up; GridParams once per block in shared memory.
constexpr uint32_t kEstStride = 8;
__global__ void k_estimate(const uint32_t* __restrict__ cfirst, const GridParams* __restrict__ gpp, uint64_t cells,
                           unsigned long long* __restrict__ est) {
  __shared__ GridParams P;
  if (threadIdx.x == 0) P = *gpp;
  __syncthreads();
  unsigned long long total = 0;
  for (uint64_t A = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) * kEstStride; A < cells;
       A += static_cast<uint64_t>(gridDim.x) * blockDim.x * kEstStride) {
    const unsigned long long na = cfirst[A + 1] - cfirst[A];
    if (na == 0) continue;
    total += na * (na - 1) / 2;
    int cc[kMaxGridKeys];
    cell_decode(P, static_cast<uint32_t>(A), cc);
    for (int s = 1; s <= forward_count(P.g); ++s) {
      uint32_t B;
      if (cell_forward(P, cc, s, &B)) total += na * (cfirst[B + 1] - cfirst[B]);
    }
  }
  for (int o = 16; o; o >>= 1) total += __shfl_xor_sync(kFull, total, o);
  if ((threadIdx.x & 31) == 0 && total) atomicAdd(est, total * kEstStride);
}

// Rows in grid order (materialised here also for window sets: the tiles
// stream them with TMA / wide loads).
// Rows in cell order, dx >= d floats each: coordinates past d are zero (the
// Gram tiles' padded width; a zero coordinate adds fmaf(0, 0, s) == s to a
// canonical distance and nothing to a norm or a dot product).
__global__ void k_gather_rows(Rows R, const uint32_t* __restrict__ sidx, uint32_t n, int d, int dx,
                              float* __restrict__ Xs) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t p = warp; p < n; p += nwarps) {
    const uint32_t i = sidx[p];
    float* dst = Xs + static_cast<size_t>(p) * dx;
    for (int t = lane; t < dx; t += 32) dst[t] = t < d ? row_at(R, i, t) : 0.f;
  }
}

// The non-empty cells (run starts of the cell-sorted ids), in arbitrary order:
// every consumer below is per cell, and a cell's pairs keep their stencil order.
__global__ void k_cell_list(const uint32_t* __restrict__ scell, uint32_t n, uint32_t* __restrict__ list,
                            unsigned long long* __restrict__ count) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  const bool start = p < n && (p == 0 || scell[p] != scell[p - 1]);
  const unsigned m = __ballot_sync(kFull, start);
  if (!m) return;
  const int lane = threadIdx.x & 31;
  unsigned long long base = 0;
  if (lane == __ffs(m) - 1) base = atomicAdd(count, static_cast<unsigned long long>(__popc(m)));
  base = __shfl_sync(kFull, base, __ffs(m) - 1);
  if (start) list[base + __popc(m & ((1u << lane) - 1u))] = scell[p];
}

// Per-cell key boxes, one warp per non-empty cell.
template <int NK>
__global__ void __launch_bounds__(256) k_cell_boxes_list(const float* __restrict__ skeys,
                                                         const uint32_t* __restrict__ cfirst,
                                                         const uint32_t* __restrict__ list, uint32_t ncells,
                                                         float* __restrict__ cbox) {
  const int lane = threadIdx.x & 31;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < ncells; k += nw) {
    const uint32_t c = list[k], lo = cfirst[c], hi = cfirst[c + 1];
    float mn[NK], mx[NK];
#pragma unroll
    for (int t = 0; t < NK; ++t) {
      mn[t] = INFINITY;
      mx[t] = -INFINITY;
    }
    for (uint32_t p = lo + lane; p < hi; p += 32) {
      float kv[NK];
      load_keys<NK>(skeys + static_cast<size_t>(p) * NK, kv);
#pragma unroll
      for (int t = 0; t < NK; ++t) {
        mn[t] = fminf(mn[t], kv[t]);
        mx[t] = fmaxf(mx[t], kv[t]);
      }
    }
#pragma unroll
    for (int t = 0; t < NK; ++t)
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        mn[t] = fminf(mn[t], __shfl_xor_sync(kFull, mn[t], o));
        mx[t] = fmaxf(mx[t], __shfl_xor_sync(kFull, mx[t], o));
      }
    if (lane < NK) {
      float a = mn[0], b = mx[0];
#pragma unroll
      for (int t = 1; t < NK; ++t)
        if (lane == t) {
          a = mn[t];
          b = mx[t];
        }
      cbox[static_cast<size_t>(c) * 2 * NK + lane] = a;
      cbox[static_cast<size_t>(c) * 2 * NK + NK + lane] = b;
    }
  }
}

// Kept cell pairs, one warp per non-empty A cell: lanes take 32 stencil
// offsets at a time (s = 0 is the own cell) and a warp appends its kept pairs
// with one atomic per 32 offsets, in lane order — so each A's pairs are in
// stencil order, as the per-thread version emitted them (the stable sort by A
// then gives the same deterministic work list).
template <int NK>
__global__ void __launch_bounds__(256) k_cell_pairs_list(const uint32_t* __restrict__ cfirst,
                                                         const GridParams* __restrict__ gpp,
                                                         const uint32_t* __restrict__ list, uint32_t ncells,
                                                         const float* __restrict__ cbox,
                                                         const Thresholds* __restrict__ th, uint32_t* __restrict__ pa,
                                                         uint32_t* __restrict__ pb, uint32_t* __restrict__ pt,
                                                         uint32_t cap, unsigned long long* __restrict__ count,
                                                         bool strips, int mode) {
  __shared__ GridParams sP;
  if (threadIdx.x == 0) sP = *gpp;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const float lb2 = th->lb2 * (1.0f + 0x1.0p-20f);  // box gaps are a lower bound of every pair's key gaps
  const int fc = forward_count(sP.g);
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < ncells; k += nw) {
    const uint32_t A = list[k];
    const uint32_t na = cfirst[A + 1] - cfirst[A];
    int cc[kMaxGridKeys];
    cell_decode(sP, A, cc);
    const float* ba = cbox + static_cast<size_t>(A) * 2 * NK;
    float alo[NK], ahi[NK];
#pragma unroll
    for (int t = 0; t < NK; ++t) {
      alo[t] = ba[t];
      ahi[t] = ba[NK + t];
    }
    const uint32_t ta = (na + kT - 1) / kT;
    for (int s0 = 0; s0 <= fc; s0 += 32) {
      const int s = s0 + lane;
      bool keep = false;
      uint32_t B = A, nb = 0;
      // mode 1: own cells only; mode 2: every stencil cell but the own one
      const bool in_mode = mode == 0 || (mode == 1 ? s == 0 : s > 0);
      if (in_mode && s <= fc && (s == 0 || cell_forward(sP, cc, s, &B))) {
        nb = cfirst[B + 1] - cfirst[B];
        keep = nb != 0 && !(s == 0 && na < 2);
        if (keep && s > 0) {
          const float* bb = cbox + static_cast<size_t>(B) * 2 * NK;
          float acc = 0.f;
#pragma unroll
          for (int t = 0; t < NK; ++t) {
            const float gap = fmaxf(0.f, fmaxf(bb[t] - ahi[t], alo[t] - bb[NK + t]));
            acc = fmaf(gap, gap, acc);
          }
          keep = acc <= lb2;
        }
      }
      const unsigned m = __ballot_sync(kFull, keep);
      if (!m) continue;
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(count, static_cast<unsigned long long>(__popc(m)));
      base = __shfl_sync(kFull, base, 0);
      if (keep) {
        const unsigned long long slot = base + __popc(m & ((1u << lane) - 1u));
        if (slot < cap) {
          pa[slot] = A;
          pb[slot] = B;
          const uint32_t tb = (nb + kT - 1) / kT;
          pt[slot] = strips ? ta : (s == 0 ? ta * (ta + 1) / 2 : ta * tb);
        }
      }
    }
  }
}

// Persistent tile kernel.  Tile t of this part is global tile t*nparts+part.
__global__ void __launch_bounds__(256) k_dense_tiles(ScanArgs a, const float* __restrict__ Xs,
                                                     const uint32_t* __restrict__ cfirst, const uint32_t* __restrict__ pa,
                                                     const uint32_t* __restrict__ pb,
                                                     const uint32_t* __restrict__ prefix, uint32_t npairs,
                                                     uint32_t part, uint32_t nparts,
                                                     unsigned long long* __restrict__ cursor) {
  __shared__ __align__(16) float As[kDK][kPad];
  __shared__ __align__(16) float Bs[kDK][kPad];
  __shared__ uint32_t s_a0, s_b0, s_alen, s_blen, s_self, s_done;
  __shared__ float s_band;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const uint32_t total = prefix[npairs];
  unsigned long long visited = 0;
  for (;;) {
    if (tid == 0) {
      const unsigned long long lt = atomicAdd(cursor, 1ull);
      const unsigned long long t = lt * nparts + part;
      s_done = t >= total;
      if (!s_done) {
        // pair k with prefix[k] <= t < prefix[k+1]
        uint32_t lo = 0, hi = npairs;
        while (hi - lo > 1) {
          const uint32_t mid = (lo + hi) >> 1;
          if (prefix[mid] <= t)
            lo = mid;
          else
            hi = mid;
        }
        const uint32_t A = pa[lo], B = pb[lo];
        const uint32_t la = cfirst[A], na = cfirst[A + 1] - la;
        const uint32_t lb = cfirst[B], nb = cfirst[B + 1] - lb;
        const uint32_t lt_in = static_cast<uint32_t>(t - prefix[lo]);
        uint32_t ti, tj;
        if (A == B) {  // upper triangle of the cell's own tiles
          uint32_t j = static_cast<uint32_t>((sqrt(8.0 * lt_in + 1.0) - 1.0) * 0.5);
          while (j * (j + 1) / 2 > lt_in) --j;
          while ((j + 1) * (j + 2) / 2 <= lt_in) ++j;
          tj = j;
          ti = lt_in - j * (j + 1) / 2;
        } else {
          const uint32_t tb = (nb + kT - 1) / kT;
          ti = lt_in / tb;
          tj = lt_in % tb;
        }
        s_a0 = la + ti * kT;
        s_b0 = lb + tj * kT;
        s_alen = min(static_cast<uint32_t>(kT), na - ti * kT);
        s_blen = min(static_cast<uint32_t>(kT), nb - tj * kT);
        s_self = A == B && ti == tj;
        s_band = budget_thresholds_s32(*a.bud, best_now(a.best)).band;
      }
    }
    __syncthreads();
    if (s_done) break;
    const uint32_t a0 = s_a0, b0 = s_b0, alen = s_alen, blen = s_blen;
    const bool self = s_self;
    const float band = s_band;
    float acc[8][8];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[r][c] = 0.f;
    for (int k0 = 0; k0 < a.d; k0 += kDK) {
      __syncthreads();
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const int idx = tid + 256 * m;
        const int r = idx >> 4, c = idx & 15;
        const int t = k0 + c;
        As[c][r] = (t < a.d && r < static_cast<int>(alen)) ? Xs[static_cast<size_t>(a0 + r) * a.d + t] : 0.f;
        Bs[c][r] = (t < a.d && r < static_cast<int>(blen)) ? Xs[static_cast<size_t>(b0 + r) * a.d + t] : 0.f;
      }
      __syncthreads();
      const int kend = min(kDK, a.d - k0);
      for (int k = 0; k < kend; ++k) {
        const float4 a4 = *reinterpret_cast<const float4*>(&As[k][ty * 8]);
        const float4 a5 = *reinterpret_cast<const float4*>(&As[k][ty * 8 + 4]);
        const float4 b4 = *reinterpret_cast<const float4*>(&Bs[k][tx * 8]);
        const float4 b5 = *reinterpret_cast<const float4*>(&Bs[k][tx * 8 + 4]);
        const float av[8] = {a4.x, a4.y, a4.z, a4.w, a5.x, a5.y, a5.z, a5.w};
        const float bv[8] = {b4.x, b4.y, b4.z, b4.w, b5.x, b5.y, b5.z, b5.w};
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float g = av[r] - bv[c];
            acc[r][c] = fmaf(g, g, acc[r][c]);
          }
      }
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const uint32_t ri = ty * 8 + r;
      if (ri >= alen) continue;
      const uint32_t i = a0 + ri;
      const uint32_t oi = a.zone > 1 ? a.sidx[i] : 0u;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint32_t cj = tx * 8 + c;
        if (cj >= blen) continue;
        const uint32_t j = b0 + cj;
        if (self && j <= i) continue;
        if (a.zone > 1 && !admissible(oi, a.sidx[j], a.zone)) continue;
        ++visited;
        const float s = acc[r][c];
        if (s <= band) record(a, i, j, s, band);
      }
    }
    __syncthreads();
  }
  for (int o = 16; o; o >>= 1) visited += __shfl_xor_sync(kFull, visited, o);
  if ((tid & 31) == 0 && visited) {
    atomicAdd(a.visited, visited);
    atomicAdd(a.evals, visited);
  }
}


// ---------------------------------------------------------------------------
// Tensor-core Gram tiles (d in {32, 64}): the 128x128 pair tiles of a kept
// cell pair as D = A'.B'^T on tcgen05 (kind::tf32, both operands K-major in
// 128 B-swizzled shared memory, the 128x128 FP32 accumulator in TMEM), where
// A', B' are the rows shifted by the strip's first row (so |a'|, |b'| are at
// the scale of the cell, not of the data).  The filter value
//   s~ = |a'|^2 + |b'|^2 - 2 g~     (norms FP32, g~ from the tensor core)
// is within gram_slack * (|a'|^2 + |b'|^2) of the pair's squared distance
// (3xTF32 on the exact hi/lo split, FP32 accumulation, the shift's rounding:
// gram_slack): a pair is evaluated as the canonical FP32 distance — and
// then treated exactly like the CUDA-core tiles — only when s~ is within that
// slack of the band.  Survivors are rare, so the tensor core does the O(n^2/c)
// work and the exact path stays bit-identical.
//
// Warp roles: 0-3 loaders (one row per thread: shift, norm, swizzled store;
// A once per strip into one of two TMEM buffers, then the strip's B tiles), 4 MMA issuer (one thread), 5
// TMEM allocation, 8-11 epilogue (tcgen05.ld 32x32b: thread = A row).  A strip
// = one A tile of a kept cell pair against every B tile of the pair (self
// pairs: tiles tj >= ti); strips are taken from a global cursor.
constexpr int kGT = 128;  // A tile rows (UMMA M)
constexpr int kGN = 128;       // B tile rows (UMMA N)
constexpr int kGAB = 2;        // A buffers (hi + lo, in TMEM): the next strip's A is written while the last one's MMAs run
constexpr int kGBB = 3;        // B buffers (hi + lo, in shared memory)
constexpr int kMaxPartners = 366;  // pairs per group (k_group_flags splits longer runs of one A)
constexpr int kGThreads = 512;  // warps 0-3 loaders, 4 MMA, 5 TMEM + strip scheduler, 8-15 epilogue
constexpr int kGEpi = 8;        // epilogue warps: two per TMEM lane quarter, 64 columns each
constexpr uint32_t kGTmemCols = 512;   // [0, 256) 2 accumulators; [256 + 2D b, 256 + 2D (b+1)) A buffer b, hi | lo
constexpr uint32_t kGAcol = 2 * kGN;

// Slack of the filter value per unit of (|a'|^2 + |b'|^2):
// the 3xTF32 product (hi.hi + hi.lo + lo.hi) misses lo.lo and the TF32
// truncation of the lo parts (<= 3 * 2^-20 |a'||b'|); the FP32 accumulation of
// the 3d products is charged 4 ulps each (3d * 2^-22); s~ = na + nb - 2g~ doubles
// the Gram error, sqrt(na nb) <= (na + nb)/2, and the norms, the shift and the
// final FP32 operations add (d + 8) 2^-24; everything is doubled once more.
template <int D>
constexpr float gram_slack() {
  return static_cast<float>(2.0 * ((3.0 * 0x1.0p-20 + 3.0 * D * 0x1.0p-22) * 1.01 + (D + 8) * 0x1.0p-24));
}

struct GramMeta {
  uint32_t a0, alen, b0, blen, abuf, npar, self, last, done;
};

// One strip's work description, resolved by the scheduler warp while the
// loaders stream the previous strip: the group (cell A and its kept partner
// cells) and which 128-row A tile of it; partners as a stream prefix.
constexpr int kGS = 2;  // strip setups in flight
struct StripSetup {
  uint32_t done, A, la, nA, own, np, tot, ti;
  uint32_t ostart[kMaxPartners + 1], obase[kMaxPartners];
};

template <int D>
struct GramSmem {
  float B[kGBB][2][kGN * D];  // [hi|lo] x D/32 chunks of 128 rows x 128 B (SW128 K-major); A lives in TMEM
  float na[kGBB][kGT];  // the strip's A-row norms, copied with every B tile (released with it by the epilogue)
  float nb[kGBB][kGN];
  float cnb[kGBB][kGN];  // (1 - 2 slack) nb, +inf past the tile's length: the epilogue's fast test
  float wmaxnb[kGBB][4];
  uint32_t jpos[kGBB][kGN];  // grid position of each B row; bit 31: the row is in A's own cell
  float mu[D];               // the current strip's shift (its first row)
  StripSetup setup[kGS];     // strips prepared ahead by the scheduler warp
  GramMeta meta[kGBB];
  uint64_t afull[kGAB], afree[kGAB], bfull[kGBB], bfree[kGBB], tfull[2], tempty[2], sfull[kGS], sfree[kGS];
  uint32_t tmem;
};

#ifdef PSG_GRAM_TIMELINE
// Diagnostic build only: per-role clock64 stamps of CTA 0's first tiles.
//   0 loader: B buffer acquired     7 loader: B tile published (bfull)
//   1 MMA: B tile ready             2 MMA: accumulator free (tempty)
//   3 MMA: MMAs + commit issued     4 epilogue: accumulator full (tfull)
//   5 epilogue: tile released
constexpr int kTlTiles = 96;
__device__ long long g_tl[kTlTiles][8];
__device__ __forceinline__ void tl_mark(int ev, uint32_t tile) {
  if (blockIdx.x == 0 && tile < kTlTiles) g_tl[tile][ev] = clock64();
}
#endif

template <int D>
__global__ void __launch_bounds__(kGThreads, 1)
    k_dense_gram(ScanArgs a, const float* __restrict__ Xs, const uint32_t* __restrict__ cfirst,
                 const uint32_t* __restrict__ pa, const uint32_t* __restrict__ pb, const uint32_t* __restrict__ gstart,
                 const uint32_t* __restrict__ gprefix, const uint32_t* __restrict__ ngroups, uint32_t npairs,
                 uint32_t part, uint32_t nparts,
                 unsigned long long* __restrict__ cursor) {
  using namespace tc;
  constexpr int NC = D / 32;
  static_assert(kGAcol + kGAB * 2 * D <= kGTmemCols, "accumulators + A buffers exceed the TMEM allocation");
  extern __shared__ uint8_t graw[];
  // 1024-aligned by offsetting the shared array itself (not via an integer
  // cast), so every sm.* access stays a shared-memory (LDS/STS) access
  GramSmem<D>& sm = *reinterpret_cast<GramSmem<D>*>(graw + ((1024u - (smem_u32(graw) & 1023u)) & 1023u));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < kGAB; ++i) {
      mbar_init(&sm.afull[i], 4);
      mbar_init(&sm.afree[i], 1);  // tcgen05.commit after the strip's last MMAs
    }
    for (int i = 0; i < kGBB; ++i) {
      mbar_init(&sm.bfull[i], 4);
      mbar_init(&sm.bfree[i], kGEpi);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.tfull[i], 1);
      mbar_init(&sm.tempty[i], kGEpi);
    }
    for (int i = 0; i < kGS; ++i) {
      mbar_init(&sm.sfull[i], 1);
      mbar_init(&sm.sfree[i], 4);  // one arrive per loader warp
    }
    fence_mbar_init();
  }
  if (warp == 5) tmem_alloc(&sm.tmem, kGTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem;
  
  if (warp < 4) {
    // ---- loaders: thread = tile row.  A cursor hands out groups (a cell A
    // with every kept partner cell; the kept pairs are sorted by A, the own
    // cell first).  A strip is one 128-row tile of A against the
    // concatenation of its partners' points (the own cell from the strip's
    // first row on), cut into 128-row B tiles: small cells fill the tiles.
    const int r = tid;
    uint32_t scount = 0, bcount = 0;
    for (uint32_t k = 0;; ++k) {
      const uint32_t slot = k % kGS;
      mbar_wait(&sm.sfull[slot], (k / kGS) & 1);
      const StripSetup& S = sm.setup[slot];
      if (S.done) {  // sentinel tile: tells the MMA and the epilogue to stop
        const uint32_t bb = bcount % kGBB, bph = (bcount / kGBB) & 1;
        mbar_wait(&sm.bfree[bb], bph ^ 1);
        if (r == 0) sm.meta[bb].done = 1;
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.bfull[bb]);
        break;
      }
      const uint32_t la = S.la, nA = S.nA, np = S.np, others = S.tot;
      const bool own = S.own != 0;
      {
        const uint32_t ti = S.ti;  // this work item's strip of the group
        const uint32_t a0 = la + ti * kGT, alen = min(static_cast<uint32_t>(kGT), nA - ti * kGT);
        const uint32_t own_len = own ? la + nA - a0 : 0u;  // own cell from the strip's first row on
        const uint32_t L = own_len + others, tb = (L + kGN - 1) / kGN;
        // the strip's shift: its first row (shared; every loader has finished
        // the previous strip's tiles once it passes this barrier)
        named_bar(1, 128);
        if (r < D) sm.mu[r] = Xs[static_cast<size_t>(a0) * D + r];
        named_bar(1, 128);
        const float* mu = sm.mu;
        const uint32_t ab = scount % kGAB, aph = (scount / kGAB) & 1;
        ++scount;
        mbar_wait(&sm.afree[ab], aph ^ 1);
        tc_fence_after();  // the previous strip's MMAs have read the A tile
        const uint32_t npar = (scount - 1) & 1;
        // the A tile goes to TMEM (the MMAs take A from there): row r = TMEM
        // lane r, hi in columns kGAcol + [0, D), lo in kGAcol + D + [0, D)
        float na_r = 0.f;
        {
          const bool va = static_cast<uint32_t>(r) < alen;
          const float4* src = reinterpret_cast<const float4*>(Xs + static_cast<size_t>(a0 + (va ? r : 0)) * D);
          const uint32_t lane_base = tmem + ((32u * warp) << 16) + kGAcol + ab * 2u * D;
#pragma unroll 1
          for (int c = 0; c < D / 32; ++c) {
            uint32_t hi[32], lo[32];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              float4 v = va ? __ldg(src + c * 8 + q) : make_float4(0.f, 0.f, 0.f, 0.f);
              const int t = c * 32 + q * 4;
              if (va) {
                v.x -= mu[t];
                v.y -= mu[t + 1];
                v.z -= mu[t + 2];
                v.w -= mu[t + 3];
              }
              const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
              for (int w2 = 0; w2 < 4; ++w2) {
                na_r = fmaf(x[w2], x[w2], na_r);
                const uint32_t h = __float_as_uint(x[w2]) & ~0x1fffu;
                hi[q * 4 + w2] = h;
                lo[q * 4 + w2] = __float_as_uint(x[w2] - __uint_as_float(h));  // exact
              }
            }
            tmem_st32(lane_base + c * 32, hi);
            tmem_st32(lane_base + D + c * 32, lo);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          tc_fence_before();
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.afull[ab]);
        // B rows are loaded warp-cooperatively: kLpr lanes per row (16 B
        // each), kRpi rows per instruction, so a load touches whole 128 B
        // lines; every load of the tile is in flight before the buffer wait
        constexpr int kLpr = D / 4, kRpi = 32 / kLpr, kNi = 32 / kRpi;
        const int sub = lane % kLpr, rsel = lane / kLpr;
        const float4 mu4 = *reinterpret_cast<const float4*>(mu + 4 * sub);
        const unsigned long long mu_a = pk2(mu4.x, mu4.y), mu_b = pk2(mu4.z, mu4.w);
        // lane l resolves the grid position of tile row 32 w + l; tile tj+1's
        // positions are resolved while tile tj's loads are in flight
        auto resolve = [&](uint32_t tj, uint32_t& pos, bool& mine) -> bool {
          const uint32_t q = tj * kGN + r;
          const bool valid = q < L;
          mine = q < own_len;
          pos = 0;
          if (valid) {
            if (mine) {
              pos = a0 + q;
            } else {  // partner k with ostart[k] <= q' < ostart[k+1]
              const uint32_t qq = q - own_len;
              uint32_t lo = 0, hi = np;
              while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) >> 1;
                if (S.ostart[mid] <= qq)
                  lo = mid;
                else
                  hi = mid;
              }
              pos = S.obase[lo] + (qq - S.ostart[lo]);
            }
          }
          return valid;
        };
        // The loads run half a tile ahead of the split: the next half's rows
        // are in flight while this half is shifted, split and stored (same
        // registers as one whole tile in flight).
        constexpr int kNh = kNi / 2;
        auto load_half = [&](float4 (&v)[kNh], uint32_t ps, int h) {
#pragma unroll
          for (int i = 0; i < kNh; ++i) {
            const int src = (h * kNh + i) * kRpi + rsel;  // the warp's row this lane loads in step i
            // unconditional (pos = 0 for invalid rows, zeroed at the split): a
            // predicated select here would serialise the loads on their results
            const uint32_t p = __shfl_sync(kFull, ps, src);
            v[i] = __ldg(reinterpret_cast<const float4*>(Xs + static_cast<size_t>(p) * D) + sub);
          }
        };
        auto split_half = [&](const float4 (&v)[kNh], int h, unsigned vmask, uint32_t bb, float& wm) {
          float* hi_tile = sm.B[bb][0];
          float* lo_tile = sm.B[bb][1];
          static_assert(kNh * 2 == kLpr, "one butterfly level per halving of the row slots");
          float part[kNh];  // this lane's partial norm of each row slot
#pragma unroll
          for (int i = 0; i < kNh; ++i) {
            const int src = (h * kNh + i) * kRpi + rsel;
            const int rr = 32 * warp + src;
            // shift, norm and the lo part in packed pairs (FADD2 / FMUL2 /
            // FFMA2, exact per lane like the scalar ops; the norm's summation
            // order is any FP32 order, which gram_slack charges)
            unsigned long long xa = 0ull, xb = 0ull;
            if ((vmask >> src) & 1u) {
              xa = sub2(pk2(v[i].x, v[i].y), mu_a);
              xb = sub2(pk2(v[i].z, v[i].w), mu_b);
            }
            const float2 n2 = up2(fma2(xb, xb, mul2(xa, xa)));
            part[i] = n2.x + n2.y;
            const float2 xlo = up2(xa), xhi = up2(xb);
            const float4 x = make_float4(xlo.x, xlo.y, xhi.x, xhi.y);
            const float4 hh = make_float4(__uint_as_float(__float_as_uint(x.x) & ~0x1fffu),
                                          __uint_as_float(__float_as_uint(x.y) & ~0x1fffu),
                                          __uint_as_float(__float_as_uint(x.z) & ~0x1fffu),
                                          __uint_as_float(__float_as_uint(x.w) & ~0x1fffu));
            const float2 la = up2(sub2(xa, pk2(hh.x, hh.y))), lb = up2(sub2(xb, pk2(hh.z, hh.w)));  // exact
            const float4 l = make_float4(la.x, la.y, lb.x, lb.y);
            const int c = sub >> 3, u = sub & 7;  // 32-float chunk, 16 B unit inside the 128 B row
            const int off = c * (kGN * 32) + rr * 32 + ((u ^ (rr & 7)) << 2);
            *reinterpret_cast<float4*>(hi_tile + off) = hh;
            *reinterpret_cast<float4*>(lo_tile + off) = l;
          }
          // the kNh row norms over the row's kLpr lanes by a transposing
          // butterfly: each level sends half of the remaining slots to the
          // partner lane and adds what comes back (kNh + ... + 1 shuffles
          // instead of kNh log2(kLpr)); lane pair (slot, slot') ends with row
          // slot idx's total
          int idx = 0;
#pragma unroll
          for (int m = kLpr / 2, cnt = kNh; m >= 2; m >>= 1, cnt >>= 1) {
            const bool up = (sub & m) != 0;
#pragma unroll
            for (int k = 0; k < cnt / 2; ++k) {
              const float send = up ? part[k] : part[k + cnt / 2];
              const float keep = up ? part[k + cnt / 2] : part[k];
              part[k] = keep + __shfl_xor_sync(kFull, send, m);
            }
            idx += up ? m / 2 : 0;
          }
          const float nrm = part[0] + __shfl_xor_sync(kFull, part[0], 1);
          if ((sub & 1) == 0) {
            const int src = (h * kNh + idx) * kRpi + rsel;
            const int rr = 32 * warp + src;
            const bool ok = (vmask >> src) & 1u;
            sm.nb[bb][rr] = nrm;
            sm.cnb[bb][rr] = ok ? (1.f - 2.f * gram_slack<D>()) * nrm : INFINITY;
          }
          wm = fmaxf(wm, nrm);
        };
        uint32_t pos = 0;
        bool mine = false;
        bool valid = tb > 0 ? resolve(0, pos, mine) : false;
        float4 vc[kNh], vn[kNh];
        if (tb > 0) load_half(vc, pos, 0);
        for (uint32_t tj = 0; tj < tb; ++tj) {
          const uint32_t bb = bcount % kGBB, bph = (bcount / kGBB) & 1;
          ++bcount;
          const uint32_t blen = min(static_cast<uint32_t>(kGN), L - tj * kGN);
          const unsigned vmask = __ballot_sync(kFull, valid);
          const uint32_t jpos_c = pos | (mine ? 0x80000000u : 0u);
          load_half(vn, pos, 1);  // this tile's second half
          if (tj + 1 < tb) valid = resolve(tj + 1, pos, mine);  // the next tile's rows
          mbar_wait(&sm.bfree[bb], bph ^ 1);
#ifdef PSG_GRAM_TIMELINE
          if (warp == 0 && lane == 0) tl_mark(0, bcount - 1);
#endif
          float wm = 0.f;
          split_half(vc, 0, vmask, bb, wm);
          if (tj + 1 < tb) load_half(vc, pos, 0);  // the next tile's first half
          split_half(vn, 1, vmask, bb, wm);
          sm.na[bb][r] = na_r;
          sm.jpos[bb][r] = jpos_c;
          wm = __uint_as_float(__reduce_max_sync(kFull, __float_as_uint(wm)));  // norms >= 0
          if (lane == 0) sm.wmaxnb[bb][warp] = wm;
          // only the strip's first B tile can hold pairs with j <= i (own-cell
          // rows start at the strip's first row, so tile tj >= 1 has every B
          // row past every A row): the other tiles take the epilogue's fast path
          if (r == 0) sm.meta[bb] = GramMeta{a0, alen, 0u, blen, ab, npar, tj == 0 && own_len > 0, tj + 1 == tb, 0u};
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm.bfull[bb]);
#ifdef PSG_GRAM_TIMELINE
          if (warp == 0 && lane == 0) tl_mark(7, bcount - 1);
#endif
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.sfree[slot]);  // this warp is done with the strip's setup
    }
  } else if (warp == 5) {
    // ---- strip scheduler: takes strips from the global cursor and resolves
    // each one's group and partner table into the setup ring while the
    // loaders stream the previous strip (warp-parallel searches and loads)
    const uint32_t ng = *ngroups, total = gprefix[ng];
    for (uint32_t k = 0;; ++k) {
      const uint32_t slot = k % kGS;
      mbar_wait(&sm.sfree[slot], ((k / kGS) & 1) ^ 1);
      StripSetup& S = sm.setup[slot];
      uint32_t st = 0;
      if (lane == 0) st = static_cast<uint32_t>(atomicAdd(cursor, 1ull) * nparts + part);
      st = __shfl_sync(kFull, st, 0);
      if (st >= total) {
        if (lane == 0) {
          S.done = 1;
          mbar_arrive(&sm.sfull[slot]);
        }
        break;
      }
      // group g with gprefix[g] <= st < gprefix[g+1] (gprefix strictly increasing):
      // 32-way search, every lane probes one point of the current range
      uint32_t lo = 0, hi = ng;  // answer in [lo, hi)
      while (hi - lo > 1) {
        const uint32_t step = (hi - lo + 31) / 32;
        const uint32_t probe = min(lo + lane * step, hi - 1);
        const int c = __popc(__ballot_sync(kFull, gprefix[probe] <= st));  // >= 1: gprefix[lo] <= st
        const uint32_t nlo = min(lo + (c - 1) * step, hi - 1);  // lane c-1's probe
        if (c < 32) hi = min(lo + c * step, hi);                 // lane c's probe failed
        lo = nlo;
      }
      const uint32_t g = lo, gs = gstart[g], gend = g + 1 < ng ? gstart[g + 1] : npairs;
      const uint32_t A = pa[gs], la = cfirst[A], nA = cfirst[A + 1] - la;
      const uint32_t own = pb[gs] == A;
      const uint32_t np = min(gend - gs - own, static_cast<uint32_t>(kMaxPartners));
      uint32_t run = 0;
      for (uint32_t b0 = 0; b0 < np; b0 += 32) {
        const uint32_t t = b0 + lane;
        uint32_t lb = 0, nB = 0;
        if (t < np) {
          const uint32_t B = pb[gs + own + t];
          lb = cfirst[B];
          nB = cfirst[B + 1] - lb;
        }
        uint32_t incl = nB;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t v = __shfl_up_sync(kFull, incl, o);
          if (lane >= o) incl += v;
        }
        if (t < np) {
          S.ostart[t] = run + incl - nB;
          S.obase[t] = lb;
        }
        run += __shfl_sync(kFull, incl, 31);
      }
      if (lane == 0) {
        S.ostart[np] = run;
        S.done = 0;
        S.A = A;
        S.la = la;
        S.nA = nA;
        S.own = own;
        S.np = np;
        S.tot = run;
        S.ti = st - gprefix[g];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.sfull[slot]);
    }
  } else if (warp == 4) {
    // ---- MMA issuer: the whole warp runs the loop (uniform registers), one
    // elected lane issues the MMAs and their commits
    constexpr uint32_t idesc = idesc_tf32(kGT, kGN);
    unsigned long long ntiles = 0;
    uint32_t bcount = 0, tcount = 0, scount = 0;
    bool need_a = true;
    for (;;) {
      const uint32_t bb = bcount % kGBB, bph = (bcount / kGBB) & 1;
      mbar_wait(&sm.bfull[bb], bph);
#ifdef PSG_GRAM_TIMELINE
      if (lane == 0) tl_mark(1, tcount);
#endif
      const uint32_t acc = tcount & 1, tph = (tcount >> 1) & 1;
      mbar_wait(&sm.tempty[acc], tph ^ 1);
#ifdef PSG_GRAM_TIMELINE
      if (lane == 0) tl_mark(2, tcount);
#endif
      const GramMeta m = sm.meta[bb];  // published before the barrier arrive
      if (m.done) {
        if (lane == 0) {
          mbar_arrive(&sm.tfull[acc]);
          atomicAdd(cursor + 1, ntiles);  // ctr[2]: tiles issued (profiling)
        }
        break;
      }
      if (need_a) {  // first tile of a strip: its A buffer is filled
        const uint32_t aph = (scount / kGAB) & 1;
        mbar_wait(&sm.afull[m.abuf], aph);
        ++scount;
        need_a = false;
      }
      tc_fence_after();
      const uint32_t dcol = tmem + acc * kGN;
      if (elect_one()) {
#pragma unroll
        for (int c = 0; c < NC; ++c) {  // 3xTF32: hi.hi + hi.lo + lo.hi; A from TMEM, B from smem
          const uint32_t ah = tmem + kGAcol + m.abuf * 2u * D + c * 32, al = ah + D;
          const uint64_t bh = sw128_desc(smem_u32(sm.B[bb][0] + c * (kGN * 32)));
          const uint64_t bl = sw128_desc(smem_u32(sm.B[bb][1] + c * (kGN * 32)));
          umma_tf32_ts_3x_chunk32(dcol, ah, al, bh, bl, idesc, c != 0);
        }
        umma_commit(&sm.tfull[acc]);
#ifdef PSG_GRAM_TIMELINE
        tl_mark(3, tcount);
#endif
        if (m.last) umma_commit(&sm.afree[m.abuf]);  // the strip's A tile is free once these MMAs have read it
      }
      __syncwarp();
      ++ntiles;
      if (m.last) need_a = true;
      ++bcount;
      ++tcount;
    }
  } else if (warp >= 8) {
    // ---- epilogue: warp w owns TMEM lanes (A rows) 32 (w%4) .. +31 and the
    // 32 columns starting at 32 ((w-8)/4).  Fast path per pair: one FMA, one
    // compare folded into a predicate, one min; a chunk with a hit (or a self
    // tile, or an exclusion zone) is re-run with every check.
    const uint32_t e = warp & 3, half = (warp - 8) >> 2, r = 32 * e + lane;
    constexpr float g2 = 2.f * gram_slack<D>();
    uint32_t bcount = 0, tcount = 0;
    unsigned long long visited = 0, evals = 0;
    unsigned band_bits = 0xffffffffu;
    float band_c = 0.f;
    unsigned next_best = lane == 0 ? ld_relaxed_u32(a.best) : 0u;
    float known = INFINITY;  // a bound at least as large as the global one (read every 16th tile)
    for (;;) {
      const uint32_t bb = bcount % kGBB, acc = tcount & 1, tph = (tcount >> 1) & 1;
      mbar_wait(&sm.tfull[acc], tph);
#ifdef PSG_GRAM_TIMELINE
      if (lane == 0 && warp == 8) tl_mark(4, tcount);
#endif
      tc_fence_after();
      const GramMeta m = sm.meta[bb];
      if (m.done) break;
      // the band from the bound read during the previous tile (a stale bound
      // only widens the band), recomputed (FP64) only when the bound moved enough;
      // the next read is issued now and lands while tiles are filtered
      {
        const unsigned cur = __shfl_sync(kFull, next_best, 0);
        known = fminf(known, __uint_as_float(cur));
        // (re-read every 16th tile: the read itself waits behind every SM's atomicMin traffic)
        if (lane == 0 && (tcount & 15) == 0) next_best = ld_relaxed_u32(a.best);
        // hysteresis: a band up to ~3 % wider than the current bound's is
        // still a superset, so the FP64 recomputation runs a few hundred
        // times per solve instead of on every small move of the bound
        if (band_bits == 0xffffffffu || __uint_as_float(cur) < 0.97f * __uint_as_float(band_bits)) {
          float b = 0.f;
          if (lane == 0) b = budget_thresholds_s32(*a.bud, __uint_as_float(cur)).band;
          band_c = __shfl_sync(kFull, b, 0);
          band_bits = cur;
        }
      }
      const float band = band_c;
      const bool vr = r < m.alen;
      const uint32_t i = m.a0 + r;
      const float na = sm.na[bb][r];
      const float maxnb = fmaxf(fmaxf(sm.wmaxnb[bb][0], sm.wmaxnb[bb][1]), fmaxf(sm.wmaxnb[bb][2], sm.wmaxnb[bb][3]));
      const float R = band - (1.f - g2) * na;  // fast test: -2g + (1-g2) nb <= R
      const bool general = m.self || a.zone > 1;
      const uint32_t oi = (vr && a.zone > 1) ? a.sidx[i] : 0u;
      float vmin = INFINITY, ubs = INFINITY;
      static_assert(kGN / 64 == 2, "two 32-column loads per epilogue warp");
      uint32_t vv[2][32];  // both loads in flight before one wait
      tmem_ld32_nowait(tmem + ((32u * e) << 16) + acc * kGN + half * (kGN / 2), vv[0]);
      tmem_ld32_nowait(tmem + ((32u * e) << 16) + acc * kGN + half * (kGN / 2) + 32, vv[1]);
      tmem_wait_ld();
#pragma unroll
      for (int q = 0; q < kGN / 64; ++q) {
        const uint32_t c0 = half * (kGN / 2) + q * 32;
        const uint32_t (&v)[32] = vv[q];
        if (!vr || c0 >= m.blen) continue;
        if (!general) {
          // fast path: x = -2 g + cnb in packed pairs (FFMA2, the scalar fmaf's
          // rounding per lane) and a 3-input running min; the chunk hits iff
          // its min is <= R.  Every column is a valid pair here.
          const unsigned long long m2 = pk2(-2.f, -2.f);
          float vc = INFINITY;
#pragma unroll
          for (int jj = 0; jj < 32; jj += 4) {
            const float4 cn = *reinterpret_cast<const float4*>(&sm.cnb[bb][c0 + jj]);
            const float2 x01 = up2(fma2(pk2(__uint_as_float(v[jj]), __uint_as_float(v[jj + 1])), m2, pk2(cn.x, cn.y)));
            const float2 x23 =
                up2(fma2(pk2(__uint_as_float(v[jj + 2]), __uint_as_float(v[jj + 3])), m2, pk2(cn.z, cn.w)));
            vc = fmin3(vc, x01.x, x01.y);
            vc = fmin3(vc, x23.x, x23.y);
          }
          vmin = fminf(vmin, vc);
          visited += min(32u, m.blen - c0);
          if (!(vc <= R)) continue;
        }
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) {  // slow path: every check, the exact slack test
          const uint32_t jl = c0 + jj;
          if (jl >= m.blen) continue;
          const uint32_t jp = sm.jpos[bb][jl], j = jp & 0x7fffffffu;
          if ((jp >> 31) && j <= i) continue;  // own cell: pairs j > i only
          if (a.zone > 1 && !admissible(oi, a.sidx[j], a.zone)) continue;
          if (general) ++visited;
          const float nbj = sm.nb[bb][jl];
          const float st = fmaf(-2.f, __uint_as_float(v[jj]), na + nbj);
          const float slack = gram_slack<D>() * (na + nbj) + 1e-30f;
          if (general) ubs = fminf(ubs, st + slack);
          if (st <= band + slack) {
            ++evals;
            const float s32 = thread_sqdist(Xs + static_cast<size_t>(i) * D, Xs + static_cast<size_t>(j) * D, D);
            if (s32 <= band) record(a, i, j, s32, band);
          }
        }
      }
      // An upper bound of some valid pair's real squared distance: with
      // slack = gs (na + nb) and vmin = -2g + (1 - 2gs) nb at the minimising
      // pair, s~ + slack = vmin + 3gs nb + (1 + gs) na <= vmin + 3gs maxnb +
      // (1 + gs) na (general tiles: the slow path's own s~ + slack).  Rounded up
      // past the FP32 distance error it is a valid bound (never below the
      // canonical minimum), and the band tightens from the tensor-core values
      // alone.
      constexpr float gs = gram_slack<D>();
      float ub = vr && vmin < INFINITY ? vmin + 3.f * gs * maxnb + (1.f + gs) * na : INFINITY;
      ub = fminf(ub, ubs);
      ub = __fmul_ru(fmaxf(ub, 0.f), 1.0f + 0x1.0p-16f);
#pragma unroll
      for (int o = 16; o; o >>= 1) ub = fminf(ub, __shfl_xor_sync(kFull, ub, o));
      // only a value below the last bound read can lower the global one: the
      // other tiles' atomics (one per warp per tile, all on one word) were the
      // epilogue's main cost
      if (lane == 0 && ub < known && !a.no_ub) {
        atomicMin(a.best, __float_as_uint(ub));
        known = ub;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&sm.tempty[acc]);
#ifdef PSG_GRAM_TIMELINE
        if (warp == 8) tl_mark(5, tcount);
#endif
        mbar_arrive(&sm.bfree[bb]);
      }
      ++bcount;
      ++tcount;
    }
    for (int o = 16; o; o >>= 1) {
      visited += __shfl_xor_sync(kFull, visited, o);
      evals += __shfl_xor_sync(kFull, evals, o);
    }
    if (lane == 0) {
      if (visited) atomicAdd(a.visited, visited);
      if (evals) atomicAdd(a.evals, evals);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_free(tmem, kGTmemCols);
  }
#ifdef PSG_GRAM_TIMELINE
  if (blockIdx.x == 0 && tid == 0) {
    const long long t0 = g_tl[0][0];
    for (int t = 0; t < kTlTiles; ++t)
      printf("TL %d %lld %lld %lld %lld %lld %lld %lld\n", t, g_tl[t][0] - t0, g_tl[t][7] - t0, g_tl[t][1] - t0,
             g_tl[t][2] - t0, g_tl[t][3] - t0, g_tl[t][4] - t0, g_tl[t][5] - t0);
  }
#endif
}

template <int D>
void launch_gram(const ScanArgs& a, const DenseWork& w, const GridIndex& gi, const uint32_t* pa, const uint32_t* pb,
                 uint32_t npairs, uint32_t part, uint32_t nparts, cudaStream_t s) {
  constexpr size_t kSmem = sizeof(GramSmem<D>) + 1024;
  set_max_dynamic_smem(reinterpret_cast<const void*>(k_dense_gram<D>), kSmem);
  k_dense_gram<D><<<ctx().sm_count, kGThreads, kSmem, s>>>(a, w.Xs.p, gi.dev.cfirst, pa, pb, w.gstart.p,
                                                           w.gprefix.p, reinterpret_cast<const uint32_t*>(w.ctr.p + 3),
                                                           npairs, part, nparts, w.ctr.p + 1);
  PSG_LAUNCHED();
}

// Strips (128-row A tiles) per group.
__global__ void k_group_strips(const uint32_t* __restrict__ pa, const uint32_t* __restrict__ gstart, uint32_t ngroups,
                               const uint32_t* __restrict__ cfirst, uint32_t* __restrict__ gstrips) {
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g > ngroups) return;
  if (g == ngroups) {
    gstrips[g] = 0;
    return;
  }
  const uint32_t A = pa[gstart[g]];
  gstrips[g] = (cfirst[A + 1] - cfirst[A] + kGT - 1) / kGT;
}

// Group flags of the pairs sorted by A: flags[k] = 1 at the first pair of a group
// (flags[npairs] = 0); after an exclusive scan, the group index of its first pair.
// A group is an A cell with at most kMaxPartners of its kept pairs (the own
// pair first): an A with more (up to 3^8/2 stencil cells) spans several groups.
__global__ void k_group_flags(const uint32_t* __restrict__ pa, uint32_t npairs, uint32_t group,
                              uint32_t* __restrict__ flags, unsigned long long* __restrict__ split) {
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k <= npairs; k += gridDim.x * blockDim.x) {
    uint32_t f = 0, cont = 0;
    if (k < npairs) {
      if (k == 0 || pa[k] != pa[k - 1]) {
        f = 1;
      } else {  // rank inside A's run: first index with pa == pa[k] (binary search, pa sorted)
        const uint32_t A = pa[k];
        uint32_t lo = 0, hi = k;
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (pa[mid] < A)
            lo = mid + 1;
          else
            hi = mid;
        }
        f = (k - lo) % group == 0;
        cont = f;  // a group continuing a longer run of the same A
      }
    }
    flags[k] = f;
    if (cont) atomicAdd(split, 1ull);  // rare: only past 366 partners
  }
}

__global__ void k_group_scatter(const uint32_t* __restrict__ flags, const uint32_t* __restrict__ gidx, uint32_t npairs,
                                uint32_t* __restrict__ gstart) {
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < npairs; k += gridDim.x * blockDim.x)
    if (flags[k]) gstart[gidx[k]] = k;
}

// CUDA-core tiles per sorted pair (self pairs: the upper triangle of tiles).
__global__ void k_pair_tiles(const uint32_t* __restrict__ pa, const uint32_t* __restrict__ pb, uint32_t npairs,
                             const uint32_t* __restrict__ cfirst, uint32_t* __restrict__ pt) {
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k <= npairs; k += gridDim.x * blockDim.x) {
    if (k == npairs) {
      pt[k] = 0;
      continue;
    }
    const uint32_t A = pa[k], B = pb[k];
    const uint32_t ta = (cfirst[A + 1] - cfirst[A] + kT - 1) / kT, tb = (cfirst[B + 1] - cfirst[B] + kT - 1) / kT;
    pt[k] = A == B ? ta * (ta + 1) / 2 : ta * tb;
  }
}

bool gram_shape(int d) { return d == 32 || d == 64; }
// The Gram tiles' width for d coordinates (zero-padded), 0 when d is too wide.
int gram_width(int d) { return d <= 32 ? 32 : d <= 64 ? 64 : 0; }
}  // namespace

uint64_t grid_pair_estimate(const GridIndex& gi, uint64_t cells, cudaStream_t s) {
  DevBuf<unsigned long long> est(1, s);
  PSG_CUDA(cudaMemsetAsync(est.p, 0, 8, s));
  k_estimate<<<std::min<unsigned>(blocks((cells + kEstStride - 1) / kEstStride, 256), 4096), 256, 0, s>>>(
      gi.dev.cfirst, gi.gp.p, cells, est.p);
  PSG_LAUNCHED();
  ++g_launches;
  unsigned long long h = 0;
  PSG_CUDA(cudaMemcpyAsync(&h, est.p, 8, cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaStreamSynchronize(s));
  return h;
}

uint64_t dense_pass(const ScanArgs& a, const GridIndex& gi, uint64_t cells, int d, int nk, Thresholds* th,
                    DenseWork& w, uint32_t part, uint32_t nparts, cudaStream_t s, bool gram, unsigned lb, uint32_t ne,
                    int mode);

// The starting thresholds from the bound reached so far (between the two
// passes of a single-part Gram solve).
__global__ void k_refresh_th(const Budget* bud, const unsigned* best, Thresholds* th) {
  *th = budget_thresholds_s32(*bud, __uint_as_float(*best));
}

uint64_t dense_scan(const ScanArgs& a, const GridIndex& gi, uint64_t cells, const Rows& X, uint32_t n, int d,
                    int nk, Thresholds* th, DenseWork& w, uint32_t part, uint32_t nparts, cudaStream_t s) {
  const int sms = ctx().sm_count;
  // tensor-core Gram tiles for d <= 64 (rows zero-padded to 32 or 64);
  // CUDA-core canonical tiles otherwise
  static const bool no_gram = std::getenv("PSG_NO_GRAM") != nullptr;
  const int dg = gram_width(d);
  const bool gram = dg > 0 && !no_gram;
  const int dx = gram ? dg : d;  // Xs row width
  if (w.Xs.n != static_cast<size_t>(n) * dx) w.Xs.alloc(static_cast<size_t>(n) * dx, s);
  if (w.cbox.n < cells * 2 * nk) w.cbox.alloc(cells * 2 * nk, s);
  if (w.ctr.n < 6) w.ctr.alloc(6, s);
  if (w.clist.n < n) w.clist.alloc(n, s);
  k_gather_rows<<<sms * 16, 256, 0, s>>>(X, gi.sidx.p, n, d, dx, w.Xs.p);
  PSG_LAUNCHED();
  // the non-empty cells: boxes and pairs are per non-empty cell (a dense grid
  // over 8 keys has up to 2^27 cells, almost all empty)
  PSG_CUDA(cudaMemsetAsync(w.ctr.p + 4, 0, 8, s));
  k_cell_list<<<blocks(n, 256), 256, 0, s>>>(gi.dev.scell, n, w.clist.p, w.ctr.p + 4);
  PSG_LAUNCHED();
  unsigned long long ne64 = 0;
  PSG_CUDA(cudaMemcpyAsync(&ne64, w.ctr.p + 4, 8, cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaStreamSynchronize(s));
  const uint32_t ne = static_cast<uint32_t>(ne64);
  const unsigned lb = std::max(1u, std::min<unsigned>(blocks(static_cast<uint64_t>(ne) * 32, 256), sms * 16));
  if (nk == 4)
    k_cell_boxes_list<4><<<lb, 256, 0, s>>>(gi.skeys.p, gi.dev.cfirst, w.clist.p, ne, w.cbox.p);
  else
    k_cell_boxes_list<8><<<lb, 256, 0, s>>>(gi.skeys.p, gi.dev.cfirst, w.clist.p, ne, w.cbox.p);
  PSG_LAUNCHED();
  g_launches += 3;
  if (w.pair_cap == 0) w.pair_cap = static_cast<uint32_t>(std::min<uint64_t>(std::max<uint64_t>(cells * 14, 1024),
                                                                             1u << 26));
  // Single-part Gram solves run in two passes: the own-cell tiles first (where
  // a clustered set's closest pairs usually are), whose tile upper bounds
  // tighten the bound; then every other kept cell pair, chosen under that
  // tighter bound.  Sharded solves keep one pass: every rank must enumerate
  // the same work list, so the list is chosen under the shared bound only.
  static const bool one_pass = std::getenv("PSG_DENSE_ONE_PASS") != nullptr;
  const bool two = gram && nparts == 1 && !one_pass;
  uint64_t kept = 0;
  for (int pass = two ? 1 : 0; pass <= (two ? 2 : 0); ++pass) {
    if (pass == 2) {
      k_refresh_th<<<1, 1, 0, s>>>(a.bud, a.best, th);
      PSG_LAUNCHED();
      ++g_launches;
    }
    kept += dense_pass(a, gi, cells, dx, nk, th, w, part, nparts, s, gram, lb, ne, pass);
  }
  return kept;
}

// One pass of dense_scan over the kept cell pairs of `mode` (0 all, 1 own
// cells, 2 all but own): list, sort by A, groups / tile prefix, launch.
uint64_t dense_pass(const ScanArgs& a, const GridIndex& gi, uint64_t cells, int d, int nk, Thresholds* th,
                    DenseWork& w, uint32_t part, uint32_t nparts, cudaStream_t s, bool gram, unsigned lb, uint32_t ne,
                    int mode) {
  const int sms = ctx().sm_count;
  unsigned long long npairs = 0;
  for (;;) {
    if (w.pa.n < w.pair_cap) {
      w.pa.alloc(w.pair_cap + 1, s);
      w.pb.alloc(w.pair_cap + 1, s);
      w.ptiles.alloc(w.pair_cap + 1, s);
      w.pprefix.alloc(w.pair_cap + 1, s);
      w.stmp.alloc(scan_temp_words(w.pair_cap + 1), s);
    }
    PSG_CUDA(cudaMemsetAsync(w.ctr.p, 0, 32, s));
    PSG_CUDA(cudaMemsetAsync(w.ctr.p + 5, 0, 8, s));
    if (nk == 4)
      k_cell_pairs_list<4><<<lb, 256, 0, s>>>(gi.dev.cfirst, gi.gp.p, w.clist.p, ne, w.cbox.p, th, w.pa.p, w.pb.p,
                                             w.ptiles.p, w.pair_cap, w.ctr.p, gram, mode);
    else
      k_cell_pairs_list<8><<<lb, 256, 0, s>>>(gi.dev.cfirst, gi.gp.p, w.clist.p, ne, w.cbox.p, th, w.pa.p, w.pb.p,
                                             w.ptiles.p, w.pair_cap, w.ctr.p, gram, mode);
    PSG_LAUNCHED();
    ++g_launches;
    PSG_CUDA(cudaMemcpyAsync(&npairs, w.ctr.p, 8, cudaMemcpyDeviceToHost, s));
    PSG_CUDA(cudaStreamSynchronize(s));
    if (npairs <= w.pair_cap) break;
    w.pair_cap = static_cast<uint32_t>(npairs);
  }
  g_prof.dense_cells = cells;
  g_prof.dense_cell_pairs += npairs;
  if (npairs == 0) return 0;
  const uint32_t np32 = static_cast<uint32_t>(npairs);
  // Deterministic work order: every rank of a sharded solve enumerates the
  // same pairs / strips, so the round-robin split covers each exactly once.
  // Stable sort by A; within an A the appending thread's stencil order (the
  // own cell first).  Sorted pairs land in (spa, spb); the other two arrays
  // are scratch.
  if (w.hist.n < radix_hist_words(w.pair_cap)) w.hist.alloc(radix_hist_words(w.pair_cap), s);
  uint32_t* kk[2] = {w.pa.p, w.ptiles.p};
  uint32_t* vv[2] = {w.pb.p, w.pprefix.p};
  int bits = 1;
  while ((1ull << bits) < cells) ++bits;
  const int which = radix_sort<uint32_t>(kk, vv, npairs, 0, ((bits + 7) / 8) * 8, w.hist.p, s);
  const uint32_t* spa = kk[which];
  const uint32_t* spb = vv[which];
  uint32_t* scr0 = kk[which ^ 1];  // npairs + 1 entries each
  uint32_t* scr1 = vv[which ^ 1];
  g_launches += 1 + (bits + 7) / 8;
  if (gram) {
    // groups (a cell A and its kept partners), in pair order
    // pairs per group: kMaxPartners (the strip setup's capacity); PSG_GROUP_PAIRS
    // lowers it so tests reach the split path at small n
    uint32_t group = kMaxPartners;
    if (const char* e = std::getenv("PSG_GROUP_PAIRS"))
      group = static_cast<uint32_t>(std::clamp(std::atoi(e), 2, kMaxPartners));
    k_group_flags<<<std::min<unsigned>(blocks(npairs + 1, 256), 4096), 256, 0, s>>>(spa, np32, group, scr0,
                                                                                    w.ctr.p + 5);
    PSG_LAUNCHED();
    exclusive_scan_u32(scr0, scr1, npairs + 1, w.stmp.p, s);
    uint32_t ng = 0;
    PSG_CUDA(cudaMemcpyAsync(&ng, scr1 + npairs, 4, cudaMemcpyDeviceToHost, s));
    if (w.gstart.n < w.pair_cap + 1) w.gstart.alloc(w.pair_cap + 1, s);
    k_group_scatter<<<std::min<unsigned>(blocks(npairs, 256), 4096), 256, 0, s>>>(scr0, scr1, np32, w.gstart.p);
    PSG_LAUNCHED();
    PSG_CUDA(cudaStreamSynchronize(s));
    PSG_CUDA(cudaMemcpyAsync(w.ctr.p + 3, &ng, 4, cudaMemcpyHostToDevice, s));
    if (w.gprefix.n < ng + 1) w.gprefix.alloc(ng + 1, s);
    if (w.gstrips.n < ng + 1) w.gstrips.alloc(ng + 1, s);
    if (w.gtmp.n < scan_temp_words(ng + 1)) w.gtmp.alloc(scan_temp_words(ng + 1), s);
    k_group_strips<<<blocks(ng + 1, 256), 256, 0, s>>>(spa, w.gstart.p, ng, gi.dev.cfirst, w.gstrips.p);
    PSG_LAUNCHED();
    exclusive_scan_u32(w.gstrips.p, w.gprefix.p, ng + 1, w.gtmp.p, s);
    g_launches += 9;
    if (d == 32)
      launch_gram<32>(a, w, gi, spa, spb, np32, part, nparts, s);
    else
      launch_gram<64>(a, w, gi, spa, spb, np32, part, nparts, s);
    unsigned long long t[6] = {};
    PSG_CUDA(cudaMemcpyAsync(t, w.ctr.p, 48, cudaMemcpyDeviceToHost, s));
    PSG_CUDA(cudaStreamSynchronize(s));
    g_prof.dense_groups += ng;
    g_prof.dense_split_groups += t[5];
    g_prof.dense_tiles += t[2];
    if (std::getenv("PSG_TRACE"))
      std::fprintf(stderr, "[psg] gram: %llu kept cell pairs, %u groups (%llu split), %llu tiles\n",
                   static_cast<unsigned long long>(npairs), ng, t[5], t[2]);
  } else {
    // tiles per sorted pair -> prefix (scr0[npairs] = 0 so prefix[npairs] = total)
    k_pair_tiles<<<std::min<unsigned>(blocks(npairs + 1, 256), 4096), 256, 0, s>>>(spa, spb, np32, gi.dev.cfirst, scr0);
    PSG_LAUNCHED();
    exclusive_scan_u32(scr0, scr1, npairs + 1, w.stmp.p, s);
    g_launches += 4;
    k_dense_tiles<<<sms * 2, 256, 0, s>>>(a, w.Xs.p, gi.dev.cfirst, spa, spb, scr1, np32, part, nparts, w.ctr.p + 1);
    PSG_LAUNCHED();
  }
  ++g_launches;
  return npairs;
}

}  // namespace psg
