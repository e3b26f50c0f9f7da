// psg_grid.cu — build the cell grid (psg_grid.cuh): cell ids from the device
// GridParams, stable radix sort by cell, cfirst by a warp-parallel search of
// the sorted cell ids, key gather.  Everything is enqueued; nothing waits on
// the host.
#include <algorithm>
#include <cstdio>
#include <cmath>
#include <vector>

#include "psg_grid.cuh"
#include "psg_points.cuh"
#include "psg_scan.cuh"
#include "psg_sort.cuh"

namespace psg {
namespace {

constexpr unsigned kGridFull = 0xffffffffu;

unsigned blocks(uint64_t n, int per) { return static_cast<unsigned>((n + per - 1) / per); }

__global__ void k_sample_keys(const float* __restrict__ keys, uint32_t n, int nk, int g, uint32_t m,
                              float* __restrict__ out) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  // multiplicative hash, not a stride: a strided sample aliases with periodic
  // structure in the index order (e.g. cluster = index mod 1024)
  const uint32_t i = static_cast<uint32_t>((static_cast<uint64_t>(k) * 2654435761ull + 12345) % n);
  for (int t = 0; t < g; ++t) out[static_cast<size_t>(t) * m + k] = keys[static_cast<size_t>(i) * nk + t];
}

template <int NK>
__global__ void k_cell_ids(const float* __restrict__ keys, uint32_t n, const GridParams* __restrict__ gpp,
                           uint32_t* __restrict__ cid, uint32_t* __restrict__ idx) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const GridParams P = *gpp;
  cid[i] = cell_of<NK>(keys + static_cast<size_t>(i) * NK, P);
  idx[i] = i;
}

// cfirst[c] = first sorted position whose cell id is >= c, for c = 0..cells.
// A warp owns kCfirstWarpCells consecutive cells: one binary search for the
// first, then groups of 32 cells (one per lane) walk forward through windows
// of 32 sorted cell ids, each lane ranking its cell in the window with a
// 5-step shuffle search.  Work ~ (cells + n) / 32 per warp-step, writes
// coalesced; no per-cell counters, atomics or scans.
constexpr uint32_t kCfirstWarpCells = 1024;

__global__ void __launch_bounds__(256) k_cfirst(const uint32_t* __restrict__ scell, uint32_t n,
                                                const GridParams* __restrict__ gp, uint32_t* __restrict__ cfirst) {
  const int lane = threadIdx.x & 31;
  const uint32_t last = static_cast<uint32_t>(gp->cells);  // entries 0..last
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t c0 = warp * kCfirstWarpCells; c0 <= last; c0 += nwarps * kCfirstWarpCells) {
    // pos = lower_bound(scell, c0): lanes split the range 32 ways per step
    uint32_t lo = 0, hi = n;  // answer in [lo, hi]
    while (hi - lo > 32) {
      const uint32_t step = (hi - lo + 31) / 32;
      const uint32_t probe = min(lo + lane * step, hi - 1);
      const unsigned below = __ballot_sync(kGridFull, scell[probe] < c0);  // prefix of lanes (sorted)
      const int k = __popc(below);  // probes 0..k-1 are < c0
      const uint32_t nlo = k == 0 ? lo : min(lo + (k - 1) * step + 1, hi);
      const uint32_t nhi = k == 32 ? hi : min(lo + k * step, hi);
      lo = nlo;
      hi = nhi;
    }
    {
      const uint32_t probe = lo + lane;
      const bool lt = probe < hi && scell[probe] < c0;
      lo += __popc(__ballot_sync(kGridFull, lt));
    }
    uint32_t pos = lo;
    const uint32_t cend = min(c0 + kCfirstWarpCells - 1, last);
    for (uint32_t cb = c0; cb <= cend; cb += 32) {
      const uint32_t c = cb + lane;
      uint32_t res = 0;
      bool done = c > cend;  // lanes past the range have nothing to write
      uint32_t base = pos;
      for (int win = 0; !__all_sync(kGridFull, done); ++win) {
        if (win == 4) {  // dense cells: stop walking, each open lane binary-searches [base, n)
          if (!done) {
            uint32_t lo2 = base, hi2 = n;
            while (lo2 < hi2) {
              const uint32_t mid = (lo2 + hi2) >> 1;
              if (scell[mid] < c)
                lo2 = mid + 1;
              else
                hi2 = mid;
            }
            res = lo2;
            done = true;
          }
          break;
        }
        const uint32_t v = base + lane < n ? scell[base + lane] : 0xffffffffu;
        // r = #(window values < c); the window is ascending across lanes
        // (every shuffle is executed by all lanes: no shuffle under a branch)
        const uint32_t v31 = __shfl_sync(kGridFull, v, 31);
        int r = 0;
#pragma unroll
        for (int st = 16; st; st >>= 1) {
          const uint32_t probe = __shfl_sync(kGridFull, v, r + st - 1);
          if (probe < c) r += st;
        }
        if (r == 31 && v31 < c) r = 32;
        if (!done && (r < 32 || base + 32 >= n)) {
          res = min(base + r, n);
          done = true;
        }
        base += 32;
      }
      if (c <= cend) cfirst[c] = res;
      pos = __shfl_sync(kGridFull, res, min(cend - cb, 31u));  // lb of the group's last cell
    }
  }
}

#ifdef PSG_DEBUG_SYNC
__global__ void k_verify_cfirst(const uint32_t* __restrict__ scell, uint32_t n, const GridParams* __restrict__ gp,
                                const uint32_t* __restrict__ cfirst) {
  const uint32_t last = static_cast<uint32_t>(gp->cells);
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c <= last; c += gridDim.x * blockDim.x) {
    const uint32_t p = cfirst[c];
    const bool ok = p <= n && (p == n || scell[p] >= c) && (p == 0 || scell[p - 1] < c);
    if (!ok) {
      uint32_t a = 0, b = n;  // true lower bound
      while (a < b) {
        const uint32_t m = (a + b) / 2;
        if (scell[m] < c) a = m + 1; else b = m;
      }
      printf("cfirst[%u] = %u want %u (c%%32 %u c%%1024 %u) prev %u next %u\n", c, p, a, c % 32, c % 1024,
             c > 0 ? cfirst[c - 1] : 0u, c < last ? cfirst[c + 1] : 0u);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (uint32_t i = 1; i < n; i += 997)
      if (scell[i] < scell[i - 1]) { printf("scell not sorted at %u\n", i); __trap(); }
}
#endif

// ---- counting build ----------------------------------------------------------
// Cell id and the point's arrival rank in its cell (atomic, so arbitrary
// order; k_cell_fix makes the final order deterministic).
template <int NK>
__global__ void k_cell_count(const float* __restrict__ keys, uint32_t n, const GridParams* __restrict__ gpp,
                             uint32_t* __restrict__ cnt, uint32_t* __restrict__ cid, uint32_t* __restrict__ rnk,
                             uint32_t* __restrict__ bctr) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) {
    bctr[0] = 0;  // big cells
    bctr[1] = 0;  // their cursor
  }
  if (i >= n) return;
  const GridParams P = *gpp;
  const uint32_t c = cell_of<NK>(keys + static_cast<size_t>(i) * NK, P);
  cid[i] = c;
  atomicAdd(cnt + c, 1u);  // result unused: a reduction (k_cell_place ranks)
}

// Arrival-order placement; the counters go back to zero for the next build
// (every non-zero counter has at least one point here).
// The arrival rank comes from counting the cell back down (atomicSub), which
// also leaves every counter at zero for the next build; the counting pass
// then needs no returned value (fire-and-forget reductions).
__global__ void k_cell_place(const uint32_t* __restrict__ cid, uint32_t n, const uint32_t* __restrict__ cfirst,
                             uint32_t* __restrict__ cnt, uint32_t* __restrict__ tmp) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t c = cid[i];
  tmp[cfirst[c] + atomicSub(cnt + c, 1u) - 1u] = i;
}

constexpr uint32_t kFixSmall = 64;  // cells up to this size are ranked per position
constexpr uint32_t kBootCand = 64;  // BootLB candidates per point (the old bootstrap's cap was 256)

// Final position of the point at arrival position p: its cell's start plus
// the number of points of the cell with a smaller original index; gathers its
// keys there.  Cells above kFixSmall points are listed for k_cell_fix_big.
template <int NK>
__global__ void k_cell_fix(const float* __restrict__ keys, const uint32_t* __restrict__ tmp,
                           const uint32_t* __restrict__ cid, uint32_t n, const uint32_t* __restrict__ cfirst,
                           float* __restrict__ skeys, uint32_t* __restrict__ sidx, uint32_t* __restrict__ scell,
                           uint32_t* __restrict__ big, uint32_t* __restrict__ bctr) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint32_t i = tmp[p], c = cid[i], b = cfirst[c], e = cfirst[c + 1];
  if (e - b > kFixSmall) {
    if (p == b) big[atomicAdd(bctr, 1u)] = c;
    return;
  }
  uint32_t r = 0;
  for (uint32_t k = b; k < e; ++k) r += tmp[k] < i;
  const uint32_t q = b + r;
  sidx[q] = i;
  scell[q] = c;
  const float4* src = reinterpret_cast<const float4*>(keys + static_cast<size_t>(i) * NK);
  float4* dst = reinterpret_cast<float4*>(skeys + static_cast<size_t>(q) * NK);
#pragma unroll
  for (int v = 0; v < NK / 4; ++v) dst[v] = src[v];
}

// (lb, i, j) order: the least lower bound, ties to the least (i, j).
__device__ __forceinline__ bool boot_less(float lb, uint32_t i, uint32_t j, float ob, uint32_t oi, uint32_t oj) {
  return lb < ob || (lb == ob && (i < oi || (i == oi && j < oj)));
}

// BootLB on the finished grid: the point at sorted position p against the
// other points of its cell and of the next cell of its row (all of them up to
// kBootCand, else a uniform stride from p), keys read by position (a warp's
// candidates are its neighbours: coalesced, mostly L1 hits); the least (lb,
// i, j) per warp of positions.
template <int NK>
__global__ void k_boot_lb(const float* __restrict__ skeys, const uint32_t* __restrict__ sidx,
                          const uint32_t* __restrict__ scell, const uint32_t* __restrict__ cfirst, uint32_t n,
                          const GridParams* __restrict__ gpp, BootLB B) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  float best = INFINITY;
  uint32_t bi = 0xffffffffu, bj = 0xffffffffu;
  if (p < n) {
    const uint32_t c = scell[p];
    const uint32_t D = gpp->dims[gpp->g - 1];
    const FastDiv fD = gpp->fD;
    const uint32_t cs = cfirst[c];
    const uint32_t c1 = c + 1;
    const uint32_t ne = fD.div(c1) * D != c1 ? cfirst[c + 2] : cfirst[c1];  // the row's next cell when there is one
    const uint32_t L = ne - cs;
    float mk[NK];
    load_keys<NK>(skeys + static_cast<size_t>(p) * NK, mk);
    const uint32_t mi = sidx[p];
    auto consider = [&](uint32_t m) {
      if (m == p) return;
      float km[NK];
      load_keys<NK>(skeys + static_cast<size_t>(m) * NK, km);
      const float lb = lb2_full<NK>(mk, km);
      if (lb > best) return;
      const uint32_t mj = sidx[m];
      if (B.zone > 1 && !admissible(mi, mj, B.zone)) return;
      const uint32_t a = min(mi, mj), z = max(mi, mj);
      if (boot_less(lb, a, z, best, bi, bj)) {
        best = lb;
        bi = a;
        bj = z;
      }
    };
    if (L <= kBootCand + 1) {
      for (uint32_t m = cs; m < ne; ++m) consider(m);
    } else {
      const uint32_t stride = L / kBootCand, o = p - cs;
      for (uint32_t t = 1; t <= kBootCand; ++t) consider(cs + (o + t * stride) % L);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float ob = __shfl_xor_sync(kGridFull, best, o);
    const uint32_t oi = __shfl_xor_sync(kGridFull, bi, o), oj = __shfl_xor_sync(kGridFull, bj, o);
    if (boot_less(ob, oi, oj, best, bi, bj)) {
      best = ob;
      bi = oi;
      bj = oj;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    B.wlb[w] = best;
    B.wpair[w] = make_uint2(bi, bj);
  }
}

// Big cells (duplicates, tight clusters): a block per cell.  The cell's
// indices are bitonic-sorted in shared memory in runs of kFixRun; a cell of
// one run is written out directly, a longer one ranks every point as the sum
// of its lower bounds in the sorted runs (indices are distinct).
constexpr int kFixBigThreads = 512, kFixRun = 8192;
template <int NK>
__device__ __forceinline__ void fix_write(const float* __restrict__ keys, uint32_t q, uint32_t i, uint32_t c,
                                          float* __restrict__ skeys, uint32_t* __restrict__ sidx,
                                          uint32_t* __restrict__ scell) {
  sidx[q] = i;
  scell[q] = c;
  const float4* src = reinterpret_cast<const float4*>(keys + static_cast<size_t>(i) * NK);
  float4* dst = reinterpret_cast<float4*>(skeys + static_cast<size_t>(q) * NK);
#pragma unroll
  for (int v = 0; v < NK / 4; ++v) dst[v] = src[v];
}

template <int NK>
__global__ void __launch_bounds__(kFixBigThreads) k_cell_fix_big(
    const float* __restrict__ keys, const uint32_t* __restrict__ tmp, uint32_t* __restrict__ runs,
    const uint32_t* __restrict__ cfirst, float* __restrict__ skeys, uint32_t* __restrict__ sidx,
    uint32_t* __restrict__ scell, const uint32_t* __restrict__ big, uint32_t* __restrict__ bctr) {
  __shared__ uint32_t sk[kFixRun];
  __shared__ uint32_t s_c;
  const uint32_t tid = threadIdx.x;
  for (;;) {
    __syncthreads();
    if (tid == 0) {
      const uint32_t k = atomicAdd(bctr + 1, 1u);
      s_c = k < bctr[0] ? big[k] : 0xffffffffu;
    }
    __syncthreads();
    const uint32_t c = s_c;
    if (c == 0xffffffffu) return;
    const uint32_t b = cfirst[c], e = cfirst[c + 1], L = e - b;
    for (uint32_t r0 = b; r0 < e; r0 += kFixRun) {
      const uint32_t len = min(static_cast<uint32_t>(kFixRun), e - r0);
      uint32_t P = 1;
      while (P < len) P <<= 1;
      __syncthreads();
      for (uint32_t k = tid; k < P; k += kFixBigThreads) sk[k] = k < len ? tmp[r0 + k] : 0xffffffffu;
      __syncthreads();
      for (uint32_t k2 = 2; k2 <= P; k2 <<= 1)
        for (uint32_t j = k2 >> 1; j > 0; j >>= 1) {
          for (uint32_t t = tid; t < P / 2; t += kFixBigThreads) {
            const uint32_t i = ((t & ~(j - 1)) << 1) | (t & (j - 1)), l = i + j;
            const uint32_t x = sk[i], y = sk[l];
            if ((x > y) == ((i & k2) == 0)) {
              sk[i] = y;
              sk[l] = x;
            }
          }
          __syncthreads();
        }
      if (L <= kFixRun) {
        for (uint32_t k = tid; k < len; k += kFixBigThreads) fix_write<NK>(keys, b + k, sk[k], c, skeys, sidx, scell);
      } else {
        for (uint32_t k = tid; k < len; k += kFixBigThreads) runs[r0 + k] = sk[k];
      }
    }
    if (L > kFixRun) {
      __threadfence_block();
      __syncthreads();
      for (uint32_t p = b + tid; p < e; p += kFixBigThreads) {
        const uint32_t i = tmp[p];
        uint32_t rank = 0;
        for (uint32_t r0 = b; r0 < e; r0 += kFixRun) {  // lower bound of i in each sorted run
          uint32_t lo = 0, hi = min(static_cast<uint32_t>(kFixRun), e - r0);
          while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (runs[r0 + mid] < i)
              lo = mid + 1;
            else
              hi = mid;
          }
          rank += lo;
        }
        fix_write<NK>(keys, b + rank, i, c, skeys, sidx, scell);
      }
    }
  }
}

template <int NK>
__global__ void k_gather_sorted(const float* __restrict__ keys, const uint32_t* __restrict__ perm, uint32_t n,
                                float* __restrict__ skeys, uint32_t* __restrict__ sidx) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint32_t i = perm[p];
  const float4* src = reinterpret_cast<const float4*>(keys + static_cast<size_t>(i) * NK);
  float4* dst = reinterpret_cast<float4*>(skeys + static_cast<size_t>(p) * NK);
#pragma unroll
  for (int v = 0; v < NK / 4; ++v) dst[v] = src[v];
  sidx[p] = i;
}

}  // namespace

void GridIndex::ensure(uint32_t n_, int nk_, cudaStream_t s) {
  if (n == n_ && nk == nk_ && skeys.p) return;
  n = n_;
  nk = nk_;
  skeys.alloc(static_cast<size_t>(n) * nk, s);
  sidx.alloc(n, s);
  cid0.alloc(n, s);
  cid1.alloc(n, s);
  idx0.alloc(n, s);
  idx1.alloc(n, s);
  hist.alloc(radix_hist_words(n), s);
  cfirst.alloc(kMaxCells + 1, s);
  if (!cnt.p) {
    cnt.alloc(kMaxCells + 1, s);
    PSG_CUDA(cudaMemsetAsync(cnt.p, 0, (kMaxCells + 1) * sizeof(uint32_t), s));  // invariant: all zero
    ctmp.alloc(scan_temp_words(kMaxCells + 1), s);
    bctr.alloc(2, s);
  }
  big.alloc(n / kFixSmall + 1, s);
  sample.alloc(kMaxKeys * kGridSample, s);
  gp.alloc(1, s);
  wlb.alloc((n + 255) / 256 * 8, s);
  wpair.alloc((n + 255) / 256 * 8, s);
}

uint32_t grid_sample(const float* keys, uint32_t n, int nk, int g, GridIndex& gi, cudaStream_t s) {
  const uint32_t m = std::min<uint32_t>(n, kGridSample);
  k_sample_keys<<<blocks(m, 256), 256, 0, s>>>(keys, n, nk, g, m, gi.sample.p);
  PSG_LAUNCHED();
  ++g_launches;
  return m;
}

// box = [mean - 3 sd, mean + 3 sd] clipped to the sample range (a tuning
// input only: clamping keeps any box exact).
void grid_box_host(const float* sample, uint32_t m, int g, double lo[3], double span[3]) {
  for (int t = 0; t < 3; ++t) {
    lo[t] = 0;
    span[t] = 0;
  }
  for (int t = 0; t < g; ++t) {
    const float* v = sample + static_cast<size_t>(t) * m;
    double s1 = 0, s2 = 0, mn = v[0], mx = v[0];
    for (uint32_t i = 0; i < m; ++i) {
      s1 += v[i];
      s2 += static_cast<double>(v[i]) * v[i];
      mn = std::min<double>(mn, v[i]);
      mx = std::max<double>(mx, v[i]);
    }
    const double mean = s1 / m, sd = std::sqrt(std::max(s2 / m - mean * mean, 0.0));
    const double a = std::max(mn, mean - 3 * sd), b = std::min(mx, mean + 3 * sd);
    lo[t] = a;
    span[t] = std::max(b - a, 1e-30);
  }
}

void build_grid(const float* keys, uint32_t n, int nk, GridIndex& gi, int sort_bits, cudaStream_t s, bool counting,
                uint64_t dense_cells, bool counted, const BootLB* boot) {
  if (counting) {
    const unsigned nb = blocks(n, 256);
    if (!counted) {  // else the projection counted (CellCount; bctr reset by k_presample)
      if (nk == 4)
        k_cell_count<4><<<nb, 256, 0, s>>>(keys, n, gi.gp.p, gi.cnt.p, gi.cid0.p, gi.idx0.p, gi.bctr.p);
      else
        k_cell_count<8><<<nb, 256, 0, s>>>(keys, n, gi.gp.p, gi.cnt.p, gi.cid0.p, gi.idx0.p, gi.bctr.p);
      PSG_LAUNCHED();
    }
    const BootLB B = boot ? *boot : BootLB{};
    // cfirst = exclusive scan of the counts over cells 0..cells (count read on device)
    exclusive_scan_u32_dev(gi.cnt.p, gi.cfirst.p, kMaxCells + 1, &gi.gp.p->cells, gi.ctmp.p, s);
    k_cell_place<<<nb, 256, 0, s>>>(gi.cid0.p, n, gi.cfirst.p, gi.cnt.p, gi.idx1.p);
    PSG_LAUNCHED();
    if (nk == 4) {
      k_cell_fix<4><<<nb, 256, 0, s>>>(keys, gi.idx1.p, gi.cid0.p, n, gi.cfirst.p, gi.skeys.p, gi.sidx.p, gi.cid1.p,
                                       gi.big.p, gi.bctr.p);
      PSG_LAUNCHED();
      k_cell_fix_big<4><<<148, kFixBigThreads, 0, s>>>(keys, gi.idx1.p, gi.idx0.p, gi.cfirst.p, gi.skeys.p,
                                                       gi.sidx.p, gi.cid1.p, gi.big.p, gi.bctr.p);
      PSG_LAUNCHED();
      if (B.keys) k_boot_lb<4><<<nb, 256, 0, s>>>(gi.skeys.p, gi.sidx.p, gi.cid1.p, gi.cfirst.p, n, gi.gp.p, B);
    } else {
      k_cell_fix<8><<<nb, 256, 0, s>>>(keys, gi.idx1.p, gi.cid0.p, n, gi.cfirst.p, gi.skeys.p, gi.sidx.p, gi.cid1.p,
                                       gi.big.p, gi.bctr.p);
      PSG_LAUNCHED();
      k_cell_fix_big<8><<<148, kFixBigThreads, 0, s>>>(keys, gi.idx1.p, gi.idx0.p, gi.cfirst.p, gi.skeys.p,
                                                       gi.sidx.p, gi.cid1.p, gi.big.p, gi.bctr.p);
      PSG_LAUNCHED();
      if (B.keys) k_boot_lb<8><<<nb, 256, 0, s>>>(gi.skeys.p, gi.sidx.p, gi.cid1.p, gi.cfirst.p, n, gi.gp.p, B);
    }
    if (B.keys) {
      PSG_LAUNCHED();
      ++g_launches;
    }
#ifdef PSG_DEBUG_SYNC
    k_verify_cfirst<<<1024, 256, 0, s>>>(gi.cid1.p, n, gi.gp.p, gi.cfirst.p);
    PSG_LAUNCHED();
#endif
    g_launches += 8;
    gi.dev.skeys = gi.skeys.p;
    gi.dev.sidx = gi.sidx.p;
    gi.dev.scell = gi.cid1.p;
    gi.dev.cfirst = gi.cfirst.p;
    gi.dev.gp = gi.gp.p;
    gi.dev.n = n;
    return;
  }
  if (nk == 4)
    k_cell_ids<4><<<blocks(n, 256), 256, 0, s>>>(keys, n, gi.gp.p, gi.cid0.p, gi.idx0.p);
  else
    k_cell_ids<8><<<blocks(n, 256), 256, 0, s>>>(keys, n, gi.gp.p, gi.cid0.p, gi.idx0.p);
  PSG_LAUNCHED();
  uint32_t* kk[2] = {gi.cid0.p, gi.cid1.p};
  uint32_t* vv[2] = {gi.idx0.p, gi.idx1.p};
  uint32_t* cfirst = gi.cfirst.p;
  if (dense_cells > kMaxCells) {
    if (gi.dcfirst.n < dense_cells + 1) gi.dcfirst.alloc(dense_cells + 1, s);
    cfirst = gi.dcfirst.p;
    while ((1ull << sort_bits) < dense_cells) ++sort_bits;
  }
  const int passes = (sort_bits + 7) / 8;
  const int which = radix_sort<uint32_t>(kk, vv, n, 0, passes * 8, gi.hist.p, s);
  // every warp resident at once: the binary searches overlap
  k_cfirst<<<2 * 148 * 8, 256, 0, s>>>(kk[which], n, gi.gp.p, cfirst);
  PSG_LAUNCHED();
#ifdef PSG_DEBUG_SYNC
  k_verify_cfirst<<<1024, 256, 0, s>>>(kk[which], n, gi.gp.p, cfirst);
  PSG_LAUNCHED();
#endif
  if (nk == 4)
    k_gather_sorted<4><<<blocks(n, 256), 256, 0, s>>>(keys, vv[which], n, gi.skeys.p, gi.sidx.p);
  else
    k_gather_sorted<8><<<blocks(n, 256), 256, 0, s>>>(keys, vv[which], n, gi.skeys.p, gi.sidx.p);
  PSG_LAUNCHED();
  g_launches += 3 + 3 * passes;
  gi.dev.skeys = gi.skeys.p;
  gi.dev.sidx = gi.sidx.p;
  gi.dev.scell = kk[which];
  gi.dev.cfirst = cfirst;
  gi.dev.gp = gi.gp.p;
  gi.dev.n = n;
}

}  // namespace psg
