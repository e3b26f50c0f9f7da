// psg_grid.cu — build the cell grid (psg_grid.cuh): cell ids from the device
// GridParams, per-cell counts -> cfirst (exclusive scan), stable radix sort by
// cell, key gather.  Everything is enqueued; nothing waits on the host.
#include <algorithm>
#include <cmath>
#include <vector>

#include "psg_grid.cuh"
#include "psg_points.cuh"
#include "psg_sort.cuh"

namespace psg {
namespace {

unsigned blocks(uint64_t n, int per) { return static_cast<unsigned>((n + per - 1) / per); }
constexpr uint32_t kSample = 4096;

__global__ void k_sample_keys(const float* __restrict__ keys, uint32_t n, int nk, int g, uint32_t m,
                              float* __restrict__ out) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  // multiplicative hash, not a stride: a strided sample aliases with periodic
  // structure in the index order (e.g. cluster = index mod 1024)
  const uint32_t i = static_cast<uint32_t>((static_cast<uint64_t>(k) * 2654435761ull + 12345) % n);
  for (int t = 0; t < g; ++t) out[static_cast<size_t>(t) * m + k] = keys[static_cast<size_t>(i) * nk + t];
}

__global__ void k_zero_counts(uint32_t* __restrict__ counts, const GridParams* __restrict__ gp) {
  const uint64_t count = gp->cells + 1;
  for (uint64_t c = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; c < count;
       c += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    counts[c] = 0;
}

template <int NK>
__global__ void k_cell_ids(const float* __restrict__ keys, uint32_t n, const GridParams* __restrict__ gpp,
                           uint32_t* __restrict__ cid, uint32_t* __restrict__ idx, uint32_t* __restrict__ counts) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const GridParams P = *gpp;
  uint32_t c = 0;
#pragma unroll
  for (int t = 0; t < (NK < kMaxGridKeys ? NK : kMaxGridKeys); ++t) {
    if (t >= P.g) break;
    const uint32_t dim = P.dims[t];
    const double v = (static_cast<double>(keys[static_cast<size_t>(i) * NK + t]) - P.lo[t]) * P.inv_w;
    const uint32_t ct = v <= 0.0 ? 0u : (v >= static_cast<double>(dim - 1) ? dim - 1 : static_cast<uint32_t>(v));
    c = c * dim + ct;
  }
  cid[i] = c;
  idx[i] = i;
  atomicAdd(counts + c, 1u);
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
  counts.alloc(kMaxCells + 1, s);
  cfirst.alloc(kMaxCells + 1, s);
  stmp.alloc(scan_temp_words(kMaxCells + 1), s);
  sample.alloc(kMaxKeys * kSample, s);
  gp.alloc(1, s);
}

uint32_t grid_sample(const float* keys, uint32_t n, int nk, int g, GridIndex& gi, cudaStream_t s) {
  const uint32_t m = std::min<uint32_t>(n, kSample);
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

void build_grid(const float* keys, uint32_t n, int nk, GridIndex& gi, int sort_bits, cudaStream_t s) {
  k_zero_counts<<<1024, 256, 0, s>>>(gi.counts.p, gi.gp.p);
  PSG_LAUNCHED();
  if (nk == 4)
    k_cell_ids<4><<<blocks(n, 256), 256, 0, s>>>(keys, n, gi.gp.p, gi.cid0.p, gi.idx0.p, gi.counts.p);
  else
    k_cell_ids<8><<<blocks(n, 256), 256, 0, s>>>(keys, n, gi.gp.p, gi.cid0.p, gi.idx0.p, gi.counts.p);
  PSG_LAUNCHED();
  // cfirst = exclusive prefix sum of the per-cell counts (cfirst[cells] = n)
  exclusive_scan_u32_dev(gi.counts.p, gi.cfirst.p, kMaxCells + 1, &gi.gp.p->cells, gi.stmp.p, s);
  uint32_t* kk[2] = {gi.cid0.p, gi.cid1.p};
  uint32_t* vv[2] = {gi.idx0.p, gi.idx1.p};
  const int passes = (sort_bits + 7) / 8;
  const int which = radix_sort<uint32_t>(kk, vv, n, 0, passes * 8, gi.hist.p, s);
  if (nk == 4)
    k_gather_sorted<4><<<blocks(n, 256), 256, 0, s>>>(keys, vv[which], n, gi.skeys.p, gi.sidx.p);
  else
    k_gather_sorted<8><<<blocks(n, 256), 256, 0, s>>>(keys, vv[which], n, gi.skeys.p, gi.sidx.p);
  PSG_LAUNCHED();
  g_launches += 6 + 3 * passes;
  gi.dev.skeys = gi.skeys.p;
  gi.dev.sidx = gi.sidx.p;
  gi.dev.scell = kk[which];
  gi.dev.cfirst = gi.cfirst.p;
  gi.dev.gp = gi.gp.p;
  gi.dev.n = n;
}

}  // namespace psg
