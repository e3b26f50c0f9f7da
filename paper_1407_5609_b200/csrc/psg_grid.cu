// psg_grid.cu — build the cell grid (psg_grid.cuh): sample box, cell ids,
// stable radix sort by cell, key gather, dense cell ranges.
#include <algorithm>
#include <cmath>
#include <vector>

#include "psg_grid.cuh"
#include "psg_points.cuh"
#include "psg_sort.cuh"

namespace psg {
namespace {

unsigned blocks(uint64_t n, int per) { return static_cast<unsigned>((n + per - 1) / per); }

__global__ void k_sample_keys(const float* __restrict__ keys, uint32_t n, int nk, int g, uint32_t m,
                              float* __restrict__ out) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const uint32_t i = static_cast<uint32_t>((static_cast<uint64_t>(k) * n) / m);
  for (int t = 0; t < g; ++t) out[static_cast<size_t>(t) * m + k] = keys[static_cast<size_t>(i) * nk + t];
}

template <int NK>
__global__ void k_cell_ids(const float* __restrict__ keys, uint32_t n, GridDev G, uint32_t* __restrict__ cid,
                           uint32_t* __restrict__ idx) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t c = 0;
  for (int t = 0; t < G.g; ++t) {
    const double v = (static_cast<double>(keys[static_cast<size_t>(i) * NK + t]) - G.lo[t]) * G.inv_w;
    uint32_t ct = v <= 0.0 ? 0u : (v >= static_cast<double>(G.dims[t] - 1) ? G.dims[t] - 1 : static_cast<uint32_t>(v));
    c = c * G.dims[t] + ct;
  }
  cid[i] = c;
  idx[i] = i;
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

// cfirst[c] = lower_bound(scell, c) for c in [0, cells]: position p (0..n)
// writes p into every cell id in (scell[p-1], scell[p]] — each entry exactly
// once, total work cells + n.
__global__ void k_cell_first(const uint32_t* __restrict__ scell, uint32_t n, uint64_t cells,
                             uint32_t* __restrict__ cfirst) {
  const uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (p > n) return;
  const int64_t prev = p == 0 ? -1 : static_cast<int64_t>(scell[p - 1]);
  const int64_t cur = p == n ? static_cast<int64_t>(cells) : static_cast<int64_t>(scell[p]);
  for (int64_t c = prev + 1; c <= cur; ++c) cfirst[c] = static_cast<uint32_t>(p);
}

}  // namespace

void grid_sample_box(const float* keys, uint32_t n, int nk, int g, double lo[3], double span[3], cudaStream_t s) {
  const uint32_t m = std::min<uint32_t>(n, 4096);
  DevBuf<float> smp(static_cast<size_t>(m) * g, s);
  k_sample_keys<<<blocks(m, 256), 256, 0, s>>>(keys, n, nk, g, m, smp.p);
  PSG_LAUNCHED();
  ++g_launches;
  std::vector<float> h(static_cast<size_t>(m) * g);
  PSG_CUDA(cudaMemcpyAsync(h.data(), smp.p, h.size() * sizeof(float), cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaStreamSynchronize(s));
  trace("grid: sample d2h");
  // box = [mean - 3 sd, mean + 3 sd] clipped to the sample range (one pass)
  for (int t = 0; t < g; ++t) {
    const float* v = h.data() + static_cast<size_t>(t) * m;
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
  trace("grid: quantiles");
  for (int t = g; t < 3; ++t) {
    lo[t] = 0;
    span[t] = 0;
  }
}

double grid_occupancy_width(uint32_t n, int g, const double span[3], double occupancy) {
  double vol = 1.0;
  for (int t = 0; t < g; ++t) vol *= span[t];
  return std::pow(vol * occupancy / std::max<double>(n, 1), 1.0 / g);
}

void build_grid(const float* keys, uint32_t n, int nk, int g, double w, const double lo[3], const double span[3],
                GridIndex& gi, cudaStream_t s) {
  gi.nk = nk;
  GridDev G;
  G.n = n;
  G.g = g;
  for (;;) {
    double cells = 1.0;
    for (int t = 0; t < g; ++t) cells *= std::floor(span[t] / w) + 1.0;
    if (cells <= static_cast<double>(1u << 24)) break;
    w *= 1.25;
  }
  gi.w = w;
  G.inv_w = 1.0 / w;
  gi.cells = 1;
  for (int t = 0; t < g; ++t) {
    G.lo[t] = lo[t];
    G.dims[t] = static_cast<uint32_t>(std::floor(span[t] / w)) + 1;
    gi.cells *= G.dims[t];
  }
  trace("grid: params");
  DevBuf<uint32_t> k0(n, s), k1(n, s), v0(n, s), v1(n, s), hist(radix_hist_words(n), s);
  trace("grid: alloc");
  if (nk == 4)
    k_cell_ids<4><<<blocks(n, 256), 256, 0, s>>>(keys, n, G, k0.p, v0.p);
  else
    k_cell_ids<8><<<blocks(n, 256), 256, 0, s>>>(keys, n, G, k0.p, v0.p);
  PSG_LAUNCHED();
  ++g_launches;
  uint32_t* kk[2] = {k0.p, k1.p};
  uint32_t* vv[2] = {v0.p, v1.p};
  int bits = 1;
  while ((1ull << bits) < gi.cells) ++bits;
  const int passes = (bits + 7) / 8;
  const int which = radix_sort<uint32_t>(kk, vv, n, 0, passes * 8, hist.p, s);
  g_launches += 3 * passes;
  trace("grid: sort launched");
  gi.skeys.alloc(static_cast<size_t>(n) * nk, s);
  gi.sidx.alloc(n, s);
  if (nk == 4)
    k_gather_sorted<4><<<blocks(n, 256), 256, 0, s>>>(keys, vv[which], n, gi.skeys.p, gi.sidx.p);
  else
    k_gather_sorted<8><<<blocks(n, 256), 256, 0, s>>>(keys, vv[which], n, gi.skeys.p, gi.sidx.p);
  PSG_LAUNCHED();
  gi.scell = std::move(which == 0 ? k0 : k1);
  gi.cfirst.alloc(gi.cells + 1, s);
  k_cell_first<<<blocks(static_cast<uint64_t>(n) + 1, 256), 256, 0, s>>>(gi.scell.p, n, gi.cells, gi.cfirst.p);
  PSG_LAUNCHED();
  g_launches += 2;
  trace("grid: ranges launched");
  G.skeys = gi.skeys.p;
  G.sidx = gi.sidx.p;
  G.scell = gi.scell.p;
  G.cfirst = gi.cfirst.p;
  gi.dev = G;
}

}  // namespace psg
