// psg_frnn.cu — exact fixed-radius neighbours (refscan.cpp:159-209).
//
//   K1 project    keys = <U_k, X_i>                         (psg_cpp.cu)
//      grid       cell = floor((k_t - min_t) / w), t < g = min(3, q), w >= the
//                 key window implied by R (+ rounding slack), so every pair
//                 within R sits in the same or an adjacent cell
//   K2 sort       radix sort by cell id (stable: original index inside a cell)
//   K4 scan       one thread per point, half stencil of neighbour cells; all
//                 nk keys prune (lower bound), then the FP32 distance decides
//                 outside the rounding band and the reference's FP64
//                 arithmetic decides inside it (boundary inclusive, <= R);
//                 pairs emitted as (min(i,j)<<32)|max(i,j), hashed in-kernel
//   lists         both directions radix-sorted -> CSR, ascending per row
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <memory>

#include "psg_cpp.cuh"
#include "psg_engines.cuh"
#include "psg_sort.cuh"

namespace psg {

uint64_t brute_emit_pairs(psg_pointset* ps, double radius, uint64_t zone, DevBuf<uint64_t>& keys, uint64_t* hash,
                          cudaStream_t s);

namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ uint64_t mix64(uint64_t x) {  // rng.cpp:46-51
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

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

struct Grid {
  int g = 1;
  double lo[3] = {0, 0, 0};
  double inv_w = 1.0;
  uint32_t dims[3] = {1, 1, 1};
  uint64_t cells = 1;
};

template <int NK>
__global__ void k_cell_ids(const float* __restrict__ keys, uint32_t n, Grid gr, uint32_t* __restrict__ cid,
                           uint32_t* __restrict__ idx) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t c = 0;
  for (int t = 0; t < gr.g; ++t) {
    double v = (static_cast<double>(keys[static_cast<size_t>(i) * NK + t]) - gr.lo[t]) * gr.inv_w;
    uint32_t ct = v <= 0.0 ? 0u : static_cast<uint32_t>(v);
    if (ct >= gr.dims[t]) ct = gr.dims[t] - 1;
    c = c * gr.dims[t] + ct;
  }
  cid[i] = c;
  idx[i] = i;
}

template <int NK>
__global__ void k_gather_cells(const float* __restrict__ keys, const uint32_t* __restrict__ perm, uint32_t n,
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

__global__ void k_cell_ranges(const uint32_t* __restrict__ scell, uint32_t n, uint32_t* __restrict__ cstart,
                              uint32_t* __restrict__ cend) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint32_t c = scell[p];
  if (p == 0 || scell[p - 1] != c) cstart[c] = p;
  if (p == n - 1 || scell[p + 1] != c) cend[c] = p + 1;
}

struct FrnnArgs {
  const float* X;
  const float* skeys;
  const uint32_t* sidx;
  const uint32_t* scell;
  const uint32_t* cstart;
  const uint32_t* cend;
  uint32_t n;
  int d;
  uint64_t zone;
  Grid gr;
  Thresholds th;
  float lo;
  double R;
  ExactSrc src;
  uint64_t* out;
  uint64_t cap;
  unsigned long long* acc;  // [0] count, [1] hash, [2] visited, [3] examined
};

template <int NK>
__device__ __forceinline__ void load_keys(const float* __restrict__ p, float (&k)[NK]) {
  const float4* p4 = reinterpret_cast<const float4*>(p);
#pragma unroll
  for (int v = 0; v < NK / 4; ++v) {
    const float4 t = p4[v];
    k[4 * v] = t.x;
    k[4 * v + 1] = t.y;
    k[4 * v + 2] = t.z;
    k[4 * v + 3] = t.w;
  }
}

template <int NK>
__global__ void __launch_bounds__(256) k_frnn_scan(FrnnArgs a) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t visited = 0, examined = 0, hsum = 0;
  if (p < a.n) {
    float mk[NK];
    load_keys<NK>(a.skeys + static_cast<size_t>(p) * NK, mk);
    const uint32_t mi = a.sidx[p];
    const float* xi = a.X + static_cast<size_t>(mi) * a.d;
    const uint32_t c = a.scell[p];
    uint32_t cc[3] = {0, 0, 0};
    {
      uint32_t r = c;
      for (int t = a.gr.g - 1; t >= 0; --t) {
        cc[t] = r % a.gr.dims[t];
        r /= a.gr.dims[t];
      }
    }
    int nst = 1;
    for (int t = 0; t < a.gr.g; ++t) nst *= 3;
    // offsets o in {-1,0,1}^g; visit o == 0 (j > p) and o lexicographically > 0
    for (int s = nst / 2; s < nst; ++s) {
      int rem = s;
      int off[3] = {0, 0, 0};
      for (int t = a.gr.g - 1; t >= 0; --t) {
        off[t] = rem % 3 - 1;
        rem /= 3;
      }
      uint32_t nc = 0;
      bool ok = true;
      for (int t = 0; t < a.gr.g; ++t) {
        const int64_t v = static_cast<int64_t>(cc[t]) + off[t];
        if (v < 0 || v >= a.gr.dims[t]) {
          ok = false;
          break;
        }
        nc = nc * a.gr.dims[t] + static_cast<uint32_t>(v);
      }
      if (!ok) continue;
      uint32_t jb = a.cstart[nc], je = a.cend[nc];
      if (s == nst / 2) jb = p + 1;  // own cell: later positions only
      for (uint32_t j = jb; j < je; ++j) {
        const uint32_t mj = a.sidx[j];
        const uint32_t gap = mi > mj ? mi - mj : mj - mi;
        if (gap < a.zone) continue;  // refscan.cpp:15-18
        ++visited;
        float kj[NK];
        load_keys<NK>(a.skeys + static_cast<size_t>(j) * NK, kj);
        float g = kj[0] - mk[0];
        float sl = g * g;
#pragma unroll
        for (int k = 1; k < NK; ++k) {
          g = kj[k] - mk[k];
          sl = fmaf(g, g, sl);
        }
        if (sl > a.th.lb2) continue;
        ++examined;
        const float* xj = a.X + static_cast<size_t>(mj) * a.d;
        float s32 = 0.f;
        for (int t = 0; t < a.d; ++t) {
          const float q = __ldg(xi + t) - __ldg(xj + t);
          s32 = fmaf(q, q, s32);
        }
        if (s32 > a.th.band) continue;
        if (s32 > a.lo && !(exact_distance(a.src, mi, mj) <= a.R)) continue;  // boundary inclusive
        const uint64_t key = mi < mj ? (static_cast<uint64_t>(mi) << 32) | mj : (static_cast<uint64_t>(mj) << 32) | mi;
        const unsigned long long slot = atomicAdd(a.acc, 1ull);
        if (slot < a.cap) a.out[slot] = key;
        hsum += mix64(key);
      }
    }
  }
  for (int o = 16; o; o >>= 1) {
    hsum += __shfl_xor_sync(kFull, hsum, o);
    visited += __shfl_xor_sync(kFull, visited, o);
    examined += __shfl_xor_sync(kFull, examined, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (hsum) atomicAdd(a.acc + 1, static_cast<unsigned long long>(hsum));
    if (visited) atomicAdd(a.acc + 2, static_cast<unsigned long long>(visited));
    if (examined) atomicAdd(a.acc + 3, static_cast<unsigned long long>(examined));
  }
}

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

int bits_for(uint64_t n) {
  int b = 1;
  while ((1ull << b) < n) ++b;
  return b;
}

unsigned blocks(uint64_t n, int per) { return static_cast<unsigned>((n + per - 1) / per); }

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
  g_launches += 3 * passes;
  if (which == 1) std::swap(buf, tmp);
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
  const int b = bits_for(n);
  DevBuf<uint64_t> dir(std::max<uint64_t>(2 * m, 1), s);
  if (m) {
    k_directed<<<blocks(m, 256), 256, 0, s>>>(pairs.p, m, b, dir.p);
    PSG_LAUNCHED();
    ++g_launches;
    sort_u64(dir, 2 * m, 2 * b, s);
  }
  DevBuf<uint64_t> off(n + 1, s);
  k_offsets<<<blocks(n + 1, 256), 256, 0, s>>>(dir.p, 2 * m, n, b, off.p);
  PSG_LAUNCHED();
  if (m) {
    k_low_bits<<<blocks(2 * m, 256), 256, 0, s>>>(dir.p, 2 * m, b);
    PSG_LAUNCHED();
  }
  g_launches += 2;
  out->offsets = static_cast<uint64_t*>(std::malloc((n + 1) * sizeof(uint64_t)));
  out->neighbors = static_cast<uint64_t*>(std::malloc(std::max<uint64_t>(2 * m, 1) * sizeof(uint64_t)));
  if (!out->offsets || !out->neighbors) throw std::bad_alloc();
  PSG_CUDA(cudaMemcpyAsync(out->offsets, off.p, (n + 1) * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  if (m) PSG_CUDA(cudaMemcpyAsync(out->neighbors, dir.p, 2 * m * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaStreamSynchronize(s));
  g_prof.d2h_bytes += (n + 1 + 2 * m) * sizeof(uint64_t);
}

namespace {

struct FrnnRun {
  DevBuf<uint64_t> pairs;
  uint64_t count = 0, hash = 0, visited = 0, examined = 0;
};

FrnnRun frnn_run(psg_pointset* ps, double radius, uint64_t q, double f, uint64_t seed, uint64_t zone) {
  const uint64_t n = ps->n;
  if (!(radius > 0.0) || !std::isfinite(radius)) throw invalid_argument("radius must be positive");
  check_reference_args(n, std::min(q, n), f);  // refscan.cpp:165 clamps q to n
  if (n >= 0xffffffffull) throw invalid_argument("point count exceeds 2^32-1");
  Ctx& c = ctx();
  cudaStream_t s = c.stream;
  StageTimer tm(s);
  FrnnRun run;
  const Directions dir = make_directions(seed, ps->d, static_cast<int>(std::min<uint64_t>(std::min(q, n), 64)));
  const int nk = dir.nk;
  DevBuf<float> keys(n * nk, s);
  const float norm2 = project(*ps, dir, keys.p, s);
  tm.mark("project");
  const Budget bud = make_budget(*ps, dir, norm2);
  const double Rw = radius * ps->scale;
  const double dmax = (Rw * (1.0 + 4.0 * bud.gamma64) + 2.0 * bud.Rn) * (1.0 + 1e-12);
  const Thresholds th = budget_thresholds(bud, dmax);
  const double inner = Rw * (1.0 - 4.0 * bud.gamma64) - 2.0 * bud.Rn;
  const float lo = inner > 0 ? static_cast<float>(((inner * inner) * (1.0 - bud.e) - bud.a) * (1.0 - 1e-6)) : -1.0f;

  // grid over the first g keys
  Grid gr;
  gr.g = std::min(3, dir.q);
  {
    DevBuf<unsigned> mm(6, s);
    const unsigned init[6] = {~0u, ~0u, ~0u, 0u, 0u, 0u};
    PSG_CUDA(cudaMemcpyAsync(mm.p, init, 24, cudaMemcpyHostToDevice, s));
    const unsigned gb = std::min<unsigned>(blocks(n, 256), c.sm_count * 8);
    if (nk == 4)
      k_key_range<4><<<gb, 256, 0, s>>>(keys.p, static_cast<uint32_t>(n), gr.g, mm.p, mm.p + 3);
    else
      k_key_range<8><<<gb, 256, 0, s>>>(keys.p, static_cast<uint32_t>(n), gr.g, mm.p, mm.p + 3);
    PSG_LAUNCHED();
    ++g_launches;
    unsigned h[6];
    PSG_CUDA(cudaMemcpyAsync(h, mm.p, 24, cudaMemcpyDeviceToHost, s));
    PSG_CUDA(cudaStreamSynchronize(s));
    double w = static_cast<double>(th.win) * (1.0 + 1e-6);
    double span[3];
    for (int t = 0; t < gr.g; ++t) {
      gr.lo[t] = f32_unorder(h[t]);
      span[t] = static_cast<double>(f32_unorder(h[3 + t])) - gr.lo[t];
    }
    for (;;) {
      double cells = 1.0;
      for (int t = 0; t < gr.g; ++t) cells *= std::floor(span[t] / w) + 1.0;
      if (cells <= static_cast<double>(1u << 26)) break;
      w *= 1.25;
    }
    gr.inv_w = 1.0 / w;
    gr.cells = 1;
    for (int t = 0; t < gr.g; ++t) {
      gr.dims[t] = static_cast<uint32_t>(std::floor(span[t] / w)) + 1;
      gr.cells *= gr.dims[t];
    }
  }
  DevBuf<uint32_t> kb0(n, s), kb1(n, s), vb0(n, s), vb1(n, s);
  DevBuf<uint32_t> hist(radix_hist_words(n), s);
  if (nk == 4)
    k_cell_ids<4><<<blocks(n, 256), 256, 0, s>>>(keys.p, static_cast<uint32_t>(n), gr, kb0.p, vb0.p);
  else
    k_cell_ids<8><<<blocks(n, 256), 256, 0, s>>>(keys.p, static_cast<uint32_t>(n), gr, kb0.p, vb0.p);
  PSG_LAUNCHED();
  ++g_launches;
  uint32_t* kk[2] = {kb0.p, kb1.p};
  uint32_t* vv[2] = {vb0.p, vb1.p};
  const int cbits = bits_for(gr.cells);
  const int passes = (cbits + 7) / 8;
  const int which = radix_sort<uint32_t>(kk, vv, n, 0, passes * 8, hist.p, s);
  g_launches += 3 * passes;
  tm.mark("sort");
  DevBuf<float> skeys(n * nk, s);
  DevBuf<uint32_t> sidx(n, s), cstart(gr.cells, s), cend(gr.cells, s);
  if (nk == 4)
    k_gather_cells<4><<<blocks(n, 256), 256, 0, s>>>(keys.p, vv[which], static_cast<uint32_t>(n), skeys.p, sidx.p);
  else
    k_gather_cells<8><<<blocks(n, 256), 256, 0, s>>>(keys.p, vv[which], static_cast<uint32_t>(n), skeys.p, sidx.p);
  PSG_LAUNCHED();
  PSG_CUDA(cudaMemsetAsync(cstart.p, 0, gr.cells * 4, s));
  PSG_CUDA(cudaMemsetAsync(cend.p, 0, gr.cells * 4, s));
  k_cell_ranges<<<blocks(n, 256), 256, 0, s>>>(kk[which], static_cast<uint32_t>(n), cstart.p, cend.p);
  PSG_LAUNCHED();
  g_launches += 2;
  keys.release();
  tm.mark("grid");

  FrnnArgs a{};
  a.X = ps->X;
  a.skeys = skeys.p;
  a.sidx = sidx.p;
  a.scell = kk[which];
  a.cstart = cstart.p;
  a.cend = cend.p;
  a.n = static_cast<uint32_t>(n);
  a.d = ps->d;
  a.zone = zone;
  a.gr = gr;
  a.th = th;
  a.lo = lo;
  a.R = radius;
  a.src = ps->exact();
  DevBuf<unsigned long long> acc(4, s);
  uint64_t cap = std::max<uint64_t>(1u << 20, 24 * n);
  for (;;) {
    run.pairs.alloc(cap, s);
    PSG_CUDA(cudaMemsetAsync(acc.p, 0, 32, s));
    a.out = run.pairs.p;
    a.cap = cap;
    a.acc = acc.p;
    if (nk == 4)
      k_frnn_scan<4><<<blocks(n, 256), 256, 0, s>>>(a);
    else
      k_frnn_scan<8><<<blocks(n, 256), 256, 0, s>>>(a);
    PSG_LAUNCHED();
    ++g_launches;
    unsigned long long h[4];
    PSG_CUDA(cudaMemcpyAsync(h, acc.p, 32, cudaMemcpyDeviceToHost, s));
    PSG_CUDA(cudaStreamSynchronize(s));
    if (h[0] <= cap) {
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
  return run;
}

}  // namespace

void frnn_solve(psg_pointset* ps, double radius, uint64_t q, double f, uint64_t seed, uint64_t zone,
                bool want_lists, psg_neighbor_result* out) {
  FrnnRun run = frnn_run(ps, radius, q, f, seed, zone);
  cudaStream_t s = ctx().stream;
  finish_neighbors(run.pairs, run.count, ps->n, want_lists, out, s);
  out->pair_hash = run.hash;
  const uint64_t adm = admissible_pairs(ps->n, zone);
  out->stats.pairs_examined = run.examined;
  out->stats.pairs_pruned_by_reference = run.visited - run.examined;
  out->stats.pairs_skipped_by_exit = adm - run.visited;
  out->stats.inner_loop_exits = 0;
}

void frnn_pairs(psg_pointset* ps, double radius, uint64_t q, double f, uint64_t seed, uint64_t zone,
                uint64_t* pairs, uint64_t capacity, uint64_t* count, uint64_t* hash) {
  FrnnRun run = frnn_run(ps, radius, q, f, seed, zone);
  cudaStream_t s = ctx().stream;
  *count = run.count;
  *hash = run.hash;
  if (!pairs || capacity == 0 || run.count == 0) return;
  const int b = bits_for(ps->n);
  DevBuf<uint64_t> packed(run.count, s);
  k_pack<<<blocks(run.count, 256), 256, 0, s>>>(run.pairs.p, run.count, b, packed.p);
  PSG_LAUNCHED();
  sort_u64(packed, run.count, 2 * b, s);
  k_unpack<<<blocks(run.count, 256), 256, 0, s>>>(packed.p, run.count, b);
  PSG_LAUNCHED();
  g_launches += 2;
  const uint64_t m = std::min(capacity, run.count);
  PSG_CUDA(cudaMemcpyAsync(pairs, packed.p, m * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaStreamSynchronize(s));
  g_prof.d2h_bytes += m * sizeof(uint64_t);
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
