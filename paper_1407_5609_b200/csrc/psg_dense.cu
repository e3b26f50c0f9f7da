// psg_dense.cu — dense cell-pair engine (psg_dense.cuh).
//
// When the grid's cells hold many points (clustered data: the closest pair
// sits at the scale of a cluster, so a key window of the bound spans whole
// clusters), per-point candidate lists degenerate: every point would walk
// ~10^4-10^5 candidates.  Here the unit of work is a pair of cells instead:
//   1. per-cell boxes over all nk keys (block per cell)
//   2. keep a forward-stencil cell pair (A, B) only if the box gap lower
//      bound is within the threshold — pairs of points of different clusters
//      are dropped a whole cell pair at a time
//   3. kept cell pairs are cut into 128x128 tiles; a persistent kernel takes
//      tiles from an atomic cursor and evaluates every pair as a canonical
//      FP32 distance (16-wide coordinate slabs in shared memory, 8x8 pairs per
//      thread — the all-pairs kernel's arithmetic and order) from rows
//      gathered into grid order, recording the band into the candidate list.
#include <algorithm>
#include <cmath>

#include "psg_dense.cuh"
#include "psg_points.cuh"
#include "psg_sort.cuh"

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

__global__ void k_estimate(const uint32_t* __restrict__ cfirst, const GridParams* __restrict__ gpp, uint64_t cells,
                           unsigned long long* __restrict__ est) {
  const GridParams P = *gpp;
  unsigned long long total = 0;
  for (uint64_t A = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; A < cells;
       A += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
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
  if ((threadIdx.x & 31) == 0 && total) atomicAdd(est, total);
}

__global__ void k_gather_rows(const float* __restrict__ X, const uint32_t* __restrict__ sidx, uint32_t n, int d,
                              float* __restrict__ Xs) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t p = warp; p < n; p += nwarps) {
    const float* src = X + static_cast<size_t>(sidx[p]) * d;
    float* dst = Xs + static_cast<size_t>(p) * d;
    for (int t = lane; t < d; t += 32) dst[t] = __ldg(src + t);
  }
}

template <int NK>
__global__ void __launch_bounds__(256) k_cell_boxes(const float* __restrict__ skeys, const uint32_t* __restrict__ cfirst,
                                                    uint64_t cells, float* __restrict__ cbox) {
  __shared__ float red[2][NK][8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (uint64_t c = blockIdx.x; c < cells; c += gridDim.x) {
    const uint32_t lo = cfirst[c], hi = cfirst[c + 1];
    if (lo == hi) continue;  // uniform per block
    float mn[NK], mx[NK];
#pragma unroll
    for (int k = 0; k < NK; ++k) {
      mn[k] = INFINITY;
      mx[k] = -INFINITY;
    }
    for (uint32_t p = lo + tid; p < hi; p += blockDim.x) {
      float kv[NK];
      load_keys<NK>(skeys + static_cast<size_t>(p) * NK, kv);
#pragma unroll
      for (int k = 0; k < NK; ++k) {
        mn[k] = fminf(mn[k], kv[k]);
        mx[k] = fmaxf(mx[k], kv[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < NK; ++k)
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        mn[k] = fminf(mn[k], __shfl_xor_sync(kFull, mn[k], o));
        mx[k] = fmaxf(mx[k], __shfl_xor_sync(kFull, mx[k], o));
      }
    __syncthreads();
    if (lane == 0)
#pragma unroll
      for (int k = 0; k < NK; ++k) {
        red[0][k][warp] = mn[k];
        red[1][k][warp] = mx[k];
      }
    __syncthreads();
    if (tid < NK) {
      float a = INFINITY, b = -INFINITY;
      for (int w = 0; w < 8; ++w) {
        a = fminf(a, red[0][tid][w]);
        b = fmaxf(b, red[1][tid][w]);
      }
      cbox[c * 2 * NK + tid] = a;
      cbox[c * 2 * NK + NK + tid] = b;
    }
  }
}

template <int NK>
__global__ void k_cell_pairs(const uint32_t* __restrict__ cfirst, const GridParams* __restrict__ gpp, uint64_t cells,
                             const float* __restrict__ cbox, const Thresholds* __restrict__ th,
                             uint32_t* __restrict__ pa, uint32_t* __restrict__ pb, uint32_t* __restrict__ pt,
                             uint32_t cap, unsigned long long* __restrict__ count) {
  const GridParams P = *gpp;
  const float lb2 = th->lb2 * (1.0f + 0x1.0p-20f);  // box gaps are a lower bound of every pair's key gaps
  for (uint64_t A = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; A < cells;
       A += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t na = cfirst[A + 1] - cfirst[A];
    if (na == 0) continue;
    int cc[kMaxGridKeys];
    cell_decode(P, static_cast<uint32_t>(A), cc);
    const float* ba = cbox + A * 2 * NK;
    for (int s = 0; s <= forward_count(P.g); ++s) {
      uint32_t B = static_cast<uint32_t>(A);
      if (s > 0 && !cell_forward(P, cc, s, &B)) continue;
      const uint32_t nb = cfirst[B + 1] - cfirst[B];
      if (nb == 0 || (s == 0 && na < 2)) continue;
      if (s > 0) {
        const float* bb = cbox + static_cast<size_t>(B) * 2 * NK;
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < NK; ++k) {
          const float gap = fmaxf(0.f, fmaxf(bb[k] - ba[NK + k], ba[k] - bb[NK + k]));
          acc = fmaf(gap, gap, acc);
        }
        if (acc > lb2) continue;
      }
      const unsigned long long slot = atomicAdd(count, 1ull);
      if (slot < cap) {
        pa[slot] = static_cast<uint32_t>(A);
        pb[slot] = B;
        const uint32_t ta = (na + kT - 1) / kT, tb = (nb + kT - 1) / kT;
        pt[slot] = s == 0 ? ta * (ta + 1) / 2 : ta * tb;
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

}  // namespace

uint64_t grid_pair_estimate(const GridIndex& gi, uint64_t cells, cudaStream_t s) {
  DevBuf<unsigned long long> est(1, s);
  PSG_CUDA(cudaMemsetAsync(est.p, 0, 8, s));
  k_estimate<<<std::min<unsigned>(blocks(cells, 256), 4096), 256, 0, s>>>(gi.cfirst.p, gi.gp.p, cells, est.p);
  PSG_LAUNCHED();
  ++g_launches;
  unsigned long long h = 0;
  PSG_CUDA(cudaMemcpyAsync(&h, est.p, 8, cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaStreamSynchronize(s));
  return h;
}

uint64_t dense_scan(const ScanArgs& a, const GridIndex& gi, uint64_t cells, const float* X, uint32_t n, int d,
                    int nk, const Thresholds* th, DenseWork& w, uint32_t part, uint32_t nparts, cudaStream_t s) {
  const int sms = ctx().sm_count;
  if (w.Xs.n != static_cast<size_t>(n) * d) w.Xs.alloc(static_cast<size_t>(n) * d, s);
  if (w.cbox.n < cells * 2 * nk) w.cbox.alloc(cells * 2 * nk, s);
  if (w.ctr.n < 3) w.ctr.alloc(3, s);
  k_gather_rows<<<sms * 16, 256, 0, s>>>(X, gi.sidx.p, n, d, w.Xs.p);
  PSG_LAUNCHED();
  if (nk == 4)
    k_cell_boxes<4><<<static_cast<unsigned>(std::min<uint64_t>(cells, 65535)), 256, 0, s>>>(gi.skeys.p, gi.cfirst.p,
                                                                                            cells, w.cbox.p);
  else
    k_cell_boxes<8><<<static_cast<unsigned>(std::min<uint64_t>(cells, 65535)), 256, 0, s>>>(gi.skeys.p, gi.cfirst.p,
                                                                                            cells, w.cbox.p);
  PSG_LAUNCHED();
  g_launches += 2;
  if (w.pair_cap == 0) w.pair_cap = static_cast<uint32_t>(std::min<uint64_t>(std::max<uint64_t>(cells * 14, 1024),
                                                                             1u << 26));
  unsigned long long npairs = 0;
  for (;;) {
    if (w.pa.n < w.pair_cap) {
      w.pa.alloc(w.pair_cap, s);
      w.pb.alloc(w.pair_cap, s);
      w.ptiles.alloc(w.pair_cap + 1, s);
      w.pprefix.alloc(w.pair_cap + 1, s);
      w.stmp.alloc(scan_temp_words(w.pair_cap + 1), s);
    }
    PSG_CUDA(cudaMemsetAsync(w.ctr.p, 0, 24, s));
    if (nk == 4)
      k_cell_pairs<4><<<std::min<unsigned>(blocks(cells, 256), 4096), 256, 0, s>>>(
          gi.cfirst.p, gi.gp.p, cells, w.cbox.p, th, w.pa.p, w.pb.p, w.ptiles.p, w.pair_cap, w.ctr.p);
    else
      k_cell_pairs<8><<<std::min<unsigned>(blocks(cells, 256), 4096), 256, 0, s>>>(
          gi.cfirst.p, gi.gp.p, cells, w.cbox.p, th, w.pa.p, w.pb.p, w.ptiles.p, w.pair_cap, w.ctr.p);
    PSG_LAUNCHED();
    ++g_launches;
    PSG_CUDA(cudaMemcpyAsync(&npairs, w.ctr.p, 8, cudaMemcpyDeviceToHost, s));
    PSG_CUDA(cudaStreamSynchronize(s));
    if (npairs <= w.pair_cap) break;
    w.pair_cap = static_cast<uint32_t>(npairs);
  }
  if (npairs == 0) return 0;
  // tile prefix over the kept pairs (ptiles[npairs] = 0 so prefix[npairs] = total)
  PSG_CUDA(cudaMemsetAsync(w.ptiles.p + npairs, 0, 4, s));
  exclusive_scan_u32(w.ptiles.p, w.pprefix.p, npairs + 1, w.stmp.p, s);
  g_launches += 3;
  k_dense_tiles<<<sms * 2, 256, 0, s>>>(a, w.Xs.p, gi.cfirst.p, w.pa.p, w.pb.p, w.pprefix.p,
                                        static_cast<uint32_t>(npairs), part, nparts, w.ctr.p + 1);
  PSG_LAUNCHED();
  ++g_launches;
  return npairs;
}

}  // namespace psg
