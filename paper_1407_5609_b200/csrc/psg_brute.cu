// psg_brute.cu — all-pairs engines (refscan.cpp:134-157 and 211-227) on
// device.  A 128x128 pair tile per block, 8x8 pairs per thread, coordinates
// staged through shared memory in 16-wide slabs; each pair's FP32 squared
// distance is accumulated sequentially in coordinate order (identical bits
// to a thread-serial fmaf loop).  Blocks enumerate the upper triangle of
// tiles linearly.  Used as the product's brute engines and as the device
// oracle for the configs the CPU oracle cannot finish.
#include <algorithm>
#include <cmath>
#include <memory>

#include "psg_cpp.cuh"
#include "psg_engines.cuh"

namespace psg {
namespace {

constexpr int kT = 128;   // tile edge
constexpr int kDK = 16;   // coordinate slab
constexpr int kPad = 132;

enum Mode : int { kMin = 0, kCollect = 1, kFrnn = 2 };

struct BruteArgs {
  Rows X;  // the working rows (materialised or virtual windows)
  uint32_t n;
  int d;
  uint64_t zone;
  unsigned* best;       // kMin
  float thr;            // kCollect: s32 <= thr ; kFrnn: s32 <= hi
  float lo;             // kFrnn: s32 <= lo is certainly inside R
  double R;             // kFrnn: reference radius (source units)
  ExactSrc src;         // kFrnn boundary decisions
  uint32_t* ci;         // kCollect
  uint32_t* cj;
  float* cs;
  unsigned long long* count;  // kCollect / kFrnn
  uint32_t cap;
  uint64_t* keys;       // kFrnn output (i<<32|j)
  uint64_t kcap;
  unsigned long long* hash;
};

__device__ __forceinline__ void tri_index(uint64_t t, uint32_t* bi, uint32_t* bj) {
  uint64_t j = static_cast<uint64_t>((sqrt(8.0 * static_cast<double>(t) + 1.0) - 1.0) * 0.5);
  while (j * (j + 1) / 2 > t) --j;
  while ((j + 1) * (j + 2) / 2 <= t) ++j;
  *bj = static_cast<uint32_t>(j);
  *bi = static_cast<uint32_t>(t - j * (j + 1) / 2);
}

// One launch covers tiles [base, base + gridDim.x) of the upper triangle
// (n = 2^24 has 8.6e9 tiles: launched in chunks below 2^31 blocks).
template <int MODE>
__global__ void __launch_bounds__(256) k_brute(BruteArgs a, uint64_t base) {
  __shared__ __align__(16) float As[kDK][kPad];
  __shared__ __align__(16) float Bs[kDK][kPad];
  uint32_t bi, bj;
  tri_index(base + blockIdx.x, &bi, &bj);
  const uint32_t i0 = bi * kT, j0 = bj * kT;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
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
      const uint32_t gi = i0 + r, gj = j0 + r;
      As[c][r] = (t < a.d && gi < a.n) ? row_at(a.X, gi, t) : 0.f;
      Bs[c][r] = (t < a.d && gj < a.n) ? row_at(a.X, gj, t) : 0.f;
    }
    __syncthreads();
    const int kend = min(kDK, a.d - k0);
    for (int k = 0; k < kend; ++k) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[k][ty * 8]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[k][ty * 8 + 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[k][tx * 8]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[k][tx * 8 + 4]);
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float g = av[r] - bv[c];
          acc[r][c] = fmaf(g, g, acc[r][c]);
        }
    }
  }
  float local_min = INFINITY;
  uint64_t cnt = 0, hsum = 0;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const uint32_t i = i0 + ty * 8 + r;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const uint32_t j = j0 + tx * 8 + c;
      if (i >= j || j >= a.n || (j - i) < a.zone) continue;
      const float s = acc[r][c];
      if (MODE == kMin) {
        local_min = fminf(local_min, s);
      } else if (MODE == kCollect) {
        if (s <= a.thr) {
          const unsigned long long slot = atomicAdd(a.count, 1ull);
          if (slot < a.cap) {
            a.ci[slot] = i;
            a.cj[slot] = j;
            a.cs[slot] = s;
          }
        }
      } else {
        if (s > a.thr) continue;
        if (s > a.lo && !(exact_distance(a.src, i, j) <= a.R)) continue;
        const uint64_t key = (static_cast<uint64_t>(i) << 32) | j;
        const unsigned long long slot = atomicAdd(a.count, 1ull);
        if (slot < a.kcap) a.keys[slot] = key;
        ++cnt;
        // SplitMix64 finaliser (rng.cpp:46-51)
        uint64_t x = key + 0x9e3779b97f4a7c15ull;
        x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
        x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
        hsum += x ^ (x >> 31);
      }
    }
  }
  if (MODE == kMin) {
    local_min = __uint_as_float(__reduce_min_sync(0xffffffffu, __float_as_uint(local_min)));
    if ((tid & 31) == 0 && local_min < INFINITY) atomicMin(a.best, __float_as_uint(local_min));
  }
  if (MODE == kFrnn) {
    for (int o = 16; o; o >>= 1) hsum += __shfl_xor_sync(0xffffffffu, hsum, o);
    (void)cnt;
    if ((tid & 31) == 0 && hsum) atomicAdd(a.hash, static_cast<unsigned long long>(hsum));
  }
}

__global__ void k_recheck_plain(ExactSrc src, const uint32_t* __restrict__ ci, const uint32_t* __restrict__ cj,
                                uint32_t count, double* __restrict__ d64, unsigned long long* __restrict__ best64) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= count) return;
  const double dd = exact_distance(src, ci[c], cj[c]);
  d64[c] = dd;
  atomicMin(best64, static_cast<unsigned long long>(__double_as_longlong(dd)));
}

__global__ void k_pick_plain(const uint32_t* __restrict__ ci, const uint32_t* __restrict__ cj, uint32_t count,
                             const double* __restrict__ d64, const unsigned long long* __restrict__ best64,
                             unsigned long long* __restrict__ lex) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= count) return;
  if (static_cast<unsigned long long>(__double_as_longlong(d64[c])) != *best64) return;
  atomicMin(lex, (static_cast<unsigned long long>(ci[c]) << 32) | cj[c]);
}

uint64_t tiles_for(uint64_t n) {
  const uint64_t t = (n + kT - 1) / kT;
  return t * (t + 1) / 2;
}

template <int MODE>
void launch(const BruteArgs& a, cudaStream_t s) {
  const uint64_t tiles = tiles_for(a.n);
  constexpr uint64_t kMaxBlocks = 1ull << 30;
  for (uint64_t base = 0; base < tiles; base += kMaxBlocks) {
    k_brute<MODE><<<static_cast<unsigned>(std::min(kMaxBlocks, tiles - base)), 256, 0, s>>>(a, base);
    PSG_LAUNCHED();
    ++g_launches;
  }
}

Budget band_budget(const psg_pointset& ps) {
  const double u = 0x1.0p-24;
  Budget b;
  b.e = (ps.d + 4) * u * 1.01;
  b.a = (2.0 * ps.d + 2.0) * 0x1.0p-149;
  b.Rn = ps.Rn;
  b.gamma64 = (ps.d + 2) * 0x1.0p-53 * 1.01;
  return b;
}

}  // namespace

// upper < 0: two passes (the FP32 minimum, then its band); upper >= 0: one
// pass over the band of FP64 distance `upper` (source units).
psg_pair_result brute_solve(psg_pointset* ps, uint64_t zone, double upper) {
  const uint64_t n = ps->n;
  if (n < 2) throw invalid_argument("closest_pair needs at least 2 points");  // refscan.cpp:136
  if (n >= 0xffffffffull) throw invalid_argument("point count exceeds 2^32-1");
  const uint64_t adm = admissible_pairs(n, zone);
  if (adm == 0) throw invalid_argument("no admissible pair");  // refscan.cpp:154
  Ctx& c = ctx();
  cudaStream_t s = c.stream;
  StageTimer tm(s);
  BruteArgs a{};
  a.X = ps->rows();
  a.n = static_cast<uint32_t>(n);
  a.d = ps->d;
  a.zone = zone;
  const Budget bud = band_budget(*ps);
  if (upper < 0.0) {
    DevBuf<unsigned> best(1, s);
    const float inf = INFINITY;
    PSG_CUDA(cudaMemcpyAsync(best.p, &inf, 4, cudaMemcpyHostToDevice, s));
    a.best = best.p;
    launch<kMin>(a, s);
    unsigned hb;
    PSG_CUDA(cudaMemcpyAsync(&hb, best.p, 4, cudaMemcpyDeviceToHost, s));
    PSG_CUDA(cudaStreamSynchronize(s));
    tm.mark("brute_min");
    float bs;
    std::memcpy(&bs, &hb, 4);
    a.thr = budget_thresholds_s32(bud, bs).band;
  } else {
    // every pair at FP64 distance <= upper (the FRNN boundary band, psg_frnn.cu)
    const double Uw = upper * ps->scale;
    a.thr = budget_thresholds(bud, (Uw * (1.0 + 4.0 * bud.gamma64) + 2.0 * bud.Rn) * (1.0 + 1e-12)).band;
  }
  uint32_t cap = 1u << 16;
  DevBuf<unsigned long long> cnt(1, s);
  DevBuf<uint32_t> ci, cj;
  DevBuf<float> cs;
  uint64_t hc = 0;
  for (;;) {
    ci.alloc(cap, s);
    cj.alloc(cap, s);
    cs.alloc(cap, s);
    PSG_CUDA(cudaMemsetAsync(cnt.p, 0, 8, s));
    a.ci = ci.p;
    a.cj = cj.p;
    a.cs = cs.p;
    a.count = cnt.p;
    a.cap = cap;
    launch<kCollect>(a, s);
    PSG_CUDA(cudaMemcpyAsync(&hc, cnt.p, 8, cudaMemcpyDeviceToHost, s));
    PSG_CUDA(cudaStreamSynchronize(s));
    if (hc <= cap) break;
    if (hc > (1ull << 30)) throw std::runtime_error("brute force: candidate band too large");
    cap = static_cast<uint32_t>(hc);
  }
  tm.mark("brute_band");
  const uint32_t nc = static_cast<uint32_t>(hc);
  DevBuf<double> d64(std::max<uint32_t>(nc, 1), s);
  DevBuf<unsigned long long> red(2, s);
  const unsigned long long init[2] = {~0ull, ~0ull};
  PSG_CUDA(cudaMemcpyAsync(red.p, init, 16, cudaMemcpyHostToDevice, s));
  const ExactSrc src = ps->exact();
  if (nc) {
    k_recheck_plain<<<(nc + 255) / 256, 256, 0, s>>>(src, ci.p, cj.p, nc, d64.p, red.p);
    PSG_LAUNCHED();
    k_pick_plain<<<(nc + 255) / 256, 256, 0, s>>>(ci.p, cj.p, nc, d64.p, red.p, red.p + 1);
    PSG_LAUNCHED();
    g_launches += 2;
  }
  unsigned long long hr[2];
  PSG_CUDA(cudaMemcpyAsync(hr, red.p, 16, cudaMemcpyDeviceToHost, s));
  tm.mark("recheck");
  PSG_CUDA(cudaStreamSynchronize(s));
  prof_stages(tm);
  psg_pair_result r{};
  r.index_i = hr[1] >> 32;
  r.index_j = hr[1] & 0xffffffffull;
  std::memcpy(&r.distance, &hr[0], 8);
  if (hr[1] == ~0ull || (upper >= 0.0 && !(r.distance <= upper))) {
    r.index_i = r.index_j = UINT64_MAX;
    r.distance = INFINITY;
  }
  r.stats.pairs_examined = adm;  // every admissible pair (refscan.cpp:145)
  g_prof.candidates = nc;
  g_prof.lb_survivors = adm;
  return r;
}

// Shared with the FRNN engine: all-pairs emission of (i<<32|j) inside R.
uint64_t brute_emit_pairs(psg_pointset* ps, double radius, uint64_t zone, DevBuf<uint64_t>& keys, uint64_t* hash,
                          cudaStream_t s);

uint64_t brute_emit_pairs(psg_pointset* ps, double radius, uint64_t zone, DevBuf<uint64_t>& keys, uint64_t* hash,
                          cudaStream_t s) {
  const uint64_t n = ps->n;
  BruteArgs a{};
  a.X = ps->rows();
  a.n = static_cast<uint32_t>(n);
  a.d = ps->d;
  a.zone = zone;
  a.R = radius;
  a.src = ps->exact();
  // FP32 band around R (working units): see frnn thresholds in psg_frnn.cu
  const Budget bud = band_budget(*ps);
  const double Rw = radius * ps->scale;
  const double dmax = (Rw * (1.0 + 4.0 * bud.gamma64) + 2.0 * bud.Rn) * (1.0 + 1e-12);
  a.thr = budget_thresholds(bud, dmax).band;
  const double inner = Rw * (1.0 - 4.0 * bud.gamma64) - 2.0 * bud.Rn;
  a.lo = inner > 0 ? static_cast<float>(((inner * inner) * (1.0 - bud.e) - bud.a) * (1.0 - 1e-6)) : -1.0f;
  DevBuf<unsigned long long> acc(2, s);
  uint64_t cap = std::max<uint64_t>(keys.n, 1u << 16);
  for (;;) {
    if (keys.n < cap) keys.alloc(cap, s);
    PSG_CUDA(cudaMemsetAsync(acc.p, 0, 16, s));
    a.keys = keys.p;
    a.kcap = cap;
    a.count = acc.p;
    a.hash = acc.p + 1;
    launch<kFrnn>(a, s);
    unsigned long long h[2];
    PSG_CUDA(cudaMemcpyAsync(h, acc.p, 16, cudaMemcpyDeviceToHost, s));
    PSG_CUDA(cudaStreamSynchronize(s));
    if (h[0] <= cap) {
      *hash = h[1];
      return h[0];
    }
    cap = h[0];
  }
}

}  // namespace psg
