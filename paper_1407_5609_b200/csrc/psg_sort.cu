// psg_sort.cu — LSD radix sort, 8 bits per pass, three kernels per pass:
//   rs_hist    per-tile digit histogram (shared-memory atomics) -> digit-major table
//   rs_scan    exclusive scan of the digit-major table (one block)
//   rs_scatter stable scatter: warp-contiguous sub-tiles, __match_any_sync
//              ranks within 32-item rounds, per-warp digit counters, a
//              cross-warp exclusive scan, then one coalesced-per-digit store.
// Work per element per pass: read key(+val) twice, write once -> HBM-bound.
#include "psg_internal.cuh"
#include "psg_sort.cuh"

namespace psg {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 16;
constexpr int kTile = kThreads * kItems;  // 4096 elements per block
constexpr int kRadix = 256;

template <class K>
__global__ void __launch_bounds__(kThreads) rs_hist(const K* __restrict__ keys, size_t n, int shift,
                                                    uint32_t* __restrict__ hist, int nblocks) {
  __shared__ uint32_t h[kRadix];
  for (int i = threadIdx.x; i < kRadix; i += kThreads) h[i] = 0;
  __syncthreads();
  const size_t base = static_cast<size_t>(blockIdx.x) * kTile;
#pragma unroll 4
  for (int r = 0; r < kItems; ++r) {
    const size_t idx = base + static_cast<size_t>(r) * kThreads + threadIdx.x;
    if (idx < n) atomicAdd(&h[static_cast<uint32_t>(keys[idx] >> shift) & 0xffu], 1u);
  }
  __syncthreads();
  for (int dgt = threadIdx.x; dgt < kRadix; dgt += kThreads)
    hist[static_cast<size_t>(dgt) * nblocks + blockIdx.x] = h[dgt];
}

// Exclusive scan in place over `total` words with one 1024-thread block.
__global__ void __launch_bounds__(1024) rs_scan(uint32_t* __restrict__ a, size_t total) {
  __shared__ uint32_t warp_sums[32];
  const size_t per = (total + 1023) / 1024;
  const size_t lo = threadIdx.x * per;
  const size_t hi = lo + per < total ? lo + per : total;
  uint32_t sum = 0;
  for (size_t i = lo; i < hi; ++i) sum += a[i];
  // block-wide exclusive scan of `sum`
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) warp_sums[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = warp_sums[lane];
    uint32_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += v;
    }
    warp_sums[lane] = wi - w;
  }
  __syncthreads();
  uint32_t run = warp_sums[warp] + incl - sum;
  for (size_t i = lo; i < hi; ++i) {
    const uint32_t v = a[i];
    a[i] = run;
    run += v;
  }
}

template <class K, bool kVals>
__global__ void __launch_bounds__(kThreads) rs_scatter(const K* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                       K* __restrict__ kout, uint32_t* __restrict__ vout, size_t n,
                                                       int shift, const uint32_t* __restrict__ hist, int nblocks) {
  __shared__ uint32_t whist[kWarps][kRadix];
  __shared__ uint32_t base[kRadix];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kWarps * kRadix; i += kThreads) (&whist[0][0])[i] = 0;
  for (int dgt = threadIdx.x; dgt < kRadix; dgt += kThreads)
    base[dgt] = hist[static_cast<size_t>(dgt) * nblocks + blockIdx.x];
  __syncthreads();

  const size_t wbase = static_cast<size_t>(blockIdx.x) * kTile + static_cast<size_t>(warp) * (32 * kItems);
  const unsigned lt_mask = (1u << lane) - 1u;
  K key[kItems];
  uint32_t val[kItems];
  uint32_t rank[kItems];
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const size_t idx = wbase + static_cast<size_t>(r) * 32 + lane;
    const bool ok = idx < n;
    key[r] = ok ? kin[idx] : K(0);
    if (kVals) val[r] = ok ? vin[idx] : 0u;
    const uint32_t dgt = ok ? (static_cast<uint32_t>(key[r] >> shift) & 0xffu) : 0x100u;
    const unsigned peers = __match_any_sync(0xffffffffu, dgt);
    const uint32_t before = __popc(peers & lt_mask);
    const uint32_t seen = ok ? whist[warp][dgt] : 0u;
    __syncwarp();
    if (ok && lane == __ffs(peers) - 1) whist[warp][dgt] = seen + __popc(peers);
    __syncwarp();
    rank[r] = seen + before;
  }
  __syncthreads();
  for (int dgt = threadIdx.x; dgt < kRadix; dgt += kThreads) {
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t c = whist[w][dgt];
      whist[w][dgt] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const size_t idx = wbase + static_cast<size_t>(r) * 32 + lane;
    if (idx < n) {
      const uint32_t dgt = static_cast<uint32_t>(key[r] >> shift) & 0xffu;
      const size_t pos = static_cast<size_t>(base[dgt]) + whist[warp][dgt] + rank[r];
      kout[pos] = key[r];
      if (kVals) vout[pos] = val[r];
    }
  }
}

}  // namespace

size_t radix_hist_words(size_t n) {
  const size_t blocks = (n + kTile - 1) / kTile;
  return (blocks ? blocks : 1) * kRadix;
}

template <class K>
int radix_sort(K* keys[2], uint32_t* vals[2], size_t n, int begin_bit, int end_bit, uint32_t* hist,
               cudaStream_t s) {
  if (n <= 1) return 0;
  const int nblocks = static_cast<int>((n + kTile - 1) / kTile);
  const size_t total = static_cast<size_t>(nblocks) * kRadix;
  int cur = 0;
  for (int shift = begin_bit; shift < end_bit; shift += 8) {
    rs_hist<K><<<nblocks, kThreads, 0, s>>>(keys[cur], n, shift, hist, nblocks);
    PSG_LAUNCHED();
    rs_scan<<<1, 1024, 0, s>>>(hist, total);
    PSG_LAUNCHED();
    if (vals[0])
      rs_scatter<K, true><<<nblocks, kThreads, 0, s>>>(keys[cur], vals[cur], keys[cur ^ 1], vals[cur ^ 1], n, shift,
                                                       hist, nblocks);
    else
      rs_scatter<K, false><<<nblocks, kThreads, 0, s>>>(keys[cur], nullptr, keys[cur ^ 1], nullptr, n, shift, hist,
                                                        nblocks);
    PSG_LAUNCHED();
    cur ^= 1;
  }
  return cur;
}

template int radix_sort<uint32_t>(uint32_t* [2], uint32_t* [2], size_t, int, int, uint32_t*, cudaStream_t);
template int radix_sort<uint64_t>(uint64_t* [2], uint32_t* [2], size_t, int, int, uint32_t*, cudaStream_t);

}  // namespace psg
