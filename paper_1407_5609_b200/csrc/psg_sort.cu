// psg_sort.cu — LSD radix sort, 8 bits per pass, three kernels per pass:
//   rs_hist    per-tile digit histogram (shared-memory atomics) -> digit-major
//              table hist[digit][tile]
//   rs_scan    one block per digit: exclusive scan along the tiles, digit total
//   rs_scatter stable scatter: the block first turns the 256 digit totals into
//              digit offsets (shared-memory scan), then ranks its tile with
//              warp-contiguous sub-tiles, __match_any_sync ranks inside 32-item
//              rounds, per-warp digit counters and a cross-warp scan
// Tiles are 256 x ITEMS elements; small inputs use ITEMS = 4 so a 1M-key pass
// still launches 1024 blocks (>= 6 per SM).  Per pass each element is read
// twice and written once, so the sort is HBM/latency bound.
#include "psg_internal.cuh"
#include "psg_sort.cuh"

namespace psg {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kRadix = 256;

template <int ITEMS>
constexpr int tile() {
  return kThreads * ITEMS;
}

int items_for(size_t n) { return n <= (size_t(1) << 22) ? 4 : 16; }

template <class K, int ITEMS>
__global__ void __launch_bounds__(kThreads) rs_hist(const K* __restrict__ keys, size_t n, int shift,
                                                    uint32_t* __restrict__ hist, int nblocks) {
  __shared__ uint32_t h[kRadix];
  h[threadIdx.x] = 0;
  __syncthreads();
  const size_t base = static_cast<size_t>(blockIdx.x) * tile<ITEMS>();
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    const size_t idx = base + static_cast<size_t>(r) * kThreads + threadIdx.x;
    if (idx < n) atomicAdd(&h[static_cast<uint32_t>(keys[idx] >> shift) & 0xffu], 1u);
  }
  __syncthreads();
  hist[static_cast<size_t>(threadIdx.x) * nblocks + blockIdx.x] = h[threadIdx.x];
}

// Block `digit`: exclusive scan of hist[digit][0..nblocks), total -> totals[digit].
__global__ void __launch_bounds__(kThreads) rs_scan(uint32_t* __restrict__ hist, int nblocks,
                                                    uint32_t* __restrict__ totals) {
  __shared__ uint32_t warp_sums[kWarps];
  __shared__ uint32_t carry;
  uint32_t* row = hist + static_cast<size_t>(blockIdx.x) * nblocks;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nblocks; base += kThreads) {
    const int i = base + threadIdx.x;
    const uint32_t v = i < nblocks ? row[i] : 0u;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) warp_sums[warp] = incl;
    __syncthreads();
    uint32_t wpre = 0, chunk = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t s = warp_sums[w];
      if (w < warp) wpre += s;
      chunk += s;
    }
    const uint32_t c = carry;
    if (i < nblocks) row[i] = c + wpre + incl - v;
    __syncthreads();
    if (threadIdx.x == 0) carry = c + chunk;
    __syncthreads();
  }
  if (threadIdx.x == 0) totals[blockIdx.x] = carry;
}

template <class K, bool kVals, int ITEMS>
__global__ void __launch_bounds__(kThreads) rs_scatter(const K* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                       K* __restrict__ kout, uint32_t* __restrict__ vout, size_t n,
                                                       int shift, const uint32_t* __restrict__ hist,
                                                       const uint32_t* __restrict__ totals, int nblocks) {
  __shared__ uint32_t whist[kWarps][kRadix];
  __shared__ uint32_t base[kRadix];
  __shared__ uint32_t wsum[kWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kWarps * kRadix; i += kThreads) (&whist[0][0])[i] = 0;
  {  // digit offsets = exclusive scan of the digit totals
    const uint32_t t = totals[threadIdx.x];
    uint32_t incl = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    uint32_t pre = 0;
    for (int w = 0; w < warp; ++w) pre += wsum[w];
    base[threadIdx.x] = pre + incl - t + hist[static_cast<size_t>(threadIdx.x) * nblocks + blockIdx.x];
  }
  __syncthreads();

  const size_t wbase =
      static_cast<size_t>(blockIdx.x) * tile<ITEMS>() + static_cast<size_t>(warp) * (32 * ITEMS);
  const unsigned lt_mask = (1u << lane) - 1u;
  K key[ITEMS];
  uint32_t val[ITEMS];
  uint32_t rank[ITEMS];
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
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
  {
    const int dgt = threadIdx.x;
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
  for (int r = 0; r < ITEMS; ++r) {
    const size_t idx = wbase + static_cast<size_t>(r) * 32 + lane;
    if (idx < n) {
      const uint32_t dgt = static_cast<uint32_t>(key[r] >> shift) & 0xffu;
      const size_t pos = static_cast<size_t>(base[dgt]) + whist[warp][dgt] + rank[r];
      kout[pos] = key[r];
      if (kVals) vout[pos] = val[r];
    }
  }
}

template <class K, int ITEMS>
int sort_impl(K* keys[2], uint32_t* vals[2], size_t n, int begin_bit, int end_bit, uint32_t* hist,
              cudaStream_t s) {
  const int nblocks = static_cast<int>((n + tile<ITEMS>() - 1) / tile<ITEMS>());
  uint32_t* totals = hist + static_cast<size_t>(nblocks) * kRadix;
  int cur = 0;
  for (int shift = begin_bit; shift < end_bit; shift += 8) {
    rs_hist<K, ITEMS><<<nblocks, kThreads, 0, s>>>(keys[cur], n, shift, hist, nblocks);
    PSG_LAUNCHED();
    rs_scan<<<kRadix, kThreads, 0, s>>>(hist, nblocks, totals);
    PSG_LAUNCHED();
    if (vals[0])
      rs_scatter<K, true, ITEMS><<<nblocks, kThreads, 0, s>>>(keys[cur], vals[cur], keys[cur ^ 1], vals[cur ^ 1], n,
                                                              shift, hist, totals, nblocks);
    else
      rs_scatter<K, false, ITEMS><<<nblocks, kThreads, 0, s>>>(keys[cur], nullptr, keys[cur ^ 1], nullptr, n, shift,
                                                               hist, totals, nblocks);
    PSG_LAUNCHED();
    cur ^= 1;
  }
  return cur;
}

}  // namespace

size_t radix_hist_words(size_t n) {
  const size_t t = static_cast<size_t>(kThreads) * items_for(n);
  const size_t blocks = (n + t - 1) / t;
  return (blocks ? blocks : 1) * kRadix + kRadix;
}

template <class K>
int radix_sort(K* keys[2], uint32_t* vals[2], size_t n, int begin_bit, int end_bit, uint32_t* hist,
               cudaStream_t s) {
  if (n <= 1) return 0;
  if (items_for(n) == 4) return sort_impl<K, 4>(keys, vals, n, begin_bit, end_bit, hist, s);
  return sort_impl<K, 16>(keys, vals, n, begin_bit, end_bit, hist, s);
}

template int radix_sort<uint32_t>(uint32_t* [2], uint32_t* [2], size_t, int, int, uint32_t*, cudaStream_t);
template int radix_sort<uint64_t>(uint64_t* [2], uint32_t* [2], size_t, int, int, uint32_t*, cudaStream_t);

}  // namespace psg
