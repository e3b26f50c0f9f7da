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

// ---- exclusive scan ---------------------------------------------------------
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;  // 4096

// Block-wide exclusive scan of one value per thread; returns the block total.
__device__ __forceinline__ uint32_t block_exclusive(uint32_t v, uint32_t* warp_sums, uint32_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) warp_sums[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint32_t w = warp_sums[lane];
    uint32_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    warp_sums[lane] = wi - w;
    if (lane == 31) warp_sums[32] = wi;
  }
  __syncthreads();
  total = warp_sums[32];
  return warp_sums[warp] + incl - v;
}

// count = *dcells + 1 when dcells is given (device-side size), else count.
__device__ __forceinline__ size_t scan_count(size_t count, const uint64_t* dcells) {
  return dcells ? static_cast<size_t>(*dcells) + 1 : count;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_tiles(const uint32_t* __restrict__ in, size_t count,
                                                             const uint64_t* __restrict__ dcells,
                                                             uint32_t* __restrict__ sums) {
  __shared__ uint32_t ws[33];
  count = scan_count(count, dcells);
  if (static_cast<size_t>(blockIdx.x) * kScanTile >= count) return;
  const size_t base = static_cast<size_t>(blockIdx.x) * kScanTile + static_cast<size_t>(threadIdx.x) * kScanItems;
  uint32_t v = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) v += base + i < count ? in[base + i] : 0u;
  uint32_t total;
  block_exclusive(v, ws, total);
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_top(uint32_t* __restrict__ sums, size_t count,
                                                           const uint64_t* __restrict__ dcells) {
  __shared__ uint32_t ws[33];
  count = scan_count(count, dcells);
  const int nb = static_cast<int>((count + kScanTile - 1) / kScanTile);
  constexpr int kPer = 8;  // up to 8192 tiles
  uint32_t v[kPer], s = 0;
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int k = threadIdx.x * kPer + i;
    v[i] = k < nb ? sums[k] : 0u;
    s += v[i];
  }
  uint32_t total;
  uint32_t run = block_exclusive(s, ws, total);
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int k = threadIdx.x * kPer + i;
    if (k < nb) sums[k] = run;
    run += v[i];
  }
}

__global__ void __launch_bounds__(kScanThreads) k_scan_apply(const uint32_t* __restrict__ in, size_t count,
                                                             const uint64_t* __restrict__ dcells,
                                                             const uint32_t* __restrict__ sums,
                                                             uint32_t* __restrict__ out) {
  __shared__ uint32_t ws[33];
  count = scan_count(count, dcells);
  if (static_cast<size_t>(blockIdx.x) * kScanTile >= count) return;
  const size_t base = static_cast<size_t>(blockIdx.x) * kScanTile + static_cast<size_t>(threadIdx.x) * kScanItems;
  uint32_t v[kScanItems], s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = base + i < count ? in[base + i] : 0u;
    s += v[i];
  }
  uint32_t total;
  uint32_t run = block_exclusive(s, ws, total) + sums[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < count) out[base + i] = run;
    run += v[i];
  }
}

}  // namespace

size_t scan_temp_words(size_t count) { return (count + kScanTile - 1) / kScanTile + 1; }

void exclusive_scan_u32(const uint32_t* in, uint32_t* out, size_t count, uint32_t* temp, cudaStream_t s) {
  exclusive_scan_u32_dev(in, out, count, nullptr, temp, s);
}

void exclusive_scan_u32_dev(const uint32_t* in, uint32_t* out, size_t max_count, const uint64_t* dcells,
                            uint32_t* temp, cudaStream_t s) {
  if (max_count == 0) return;
  const int nb = static_cast<int>((max_count + kScanTile - 1) / kScanTile);
  if (nb > 8 * kScanThreads) throw std::runtime_error("exclusive_scan_u32: input too large");
  k_scan_tiles<<<nb, kScanThreads, 0, s>>>(in, max_count, dcells, temp);
  PSG_LAUNCHED();
  k_scan_top<<<1, kScanThreads, 0, s>>>(temp, max_count, dcells);
  PSG_LAUNCHED();
  k_scan_apply<<<nb, kScanThreads, 0, s>>>(in, max_count, dcells, temp, out);
  PSG_LAUNCHED();
}

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
