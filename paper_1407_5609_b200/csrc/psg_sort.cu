// psg_sort.cu — LSD radix sort, 8-bit digits, one pass = ONE kernel:
//   os_hist     once per sort: the digit histograms of every pass (one read
//               of the keys, shared-memory counters, global atomics)
//   os_scatter  per pass: a block takes the next tile (atomic ticket, so
//               tiles are claimed in order), ranks its 2048 keys stably
//               (warp __match_any_sync inside 32-key rounds, per-warp digit
//               counters, a cross-warp scan), publishes its digit counts and
//               resolves its global offsets by decoupled look-back over the
//               tiles before it (flag+value words tagged with the pass, so
//               one memset per sort serves every pass), then stages the tile
//               in shared memory in digit order and writes it out in
//               contiguous per-digit runs (coalesced)
// Stable: ties keep input order, so sorting (key, index) with the identity
// payload reproduces std::sort by (key, index).
#include "psg_internal.cuh"
#include "psg_sort.cuh"

namespace psg {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kRadix = 256;
// keys per thread: 16 for u32 keys (4096-key tiles), 8 for u64 (2048) —
// fewer, larger tiles shorten the look-back chains
template <class K>
constexpr int items() {
  return sizeof(K) == 4 ? 16 : 8;
}
template <class K>
constexpr int tile_keys() {
  return kThreads * items<K>();
}
constexpr int kMaxPasses = 8;
constexpr uint64_t kValMask = (1ull << 56) - 1;
constexpr uint64_t kFlagAgg = 1ull << 56;     // tile's own digit count
constexpr uint64_t kFlagPre = 2ull << 56;     // inclusive prefix over tiles 0..t

__device__ __forceinline__ uint64_t status_word(int pass, uint64_t flag, uint64_t v) {
  return (static_cast<uint64_t>(pass + 1) << 58) | flag | v;
}

template <class K>
__global__ void __launch_bounds__(kThreads) os_hist(const K* __restrict__ keys, size_t n, int begin_bit, int passes,
                                                    uint32_t* __restrict__ ghist) {
  __shared__ uint32_t h[kMaxPasses][kRadix];
  for (int i = threadIdx.x; i < kMaxPasses * kRadix; i += kThreads) (&h[0][0])[i] = 0;
  __syncthreads();
  for (size_t i = blockIdx.x * static_cast<size_t>(kThreads) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * kThreads) {
    const K k = keys[i];
    for (int p = 0; p < passes; ++p) atomicAdd(&h[p][static_cast<uint32_t>(k >> (begin_bit + 8 * p)) & 0xffu], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * kRadix; i += kThreads) {
    const uint32_t v = (&h[0][0])[i];
    if (v) atomicAdd(ghist + i, v);
  }
}

template <class K, bool kVals>
__global__ void __launch_bounds__(kThreads, 2) os_scatter(const K* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                       K* __restrict__ kout, uint32_t* __restrict__ vout, size_t n,
                                                       int shift, int pass, const uint32_t* __restrict__ ghist,
                                                       unsigned long long* __restrict__ status,
                                                       uint32_t* __restrict__ ticket) {
  __shared__ uint32_t whist[kWarps][kRadix];  // per-warp digit counts -> exclusive offsets
  __shared__ uint32_t bexcl[kRadix];          // digit start inside the tile
  __shared__ unsigned long long gbase[kRadix];  // global position of the tile's first key of each digit
  __shared__ uint32_t wsum[kWarps];
  __shared__ uint32_t s_tile;
  constexpr int kItems = items<K>(), kTile = tile_keys<K>();
  __shared__ K skeys[kTile];
  __shared__ uint32_t svals[kVals ? kTile : 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(ticket, 1u);
  for (int i = tid; i < kWarps * kRadix; i += kThreads) (&whist[0][0])[i] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const size_t base = static_cast<size_t>(tile) * kTile;
  const uint32_t tile_n = static_cast<uint32_t>(min(static_cast<size_t>(kTile), n - base));

  // stable ranks: warp w owns keys [w*32*kItems, (w+1)*32*kItems) of the tile in rounds of 32
  const size_t wbase = base + static_cast<size_t>(warp) * (32 * kItems);
  const unsigned lt_mask = (1u << lane) - 1u;
  K key[kItems];
  uint32_t val[kItems], rank[kItems], dg[kItems];
#pragma unroll
  for (int r = 0; r < kItems; ++r) {  // every load in flight before any ranking
    const size_t idx = wbase + static_cast<size_t>(r) * 32 + lane;
    const bool ok = idx < n;
    key[r] = ok ? kin[idx] : K(0);
    if (kVals) val[r] = ok ? vin[idx] : 0u;
    dg[r] = ok ? 0u : 0x100u;
  }
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const bool ok = dg[r] == 0u;
    if (ok) dg[r] = static_cast<uint32_t>(key[r] >> shift) & 0xffu;
    const unsigned peers = __match_any_sync(0xffffffffu, dg[r]);
    const uint32_t seen = ok ? whist[warp][dg[r]] : 0u;
    __syncwarp();
    if (ok && lane == __ffs(peers) - 1) whist[warp][dg[r]] = seen + __popc(peers);
    __syncwarp();
    rank[r] = seen + __popc(peers & lt_mask);
  }
  __syncthreads();
  // thread = digit: counts over warps, tile total, publish, look back
  const int d = tid;
  uint32_t count = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    const uint32_t c = whist[w][d];
    whist[w][d] = count;
    count += c;
  }
  unsigned long long* mine = status + static_cast<size_t>(tile) * kRadix + d;
  if (tile == 0) {
    atomicExch(mine, status_word(pass, kFlagPre, count));
  } else {
    atomicExch(mine, status_word(pass, kFlagAgg, count));
  }
  // look back in windows of kLook predecessors: their status words are
  // loaded together (independent loads in flight), then summed from the
  // nearest tile until one carries an inclusive prefix
  constexpr int kLook = 16;
  uint64_t excl = 0;
  bool done = tile == 0;
  for (int64_t t0 = static_cast<int64_t>(tile) - 1; !done; t0 -= kLook) {
    uint64_t v[kLook];
#pragma unroll
    for (int w = 0; w < kLook; ++w)
      v[w] = t0 - w >= 0 ? *(reinterpret_cast<const volatile unsigned long long*>(status) +
                             static_cast<size_t>(t0 - w) * kRadix + d)
                         : status_word(pass, kFlagPre, 0);
#pragma unroll
    for (int w = 0; w < kLook; ++w) {
      if (done) break;
      while ((v[w] >> 58) != static_cast<uint64_t>(pass + 1))  // not yet published in this pass
        v[w] = *(reinterpret_cast<const volatile unsigned long long*>(status) + static_cast<size_t>(t0 - w) * kRadix + d);
      excl += v[w] & kValMask;
      if (v[w] & kFlagPre) done = true;
    }
  }
  if (tile > 0) atomicExch(mine, status_word(pass, kFlagPre, excl + count));
  // global digit start: exclusive scan of the pass histogram (every block, 256 values)
  const uint32_t hcount = ghist[d];
  uint32_t incl = hcount, inclb = count;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    const uint32_t tb = __shfl_up_sync(0xffffffffu, inclb, o);
    if (lane >= o) {
      incl += t;
      inclb += tb;
    }
  }
  __shared__ uint32_t wsum_b[kWarps];
  if (lane == 31) {
    wsum[warp] = incl;
    wsum_b[warp] = inclb;
  }
  __syncthreads();
  uint32_t pre = 0, preb = 0;
  for (int w = 0; w < warp; ++w) {
    pre += wsum[w];
    preb += wsum_b[w];
  }
  gbase[d] = static_cast<unsigned long long>(pre + incl - hcount) + excl;
  bexcl[d] = preb + inclb - count;
  __syncthreads();
  // stage the tile in digit order
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    if (dg[r] < 0x100u) {
      const uint32_t local = bexcl[dg[r]] + whist[warp][dg[r]] + rank[r];
      skeys[local] = key[r];
      if (kVals) svals[local] = val[r];
    }
  }
  __syncthreads();
  // contiguous per-digit runs out
  for (uint32_t i = tid; i < tile_n; i += kThreads) {
    const K k = skeys[i];
    const uint32_t dd = static_cast<uint32_t>(k >> shift) & 0xffu;
    const size_t pos = gbase[dd] + (i - bexcl[dd]);
    kout[pos] = k;
    if (kVals) vout[pos] = svals[i];
  }
}

template <class K>
size_t tiles_for(size_t n) {
  return (n + tile_keys<K>() - 1) / tile_keys<K>();
}

// hist layout (u32 words): [kMaxPasses x 256 histograms][kMaxPasses tickets][pad][tiles x 256 u64 status]
size_t status_offset_words() { return ((kMaxPasses * kRadix + kMaxPasses) + 1) & ~size_t(1); }

template <class K>
int sort_impl(K* keys[2], uint32_t* vals[2], size_t n, int begin_bit, int end_bit, uint32_t* hist, cudaStream_t s) {
  const int passes = (end_bit - begin_bit + 7) / 8;
  if (passes > kMaxPasses) throw std::runtime_error("radix_sort: too many passes");
  const size_t tiles = tiles_for<K>(n);
  uint32_t* ghist = hist;
  uint32_t* tickets = hist + kMaxPasses * kRadix;
  auto* status = reinterpret_cast<unsigned long long*>(hist + status_offset_words());
  PSG_CUDA(cudaMemsetAsync(hist, 0, (status_offset_words() + 2 * tiles * kRadix) * sizeof(uint32_t), s));
  const int hb = static_cast<int>(std::min<size_t>((n + kThreads * 16 - 1) / (kThreads * 16), 148 * 8));
  os_hist<K><<<std::max(hb, 1), kThreads, 0, s>>>(keys[0], n, begin_bit, passes, ghist);
  PSG_LAUNCHED();
  int cur = 0;
  for (int p = 0; p < passes; ++p) {
    const int shift = begin_bit + 8 * p;
    if (vals[0])
      os_scatter<K, true><<<static_cast<unsigned>(tiles), kThreads, 0, s>>>(
          keys[cur], vals[cur], keys[cur ^ 1], vals[cur ^ 1], n, shift, p, ghist + p * kRadix, status, tickets + p);
    else
      os_scatter<K, false><<<static_cast<unsigned>(tiles), kThreads, 0, s>>>(
          keys[cur], nullptr, keys[cur ^ 1], nullptr, n, shift, p, ghist + p * kRadix, status, tickets + p);
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

size_t radix_hist_words(size_t n) { return status_offset_words() + 2 * tiles_for<uint64_t>(n) * kRadix; }

template <class K>
int radix_sort(K* keys[2], uint32_t* vals[2], size_t n, int begin_bit, int end_bit, uint32_t* hist,
               cudaStream_t s) {
  if (n <= 1) return 0;
  return sort_impl<K>(keys, vals, n, begin_bit, end_bit, hist, s);
}

template int radix_sort<uint32_t>(uint32_t* [2], uint32_t* [2], size_t, int, int, uint32_t*, cudaStream_t);
template int radix_sort<uint64_t>(uint64_t* [2], uint32_t* [2], size_t, int, int, uint32_t*, cudaStream_t);

}  // namespace psg
