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
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;  // 16384

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

// Single pass (decoupled look-back): each block takes tiles in order, scans
// a tile's 16384 values (four 16-byte loads per thread), publishes its
// aggregate, then one warp looks back over its predecessors' status words
// (flag in the top bits, value in the low 32; zeroed before the launch) until
// it reaches an inclusive prefix.  Reads the input once and writes the output
// once (the three-kernel tile/top/apply scan read it twice).
constexpr uint64_t kScanAgg = 1ull << 62, kScanInc = 2ull << 62;

__global__ void __launch_bounds__(kScanThreads) k_scan_lookback(const uint32_t* __restrict__ in, size_t count,
                                                                const uint64_t* __restrict__ dcells,
                                                                unsigned long long* __restrict__ status,
                                                                uint32_t* __restrict__ ticket,
                                                                uint32_t* __restrict__ out) {
  pdl_wait();  // PDL: the predecessor's writes are visible from here
  pdl_trigger();
  __shared__ uint32_t ws[33];
  __shared__ uint32_t tile_s, prefix_s;
  count = scan_count(count, dcells);
  (void)ticket;
  // persistent, static striding: block b scans tiles b, b + grid, ... in
  // order; every tile a block waits on is held by a block that started (all
  // blocks are resident: the grid is sized by the occupancy), so no ticket (a
  // shared ticket serialises every tile on one L2 address)
  for (uint32_t tile = blockIdx.x;; tile += gridDim.x) {
  __syncthreads();  // the previous tile's shared state is consumed
  if (static_cast<size_t>(tile) * kScanTile >= count) return;
  const size_t base = static_cast<size_t>(tile) * kScanTile + static_cast<size_t>(threadIdx.x) * kScanItems;
  uint32_t v[kScanItems];
  if (base + kScanItems <= count) {
#pragma unroll
    for (int q4 = 0; q4 < kScanItems / 4; ++q4) {
      const uint4 q = *reinterpret_cast<const uint4*>(in + base + 4 * q4);
      v[4 * q4] = q.x;
      v[4 * q4 + 1] = q.y;
      v[4 * q4 + 2] = q.z;
      v[4 * q4 + 3] = q.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) v[i] = base + i < count ? in[base + i] : 0u;
  }
  uint32_t sum = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) sum += v[i];
  uint32_t total;
  const uint32_t excl = block_exclusive(sum, ws, total);
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    uint32_t prefix = 0;
    if (tile == 0) {
      if (lane == 0) atomicExch(status, kScanInc | total);
    } else {
      if (lane == 0) atomicExch(status + tile, kScanAgg | total);
      const volatile unsigned long long* st = status;
      int64_t t0 = static_cast<int64_t>(tile) - 1;
      for (;;) {
        const int64_t idx = t0 - lane;
        unsigned long long w = idx >= 0 ? st[idx] : (kScanInc | 0ull);
        while (__any_sync(0xffffffffu, (w >> 62) == 0))  // a predecessor has not published yet
          if ((w >> 62) == 0) w = st[idx];
        const unsigned inc = __ballot_sync(0xffffffffu, (w >> 62) == 2);
        const int stop = inc ? __ffs(inc) - 1 : 31;  // nearest inclusive prefix, or the whole window
        uint32_t part = lane <= stop ? static_cast<uint32_t>(w) : 0u;
#pragma unroll
        for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        prefix += part;
        if (inc) break;
        t0 -= 32;
      }
      if (lane == 0) atomicExch(status + tile, kScanInc | static_cast<uint32_t>(prefix + total));
    }
    if (lane == 0) prefix_s = prefix;
  }
  __syncthreads();
  uint32_t run = excl + prefix_s;
  uint32_t o[kScanItems];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    o[i] = run;
    run += v[i];
  }
  if (base + kScanItems <= count) {
#pragma unroll
    for (int q4 = 0; q4 < kScanItems / 4; ++q4)
      *reinterpret_cast<uint4*>(out + base + 4 * q4) = make_uint4(o[4 * q4], o[4 * q4 + 1], o[4 * q4 + 2], o[4 * q4 + 3]);
  } else {
#pragma unroll
    for (int i = 0; i < kScanItems; ++i)
      if (base + i < count) out[base + i] = o[i];
  }
  }
}

}  // namespace

// temp layout: [tiles + 1 u64 status words][ticket]
size_t scan_temp_words(size_t count) { return 2 * ((count + kScanTile - 1) / kScanTile + 1) + 2; }

void exclusive_scan_u32(const uint32_t* in, uint32_t* out, size_t count, uint32_t* temp, cudaStream_t s) {
  exclusive_scan_u32_dev(in, out, count, nullptr, temp, s);
}

void exclusive_scan_u32_dev(const uint32_t* in, uint32_t* out, size_t max_count, const uint64_t* dcells,
                            uint32_t* temp, cudaStream_t s, bool zeroed) {
  if (max_count == 0) return;
  const size_t nb = (max_count + kScanTile - 1) / kScanTile;
  if (reinterpret_cast<uintptr_t>(in) % 16 || reinterpret_cast<uintptr_t>(out) % 16)
    throw std::runtime_error("exclusive_scan_u32: buffers must be 16-byte aligned");
  const size_t words = scan_temp_words(max_count);
  if (!zeroed) PSG_CUDA(cudaMemsetAsync(temp, 0, words * sizeof(uint32_t), s));
  auto* status = reinterpret_cast<unsigned long long*>(temp);
  // every block resident at once (the static tile striding waits on blocks
  // that must be running); they loop over the tiles
  static const int per_sm = [] {
    int per = 0;
    PSG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_scan_lookback, kScanThreads, 0));
    return std::max(per, 1);
  }();
  const unsigned grid = static_cast<unsigned>(std::min<size_t>(nb, static_cast<size_t>(ctx().sm_count) * per_sm));
  launch_pdl(k_scan_lookback, grid, kScanThreads, 0, s, in, max_count, dcells, status, temp + 2 * (nb + 1), out);
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
