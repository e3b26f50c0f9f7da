// psg_scan.cuh — device helpers shared by the candidate engines (sparse
// grid / window scans in psg_cpp.cu, dense cell-pair tiles in psg_dense.cu).
#pragma once

#include "psg_internal.cuh"
#include "psg_points.cuh"

namespace psg {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ bool admissible(uint32_t a, uint32_t b, uint64_t zone) {
  const uint32_t gap = a > b ? a - b : b - a;
  return gap >= zone;  // refscan.cpp:15-18
}

template <int NK>
__device__ __forceinline__ void load_keys(const float* __restrict__ p, float (&k)[NK]) {
  const float4* p4 = reinterpret_cast<const float4*>(p);
#pragma unroll
  for (int v = 0; v < NK / 4; ++v) {
    const float4 t = p4[v];
    k[4 * v + 0] = t.x;
    k[4 * v + 1] = t.y;
    k[4 * v + 2] = t.z;
    k[4 * v + 3] = t.w;
  }
}

// Lower-bound accumulator: the ONE expression both the scan and the recheck
// use, so the recheck filter is a deterministic subset of what the scan kept.
template <int NK>
__device__ __forceinline__ float lb2_full(const float (&a)[NK], const float (&b)[NK]) {
  float g = b[0] - a[0];
  float s = g * g;
#pragma unroll
  for (int k = 1; k < NK; ++k) {
    g = b[k] - a[k];
    s = fmaf(g, g, s);
  }
  return s;
}

// The canonical FP32 squared distance: one thread, fmaf accumulated in
// coordinate order t = 0..d-1 — the same order as the all-pairs kernel
// (psg_brute.cu), so every engine and every code path (queue flush, inline
// evaluation on a full queue, bootstrap, brute force) produces the same bits
// for a pair.  float4 loads when rows are 16-byte aligned (d % 4 == 0).
__device__ __forceinline__ float thread_sqdist(const float* __restrict__ a, const float* __restrict__ b, int d) {
  float s = 0.f;
  if ((d & 3) == 0) {
    const float4* a4 = reinterpret_cast<const float4*>(a);
    const float4* b4 = reinterpret_cast<const float4*>(b);
    for (int t = 0; t < (d >> 2); ++t) {
      const float4 x = __ldg(a4 + t), y = __ldg(b4 + t);
      float g = x.x - y.x;
      s = fmaf(g, g, s);
      g = x.y - y.y;
      s = fmaf(g, g, s);
      g = x.z - y.z;
      s = fmaf(g, g, s);
      g = x.w - y.w;
      s = fmaf(g, g, s);
    }
  } else {
    for (int t = 0; t < d; ++t) {
      const float g = __ldg(a + t) - __ldg(b + t);
      s = fmaf(g, g, s);
    }
  }
  return s;
}

// The same canonical distance between rows i and j of a row set, materialised
// or virtual (window sets: psg_points.cuh Rows): coordinate order, one fmaf
// per coordinate, identical bits for a pair on every path.
__device__ __forceinline__ float thread_sqdist(const Rows& R, uint64_t i, uint64_t j) {
  if (R.X) return thread_sqdist(R.X + i * R.d, R.X + j * R.d, R.d);
  const float* a = R.s32 + i;
  const float* b = R.s32 + j;
  float s = 0.f;
  if (R.m32) {
    const float ma = __ldg(R.m32 + i), ra = __ldg(R.r32 + i), mb = __ldg(R.m32 + j), rb = __ldg(R.r32 + j);
    for (int t = 0; t < R.d; ++t) {
      const float g = __fsub_rn(__fmul_rn(__fsub_rn(__ldg(a + t), ma), ra), __fmul_rn(__fsub_rn(__ldg(b + t), mb), rb));
      s = fmaf(g, g, s);
    }
  } else {
    for (int t = 0; t < R.d; ++t) {
      const float g = __ldg(a + t) - __ldg(b + t);
      s = fmaf(g, g, s);
    }
  }
  return s;
}

// Warp-level call site of the canonical distance (lane 0 computes, broadcast).
__device__ __forceinline__ float warp_sqdist(const float* __restrict__ a, const float* __restrict__ b, int d,
                                             int lane) {
  float s = 0.f;
  if (lane == 0) s = thread_sqdist(a, b, d);
  return __shfl_sync(kFull, s, 0);
}

__device__ __forceinline__ float warp_sqdist(const Rows& R, uint64_t i, uint64_t j, int lane) {
  float s = 0.f;
  if (lane == 0) s = thread_sqdist(R, i, j);
  return __shfl_sync(kFull, s, 0);
}

__device__ __forceinline__ float best_now(const unsigned* best) {
  return __uint_as_float(*reinterpret_cast<const volatile unsigned*>(best));
}

// ---------------------------------------------------------------------------
// The (FP64 distance, i, j) minimum as one 128-bit word: hi = the distance's
// bits (non-negative doubles order as unsigned), lo = (i << 32) | j with i < j
// original indices — the reference's "d < best, or d == best and (i, j)
// lexicographically smaller" (refscan.cpp:118-126) is unsigned 128-bit order.
// w[0] = lo, w[1] = hi; 16-byte aligned; initial value all ones.
__device__ __forceinline__ void load_u128(const unsigned long long* w, unsigned long long& lo, unsigned long long& hi) {
  asm volatile("{\n\t.reg .b128 r;\n\tld.relaxed.gpu.global.b128 r, [%2];\n\tmov.b128 {%0, %1}, r;\n\t}"
               : "=l"(lo), "=l"(hi)
               : "l"(w)
               : "memory");
}

__device__ __forceinline__ void atomic_min_u128(unsigned long long* w, unsigned long long hi, unsigned long long lo) {
  unsigned long long cl, ch;
  load_u128(w, cl, ch);  // one 16-byte access: a snapshot; the word only decreases
  while (hi < ch || (hi == ch && lo < cl)) {
    unsigned long long ol, oh;
    asm volatile(
        "{\n\t.reg .b128 c, v, r;\n\tmov.b128 c, {%2, %3};\n\tmov.b128 v, {%4, %5};\n\t"
        "atom.relaxed.gpu.global.cas.b128 r, [%6], c, v;\n\tmov.b128 {%0, %1}, r;\n\t}"
        : "=l"(ol), "=l"(oh)
        : "l"(cl), "l"(ch), "l"(lo), "l"(hi), "l"(w)
        : "memory");
    if (ol == cl && oh == ch) return;
    cl = ol;
    ch = oh;
  }
}

__device__ __forceinline__ unsigned long long lex_key(uint32_t i, uint32_t j) {
  return i < j ? (static_cast<unsigned long long>(i) << 32) | j : (static_cast<unsigned long long>(j) << 32) | i;
}

// What the inline FP64 evaluation of an overflowing band pair needs, kept in
// device memory (DevState) so the hot kernels carry one pointer for it and
// the cold path stays out of their register allocation.
struct InlineCtx {
  ExactSrc src;                  // the reference's values
  const uint32_t* sidx;          // sorted position -> original index
  unsigned long long* best128;   // (distance bits, (i << 32) | j) minimum, see atomic_min_u128
  unsigned long long* examined;  // FP64 evaluations
  unsigned long long* inline_n;  // of which inline
};

// Out of line (noinline): only ever reached past the candidate list.
static __device__ __noinline__ void record_inline(const InlineCtx* __restrict__ ic, uint32_t p, uint32_t j) {
  const uint32_t oi = ic->sidx[p], oj = ic->sidx[j];
  const double dd = exact_distance(ic->src, oi, oj);
  atomic_min_u128(ic->best128, static_cast<unsigned long long>(__double_as_longlong(dd)), lex_key(oi, oj));
  const unsigned m = __activemask();
  if ((threadIdx.x & 31) == __ffs(m) - 1) {
    atomicAdd(ic->examined, static_cast<unsigned long long>(__popc(m)));
    atomicAdd(ic->inline_n, static_cast<unsigned long long>(__popc(m)));
  }
}

struct ScanArgs {
  Rows rows;  // the FP32 working rows (X or virtual windows)
  const float* skeys;
  const uint32_t* sidx;
  uint32_t n;
  int d;
  uint64_t zone;
  const Budget* bud;  // device (DevState::bud)
  unsigned* best;
  uint32_t* cand_p;
  uint32_t* cand_j;
  float* cand_s;
  unsigned long long* cand_n;  // 64-bit: counts every band pair, never wraps
  uint32_t cand_cap;
  const InlineCtx* ic;            // band pairs past the list (DevState::ic)
  unsigned long long* evals;
  unsigned long long* visited;  // grid engine: admissible stencil pairs
  int no_ub;                    // debugging: dense Gram tiles do not feed their upper bounds to `best`
};

// A pair inside the FP32 band of the bound seen so far.  The first cand_cap
// band pairs of a scan are listed for the deterministic recheck (k_recheck /
// k_pick, against the FINAL bound); every later one is evaluated here in the
// reference's FP64 order and folded into the 128-bit (distance, i, j) minimum.
// Both sets are real admissible pairs and together they hold every pair the
// final band holds, so the minimum of the two is the reference's answer with
// no rescan and O(1) memory, however many exact ties the data has (a run of
// duplicate points puts all its pairs in the band).
__device__ __forceinline__ void record(const ScanArgs& a, uint32_t p, uint32_t j, float s32, float band) {
  atomicMin(a.best, __float_as_uint(s32));
  if (s32 <= band) {
    const unsigned long long c = atomicAdd(a.cand_n, 1ull);
    if (c < a.cand_cap) {
      a.cand_p[c] = p;
      a.cand_j[c] = j;
      a.cand_s[c] = s32;
    } else {
      record_inline(a.ic, p, j);
    }
  }
}

// The sparse scans' two variants (no function call in the list variant: the
// call's ABI would cost their candidate loops registers).  kExact = false: the
// list only, every band pair counted (cand_n > cand_cap tells the host the
// list lost pairs); kExact = true, the rescan after such an overflow: every
// band pair evaluated inline in FP64 into the 128-bit minimum, nothing listed.
template <bool kExact>
__device__ __forceinline__ void record_scan(const ScanArgs& a, uint32_t p, uint32_t j, float s32, float band) {
  atomicMin(a.best, __float_as_uint(s32));
  if (s32 <= band) {
    if constexpr (kExact) {
      record_inline(a.ic, p, j);
    } else {
      const unsigned long long c = atomicAdd(a.cand_n, 1ull);
      if (c < a.cand_cap) {
        a.cand_p[c] = p;
        a.cand_j[c] = j;
        a.cand_s[c] = s32;
      }
    }
  }
}

}  // namespace psg
