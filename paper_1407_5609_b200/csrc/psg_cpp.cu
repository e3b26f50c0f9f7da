// psg_cpp.cu — exact closest pair on B200.
//
// Pipeline (reference loop refscan.cpp:67-132):
//   K1 project    keys = <U_k, X_i>, k < nk, one warp per row, U in registers
//   K2 sort       LSD radix sort of key 0 (+ index payload)          (psg_sort.cu)
//      gather     keys into sorted order (AoS, nk floats per point)
//   K3a bootstrap each sorted row vs its next `width` rows: min lower bound
//                 sum_k gap_k^2 per row, exact FP32 distance of each warp's
//                 best -> global upper bound delta_0 (atomicMin on FP32 bits)
//   K3b scan      each sorted row vs the rows whose key-0 gap is <= delta
//                 (the reference's sorted-order exit, refscan.cpp:85-92),
//                 pruned by all nk keys (its secondary references, 95-105),
//                 survivors queued in shared memory and evaluated as exact
//                 FP32 distances by whole warps (coalesced row loads, shuffle
//                 reduction); delta tightens as the atomic minimum falls
//   K6 recheck    every candidate inside the FP32 error band of the final
//                 delta re-evaluated in the reference's FP64 order; ties to the
//                 lowest (i, j) (refscan.cpp:118-126)
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <memory>

#include "psg_cpp.cuh"
#include "psg_engines.cuh"
#include "psg_scan.cuh"
#include "psg_sort.cuh"

namespace psg {

thread_local psg_profile g_prof;

void prof_begin() {
  std::memset(&g_prof, 0, sizeof(g_prof));
  g_launches = 0;
}

void prof_stages(const StageTimer& t) {
  if (!t.on || t.capture) return;  // a captured timer is read per replay (solve_graph)
  for (int i = 0; i < t.count && g_prof.stages < 16; ++i) {
    float ms = 0.f;
    PSG_CUDA(cudaEventElapsedTime(&ms, t.ev[i], t.ev[i + 1]));
    std::strncpy(g_prof.stage_name[g_prof.stages], t.name[i], 23);
    g_prof.stage_ms[g_prof.stages] = ms;
    ++g_prof.stages;
  }
}

namespace {

constexpr int kThreads = 256;
constexpr int kChunk = 256;
constexpr int kQueue = 1024;
constexpr int kInlineD = 16;  // d <= 16: one thread per exact evaluation
constexpr double kGridOccupancy = 0.25;   // mean points per cell over the key box (sweep: tools/occ_sweep.sh)
// window sets (motifs): near-duplicate windows straddle cell faces far more
// often; wider cells cost less than the regrid / full-stencil bootstrap the
// narrow ones trigger (C3 graph solve 0.77 -> 0.67 ms; tools/gpu_r2s2_ac2.sh)
constexpr double kGridOccupancyWindows = 1.5;
constexpr double kGridBoxSd = 2.5;        // key box: mean +- kGridBoxSd sd (clipped to the sample range)
constexpr int kGridBootCap = 256;         // candidates per point in the grid bootstrap
int boot_own_row() {  // the first bootstrap looks at the own cell row only (one cfirst lookup)
  static const int v = std::getenv("PSG_BOOT_FULL") ? 0 : 1;
  return v;
}
constexpr uint64_t kDenseFactor = 512;    // mean stencil candidates per point above which cells go dense

// ---------------------------------------------------------------------------
// K1: projection on CUDA cores for the shapes the tensor-core kernel does not
// take (psg_project_tc.cu handles d in {32, 64, 128, 256}).
// d < 32 (C1 d=2, C4 d=3, ...): one thread per row, U by value in the
// constant bank (so the launch carries no host-side buffer: graph-safe).
struct USmall {
  float u[kMaxKeys][32];
};

template <int NK>
__global__ void __launch_bounds__(256) k_project_small(const float* __restrict__ X, uint32_t n, int d,
                                                       const __grid_constant__ USmall U, float* __restrict__ keys,
                                                       unsigned* __restrict__ norm2_bits, CellCount cc) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  float nn = 0.f;
  if (r < n) {
    float acc[NK];
#pragma unroll
    for (int k = 0; k < NK; ++k) acc[k] = 0.f;
    const float* row = X + static_cast<size_t>(r) * d;
    for (int t = 0; t < d; ++t) {
      const float x = __ldg(row + t);
      nn = fmaf(x, x, nn);
#pragma unroll
      for (int k = 0; k < NK; ++k) acc[k] = fmaf(U.u[k][t], x, acc[k]);
    }
    float4* out = reinterpret_cast<float4*>(keys + static_cast<size_t>(r) * NK);
#pragma unroll
    for (int v = 0; v < NK / 4; ++v) out[v] = make_float4(acc[4 * v], acc[4 * v + 1], acc[4 * v + 2], acc[4 * v + 3]);
    if (cc.gp) count_cell<NK>(acc, r, cc);
  }
  block_max_to(norm2_bits, __float_as_uint(nn));
}

// Small or irregular d: one thread per row, U staged in shared memory.
template <int NK>
__global__ void __launch_bounds__(256) k_project_thread(const float* __restrict__ X, uint32_t n, int d,
                                                        const float* __restrict__ U, float* __restrict__ keys,
                                                        unsigned* __restrict__ norm2_bits, int u_in_smem) {
  extern __shared__ float su[];
  if (u_in_smem) {
    for (int i = threadIdx.x; i < NK * d; i += blockDim.x) su[i] = U[i];
    __syncthreads();
  }
  const float* Us = u_in_smem ? su : U;
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  float nn = 0.f;
  if (r < n) {
    float acc[NK];
#pragma unroll
    for (int k = 0; k < NK; ++k) acc[k] = 0.f;
    const float* row = X + static_cast<size_t>(r) * d;
    for (int t = 0; t < d; ++t) {
      const float x = __ldg(row + t);
      nn = fmaf(x, x, nn);
#pragma unroll
      for (int k = 0; k < NK; ++k) acc[k] = fmaf(Us[k * d + t], x, acc[k]);
    }
    float4* out = reinterpret_cast<float4*>(keys + static_cast<size_t>(r) * NK);
#pragma unroll
    for (int v = 0; v < NK / 4; ++v) out[v] = make_float4(acc[4 * v], acc[4 * v + 1], acc[4 * v + 2], acc[4 * v + 3]);
  }
  block_max_to(norm2_bits, __float_as_uint(nn));
}

// Window sets (virtual rows, psg_points.cuh Rows): kWinW consecutive windows
// per thread.  A block stages the series segment its kWinRows * kWinW windows
// span and, when it fits, U transposed (d x NK: one broadcast per tap and key
// quad); each thread slides a register window of kWinW series values along
// the taps, forms its rows on the fly — the same FP32 values every other
// reader sees — and accumulates each window's NK keys in coordinate order.
// Per tap the series value and U are loaded once for kWinW windows.  No
// n_w x d buffer is read or written: the C3 projection reads the 4 MiB series
// instead of 1 GiB of rows.  (The window rows' norms are measured once, when
// the set is built: k_window_check.)
constexpr int kWinRows = 128;
constexpr int kWinW = 4;
template <int NK>
__global__ void __launch_bounds__(kWinRows) k_project_windows(Rows R, uint32_t n, const float* __restrict__ Ut,
                                                              float* __restrict__ keys, int u_smem, int seg_smem,
                                                              CellCount cc) {
  extern __shared__ float4 sh4[];
  float* sh = reinterpret_cast<float*>(sh4);
  const int d = R.d;
  const uint32_t i0 = blockIdx.x * (kWinRows * kWinW);
  const uint32_t cnt = min(static_cast<uint32_t>(kWinRows * kWinW), n - i0);
  float* su = sh;  // d x NK (16-byte aligned)
  float* seg = sh + (u_smem ? d * NK : 0);
  if (u_smem)
    for (int k = threadIdx.x; k < d * NK; k += kWinRows) su[k] = Ut[k];
  if (seg_smem)
    for (uint32_t k = threadIdx.x; k < cnt + d - 1; k += kWinRows) seg[k] = R.s32[i0 + k];
  __syncthreads();
  const uint32_t r0 = threadIdx.x * kWinW;  // this thread's first window, block-relative
  if (r0 >= cnt) return;
  const float* Us = u_smem ? su : Ut;
  const float* x = seg_smem ? seg + r0 : R.s32 + i0 + r0;
  const bool z = R.m32 != nullptr;
  float m[kWinW], rr[kWinW], acc[kWinW][NK], ring[kWinW];
#pragma unroll
  for (int w = 0; w < kWinW; ++w) {
    const uint32_t i = min(i0 + r0 + w, n - 1);  // past the end: a duplicate, not stored
    m[w] = z ? R.m32[i] : 0.f;
    rr[w] = z ? R.r32[i] : 1.f;
#pragma unroll
    for (int k = 0; k < NK; ++k) acc[w][k] = 0.f;
  }
  // ring[w] = series value at tap t of window r0 + w = x[t + w]; offsets past
  // the last valid one (windows beyond the set's end, never stored) are
  // clamped so no read leaves the segment / series
  const uint32_t last = cnt - r0 - 1 + d - 1;
#pragma unroll
  for (int w = 0; w < kWinW - 1; ++w) ring[w] = x[min(static_cast<uint32_t>(w), last)];
  for (int t = 0; t < d; ++t) {
    ring[kWinW - 1] = x[min(static_cast<uint32_t>(t + kWinW - 1), last)];
    float4 u[NK / 4];
    const float4* u4 = reinterpret_cast<const float4*>(Us + t * NK);
#pragma unroll
    for (int q = 0; q < NK / 4; ++q) u[q] = u4[q];
#pragma unroll
    for (int w = 0; w < kWinW; ++w) {
      const float v = z ? __fmul_rn(__fsub_rn(ring[w], m[w]), rr[w]) : ring[w];
#pragma unroll
      for (int q = 0; q < NK / 4; ++q) {
        acc[w][4 * q + 0] = fmaf(u[q].x, v, acc[w][4 * q + 0]);
        acc[w][4 * q + 1] = fmaf(u[q].y, v, acc[w][4 * q + 1]);
        acc[w][4 * q + 2] = fmaf(u[q].z, v, acc[w][4 * q + 2]);
        acc[w][4 * q + 3] = fmaf(u[q].w, v, acc[w][4 * q + 3]);
      }
    }
#pragma unroll
    for (int w = 0; w < kWinW - 1; ++w) ring[w] = ring[w + 1];
  }
#pragma unroll
  for (int w = 0; w < kWinW; ++w) {
    if (r0 + w >= cnt) break;
    float4* out = reinterpret_cast<float4*>(keys + static_cast<size_t>(i0 + r0 + w) * NK);
#pragma unroll
    for (int q = 0; q < NK / 4; ++q)
      out[q] = make_float4(acc[w][4 * q], acc[w][4 * q + 1], acc[w][4 * q + 2], acc[w][4 * q + 3]);
    if (cc.gp) count_cell<NK>(acc[w], i0 + r0 + w, cc);
  }
}

template <int NK>
__global__ void k_sort_keys(const float* __restrict__ keys, uint32_t n, uint32_t* __restrict__ k_out,
                            uint32_t* __restrict__ v_out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  k_out[i] = f32_order(keys[static_cast<size_t>(i) * NK]);
  v_out[i] = i;
}

template <int NK>
__global__ void k_gather(const float* __restrict__ keys, const uint32_t* __restrict__ perm, uint32_t n,
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

// Seed: pair (0, max(zone,1)) is admissible whenever any pair is, so delta
// is finite from the start.
__global__ void k_seed_pair(ScanArgs a, uint32_t z) {
  const int lane = threadIdx.x & 31;
  const float s = a.d <= kInlineD ? (lane == 0 ? thread_sqdist(a.rows, 0, z) : 0.f) : warp_sqdist(a.rows, 0, z, lane);
  if (lane == 0) atomicMin(a.best, __float_as_uint(s));
}

// K3a: bootstrap.  All threads walk the same j (shared-memory broadcast).
template <int NK>
__global__ void __launch_bounds__(kThreads) k_bootstrap(ScanArgs a, uint32_t lo, uint32_t hi, uint32_t width) {
  __shared__ __align__(16) float sk[kChunk * NK];
  __shared__ uint32_t so[kChunk];
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t p0 = lo + blockIdx.x * kThreads;
  const uint32_t p = p0 + tid;
  const bool valid = p < hi;
  float mk[NK];
  uint32_t mo = 0;
  if (valid) {
    load_keys<NK>(a.skeys + static_cast<size_t>(p) * NK, mk);
    mo = a.sidx[p];
  } else {
#pragma unroll
    for (int k = 0; k < NK; ++k) mk[k] = 0.f;
  }
  float best_lb = INFINITY;
  uint32_t best_j = 0xffffffffu;
  const uint64_t jend64 = static_cast<uint64_t>(p0) + kThreads + width;
  const uint32_t jend = static_cast<uint32_t>(jend64 < a.n ? jend64 : a.n);
  for (uint32_t c0 = p0 + 1; c0 < jend; c0 += kChunk) {
    const uint32_t cnt = min(static_cast<uint32_t>(kChunk), jend - c0);
    __syncthreads();
    if (tid < cnt) {
      const float4* src = reinterpret_cast<const float4*>(a.skeys + static_cast<size_t>(c0 + tid) * NK);
      float4* dst = reinterpret_cast<float4*>(sk + tid * NK);
#pragma unroll
      for (int v = 0; v < NK / 4; ++v) dst[v] = src[v];
      so[tid] = a.sidx[c0 + tid];
    }
    __syncthreads();
    if (valid) {
      for (uint32_t jj = 0; jj < cnt; ++jj) {
        const uint32_t j = c0 + jj;
        if (j <= p || j > p + width) continue;
        const float* kj = sk + jj * NK;
        float g = kj[0] - mk[0];
        float s = g * g;
        g = kj[1] - mk[1];
        s = fmaf(g, g, s);
        if (s >= best_lb) continue;
#pragma unroll
        for (int k = 2; k < NK; ++k) {
          g = kj[k] - mk[k];
          s = fmaf(g, g, s);
        }
        if (s < best_lb && admissible(mo, so[jj], a.zone)) {
          best_lb = s;
          best_j = j;
        }
      }
    }
  }
  // warp argmin of the per-row best lower bound, then one exact evaluation
  float wlb = best_lb;
  uint32_t wj = best_j, wp = p;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float olb = __shfl_xor_sync(kFull, wlb, o);
    const uint32_t oj = __shfl_xor_sync(kFull, wj, o);
    const uint32_t op = __shfl_xor_sync(kFull, wp, o);
    if (olb < wlb || (olb == wlb && op < wp)) {
      wlb = olb;
      wj = oj;
      wp = op;
    }
  }
  if (wj == 0xffffffffu) return;
  const Thresholds th = budget_thresholds_s32(*a.bud,best_now(a.best));
  if (!(wlb <= th.lb2)) return;
  const uint32_t xi = a.sidx[wp], xj = a.sidx[wj];
  float s;
  if (a.d <= kInlineD)
    s = lane == 0 ? thread_sqdist(a.rows, xi, xj) : 0.f;
  else
    s = warp_sqdist(a.rows, xi, xj, lane);
  if (lane == 0) atomicMin(a.best, __float_as_uint(s));
}

// K3b: the windowed candidate scan.
template <int NK, bool kExact>
__global__ void __launch_bounds__(kThreads) k_scan(ScanArgs a, uint32_t lo, uint32_t hi) {
  __shared__ __align__(16) float sk[kChunk * NK];
  __shared__ uint32_t so[kChunk];
  __shared__ uint32_t qp[kQueue], qj[kQueue];
  __shared__ int qn;
  __shared__ Thresholds th;
  __shared__ unsigned long long nevals;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t p0 = lo + blockIdx.x * kThreads;
  const uint32_t p = p0 + tid;
  const uint32_t plast = min(p0 + kThreads, hi) - 1;
  bool active = p < hi;
  float mk[NK];
  uint32_t mo = 0;
  if (active) {
    load_keys<NK>(a.skeys + static_cast<size_t>(p) * NK, mk);
    mo = a.sidx[p];
  } else {
#pragma unroll
    for (int k = 0; k < NK; ++k) mk[k] = 0.f;
  }
  const float kmax = a.skeys[static_cast<size_t>(plast) * NK];
  if (tid == 0) {
    qn = 0;
    nevals = 0;
    th = budget_thresholds_s32(*a.bud,best_now(a.best));
  }
  __syncthreads();
  for (uint32_t c0 = p0 + 1; c0 < a.n; c0 += kChunk) {
    if (a.skeys[static_cast<size_t>(c0) * NK] - kmax > th.win) break;  // block-wide exit
    const uint32_t cnt = min(static_cast<uint32_t>(kChunk), a.n - c0);
    if (tid < cnt) {
      const float4* src = reinterpret_cast<const float4*>(a.skeys + static_cast<size_t>(c0 + tid) * NK);
      float4* dst = reinterpret_cast<float4*>(sk + tid * NK);
#pragma unroll
      for (int v = 0; v < NK / 4; ++v) dst[v] = src[v];
      so[tid] = a.sidx[c0 + tid];
    }
    __syncthreads();
    if (active) {
      const float win = th.win, lb2 = th.lb2;
      for (uint32_t jj = 0; jj < cnt; ++jj) {
        const uint32_t j = c0 + jj;
        if (j <= p) continue;
        const float* kj = sk + jj * NK;
        float g = kj[0] - mk[0];
        if (g > win) {  // sorted: every later j is farther (refscan.cpp:85)
          active = false;
          break;
        }
        float s = g * g;
        g = kj[1] - mk[1];
        s = fmaf(g, g, s);
        if (s > lb2) continue;
#pragma unroll
        for (int k = 2; k < NK; ++k) {
          g = kj[k] - mk[k];
          s = fmaf(g, g, s);
        }
        if (s > lb2 || !admissible(mo, so[jj], a.zone)) continue;
        const int slot = atomicAdd(&qn, 1);
        if (slot < kQueue) {
          qp[slot] = p;
          qj[slot] = j;
        } else {  // queue full: evaluate here (canonical order, bounded memory)
          record_scan<kExact>(a, p, j, thread_sqdist(a.rows, mo, so[jj]), th.band);
        }
      }
    }
    __syncthreads();
    const int nq = min(qn, kQueue);
    if (nq > 0) {
      const float band = th.band;
      for (int i = tid; i < nq; i += kThreads) {  // one queued pair per thread
        const uint32_t pi = qp[i], pj = qj[i];
        const float s = thread_sqdist(a.rows, a.sidx[pi], a.sidx[pj]);
        record_scan<kExact>(a, pi, pj, s, band);
      }
    }
    __syncthreads();
    if (tid == 0) {
      nevals += static_cast<unsigned long long>(nq);
      qn = 0;
      th = budget_thresholds_s32(*a.bud,best_now(a.best));
    }
    if (!__syncthreads_or(active)) break;
  }
  if (tid == 0 && nevals) atomicAdd(a.evals, nevals);
}

// ---------------------------------------------------------------------------
// Grid engine (psg_grid.cuh): candidates of sorted position p are the later
// positions of its own cell and every position of the forward half of the
// 3^g cell stencil, so each unordered pair is visited exactly once.

// Warp argmin of (lb, p) and one exact FP32 evaluation of the winner.
// Returns the (rounded-up) FP32 squared distance of the warp's winner, +inf
// when the warp has none; the caller min-reduces it per block.
__device__ __forceinline__ float warp_eval_best(const ScanArgs& a, float lb, uint32_t j, uint32_t p, int lane) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float olb = __shfl_xor_sync(kFull, lb, o);
    const uint32_t oj = __shfl_xor_sync(kFull, j, o);
    const uint32_t op = __shfl_xor_sync(kFull, p, o);
    if (olb < lb || (olb == lb && op < p)) {
      lb = olb;
      j = oj;
      p = op;
    }
  }
  if (j == 0xffffffffu) return INFINITY;
  const uint32_t xi = a.sidx[p], xj = a.sidx[j];
  // Warp-parallel sum (not the canonical order), rounded up by (2d+8) ulps
  // relative: two FP32 orders of a sum of d non-negative terms differ by at
  // most 2d*2^-24 relative, so this stays >= the canonical value the scan
  // computes for the same pair (the final bound is always a canonical value),
  // and any value >= a computed one is a valid bound for the thresholds.
  float s = 0.f;
  for (int t = lane; t < a.d; t += 32) {
    const float g = row_at(a.rows, xi, t) - row_at(a.rows, xj, t);
    s = fmaf(g, g, s);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  return __fmul_ru(s, 1.0f + static_cast<float>(2 * a.d + 8) * 0x1.0p-24f);
}

// K3a (grid): per position, the stencil candidate with the least key lower
// bound (at most `cap` candidates looked at); each warp evaluates its best.
template <int NK>
__global__ void __launch_bounds__(kThreads) k_grid_bootstrap(ScanArgs a, GridDev G, uint32_t lo, uint32_t hi,
                                                             int cap, int own_row) {
  __shared__ GridParams sP;  // one copy per block, not per thread (registers)
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) sP = *G.gp;
  __syncthreads();
  const uint32_t p = lo + blockIdx.x * kThreads + threadIdx.x;
  float best_lb = INFINITY;
  uint32_t best_j = 0xffffffffu;
  if (p < hi) {
    float mk[NK];
    load_keys<NK>(a.skeys + static_cast<size_t>(p) * NK, mk);
    const uint32_t mo = a.sidx[p];
    const GridFlat F = grid_flat(own_row ? grid_own_row(G.cfirst, sP, p, G.scell[p])
                                         : grid_ranges(G.cfirst, sP, p, G.scell[p]));
    const uint32_t L = min(F.total, static_cast<uint32_t>(cap));
    // more candidates than the cap: a uniform stride over all of them (a
    // cell lists its points in index order, which can correlate with
    // structure in the data, e.g. cluster = index mod k)
    const uint32_t stride = F.total > L ? F.total / L : 1u;
    // four candidates per step: all key loads in flight before any math
    constexpr int B = 2;  // candidates in flight per step (registers vs latency)
    for (uint32_t t0 = 0; t0 < L; t0 += B) {
      uint32_t jj[B];
      float kk[B][NK];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        jj[u] = t0 + u < L ? F.at((t0 + u) * stride) : p;
        load_keys<NK>(a.skeys + static_cast<size_t>(jj[u]) * NK, kk[u]);
      }
#pragma unroll
      for (int u = 0; u < B; ++u) {
        if (t0 + u >= L) break;
        const float sl = lb2_full<NK>(mk, kk[u]);
        if (sl < best_lb && (a.zone <= 1 || admissible(mo, a.sidx[jj[u]], a.zone))) {
          best_lb = sl;
          best_j = jj[u];
        }
      }
    }
  }
  const float s = warp_eval_best(a, best_lb, best_j, p, lane);
  // one atomic per block (per-warp atomics on one address serialise at the L2)
  __shared__ float wmin[kThreads / 32];
  if (lane == 0) wmin[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = wmin[0];
    for (int w = 1; w < kThreads / 32; ++w) m = fminf(m, wmin[w]);
    if (m < INFINITY) atomicMin(a.best, __float_as_uint(m));
  }
}

// Before the scan: the grid must hold every pair whose key gaps are within
// the window of the bound reached by the bootstrap; otherwise flag a rebuild
// (the host widens the cells and reruns the scan).  One thread, so every
// block of the scan sees the same decision.
// Also resets the attempt's counters and minima (one launch for both).
__global__ void k_scan_prepare(DevState* st, const GridParams* gp) {
  st->cand_n = 0;
  st->best64 = ~0ull;
  st->lex = ~0ull;
  st->best128[0] = st->best128[1] = ~0ull;
  st->examined = st->evals = st->visited = st->inline_n = 0;
  const unsigned b = st->best;
  const Thresholds th = budget_thresholds_s32(st->bud, __uint_as_float(b));
  st->check_best = b;
  st->th = th;  // the scan's starting thresholds, computed once
  st->regrid = gp ? !(gp->w >= static_cast<double>(th.win) * (1.0 + 1e-5)) : 0u;
}

// K3b (grid): one pass per sorted position over its (at most five) stencil
// ranges with the key lower bound at the threshold it read at start (the
// bound only tightens, so a stale threshold only admits more); survivors go to
// the warp's shared-memory queue (evaluated in place when full) and the warp's
// lanes evaluate them as exact FP32 distances after its own loop — no block
// barrier after the candidate loops, so a warp never waits for the block's
// slowest position.  The block's counts reach global memory through the last
// warp to finish (a shared-memory ticket): one atomic per block and counter.
constexpr int kScanWarps = kThreads / 32;
constexpr int kWarpQueue = kQueue / kScanWarps;
template <int NK, bool kExact>
__global__ void __launch_bounds__(kThreads) k_grid_scan2(ScanArgs a, GridDev G, uint32_t lo, uint32_t hi,
                                                         const unsigned* __restrict__ regrid,
                                                         const Thresholds* __restrict__ th0) {
  __shared__ uint32_t qp[kScanWarps][kWarpQueue], qj[kScanWarps][kWarpQueue];
  __shared__ int qn[kScanWarps];
  __shared__ unsigned long long s_visited, s_evals;
  __shared__ unsigned s_done;
  __shared__ double s_win;
  __shared__ GridParams sP;  // one copy per block, not per thread (registers)
  if (*regrid) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t p = lo + blockIdx.x * kThreads + tid;
  // the position's own loads go out before the block barrier (they do not
  // need the shared grid parameters)
  const uint32_t pc = p < hi ? p : lo;
  float mk[NK];
  load_keys<NK>(a.skeys + static_cast<size_t>(pc) * NK, mk);
  const uint32_t mo = a.sidx[pc], mcell = G.scell[pc];
  const float lb2 = th0->lb2;
  if (tid < kScanWarps) qn[tid] = 0;
  if (tid == 0) {
    sP = *G.gp;
    s_visited = s_evals = 0;
    s_done = 0;
    // rows the point is too far from to hold a passing pair are skipped
    // (margin: cell faces are computed in FP64 like the cell ids, keys are
    // FP32); one FP64 square root per block
    s_win = sqrt(static_cast<double>(lb2)) * (1.0 + 0x1.0p-20) + 1e-6 * sP.w;
  }
  __syncthreads();
  unsigned long long visited = 0, inline_evals = 0;
  if (p < hi) {
    const GridFlat F = grid_flat(grid_ranges_pruned(G.cfirst, sP, p, mcell, mk, s_win));
    const bool zoned = a.zone > 1;
    // two candidates per step: all loads in flight before any math
    constexpr int B = 2;  // candidates in flight per step (registers vs latency)
    for (uint32_t t0 = 0; t0 < F.total; t0 += B) {
      uint32_t jj[B], oo[B];
      float4 k0[B];  // keys 0-3 first: most candidates fail on them (16 B instead of 32 B)
#pragma unroll
      for (int u = 0; u < B; ++u) {
        jj[u] = t0 + u < F.total ? F.at(t0 + u) : p;
        k0[u] = *reinterpret_cast<const float4*>(a.skeys + static_cast<size_t>(jj[u]) * NK);
        oo[u] = zoned ? a.sidx[jj[u]] : 0u;
      }
#pragma unroll
      for (int u = 0; u < B; ++u) {
        if (t0 + u >= F.total) break;
        if (zoned && !admissible(mo, oo[u], a.zone)) continue;
        ++visited;
        const uint32_t j = jj[u];
        // the lb2_full accumulation order, split after key 3: the partial sum
        // only grows, so rejecting on it rejects exactly what the full sum would
        float g = k0[u].x - mk[0];
        float sl = g * g;
        g = k0[u].y - mk[1];
        sl = fmaf(g, g, sl);
        g = k0[u].z - mk[2];
        sl = fmaf(g, g, sl);
        g = k0[u].w - mk[3];
        sl = fmaf(g, g, sl);
        if (sl > lb2) continue;
        if constexpr (NK == 8) {
          const float4 k1 = *reinterpret_cast<const float4*>(a.skeys + static_cast<size_t>(j) * NK + 4);
          g = k1.x - mk[4];
          sl = fmaf(g, g, sl);
          g = k1.y - mk[5];
          sl = fmaf(g, g, sl);
          g = k1.z - mk[6];
          sl = fmaf(g, g, sl);
          g = k1.w - mk[7];
          sl = fmaf(g, g, sl);
          if (sl > lb2) continue;
        }
        const int slot = atomicAdd(&qn[warp], 1);
        if (slot < kWarpQueue) {
          qp[warp][slot] = p;
          qj[warp][slot] = j;
        } else {  // queue full: evaluate here (canonical order, bounded memory)
          record_scan<kExact>(a, p, j, thread_sqdist(a.rows, mo, a.sidx[j]), th0->band);
          ++inline_evals;
        }
      }
    }
  }
  __syncwarp();
  const int nq = min(qn[warp], kWarpQueue);
  if (nq > 0) {
    const float band = th0->band;  // >= the band of any tighter bound: a superset, refiltered by k_recheck
    for (int i = lane; i < nq; i += 32) {  // one queued pair per lane
      const uint32_t pi = qp[warp][i], pj = qj[warp][i];
      const float sd = thread_sqdist(a.rows, a.sidx[pi], a.sidx[pj]);
      record_scan<kExact>(a, pi, pj, sd, band);
    }
  }
  for (int o = 16; o; o >>= 1) {
    visited += __shfl_xor_sync(kFull, visited, o);
    inline_evals += __shfl_xor_sync(kFull, inline_evals, o);
  }
  if (lane == 0) {
    if (visited) atomicAdd(&s_visited, visited);
    const unsigned long long e = inline_evals + static_cast<unsigned long long>(nq);
    if (e) atomicAdd(&s_evals, e);
    __threadfence_block();
    if (atomicAdd(&s_done, 1u) == kScanWarps - 1) {  // the block's last warp
      __threadfence_block();
      const unsigned long long v = atomicAdd(&s_visited, 0ull), ev = atomicAdd(&s_evals, 0ull);
      if (v) atomicAdd(a.visited, v);
      if (ev) atomicAdd(a.evals, ev);
    }
  }
}

// K6: deterministic final filter + FP64 recheck in the reference's order.
// Thresholds come from the final FP32 bound on device; the candidate count is
// min(candidates, capacity) read on device; grid-stride over candidates.
// kWarp: one warp per candidate, the exact distance's terms in parallel
// (warp_exact_distance) — for d >= 32, where one thread per candidate is
// latency-bound (a z-normalised window term costs two FP64 divisions: one
// thread spent 76 us on C3's single candidate); else one thread per candidate.
template <int NK, bool kWindow, bool kWarp>
__global__ void k_recheck(ScanArgs a, ExactSrc src, double* __restrict__ d64, unsigned long long* __restrict__ best64,
                          unsigned long long* __restrict__ examined) {
  const uint32_t count = static_cast<uint32_t>(min(*a.cand_n, static_cast<unsigned long long>(a.cand_cap)));
  constexpr uint32_t kPer = kWarp ? 32 : 1;  // threads per candidate
  const uint32_t per_block = blockDim.x / kPer;
  if (blockIdx.x * per_block >= count) return;  // usually one block has work (C2: one candidate)
  // the final bound's thresholds, once per block (FP64 sqrt / divisions)
  __shared__ Thresholds sth;
  if (threadIdx.x == 0) sth = budget_thresholds_s32(*a.bud, best_now(a.best));
  __syncthreads();
  const Thresholds th = sth;
  const int lane = threadIdx.x & 31;
  const uint32_t u0 = (blockIdx.x * blockDim.x + threadIdx.x) / kPer, nu = gridDim.x * per_block;
  unsigned long long pass = 0;
  for (uint32_t base = (u0 / per_block) * per_block; base < count; base += nu) {
    const uint32_t c = base + (threadIdx.x / kPer);
    bool keep = false;
    uint32_t p = 0, j = 0;
    if (c < count) {
      p = a.cand_p[c];
      j = a.cand_j[c];
      float kp[NK], kj[NK];
      load_keys<NK>(a.skeys + static_cast<size_t>(p) * NK, kp);
      load_keys<NK>(a.skeys + static_cast<size_t>(j) * NK, kj);
      keep = (!kWindow || kj[0] - kp[0] <= th.win) && (lb2_full<NK>(kp, kj) <= th.lb2) && (a.cand_s[c] <= th.band);
    }
    double dd = -1.0;
    if constexpr (kWarp) {
      if (keep) {  // warp-uniform: every lane read the same candidate
        dd = warp_exact_distance(src, a.sidx[p], a.sidx[j], lane);
        if (lane == 0) atomicMin(best64, static_cast<unsigned long long>(__double_as_longlong(dd)));
        ++pass;
      }
      if (c < count && lane == 0) d64[c] = dd;
    } else {
      if (keep) {
        dd = exact_distance(src, a.sidx[p], a.sidx[j]);
        atomicMin(best64, static_cast<unsigned long long>(__double_as_longlong(dd)));
        ++pass;
      }
      if (c < count) d64[c] = dd;
    }
  }
  if constexpr (!kWarp) pass = __reduce_add_sync(kFull, static_cast<unsigned>(pass));
  if (lane == 0 && pass) atomicAdd(examined, pass);
}

__global__ void k_pick(const ScanArgs a, const double* __restrict__ d64, const unsigned long long* __restrict__ best64,
                       unsigned long long* __restrict__ lex) {
  const uint32_t count = static_cast<uint32_t>(min(*a.cand_n, static_cast<unsigned long long>(a.cand_cap)));
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < count; c += gridDim.x * blockDim.x) {
    if (static_cast<unsigned long long>(__double_as_longlong(d64[c])) != *best64 || d64[c] < 0.0) continue;
    atomicMin(lex, lex_key(a.sidx[a.cand_p[c]], a.sidx[a.cand_j[c]]));
  }
}

// Lower the device bound to min(current, bound) (multi-rank global bound).
__global__ void k_min_bound(unsigned* best, float bound) {
  if (bound >= 0.f) atomicMin(best, __float_as_uint(bound));
}

// Window statistics at the final delta: pairs with fl(k0_j - k0_p) <= win,
// and rows whose window ends before the last point.
template <int NK>
__global__ void k_window_stats(const float* __restrict__ skeys, uint32_t n, uint32_t lo, uint32_t hi, float win,
                               unsigned long long* __restrict__ pairs, unsigned long long* __restrict__ exits) {
  const uint32_t p = lo + blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long cnt = 0;
  unsigned ex = 0;
  if (p < hi) {
    const float kp = skeys[static_cast<size_t>(p) * NK];
    uint32_t a = p + 1, b = n;  // first j in [p+1, n) with gap > win
    while (a < b) {
      const uint32_t m = a + ((b - a) >> 1);
      if (skeys[static_cast<size_t>(m) * NK] - kp <= win)
        a = m + 1;
      else
        b = m;
    }
    cnt = a - p - 1;
    ex = a < n;
  }
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(kFull, cnt, o);
  ex = __reduce_add_sync(kFull, ex);
  if ((threadIdx.x & 31) == 0) {
    if (cnt) atomicAdd(pairs, cnt);
    if (ex) atomicAdd(exits, static_cast<unsigned long long>(ex));
  }
}

int blocks_for(uint64_t n, int per) { return static_cast<int>((n + per - 1) / per); }

template <class T>
T read1(const T* dptr, cudaStream_t s) {
  T h;
  PSG_CUDA(cudaMemcpyAsync(&h, dptr, sizeof(T), cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaStreamSynchronize(s));
  return h;
}

// The running best lives on device as FP32 bits (atomicMin on unsigned).
float read_best(const unsigned* dptr, cudaStream_t s) {
  const unsigned bits = read1(dptr, s);
  float v;
  std::memcpy(&v, &bits, 4);
  return v;
}

void part_range(uint64_t n, uint64_t part, uint64_t nparts, uint32_t* lo, uint32_t* hi) {
  *lo = static_cast<uint32_t>(n * part / nparts);
  *hi = static_cast<uint32_t>(n * (part + 1) / nparts);
}

// ---------------------------------------------------------------------------
// Device-side solve state (DevState): initialised, filled and read back once.
__global__ void k_state_init(DevState* st, ExactSrc src, const uint32_t* sidx, Budget bud) {
  st->bud = bud;
  st->pre_ticket = 0;
  st->ic.src = src;
  st->ic.sidx = sidx;
  st->ic.best128 = st->best128;
  st->ic.examined = &st->examined;
  st->ic.inline_n = &st->inline_n;
  st->norm2_bits = 0;
  st->best = 0x7f800000u;  // +inf
  st->cand_n = 0;
  st->best64 = ~0ull;
  st->lex = ~0ull;
  st->best128[0] = st->best128[1] = ~0ull;
  st->examined = st->evals = st->visited = st->inline_n = 0;
}


// ---------------------------------------------------------------------------
// The grid's key box and cell width before the projection runs (so the
// projection can count cells): kPreBlocks x 8 warps project a hashed sample of
// kPreRows rows on CUDA cores (warp per row, lanes over coordinates; a
// tuning input only, so any summation order), reduce per-key moments, and the
// last block to finish turns them into the box (mean +- box_sd sd clipped to
// the sample range) and GridParams at the occupancy width.
constexpr int kPreBlocks = 128;
constexpr uint32_t kPreRows = 1024;  // one sample row per warp: the box is a tuning input
struct PresampleArgs {
  Rows R;
  const float* Ut;  // d x nk (transposed directions)
  int ut_smem;      // Ut staged in shared memory (d * nk * 4 bytes)
  int nk, g, gbox;  // gbox: keys boxed (the dense engine may regrid on up to kMaxGridKeys)
  uint32_t n, m;
  double occupancy, box_sd, min_w;
};

__global__ void __launch_bounds__(256) k_presample(PresampleArgs a, DevState* st, GridParams* gp,
                                                   double* __restrict__ part, unsigned* __restrict__ ticket,
                                                   uint32_t* __restrict__ bctr) {
  extern __shared__ float sut[];  // U transposed (d x nk), when it fits
  __shared__ double red[8][kMaxGridKeys][4];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int d = a.R.d, nk = a.nk;
  const bool ut_smem = a.ut_smem;
  // PDL: the tensor-core projection that follows reads nothing this kernel
  // writes before its epilogue warps' own wait, so it may be scheduled now
  // (k_project_tc); any other successor waits at its top or is a plain launch
  pdl_trigger();
  if (ut_smem)
    for (int k = threadIdx.x; k < d * nk; k += blockDim.x) sut[k] = a.Ut[k];
  __syncthreads();
  const float* Ut = ut_smem ? sut : a.Ut;
  double s1[kMaxGridKeys], s2[kMaxGridKeys];
  float mn[kMaxGridKeys], mx[kMaxGridKeys];
#pragma unroll
  for (int t = 0; t < kMaxGridKeys; ++t) {
    s1[t] = s2[t] = 0.0;
    mn[t] = INFINITY;
    mx[t] = -INFINITY;
  }
  constexpr int kRows = 1;  // sample rows per warp step (kPreRows = one per warp)
  const uint32_t gw = blockIdx.x * 8 + warp, nw = gridDim.x * 8;
  for (uint32_t k0 = gw * kRows; k0 < a.m; k0 += nw * kRows) {
    uint32_t i[kRows];
#pragma unroll
    for (int r = 0; r < kRows; ++r)  // a bijective 32-bit hash scaled to [0, n): no aliasing with
      i[r] = __umulhi((k0 + r) * 2654435761u + 12345u, a.n);  // index-periodic structure
    float acc[kRows][kMaxGridKeys];
#pragma unroll
    for (int r = 0; r < kRows; ++r)
#pragma unroll
      for (int t = 0; t < kMaxGridKeys; ++t) acc[r][t] = 0.f;
#pragma unroll 2
    for (int c = lane; c < d; c += 32) {
      float x[kRows];
#pragma unroll
      for (int r = 0; r < kRows; ++r) x[r] = k0 + r < a.m ? row_at(a.R, i[r], c) : 0.f;
#pragma unroll
      for (int t = 0; t < kMaxGridKeys; ++t) {
        if (t >= a.gbox) break;
        const float u = Ut[c * nk + t];
#pragma unroll
        for (int r = 0; r < kRows; ++r) acc[r][t] = fmaf(u, x[r], acc[r][t]);
      }
    }
#pragma unroll
    for (int r = 0; r < kRows; ++r)
#pragma unroll
      for (int t = 0; t < kMaxGridKeys; ++t) {
        float v = acc[r][t];
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
        if (t < a.gbox && k0 + r < a.m) {
          s1[t] += v;
          s2[t] = fma(static_cast<double>(v), static_cast<double>(v), s2[t]);
          mn[t] = fminf(mn[t], v);
          mx[t] = fmaxf(mx[t], v);
        }
      }
  }
  if (lane == 0)
    for (int t = 0; t < a.gbox; ++t) {
      red[warp][t][0] = s1[t];
      red[warp][t][1] = s2[t];
      red[warp][t][2] = mn[t];
      red[warp][t][3] = mx[t];
    }
  __syncthreads();
  if (threadIdx.x < a.gbox) {
    const int t = threadIdx.x;
    double q[4] = {0.0, 0.0, INFINITY, -INFINITY};
    for (int w = 0; w < 8; ++w) {
      q[0] += red[w][t][0];
      q[1] += red[w][t][1];
      q[2] = fmin(q[2], red[w][t][2]);
      q[3] = fmax(q[3], red[w][t][3]);
    }
    for (int c = 0; c < 4; ++c) part[(static_cast<size_t>(blockIdx.x) * kMaxGridKeys + t) * 4 + c] = q[c];
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  // the last block: warp t reduces key t's per-block partials (lanes over blocks)
  __shared__ double s_lo[kMaxGridKeys], s_span[kMaxGridKeys];
  if (warp < a.gbox) {
    const int t = warp;
    double q[4] = {0.0, 0.0, INFINITY, -INFINITY};
    for (uint32_t b = lane; b < gridDim.x; b += 32) {
      const double* pp = part + (static_cast<size_t>(b) * kMaxGridKeys + t) * 4;
      q[0] += pp[0];
      q[1] += pp[1];
      q[2] = fmin(q[2], pp[2]);
      q[3] = fmax(q[3], pp[3]);
    }
    for (int o = 16; o; o >>= 1) {
      q[0] += __shfl_xor_sync(kFull, q[0], o);
      q[1] += __shfl_xor_sync(kFull, q[1], o);
      q[2] = fmin(q[2], __shfl_xor_sync(kFull, q[2], o));
      q[3] = fmax(q[3], __shfl_xor_sync(kFull, q[3], o));
    }
    if (lane == 0) {
      const double mean = q[0] / a.m, sd = sqrt(fmax(q[1] / a.m - mean * mean, 0.0));
      const double lo_t = fmax(q[2], mean - a.box_sd * sd), hi_t = fmin(q[3], mean + a.box_sd * sd);
      s_lo[t] = lo_t;
      s_span[t] = fmax(hi_t - lo_t, 1e-30);
    }
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  *ticket = 0;  // ready for the next solve
  bctr[0] = bctr[1] = 0;  // the counting build's big-cell list (k_cell_count's reset)
  double lo[kMaxGridKeys] = {}, span[kMaxGridKeys] = {};
  for (int t = 0; t < a.gbox; ++t) {
    lo[t] = s_lo[t];
    span[t] = s_span[t];
  }
  for (int t = 0; t < kMaxGridKeys; ++t) {
    st->box_lo[t] = lo[t];
    st->box_span[t] = span[t];
  }
  const double w = fmax(grid_occupancy_width(a.n, a.g, span, a.occupancy), a.min_w);
  GridParams P;
  grid_params_for(P, a.g, w, lo, span);
  *gp = P;
}

// The bootstrap bound from the lower bounds k_cell_fix left per warp
// (BootLB): up to kBootEvals warps each take a chunk of the entries (one entry
// each up to 2^20 points), pick the least lower bound and evaluate that pair
// warp-parallel (coalesced row reads), rounded up past any FP32 summation
// order so the value is a valid bound (warp_eval_best); block 0 also takes the
// seed pair (0, max(zone, 1)), admissible whenever any pair is.
constexpr uint32_t kBootEvals = 4096;
__global__ void __launch_bounds__(256) k_boot_select(ScanArgs a, const float* __restrict__ wlb,
                                                     const uint2* __restrict__ wpair, uint32_t W, uint32_t nw,
                                                     uint32_t z) {
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (gw == 0 && z < a.n) {
    const float s = a.d <= kInlineD ? (lane == 0 ? thread_sqdist(a.rows, 0, z) : 0.f) : warp_sqdist(a.rows, 0, z, lane);
    if (lane == 0) atomicMin(a.best, __float_as_uint(s));
  }
  // every warp of the block reaches the block minimum below (one atomic per
  // block: per-warp atomics on one address serialise at the L2)
  const uint32_t chunk = (W + nw - 1) / nw;
  const uint32_t e0 = gw < nw ? gw * chunk : W, e1 = min(W, e0 + chunk);
  float lb = INFINITY;
  uint32_t at = 0;
  for (uint32_t e = e0 + lane; e < e1; e += 32) {
    const float x = wlb[e];
    if (x < lb) {
      lb = x;
      at = e;
    }
  }
  for (int o = 16; o; o >>= 1) {
    const float ol = __shfl_xor_sync(kFull, lb, o);
    const uint32_t oa = __shfl_xor_sync(kFull, at, o);
    if (ol < lb || (ol == lb && oa < at)) {
      lb = ol;
      at = oa;
    }
  }
  float s = INFINITY;
  if (lb < INFINITY) {
    const uint2 pr = wpair[at];
    s = 0.f;
    for (int t = lane; t < a.d; t += 32) {
      const float g = row_at(a.rows, pr.x, t) - row_at(a.rows, pr.y, t);
      s = fmaf(g, g, s);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    s = __fmul_ru(s, 1.0f + static_cast<float>(2 * a.d + 8) * 0x1.0p-24f);  // see warp_eval_best
  }
  __shared__ float wmin[8];
  if (lane == 0) wmin[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = wmin[0];
    for (int w = 1; w < 8; ++w) m = fminf(m, wmin[w]);
    if (m < INFINITY) atomicMin(a.best, __float_as_uint(m));
  }
}

}  // namespace

// ===========================================================================
void check_reference_args(uint64_t n, uint64_t q, double f) {
  // build_reference_set validation order (refscan.cpp:33-35)
  if (q == 0) throw invalid_argument("reference count must be positive");
  if (q > n) throw invalid_argument("reference count exceeds point count");
  if (!(f > 0.0) || !std::isfinite(f)) throw invalid_argument("projection factor must be positive");
}

bool project_async(const psg_pointset& ps, const Directions& dir, float* keys, unsigned* norm2_bits,
                   cudaStream_t s, const CellCount& cc) {
  const uint32_t n = static_cast<uint32_t>(ps.n);
  const int d = ps.d;
  bool counted = cc.gp != nullptr;
  if (!ps.X) {
    project_windows(ps, dir, keys, norm2_bits, s, cc);  // virtual window rows (Rows)
  } else if (tc_projection(d, ps.n)) {
    project_tc(ps, dir, keys, norm2_bits, s, cc);  // psg_project_tc.cu
  } else if (d < 32) {
    USmall u{};
    for (int k = 0; k < dir.nk; ++k)
      for (int t = 0; t < d; ++t) u.u[k][t] = dir.U[static_cast<size_t>(k) * d + t];
    if (dir.nk == 4)
      k_project_small<4><<<blocks_for(n, 256), 256, 0, s>>>(ps.X, n, d, u, keys, norm2_bits, cc);
    else
      k_project_small<8><<<blocks_for(n, 256), 256, 0, s>>>(ps.X, n, d, u, keys, norm2_bits, cc);
  } else {
    counted = false;
    // irregular d: thread per row, U staged in shared memory (not graph-safe:
    // solve_graph skips these)
    DevBuf<float> U(dir.U.size(), s);  // freed stream-ordered after the launch
    PSG_CUDA(cudaMemcpyAsync(U.p, dir.U.data(), dir.U.size() * sizeof(float), cudaMemcpyHostToDevice, s));
    const size_t ubytes = static_cast<size_t>(dir.nk) * d * sizeof(float);
    const int smem_ok = ubytes <= 48 * 1024;
    if (dir.nk == 4)
      k_project_thread<4><<<blocks_for(n, 256), 256, smem_ok ? ubytes : 0, s>>>(ps.X, n, d, U.p, keys, norm2_bits,
                                                                               smem_ok);
    else
      k_project_thread<8><<<blocks_for(n, 256), 256, smem_ok ? ubytes : 0, s>>>(ps.X, n, d, U.p, keys, norm2_bits,
                                                                               smem_ok);
  }
  PSG_LAUNCHED();
  ++g_launches;
  return counted;
}

// Window sets: U transposed (d x nk), kept on the point set and uploaded
// when the directions change (solve_graph primes it before a capture, so a
// captured solve holds no host buffer).
const float* window_directions(const psg_pointset& ps, const Directions& dir, cudaStream_t s) {
  if (ps.win_ut.p && ps.win_ut_seed == dir.seed && ps.win_ut_q == dir.q) return ps.win_ut.p;  // same (seed, q)
  const int d = ps.d, nk = dir.nk;
  std::vector<float> ut(static_cast<size_t>(d) * nk);
  for (int k = 0; k < nk; ++k)
    for (int t = 0; t < d; ++t) ut[static_cast<size_t>(t) * nk + k] = dir.U[static_cast<size_t>(k) * d + t];
  if (g_capturing) throw std::runtime_error("window directions changed inside a graph capture");
  ps.win_ut_host = std::move(ut);
  ps.win_ut.alloc(ps.win_ut_host.size(), s);
  PSG_CUDA(cudaMemcpyAsync(ps.win_ut.p, ps.win_ut_host.data(), ps.win_ut_host.size() * 4, cudaMemcpyHostToDevice, s));
  ps.win_ut_seed = dir.seed;
  ps.win_ut_q = dir.q;
  return ps.win_ut.p;
}

void project_windows(const psg_pointset& ps, const Directions& dir, float* keys, unsigned* norm2_bits,
                     cudaStream_t s, const CellCount& cc) {
  const uint32_t n = static_cast<uint32_t>(ps.n);
  const int d = ps.d, nk = dir.nk;
  const float* Ut = window_directions(ps, dir, s);
  const size_t ubytes = static_cast<size_t>(d) * nk * 4,
               sbytes = (static_cast<size_t>(kWinRows) * kWinW + d + kWinW) * 4;
  constexpr size_t kMaxSmem = 200 * 1024;
  const int u_smem = ubytes <= kMaxSmem - std::min(sbytes, kMaxSmem / 2) ? 1 : 0;
  const int seg_smem = (u_smem ? ubytes : 0) + sbytes <= kMaxSmem ? 1 : 0;
  const size_t smem = (u_smem ? ubytes : 0) + (seg_smem ? sbytes : 0);
  if (nk == 4) {
    if (smem > 48 * 1024)
      PSG_CUDA(cudaFuncSetAttribute(k_project_windows<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    k_project_windows<4><<<blocks_for(n, kWinRows * kWinW), kWinRows, smem, s>>>(ps.rows(), n, Ut, keys, u_smem,
                                                                                  seg_smem, cc);
  } else {
    if (smem > 48 * 1024)
      PSG_CUDA(cudaFuncSetAttribute(k_project_windows<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    k_project_windows<8><<<blocks_for(n, kWinRows * kWinW), kWinRows, smem, s>>>(ps.rows(), n, Ut, keys, u_smem,
                                                                                  seg_smem, cc);
  }
}

float project(const psg_pointset& ps, const Directions& dir, float* keys, cudaStream_t s) {
  DevBuf<unsigned> nb(1, s);
  PSG_CUDA(cudaMemsetAsync(nb.p, 0, 4, s));
  KernelSpan span(s);
  project_async(ps, dir, keys, nb.p, s);
  g_prof.project_kernel_ms += span.stop();
  const unsigned bits = read1(nb.p, s);
  float v;
  std::memcpy(&v, &bits, 4);
  return v;
}

Budget make_budget(const psg_pointset& ps, const Directions& dir, float max_norm2) {
  const double u = 0x1.0p-24;
  const int d = ps.d;
  Budget b;
  b.e = (d + 4) * u * 1.01;
  b.a = (2.0 * d + 2.0) * 0x1.0p-149;
  const double maxnorm = std::sqrt(static_cast<double>(max_norm2) * (1.0 + (d + 4) * u)) * (1.0 + 1e-7);
  const bool tc = tc_projection(d, ps.n) && ps.X;
  b.E = key_gamma(d, tc) * dir.unorm * maxnorm * 1.0001 + key_abs(d, tc);
  b.Rn = ps.Rn;
  b.sigma = dir.sigma;
  b.unorm = dir.unorm;
  b.gamma64 = (d + 2) * 0x1.0p-53 * 1.01;
  b.nk = dir.nk;
  return b;
}

void CppWork::drop_graph() {
  if (gexec) cudaGraphExecDestroy(gexec);
  gexec = nullptr;
}

CppWork::~CppWork() {
  pinned_small_put(host_st);
  if (gexec) cudaGraphExecDestroy(gexec);
  for (cudaEvent_t e : gev)
    if (e) cudaEventDestroy(e);
}

namespace {

std::shared_ptr<CppWork> get_work(psg_pointset* ps, int nk, cudaStream_t s) {
  std::shared_ptr<void>& slot = ps->cpp_work[nk == 8 ? 1 : 0];
  std::shared_ptr<CppWork> w = std::static_pointer_cast<CppWork>(slot);
  if (!w) {
    w = std::make_shared<CppWork>();
    w->n = static_cast<uint32_t>(ps->n);
    w->nk = nk;
    w->keys.alloc(ps->n * nk, s);
    w->st.alloc(1, s);
    w->pre_part.alloc(kPreBlocks * kMaxGridKeys * 4, s);  // not inside a graph capture
    static_assert(sizeof(DevState) <= kPinnedSmall, "DevState mirror outgrew the pinned pool's blocks");
    w->host_st = static_cast<DevState*>(pinned_small_get());
    slot = w;
  }
  return w;
}

// One synchronisation: DevState (and the grid parameters) back to the host.
void read_state(CppPlan& plan, cudaStream_t s) {
  CppWork& W = *plan.work;
  PSG_CUDA(cudaMemcpyAsync(W.host_st, W.st.p, sizeof(DevState), cudaMemcpyDeviceToHost, s));
  if (plan.grid) PSG_CUDA(cudaMemcpyAsync(&plan.gp, W.gi.gp.p, sizeof(GridParams), cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaStreamSynchronize(s));
  plan.bud = W.host_st->bud;
}

float bits_to_float(unsigned b) {
  float v;
  std::memcpy(&v, &b, 4);
  return v;
}

ScanArgs make_args(CppPlan& plan) {
  CppWork& W = *plan.work;
  ScanArgs a{};
  a.rows = plan.ps->rows();
  a.skeys = plan.grid ? W.gi.skeys.p : W.wskeys.p;
  a.sidx = plan.grid ? W.gi.sidx.p : W.wsidx.p;
  a.n = static_cast<uint32_t>(plan.ps->n);
  a.d = plan.ps->d;
  a.zone = plan.zone;
  DevState* st = W.st.p;
  a.bud = &st->bud;
  a.best = &st->best;
  a.cand_p = W.cand_p.p;
  a.cand_j = W.cand_j.p;
  a.cand_s = W.cand_s.p;
  a.cand_n = &st->cand_n;
  a.cand_cap = W.cand_cap;
  a.ic = &st->ic;
  a.evals = &st->evals;
  a.visited = &st->visited;
  a.no_ub = std::getenv("PSG_NO_UB") != nullptr;
  return a;
}

uint64_t window_pairs(CppPlan& plan, uint32_t lo, uint32_t hi, float win, uint64_t* exits, cudaStream_t s) {
  CppWork& W = *plan.work;
  DevBuf<unsigned long long> acc(2, s);
  PSG_CUDA(cudaMemsetAsync(acc.p, 0, 16, s));
  if (hi > lo) {
    if (plan.dir.nk == 4)
      k_window_stats<4><<<blocks_for(hi - lo, 256), 256, 0, s>>>(W.wskeys.p, W.n, lo, hi, win, acc.p, acc.p + 1);
    else
      k_window_stats<8><<<blocks_for(hi - lo, 256), 256, 0, s>>>(W.wskeys.p, W.n, lo, hi, win, acc.p, acc.p + 1);
    PSG_LAUNCHED();
    ++g_launches;
  }
  unsigned long long h[2];
  PSG_CUDA(cudaMemcpyAsync(h, acc.p, 16, cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaStreamSynchronize(s));
  if (exits) *exits = h[1];
  return h[0];
}

}  // namespace

CppPlan* cpp_plan_create(psg_pointset* ps, uint64_t q, double f, uint64_t seed, uint64_t zone, bool sharded) {
  const uint64_t n = ps->n;
  if (n < 2) throw invalid_argument("closest_pair needs at least 2 points");  // refscan.cpp:70
  check_reference_args(n, q, f);
  if (n >= 0xffffffffull) throw invalid_argument("point count exceeds 2^32-1");
  if (admissible_pairs(n, zone) == 0) throw invalid_argument("no admissible pair");  // refscan.cpp:129
  Ctx& c = ctx();
  cudaStream_t s = c.stream;
  auto plan = std::make_unique<CppPlan>();
  plan->ps = ps;
  plan->zone = zone;
  plan->q_arg = q;
  plan->seed_arg = seed;
  plan->sharded = sharded;
  plan->dir = make_directions(seed, ps->d, static_cast<int>(std::min<uint64_t>(q, 1u << 20)));
  const int nk = plan->dir.nk;
  plan->work = get_work(ps, nk, s);
  CppWork& W = *plan->work;
  trace("plan: workspace");
  const char* eng = std::getenv("PSG_ENGINE");
  plan->grid = plan->dir.q >= 2 && !(eng && std::string(eng) == "window");
  plan->g = plan->grid ? std::min(3, plan->dir.q) : 0;
  plan->prep_tm = std::make_unique<StageTimer>(s);
  StageTimer& tm = *plan->prep_tm;
  // every buffer the kernels see is allocated before the state that points into them
  if (plan->grid) {
    W.gi.ensure(static_cast<uint32_t>(n), nk, s);
  } else if (W.wsidx.n != n) {
    W.wskeys.alloc(n * nk, s);
    W.wsidx.alloc(n, s);
    W.wk0.alloc(n, s);
    W.wk1.alloc(n, s);
    W.wv0.alloc(n, s);
    W.wv1.alloc(n, s);
    W.whist.alloc(radix_hist_words(n), s);
  }
  // the error budget is a property of the point set and the directions: host
  plan->bud = make_budget(*ps, plan->dir, ps->norm2max);
  trace_sync("plan: buffers + budget", s);
  k_state_init<<<1, 1, 0, s>>>(W.st.p, ps->exact(), plan->grid ? W.gi.sidx.p : W.wsidx.p, plan->bud);
  PSG_LAUNCHED();
  {
    static const double occ_env = std::getenv("PSG_OCC") ? std::atof(std::getenv("PSG_OCC")) : 0.0;
    const bool windows = ps->kind == kWindowsZ || ps->kind == kWindowsRaw;
    const double occupancy = occ_env > 0.0 ? occ_env : windows ? kGridOccupancyWindows : kGridOccupancy;
    static const double box_sd = std::getenv("PSG_BOXSD") ? std::atof(std::getenv("PSG_BOXSD")) : kGridBoxSd;
    // Learned hints (a width, the engine, the bootstrap mode) come from this
    // process's earlier solves; a sharded plan must not use them: every rank
    // has to build the same grid, whatever each rank solved before.
    const bool hints = !sharded && W.learned_q == q && W.learned_seed == seed && W.learned_zone == zone;
    const double min_w = hints ? W.learned_w : 0.0;
    // a width learned on dense data makes big cells: the radix build then
    const bool counting = plan->grid && !(min_w > 0.0 && W.learned_dense);
    CellCount cc{};
    if (plan->grid) {
      // K2 (grid) set-up before K1: the key box from a projected sample and the
      // cell width, on device, so the projection can count the cells
      const size_t ut_bytes = static_cast<size_t>(ps->d) * nk * 4;
      const int ut_smem = ut_bytes <= 32 * 1024;
      PresampleArgs pa{ps->rows(), window_directions(*ps, plan->dir, s), ut_smem, nk, plan->g,
                       std::min(plan->dir.q, kMaxGridKeys), static_cast<uint32_t>(n),
                       static_cast<uint32_t>(std::min<uint64_t>(n, kPreRows)), occupancy, box_sd, min_w};
      k_presample<<<kPreBlocks, 256, ut_smem ? ut_bytes : 0, s>>>(pa, W.st.p, W.gi.gp.p, W.pre_part.p,
                                                                  &W.st.p->pre_ticket, W.gi.bctr.p);
      PSG_LAUNCHED();
      ++g_launches;
      static const bool no_fuse = std::getenv("PSG_NO_FUSED_COUNT") != nullptr;  // A/B
      if (counting && !no_fuse) cc = CellCount{W.gi.gp.p, W.gi.cnt.p, W.gi.cid0.p};
    }
    tm.mark("presample");
    trace_sync("plan: presample", s);
    plan->proj_span = std::make_unique<KernelSpan>(s, "project");
    const bool counted = project_async(*ps, plan->dir, W.keys.p, &W.st.p->norm2_bits, s, cc);
    plan->proj_span->end();
    tm.mark("project");
    trace_sync("plan: project", s);
    if (plan->grid) {
      // K2 (grid): cells over the first g keys at the occupancy width, sorted;
      // the counting build also leaves the bootstrap's lower bounds (BootLB)
      const BootLB boot{W.keys.p, W.gi.wlb.p, W.gi.wpair.p, zone};
      build_grid(W.keys.p, static_cast<uint32_t>(n), nk, W.gi, 24, s, counting, 0, counted, counting ? &boot : nullptr);
      static const bool old_boot = std::getenv("PSG_OLD_BOOT") != nullptr;  // A/B: the standalone bootstrap
      plan->boot_lb = counting && !old_boot;
      g_launches += 3;
      tm.mark("grid");
    } else {
      // K2 (window): sort by key 0 (stable, index payload)
      if (nk == 4)
        k_sort_keys<4><<<blocks_for(n, 256), 256, 0, s>>>(W.keys.p, static_cast<uint32_t>(n), W.wk0.p, W.wv0.p);
      else
        k_sort_keys<8><<<blocks_for(n, 256), 256, 0, s>>>(W.keys.p, static_cast<uint32_t>(n), W.wk0.p, W.wv0.p);
      PSG_LAUNCHED();
      uint32_t* kk[2] = {W.wk0.p, W.wk1.p};
      uint32_t* vv[2] = {W.wv0.p, W.wv1.p};
      const int which = radix_sort<uint32_t>(kk, vv, n, 0, 32, W.whist.p, s);
      if (nk == 4)
        k_gather<4><<<blocks_for(n, 256), 256, 0, s>>>(W.keys.p, vv[which], static_cast<uint32_t>(n), W.wskeys.p,
                                                       W.wsidx.p);
      else
        k_gather<8><<<blocks_for(n, 256), 256, 0, s>>>(W.keys.p, vv[which], static_cast<uint32_t>(n), W.wskeys.p,
                                                       W.wsidx.p);
      PSG_LAUNCHED();
      g_launches += 16;
      tm.mark("sort");
    }
    trace("plan: enqueued");  // timings are collected at the bootstrap's synchronisation
  }
  return plan.release();
}

namespace {
// Stage/kernel times of plan_create and the bootstrap, read once the stream
// has synchronised.
void collect_prep(CppPlan& plan) {
  if (plan.proj_span) g_prof.project_kernel_ms += plan.proj_span->ms();
  if (plan.boot_span) g_prof.bootstrap_kernel_ms += plan.boot_span->ms();
  if (plan.prep_tm) prof_stages(*plan.prep_tm);
  plan.proj_span.reset();
  plan.boot_span.reset();
  plan.prep_tm.reset();
}
}  // namespace

// Tuning hints learned by a solve hold for its (q, seed, zone) on this point
// set: switching to another triple drops them.
void learn_for(CppWork& W, const CppPlan& plan) {
  if (W.learned_q != plan.q_arg || W.learned_seed != plan.seed_arg || W.learned_zone != plan.zone) {
    W.learned_w = 0.0;
    W.learned_dense = false;
    W.learned_full_boot = false;
    W.learned_brute = false;
  }
  W.learned_q = plan.q_arg;
  W.learned_seed = plan.seed_arg;
  W.learned_zone = plan.zone;
}

// The bootstrap over every position's whole forward 3^g stencil (at most
// kGridBootCap candidates each, a uniform stride beyond): the rescue when the
// own-row bound is too wide for the cells.
void launch_full_bootstrap(CppPlan& plan, cudaStream_t s) {
  ScanArgs a = make_args(plan);
  const uint32_t n = static_cast<uint32_t>(plan.ps->n);
  if (plan.dir.nk == 4)
    k_grid_bootstrap<4><<<blocks_for(n, kThreads), kThreads, 0, s>>>(a, plan.work->gi.dev, 0, n, kGridBootCap, 0);
  else
    k_grid_bootstrap<8><<<blocks_for(n, kThreads), kThreads, 0, s>>>(a, plan.work->gi.dev, 0, n, kGridBootCap, 0);
  PSG_LAUNCHED();
  ++g_launches;
}

float cpp_plan_bootstrap(CppPlan& plan, uint64_t part, uint64_t nparts) {
  Ctx& c = ctx();
  cudaStream_t s = c.stream;
  uint32_t lo, hi;
  part_range(plan.ps->n, part, nparts, &lo, &hi);
  ScanArgs a = make_args(plan);
  StageTimer tm(s);
  const uint32_t z = static_cast<uint32_t>(std::max<uint64_t>(plan.zone, 1));
  if (plan.grid && plan.boot_lb) {
    // the lower bounds the grid build left (BootLB): the best of them
    // evaluated exactly, plus the seed pair — one small kernel; the same global
    // bound on every rank of a sharded solve (every rank built the same grid)
    plan.boot_span = std::make_unique<KernelSpan>(s, "bootstrap");
    const uint32_t nwarps = static_cast<uint32_t>((plan.ps->n + 255) / 256 * 8);
    static const uint32_t evals =
        std::getenv("PSG_BOOT_EVALS") ? static_cast<uint32_t>(std::atoi(std::getenv("PSG_BOOT_EVALS"))) : kBootEvals;
    const uint32_t nw = std::max(1u, std::min(nwarps, evals));
    k_boot_select<<<(nw + 7) / 8, 256, 0, s>>>(a, plan.work->gi.wlb.p, plan.work->gi.wpair.p, nwarps, nw, z);
    PSG_LAUNCHED();
    ++g_launches;
    const CppWork& W = *plan.work;
    if (!plan.sharded && W.learned_full_boot && W.learned_q == plan.q_arg && W.learned_seed == plan.seed_arg &&
        W.learned_zone == plan.zone)
      launch_full_bootstrap(plan, s);  // this (q, seed, zone) needed the whole stencil before
    plan.boot_span->end();
    tm.mark("bootstrap");
    if (!plan.sync_bootstrap) return INFINITY;
    read_state(plan, s);
    collect_prep(plan);
    return bits_to_float(plan.work->host_st->best);
  }
  if (z < plan.ps->n) {
    k_seed_pair<<<1, 32, 0, s>>>(a, z);
    PSG_LAUNCHED();
    ++g_launches;
  }
  if (plan.grid) {
    plan.boot_span = std::make_unique<KernelSpan>(s);
    if (hi > lo) {
      if (plan.dir.nk == 4)
        k_grid_bootstrap<4><<<blocks_for(hi - lo, kThreads), kThreads, 0, s>>>(a, plan.work->gi.dev, lo, hi,
                                                                             kGridBootCap, boot_own_row());
      else
        k_grid_bootstrap<8><<<blocks_for(hi - lo, kThreads), kThreads, 0, s>>>(a, plan.work->gi.dev, lo, hi,
                                                                             kGridBootCap, boot_own_row());
      PSG_LAUNCHED();
      ++g_launches;
    }
    plan.boot_span->end();
    if (!plan.sync_bootstrap) return INFINITY;  // single-part solve: no host round trip here
    read_state(plan, s);  // synchronises the stream
    collect_prep(plan);
    trace("bootstrap: done");
    return bits_to_float(plan.work->host_st->best);
  }
  // Window engine.  Adaptive width: widen while the window the bound implies
  // is far more work than the bootstrap that produced it.
  PSG_CUDA(cudaStreamSynchronize(s));  // the plan's stage events
  collect_prep(plan);
  uint32_t width = 1024;
  for (int round = 0; round < 4; ++round) {
    if (hi > lo) {
      KernelSpan ks(s);
      if (plan.dir.nk == 4)
        k_bootstrap<4><<<blocks_for(hi - lo, kThreads), kThreads, 0, s>>>(a, lo, hi, width);
      else
        k_bootstrap<8><<<blocks_for(hi - lo, kThreads), kThreads, 0, s>>>(a, lo, hi, width);
      PSG_LAUNCHED();
      ++g_launches;
      g_prof.bootstrap_kernel_ms += ks.stop();
    }
    const float b = read_best(a.best, s);
    const Thresholds th = budget_thresholds_s32(plan.bud, b);
    const uint64_t est = window_pairs(plan, lo, hi, th.win, nullptr, s);
    if (est <= 8ull * (hi - lo) * width || width >= 16384) break;
    width *= 4;
  }
  plan.width = width;
  tm.mark("bootstrap");
  PSG_CUDA(cudaStreamSynchronize(s));
  prof_stages(tm);
  g_prof.bootstrap_width = width;
  return read_best(a.best, s);
}

namespace {

constexpr uint32_t kCandMax = 1u << 24;  // list capacity ceiling; band pairs past it are evaluated inline

void ensure_candidates(CppWork& W, cudaStream_t s) {
  if (W.cand_cap == 0) W.cand_cap = 1u << 16;
  if (W.cand_p.n < W.cand_cap) {
    W.drop_graph();  // a captured solve holds the old buffers
    W.cand_p.alloc(W.cand_cap, s);
    W.cand_j.alloc(W.cand_cap, s);
    W.cand_s.alloc(W.cand_cap, s);
    W.d64.alloc(W.cand_cap, s);
  }
}

// After a scan whose band held more pairs than the list: the answer is still
// exact (record() evaluated the rest inline), but later solves on this point
// set get a longer list, so the bulk of their band goes through the
// deterministic recheck again.
void grow_after_overflow(CppWork& W, const DevState& h) {
  if (h.cand_n > W.cand_cap && W.cand_cap < kCandMax)
    W.cand_cap = static_cast<uint32_t>(std::min<unsigned long long>(h.cand_n * 2, kCandMax));
}

// One scan attempt, enqueued only (no host synchronisation): reset, grid
// check, candidate scan, spill-list evaluation, speculative FP64 recheck
// (correct whenever nothing overflowed; the caller checks), pick, and the
// state copy to the pinned host mirror.  Returns the scan kernel's span.
KernelSpan* scan_enqueue(CppPlan& plan, uint32_t lo, uint32_t hi, uint32_t part, uint32_t nparts, cudaStream_t s) {
  Ctx& c = ctx();
  CppWork& W = *plan.work;
  DevState* st = W.st.p;
  ScanArgs a = make_args(plan);
  // Reset, and (grid) the check that the cells hold every pair whose key gaps
  // are within the window of the bound — decided on device from the bound
  // every rank shares.
  StageTimer tm(s, g_capturing);  // stage marks inside a captured solve (replays report them)
  k_scan_prepare<<<1, 1, 0, s>>>(st, plan.grid ? W.gi.gp.p : nullptr);
  PSG_LAUNCHED();
  tm.mark("prepare");
  KernelSpan* span = new KernelSpan(s, "scan");
  if (plan.grid && plan.dense) {
    // dense cells: cell-pair tiles (the caller decided after the grid check
    // passed on the host, so the cells are wide enough for the bound)
    unsigned regrid = 0;
    PSG_CUDA(cudaMemcpyAsync(&regrid, &st->regrid, 4, cudaMemcpyDeviceToHost, s));
    PSG_CUDA(cudaStreamSynchronize(s));
    if (!regrid)
      dense_scan(a, W.gi, plan.gp.cells, plan.ps->rows(), static_cast<uint32_t>(plan.ps->n), plan.ps->d, plan.dir.nk,
                 &st->th, W.dense, part, nparts, s);
  } else if (hi > lo) {
    const unsigned nb = blocks_for(hi - lo, kThreads);
    const int v = (plan.grid ? 4 : 0) + (plan.dir.nk == 8 ? 2 : 0) + (plan.exact_scan ? 1 : 0);
    switch (v) {
      case 0: k_scan<4, false><<<nb, kThreads, 0, s>>>(a, lo, hi); break;
      case 1: k_scan<4, true><<<nb, kThreads, 0, s>>>(a, lo, hi); break;
      case 2: k_scan<8, false><<<nb, kThreads, 0, s>>>(a, lo, hi); break;
      case 3: k_scan<8, true><<<nb, kThreads, 0, s>>>(a, lo, hi); break;
      case 4: k_grid_scan2<4, false><<<nb, kThreads, 0, s>>>(a, W.gi.dev, lo, hi, &st->regrid, &st->th); break;
      case 5: k_grid_scan2<4, true><<<nb, kThreads, 0, s>>>(a, W.gi.dev, lo, hi, &st->regrid, &st->th); break;
      case 6: k_grid_scan2<8, false><<<nb, kThreads, 0, s>>>(a, W.gi.dev, lo, hi, &st->regrid, &st->th); break;
      default: k_grid_scan2<8, true><<<nb, kThreads, 0, s>>>(a, W.gi.dev, lo, hi, &st->regrid, &st->th); break;
    }
    PSG_LAUNCHED();
    ++g_prof.scan_launches;
  }
  span->end();
  tm.mark("scan");
  const ExactSrc ex = plan.ps->exact();
  const int nb = c.sm_count * 2;
  const bool wide = plan.ps->d >= 32;  // a warp per candidate (k_recheck)
  const int v = (plan.grid ? 0 : 4) + (plan.dir.nk == 8 ? 2 : 0) + (wide ? 1 : 0);
  switch (v) {
    case 0: k_recheck<4, false, false><<<nb, 256, 0, s>>>(a, ex, W.d64.p, &st->best64, &st->examined); break;
    case 1: k_recheck<4, false, true><<<nb, 256, 0, s>>>(a, ex, W.d64.p, &st->best64, &st->examined); break;
    case 2: k_recheck<8, false, false><<<nb, 256, 0, s>>>(a, ex, W.d64.p, &st->best64, &st->examined); break;
    case 3: k_recheck<8, false, true><<<nb, 256, 0, s>>>(a, ex, W.d64.p, &st->best64, &st->examined); break;
    case 4: k_recheck<4, true, false><<<nb, 256, 0, s>>>(a, ex, W.d64.p, &st->best64, &st->examined); break;
    case 5: k_recheck<4, true, true><<<nb, 256, 0, s>>>(a, ex, W.d64.p, &st->best64, &st->examined); break;
    case 6: k_recheck<8, true, false><<<nb, 256, 0, s>>>(a, ex, W.d64.p, &st->best64, &st->examined); break;
    default: k_recheck<8, true, true><<<nb, 256, 0, s>>>(a, ex, W.d64.p, &st->best64, &st->examined); break;
  }
  PSG_LAUNCHED();
  k_pick<<<nb, 256, 0, s>>>(a, W.d64.p, &st->best64, &st->lex);
  PSG_LAUNCHED();
  tm.mark("recheck");
  PSG_CUDA(cudaMemcpyAsync(W.host_st, st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
  g_launches += 4;
  return span;
}

psg_pair_result result_from(const DevState& h, uint64_t wp, uint64_t exits) {
  psg_pair_result r{};
  // the listed candidates' (best64, lex) against the inline 128-bit minimum
  unsigned long long hi = h.best64, lo = h.lex;
  if (h.lex == ~0ull || h.best128[1] < hi || (h.best128[1] == hi && h.best128[0] < lo)) {
    hi = h.best128[1];
    lo = h.best128[0];
  }
  if (lo == ~0ull) {
    r.index_i = r.index_j = UINT64_MAX;
    r.distance = INFINITY;
  } else {
    r.index_i = lo >> 32;
    r.index_j = lo & 0xffffffffull;
    std::memcpy(&r.distance, &hi, 8);
  }
  r.stats.pairs_examined = h.examined;
  r.stats.pairs_pruned_by_reference = wp > h.examined ? wp - h.examined : 0;
  r.stats.inner_loop_exits = exits;
  g_prof.window_pairs += wp;
  g_prof.lb_survivors += h.evals;
  g_prof.candidates += h.cand_n;
  g_prof.inline_fp64 += h.inline_n;
  return r;
}

}  // namespace

psg_pair_result cpp_plan_scan(CppPlan& plan, uint64_t part, uint64_t nparts, float bound_s32) {
  Ctx& c = ctx();
  cudaStream_t s = c.stream;
  const uint64_t n = plan.ps->n;
  CppWork& W = *plan.work;
  uint32_t lo, hi;
  part_range(n, part, nparts, &lo, &hi);
  StageTimer tm(s);
  // The bound handed in is the (global) minimum of what the bootstraps
  // returned; lower the device copy to it.
  k_min_bound<<<1, 1, 0, s>>>(&W.st.p->best, bound_s32);
  PSG_LAUNCHED();
  ++g_launches;
  KernelSpan* scan_span = nullptr;
  uint64_t last_est = 0;  // the grid's pair estimate (sparse grids)
  for (int attempt = 0;; ++attempt) {
    if (attempt > 16) throw std::runtime_error("closest_pair: the cell grid did not settle after 16 rebuilds");
    ensure_candidates(W, s);
    if (plan.grid) {
      // dense cells (clustered data): cell-pair tiles beat per-point lists
      PSG_CUDA(cudaMemcpyAsync(&plan.gp, W.gi.gp.p, sizeof(GridParams), cudaMemcpyDeviceToHost, s));
      PSG_CUDA(cudaMemcpyAsync(W.host_st, W.st.p, sizeof(DevState), cudaMemcpyDeviceToHost, s));
      // a grid over more than 3 keys is already the dense engine's (a regrid
      // of it): no estimate (it would walk the 3^g stencil of every cell)
      if (plan.g > 3) {
        PSG_CUDA(cudaStreamSynchronize(s));
        plan.dense = true;
      } else {
        const uint64_t est = grid_pair_estimate(W.gi, plan.gp.cells, s);  // synchronises
        last_est = est;
        plan.dense = est > kDenseFactor * n;
        if (std::getenv("PSG_TRACE")) {
          const DevState& h0 = *W.host_st;
          std::fprintf(stderr, "[psg] grid: g %d w %.6g cells %llu dims %u %u %u box %.4g+%.4g %.4g+%.4g %.4g+%.4g "
                       "bound %.6g est %llu dense %d learned_w %.6g\n", plan.gp.g, plan.gp.w,
                       static_cast<unsigned long long>(plan.gp.cells), plan.gp.dims[0], plan.gp.dims[1],
                       plan.gp.dims[2], h0.box_lo[0], h0.box_span[0], h0.box_lo[1], h0.box_span[1], h0.box_lo[2],
                       h0.box_span[2], static_cast<double>(bits_to_float(h0.best)),
                       static_cast<unsigned long long>(est), static_cast<int>(plan.dense), W.learned_w);
        }
      }
      // Small sets the grid cannot separate (a pair estimate over 1/64 of all
      // pairs, under ~4e9 pair-coordinates: ~0.6 ms all-pairs) go to the
      // all-pairs engine: the dense engine's set-up (pair lists, sorts, host
      // synchronisations) costs more than that (4096 x 32 Gaussian: 0.95 ->
      // 0.18 ms).  Larger ones stay on the dense engine, which beats the
      // all-pairs kernel at every d measured (tools/cmp_switch.py: 2^16 x 100
      // Gaussian 20 ms against 47 ms).  Same exact answer either way
      // (refscan.cpp:134-157 is the definition the all-pairs engine implements).
      if (nparts == 1 && plan.dense && plan.g <= 3 && !std::getenv("PSG_NO_BRUTE_SWITCH")) {
        const double all = 0.5 * static_cast<double>(n) * static_cast<double>(n - 1);
        const bool small = all * plan.ps->d < 4e9;
        if (static_cast<double>(last_est) > all / 64.0 && small) {
          trace("scan: small unseparable set -> all-pairs engine");
          learn_for(W, plan);
          W.learned_brute = true;  // later solves of this (q, seed, zone) go there directly (cpp_solve)
          delete scan_span;
          return brute_solve(plan.ps, plan.zone);
        }
      }
      if (nparts == 1 && plan.dense) {  // later solves of this (q, seed, zone) skip the graph attempt
        learn_for(W, plan);
        W.learned_dense = true;
      }
      static const int dense_keys = std::getenv("PSG_DENSE_KEYS") ? std::atoi(std::getenv("PSG_DENSE_KEYS")) : kMaxGridKeys;
      const int gd = std::min(plan.dir.q, dense_keys);
      if (plan.dense && plan.g < gd) {
        // Dense: rebuild the cells on more keys at the same width (still >=
        // the bound's key window): in 3 projected keys clusters overlap; every
        // further key divides the clusters a cell pair mixes by ~2.5 (C5:
        // 4 -> 5 -> 6 keys = 5.0e12 -> 1.9e12 -> 7.7e11 tile pairs).  Up to 8
        // keys and 2^27 cells (the table is a 512 MiB radix-sorted grid).
        grid_params_for(plan.gp, gd, plan.gp.w, W.host_st->box_lo, W.host_st->box_span, kMaxDenseCells);
        PSG_CUDA(cudaMemcpyAsync(W.gi.gp.p, &plan.gp, sizeof(GridParams), cudaMemcpyHostToDevice, s));
        build_grid(W.keys.p, static_cast<uint32_t>(n), plan.dir.nk, W.gi, 24, s, /*counting=*/false,
                   plan.gp.cells);  // large cells
        plan.g = gd;
        tm.mark("dense grid");
      }
    }
    delete scan_span;
    scan_span = scan_enqueue(plan, lo, hi, static_cast<uint32_t>(part), static_cast<uint32_t>(nparts), s);
    PSG_CUDA(cudaStreamSynchronize(s));
    plan.bud = W.host_st->bud;
    if (plan.grid) PSG_CUDA(cudaMemcpy(&plan.gp, W.gi.gp.p, sizeof(GridParams), cudaMemcpyDeviceToHost));
    collect_prep(plan);
    const DevState& h = *W.host_st;
    if (plan.grid && h.regrid && !plan.rescued && plan.g <= 3) {
      // The bootstrap looked at each point's own cell row only; before
      // widening the cells, try the whole 3^g stencil on these cells (a
      // near pair split across a row boundary: e.g. a motif whose windows
      // straddle a cell face).  Over all positions, so every rank of a
      // sharded solve derives the same bound; later solves of this (q, seed,
      // zone) run it up front (learned_full_boot).
      plan.rescued = true;
      launch_full_bootstrap(plan, s);
      if (nparts == 1) {
        learn_for(W, plan);
        W.learned_full_boot = true;
        W.drop_graph();  // recaptured with the full bootstrap
      }
      continue;  // k_scan_prepare checks the cells again against the new bound
    }
    if (plan.grid && h.regrid) {
      // Widen the cells to the key window of the bound the check saw and
      // rebuild.  Single part: the wider cells hold far better partners, so
      // re-bootstrap on them and shrink again while the bound keeps falling
      // (clustered data: the occupancy grid's bootstrap bound is poor).
      float bound = bits_to_float(h.check_best);
      for (int round = 0; round < 4; ++round) {
        const double need =
            static_cast<double>(budget_thresholds_s32(plan.bud, bound).win) * (1.0 + 2e-5);
        if (!(need < 1e300)) throw std::runtime_error("closest_pair: no finite bound before the scan");
        const bool dense_grid = plan.g > 3;  // the dense engine's grid (more keys, radix-sorted, up to 2^27 cells)
        grid_params_for(plan.gp, plan.g, need, h.box_lo, h.box_span, dense_grid ? kMaxDenseCells : kMaxCells);
        PSG_CUDA(cudaMemcpyAsync(W.gi.gp.p, &plan.gp, sizeof(GridParams), cudaMemcpyHostToDevice, s));
        build_grid(W.keys.p, static_cast<uint32_t>(n), plan.dir.nk, W.gi, 24, s, !dense_grid,
                   dense_grid ? plan.gp.cells : 0);
        tm.mark("regrid");
        // every rank must derive the same grid from the shared bound; the
        // stencil bootstrap walks g <= 3 grids only (the dense engine's own
        // Gram tiles lower the bound as they go)
        if (nparts != 1 || dense_grid) break;
        ScanArgs a = make_args(plan);
        if (plan.dir.nk == 4)
          k_grid_bootstrap<4><<<blocks_for(n, kThreads), kThreads, 0, s>>>(a, W.gi.dev, 0, static_cast<uint32_t>(n),
                                                                           kGridBootCap, 0);
        else
          k_grid_bootstrap<8><<<blocks_for(n, kThreads), kThreads, 0, s>>>(a, W.gi.dev, 0, static_cast<uint32_t>(n),
                                                                           kGridBootCap, 0);
        PSG_LAUNCHED();
        g_launches += 1;
        const float nb = read_best(&W.st.p->best, s);
        const double next = static_cast<double>(budget_thresholds_s32(plan.bud, nb).win) * (1.0 + 2e-5);
        if (std::getenv("PSG_TRACE"))
          std::fprintf(stderr, "[psg] regrid %d: bound %.6g need %.6g cells %llu -> rebootstrap bound %.6g need %.6g\n",
                       round, static_cast<double>(bound), need, static_cast<unsigned long long>(plan.gp.cells),
                       static_cast<double>(nb), next);
        if (!(next < need / 1.25)) break;  // converged: keep these cells
        bound = nb;
      }
      if (nparts == 1) {
        // Remember the width for later solves of the same (q, seed, zone) on
        // this point set: their first grid is built at it, so the captured
        // graph solve needs no regrid (a tuning hint; every stage still runs).
        learn_for(W, plan);
        W.learned_w = plan.gp.w;
        W.drop_graph();
      }
      continue;
    }
    if (!plan.dense && !plan.exact_scan && h.cand_n > W.cand_cap) {
      // the band outgrew the list: grow it for later solves and rescan this
      // part with every band pair evaluated inline (the bound only tightened)
      grow_after_overflow(W, h);
      plan.exact_scan = true;
      continue;
    }
    grow_after_overflow(W, h);
    break;
  }
  g_prof.scan_kernel_ms += scan_span->ms();
  delete scan_span;
  tm.mark("scan+recheck");
  trace("scan+recheck: done");
  const DevState h = *W.host_st;
  uint64_t exits = 0, wp = h.visited;
  if (!plan.grid) {
    const Thresholds th = budget_thresholds_s32(plan.bud, bits_to_float(h.best));
    wp = window_pairs(plan, lo, hi, th.win, &exits, s);
    tm.mark("stats");
  }
  PSG_CUDA(cudaStreamSynchronize(s));
  prof_stages(tm);
  return result_from(h, wp, exits);
}

namespace {

psg_pair_result finalize(psg_pair_result r, uint64_t n, uint64_t zone) {
  if (r.index_i == UINT64_MAX) throw invalid_argument("no admissible pair");
  const uint64_t adm = admissible_pairs(n, zone);
  const uint64_t used = r.stats.pairs_examined + r.stats.pairs_pruned_by_reference;
  if (used > adm) r.stats.pairs_pruned_by_reference = adm - r.stats.pairs_examined;
  r.stats.pairs_skipped_by_exit = adm - r.stats.pairs_examined - r.stats.pairs_pruned_by_reference;
  return r;
}

bool graphs_enabled() {
  static const bool off = std::getenv("PSG_NO_GRAPH") != nullptr;
  return !off;
}

// The single-part grid solve as one CUDA graph: plan (projection, grid
// build), bootstrap and one scan attempt, all device-resident, ending with the
// state copy to pinned host memory.  Captured on first use per (q, seed, zone)
// and replayed afterwards: one launch per solve instead of ~30.  Returns false
// when the replay's state asks for a regrid / bigger buffers (the caller then
// runs the regular path, which handles those).
bool solve_graph(psg_pointset* ps, uint64_t q, double f, uint64_t seed, uint64_t zone, psg_pair_result* out) {
  Ctx& c = ctx();
  cudaStream_t s = c.stream;
  const Directions dir = make_directions(seed, ps->d, static_cast<int>(std::min<uint64_t>(q, 1u << 20)));
  const char* eng = std::getenv("PSG_ENGINE");
  if (dir.q < 2 || (eng && std::string(eng) == "window")) return false;
  const int d = ps->d;
  if (ps->X && !(d < 32 || d == 32 || d == 64 || d == 128 || d == 256)) return false;  // projection needs a host buffer
  std::shared_ptr<CppWork> work = get_work(ps, dir.nk, s);
  CppWork& W = *work;
  // a point set's first solve runs uncaptured (it also learns the width and
  // the engine): a graph pays off only once the set is solved again (the
  // one-shot entries build a fresh set per call)
  if (W.solves++ == 0) return false;
  if (W.learned_dense && W.learned_q == q && W.learned_seed == seed && W.learned_zone == zone) return false;
  // every allocation happens before capture (and drops a graph that holds
  // buffers it replaces)
  window_directions(*ps, dir, s);  // the presample / window projection read it
  W.gi.ensure(static_cast<uint32_t>(ps->n), dir.nk, s);
  ensure_candidates(W, s);
  if (!W.gexec || W.gq != q || W.gseed != seed || W.gzone != zone || W.gcap != W.cand_cap ||
      W.glevel != graph_profiling()) {
    W.drop_graph();
    for (cudaEvent_t& e : W.gev)
      if (!e) PSG_CUDA(cudaEventCreate(&e));
    PSG_CUDA(cudaStreamSynchronize(s));
    cudaGraph_t graph = nullptr;
    const uint64_t launches0 = g_launches;
    PSG_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    g_capturing = true;
    g_cap_ev = W.gev;
    g_cap_next = 0;
    g_cap_max = static_cast<int>(std::size(W.gev));
    g_cap_spans.clear();
    g_cap_stages.clear();
    W.glevel = graph_profiling();
    g_cap_span_marks = W.glevel >= 1;
    g_cap_stage_marks = W.glevel >= 2;
    try {
      std::unique_ptr<CppPlan> plan(cpp_plan_create(ps, q, f, seed, zone));
      plan->sync_bootstrap = false;
      cpp_plan_bootstrap(*plan, 0, 1);
      delete scan_enqueue(*plan, 0, static_cast<uint32_t>(ps->n), 0, 1, s);
    } catch (...) {
      g_capturing = false;
      g_cap_ev = nullptr;
      cudaStreamEndCapture(s, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    g_capturing = false;
    g_cap_ev = nullptr;
    PSG_CUDA(cudaStreamEndCapture(s, &graph));
    const cudaError_t ie = cudaGraphInstantiate(&W.gexec, graph, 0);
    cudaGraphDestroy(graph);
    PSG_CUDA(ie);
    W.gq = q;
    W.gseed = seed;
    W.gzone = zone;
    W.gspans = g_cap_spans;
    W.gstages = g_cap_stages;
    W.gcap = W.cand_cap;
    W.glaunches = g_launches - launches0;
    g_launches = launches0;
  }
  PSG_CUDA(cudaGraphLaunch(W.gexec, s));
  PSG_CUDA(cudaStreamSynchronize(s));
  g_launches += W.glaunches;
  const DevState h = *W.host_st;
  // cells narrower than the bound's window, or a band longer than the list:
  // the regular path rebuilds the cells / rescans exactly
  if (h.regrid || h.cand_n > W.cand_cap) {
    grow_after_overflow(W, h);
    return false;
  }
  // the captured spans and stages, read from this replay's event nodes
  for (const CapMark& m : W.gspans) {
    float ms = 0.f;
    PSG_CUDA(cudaEventElapsedTime(&ms, W.gev[m.a], W.gev[m.b]));
    const std::string nm = m.name;
    if (nm == "project") g_prof.project_kernel_ms += ms;
    else if (nm == "bootstrap") g_prof.bootstrap_kernel_ms += ms;
    else if (nm == "scan") g_prof.scan_kernel_ms += ms;
  }
  for (const CapMark& m : W.gstages) {
    if (g_prof.stages >= 16) break;
    float ms = 0.f;
    PSG_CUDA(cudaEventElapsedTime(&ms, W.gev[m.a], W.gev[m.b]));
    std::strncpy(g_prof.stage_name[g_prof.stages], m.name, 23);
    g_prof.stage_ms[g_prof.stages++] = ms;
  }
  ++g_prof.scan_launches;
  *out = result_from(h, h.visited, 0);
  return true;
}

}  // namespace

psg_pair_result cpp_solve(psg_pointset* ps, uint64_t q, double f, uint64_t seed, uint64_t zone) {
  // validation first (same order as the reference), then the graph path
  if (ps->n < 2) throw invalid_argument("closest_pair needs at least 2 points");
  check_reference_args(ps->n, q, f);
  if (admissible_pairs(ps->n, zone) == 0) throw invalid_argument("no admissible pair");
  psg_pair_result r;
  {  // a set this (q, seed, zone) already sent to the all-pairs engine (cpp_plan_scan)
    const Directions dir = make_directions(seed, ps->d, static_cast<int>(std::min<uint64_t>(q, 1u << 20)));
    const std::shared_ptr<void>& slot = ps->cpp_work[dir.nk == 8 ? 1 : 0];
    const auto* W = static_cast<const CppWork*>(slot.get());
    if (W && W->learned_brute && W->learned_q == q && W->learned_seed == seed && W->learned_zone == zone)
      return finalize(brute_solve(ps, zone), ps->n, zone);
  }
  if (graphs_enabled() && ps->n < 0xffffffffull && solve_graph(ps, q, f, seed, zone, &r))
    return finalize(r, ps->n, zone);
  std::unique_ptr<CppPlan> plan(cpp_plan_create(ps, q, f, seed, zone));
  plan->sync_bootstrap = false;  // the bound stays on device between bootstrap and scan
  const float b = cpp_plan_bootstrap(*plan, 0, 1);
  return finalize(cpp_plan_scan(*plan, 0, 1, b), ps->n, zone);
}

}  // namespace psg
