// psg_internal.cuh — shared host/device plumbing for the sm_100a pair-search
// library: error handling, stream-ordered device buffers, the per-device
// context, and the rigorous FP32 error-budget arithmetic every filter uses.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace psg {

// Mirrors the reference's std::invalid_argument contract (refscan.cpp:33-35,
// 70, 129, 136, 162-163, 214; series.cpp:9, 20-24); surfaced through the C ABI
// as PSG_ERR_INVALID with the identical message.
#ifndef PSG_INVALID_ARGUMENT_DEFINED
#define PSG_INVALID_ARGUMENT_DEFINED
struct invalid_argument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
#endif
struct cuda_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define PSG_CUDA(call)                                                                  \
  do {                                                                                  \
    cudaError_t psg_e_ = (call);                                                        \
    if (psg_e_ != cudaSuccess)                                                          \
      throw ::psg::cuda_error(std::string(#call) + ": " + cudaGetErrorString(psg_e_) + \
                              " (" __FILE__ ":" + std::to_string(__LINE__) + ")");      \
  } while (0)
// PSG_DEBUG_SYNC builds synchronise after every launch so a faulting kernel
// is named by the failing check (there is no compute-sanitizer on the pool).
#ifdef PSG_DEBUG_SYNC
#define PSG_LAUNCHED()                 \
  do {                                 \
    PSG_CUDA(cudaGetLastError());      \
    PSG_CUDA(cudaDeviceSynchronize()); \
  } while (0)
#else
#define PSG_LAUNCHED() PSG_CUDA(cudaGetLastError())
#endif

// ---------------------------------------------------------------------------
// Programmatic dependent launch (PDL).  A kernel enqueued by launch_pdl may be
// scheduled while its predecessor on the stream is still draining; it calls
// pdl_wait() before touching anything the predecessor writes (the wait also
// makes the predecessor's writes visible) and pdl_trigger() right after, so
// its own successor can be scheduled in turn.  Because every kernel triggers
// only after its wait, a kernel's pre-wait prologue may read whatever the
// kernel two back wrote.  Outside a PDL chain both are no-ops.
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// The block's maximum of v into *dst: one atomic per block, and none when
// the current value is already as large (after the first blocks it usually
// is; every warp hitting one address serialises at the L2).  Every thread
// of the block calls it.
__device__ __forceinline__ void block_max_to(unsigned* dst, unsigned v) {
  __shared__ unsigned wmax[32];
  __syncthreads();  // a previous call's readers are done with wmax
  v = __reduce_max_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    const unsigned nw = (blockDim.x + 31) >> 5;
    unsigned m = threadIdx.x < nw ? wmax[threadIdx.x] : 0u;
    m = __reduce_max_sync(0xffffffffu, m);
    if (threadIdx.x == 0 && m > *reinterpret_cast<volatile unsigned*>(dst)) atomicMax(dst, m);
  }
}

#endif
// cudaFuncAttributeMaxDynamicSharedMemorySize once per (kernel, device): the
// attribute is per device, so a process driving several GPUs sets it on each.
void set_max_dynamic_smem(const void* kernel, size_t bytes);
// Small page-locked blocks (kPinnedSmall bytes: per-workspace state mirrors)
// from a process-wide pool of portable slabs: cudaMallocHost / cudaFreeHost
// cost milliseconds per call, which a one-shot solve would pay every time.
constexpr size_t kPinnedSmall = 4096;
void* pinned_small_get();
void pinned_small_put(void* p);
bool pdl_enabled();  // PSG_NO_PDL=1: plain launches (A/B)
template <class... P, class... A>
void launch_pdl(void (*kernel)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, A&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  PSG_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<A>(args)...));
}

// ---------------------------------------------------------------------------
// Per-device context: one stream, a stream-ordered pool that keeps freed
// blocks (so repeated solves do not pay cudaMalloc), timing events.
struct Ctx {
  int device = 0;
  int sm_count = 148;
  cudaStream_t stream = nullptr;
  std::mutex mu;  // the reference is reentrant; we serialise per device
  std::vector<cudaEvent_t> events;  // pool: creating events per call costs microseconds each
  cudaEvent_t get_event() {
    if (events.empty()) {
      cudaEvent_t e;
      PSG_CUDA(cudaEventCreate(&e));
      return e;
    }
    cudaEvent_t e = events.back();
    events.pop_back();
    return e;
  }
  void put_event(cudaEvent_t e) { events.push_back(e); }
  // Two pinned staging chunks for pageable host input (h2d_staged,
  // psg_points.cu), created on first use on this device; stage_done[k] marks
  // the end of the last upload out of chunk k.
  static constexpr size_t kStageBytes = size_t(32) << 20;
  char* stage[2] = {nullptr, nullptr};
  cudaEvent_t stage_done[2] = {nullptr, nullptr};
  cudaStream_t copy_stream = nullptr;  // D2H overlapped with work on `stream` (created on first use)
};
Ctx& ctx();  // context of the current CUDA device (created on first use)

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(size_t count, cudaStream_t st) { alloc(count, st); }
  void alloc(size_t count, cudaStream_t st) {
    release();
    s = st;
    n = count;
    if (count) PSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), st));
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; n = o.n; s = o.s;
      o.p = nullptr; o.n = 0;
    }
    return *this;
  }
  size_t bytes() const { return n * sizeof(T); }
};

// True while the calling thread is capturing a CUDA graph: stage timers stay
// out of the captured work (their events are pooled and reused); KernelSpans
// take dedicated events from g_cap_ev (owned by the graph's workspace), in
// creation order, so kernel times can still be read after each replay.
extern thread_local bool g_capturing;
extern thread_local cudaEvent_t* g_cap_ev;
extern thread_local int g_cap_next, g_cap_max;
// What a capture recorded: named spans (KernelSpan) and stages (StageTimer)
// as indices into g_cap_ev, so a replay can read each one's device time.
struct CapMark {
  const char* name;
  int a, b;  // event indices
};
extern thread_local std::vector<CapMark> g_cap_spans, g_cap_stages;
// Event nodes inside a captured solve cost ~5 us of graph time each, so the
// graphs carry them only on request (psg_set_graph_profiling): level 0 none,
// 1 the named spans (project / bootstrap / scan), 2 spans and stage marks.
// PSG_GRAPH_STAGES=1 starts at level 2.
extern thread_local bool g_cap_stage_marks, g_cap_span_marks;
int graph_profiling();
void set_graph_profiling(int level);
// next capture event (external record node), or -1 when the pool is used up
inline int cap_event() { return g_cap_ev && g_cap_next < g_cap_max ? g_cap_next++ : -1; }

// Stage timer: CUDA events on the library stream; read after the final sync.
// Inside a graph capture it records external event nodes from g_cap_ev and
// logs its stages in g_cap_stages (read after each replay, solve_graph).
struct StageTimer {
  static constexpr int kMax = 16;
  cudaEvent_t ev[kMax + 1] = {};
  int cap[kMax + 1] = {};
  const char* name[kMax] = {};
  int count = 0;
  cudaStream_t s = nullptr;
  bool on = true, capture = false;
  explicit StageTimer(cudaStream_t st, bool enabled = true)
      : s(st), on(enabled && (!g_capturing || g_cap_stage_marks)), capture(g_capturing) {
    if (!on) return;
    if (capture) {
      cap[0] = cap_event();
      if (cap[0] < 0) {
        on = false;
        return;
      }
      PSG_CUDA(cudaEventRecordWithFlags(g_cap_ev[cap[0]], s, cudaEventRecordExternal));
      return;
    }
    ev[0] = ctx().get_event();
    PSG_CUDA(cudaEventRecord(ev[0], s));
  }
  void mark(const char* stage) {
    if (!on || count >= kMax) return;
    if (capture) {
      const int e = cap_event();
      if (e < 0) return;
      name[count] = stage;
      cap[++count] = e;
      PSG_CUDA(cudaEventRecordWithFlags(g_cap_ev[e], s, cudaEventRecordExternal));
      return;
    }
    name[count] = stage;
    ++count;
    ev[count] = ctx().get_event();
    PSG_CUDA(cudaEventRecord(ev[count], s));
  }
  ~StageTimer() {
    if (!on) return;
    if (capture) {
      for (int i = 0; i < count; ++i) g_cap_stages.push_back(CapMark{name[i], cap[i], cap[i + 1]});
      return;
    }
    Ctx& c = ctx();
    for (int i = 0; i <= count; ++i) c.put_event(ev[i]);
  }
};

// Host-side trace (PSG_TRACE=1): wall time since the previous mark, stderr.
void trace(const char* what);
void trace_sync(const char* what, cudaStream_t s);

// Device time of one kernel (or a short launch sequence) on a stream.  A
// named span inside a capture is logged in g_cap_spans.
struct KernelSpan {
  cudaEvent_t a = nullptr, b = nullptr;
  cudaStream_t s = nullptr;
  bool pooled = true;
  const char* name = nullptr;
  int ia = -1, ib = -1;
  explicit KernelSpan(cudaStream_t st, const char* nm = nullptr) : s(st), name(nm) {
    if (g_capturing) {
      pooled = false;
      if (!g_cap_span_marks) return;
      ia = cap_event();
      ib = cap_event();
      if (ia < 0 || ib < 0) return;
      a = g_cap_ev[ia];
      b = g_cap_ev[ib];
    } else {
      a = ctx().get_event();
      b = ctx().get_event();
    }
    record(a);
  }
  // Inside a capture, an external record is needed to become a graph node.
  void record(cudaEvent_t e) {
    PSG_CUDA(cudaEventRecordWithFlags(e, s, pooled ? cudaEventRecordDefault : cudaEventRecordExternal));
  }
  // Records the end event, waits for it, returns milliseconds.
  double stop() {
    end();
    if (!b) return 0.0;
    PSG_CUDA(cudaEventSynchronize(b));
    return ms();
  }
  // Deferred form: end() now, ms() after a later stream synchronisation.
  void end() {
    if (b) record(b);
    if (!pooled && name && b) g_cap_spans.push_back(CapMark{name, ia, ib});
  }
  double ms() const {
    if (!a || !b) return 0.0;
    float v = 0.f;
    PSG_CUDA(cudaEventElapsedTime(&v, a, b));
    return v;
  }
  ~KernelSpan() {
    if (!pooled) return;
    Ctx& c = ctx();
    if (a) c.put_event(a);
    if (b) c.put_event(b);
  }
};

// ---------------------------------------------------------------------------
// Orderable integer images of floats (radix sort keys, atomic min/max).
#ifdef __CUDACC__
// A relaxed GPU-scope load of a word other blocks update with atomics (the
// shared bound): not cached in L1, no system-scope ordering cost.
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
#endif

__host__ __device__ __forceinline__ uint32_t f32_order(float f) {
#ifdef __CUDA_ARCH__
  uint32_t u = __float_as_uint(f);
#else
  uint32_t u;
  std::memcpy(&u, &f, 4);
#endif
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__host__ __device__ __forceinline__ float f32_unorder(uint32_t u) {
  u = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
#ifdef __CUDA_ARCH__
  return __uint_as_float(u);
#else
  float f;
  std::memcpy(&f, &u, 4);
  return f;
#endif
}
__host__ __device__ __forceinline__ uint64_t f64_order(double f) {
#ifdef __CUDA_ARCH__
  uint64_t u = static_cast<uint64_t>(__double_as_longlong(f));
#else
  uint64_t u;
  std::memcpy(&u, &f, 8);
#endif
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

// ---------------------------------------------------------------------------
// Error budget of the FP32 filters (all quantities in the scaled working
// units of the FP32 copy; see DESIGN.md §4 for the derivation).
//
//   s32 = FP32 squared distance (FMA accumulation, any fixed order):
//         |s32 - S| <= e*S + a,  e = (d+4)u(1.01), a = (2d+2)*2^-149
//   key error |k^ - k| <= E = gamma_d * max||U_k|| * max||x||
//   narrowing radius Rn = max_i ||x_src,i*scale - x_f32,i||   (0 if exact)
//   sigma = spectral-norm bound of the FP32 direction matrix U
struct Budget {
  double e = 0, a = 0;     // s32 relative / absolute error
  double E = 0;            // per-key absolute error
  double Rn = 0;           // narrowing radius
  double sigma = 1;        // ||U||_2 bound
  double unorm = 1;        // max_k ||U_k||_2
  double gamma64 = 0;      // relative error of the reference's FP64 distance
  int nk = 1;              // keys used in the LB
};

// The projection runs on the tensor cores (tcgen05 kind::tf32, psg_project_tc.cu)
// for d in {32, 64, 128, 256}; elsewhere on FP32 CUDA cores.
__host__ __device__ inline bool tc_projection(int d, uint64_t n) {
  return (d == 32 || d == 64 || d == 128 || d == 256) && n < (1ull << 31);
}
// Relative key-error factor gamma (|k^ - k| <= gamma * sum_t |u_t x_t| + abs):
//   CUDA cores: FP32 FMA chain, any order: d u / (1 - d u);
//   tensor cores (psg_project_tc.cu): U is an exact TF32 operand, x = hi + lo
//   exactly with hi exact TF32 and lo losing <= 2^-10 |lo| <= 2^-20 |x| to the
//   TF32 conversion; products are exact in FP32.  The FP32 accumulation inside
//   and across the 2d/8 MMAs is charged 4 ulps (2^-22) per product term, 4x an
//   every-addition-truncates model, plus 2^-19 for lo.  tests/test_gpu_keys.py
//   measures the realised error against FP64 projections.  Values the tensor
//   core may flush (|x| < 2^-126) add at most d 2^-126 (key_abs).
//   `tc` = the keys came from the tensor-core projection (materialised rows of
//   a tc_projection shape; window sets are projected on CUDA cores).
__host__ __device__ inline double key_gamma(int d, bool tc) {
  const double u = 0x1.0p-24;
  if (tc) return (0x1.0p-19 + 2.0 * d * 0x1.0p-22) * 1.01;
  return d * u / (1.0 - d * u);
}
__host__ __device__ inline double key_abs(int d, bool tc) { return tc ? d * 0x1.0p-120 : 0.0; }

// Thresholds derived from an upper bound `dmax` (working units) on the real
// distance of any pair that may still matter.
struct Thresholds {
  float win;   // key-0 window: keep if fl(k0_j - k0_i) <= win
  float lb2;   // keep if sum_k fl(k_j - k_i)^2 (FP32) <= lb2
  float band;  // keep as FP64-recheck candidate if s32 <= band
};

__host__ __device__ inline double budget_dmax_from_s32(const Budget& b, float best_s32) {
  // real distance (float points) of the best-seen pair, then of the best
  // source pair, widened so every pair the FP64 reference could prefer fits.
  const double s = static_cast<double>(best_s32);
  const double df = sqrt((s + b.a) / (1.0 - b.e)) * (1.0 + 1e-12);
  return (df + 2.0 * b.Rn) * (1.0 + 4.0 * b.gamma64) + 2.0 * b.Rn;
}

__host__ __device__ inline Thresholds budget_thresholds(const Budget& b, double dmax) {
  const double u = 0x1.0p-24;
  Thresholds t;
  if (!(dmax < 1e300)) {  // +inf: everything passes
    t.win = t.lb2 = t.band = INFINITY;
    return t;
  }
  const double w = (dmax * b.unorm + 2.0 * b.E) * (1.0 + 4.0 * u);
  const double lb = (dmax * b.sigma + 2.0 * b.E * sqrt(static_cast<double>(b.nk))) * (1.0 + 4.0 * u);
  const double lb2 = lb * lb * (1.0 + (2.0 * b.nk + 8.0) * u);
  const double band = (dmax * dmax * (1.0 + b.e) + b.a) * (1.0 + 4.0 * u);
  // round up to float
  t.win = static_cast<float>(w * (1.0 + 2.0 * u));
  t.lb2 = static_cast<float>(lb2 * (1.0 + 2.0 * u));
  t.band = static_cast<float>(band * (1.0 + 2.0 * u));
  return t;
}

__host__ __device__ inline Thresholds budget_thresholds_s32(const Budget& b, float best_s32) {
  if (!(best_s32 < INFINITY)) return budget_thresholds(b, INFINITY);
  return budget_thresholds(b, budget_dmax_from_s32(b, best_s32));
}

// ---------------------------------------------------------------------------
// The algebra shared by the closest-pair and fixed-radius engines.
constexpr int kMaxKeys = 8;

// Host-built orthonormal projection directions (random, seeded), in FP32.
struct Directions {
  uint64_t seed = 0;          // make_directions(seed, d, q) is a pure function of these
  int d = 0, q = 0, nk = 0;   // q used rows, nk = padded rows (power of 2)
  std::vector<float> U;       // nk x d, rows >= q are zero
  double sigma = 1.0, unorm = 1.0;
};
Directions make_directions(uint64_t seed, int d, int q);

// Closed-form admissible pair count (main.cpp:388-395).
inline uint64_t admissible_pairs(uint64_t n, uint64_t zone) {
  if (zone <= 1) return n * (n - 1) / 2;
  if (zone >= n) return 0;
  const uint64_t m = n - zone;
  return m * (m + 1) / 2;
}

}  // namespace psg
