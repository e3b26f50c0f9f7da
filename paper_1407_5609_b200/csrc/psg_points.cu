// psg_points.cu — device context, point-set construction (validation,
// narrowing to the FP32 working copy, z-normalised windows), and the seeded
// projection directions.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <set>
#include <map>
#include <memory>
#include <thread>
#include <tuple>

#include "host_pool.hpp"
#include "host_rng.hpp"
#include "psg_points.cuh"

namespace psg {

thread_local uint64_t g_launches = 0;
thread_local bool g_capturing = false;
thread_local cudaEvent_t* g_cap_ev = nullptr;
thread_local int g_cap_next = 0, g_cap_max = 0;
thread_local std::vector<CapMark> g_cap_spans, g_cap_stages;
thread_local bool g_cap_stage_marks = false, g_cap_span_marks = false;
namespace {
std::atomic<int> g_graph_prof{std::getenv("PSG_GRAPH_STAGES") ? 2 : 0};
}
int graph_profiling() { return g_graph_prof.load(); }
void set_graph_profiling(int level) { g_graph_prof.store(std::clamp(level, 0, 2)); }

void trace(const char* what) {
  static const bool on = std::getenv("PSG_TRACE") != nullptr;
  if (!on) return;
  static thread_local auto last = std::chrono::steady_clock::now();
  const auto now = std::chrono::steady_clock::now();
  std::fprintf(stderr, "[psg] %-24s %9.1f us\n", what,
               std::chrono::duration<double, std::micro>(now - last).count());
  last = now;
}

namespace {
std::mutex g_pinned_mu;
std::vector<void*> g_pinned_free;
}  // namespace

void* pinned_small_get() {
  std::lock_guard<std::mutex> g(g_pinned_mu);
  if (g_pinned_free.empty()) {
    constexpr size_t kSlab = 64;
    void* slab = nullptr;
    PSG_CUDA(cudaHostAlloc(&slab, kSlab * kPinnedSmall, cudaHostAllocPortable));  // never freed: a pool
    for (size_t k = 0; k < kSlab; ++k) g_pinned_free.push_back(static_cast<char*>(slab) + k * kPinnedSmall);
  }
  void* p = g_pinned_free.back();
  g_pinned_free.pop_back();
  return p;
}

void pinned_small_put(void* p) {
  if (!p) return;
  std::lock_guard<std::mutex> g(g_pinned_mu);
  g_pinned_free.push_back(p);
}

// trace() after draining the stream when PSG_TRACE_SYNC is set too (stage
// timing of normally asynchronous sequences; diagnostics only)
void trace_sync(const char* what, cudaStream_t s) {
  static const bool on = std::getenv("PSG_TRACE") != nullptr && std::getenv("PSG_TRACE_SYNC") != nullptr;
  if (on) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cs);
    if (cs == cudaStreamCaptureStatusNone) cudaStreamSynchronize(s);  // never inside a graph capture
  }
  trace(what);
}

void set_max_dynamic_smem(const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  PSG_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(mu);
  if (!done.insert({kernel, dev}).second) return;
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
  if (e != cudaSuccess) {
    done.erase({kernel, dev});
    throw cuda_error(std::string("dynamic shared memory of ") + std::to_string(bytes) + " bytes refused: " +
                     cudaGetErrorString(e));
  }
}

bool pdl_enabled() {
  static const bool off = std::getenv("PSG_NO_PDL") != nullptr;
  return !off;
}

Ctx& ctx() {
  static std::mutex mu;
  static std::map<int, std::unique_ptr<Ctx>> all;
  int dev = 0;
  PSG_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(mu);
  auto& c = all[dev];
  if (!c) {
    auto nc = std::make_unique<Ctx>();
    nc->device = dev;
    cudaDeviceProp prop;
    PSG_CUDA(cudaGetDeviceProperties(&prop, dev));
    if (prop.major != 10)
      throw cuda_error("pairscan_b200 is built for sm_100a; device " + std::to_string(dev) + " is sm_" +
                       std::to_string(prop.major) + std::to_string(prop.minor));
    nc->sm_count = prop.multiProcessorCount;
    PSG_CUDA(cudaStreamCreateWithFlags(&nc->stream, cudaStreamNonBlocking));
    cudaMemPool_t pool;
    PSG_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t keep = UINT64_MAX;  // keep freed blocks: repeated solves reuse them
    PSG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    c = std::move(nc);
  }
  return *c;
}

void h2d_staged(void* dst, uint64_t bytes, const std::function<size_t(char*, uint64_t, size_t)>& fill,
                cudaStream_t s) {
  Ctx& c = ctx();
  for (int k = 0; k < 2; ++k) {
    if (!c.stage[k]) PSG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&c.stage[k]), Ctx::kStageBytes));
    if (!c.stage_done[k]) PSG_CUDA(cudaEventCreateWithFlags(&c.stage_done[k], cudaEventDisableTiming));
  }
  char* out = static_cast<char*>(dst);
  const uint64_t chunk = Ctx::kStageBytes;
  int k = 0;
  for (uint64_t off = 0; off < bytes; off += chunk, k ^= 1) {
    const size_t len = static_cast<size_t>(std::min<uint64_t>(chunk, bytes - off));
    PSG_CUDA(cudaEventSynchronize(c.stage_done[k]));  // chunk k's previous upload has left it
    trace("h2d: buffer free");
    if (fill(c.stage[k], off, len) != len) {
      cudaStreamSynchronize(s);
      throw std::runtime_error("short read while staging host input");
    }
    trace("h2d: filled");
    PSG_CUDA(cudaMemcpyAsync(out + off, c.stage[k], len, cudaMemcpyHostToDevice, s));
    PSG_CUDA(cudaEventRecord(c.stage_done[k], s));
  }
}

void h2d_copy(void* dst, const void* src, uint64_t bytes, cudaStream_t s) {
  if (!bytes) return;
  cudaPointerAttributes at{};
  const bool pinned = cudaPointerGetAttributes(&at, src) == cudaSuccess && at.type == cudaMemoryTypeHost;
  cudaGetLastError();  // an unregistered pointer may leave a sticky "invalid value" on old drivers
  // small copies: the driver's own staging is as fast.  Mid-size ones too
  // until this device's pinned chunks exist: allocating them (64 MiB of
  // page-locked memory) costs ~30 ms once, which a process making one call
  // (the CLI) would pay for a copy the driver stages in about a millisecond
  const bool staged = ctx().stage[0] != nullptr;
  if (pinned || bytes <= (size_t(1) << 20) || (!staged && bytes <= (size_t(64) << 20))) {
    PSG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    return;
  }
  // memcpy fan-out over a persistent pool: one host thread moves ~10 GB/s,
  // the PCIe link ~50
  static HostPool pool(std::max(1u, std::min(16u, std::thread::hardware_concurrency())) - 1);
  const char* in = static_cast<const char*>(src);
  h2d_staged(dst, bytes, [&](char* stage, uint64_t off, size_t len) {
    const size_t per = ((len + pool.size() - 1) / pool.size() + 4095) & ~size_t(4095);
    const unsigned tasks = static_cast<unsigned>((len + per - 1) / per);
    pool.run(tasks, [&](unsigned k) {
      const size_t a = static_cast<size_t>(k) * per;
      std::memcpy(stage + a, in + off + a, std::min(per, len - a));
    });
    return len;
  }, s);
}

namespace {

__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* a, double v) {
  atomicMax(a, static_cast<unsigned long long>(__double_as_longlong(v)));
}

// One pass over float rows: finiteness (series.cpp:20-24), max |x| and the
// max row sum of squares (FP32, any order).  A warp per row (float4 lanes when
// d % 4 == 0) for d >= 32, a thread per row below.
__global__ void __launch_bounds__(256) k_check_rows_f32(const float* __restrict__ x, uint64_t n, int d,
                                                        unsigned* __restrict__ flags /* bad, maxabs, norm2 */) {
  unsigned m = 0, nonfinite = 0;
  float worst = 0.f;
  const uint64_t tid = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const uint64_t nth = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  auto take = [&](float v, float& acc) {
    nonfinite |= !isfinite(v);
    m = max(m, __float_as_uint(fabsf(v)));
    acc = fmaf(v, v, acc);
  };
  if (d >= 32) {
    const int lane = threadIdx.x & 31;
    for (uint64_t r = tid >> 5; r < n; r += nth >> 5) {
      const float* row = x + r * d;
      float acc = 0.f;
      if ((d & 3) == 0) {
        const float4* r4 = reinterpret_cast<const float4*>(row);
        for (int t = lane; t < (d >> 2); t += 32) {
          const float4 v = __ldcs(r4 + t);
          take(v.x, acc);
          take(v.y, acc);
          take(v.z, acc);
          take(v.w, acc);
        }
      } else {
        for (int t = lane; t < d; t += 32) take(__ldcs(row + t), acc);
      }
      for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      worst = fmaxf(worst, acc);
    }
  } else {
    for (uint64_t r = tid; r < n; r += nth) {
      const float* row = x + r * d;
      float acc = 0.f;
      for (int t = 0; t < d; ++t) take(row[t], acc);
      worst = fmaxf(worst, acc);
    }
  }
  m = __reduce_max_sync(0xffffffffu, m);
  nonfinite = __reduce_or_sync(0xffffffffu, nonfinite);
  const unsigned wb = __reduce_max_sync(0xffffffffu, __float_as_uint(worst));
  if ((threadIdx.x & 31) == 0 && nonfinite) atomicOr(flags, 1u);
  block_max_to(flags + 1, m);
  block_max_to(flags + 2, wb);
}

// max over rows of the FP32 sum of squares of a row (a per-set invariant the
// closest-pair error budget needs; computed once here, not per solve).  A warp
// per row for d >= 32, a thread per row below.
__global__ void k_row_norm2max(const float* __restrict__ X, uint64_t n, int d, unsigned* __restrict__ out) {
  float worst = 0.f;
  const uint64_t tid = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const uint64_t nth = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  if (d >= 32) {
    const int lane = threadIdx.x & 31;
    for (uint64_t r = tid >> 5; r < n; r += nth >> 5) {
      const float* row = X + r * d;
      float s = 0.f;
      for (int t = lane; t < d; t += 32) s = fmaf(row[t], row[t], s);
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      worst = fmaxf(worst, s);
    }
  } else {
    for (uint64_t r = tid; r < n; r += nth) {
      const float* row = X + r * d;
      float s = 0.f;
      for (int t = 0; t < d; ++t) s = fmaf(row[t], row[t], s);
      worst = fmaxf(worst, s);
    }
  }
  worst = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(worst)));
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(worst));
}

__global__ void k_check_f64(const double* __restrict__ x, uint64_t count, unsigned* __restrict__ bad,
                            unsigned long long* __restrict__ maxabs_bits) {
  unsigned long long m = 0;
  unsigned nonfinite = 0;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const double v = x[i];
    if (!isfinite(v)) nonfinite = 1;
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(fabs(v)));
    m = b > m ? b : m;
  }
  for (int o = 16; o; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(0xffffffffu, m, o);
    m = t > m ? t : m;
  }
  nonfinite = __reduce_or_sync(0xffffffffu, nonfinite);
  if ((threadIdx.x & 31) == 0) {
    if (nonfinite) atomicOr(bad, 1u);
    atomicMax(maxabs_bits, m);
  }
}

// Rows (f32 or f64 source) -> scaled FP32 rows; per-row narrowing radius
// ||scale*x - fl(scale*x)|| accumulated in FP64 and max-reduced.
template <class T>
__global__ void k_narrow_rows(const T* __restrict__ src, uint64_t n, int d, double scale, float* __restrict__ X,
                              unsigned long long* __restrict__ r2max_bits) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  double worst = 0.0;
  for (uint64_t r = warp; r < n; r += nwarps) {
    double acc = 0.0;
    for (int t = lane; t < d; t += 32) {
      const double v = scale * static_cast<double>(src[r * d + t]);
      const float f = static_cast<float>(v);
      X[r * d + t] = f;
      const double e = v - static_cast<double>(f);
      acc += e * e;
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    worst = fmax(worst, acc);
  }
  if (lane == 0) atomic_max_nonneg(r2max_bits, worst);
}

// Per-window FP64 statistics, two-pass and sequential like the oracle
// (the FP64 recheck reads them: exact_coord), plus the virtual rows' FP32
// mean and inverse sigma (psg_points.cuh Rows).
__global__ void k_window_stats(const double* __restrict__ s, uint64_t nw, int len, double* __restrict__ mu,
                               double* __restrict__ sigma, float* __restrict__ m32, float* __restrict__ r32) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= nw) return;
  const double* w = s + i;
  double acc = 0.0;
  for (int t = 0; t < len; ++t) acc = __dadd_rn(acc, w[t]);
  const double m = __ddiv_rn(acc, static_cast<double>(len));
  double v = 0.0;
  for (int t = 0; t < len; ++t) {
    const double c = __dsub_rn(w[t], m);
    v = __dadd_rn(v, __dmul_rn(c, c));
  }
  const double sg = __dsqrt_rn(__ddiv_rn(v, static_cast<double>(len)));
  mu[i] = m;
  sigma[i] = sg;
  m32[i] = __double2float_rn(m);
  r32[i] = sg == 0.0 ? 0.f : __double2float_rn(__drcp_rn(sg));
}

// The FP32 series of a window set: fl(scale * s) (raw windows; scale is a
// power of two) or fl(s) (z-normalised: the scale-free values are O(sqrt(len))).
__global__ void k_series_f32(const double* __restrict__ s, uint64_t len, double scale, float* __restrict__ out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < len;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = __double2float_rn(s[i] * scale);
}

// The narrowing radius of each virtual FP32 window row against the
// reference's FP64 window values (exact_coord order, times scale), in FP64,
// and the row's FP32 sum of squares; both max-reduced.
__global__ void __launch_bounds__(256) k_window_check(Rows R, ExactSrc src, uint64_t nw, double scale,
                                                      unsigned long long* __restrict__ r2max_bits,
                                                      unsigned* __restrict__ norm2_bits) {
  // one thread per window, coordinates in order: a warp's 32 windows read the
  // same 32 + t series values per step (coalesced, L1), and the per-value work
  // is a handful of instructions (a warp per window spent ~55 per value on
  // lane bookkeeping and shuffles: 1.5 ms at C3)
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  double worst = 0.0;
  float wn = 0.f;
  if (i < nw) {
    // z-normalised: the reference's (s - mu) / sigma as (s - mu) * (1 / sigma),
    // within 2^-51 |x| of it (one FP64 division per window; the host adds
    // len * 2^-50 to Rn for it)
    const bool z = src.kind == kWindowsZ;
    float m = 0.f, rr = 1.f;
    double mu = 0.0, inv = scale;
    if (z) {
      m = R.m32[i];
      rr = R.r32[i];
      mu = src.mu[i];
      const double sg = src.sigma[i];
      inv = sg == 0.0 ? 0.0 : 1.0 / sg;
    }
    const float* sp = R.s32 + i;
    const double* dp = src.f64 + i;
    double acc = 0.0;
    float nn = 0.f;
    for (int t = 0; t < R.d; ++t) {
      const float v = sp[t];
      const float x = z ? __fmul_rn(__fsub_rn(v, m), rr) : v;  // row_at, virtual window row
      const double xe = (dp[t] - mu) * inv;                     // raw: mu = 0, inv = scale
      const double e = xe - static_cast<double>(x);
      acc = fma(e, e, acc);
      nn = fmaf(x, x, nn);
    }
    worst = acc;
    wn = nn;
  }
  // one atomic per block for each maximum (non-negative doubles order as their bits)
  __shared__ unsigned long long wr[32];
  unsigned long long wm = static_cast<unsigned long long>(__double_as_longlong(worst));
  for (int o = 16; o; o >>= 1) wm = max(wm, __shfl_xor_sync(0xffffffffu, wm, o));
  if ((threadIdx.x & 31) == 0) wr[threadIdx.x >> 5] = wm;
  block_max_to(norm2_bits, __float_as_uint(wn));  // its barrier also publishes wr
  if (threadIdx.x == 0) {
    unsigned long long mx = 0;
    for (unsigned w = 0; w < (blockDim.x + 31) / 32; ++w) mx = max(mx, wr[w]);
    if (mx) atomicMax(r2max_bits, mx);
  }
}

__global__ void k_widen(const float* __restrict__ in, uint64_t count, double* __restrict__ out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<double>(in[i]);
}

int grid_for(uint64_t work, int per_block, int sms) {
  const uint64_t want = (work + per_block - 1) / per_block;
  const uint64_t cap = static_cast<uint64_t>(sms) * 16;
  return static_cast<int>(want < cap ? (want ? want : 1) : cap);
}

// Power-of-two scale that keeps FP32 squares far from overflow/underflow.
double choose_scale(double maxabs) {
  if (maxabs == 0.0 || (maxabs < 0x1.0p60 && maxabs > 0x1.0p-60)) return 1.0;
  int e = 0;
  std::frexp(maxabs, &e);
  return std::ldexp(1.0, 8 - e);
}

template <class T>
void upload(DevBuf<T>& dst, const T* src, uint64_t count, bool dev_src, cudaStream_t s, uint64_t* h2d) {
  dst.alloc(count, s);
  if (!count) return;
  if (dev_src) {
    PSG_CUDA(cudaMemcpyAsync(dst.p, src, count * sizeof(T), cudaMemcpyDeviceToDevice, s));
    return;
  }
  h2d_copy(dst.p, src, count * sizeof(T), s);
  *h2d += count * sizeof(T);
}

double read_r2(unsigned long long* dbits, cudaStream_t s) {
  unsigned long long h = 0;
  PSG_CUDA(cudaMemcpyAsync(&h, dbits, 8, cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaStreamSynchronize(s));
  double r2;
  std::memcpy(&r2, &h, 8);
  return r2;
}

// sqrt of an FP64-accumulated sum of squares, widened to a safe upper bound.
float row_norm2max(const float* X, uint64_t n, int d, cudaStream_t s, int sms) {
  if (n == 0 || d == 0) return 0.f;
  DevBuf<unsigned> out(1, s);
  PSG_CUDA(cudaMemsetAsync(out.p, 0, 4, s));
  k_row_norm2max<<<grid_for(d >= 32 ? n * 32 : n, 256, sms), 256, 0, s>>>(X, n, d, out.p);
  PSG_LAUNCHED();
  ++g_launches;
  unsigned h = 0;
  PSG_CUDA(cudaMemcpyAsync(&h, out.p, 4, cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaStreamSynchronize(s));
  float v;
  std::memcpy(&v, &h, 4);
  return v;
}

double radius_bound(double r2, int d) {
  if (r2 <= 0.0) return 0.0;
  return std::sqrt(r2 * (1.0 + 4.0 * d * 0x1.0p-53)) * (1.0 + 1e-12);
}

}  // namespace

psg_pointset* pointset_rows_f32(const float* p, uint64_t n, uint64_t d, bool dev_src) {
  Ctx& c = ctx();
  cudaStream_t s = c.stream;
  auto ps = std::make_unique<psg_pointset>();
  ps->n = n;
  ps->d = static_cast<int>(d);
  ps->kind = kRowsF32;
  ps->device = c.device;
  trace("rows32: enter");
  upload(ps->src32, p, n * d, dev_src, s, &ps->h2d_bytes);
  trace("rows32: upload enqueued");
  DevBuf<unsigned> flags(3, s);
  PSG_CUDA(cudaMemsetAsync(flags.p, 0, 12, s));
  if (n * d) {
    k_check_rows_f32<<<grid_for(d >= 32 ? n * 32 : n, 256, c.sm_count), 256, 0, s>>>(ps->src32.p, n, ps->d,
                                                                                      flags.p);
    PSG_LAUNCHED();
    ++g_launches;
  }
  unsigned h[3];
  PSG_CUDA(cudaMemcpyAsync(h, flags.p, 12, cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaStreamSynchronize(s));
  trace("rows32: checked");
  if (h[0]) throw invalid_argument("point coordinate must be finite");
  float mx;
  std::memcpy(&mx, &h[1], 4);
  ps->scale = choose_scale(mx);
  ps->X = ps->src32.p;
  if (ps->scale != 1.0) {
    ps->work.alloc(n * d, s);
    DevBuf<unsigned long long> r2(1, s);
    PSG_CUDA(cudaMemsetAsync(r2.p, 0, 8, s));
    k_narrow_rows<float><<<grid_for(n * 32, 256, c.sm_count), 256, 0, s>>>(ps->src32.p, n, ps->d, ps->scale,
                                                                           ps->work.p, r2.p);
    PSG_LAUNCHED();
    ++g_launches;
    ps->Rn = radius_bound(read_r2(r2.p, s), ps->d);
    ps->X = ps->work.p;
  }
  ps->maxabs = static_cast<double>(mx) * ps->scale;
  if (ps->scale == 1.0)
    std::memcpy(&ps->norm2max, &h[2], 4);  // X is the input: its norms came with the check
  else
    ps->norm2max = row_norm2max(ps->X, n, ps->d, s, c.sm_count);
  return ps.release();
}

psg_pointset* pointset_rows_f64(const double* p, uint64_t n, uint64_t d, bool dev_src) {
  Ctx& c = ctx();
  cudaStream_t s = c.stream;
  auto ps = std::make_unique<psg_pointset>();
  ps->n = n;
  ps->d = static_cast<int>(d);
  ps->kind = kRowsF64;
  ps->device = c.device;
  upload(ps->src64, p, n * d, dev_src, s, &ps->h2d_bytes);
  DevBuf<unsigned> bad(1, s);
  DevBuf<unsigned long long> mx(2, s);
  PSG_CUDA(cudaMemsetAsync(bad.p, 0, 4, s));
  PSG_CUDA(cudaMemsetAsync(mx.p, 0, 16, s));
  if (n * d) {
    k_check_f64<<<grid_for(n * d, 256 * 8, c.sm_count), 256, 0, s>>>(ps->src64.p, n * d, bad.p, mx.p);
    PSG_LAUNCHED();
    ++g_launches;
  }
  unsigned hb = 0;
  unsigned long long hm = 0;
  PSG_CUDA(cudaMemcpyAsync(&hb, bad.p, 4, cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaMemcpyAsync(&hm, mx.p, 8, cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaStreamSynchronize(s));
  if (hb) throw invalid_argument("point coordinate must be finite");
  double maxabs;
  std::memcpy(&maxabs, &hm, 8);
  ps->scale = choose_scale(maxabs);
  ps->work.alloc(n * d, s);
  if (n * d) {
    k_narrow_rows<double><<<grid_for(n * 32, 256, c.sm_count), 256, 0, s>>>(ps->src64.p, n, ps->d, ps->scale,
                                                                            ps->work.p, mx.p + 1);
    PSG_LAUNCHED();
    ++g_launches;
    ps->Rn = radius_bound(read_r2(mx.p + 1, s), ps->d);
  }
  ps->X = ps->work.p;
  ps->maxabs = maxabs * ps->scale;
  ps->norm2max = row_norm2max(ps->X, ps->n, ps->d, s, c.sm_count);
  return ps.release();
}

psg_pointset* pointset_windows(const double* series64, const float* series32, uint64_t length, uint64_t len,
                               bool znorm, bool dev_src) {
  // TimeSeries::window_count (series.cpp:8-11)
  if (len == 0 || len > length) throw invalid_argument("window length out of range");
  Ctx& c = ctx();
  cudaStream_t s = c.stream;
  auto ps = std::make_unique<psg_pointset>();
  const uint64_t nw = length - len + 1;
  ps->n = nw;
  ps->d = static_cast<int>(len);
  ps->kind = znorm ? kWindowsZ : kWindowsRaw;
  ps->device = c.device;
  trace("windows: enter");
  if (series64) {
    upload(ps->src64, series64, length, dev_src, s, &ps->h2d_bytes);
    trace_sync("windows: uploaded", s);
  } else {
    DevBuf<float> tmp;
    upload(tmp, series32, length, dev_src, s, &ps->h2d_bytes);
    ps->src64.alloc(length, s);
    k_widen<<<grid_for(length, 256 * 4, c.sm_count), 256, 0, s>>>(tmp.p, length, ps->src64.p);
    PSG_LAUNCHED();
    ++g_launches;
  }
  DevBuf<unsigned> bad(1, s);
  DevBuf<unsigned long long> mx(2, s);
  PSG_CUDA(cudaMemsetAsync(bad.p, 0, 4, s));
  PSG_CUDA(cudaMemsetAsync(mx.p, 0, 16, s));
  k_check_f64<<<grid_for(length, 256 * 8, c.sm_count), 256, 0, s>>>(ps->src64.p, length, bad.p, mx.p);
  PSG_LAUNCHED();
  ++g_launches;
  unsigned hb = 0;
  unsigned long long hm = 0;
  PSG_CUDA(cudaMemcpyAsync(&hb, bad.p, 4, cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaMemcpyAsync(&hm, mx.p, 8, cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaStreamSynchronize(s));
  trace("windows: checked");
  if (hb) throw invalid_argument("series value must be finite");
  double maxabs;
  std::memcpy(&maxabs, &hm, 8);
  ps->scale = znorm ? 1.0 : choose_scale(maxabs);  // z-normalised: |x| <= sqrt(len)
  if (znorm) {
    ps->mu.alloc(nw, s);
    ps->sigma.alloc(nw, s);
    ps->m32.alloc(nw, s);
    ps->r32.alloc(nw, s);
    k_window_stats<<<static_cast<int>((nw + 255) / 256), 256, 0, s>>>(ps->src64.p, nw, ps->d, ps->mu.p, ps->sigma.p,
                                                                       ps->m32.p, ps->r32.p);
    PSG_LAUNCHED();
    ++g_launches;
    maxabs = std::sqrt(static_cast<double>(len));
    trace_sync("windows: stats", s);
  }
  ps->s32.alloc(length, s);
  k_series_f32<<<grid_for(length, 256 * 4, c.sm_count), 256, 0, s>>>(ps->src64.p, length, ps->scale, ps->s32.p);
  PSG_LAUNCHED();
  DevBuf<unsigned> nb(1, s);
  PSG_CUDA(cudaMemsetAsync(nb.p, 0, 4, s));
  k_window_check<<<static_cast<unsigned>((nw + 255) / 256), 256, 0, s>>>(ps->rows(), ps->exact(), nw, ps->scale,
                                                                          mx.p + 1, nb.p);
  PSG_LAUNCHED();
  g_launches += 2;
  ps->Rn = radius_bound(read_r2(mx.p + 1, s), ps->d) + (znorm ? static_cast<double>(len) * 0x1.0p-50 : 0.0);
  trace("windows: error check");
  unsigned hn = 0;
  PSG_CUDA(cudaMemcpy(&hn, nb.p, 4, cudaMemcpyDeviceToHost));
  std::memcpy(&ps->norm2max, &hn, 4);
  ps->X = nullptr;  // virtual rows (Rows): no n_w x len buffer
  ps->maxabs = maxabs * ps->scale;
  return ps.release();
}

// ---------------------------------------------------------------------------
// Seeded orthonormal projection directions.  These replace the reference's
// scaled reference points (refscan.cpp:30-56): a key is <u_k, x> instead of
// ||f*x_r - x||, the f -> infinity limit of the same 1-Lipschitz bound
// (test_refscan.cpp:85-99).  Rows are drawn from the
// reference Rng stream derive_seed(seed, 0x5eed), orthonormalised in FP64
// (modified Gram-Schmidt), then rounded to FP32; the spectral norm of the
// rounded matrix is bounded (Gershgorin on U U^T) for the LB filter.
namespace {
Directions make_directions_uncached(uint64_t seed, int d, int q);
}

// Cached: repeated solves with the same (seed, d, q) reuse the matrix.
Directions make_directions(uint64_t seed, int d, int q) {
  static std::mutex mu;
  static std::map<std::tuple<uint64_t, int, int>, Directions> cache;
  std::lock_guard<std::mutex> g(mu);
  const auto key = std::make_tuple(seed, d, q);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  if (cache.size() > 64) cache.clear();
  return cache[key] = make_directions_uncached(seed, d, q);
}

namespace {
Directions make_directions_uncached(uint64_t seed, int d, int q) {
  Directions dir;
  dir.seed = seed;
  dir.d = d;
  dir.q = std::max(1, std::min(std::min(q, d), kMaxKeys));
  dir.nk = dir.q <= 4 ? 4 : 8;
  std::vector<double> V(static_cast<size_t>(dir.q) * d);
  HostRng rng(stream_seed(seed, 0x5eed));
  for (int k = 0; k < dir.q; ++k) {
    for (;;) {
      double* v = &V[static_cast<size_t>(k) * d];
      for (int t = 0; t < d; ++t) v[t] = rng.gauss(0.0, 1.0);
      for (int pass = 0; pass < 2; ++pass)
        for (int l = 0; l < k; ++l) {
          const double* w = &V[static_cast<size_t>(l) * d];
          double dot = 0.0;
          for (int t = 0; t < d; ++t) dot += v[t] * w[t];
          for (int t = 0; t < d; ++t) v[t] -= dot * w[t];
        }
      double nrm = 0.0;
      for (int t = 0; t < d; ++t) nrm += v[t] * v[t];
      nrm = std::sqrt(nrm);
      if (nrm < 1e-6) continue;  // degenerate draw: redraw
      for (int t = 0; t < d; ++t) v[t] /= nrm;
      break;
    }
  }
  dir.U.assign(static_cast<size_t>(dir.nk) * d, 0.0f);
  // tensor-core projection shapes take U as an exact TF32 operand: round to
  // 10 mantissa bits here, so sigma / unorm below describe the matrix used
  const bool tf32 = d == 32 || d == 64 || d == 128 || d == 256;
  for (size_t i = 0; i < V.size(); ++i) {
    float v = static_cast<float>(V[i]);
    if (tf32) {
      uint32_t b;
      std::memcpy(&b, &v, 4);
      b = (b + 0x1000u) & ~0x1fffu;  // nearest, ties away (|v| <= 1: no overflow)
      std::memcpy(&v, &b, 4);
    }
    dir.U[i] = v;
  }
  double gmax = 0.0, unorm = 0.0;
  for (int k = 0; k < dir.q; ++k) {
    double row = 0.0;
    for (int l = 0; l < dir.q; ++l) {
      double g = 0.0;
      for (int t = 0; t < d; ++t)
        g += static_cast<double>(dir.U[static_cast<size_t>(k) * d + t]) * dir.U[static_cast<size_t>(l) * d + t];
      row += std::fabs(g);
      if (k == l) unorm = std::max(unorm, std::sqrt(g));
    }
    gmax = std::max(gmax, row);
  }
  dir.sigma = std::sqrt(gmax) * (1.0 + 1e-9);
  dir.unorm = unorm * (1.0 + 1e-9);
  return dir;
}
}  // namespace

}  // namespace psg
