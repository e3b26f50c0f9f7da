// psg_refset.cu — build_reference_set (refscan.cpp:30-65) bit-exact on
// device: the seeded reference choice (host Rng stream, rng.cpp:34-44),
// references = x_ref * f, the k-major FP64 distance table in the reference's
// summation order, and the order permutation by (d1, index) via a stable
// 64-bit radix sort of the orderable image of d1 with the identity payload.
#include <algorithm>
#include <cmath>

#include "host_rng.hpp"
#include "psg_cpp.cuh"
#include "psg_engines.cuh"
#include "psg_sort.cuh"

namespace psg {
namespace {

__global__ void k_scale_refs(ExactSrc src, const uint64_t* __restrict__ idx, uint64_t q, double f,
                             double* __restrict__ refs) {
  const uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (e >= q * src.d) return;
  const uint64_t k = e / src.d;
  const int t = static_cast<int>(e % src.d);
  refs[e] = __dmul_rn(exact_coord(src, idx[k], t), f);  // refscan.cpp:47
}

__global__ void k_table(ExactSrc src, uint64_t n, uint64_t q, const double* __restrict__ refs,
                        double* __restrict__ table) {
  const uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (e >= q * n) return;
  const uint64_t k = e / n, i = e % n;
  const double* r = refs + k * src.d;
  double acc = 0.0;
  for (int t = 0; t < src.d; ++t) {  // metrics.cpp:19-22, euclidean_distance(ref, point)
    const double g = __dsub_rn(r[t], exact_coord(src, i, t));
    acc = __dadd_rn(acc, __dmul_rn(g, g));
  }
  table[e] = __dsqrt_rn(acc);
}

__global__ void k_order_keys(const double* __restrict__ d1, uint64_t n, uint64_t* __restrict__ k,
                             uint32_t* __restrict__ v) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  k[i] = f64_order(d1[i]);
  v[i] = static_cast<uint32_t>(i);
}

__global__ void k_widen_idx(const uint32_t* __restrict__ v, uint64_t n, uint64_t* __restrict__ out) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = v[i];
}

__global__ void k_bound(const double* __restrict__ v, int d, double* __restrict__ out) {
  // v = [r | x | y]; reference_bound = d(r,x) - d(r,y)  (refscan.cpp:229-232)
  double a = 0.0, b = 0.0;
  for (int t = 0; t < d; ++t) {
    const double g = __dsub_rn(v[t], v[d + t]);
    a = __dadd_rn(a, __dmul_rn(g, g));
  }
  for (int t = 0; t < d; ++t) {
    const double g = __dsub_rn(v[t], v[2 * d + t]);
    b = __dadd_rn(b, __dmul_rn(g, g));
  }
  *out = __dsub_rn(__dsqrt_rn(a), __dsqrt_rn(b));
}

unsigned blocks(uint64_t n, int per) { return static_cast<unsigned>((n + per - 1) / per); }

}  // namespace

void reference_set(psg_pointset* ps, uint64_t q, double f, uint64_t seed, uint64_t* ref_indices,
                   double* references, double* table, uint64_t* order) {
  const uint64_t n = ps->n;
  check_reference_args(n, q, f);
  if (n >= 0xffffffffull) throw invalid_argument("point count exceeds 2^32-1");
  cudaStream_t s = ctx().stream;
  HostRng rng(seed);
  const std::vector<uint64_t> chosen = rng.choose(n, q);  // refscan.cpp:41-42
  std::copy(chosen.begin(), chosen.end(), ref_indices);
  const ExactSrc src = ps->exact();
  const int d = ps->d;
  DevBuf<uint64_t> idx(q, s);
  DevBuf<double> refs(q * d, s), tab(q * n, s);
  PSG_CUDA(cudaMemcpyAsync(idx.p, chosen.data(), q * 8, cudaMemcpyHostToDevice, s));
  k_scale_refs<<<blocks(q * d, 256), 256, 0, s>>>(src, idx.p, q, f, refs.p);
  PSG_LAUNCHED();
  k_table<<<blocks(q * n, 256), 256, 0, s>>>(src, n, q, refs.p, tab.p);
  PSG_LAUNCHED();
  DevBuf<uint64_t> k0(n, s), k1(n, s);
  DevBuf<uint32_t> v0(n, s), v1(n, s), hist(radix_hist_words(n), s);
  k_order_keys<<<blocks(n, 256), 256, 0, s>>>(tab.p, n, k0.p, v0.p);
  PSG_LAUNCHED();
  uint64_t* kk[2] = {k0.p, k1.p};
  uint32_t* vv[2] = {v0.p, v1.p};
  const int which = radix_sort<uint64_t>(kk, vv, n, 0, 64, hist.p, s);
  DevBuf<uint64_t> ord(n, s);
  k_widen_idx<<<blocks(n, 256), 256, 0, s>>>(vv[which], n, ord.p);
  PSG_LAUNCHED();
  g_launches += 4 + 24;
  PSG_CUDA(cudaMemcpyAsync(references, refs.p, q * d * 8, cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaMemcpyAsync(table, tab.p, q * n * 8, cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaMemcpyAsync(order, ord.p, n * 8, cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaStreamSynchronize(s));
}

double reference_bound_dev(const double* r, const double* x, const double* y, uint64_t d) {
  cudaStream_t s = ctx().stream;
  DevBuf<double> v(3 * d + 1, s);
  PSG_CUDA(cudaMemcpyAsync(v.p, r, d * 8, cudaMemcpyHostToDevice, s));
  PSG_CUDA(cudaMemcpyAsync(v.p + d, x, d * 8, cudaMemcpyHostToDevice, s));
  PSG_CUDA(cudaMemcpyAsync(v.p + 2 * d, y, d * 8, cudaMemcpyHostToDevice, s));
  k_bound<<<1, 1, 0, s>>>(v.p, static_cast<int>(d), v.p + 3 * d);
  PSG_LAUNCHED();
  ++g_launches;
  double out;
  PSG_CUDA(cudaMemcpyAsync(&out, v.p + 3 * d, 8, cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaStreamSynchronize(s));
  return out;
}

}  // namespace psg
