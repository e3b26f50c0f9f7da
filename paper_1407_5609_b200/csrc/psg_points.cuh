// psg_points.cuh — the device-resident point set (series.hpp:28-44 PointSet)
// and the reference's exact FP64 distance (metrics.cpp:16-24) on device.
//
// HBM layout:
//   src   the caller's values, kept for the FP64 recheck: f32 rows (n x d),
//         f64 rows (n x d), or an f64 series for window point sets
//   X     FP32 working rows, n x d row-major, = fl(scale * src) (aliases src
//         for exact float input); every FP32 filter reads only X
//   mu/sigma  per-window FP64 statistics of z-normalised window sets
#pragma once

#include <functional>
#include <memory>
#include <vector>

#include "psg_internal.cuh"

namespace psg {

enum SrcKind : int { kRowsF32 = 0, kRowsF64 = 1, kWindowsRaw = 2, kWindowsZ = 3 };

// What the FP64 recheck reads.
struct ExactSrc {
  int kind = kRowsF32;
  int d = 0;
  const float* f32 = nullptr;    // kRowsF32
  const double* f64 = nullptr;   // kRowsF64 rows, or the series for windows
  const double* mu = nullptr;    // kWindowsZ
  const double* sigma = nullptr; // kWindowsZ
};

// Coordinate t of point i exactly as the reference's PointSet would hold it.
__device__ __forceinline__ double exact_coord(const ExactSrc& s, uint64_t i, int t) {
  switch (s.kind) {
    case kRowsF32: return static_cast<double>(s.f32[i * s.d + t]);
    case kRowsF64: return s.f64[i * s.d + t];
    case kWindowsRaw: return s.f64[i + t];
    default: {
      const double sg = s.sigma[i];
      return sg == 0.0 ? 0.0 : __ddiv_rn(__dsub_rn(s.f64[i + t], s.mu[i]), sg);
    }
  }
}

// metrics.cpp:16-24: sum over t in index order of (x_t - y_t)^2, then sqrt;
// explicit _rn intrinsics forbid FMA contraction, matching x86-64 SSE2.
__device__ __forceinline__ double exact_distance(const ExactSrc& s, uint64_t i, uint64_t j) {
  double acc = 0.0;
  for (int t = 0; t < s.d; ++t) {
    const double diff = __dsub_rn(exact_coord(s, i, t), exact_coord(s, j, t));
    acc = __dadd_rn(acc, __dmul_rn(diff, diff));
  }
  return __dsqrt_rn(acc);
}

// exact_distance by a whole warp (every lane returns it): the squared
// differences — for z-normalised windows two FP64 divisions each, the slow
// part — are formed 32 at a time in parallel, then every lane adds the same
// terms in the same index order, so the result is bit-identical.
__device__ __forceinline__ double warp_exact_distance(const ExactSrc& s, uint64_t i, uint64_t j, int lane) {
  double acc = 0.0;
  for (int t0 = 0; t0 < s.d; t0 += 32) {
    const int t = t0 + lane;
    double term = 0.0;
    if (t < s.d) {
      const double diff = __dsub_rn(exact_coord(s, i, t), exact_coord(s, j, t));
      term = __dmul_rn(diff, diff);
    }
    const int m = s.d - t0 < 32 ? s.d - t0 : 32;
    for (int k = 0; k < m; ++k) acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, term, k));
  }
  return __dsqrt_rn(acc);
}

// The FP32 working rows every filter reads.  Row sets: X, n x d row-major.
// Window sets (windows_of, series.cpp:34-42) are virtual, as the reference's
// are: row i is computed where it is read from the FP32 series in working
// units (4 MiB at C3, L2-resident), so no n_w x len buffer exists:
//   raw          x_t = s32[i + t]
//   z-normalised x_t = fl(fl(s32[i + t] - m32[i]) * r32[i])
// (m32 = fl(mu), r32 = fl(scale / sigma), 0 when sigma == 0).  Rn and the row
// norms are measured on exactly these values (psg_points.cu), so the error
// budget covers them like materialised rows.
struct Rows {
  const float* X = nullptr;    // materialised rows, or nullptr for a window set
  const float* s32 = nullptr;  // window sets: the series
  const float* m32 = nullptr;  // z-normalised windows: per-window mean / inverse sigma
  const float* r32 = nullptr;
  int d = 0;
};

#ifdef __CUDACC__
__device__ __forceinline__ float row_at(const Rows& R, uint64_t i, int t) {
  if (R.X) return __ldg(R.X + i * R.d + t);
  const float v = __ldg(R.s32 + i + t);
  return R.m32 ? __fmul_rn(__fsub_rn(v, __ldg(R.m32 + i)), __ldg(R.r32 + i)) : v;
}
#endif

}  // namespace psg

struct psg_pointset {
  uint64_t n = 0;
  int d = 0;
  int kind = psg::kRowsF32;
  int device = 0;
  psg::DevBuf<float> src32;    // kRowsF32
  psg::DevBuf<double> src64;   // kRowsF64 rows / window series
  psg::DevBuf<double> mu, sigma;
  psg::DevBuf<float> work;     // FP32 working copy when X != src32
  psg::DevBuf<float> s32, m32, r32;  // window sets: virtual rows (psg::Rows)
  mutable psg::DevBuf<float> win_ut;      // the last directions used, transposed (d x nk)
  mutable std::vector<float> win_ut_host;
  mutable uint64_t win_ut_seed = 0;
  mutable int win_ut_q = -1;
  const float* X = nullptr;    // nullptr for window sets
  double scale = 1.0;          // X = fl(scale * src)
  double Rn = 0.0;             // max narrowing radius, working units
  double maxabs = 0.0;         // max |X|
  float norm2max = 0.f;        // max over rows of the FP32 sum of squares of X (any order)
  uint64_t h2d_bytes = 0;
  // solve workspaces reused across calls on this point set (nk = 4 / 8);
  // type-erased here, owned by the closest-pair engine (psg_cpp.cu)
  std::shared_ptr<void> cpp_work[2];

  psg::Rows rows() const {
    psg::Rows r;
    r.X = X;
    r.s32 = s32.p;
    r.m32 = m32.p;
    r.r32 = r32.p;
    r.d = d;
    return r;
  }
  psg::ExactSrc exact() const {
    psg::ExactSrc s;
    s.kind = kind;
    s.d = d;
    s.f32 = src32.p;
    s.f64 = src64.p;
    s.mu = mu.p;
    s.sigma = sigma.p;
    return s;
  }
};

namespace psg {
// Builders (psg_points.cu).  `dev_src` = the pointer is device memory.
psg_pointset* pointset_rows_f32(const float* p, uint64_t n, uint64_t d, bool dev_src);
psg_pointset* pointset_rows_f64(const double* p, uint64_t n, uint64_t d, bool dev_src);
psg_pointset* pointset_windows(const double* series64, const float* series32, uint64_t length, uint64_t len,
                               bool znorm, bool dev_src);
// Host -> device copies.  Pinned (page-locked or registered) sources go in one
// cudaMemcpyAsync; pageable ones (a std::vector, a numpy array) stream through
// the context's two pinned chunks: host threads fill chunk k+1 while the copy
// engine drains chunk k, so the upload runs near the pinned PCIe rate instead
// of the driver's pageable path.  `fill(stage, off, len)` writes source bytes
// [off, off + len) into a pinned chunk and returns how many it wrote.
void h2d_staged(void* dst, uint64_t bytes, const std::function<size_t(char*, uint64_t, size_t)>& fill,
                cudaStream_t s);
void h2d_copy(void* dst, const void* src, uint64_t bytes, cudaStream_t s);
// Launch accounting for the profile (incremented by every launch site).
extern thread_local uint64_t g_launches;
}  // namespace psg
