// psg_capi.cu — the extern "C" boundary (include/pairscan_b200.h).
// Every entry: clear the per-thread profile, run, translate exceptions into
// status codes, keep the message for psg_last_error().
#include <algorithm>
#include <cmath>
#include <memory>
#include <new>
#include <string>

#include "host_rng.hpp"
#include "psg_cpp.cuh"
#include "psg_engines.cuh"
#include "psg_io.hpp"

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    psg::prof_begin();
    psg::Ctx& c = psg::ctx();
    std::lock_guard<std::mutex> lock(c.mu);  // one call at a time per device (shared workspaces)
    psg::KernelSpan span(c.stream);          // device span of the whole call
    f();
    psg::g_prof.total_ms = span.stop();
    psg::g_prof.launches = psg::g_launches;
    return PSG_OK;
  } catch (const psg::invalid_argument& e) {
    g_err = e.what();
    return PSG_ERR_INVALID;
  } catch (const psg::io_error& e) {
    g_err = e.what();
    return PSG_ERR_IO;
  } catch (const psg::cuda_error& e) {
    g_err = e.what();
    return PSG_ERR_CUDA;
  } catch (const std::bad_alloc&) {
    g_err = "out of memory";
    return PSG_ERR_NOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PSG_ERR_INTERNAL;
  }
}

// Host-only entries (file formats): no device context is touched.
template <class F>
int guarded_host(F&& f) {
  try {
    f();
    return PSG_OK;
  } catch (const psg::invalid_argument& e) {
    g_err = e.what();
    return PSG_ERR_INVALID;
  } catch (const psg::io_error& e) {
    g_err = e.what();
    return PSG_ERR_IO;
  } catch (const std::bad_alloc&) {
    g_err = "out of memory";
    return PSG_ERR_NOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PSG_ERR_INTERNAL;
  }
}

// Stream a .psgb payload into device memory through the context's pinned
// chunks: the parallel read of chunk k+1 overlaps the upload of chunk k.
psg::DevBuf<char> upload_file(psg::BinaryFile& bf, cudaStream_t s) {
  psg::DevBuf<char> dev(std::max<uint64_t>(bf.bytes, 1), s);
  psg::h2d_staged(dev.p, bf.bytes, [&](char* stage, uint64_t off, size_t len) {
    if (bf.pread_payload(stage, off, len, 8) != len) {
      cudaStreamSynchronize(s);
      throw psg::io_error("short read from a .psgb file");
    }
    return len;
  }, s);
  PSG_CUDA(cudaStreamSynchronize(s));
  psg::g_prof.h2d_bytes += bf.bytes;
  return dev;
}

void require_dim(uint64_t dim) {
  if (dim == 0) throw psg::invalid_argument("point dimension must be positive");  // series.cpp:20
}

// PointSet::from_flat takes a flat buffer whose length is a multiple of dim
// (series.cpp:19-32); here n and dim are given separately.
std::unique_ptr<psg_pointset> rows32(const float* p, uint64_t n, uint64_t dim, bool dev = false) {
  require_dim(dim);
  return std::unique_ptr<psg_pointset>(psg::pointset_rows_f32(p, n, dim, dev));
}
std::unique_ptr<psg_pointset> rows64(const double* p, uint64_t n, uint64_t dim, bool dev = false) {
  require_dim(dim);
  return std::unique_ptr<psg_pointset>(psg::pointset_rows_f64(p, n, dim, dev));
}

void account_io(const psg_pointset& ps, uint64_t d2h) {
  psg::g_prof.h2d_bytes += ps.h2d_bytes;
  psg::g_prof.d2h_bytes += d2h;
}

struct psg_cpp_plan_box {};
}  // namespace

struct psg_cpp_plan {
  std::unique_ptr<psg::CppPlan> plan;
};

extern "C" {

const char* psg_last_error(void) { return g_err.c_str(); }
const char* psg_version(void) { return "pairscan_b200 0.1.0 (sm_100a)"; }

int psg_last_profile(psg_profile* out) {
  if (!out) return PSG_ERR_INVALID;
  *out = psg::g_prof;
  return PSG_OK;
}

int psg_set_graph_profiling(int level) {
  psg::set_graph_profiling(level);
  return PSG_OK;
}

int psg_set_device(int device) {
  const cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    g_err = cudaGetErrorString(e);
    return PSG_ERR_CUDA;
  }
  return PSG_OK;
}

void* psg_stream(void) {
  try {
    return static_cast<void*>(psg::ctx().stream);
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

int psg_device_ok(int device) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || device < 0 || device >= count) return 0;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return 0;
  return prop.major == 10;
}

// ---- closest pair -----------------------------------------------------------
int psg_closest_pair_f64(const double* points, uint64_t n, uint64_t dim, uint64_t q, double f, uint64_t seed,
                         uint64_t exclusion_zone, psg_pair_result* out) {
  return guarded([&] {
    auto ps = rows64(points, n, dim);
    *out = psg::cpp_solve(ps.get(), q, f, seed, exclusion_zone);
    account_io(*ps, 0);
  });
}
int psg_closest_pair_f32(const float* points, uint64_t n, uint64_t dim, uint64_t q, double f, uint64_t seed,
                         uint64_t exclusion_zone, psg_pair_result* out) {
  return guarded([&] {
    auto ps = rows32(points, n, dim);
    *out = psg::cpp_solve(ps.get(), q, f, seed, exclusion_zone);
    account_io(*ps, 0);
  });
}
int psg_brute_force_closest_pair_f64(const double* points, uint64_t n, uint64_t dim, uint64_t exclusion_zone,
                                     psg_pair_result* out) {
  return guarded([&] {
    auto ps = rows64(points, n, dim);
    *out = psg::brute_solve(ps.get(), exclusion_zone);
  });
}
int psg_brute_force_closest_pair_f32(const float* points, uint64_t n, uint64_t dim, uint64_t exclusion_zone,
                                     psg_pair_result* out) {
  return guarded([&] {
    auto ps = rows32(points, n, dim);
    *out = psg::brute_solve(ps.get(), exclusion_zone);
  });
}

// ---- motif -------------------------------------------------------------------
int psg_motif_f64(const double* series, uint64_t length, uint64_t len, int znorm, uint64_t q, double f,
                  uint64_t seed, uint64_t exclusion_zone, psg_pair_result* out) {
  return guarded([&] {
    std::unique_ptr<psg_pointset> ps(psg::pointset_windows(series, nullptr, length, len, znorm != 0, false));
    *out = psg::cpp_solve(ps.get(), q, f, seed, exclusion_zone);
    account_io(*ps, 0);
  });
}
int psg_motif_f32(const float* series, uint64_t length, uint64_t len, int znorm, uint64_t q, double f,
                  uint64_t seed, uint64_t exclusion_zone, psg_pair_result* out) {
  return guarded([&] {
    std::unique_ptr<psg_pointset> ps(psg::pointset_windows(nullptr, series, length, len, znorm != 0, false));
    *out = psg::cpp_solve(ps.get(), q, f, seed, exclusion_zone);
    account_io(*ps, 0);
  });
}
int psg_brute_force_motif_f64(const double* series, uint64_t length, uint64_t len, int znorm,
                              uint64_t exclusion_zone, psg_pair_result* out) {
  return guarded([&] {
    std::unique_ptr<psg_pointset> ps(psg::pointset_windows(series, nullptr, length, len, znorm != 0, false));
    *out = psg::brute_solve(ps.get(), exclusion_zone);
  });
}

// ---- fixed radius --------------------------------------------------------------
int psg_fixed_radius_neighbors_f64(const double* points, uint64_t n, uint64_t dim, double radius, uint64_t q,
                                   double f, uint64_t seed, uint64_t exclusion_zone, int want_lists,
                                   psg_neighbor_result* out) {
  return guarded([&] {
    if (n == 0) throw psg::invalid_argument("empty input");  // refscan.cpp:162, before from_flat checks
    auto ps = rows64(points, n, dim);
    psg::frnn_solve(ps.get(), radius, q, f, seed, exclusion_zone, want_lists != 0, out);
    account_io(*ps, 0);
  });
}
int psg_fixed_radius_neighbors_f32(const float* points, uint64_t n, uint64_t dim, double radius, uint64_t q,
                                   double f, uint64_t seed, uint64_t exclusion_zone, int want_lists,
                                   psg_neighbor_result* out) {
  return guarded([&] {
    if (n == 0) throw psg::invalid_argument("empty input");
    auto ps = rows32(points, n, dim);
    psg::frnn_solve(ps.get(), radius, q, f, seed, exclusion_zone, want_lists != 0, out);
    account_io(*ps, 0);
  });
}
int psg_brute_force_neighbors_f64(const double* points, uint64_t n, uint64_t dim, double radius,
                                  uint64_t exclusion_zone, int want_lists, psg_neighbor_result* out) {
  return guarded([&] {
    if (n == 0) throw psg::invalid_argument("empty input");  // refscan.cpp:214
    auto ps = rows64(points, n, dim);
    psg::brute_neighbors(ps.get(), radius, exclusion_zone, want_lists != 0, out);
  });
}
int psg_frnn_pairs_f32(const float* points, uint64_t n, uint64_t dim, double radius, uint64_t q, double f,
                       uint64_t seed, uint64_t exclusion_zone, uint64_t* pairs, uint64_t capacity,
                       uint64_t* pair_count, uint64_t* pair_hash) {
  return guarded([&] {
    if (n == 0) throw psg::invalid_argument("empty input");
    auto ps = rows32(points, n, dim);
    psg::frnn_pairs(ps.get(), radius, q, f, seed, exclusion_zone, pairs, capacity, pair_count, pair_hash);
    account_io(*ps, 0);
  });
}
int psg_frnn_pairs_csr_f32(const float* points, uint64_t n, uint64_t dim, double radius, uint64_t q, double f,
                           uint64_t seed, uint64_t exclusion_zone, uint64_t* offsets, uint32_t* cols,
                           uint64_t capacity, uint64_t* pair_count, uint64_t* pair_hash) {
  return guarded([&] {
    if (n == 0) throw psg::invalid_argument("empty input");
    psg::trace("csr: enter");
    auto ps = rows32(points, n, dim);
    psg::trace("csr: point set");
    psg::frnn_pairs_csr(ps.get(), radius, q, f, seed, exclusion_zone, offsets, cols, capacity, pair_count,
                        pair_hash);
    account_io(*ps, 0);
  });
}
void psg_neighbor_result_free(psg_neighbor_result* r) {
  if (!r) return;
  std::free(r->offsets);
  std::free(r->neighbors);
  r->offsets = nullptr;
  r->neighbors = nullptr;
}

// ---- reference set -------------------------------------------------------------
int psg_build_reference_set_f64(const double* points, uint64_t n, uint64_t dim, uint64_t q, double f,
                                uint64_t seed, uint64_t* ref_indices, double* references, double* dist_table,
                                uint64_t* order) {
  return guarded([&] {
    auto ps = rows64(points, n, dim);
    psg::reference_set(ps.get(), q, f, seed, ref_indices, references, dist_table, order);
  });
}
int psg_reference_bound(const double* r, const double* x, const double* y, uint64_t dim, double* out) {
  return guarded([&] { *out = psg::reference_bound_dev(r, x, y, dim); });
}

// ---- device-resident point sets ------------------------------------------------
int psg_pointset_from_f32(const float* points, uint64_t n, uint64_t dim, int flags, psg_pointset** out) {
  return guarded([&] { *out = rows32(points, n, dim, flags & PSG_SRC_DEVICE).release(); });
}
int psg_pointset_from_f64(const double* points, uint64_t n, uint64_t dim, int flags, psg_pointset** out) {
  return guarded([&] { *out = rows64(points, n, dim, flags & PSG_SRC_DEVICE).release(); });
}
int psg_pointset_windows_f64(const double* series, uint64_t length, uint64_t len, int znorm, int flags,
                             psg_pointset** out) {
  return guarded([&] {
    *out = psg::pointset_windows(series, nullptr, length, len, znorm != 0, flags & PSG_SRC_DEVICE);
  });
}
int psg_pointset_windows_f32(const float* series, uint64_t length, uint64_t len, int znorm, int flags,
                             psg_pointset** out) {
  return guarded([&] {
    *out = psg::pointset_windows(nullptr, series, length, len, znorm != 0, flags & PSG_SRC_DEVICE);
  });
}
void psg_pointset_free(psg_pointset* ps) { delete ps; }
uint64_t psg_pointset_size(const psg_pointset* ps) { return ps ? ps->n : 0; }
uint64_t psg_pointset_dim(const psg_pointset* ps) { return ps ? static_cast<uint64_t>(ps->d) : 0; }

int psg_closest_pair_ps(psg_pointset* ps, uint64_t q, double f, uint64_t seed, uint64_t exclusion_zone,
                        psg_pair_result* out) {
  return guarded([&] { *out = psg::cpp_solve(ps, q, f, seed, exclusion_zone); });
}
int psg_brute_force_closest_pair_ps(psg_pointset* ps, uint64_t exclusion_zone, psg_pair_result* out) {
  return guarded([&] { *out = psg::brute_solve(ps, exclusion_zone); });
}
int psg_debug_brute_bounded_ps(psg_pointset* ps, uint64_t exclusion_zone, double upper, psg_pair_result* out) {
  return guarded([&] {
    if (!(upper >= 0.0) || !std::isfinite(upper)) throw psg::invalid_argument("upper bound must be finite and >= 0");
    *out = psg::brute_solve(ps, exclusion_zone, upper);
  });
}
int psg_brute_force_neighbors_ps(psg_pointset* ps, double radius, uint64_t exclusion_zone, int want_lists,
                                 psg_neighbor_result* out) {
  return guarded([&] {
    if (ps->n == 0) throw psg::invalid_argument("empty input");  // refscan.cpp:214
    psg::brute_neighbors(ps, radius, exclusion_zone, want_lists != 0, out);
  });
}
int psg_fixed_radius_neighbors_ps(psg_pointset* ps, double radius, uint64_t q, double f, uint64_t seed,
                                  uint64_t exclusion_zone, int want_lists, psg_neighbor_result* out) {
  return guarded([&] { psg::frnn_solve(ps, radius, q, f, seed, exclusion_zone, want_lists != 0, out); });
}

// ---- sharded closest pair ------------------------------------------------------
int psg_cpp_plan_create(psg_pointset* ps, uint64_t q, double f, uint64_t seed, uint64_t exclusion_zone,
                        psg_cpp_plan** out) {
  return guarded([&] {
    auto p = std::make_unique<psg_cpp_plan>();
    p->plan.reset(psg::cpp_plan_create(ps, q, f, seed, exclusion_zone, /*sharded=*/true));
    *out = p.release();
  });
}
int psg_cpp_plan_bootstrap(psg_cpp_plan* plan, uint64_t part, uint64_t nparts, float* bound_s32) {
  return guarded([&] {
    if (nparts == 0 || part >= nparts) throw psg::invalid_argument("part out of range");
    *bound_s32 = psg::cpp_plan_bootstrap(*plan->plan, part, nparts);
  });
}
int psg_cpp_plan_scan(psg_cpp_plan* plan, uint64_t part, uint64_t nparts, float bound_s32, psg_pair_result* out) {
  return guarded([&] {
    if (nparts == 0 || part >= nparts) throw psg::invalid_argument("part out of range");
    *out = psg::cpp_plan_scan(*plan->plan, part, nparts, bound_s32);
  });
}
void psg_cpp_plan_free(psg_cpp_plan* plan) { delete plan; }

// ---- sharded fixed-radius neighbours -------------------------------------------
int psg_frnn_plan_create(psg_pointset* ps, double radius, uint64_t q, double f, uint64_t seed,
                         uint64_t exclusion_zone, psg_frnn_plan** out) {
  return guarded([&] {
    if (ps->n == 0) throw psg::invalid_argument("empty input");  // refscan.cpp:162
    *out = reinterpret_cast<psg_frnn_plan*>(psg::frnn_plan_create(ps, radius, q, f, seed, exclusion_zone));
  });
}
int psg_frnn_plan_scan(psg_frnn_plan* plan, uint64_t part, uint64_t nparts, int keep_pairs, uint64_t* pair_count,
                       uint64_t* pair_hash, psg_scan_stats* stats) {
  return guarded([&] {
    if (nparts == 0 || part >= nparts) throw psg::invalid_argument("part out of range");
    psg::FrnnPlan& p = *reinterpret_cast<psg::FrnnPlan*>(plan);
    psg::frnn_plan_scan(p, part, nparts, keep_pairs != 0);
    psg::frnn_plan_result(p, pair_count, pair_hash, stats);
  });
}
int psg_frnn_plan_pairs(psg_frnn_plan* plan, uint64_t nbuckets, uint64_t* bucket_counts, uint64_t* out,
                        uint64_t capacity) {
  return guarded([&] {
    if (nbuckets == 0) throw psg::invalid_argument("bucket count must be positive");
    psg::frnn_plan_pairs(*reinterpret_cast<psg::FrnnPlan*>(plan), nbuckets, bucket_counts, out, capacity);
  });
}
void psg_frnn_plan_free(psg_frnn_plan* plan) { psg::frnn_plan_free(reinterpret_cast<psg::FrnnPlan*>(plan)); }

// ---- host helpers ----------------------------------------------------------------
int psg_host_alloc(size_t bytes, void** out) {
  return guarded([&] { PSG_CUDA(cudaMallocHost(out, bytes)); });
}
void psg_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

}  // extern "C"

// ---- inspection (tests) -----------------------------------------------------------
int psg_debug_projection(psg_pointset* ps, uint64_t q, uint64_t seed, int* nk, float* keys, float* dirs,
                         double* key_error, double* scale) {
  return guarded([&] {
    if (!ps || !nk) throw psg::invalid_argument("null argument");
    const psg::Directions dir =
        psg::make_directions(seed, ps->d, static_cast<int>(std::min<uint64_t>(std::max<uint64_t>(q, 1), 1u << 20)));
    *nk = dir.nk;
    cudaStream_t s = psg::ctx().stream;
    psg::DevBuf<float> k(ps->n * dir.nk, s);
    psg::project(*ps, dir, k.p, s);
    const psg::Budget b = psg::make_budget(*ps, dir, ps->norm2max);  // as the solves charge it
    if (keys) PSG_CUDA(cudaMemcpyAsync(keys, k.p, ps->n * dir.nk * sizeof(float), cudaMemcpyDeviceToHost, s));
    PSG_CUDA(cudaStreamSynchronize(s));
    if (dirs) std::copy(dir.U.begin(), dir.U.end(), dirs);
    if (key_error) *key_error = b.E;
    if (scale) *scale = ps->scale;
  });
}

// ---- data formats --------------------------------------------------
int psg_load_series_text(const char* path, double** values, uint64_t* length) {
  return guarded_host([&] {
    if (!path || !values || !length) throw psg::invalid_argument("null argument");
    const std::vector<double> v = psg::load_series_text(path);
    double* out = static_cast<double*>(std::malloc(v.size() * sizeof(double)));
    if (!out) throw std::bad_alloc();
    std::copy(v.begin(), v.end(), out);
    *values = out;
    *length = v.size();
  });
}

int psg_save_series_text(const char* path, const double* values, uint64_t length) {
  return guarded_host([&] {
    if (!path || (!values && length)) throw psg::invalid_argument("null argument");
    psg::save_series_text(path, values, length);
  });
}

void psg_free(void* p) { std::free(p); }

int psg_save_binary(const char* path, const void* data, int dtype, uint64_t rows, uint64_t cols) {
  return guarded_host([&] {
    if (!path || (!data && rows * cols)) throw psg::invalid_argument("null argument");
    psg::save_binary(path, data, dtype, rows, cols);
  });
}

int psg_pointset_from_file(const char* path, psg_pointset** out) {
  return guarded([&] {
    if (!path || !out) throw psg::invalid_argument("null argument");
    psg::BinaryFile bf = psg::open_binary(path);
    require_dim(bf.cols);
    cudaStream_t s = psg::ctx().stream;
    psg::DevBuf<char> dev = upload_file(bf, s);
    *out = bf.dtype == 2 ? rows32(reinterpret_cast<const float*>(dev.p), bf.rows, bf.cols, true).release()
                         : rows64(reinterpret_cast<const double*>(dev.p), bf.rows, bf.cols, true).release();
  });
}

int psg_pointset_windows_from_file(const char* path, uint64_t len, int znorm, psg_pointset** out) {
  return guarded([&] {
    if (!path || !out) throw psg::invalid_argument("null argument");
    psg::BinaryFile bf = psg::open_binary(path);
    if (bf.cols != 1) throw psg::invalid_argument("a series file has one column");
    cudaStream_t s = psg::ctx().stream;
    psg::DevBuf<char> dev = upload_file(bf, s);
    *out = bf.dtype == 2 ? psg::pointset_windows(nullptr, reinterpret_cast<const float*>(dev.p), bf.rows, len,
                                                 znorm != 0, true)
                         : psg::pointset_windows(reinterpret_cast<const double*>(dev.p), nullptr, bf.rows, len,
                                                 znorm != 0, true);
  });
}
