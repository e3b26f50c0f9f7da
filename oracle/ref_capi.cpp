// ref_capi.cpp — a C entry-point wrapper around the UNMODIFIED reference
// library, compiled together with /root/reference/proj/core/src/*.cpp by
// oracle/Makefile into oracle/_ref/libpairscan_ref.so.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  Used by tests/ to pin the C oracle
// restatement and to generate golden fixtures, and by bench.py's
// cpu_baseline / --impl reference legs to time the reference's own CPU path.
// Nothing in paper_1407_5609_b200/ loads it.
//
// Every function returns 0 on success and -1 when the reference threw
// std::invalid_argument (message retrievable with ref_last_error()).

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "pairscan/datagen.hpp"
#include "pairscan/io.hpp"
#include "pairscan/metrics.hpp"
#include "pairscan/refscan.hpp"
#include "pairscan/rng.hpp"
#include "pairscan/series.hpp"

using namespace pairscan;

namespace {
thread_local std::string g_err;

struct RefPair {
  uint64_t index_i, index_j;
  double distance;
  uint64_t pairs_examined, pairs_pruned_by_reference, pairs_skipped_by_exit, inner_loop_exits;
};

void fill(const PairResult& r, RefPair* out) {
  out->index_i = r.index_i;
  out->index_j = r.index_j;
  out->distance = r.distance;
  out->pairs_examined = r.stats.pairs_examined;
  out->pairs_pruned_by_reference = r.stats.pairs_pruned_by_reference;
  out->pairs_skipped_by_exit = r.stats.pairs_skipped_by_exit;
  out->inner_loop_exits = r.stats.inner_loop_exits;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return -1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -2;
  }
}

PointSet flat_points(const double* pts, uint64_t n, uint64_t d) {
  return PointSet::from_flat(std::vector<double>(pts, pts + n * d), d);
}

void summarise(const std::vector<std::vector<std::size_t>>& lists, uint64_t* count, uint64_t* hash,
               uint64_t* pairs, uint64_t cap) {
  uint64_t c = 0, h = 0;
  for (std::size_t i = 0; i < lists.size(); ++i)
    for (std::size_t j : lists[i])
      if (j > i) {
        const uint64_t key = (static_cast<uint64_t>(i) << 32) | j;
        if (pairs && c < cap) pairs[c] = key;
        ++c;
        h += mix_seed(key);
      }
  *count = c;
  *hash = h;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_rng_stream(uint64_t seed, uint64_t count, uint64_t* out) {
  Rng r(seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = r.next_u64();
}
void ref_gaussian_stream(uint64_t seed, double mean, double sd, uint64_t count, double* out) {
  Rng r(seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = r.gaussian(mean, sd);
}
void ref_uniform_below_stream(uint64_t seed, uint64_t bound, uint64_t count, uint64_t* out) {
  Rng r(seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = r.uniform_below(bound);
}
int ref_sample_without_replacement(uint64_t seed, uint64_t n, uint64_t k, uint64_t* out) {
  return guarded([&] {
    Rng r(seed);
    const auto v = r.sample_without_replacement(n, k);
    for (uint64_t i = 0; i < k; ++i) out[i] = v[i];
  });
}
uint64_t ref_mix_seed(uint64_t x) { return mix_seed(x); }
uint64_t ref_derive_seed(uint64_t base, uint64_t stream) { return derive_seed(base, stream); }

int ref_gen_random_walk(uint64_t n, uint64_t seed, double sd, double* out) {
  return guarded([&] {
    const TimeSeries ts = gen_random_walk(n, seed, sd);
    std::memcpy(out, ts.values.data(), n * sizeof(double));
  });
}

double ref_euclidean(const double* x, const double* y, uint64_t d) {
  return euclidean_distance({x, d}, {y, d});
}
int ref_euclidean_early_abandon(const double* x, const double* y, uint64_t d, double thr,
                                double* out) {
  const auto r = euclidean_distance_early_abandon({x, d}, {y, d}, thr);
  if (!r) return 0;
  *out = *r;
  return 1;
}
double ref_reference_bound(const double* r, const double* x, const double* y, uint64_t d) {
  return reference_bound({r, d}, {x, d}, {y, d});
}

int ref_closest_pair(const double* pts, uint64_t n, uint64_t d, uint64_t q, double f,
                     uint64_t seed, uint64_t zone, RefPair* out) {
  return guarded([&] { fill(closest_pair(flat_points(pts, n, d), q, f, seed, zone), out); });
}
int ref_brute_force_closest_pair(const double* pts, uint64_t n, uint64_t d, uint64_t zone,
                                 RefPair* out) {
  return guarded([&] { fill(brute_force_closest_pair(flat_points(pts, n, d), zone), out); });
}
// The reference's motif path: closest_pair over PointSet::windows_of (raw windows).
int ref_closest_pair_windows(const double* series, uint64_t N, uint64_t len, uint64_t q, double f,
                             uint64_t seed, uint64_t zone, RefPair* out) {
  return guarded([&] {
    TimeSeries ts;
    ts.values.assign(series, series + N);
    fill(closest_pair(PointSet::windows_of(ts, len), q, f, seed, zone), out);
  });
}
int ref_brute_force_closest_pair_windows(const double* series, uint64_t N, uint64_t len,
                                         uint64_t zone, RefPair* out) {
  return guarded([&] {
    TimeSeries ts;
    ts.values.assign(series, series + N);
    fill(brute_force_closest_pair(PointSet::windows_of(ts, len), zone), out);
  });
}

// FRNN: count/hash of pairs i<j, optional pair list, plus the scan stats.
int ref_fixed_radius_neighbors(const double* pts, uint64_t n, uint64_t d, double radius,
                               uint64_t q, double f, uint64_t seed, uint64_t zone,
                               uint64_t* count, uint64_t* hash, uint64_t* pairs, uint64_t cap,
                               uint64_t* stats4) {
  return guarded([&] {
    const NeighborResult r = fixed_radius_neighbors(flat_points(pts, n, d), radius, q, f, seed, zone);
    summarise(r.neighbors, count, hash, pairs, cap);
    if (stats4) {
      stats4[0] = r.stats.pairs_examined;
      stats4[1] = r.stats.pairs_pruned_by_reference;
      stats4[2] = r.stats.pairs_skipped_by_exit;
      stats4[3] = r.stats.inner_loop_exits;
    }
  });
}
int ref_brute_force_neighbors(const double* pts, uint64_t n, uint64_t d, double radius,
                              uint64_t zone, uint64_t* count, uint64_t* hash, uint64_t* pairs,
                              uint64_t cap) {
  return guarded([&] {
    summarise(brute_force_neighbors(flat_points(pts, n, d), radius, zone), count, hash, pairs, cap);
  });
}

int ref_build_reference_set(const double* pts, uint64_t n, uint64_t d, uint64_t q, double f,
                            uint64_t seed, uint64_t* ref_indices, double* references,
                            double* table, uint64_t* order) {
  return guarded([&] {
    const ReferenceSet rs = build_reference_set(flat_points(pts, n, d), q, f, seed);
    for (uint64_t k = 0; k < q; ++k) ref_indices[k] = rs.ref_indices[k];
    std::memcpy(references, rs.references.data(), q * d * sizeof(double));
    std::memcpy(table, rs.dist_table.data(), q * n * sizeof(double));
    for (uint64_t i = 0; i < n; ++i) order[i] = rs.order[i];
  });
}

// io.cpp:44-60 / 62-70: the series text format.  Returns 0, -1 (invalid_argument)
// or -2 (runtime_error); *out is malloc'd.
int ref_load_series(const char* path, double** out, uint64_t* n) {
  return guarded([&] {
    const TimeSeries ts = load_series(path);
    *n = ts.values.size();
    *out = static_cast<double*>(std::malloc(ts.values.size() * sizeof(double)));
    std::memcpy(*out, ts.values.data(), ts.values.size() * sizeof(double));
  });
}

int ref_save_series(const double* v, uint64_t n, const char* path) {
  return guarded([&] {
    TimeSeries ts;
    ts.values.assign(v, v + n);
    save_series(ts, path);
  });
}

void ref_free(void* p) { std::free(p); }

// io.cpp:177-225: one Report rendered as JSON (report_to_json) and CSV
// (reports_to_csv); both strings malloc'd.
int ref_report_render(const char* algorithm, const char* params, const char* dataset, uint64_t i1, uint64_t i2,
                      double dom, uint64_t examined, uint64_t iterations, double wall, uint64_t seed, char** json,
                      char** csv) {
  return guarded([&] {
    Report r;
    r.algorithm = algorithm;
    r.params = params;
    r.dataset = dataset;
    r.pair_index_1 = i1;
    r.pair_index_2 = i2;
    r.distance_or_matches = dom;
    r.pairs_examined = examined;
    r.iterations = iterations;
    r.wall_seconds = wall;
    r.seed = seed;
    const std::string j = report_to_json(r), c = reports_to_csv({r});
    *json = strdup(j.c_str());
    *csv = strdup(c.c_str());
  });
}

uint64_t ref_derive_seed3(uint64_t base, uint64_t s1, uint64_t s2) { return derive_seed(base, s1, s2); }

}  // extern "C"
