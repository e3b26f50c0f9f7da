// pairscan_b200.hpp — C++ drop-in for the reference library's hot path, a
// header-only layer over the C ABI in pairscan_b200.h.
//
// Same names, argument meaning and error behaviour as the reference
// (/root/reference/proj/core/include/pairscan/{series,refscan}.hpp):
//   TimeSeries, PointSet::from_flat / windows_of, ReferenceSet, ScanStats,
//   PairResult, NeighborResult, build_reference_set, closest_pair,
//   brute_force_closest_pair, fixed_radius_neighbors, brute_force_neighbors,
//   reference_bound.  Contract violations throw std::invalid_argument with
//   the reference's messages; device failures throw std::runtime_error.
//
// Define PAIRSCAN_B200_AS_PAIRSCAN before including to make the names
// available as namespace `pairscan` (switch an existing caller by changing
// only its include and link line).
//
// Differences a caller can observe: ScanStats counts the GPU engine's work
// (FP64 rechecks / key-bound prunes / pairs outside the key cells) and still
// partitions the admissible pairs exactly; PointSet keeps a device-resident
// copy after the first solve.
#pragma once

#include <cmath>
#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "pairscan_b200.h"

namespace pairscan_b200 {

namespace detail {
inline void check(int rc) {
  if (rc == PSG_OK) return;
  const std::string msg = psg_last_error();
  if (rc == PSG_ERR_INVALID) throw std::invalid_argument(msg);
  if (rc == PSG_ERR_NOMEM) throw std::bad_alloc();
  throw std::runtime_error("pairscan_b200: " + msg);
}
struct PointsetFree {
  void operator()(psg_pointset* p) const { psg_pointset_free(p); }
};
}  // namespace detail

struct TimeSeries {
  std::vector<double> values;

  std::size_t length() const { return values.size(); }
  std::size_t window_count(std::size_t len) const {
    if (len == 0 || len > values.size()) throw std::invalid_argument("window length out of range");
    return values.size() - len + 1;
  }
  std::span<const double> window(std::size_t i, std::size_t len) const { return {values.data() + i, len}; }
};

inline void validate(const TimeSeries& s) {
  for (double v : s.values)
    if (!std::isfinite(v)) throw std::invalid_argument("series value must be finite");
}

class PointSet {
 public:
  static PointSet from_flat(std::vector<double> flat, std::size_t dim) {
    if (dim == 0) throw std::invalid_argument("point dimension must be positive");
    if (flat.size() % dim != 0) throw std::invalid_argument("flat buffer not a multiple of dim");
    for (double v : flat)
      if (!std::isfinite(v)) throw std::invalid_argument("point coordinate must be finite");
    PointSet ps;
    ps.owned_ = std::make_shared<std::vector<double>>(std::move(flat));
    ps.base_ = ps.owned_->data();
    ps.count_ = ps.owned_->size() / dim;
    ps.dim_ = dim;
    ps.stride_ = dim;
    return ps;
  }
  // Borrowed stride-1 window view; `series` must outlive the point set.
  static PointSet windows_of(const TimeSeries& series, std::size_t len) {
    PointSet ps;
    ps.count_ = series.window_count(len);
    ps.base_ = series.values.data();
    ps.series_len_ = series.values.size();
    ps.dim_ = len;
    ps.stride_ = 1;
    return ps;
  }

  std::size_t size() const { return count_; }
  std::size_t dim() const { return dim_; }
  std::span<const double> point(std::size_t i) const { return {base_ + i * stride_, dim_}; }

  // Device-resident copy, created on first use and reused by later solves.
  psg_pointset* device() const {
    if (!dev_) {
      psg_pointset* h = nullptr;
      if (stride_ == 1 && dim_ != 1 && !owned_)
        detail::check(psg_pointset_windows_f64(base_, series_len_, dim_, 0, 0, &h));
      else
        detail::check(psg_pointset_from_f64(base_, count_, dim_, 0, &h));
      dev_.reset(h, detail::PointsetFree{});
    }
    return dev_.get();
  }

 private:
  PointSet() = default;
  std::shared_ptr<std::vector<double>> owned_;
  const double* base_ = nullptr;
  std::size_t count_ = 0, dim_ = 0, stride_ = 0, series_len_ = 0;
  mutable std::shared_ptr<psg_pointset> dev_;
};

struct ReferenceSet {
  std::size_t q = 0;
  double f = 1.0;
  std::size_t dim = 0;
  std::vector<std::size_t> ref_indices;
  std::vector<double> references;  // q x dim
  std::vector<double> dist_table;  // q x n, k-major
  std::vector<std::size_t> order;
  double dist(std::size_t ref, std::size_t point_index, std::size_t n) const {
    return dist_table[ref * n + point_index];
  }
};

struct ScanStats {
  std::uint64_t pairs_examined = 0;
  std::uint64_t pairs_pruned_by_reference = 0;
  std::uint64_t pairs_skipped_by_exit = 0;
  std::uint64_t inner_loop_exits = 0;
  std::uint64_t admissible_pairs() const {
    return pairs_examined + pairs_pruned_by_reference + pairs_skipped_by_exit;
  }
};

struct PairResult {
  std::size_t index_i = 0;
  std::size_t index_j = 0;
  double distance = 0.0;
  ScanStats stats;
};

struct NeighborResult {
  std::vector<std::vector<std::size_t>> neighbors;
  ScanStats stats;
};

namespace detail {
inline ScanStats stats(const psg_scan_stats& s) {
  return {s.pairs_examined, s.pairs_pruned_by_reference, s.pairs_skipped_by_exit, s.inner_loop_exits};
}
inline PairResult pair(const psg_pair_result& r) {
  return {static_cast<std::size_t>(r.index_i), static_cast<std::size_t>(r.index_j), r.distance, stats(r.stats)};
}
inline NeighborResult lists(psg_neighbor_result& r) {
  NeighborResult out;
  out.stats = stats(r.stats);
  out.neighbors.resize(r.n);
  for (std::uint64_t i = 0; i < r.n; ++i)
    out.neighbors[i].assign(r.neighbors + r.offsets[i], r.neighbors + r.offsets[i + 1]);
  psg_neighbor_result_free(&r);
  return out;
}
inline std::vector<double> flat_copy(const PointSet& p) {
  std::vector<double> v(p.size() * p.dim());
  for (std::size_t i = 0; i < p.size(); ++i) {
    const auto x = p.point(i);
    std::copy(x.begin(), x.end(), v.begin() + i * p.dim());
  }
  return v;
}
}  // namespace detail

inline ReferenceSet build_reference_set(const PointSet& points, std::size_t q, double f, std::uint64_t seed) {
  const std::vector<double> flat = detail::flat_copy(points);
  const std::size_t n = points.size(), d = points.dim();
  ReferenceSet rs;
  rs.q = q;
  rs.f = f;
  rs.dim = d;
  std::vector<std::uint64_t> ri(q ? q : 1), ord(n ? n : 1);
  rs.references.resize(q * d);
  rs.dist_table.resize(q * n);
  detail::check(psg_build_reference_set_f64(flat.data(), n, d, q, f, seed, ri.data(), rs.references.data(),
                                            rs.dist_table.data(), ord.data()));
  rs.ref_indices.assign(ri.begin(), ri.begin() + q);
  rs.order.assign(ord.begin(), ord.begin() + n);
  return rs;
}

inline PairResult closest_pair(const PointSet& points, std::size_t q, double f, std::uint64_t seed,
                               std::size_t exclusion_zone) {
  if (points.size() < 2) throw std::invalid_argument("closest_pair needs at least 2 points");
  psg_pair_result r{};
  detail::check(psg_closest_pair_ps(points.device(), q, f, seed, exclusion_zone, &r));
  return detail::pair(r);
}

inline PairResult brute_force_closest_pair(const PointSet& points, std::size_t exclusion_zone) {
  if (points.size() < 2) throw std::invalid_argument("closest_pair needs at least 2 points");
  psg_pair_result r{};
  detail::check(psg_brute_force_closest_pair_ps(points.device(), exclusion_zone, &r));
  return detail::pair(r);
}

inline NeighborResult fixed_radius_neighbors(const PointSet& points, double radius, std::size_t q, double f,
                                             std::uint64_t seed, std::size_t exclusion_zone = 0) {
  if (points.size() == 0) throw std::invalid_argument("empty input");
  psg_neighbor_result r{};
  detail::check(psg_fixed_radius_neighbors_ps(points.device(), radius, q, f, seed, exclusion_zone, 1, &r));
  return detail::lists(r);
}

inline std::vector<std::vector<std::size_t>> brute_force_neighbors(const PointSet& points, double radius,
                                                                   std::size_t exclusion_zone = 0) {
  if (points.size() == 0) throw std::invalid_argument("empty input");
  const std::vector<double> flat = detail::flat_copy(points);
  psg_neighbor_result r{};
  detail::check(
      psg_brute_force_neighbors_f64(flat.data(), points.size(), points.dim(), radius, exclusion_zone, 1, &r));
  return detail::lists(r).neighbors;
}

inline double reference_bound(std::span<const double> r, std::span<const double> x, std::span<const double> y) {
  if (r.size() != x.size() || x.size() != y.size()) throw std::invalid_argument("dimension mismatch");
  double out = 0.0;
  detail::check(psg_reference_bound(r.data(), x.data(), y.data(), x.size(), &out));
  return out;
}

}  // namespace pairscan_b200

#ifdef PAIRSCAN_B200_AS_PAIRSCAN
namespace pairscan = pairscan_b200;
#endif
