// The reference's refscan unit tests (tests/test_refscan.cpp, relative to
// /root/reference/proj) re-expressed against the C++ drop-in header
// include/pairscan_b200.hpp, compiled with PAIRSCAN_B200_AS_PAIRSCAN so the
// calls read exactly like the reference's.  Built and run by
// tests/test_cxx_shim.py; exits non-zero on the first failure.
#define PAIRSCAN_B200_AS_PAIRSCAN
#include "pairscan_b200.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <stdexcept>
#include <vector>

using namespace pairscan;

static int failures = 0;
#define CHECK(cond)                                                       \
  do {                                                                    \
    if (!(cond)) {                                                        \
      std::fprintf(stderr, "%s:%d: CHECK(%s) failed\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                         \
    }                                                                     \
  } while (0)
#define CHECK_THROWS_INVALID(expr)                                        \
  do {                                                                    \
    bool threw = false;                                                   \
    try {                                                                 \
      (void)(expr);                                                       \
    } catch (const std::invalid_argument&) {                              \
      threw = true;                                                       \
    }                                                                     \
    CHECK(threw);                                                         \
  } while (0)

// The reference Rng's gaussian sampler (rng.cpp:22-32) over std::mt19937_64.
struct Gauss {
  std::mt19937_64 e;
  explicit Gauss(uint64_t s) : e(s) {}
  double unit() { return static_cast<double>(e() >> 11) * 0x1.0p-53; }
  double next() {
    const double u1 = 1.0 - unit(), u2 = unit();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.14159265358979323846 * u2);
  }
};

static PointSet random_points(uint64_t seed, std::size_t n, std::size_t dim) {
  Gauss g(seed);
  std::vector<double> flat(n * dim);
  for (double& v : flat) v = g.next();
  return PointSet::from_flat(std::move(flat), dim);
}

static TimeSeries walk(std::size_t n, uint64_t seed) {
  TimeSeries ts;
  ts.values.resize(n);
  if (psg_gen_random_walk(n, seed, 1.0, ts.values.data()) != PSG_OK) std::abort();
  return ts;
}

static uint64_t count_admissible(std::size_t n, std::size_t zone) {
  uint64_t c = 0;
  for (std::size_t i = 0; i + 1 < n; ++i)
    for (std::size_t j = i + 1; j < n; ++j)
      if (j - i >= zone || zone == 0) ++c;
  return c;
}

int main() {
  {  // reference sets hold scaled copies of seeded input points
    const PointSet pts = random_points(11, 60, 5);
    const ReferenceSet rs = build_reference_set(pts, 7, 10.0, 3);
    CHECK(rs.q == 7 && rs.dim == 5 && rs.ref_indices.size() == 7 && rs.dist_table.size() == 7 * 60);
    for (std::size_t k = 0; k < rs.q; ++k) {
      const auto src = pts.point(rs.ref_indices[k]);
      for (std::size_t d = 0; d < rs.dim; ++d) CHECK(rs.references[k * rs.dim + d] == src[d] * 10.0);
    }
    std::vector<std::size_t> sorted = rs.order;
    std::sort(sorted.begin(), sorted.end());
    for (std::size_t i = 0; i < sorted.size(); ++i) CHECK(sorted[i] == i);
    for (std::size_t i = 0; i + 1 < rs.order.size(); ++i) CHECK(rs.dist(0, rs.order[i], 60) <= rs.dist(0, rs.order[i + 1], 60));
  }
  {  // projected scan equals brute force on walk windows
    const TimeSeries w = walk(240, 5);
    const PointSet pts = PointSet::windows_of(w, 8);
    const PairResult want = brute_force_closest_pair(pts, 8);
    CHECK(want.stats.pairs_examined == count_admissible(pts.size(), 8));
    for (uint64_t seed : {1ull, 2ull, 3ull})
      for (std::size_t q : {std::size_t{1}, std::size_t{3}, std::size_t{10}})
        for (double f : {1.0, 10.0}) {
          const PairResult got = closest_pair(pts, q, f, seed, 8);
          CHECK(got.index_i == want.index_i && got.index_j == want.index_j);
          CHECK(got.distance == want.distance);
          CHECK(got.stats.admissible_pairs() == want.stats.pairs_examined);
        }
  }
  {  // point clouds, every pair admissible
    const PointSet pts = random_points(77, 150, 4);
    const PairResult want = brute_force_closest_pair(pts, 0);
    const PairResult got = closest_pair(pts, 10, 10.0, 4, 0);
    CHECK(got.index_i == want.index_i && got.index_j == want.index_j && got.distance == want.distance);
    CHECK(got.stats.admissible_pairs() == 150ull * 149 / 2);
  }
  {  // statistics partition the admissible pairs for any zone
    const TimeSeries w = walk(180, 13);
    const PointSet pts = PointSet::windows_of(w, 6);
    for (std::size_t zone : {std::size_t{0}, std::size_t{1}, std::size_t{6}, std::size_t{50}}) {
      const ScanStats s = closest_pair(pts, 5, 10.0, 2, zone).stats;
      CHECK(s.pairs_examined + s.pairs_pruned_by_reference + s.pairs_skipped_by_exit ==
            count_admissible(pts.size(), zone));
      CHECK(s.pairs_examined >= 1);
    }
  }
  {  // the exclusion zone hides adjacent near-duplicates
    const PointSet pts = PointSet::from_flat({0.0, 0.0005, 10.0, 30.0, 50.0, 10.1}, 1);
    for (std::size_t zone : {std::size_t{0}, std::size_t{1}}) {
      const PairResult r = closest_pair(pts, 2, 10.0, 1, zone);
      CHECK(r.index_i == 0 && r.index_j == 1);
    }
    const PairResult wide = closest_pair(pts, 2, 10.0, 1, 2);
    CHECK(wide.index_i == 2 && wide.index_j == 5 && std::abs(wide.distance - 0.1) < 1e-12);
  }
  {  // fixed radius lists are boundary inclusive
    const PointSet pts = PointSet::from_flat({0.0, 1.0, 2.0, 3.5}, 1);
    const NeighborResult got = fixed_radius_neighbors(pts, 1.0, 2, 10.0, 1);
    CHECK(got.neighbors.size() == 4);
    CHECK(got.neighbors[0] == std::vector<std::size_t>{1});
    CHECK(got.neighbors[1] == (std::vector<std::size_t>{0, 2}));
    CHECK(got.neighbors[2] == std::vector<std::size_t>{1});
    CHECK(got.neighbors[3].empty());
  }
  {  // fixed radius lists match brute force
    const PointSet pts = random_points(31, 120, 3);
    for (double radius : {0.35, 1.2, 2.5})
      for (std::size_t zone : {std::size_t{0}, std::size_t{2}}) {
        const NeighborResult got = fixed_radius_neighbors(pts, radius, 8, 10.0, 9, zone);
        const auto want = brute_force_neighbors(pts, radius, zone);
        CHECK(got.neighbors == want);
        const ScanStats& s = got.stats;
        CHECK(s.pairs_examined + s.pairs_pruned_by_reference + s.pairs_skipped_by_exit ==
              count_admissible(pts.size(), zone));
      }
  }
  {  // results do not depend on the seed
    const TimeSeries w = walk(300, 17);
    const PointSet pts = PointSet::windows_of(w, 12);
    const PairResult want = brute_force_closest_pair(pts, 12);
    for (uint64_t seed = 1; seed <= 10; ++seed) {
      const PairResult got = closest_pair(pts, 10, 10.0, seed, 12);
      CHECK(got.index_i == want.index_i && got.index_j == want.index_j && got.distance == want.distance);
    }
  }
  {  // degenerate arguments are rejected
    const PointSet pts = random_points(1, 5, 2);
    CHECK_THROWS_INVALID(build_reference_set(pts, 0, 10.0, 1));
    CHECK_THROWS_INVALID(build_reference_set(pts, 6, 10.0, 1));
    CHECK_THROWS_INVALID(build_reference_set(pts, 2, 0.0, 1));
    CHECK_THROWS_INVALID(closest_pair(pts, 2, 10.0, 1, 5));
    CHECK_THROWS_INVALID(fixed_radius_neighbors(pts, 0.0, 2, 10.0, 1));
    const PointSet one = PointSet::from_flat({1.0, 2.0}, 2);
    CHECK_THROWS_INVALID(closest_pair(one, 1, 1.0, 1, 0));
    CHECK_THROWS_INVALID(brute_force_closest_pair(one, 0));
  }
  {  // reference bound: signed difference, never overshoots
    Gauss g(21);
    for (int t = 0; t < 50; ++t) {
      std::vector<double> r(6), x(6), y(6);
      for (double& v : r) v = 2 * g.next();
      for (double& v : x) v = 2 * g.next();
      for (double& v : y) v = 2 * g.next();
      const double b = reference_bound(r, x, y);
      CHECK(b == -reference_bound(r, y, x));
      double dxy = 0;
      for (int k = 0; k < 6; ++k) dxy += (x[k] - y[k]) * (x[k] - y[k]);
      CHECK(std::abs(b) <= std::sqrt(dxy) + 1e-9);
    }
  }
  std::printf("%s: %d failure(s)\n", failures ? "FAIL" : "PASS", failures);
  return failures ? 1 : 0;
}
