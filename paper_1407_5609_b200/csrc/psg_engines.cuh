// psg_engines.cuh — the engines behind the C ABI besides the closest-pair
// scan: fixed-radius neighbours, brute force (device oracle and API), the
// exact reference set, and the reference bound.
#pragma once

#include "../../include/pairscan_b200.h"
#include "psg_internal.cuh"
#include "psg_points.cuh"

namespace psg {

// refscan.cpp:134-157 on device: exact over every admissible pair.
// upper >= 0: one pass over the pairs at FP64 distance <= upper (inspection)
psg_pair_result brute_solve(psg_pointset* ps, uint64_t zone, double upper = -1.0);

// refscan.cpp:159-209: cell grid on the first min(3, q) projection keys,
// FP32 filter + FP64 decision on the boundary band.
void frnn_solve(psg_pointset* ps, double radius, uint64_t q, double f, uint64_t seed, uint64_t zone,
                bool want_lists, psg_neighbor_result* out);
void frnn_pairs(psg_pointset* ps, double radius, uint64_t q, double f, uint64_t seed, uint64_t zone,
                uint64_t* pairs, uint64_t capacity, uint64_t* count, uint64_t* hash);
// The same list as upper-triangular CSR: offsets[n + 1] (row i = j > i,
// ascending) and the first `capacity` columns.
void frnn_pairs_csr(psg_pointset* ps, double radius, uint64_t q, double f, uint64_t seed, uint64_t zone,
                    uint64_t* offsets, uint32_t* cols, uint64_t capacity, uint64_t* count, uint64_t* hash);
// Sharded FRNN: the plan (projection + grid, identical on every rank), then
// per-part scans; a pair belongs to the part holding its earlier sorted
// position.  frnn_plan_pairs: the last scanned part's pairs, sorted, with
// per-i-range bucket counts (the all-to-all split of the sorted list).
struct FrnnPlan;
FrnnPlan* frnn_plan_create(psg_pointset* ps, double radius, uint64_t q, double f, uint64_t seed, uint64_t zone);
void frnn_plan_scan(FrnnPlan& plan, uint64_t part, uint64_t nparts, bool emit);
void frnn_plan_result(const FrnnPlan& plan, uint64_t* count, uint64_t* hash, psg_scan_stats* stats);
void frnn_plan_pairs(FrnnPlan& plan, uint64_t nbuckets, uint64_t* bucket_counts, uint64_t* out, uint64_t capacity);
void frnn_plan_free(FrnnPlan* plan);

// refscan.cpp:211-227 on device.
void brute_neighbors(psg_pointset* ps, double radius, uint64_t zone, bool want_lists, psg_neighbor_result* out);

// refscan.cpp:30-65, bit-exact.
void reference_set(psg_pointset* ps, uint64_t q, double f, uint64_t seed, uint64_t* ref_indices,
                   double* references, double* table, uint64_t* order);
// refscan.cpp:229-232.
double reference_bound_dev(const double* r, const double* x, const double* y, uint64_t d);

}  // namespace psg
