// psg_cpp.cuh — the closest-pair engine (refscan.cpp:67-132 closest_pair) and
// the pieces the fixed-radius engine shares with it.
#pragma once

#include "../../include/pairscan_b200.h"
#include "psg_grid.cuh"
#include "psg_internal.cuh"
#include "psg_points.cuh"

namespace psg {

// Per-call profile (filled by the engines, copied out by psg_last_profile).
extern thread_local psg_profile g_prof;
void prof_begin();
void prof_stages(const StageTimer& t);

// Projection of the FP32 working rows onto the seeded directions:
// keys[i*nk + k] = <U_k, X_i>.  Returns max ||X_i||^2 (FP32 upper bound).
float project(const psg_pointset& ps, const Directions& dir, float* keys, cudaStream_t s);
// Error budget for the keys of `ps` under `dir`.
Budget make_budget(const psg_pointset& ps, const Directions& dir, float max_norm2);

struct CppPlan {
  psg_pointset* ps = nullptr;
  uint64_t zone = 0;
  Directions dir;
  Budget bud;
  // engine "window": keys sorted by key 0, candidates = the key-0 window
  // engine "grid":   keys sorted by cell of the first g keys (psg_grid.cuh)
  bool grid = false;
  DevBuf<float> skeys;     // window engine: n x nk keys in key-0 order (AoS)
  DevBuf<uint32_t> sidx;   // window engine: sorted position -> original index
  DevBuf<float> keys;      // grid engine: unsorted keys, kept for a rebuild
  GridIndex gi;            // grid engine
  int g = 0;
  double box_lo[3] = {0, 0, 0}, box_span[3] = {0, 0, 0};
  DevBuf<unsigned> best;   // FP32 bits of the best squared distance seen
  uint32_t width = 0;      // bootstrap width (sorted neighbours)
  float prep_ms[3] = {0, 0, 0};
};

CppPlan* cpp_plan_create(psg_pointset* ps, uint64_t q, double f, uint64_t seed, uint64_t zone);
float cpp_plan_bootstrap(CppPlan& plan, uint64_t part, uint64_t nparts);
// Result: index_i == UINT64_MAX when the part has no admissible pair.
psg_pair_result cpp_plan_scan(CppPlan& plan, uint64_t part, uint64_t nparts, float bound_s32);
psg_pair_result cpp_solve(psg_pointset* ps, uint64_t q, double f, uint64_t seed, uint64_t zone);

// Validation shared with the reference contract (refscan.cpp:33-35).
void check_reference_args(uint64_t n, uint64_t q, double f);

}  // namespace psg
