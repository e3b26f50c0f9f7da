// psg_cpp.cuh — the closest-pair engine (refscan.cpp:67-132 closest_pair) and
// the pieces the fixed-radius engine shares with it.
#pragma once

#include <memory>

#include "../../include/pairscan_b200.h"
#include "psg_dense.cuh"
#include "psg_grid.cuh"
#include "psg_internal.cuh"
#include "psg_points.cuh"

namespace psg {

// Per-call profile (filled by the engines, copied out by psg_last_profile).
extern thread_local psg_profile g_prof;
void prof_begin();
void prof_stages(const StageTimer& t);

// Projection of the FP32 working rows onto the seeded directions:
// keys[i*nk + k] = <U_k, X_i>; max ||X_i||^2 (FP32 bits) is atomically maxed
// into *norm2_bits (device).  Enqueued only.
// With cc.gp set, shapes that can count cells while projecting do so (and
// return true): cell id and arrival rank of every row (CellCount).
bool project_async(const psg_pointset& ps, const Directions& dir, float* keys, unsigned* norm2_bits,
                   cudaStream_t s, const CellCount& cc = CellCount{});
// The tensor-core projection (psg_project_tc.cu): tc_projection(d, n) shapes.
void project_tc(const psg_pointset& ps, const Directions& dir, float* keys, unsigned* norm2_bits, cudaStream_t s,
                const CellCount& cc);
// Window sets (virtual rows): CUDA-core projection from the series.
void project_windows(const psg_pointset& ps, const Directions& dir, float* keys, unsigned* norm2_bits, cudaStream_t s,
                     const CellCount& cc = CellCount{});
const float* window_directions(const psg_pointset& ps, const Directions& dir, cudaStream_t s);
// Host-synchronous variant: returns max ||X_i||^2.
float project(const psg_pointset& ps, const Directions& dir, float* keys, cudaStream_t s);
// Error budget for the keys of `ps` under `dir` (host).
Budget make_budget(const psg_pointset& ps, const Directions& dir, float max_norm2);

// Device-resident solve state: every threshold and counter the kernels need,
// so a solve is enqueued with two host synchronisations (after the bootstrap,
// at the end).
struct DevState {
  // (FP64 distance bits, (i << 32) | j) minimum of the band pairs past the
  // candidate list, evaluated inline (record(), psg_scan.cuh): [0] lo, [1] hi
  alignas(16) unsigned long long best128[2];
  unsigned long long cand_n;  // band pairs recorded (may exceed the list capacity)
  unsigned pre_ticket;  // k_presample's last-block ticket
  unsigned norm2_bits;  // max ||x||^2 (FP32 bits), from the projection
  unsigned best;        // FP32 bits of the best squared distance seen
  unsigned regrid;      // set by k_check_grid: cells narrower than the bound's key window
  unsigned check_best;  // FP32 bits of the bound k_check_grid tested
  Thresholds th;        // the scan's starting thresholds (from check_best)
  unsigned long long best64, lex, examined, evals, visited, inline_n;
  Budget bud;
  double box_lo[kMaxGridKeys], box_span[kMaxGridKeys];
  InlineCtx ic;  // set by k_state_init
};

// Buffers reused by every solve on one point set (per key count).
struct CppWork {
  uint32_t n = 0;
  int nk = 0;
  DevBuf<float> keys;      // n x nk, original order
  GridIndex gi;            // grid engine
  DevBuf<float> wskeys;    // window engine: keys in key-0 order
  DevBuf<uint32_t> wsidx, wk0, wk1, wv0, wv1, whist;
  DevBuf<DevState> st;
  DevState* host_st = nullptr;  // pinned mirror
  DevBuf<uint32_t> cand_p, cand_j;
  DevBuf<float> cand_s;
  DevBuf<double> d64;
  uint32_t cand_cap = 0;
  DenseWork dense;         // dense cell-pair engine (clustered data)
  DevBuf<double> pre_part; // k_presample's per-block key moments
  // The whole single-part grid solve captured once as a CUDA graph and
  // replayed by later solves with the same (q, seed, zone) on this point set.
  // Its kernels hold the buffer pointers of capture time: any reallocation
  // (ensure_candidates, GridIndex::ensure) destroys it (drop_graph).
  cudaGraphExec_t gexec = nullptr;
  uint64_t gq = 0, gseed = 0, gzone = 0;
  uint32_t gcap = 0;  // cand_cap at capture
  int glevel = -1;    // graph_profiling() at capture
  uint64_t glaunches = 0;
  uint64_t solves = 0;  // closest-pair solves on this point set (the first one is not captured)
  // cell width a regrid converged to, for the same (q, seed, zone)
  double learned_w = 0.0;
  uint64_t learned_q = 0, learned_seed = 0, learned_zone = 0;
  bool learned_dense = false;  // the solve went to the dense engine (not graph-capturable: host decisions)
  bool learned_full_boot = false;  // the own-row bootstrap was too weak: run the full-stencil one up front
  bool learned_brute = false;  // the grid could not separate the pairs: later solves go to the all-pairs engine
  cudaEvent_t gev[32] = {};  // event nodes recorded inside the graph (spans and stages)
  std::vector<CapMark> gspans, gstages;  // which gev pairs time which span / stage
  void drop_graph();
  ~CppWork();
};

struct CppPlan {
  psg_pointset* ps = nullptr;
  uint64_t zone = 0;
  uint64_t q_arg = 0, seed_arg = 0;  // the call's q and seed (learned-width key)
  Directions dir;
  Budget bud;              // host copy (valid after the first readback)
  GridParams gp;           // host copy of the grid parameters
  // engine "window": keys sorted by key 0, candidates = the key-0 window
  // engine "grid":   keys sorted by cell of the first g keys (psg_grid.cuh)
  bool grid = false;
  bool dense = false;      // grid engine: cell-pair tiles instead of per-point candidates
  bool exact_scan = false; // sparse engines: rescan with inline FP64 for every band pair (list overflow)
  bool boot_lb = false;    // the grid build left per-warp bootstrap lower bounds (BootLB)
  bool rescued = false;    // the full-stencil bootstrap already ran after a failed cell check
  bool sharded = false;    // a part plan: no learned hints (cpp_plan_create)
  int g = 0;
  std::shared_ptr<CppWork> work;
  uint32_t width = 0;      // window engine: bootstrap width (sorted neighbours)
  std::unique_ptr<StageTimer> prep_tm;   // plan_create's stages, read at the first sync
  std::unique_ptr<KernelSpan> proj_span, boot_span;
  bool sync_bootstrap = true;  // false inside cpp_solve: bootstrap -> scan without a host round trip
};

// sharded = a key-range part plan (psg_cpp_plan_*): ignores the hints learned
// by earlier solves on this point set, so every rank builds the same grid.
CppPlan* cpp_plan_create(psg_pointset* ps, uint64_t q, double f, uint64_t seed, uint64_t zone,
                         bool sharded = false);
float cpp_plan_bootstrap(CppPlan& plan, uint64_t part, uint64_t nparts);
// Result: index_i == UINT64_MAX when the part has no admissible pair.
psg_pair_result cpp_plan_scan(CppPlan& plan, uint64_t part, uint64_t nparts, float bound_s32);
psg_pair_result cpp_solve(psg_pointset* ps, uint64_t q, double f, uint64_t seed, uint64_t zone);

// Validation shared with the reference contract (refscan.cpp:33-35).
void check_reference_args(uint64_t n, uint64_t q, double f);

}  // namespace psg
