/*
 * pairscan_b200.h — C ABI of the B200 (sm_100a) exact pair-search library.
 *
 * It replaces the hot path of the reference C++ library `pairscan`
 * (paths below relative to /root/reference/proj):
 *
 *   core/include/pairscan/refscan.hpp:50-51  build_reference_set  -> psg_build_reference_set_f64
 *   core/include/pairscan/refscan.hpp:55-56  closest_pair          -> psg_closest_pair_f64 / _f32
 *   core/include/pairscan/refscan.hpp:58     brute_force_closest_pair -> psg_brute_force_closest_pair_f64
 *   core/include/pairscan/refscan.hpp:61-63  fixed_radius_neighbors -> psg_fixed_radius_neighbors_f64 / _f32
 *   core/include/pairscan/refscan.hpp:65-66  brute_force_neighbors -> psg_brute_force_neighbors_f64
 *   core/include/pairscan/refscan.hpp:70-71  reference_bound       -> psg_reference_bound
 *   core/include/pairscan/series.hpp:30-31   PointSet::from_flat / windows_of -> psg_pointset_*
 *   tools/src/main.cpp:332-346 (cmd_motif: closest_pair over windows_of)   -> psg_motif_f64 / _f32
 *
 * Conventions
 *  - Plain pointers and sizes only; all host buffers are caller-owned except
 *    the arrays inside psg_neighbor_result, released by psg_neighbor_result_free.
 *  - Every entry returns PSG_OK or an error code.  PSG_ERR_INVALID carries the
 *    reference's std::invalid_argument message verbatim (psg_last_error()).
 *  - Results are the reference's exactly: indices bit-exact (ties to the
 *    lowest (i, j)), distances computed in the reference's FP64 order.
 *  - The library runs on the calling thread's current CUDA device, on its own
 *    stream, and is synchronous at return.  There is no CPU fallback: without
 *    a usable sm_100 device every compute entry returns PSG_ERR_CUDA.
 */
#ifndef PAIRSCAN_B200_H
#define PAIRSCAN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PSG_OK 0
#define PSG_ERR_INVALID 1 /* reference std::invalid_argument */
#define PSG_ERR_CUDA 2    /* CUDA runtime / device failure */
#define PSG_ERR_NOMEM 3
#define PSG_ERR_INTERNAL 4
#define PSG_ERR_IO 5      /* reference std::runtime_error from io.cpp (file open / parse) */

/* refscan.hpp:27-36 ScanStats */
typedef struct psg_scan_stats {
  uint64_t pairs_examined;            /* pairs re-evaluated in the reference's FP64 arithmetic */
  uint64_t pairs_pruned_by_reference; /* inside the final key window, removed by key/FP32 bounds */
  uint64_t pairs_skipped_by_exit;     /* outside the final key window */
  uint64_t inner_loop_exits;          /* rows whose key window ended before the last point */
} psg_scan_stats;

/* refscan.hpp:38-43 PairResult */
typedef struct psg_pair_result {
  uint64_t index_i; /* original indices, index_i < index_j */
  uint64_t index_j;
  double distance;
  psg_scan_stats stats;
} psg_pair_result;

/* refscan.hpp:45-48 NeighborResult as CSR: neighbors of i are
 * neighbors[offsets[i] .. offsets[i+1]), ascending, symmetric.
 * pair_count = #{i<j}, pair_hash = sum of mix_seed((i<<32)|j) mod 2^64. */
typedef struct psg_neighbor_result {
  uint64_t n;
  uint64_t* offsets;   /* n+1, or NULL when only counts were requested */
  uint64_t* neighbors; /* offsets[n] entries */
  uint64_t pair_count;
  uint64_t pair_hash;
  psg_scan_stats stats;
} psg_neighbor_result;

/* Per-call measurements of the last compute entry on this thread. */
typedef struct psg_profile {
  int stages;
  char stage_name[16][24];
  float stage_ms[16];        /* CUDA-event time of each stage on the library stream */
  uint64_t launches;         /* kernels launched by the library in the call */
  uint64_t window_pairs;     /* pairs inside the final key-0 window */
  uint64_t lb_survivors;     /* pairs that reached an FP32 distance evaluation */
  uint64_t candidates;       /* FP32 band candidates sent to FP64 recheck */
  uint64_t bootstrap_width;  /* sorted-neighbour width of the delta bootstrap */
  uint64_t h2d_bytes, d2h_bytes;
  double scan_kernel_ms;     /* device time of the candidate (window) kernel(s) */
  double project_kernel_ms;  /* device time of the projection kernel */
  double bootstrap_kernel_ms;/* device time of the delta-bootstrap kernel(s) */
  double total_ms;           /* device span of the whole call on the library stream */
  uint64_t scan_launches;    /* launches of the candidate kernel */
  /* dense cell-pair engine (clustered data) of the last solve; 0 when unused */
  uint64_t dense_cells;        /* cells of the dense grid (up to 2^27) */
  uint64_t dense_cell_pairs;   /* kept (A, B) cell pairs */
  uint64_t dense_groups;       /* Gram groups (an A cell and <= 366 partners) */
  uint64_t dense_split_groups; /* groups that continue an A cell with more than 366 kept partners */
  uint64_t dense_tiles;        /* 128 x 128 Gram tiles issued */
  uint64_t inline_fp64;        /* band pairs past the candidate list, evaluated inline in FP64 */
} psg_profile;

const char* psg_last_error(void);
const char* psg_version(void);
int psg_last_profile(psg_profile* out);
/* Whether CUDA device `device` is usable (compute capability 10.x). */
int psg_device_ok(int device);
/* The library's cudaStream_t on the current device (for callers that want to
 * bracket calls with their own CUDA events); NULL on failure. */
void* psg_stream(void);
/* Select the CUDA device for this thread's subsequent calls (one process per
 * GPU: pass LOCAL_RANK). */
int psg_set_device(int device);
/* Timing inside the captured solves that repeated calls on a point set
 * replay: 0 (default) none — the fastest replay; 1 the projection, bootstrap
 * and scan spans (psg_profile.*_kernel_ms); 2 also every stage
 * (psg_profile.stage_*).  Each event node costs ~5 us of device time per
 * solve.  Graphs captured at another level are recaptured on their next use. */
int psg_set_graph_profiling(int level);

/* ---- one-shot entries (host buffers in, result out) --------------------- */
int psg_closest_pair_f64(const double* points, uint64_t n, uint64_t dim, uint64_t q, double f,
                         uint64_t seed, uint64_t exclusion_zone, psg_pair_result* out);
int psg_closest_pair_f32(const float* points, uint64_t n, uint64_t dim, uint64_t q, double f,
                         uint64_t seed, uint64_t exclusion_zone, psg_pair_result* out);
int psg_brute_force_closest_pair_f64(const double* points, uint64_t n, uint64_t dim,
                                     uint64_t exclusion_zone, psg_pair_result* out);
int psg_brute_force_closest_pair_f32(const float* points, uint64_t n, uint64_t dim,
                                     uint64_t exclusion_zone, psg_pair_result* out);

/* Motif: closest pair over the length-`len` windows of a series.  znorm=0 is
 * the reference's raw windows (series.cpp:34-42); znorm=1 z-normalises every
 * window in FP64 (two-pass mean, population sigma, 0 when sigma==0). */
int psg_motif_f64(const double* series, uint64_t length, uint64_t len, int znorm, uint64_t q,
                  double f, uint64_t seed, uint64_t exclusion_zone, psg_pair_result* out);
int psg_motif_f32(const float* series, uint64_t length, uint64_t len, int znorm, uint64_t q,
                  double f, uint64_t seed, uint64_t exclusion_zone, psg_pair_result* out);
int psg_brute_force_motif_f64(const double* series, uint64_t length, uint64_t len, int znorm,
                              uint64_t exclusion_zone, psg_pair_result* out);

/* FRNN, boundary inclusive (refscan.cpp:159-209).  want_lists=0 fills only
 * pair_count / pair_hash / stats (offsets = neighbors = NULL). */
int psg_fixed_radius_neighbors_f64(const double* points, uint64_t n, uint64_t dim, double radius,
                                   uint64_t q, double f, uint64_t seed, uint64_t exclusion_zone,
                                   int want_lists, psg_neighbor_result* out);
int psg_fixed_radius_neighbors_f32(const float* points, uint64_t n, uint64_t dim, double radius,
                                   uint64_t q, double f, uint64_t seed, uint64_t exclusion_zone,
                                   int want_lists, psg_neighbor_result* out);
int psg_brute_force_neighbors_f64(const double* points, uint64_t n, uint64_t dim, double radius,
                                  uint64_t exclusion_zone, int want_lists, psg_neighbor_result* out);
/* The sorted pair list itself: pairs[k] = (i<<32)|j, i<j, lexicographic. */
int psg_frnn_pairs_f32(const float* points, uint64_t n, uint64_t dim, double radius, uint64_t q,
                       double f, uint64_t seed, uint64_t exclusion_zone, uint64_t* pairs,
                       uint64_t capacity, uint64_t* pair_count, uint64_t* pair_hash);
/* The same sorted list as upper-triangular CSR (12 bytes per pair less 4 on
 * the wire): row i = offsets[i] .. offsets[i+1] of cols, every j > i with
 * d(i,j) <= R, ascending (main.cpp:465-478 --pairs-out order).  offsets holds
 * n+1 entries (always complete); cols receives the first `capacity` columns. */
int psg_frnn_pairs_csr_f32(const float* points, uint64_t n, uint64_t dim, double radius, uint64_t q,
                           double f, uint64_t seed, uint64_t exclusion_zone, uint64_t* offsets,
                           uint32_t* cols, uint64_t capacity, uint64_t* pair_count, uint64_t* pair_hash);
void psg_neighbor_result_free(psg_neighbor_result* r);

/* build_reference_set (refscan.cpp:30-65), bit-exact: ref_indices[q],
 * references[q*dim], dist_table[q*n] (k-major), order[n]. */
int psg_build_reference_set_f64(const double* points, uint64_t n, uint64_t dim, uint64_t q,
                                double f, uint64_t seed, uint64_t* ref_indices,
                                double* references, double* dist_table, uint64_t* order);
/* reference_bound (refscan.cpp:229-232): d(r,x) - d(r,y) in the reference's FP64 order. */
int psg_reference_bound(const double* r, const double* x, const double* y, uint64_t dim,
                        double* out);

/* ---- device-resident point sets -------------------------
 * A point set lives in HBM across calls; repeated solves skip the upload. */
typedef struct psg_pointset psg_pointset;
#define PSG_SRC_DEVICE 1 /* the input pointer is device memory (copied D2D) */
int psg_pointset_from_f32(const float* points, uint64_t n, uint64_t dim, int flags, psg_pointset** out);
int psg_pointset_from_f64(const double* points, uint64_t n, uint64_t dim, int flags, psg_pointset** out);
/* windows_of (series.cpp:34-42), optionally z-normalised */
int psg_pointset_windows_f64(const double* series, uint64_t length, uint64_t len, int znorm, int flags,
                             psg_pointset** out);
int psg_pointset_windows_f32(const float* series, uint64_t length, uint64_t len, int znorm, int flags,
                             psg_pointset** out);
void psg_pointset_free(psg_pointset* ps);
uint64_t psg_pointset_size(const psg_pointset* ps);
uint64_t psg_pointset_dim(const psg_pointset* ps);

int psg_closest_pair_ps(psg_pointset* ps, uint64_t q, double f, uint64_t seed, uint64_t exclusion_zone,
                        psg_pair_result* out);
int psg_brute_force_closest_pair_ps(psg_pointset* ps, uint64_t exclusion_zone, psg_pair_result* out);
int psg_fixed_radius_neighbors_ps(psg_pointset* ps, double radius, uint64_t q, double f, uint64_t seed,
                                  uint64_t exclusion_zone, int want_lists, psg_neighbor_result* out);
/* brute_force_neighbors (refscan.cpp:211-227) over a device point set. */
int psg_brute_force_neighbors_ps(psg_pointset* ps, double radius, uint64_t exclusion_zone, int want_lists,
                                 psg_neighbor_result* out);

/* ---- key-range sharding across ranks (one process per GPU) --------------
 * plan_create projects + sorts (identical on every rank); bootstrap returns a
 * rank-local FP32 squared-distance bound for sorted positions of part `part`
 * of `nparts`; the caller all-reduces (MIN) it; scan then searches the part's
 * rows with the global bound and returns the part's best pair (index_i =
 * UINT64_MAX when the part holds none); the caller all-reduces
 * (distance, index_i, index_j) lexicographically and sums stats. */
typedef struct psg_cpp_plan psg_cpp_plan;
int psg_cpp_plan_create(psg_pointset* ps, uint64_t q, double f, uint64_t seed, uint64_t exclusion_zone,
                        psg_cpp_plan** out);
int psg_cpp_plan_bootstrap(psg_cpp_plan* plan, uint64_t part, uint64_t nparts, float* bound_s32);
int psg_cpp_plan_scan(psg_cpp_plan* plan, uint64_t part, uint64_t nparts, float bound_s32,
                      psg_pair_result* out);
void psg_cpp_plan_free(psg_cpp_plan* plan);

/* Fixed-radius neighbours sharded the same way (refscan.cpp:159-209):
 * plan_create projects and builds the cell grid (identical on every rank);
 * plan_scan enumerates the pairs owned by part `part` of `nparts` (a pair is
 * owned by the part holding its earlier grid-sorted position) and returns
 * their count, order-independent hash and stats — the caller all-reduces
 * (SUM) count, hash (mod 2^64) and stats; keep_pairs = 1 keeps the part's
 * pairs on device for plan_pairs, which writes them sorted ascending
 * ((i << 32) | j, i < j) into out[capacity] and fills bucket_counts[b] with
 * how many have i in [n b / nbuckets, n (b + 1) / nbuckets) — the split of an
 * all-to-all that leaves rank b the globally sorted list of its i-range. */
typedef struct psg_frnn_plan psg_frnn_plan;
int psg_frnn_plan_create(psg_pointset* ps, double radius, uint64_t q, double f, uint64_t seed,
                         uint64_t exclusion_zone, psg_frnn_plan** out);
int psg_frnn_plan_scan(psg_frnn_plan* plan, uint64_t part, uint64_t nparts, int keep_pairs, uint64_t* pair_count,
                       uint64_t* pair_hash, psg_scan_stats* stats);
int psg_frnn_plan_pairs(psg_frnn_plan* plan, uint64_t nbuckets, uint64_t* bucket_counts, uint64_t* out,
                        uint64_t capacity);
void psg_frnn_plan_free(psg_frnn_plan* plan);

/* ---- data formats --------------------------------------------
 * Text series: io.cpp:44-60 load_series — one decimal real per line, strtod
 * values, the reference's messages ("path:line: ..."; PSG_ERR_IO) and the
 * finiteness check (series.cpp:13-17; PSG_ERR_INVALID); parsed in parallel.
 * Needs no GPU.  *values is library-allocated: release with psg_free. */
int psg_load_series_text(const char* path, double** values, uint64_t* length);
/* io.cpp:62-70 save_series: "%.17g\n" per value, so load(save(x)) == x. */
int psg_save_series_text(const char* path, const double* values, uint64_t length);
void psg_free(void* p);
/* Binary ".psgb": 32-byte header {"PSGB", u32 version=1, u32 dtype (1 = f64,
 * 2 = f32), u32 0, u64 rows, u64 cols} + rows*cols little-endian values,
 * row-major (a series is one column). */
int psg_save_binary(const char* path, const void* data, int dtype, uint64_t rows, uint64_t cols);
/* A device point set straight from a .psgb file: the rows stream through two
 * pinned staging buffers into HBM (no pageable copy of the whole file). */
int psg_pointset_from_file(const char* path, psg_pointset** out);
/* windows_of over a one-column .psgb series (optionally z-normalised). */
int psg_pointset_windows_from_file(const char* path, uint64_t len, int znorm, psg_pointset** out);

/* ---- inspection (tests): the projection keys of a point set ---------------
 * keys[i*nk + k] = <U_k, X_i> as the solve computes them (tensor cores for
 * d in {32,64,128,256}), the directions U (nk x dim, FP32), the charged key
 * error bound E (working units) and the working-unit scale
 * (X = fl(scale * points)).  nk = 4 or 8 for q clamped to [1, 8]. */
int psg_debug_projection(psg_pointset* ps, uint64_t q, uint64_t seed, int* nk, float* keys, float* dirs,
                         double* key_error, double* scale);

/* ---- inspection (tests): exhaustive search under a known upper bound --------
 * brute_force_closest_pair (refscan.cpp:134-157) in ONE all-pairs pass: every
 * admissible pair whose FP32 distance lies inside the rounding band of
 * `upper` (an FP64 distance some admissible pair is known to reach, e.g. the
 * distance of a returned pair recomputed by the caller) is re-evaluated in the
 * reference's FP64 order.  The band holds every pair at FP64 distance
 * <= upper, so the result is the exact minimum whenever upper >= it; it
 * reports index_i = UINT64_MAX if no pair is that close.  Half the work of the
 * two-pass brute force at sizes where that takes minutes (C5: 1.4e14 pairs). */
int psg_debug_brute_bounded_ps(psg_pointset* ps, uint64_t exclusion_zone, double upper, psg_pair_result* out);

/* ---- host helpers: the reference's seeded synthetic data (datagen.cpp) --- */
int psg_gen_random_walk(uint64_t n, uint64_t seed, double stddev, double* out);
/* SURVEY §8(d) recipes: blocks of 65,536 points from Rng(derive_seed(master, 1000+b)). */
void psg_gen_uniform(uint64_t master, uint64_t n, uint64_t dim, float* out);
void psg_gen_gauss_planted(uint64_t master, uint64_t n, uint64_t dim, double noise, float* out,
                           uint64_t* planted_i, uint64_t* planted_j);
void psg_gen_walk_motif(uint64_t master, uint64_t length, uint64_t len, double noise, float* out,
                        uint64_t* planted_a, uint64_t* planted_b);
void psg_gen_mixture(uint64_t master, uint64_t n, uint64_t dim, uint64_t clusters, double sigma,
                     float* out);
uint64_t psg_mix_seed(uint64_t x);
uint64_t psg_derive_seed(uint64_t base, uint64_t stream);

/* pinned host memory for callers that want the fast H2D path */
int psg_host_alloc(size_t bytes, void** out);
void psg_host_free(void* p);

#ifdef __cplusplus
}
#endif
#endif
