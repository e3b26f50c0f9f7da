/*
 * oracle.c — CPU restatement of the reference hot path (see oracle.h).
 * TEST INFRASTRUCTURE ONLY: never linked into the product library.
 * File:line citations are relative to /root/reference/proj.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ======================================================================
 * mt19937_64 (Matsumoto & Nishimura 2000, the published 64-bit variant),
 * which std::mt19937_64 is required to produce bit-exactly; the reference
 * draws every seeded value from it (core/include/pairscan/rng.hpp:14-41).
 * ==================================================================== */
#define MT_N 312
#define MT_M 156
#define MT_A 0xB5026F5AA96619E9ULL
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x000000007FFFFFFFULL

void orc_rng_seed(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i) {
    const uint64_t prev = r->mt[i - 1];
    r->mt[i] = 6364136223846793005ULL * (prev ^ (prev >> 62)) + (uint64_t)i;
  }
  r->mti = MT_N;
}

static void mt_refill(orc_rng* r) {
  uint64_t* mt = r->mt;
  for (int k = 0; k < MT_N; ++k) {
    const uint64_t y = (mt[k] & MT_UPPER) | (mt[(k + 1) % MT_N] & MT_LOWER);
    const uint64_t twisted = (y >> 1) ^ ((y & 1ULL) ? MT_A : 0ULL);
    mt[k] = mt[(k + MT_M) % MT_N] ^ twisted;
  }
  r->mti = 0;
}

uint64_t orc_rng_next(orc_rng* r) {
  if (r->mti >= MT_N) mt_refill(r);
  uint64_t z = r->mt[r->mti++];
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= z >> 43;
  return z;
}

/* rng.cpp:10-20: masked rejection with the smallest all-ones mask >= bound-1. */
uint64_t orc_uniform_below(orc_rng* r, uint64_t bound) {
  if (bound <= 1) return 0; /* bound==0 is a contract violation upstream */
  const uint64_t top = bound - 1;
  const int bits = 64 - __builtin_clzll(top);
  const uint64_t mask = bits == 64 ? ~0ULL : ((1ULL << bits) - 1ULL);
  for (;;) {
    const uint64_t v = orc_rng_next(r) & mask;
    if (v < bound) return v;
  }
}

/* rng.cpp:22-24: 53 high bits scaled by 2^-53. */
double orc_uniform_unit(orc_rng* r) { return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53; }

/* rng.cpp:26-32: Box-Muller, cosine branch only, u1 = 1 - U so log is finite. */
double orc_gaussian(orc_rng* r, double mean, double sd) {
  const double u1 = 1.0 - orc_uniform_unit(r);
  const double u2 = orc_uniform_unit(r);
  const double two_pi = 2.0 * 3.14159265358979323846;
  const double radius = sqrt(-2.0 * log(u1));
  return mean + sd * radius * cos(two_pi * u2);
}

/* rng.cpp:34-44: partial Fisher-Yates over the identity pool. */
int orc_sample_without_replacement(orc_rng* r, uint64_t n, uint64_t k, uint64_t* out) {
  if (k > n) return -1;
  uint64_t* pool = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
  if (!pool) return -3;
  for (uint64_t i = 0; i < n; ++i) pool[i] = i;
  for (uint64_t i = 0; i < k; ++i) {
    const uint64_t j = i + orc_uniform_below(r, n - i);
    const uint64_t t = pool[i];
    pool[i] = pool[j];
    pool[j] = t;
  }
  memcpy(out, pool, k * sizeof(uint64_t));
  free(pool);
  return 0;
}

/* rng.cpp:46-51 (SplitMix64 finaliser) and 53-55. */
uint64_t orc_mix_seed(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

uint64_t orc_derive_seed(uint64_t base, uint64_t stream) {
  return orc_mix_seed(base ^ orc_mix_seed(stream + 1));
}

/* datagen.cpp:10-23 */
int orc_gen_random_walk(uint64_t n, uint64_t seed, double sd, double* out) {
  if (n == 0) return -1;
  if (!(sd > 0.0) || !isfinite(sd)) return -1;
  orc_rng r;
  orc_rng_seed(&r, seed);
  out[0] = 0.0;
  for (uint64_t i = 1; i < n; ++i) out[i] = out[i - 1] + orc_gaussian(&r, 0.0, sd);
  return 0;
}

/* ======================================================================
 * metrics.cpp
 * ==================================================================== */
double orc_euclidean(const double* x, const double* y, uint64_t d) {
  double acc = 0.0;
  for (uint64_t t = 0; t < d; ++t) {
    const double diff = x[t] - y[t];
    acc += diff * diff;
  }
  return sqrt(acc);
}

int orc_euclidean_early_abandon(const double* x, const double* y, uint64_t d, double thr,
                                double* out) {
  const double limit = thr * thr * (1.0 + 4e-15); /* metrics.cpp:36 */
  double acc = 0.0;
  for (uint64_t t = 0; t < d; ++t) {
    const double diff = x[t] - y[t];
    acc += diff * diff;
    if (acc > limit) return 0;
  }
  const double dist = sqrt(acc);
  if (dist > thr) return 0; /* metrics.cpp:44 */
  *out = dist;
  return 1;
}

double orc_reference_bound(const double* r, const double* x, const double* y, uint64_t d) {
  return orc_euclidean(r, x, d) - orc_euclidean(r, y, d);
}

static double dist_f32(const float* x, const float* y, uint64_t d) {
  double acc = 0.0;
  for (uint64_t t = 0; t < d; ++t) {
    const double diff = (double)x[t] - (double)y[t];
    acc += diff * diff;
  }
  return sqrt(acc);
}

static int admissible(uint64_t i, uint64_t j, uint64_t zone) {
  const uint64_t gap = i > j ? i - j : j - i;
  return gap >= zone; /* refscan.cpp:15-18 */
}

/* ======================================================================
 * refscan.cpp:134-157 — the definition every engine must reproduce.
 * ==================================================================== */
int orc_brute_force_closest_pair(const double* pts, uint64_t n, uint64_t d, uint64_t zone,
                                 orc_pair* out) {
  if (n < 2) return -1;
  int found = 0;
  orc_pair best = {0, 0, INFINITY, 0};
  for (uint64_t i = 0; i + 1 < n; ++i) {
    for (uint64_t j = i + 1; j < n; ++j) {
      if (!admissible(i, j, zone)) continue;
      ++best.pairs_examined;
      const double dist = orc_euclidean(pts + i * d, pts + j * d, d);
      if (dist < best.distance) {
        best.index_i = i;
        best.index_j = j;
        best.distance = dist;
        found = 1;
      }
    }
  }
  if (!found) return -2;
  *out = best;
  return 0;
}

int orc_brute_force_closest_pair_f32(const float* pts, uint64_t n, uint64_t d, uint64_t zone,
                                     orc_pair* out) {
  if (n < 2) return -1;
  int found = 0;
  orc_pair best = {0, 0, INFINITY, 0};
  for (uint64_t i = 0; i + 1 < n; ++i) {
    for (uint64_t j = i + 1; j < n; ++j) {
      if (!admissible(i, j, zone)) continue;
      ++best.pairs_examined;
      const double dist = dist_f32(pts + i * d, pts + j * d, d);
      if (dist < best.distance) {
        best.index_i = i;
        best.index_j = j;
        best.distance = dist;
        found = 1;
      }
    }
  }
  if (!found) return -2;
  *out = best;
  return 0;
}

/* refscan.cpp:211-227 (boundary inclusive <= R), summarised. */
int orc_brute_force_neighbors(const double* pts, uint64_t n, uint64_t d, double R, uint64_t zone,
                              uint64_t* count, uint64_t* hash, uint64_t* lists, uint64_t cap) {
  if (n == 0) return -1;
  if (!(R > 0.0) || !isfinite(R)) return -1;
  uint64_t c = 0, h = 0;
  for (uint64_t i = 0; i + 1 < n; ++i) {
    for (uint64_t j = i + 1; j < n; ++j) {
      if (!admissible(i, j, zone)) continue;
      if (orc_euclidean(pts + i * d, pts + j * d, d) <= R) {
        const uint64_t key = (i << 32) | j;
        if (lists && c < cap) lists[c] = key;
        ++c;
        h += orc_mix_seed(key);
      }
    }
  }
  *count = c;
  *hash = h;
  return 0;
}

/* Exact cell-grid FRNN: same decision as brute_force_neighbors, candidates
 * restricted to the 3^g neighbouring cells of width w > R.  A pair inside R
 * differs by at most R*(1+1e-15) per coordinate, so it lies in adjacent cells. */
int orc_frnn_grid_f32(const float* pts, uint64_t n, uint64_t d, double R, uint64_t zone,
                      uint64_t* count, uint64_t* hash) {
  if (n == 0) return -1;
  if (!(R > 0.0) || !isfinite(R)) return -1;
  const int g = d < 3 ? (int)d : 3;
  double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  for (int t = 0; t < g; ++t) {
    lo[t] = INFINITY;
    hi[t] = -INFINITY;
  }
  for (uint64_t i = 0; i < n; ++i)
    for (int t = 0; t < g; ++t) {
      const double v = pts[i * d + t];
      if (v < lo[t]) lo[t] = v;
      if (v > hi[t]) hi[t] = v;
    }
  double w = R * (1.0 + 0x1.0p-30);
  int64_t dims[3] = {1, 1, 1};
  for (;;) {
    double cells = 1.0;
    for (int t = 0; t < g; ++t) {
      dims[t] = (int64_t)floor((hi[t] - lo[t]) / w) + 1;
      cells *= (double)dims[t];
    }
    if (cells <= (double)(1u << 26)) break;
    w *= 2.0;
  }
  const uint64_t ncell = (uint64_t)(dims[0] * dims[1] * dims[2]);
  uint64_t* cell_of = (uint64_t*)malloc(n * sizeof(uint64_t));
  uint64_t* start = (uint64_t*)calloc(ncell + 1, sizeof(uint64_t));
  uint64_t* sorted = (uint64_t*)malloc(n * sizeof(uint64_t));
  if (!cell_of || !start || !sorted) {
    free(cell_of);
    free(start);
    free(sorted);
    return -3;
  }
  for (uint64_t i = 0; i < n; ++i) {
    int64_t c[3] = {0, 0, 0};
    for (int t = 0; t < g; ++t) {
      c[t] = (int64_t)floor(((double)pts[i * d + t] - lo[t]) / w);
      if (c[t] >= dims[t]) c[t] = dims[t] - 1;
    }
    cell_of[i] = (uint64_t)((c[0] * dims[1] + c[1]) * dims[2] + c[2]);
    start[cell_of[i] + 1]++;
  }
  for (uint64_t c = 0; c < ncell; ++c) start[c + 1] += start[c];
  {
    uint64_t* fill = (uint64_t*)malloc(ncell * sizeof(uint64_t));
    memcpy(fill, start, ncell * sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i) sorted[fill[cell_of[i]]++] = i; /* ascending i per cell */
    free(fill);
  }
  uint64_t c_total = 0, h_total = 0;
#pragma omp parallel for schedule(dynamic, 4096) reduction(+ : c_total, h_total)
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t cell = cell_of[i];
    int64_t ci[3];
    ci[2] = (int64_t)(cell % (uint64_t)dims[2]);
    ci[1] = (int64_t)((cell / (uint64_t)dims[2]) % (uint64_t)dims[1]);
    ci[0] = (int64_t)(cell / (uint64_t)(dims[2] * dims[1]));
    for (int64_t a = -1; a <= 1; ++a) {
      const int64_t x0 = ci[0] + a;
      if (x0 < 0 || x0 >= dims[0]) continue;
      for (int64_t b = -1; b <= 1; ++b) {
        const int64_t x1 = ci[1] + b;
        if (x1 < 0 || x1 >= dims[1]) continue;
        for (int64_t e = -1; e <= 1; ++e) {
          const int64_t x2 = ci[2] + e;
          if (x2 < 0 || x2 >= dims[2]) continue;
          const uint64_t nc = (uint64_t)((x0 * dims[1] + x1) * dims[2] + x2);
          for (uint64_t s = start[nc]; s < start[nc + 1]; ++s) {
            const uint64_t j = sorted[s];
            if (j <= i || !admissible(i, j, zone)) continue;
            if (dist_f32(pts + i * d, pts + j * d, d) <= R) {
              ++c_total;
              h_total += orc_mix_seed((i << 32) | j);
            }
          }
        }
      }
    }
  }
  free(cell_of);
  free(start);
  free(sorted);
  *count = c_total;
  *hash = h_total;
  return 0;
}

/* ======================================================================
 * refscan.cpp:30-65 build_reference_set
 * ==================================================================== */
static const double* g_sort_key;
static int cmp_by_key_then_index(const void* a, const void* b) {
  const uint64_t ia = *(const uint64_t*)a, ib = *(const uint64_t*)b;
  const double ka = g_sort_key[ia], kb = g_sort_key[ib];
  if (ka != kb) return ka < kb ? -1 : 1;
  return ia < ib ? -1 : (ia > ib ? 1 : 0);
}

int orc_build_reference_set(const double* pts, uint64_t n, uint64_t d, uint64_t q, double f,
                            uint64_t seed, uint64_t* ref_indices, double* references,
                            double* table, uint64_t* order) {
  if (q == 0 || q > n) return -1;
  if (!(f > 0.0) || !isfinite(f)) return -1;
  orc_rng r;
  orc_rng_seed(&r, seed);
  if (orc_sample_without_replacement(&r, n, q, ref_indices) != 0) return -3;
  for (uint64_t k = 0; k < q; ++k)
    for (uint64_t t = 0; t < d; ++t) references[k * d + t] = pts[ref_indices[k] * d + t] * f;
  for (uint64_t k = 0; k < q; ++k)
    for (uint64_t i = 0; i < n; ++i) table[k * n + i] = orc_euclidean(references + k * d, pts + i * d, d);
  for (uint64_t i = 0; i < n; ++i) order[i] = i;
  g_sort_key = table;
  qsort(order, n, sizeof(uint64_t), cmp_by_key_then_index);
  return 0;
}

/* ======================================================================
 * z-normalised windows (SURVEY.md §8(d) C3 recipe; not in the reference)
 * ==================================================================== */
static void window_stats(const double* s, uint64_t l, double* mu, double* sigma) {
  double acc = 0.0;
  for (uint64_t t = 0; t < l; ++t) acc += s[t];
  const double m = acc / (double)l;
  double v = 0.0;
  for (uint64_t t = 0; t < l; ++t) {
    const double c = s[t] - m;
    v += c * c;
  }
  *mu = m;
  *sigma = sqrt(v / (double)l);
}

int orc_znorm_windows(const double* series, uint64_t N, uint64_t l, double* out) {
  if (l == 0 || l > N) return -1;
  const uint64_t nw = N - l + 1;
  for (uint64_t i = 0; i < nw; ++i) {
    double mu, sigma;
    window_stats(series + i, l, &mu, &sigma);
    for (uint64_t t = 0; t < l; ++t)
      out[i * l + t] = sigma == 0.0 ? 0.0 : (series[i + t] - mu) / sigma;
  }
  return 0;
}

double orc_znorm_pair_distance(const double* series, uint64_t l, uint64_t i, uint64_t j) {
  double mi, si, mj, sj, acc = 0.0;
  window_stats(series + i, l, &mi, &si);
  window_stats(series + j, l, &mj, &sj);
  for (uint64_t t = 0; t < l; ++t) {
    const double a = si == 0.0 ? 0.0 : (series[i + t] - mi) / si;
    const double b = sj == 0.0 ? 0.0 : (series[j + t] - mj) / sj;
    const double diff = a - b;
    acc += diff * diff;
  }
  return sqrt(acc);
}

int orc_motif_brute_znorm(const double* series, uint64_t N, uint64_t l, uint64_t zone,
                          orc_pair* out) {
  if (l == 0 || l > N) return -1;
  const uint64_t nw = N - l + 1;
  double* z = (double*)malloc(nw * l * sizeof(double));
  if (!z) return -3;
  orc_znorm_windows(series, N, l, z);
  const int rc = orc_brute_force_closest_pair(z, nw, l, zone, out);
  free(z);
  return rc;
}

/* ======================================================================
 * Synthetic configs.
 * ==================================================================== */
#define BLOCK_POINTS 65536ULL

static float u24(orc_rng* r) { return (float)((double)(orc_rng_next(r) >> 40) * 0x1.0p-24); }

void orc_gen_uniform_u24(uint64_t master, uint64_t n, uint64_t d, float* out) {
  for (uint64_t b = 0; b * BLOCK_POINTS < n; ++b) {
    orc_rng r;
    orc_rng_seed(&r, orc_derive_seed(master, 1000 + b));
    const uint64_t end = (b + 1) * BLOCK_POINTS < n ? (b + 1) * BLOCK_POINTS : n;
    for (uint64_t i = b * BLOCK_POINTS; i < end; ++i)
      for (uint64_t t = 0; t < d; ++t) out[i * d + t] = u24(&r);
  }
}

void orc_gen_gauss_planted(uint64_t master, uint64_t n, uint64_t d, double noise, float* out,
                           uint64_t* pi, uint64_t* pj) {
  for (uint64_t b = 0; b * BLOCK_POINTS < n; ++b) {
    orc_rng r;
    orc_rng_seed(&r, orc_derive_seed(master, 1000 + b));
    const uint64_t end = (b + 1) * BLOCK_POINTS < n ? (b + 1) * BLOCK_POINTS : n;
    for (uint64_t i = b * BLOCK_POINTS; i < end; ++i)
      for (uint64_t t = 0; t < d; ++t) out[i * d + t] = (float)orc_gaussian(&r, 0.0, 1.0);
  }
  orc_rng p;
  orc_rng_seed(&p, orc_derive_seed(master, 1));
  const uint64_t i = orc_uniform_below(&p, n);
  uint64_t j = orc_uniform_below(&p, n - 1);
  if (j >= i) ++j;
  for (uint64_t t = 0; t < d; ++t)
    out[j * d + t] = (float)((double)out[i * d + t] + orc_gaussian(&p, 0.0, noise));
  *pi = i;
  *pj = j;
}

void orc_gen_walk_motif(uint64_t master, uint64_t N, uint64_t l, double noise, float* out,
                        uint64_t* pa, uint64_t* pb) {
  double* walk = (double*)malloc(N * sizeof(double));
  orc_gen_random_walk(N, orc_derive_seed(master, 0), 1.0, walk);
  for (uint64_t t = 0; t < N; ++t) out[t] = (float)walk[t];
  free(walk);
  orc_rng p;
  orc_rng_seed(&p, orc_derive_seed(master, 1));
  const uint64_t nw = N - l + 1;
  const uint64_t a = orc_uniform_below(&p, nw);
  uint64_t b;
  do {
    b = orc_uniform_below(&p, nw);
  } while ((a > b ? a - b : b - a) < l);
  for (uint64_t t = 0; t < l; ++t) out[b + t] = (float)((double)out[a + t] + orc_gaussian(&p, 0.0, noise));
  *pa = a;
  *pb = b;
}

void orc_gen_mixture(uint64_t master, uint64_t n, uint64_t d, uint64_t k, double sigma, float* out) {
  double* centres = (double*)malloc(k * d * sizeof(double));
  orc_rng c;
  orc_rng_seed(&c, orc_derive_seed(master, 0));
  for (uint64_t t = 0; t < k * d; ++t) centres[t] = -1.0 + 2.0 * (double)u24(&c);
  for (uint64_t b = 0; b * BLOCK_POINTS < n; ++b) {
    orc_rng r;
    orc_rng_seed(&r, orc_derive_seed(master, 1000 + b));
    const uint64_t end = (b + 1) * BLOCK_POINTS < n ? (b + 1) * BLOCK_POINTS : n;
    for (uint64_t i = b * BLOCK_POINTS; i < end; ++i) {
      const double* ctr = centres + (i % k) * d;
      for (uint64_t t = 0; t < d; ++t) out[i * d + t] = (float)(ctr[t] + orc_gaussian(&r, 0.0, sigma));
    }
  }
  free(centres);
}
