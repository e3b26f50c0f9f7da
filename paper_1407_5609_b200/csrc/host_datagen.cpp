// host_datagen.cpp — seeded synthetic inputs (host side, generated once and
// shipped to the device as bytes).  gen_random_walk follows
// datagen.cpp:10-23; the config recipes draw block b of 65,536 points from
// Rng(derive_seed(master, 1000 + b)) so blocks generate in parallel and the
// result does not depend on the thread count.
#include <algorithm>
#include <cmath>
#include <thread>
#include <vector>

#include "../../include/pairscan_b200.h"
#include "host_rng.hpp"

namespace {

constexpr uint64_t kBlock = 65536;

template <class F>
void for_blocks(uint64_t n, F&& body) {
  const uint64_t nb = (n + kBlock - 1) / kBlock;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const unsigned nt = static_cast<unsigned>(std::min<uint64_t>(nb, hw));
  std::vector<std::thread> pool;
  for (unsigned w = 0; w < nt; ++w)
    pool.emplace_back([&, w] {
      for (uint64_t b = w; b < nb; b += nt) body(b, b * kBlock, std::min(n, (b + 1) * kBlock));
    });
  for (auto& t : pool) t.join();
}

}  // namespace

extern "C" {

uint64_t psg_mix_seed(uint64_t x) { return psg::splitmix(x); }
uint64_t psg_derive_seed(uint64_t base, uint64_t stream) { return psg::stream_seed(base, stream); }

int psg_gen_random_walk(uint64_t n, uint64_t seed, double stddev, double* out) {
  if (n == 0 || !(stddev > 0.0) || !std::isfinite(stddev)) return PSG_ERR_INVALID;
  psg::HostRng r(seed);
  out[0] = 0.0;
  for (uint64_t i = 1; i < n; ++i) out[i] = out[i - 1] + r.gauss(0.0, stddev);
  return PSG_OK;
}

void psg_gen_uniform(uint64_t master, uint64_t n, uint64_t dim, float* out) {
  for_blocks(n, [&](uint64_t b, uint64_t lo, uint64_t hi) {
    psg::HostRng r(psg::stream_seed(master, 1000 + b));
    for (uint64_t i = lo * dim; i < hi * dim; ++i) out[i] = r.u24();
  });
}

void psg_gen_gauss_planted(uint64_t master, uint64_t n, uint64_t dim, double noise, float* out, uint64_t* pi,
                           uint64_t* pj) {
  for_blocks(n, [&](uint64_t b, uint64_t lo, uint64_t hi) {
    psg::HostRng r(psg::stream_seed(master, 1000 + b));
    for (uint64_t i = lo * dim; i < hi * dim; ++i) out[i] = static_cast<float>(r.gauss(0.0, 1.0));
  });
  psg::HostRng p(psg::stream_seed(master, 1));
  const uint64_t i = p.below(n);
  uint64_t j = p.below(n - 1);
  if (j >= i) ++j;
  for (uint64_t t = 0; t < dim; ++t)
    out[j * dim + t] = static_cast<float>(static_cast<double>(out[i * dim + t]) + p.gauss(0.0, noise));
  *pi = i;
  *pj = j;
}

void psg_gen_walk_motif(uint64_t master, uint64_t length, uint64_t len, double noise, float* out, uint64_t* pa,
                        uint64_t* pb) {
  std::vector<double> walk(length);
  psg_gen_random_walk(length, psg::stream_seed(master, 0), 1.0, walk.data());
  for (uint64_t t = 0; t < length; ++t) out[t] = static_cast<float>(walk[t]);
  psg::HostRng p(psg::stream_seed(master, 1));
  const uint64_t nw = length - len + 1;
  const uint64_t a = p.below(nw);
  uint64_t b;
  do {
    b = p.below(nw);
  } while ((a > b ? a - b : b - a) < len);
  for (uint64_t t = 0; t < len; ++t)
    out[b + t] = static_cast<float>(static_cast<double>(out[a + t]) + p.gauss(0.0, noise));
  *pa = a;
  *pb = b;
}

void psg_gen_mixture(uint64_t master, uint64_t n, uint64_t dim, uint64_t clusters, double sigma, float* out) {
  std::vector<double> centres(clusters * dim);
  psg::HostRng c(psg::stream_seed(master, 0));
  for (auto& v : centres) v = -1.0 + 2.0 * static_cast<double>(c.u24());
  for_blocks(n, [&](uint64_t b, uint64_t lo, uint64_t hi) {
    psg::HostRng r(psg::stream_seed(master, 1000 + b));
    for (uint64_t i = lo; i < hi; ++i) {
      const double* ctr = centres.data() + (i % clusters) * dim;
      for (uint64_t t = 0; t < dim; ++t) out[i * dim + t] = static_cast<float>(ctr[t] + r.gauss(0.0, sigma));
    }
  });
}

}  // extern "C"
