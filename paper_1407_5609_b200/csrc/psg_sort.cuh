// psg_sort.cuh — on-device LSD radix sort (8-bit digits) of u32/u64 keys with
// an optional u32 payload.  Stable, so sorting (key, index) with the identity
// payload reproduces the reference's `std::sort` by (d1, index)
// (refscan.cpp:58-63) bit-exactly.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace psg {

// Sorts keys[0]/vals[0] (length n) on bits [begin_bit, end_bit).  keys[1] and
// vals[1] are scratch of the same length.  Returns the index (0 or 1) of the
// buffer holding the result.  vals may be {nullptr, nullptr}.  `hist` needs
// radix_hist_words(n) u32 words.
size_t radix_hist_words(size_t n);
template <class K>
int radix_sort(K* keys[2], uint32_t* vals[2], size_t n, int begin_bit, int end_bit, uint32_t* hist,
               cudaStream_t s);

}  // namespace psg
