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

// out[i] = in[0] + ... + in[i-1] (u32), count <= 2^25; `temp` needs
// scan_temp_words(count) words.  One single-pass kernel (decoupled
// look-back) after a memset of the temp; in/out 16-byte aligned.
size_t scan_temp_words(size_t count);
void exclusive_scan_u32(const uint32_t* in, uint32_t* out, size_t count, uint32_t* temp, cudaStream_t s);
// Same with the length read on device: count = *dcells + 1 (<= max_count).
// zeroed: the caller already zeroed the temp (no memset node between kernels).
void exclusive_scan_u32_dev(const uint32_t* in, uint32_t* out, size_t max_count, const uint64_t* dcells,
                            uint32_t* temp, cudaStream_t s, bool zeroed = false);
template <class K>
int radix_sort(K* keys[2], uint32_t* vals[2], size_t n, int begin_bit, int end_bit, uint32_t* hist,
               cudaStream_t s);

}  // namespace psg
