// psg_io.hpp — host-side file formats (psg_io.cpp): the reference's text series
// format (io.cpp:44-60) and the binary ".psgb" points/series format.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

namespace psg {

// The reference's io errors are std::runtime_error; its argument errors are
// std::invalid_argument (series.cpp).
struct io_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
#ifndef PSG_INVALID_ARGUMENT_DEFINED
#define PSG_INVALID_ARGUMENT_DEFINED
struct invalid_argument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
#endif

std::vector<double> load_series_text(const std::string& path);
void save_series_text(const std::string& path, const double* v, uint64_t n);
void save_binary(const std::string& path, const void* data, int dtype, uint64_t rows, uint64_t cols);

struct BinaryFile {
  FILE* f = nullptr;
  int dtype = 0;  // 1 = f64, 2 = f32
  uint64_t rows = 0, cols = 0, bytes = 0;
  size_t read(void* dst, size_t bytes);
  // payload bytes [off, off+len) into dst, read by `threads` parallel preads
  size_t pread_payload(void* dst, uint64_t off, size_t len, int threads) const;
  BinaryFile() = default;
  BinaryFile(BinaryFile&& o) noexcept : f(o.f), dtype(o.dtype), rows(o.rows), cols(o.cols), bytes(o.bytes) {
    o.f = nullptr;
  }
  BinaryFile(const BinaryFile&) = delete;
  ~BinaryFile();
};
BinaryFile open_binary(const std::string& path);

}  // namespace psg
