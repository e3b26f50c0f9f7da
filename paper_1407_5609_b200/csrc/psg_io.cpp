// psg_io.cpp — the data formats on either side of the path.
//
// Text series (io.cpp:44-60 load_series): one decimal real per line, no
// header, strtod semantics and the same error messages; parsed here by up to
// 16 threads over newline-aligned chunks (the reference's single-threaded
// getline/istringstream/strtod loop is the host bottleneck once the solve takes
// milliseconds).  Values are identical: every token goes through strtod.
//
// Binary points/series (".psgb", new): a 32-byte header
//   char magic[4] = "PSGB"; uint32 version = 1; uint32 dtype (1 = f64, 2 = f32);
//   uint32 reserved = 0; uint64 rows; uint64 cols
// followed by rows*cols little-endian values, row-major.  A series is one column.
#include <algorithm>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <unistd.h>
#include <stdexcept>
#include <string>
#include <functional>
#include <thread>
#include <vector>

#include "psg_io.hpp"

namespace psg {
namespace {

bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

[[noreturn]] void fail_line(const std::string& path, uint64_t line, const std::string& what) {
  throw io_error(path + ":" + std::to_string(line) + ": " + what);  // io.cpp:16-18
}

std::vector<char> read_file(const std::string& path) {
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw io_error("cannot open " + path + " for reading");  // io.cpp:20-24
  std::vector<char> buf;
  if (std::fseek(f, 0, SEEK_END) == 0) {
    const long sz = std::ftell(f);
    if (sz > 0) buf.resize(static_cast<size_t>(sz));
    std::fseek(f, 0, SEEK_SET);
  }
  const size_t got = buf.empty() ? 0 : std::fread(buf.data(), 1, buf.size(), f);
  std::fclose(f);
  buf.resize(got);
  return buf;
}

// Parse lines [b, e) of the buffer (b at a line start); line numbers from first_line.
struct Chunk {
  const char* b;
  const char* e;
  uint64_t first_line;
  std::vector<double> values;
  std::string error;  // first error of the chunk ("path:line: what")
  uint64_t error_line = 0;
};

void parse_chunk(Chunk& c, const std::string& path) {
  uint64_t line = c.first_line;
  std::string token;
  for (const char* p = c.b; p < c.e; ++line) {
    const char* eol = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(c.e - p)));
    const char* end = eol ? eol : c.e;
    const char* q = p;
    while (q < end && is_space(*q)) ++q;
    if (q == end) {  // io.cpp:53
      c.error = path + ":" + std::to_string(line) + ": empty line in series file";
      c.error_line = line;
      return;
    }
    const char* t = q;
    while (t < end && !is_space(*t)) ++t;
    token.assign(q, t);
    const char* r = t;
    while (r < end && is_space(*r)) ++r;
    if (r != end) {  // io.cpp:54
      c.error = path + ":" + std::to_string(line) + ": expected one value per line";
      c.error_line = line;
      return;
    }
    errno = 0;  // io.cpp:26-34 parse_real
    char* stop = nullptr;
    const double v = std::strtod(token.c_str(), &stop);
    if (stop == token.c_str() || *stop != '\0' || errno == ERANGE) {
      c.error = path + ":" + std::to_string(line) + ": expected a decimal real, got '" + token + "'";
      c.error_line = line;
      return;
    }
    c.values.push_back(v);
    p = eol ? eol + 1 : c.e;
  }
}

struct Header {
  char magic[4];
  uint32_t version, dtype, reserved;
  uint64_t rows, cols;
};
static_assert(sizeof(Header) == 32, "psgb header");

}  // namespace

std::vector<double> load_series_text(const std::string& path) {
  const std::vector<char> buf = read_file(path);
  const char* b = buf.data();
  const char* e = b + buf.size();
  // newline-aligned chunks; each chunk's first line number from a newline count
  const unsigned hw = std::thread::hardware_concurrency();
  const size_t nt = std::max<size_t>(1, std::min<size_t>({hw ? hw : 1, 16, buf.size() / (1 << 16) + 1}));
  std::vector<Chunk> chunks;
  const char* p = b;
  for (size_t k = 0; k < nt && p < e; ++k) {
    const char* ce = k + 1 == nt ? e : b + buf.size() * (k + 1) / nt;
    if (ce < p) ce = p;
    if (ce < e) {
      const char* nl = static_cast<const char*>(std::memchr(ce, '\n', static_cast<size_t>(e - ce)));
      ce = nl ? nl + 1 : e;
    }
    chunks.push_back(Chunk{p, ce, 0, {}, {}, 0});
    p = ce;
  }
  uint64_t line = 1;
  for (Chunk& c : chunks) {
    c.first_line = line;
    for (const char* q = c.b; q < c.e; ++q) line += *q == '\n';
    if (c.e > c.b && c.e[-1] != '\n') ++line;  // last line without a newline
  }
  std::vector<std::thread> th;
  for (size_t k = 1; k < chunks.size(); ++k) th.emplace_back(parse_chunk, std::ref(chunks[k]), std::cref(path));
  if (!chunks.empty()) parse_chunk(chunks[0], path);
  for (std::thread& t : th) t.join();
  std::vector<double> out;
  size_t total = 0;
  for (const Chunk& c : chunks) {
    if (!c.error.empty()) throw io_error(c.error);  // the first failing line, as the sequential loop reports
    total += c.values.size();
  }
  if (total == 0) throw io_error(path + ": empty series file");  // io.cpp:58
  out.reserve(total);
  for (const Chunk& c : chunks) out.insert(out.end(), c.values.begin(), c.values.end());
  for (const double v : out)
    if (!std::isfinite(v)) throw invalid_argument("series value must be finite");  // series.cpp:13-17
  return out;
}

void save_series_text(const std::string& path, const double* v, uint64_t n) {
  std::string out;
  out.reserve(n * 20);
  char tmp[40];
  for (uint64_t i = 0; i < n; ++i) {
    std::snprintf(tmp, sizeof(tmp), "%.17g", v[i]);  // io.cpp:36-40 format_real
    out += tmp;
    out += '\n';
  }
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw io_error("cannot open " + path + " for writing");
  const size_t w = std::fwrite(out.data(), 1, out.size(), f);
  std::fclose(f);
  if (w != out.size()) throw io_error("short write to " + path);
}

void save_binary(const std::string& path, const void* data, int dtype, uint64_t rows, uint64_t cols) {
  if (dtype != 1 && dtype != 2) throw invalid_argument("binary dtype must be 1 (f64) or 2 (f32)");
  Header h{{'P', 'S', 'G', 'B'}, 1, static_cast<uint32_t>(dtype), 0, rows, cols};
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw io_error("cannot open " + path + " for writing");
  const size_t bytes = rows * cols * (dtype == 1 ? 8 : 4);
  const bool ok = std::fwrite(&h, sizeof(h), 1, f) == 1 && (bytes == 0 || std::fwrite(data, 1, bytes, f) == bytes);
  std::fclose(f);
  if (!ok) throw io_error("short write to " + path);
}

BinaryFile open_binary(const std::string& path) {
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw io_error("cannot open " + path + " for reading");
  Header h{};
  const bool got = std::fread(&h, sizeof(h), 1, f) == 1;
  if (!got || std::memcmp(h.magic, "PSGB", 4) != 0 || h.version != 1 || (h.dtype != 1 && h.dtype != 2)) {
    std::fclose(f);
    throw io_error(path + ": not a PSGB v1 file");
  }
  BinaryFile b;
  b.f = f;
  b.dtype = static_cast<int>(h.dtype);
  b.rows = h.rows;
  b.cols = h.cols;
  b.bytes = h.rows * h.cols * (h.dtype == 1 ? 8 : 4);
  return b;
}

size_t BinaryFile::read(void* dst, size_t bytes) { return std::fread(dst, 1, bytes, f); }

size_t BinaryFile::pread_payload(void* dst, uint64_t off, size_t len, int threads) const {
  const int fd = fileno(f);
  std::vector<size_t> got(static_cast<size_t>(std::max(threads, 1)), 0);
  auto work = [&](int k) {
    const size_t b = len * k / got.size(), e = len * (k + 1) / got.size();
    size_t done = 0;
    while (b + done < e) {
      const ssize_t r = ::pread(fd, static_cast<char*>(dst) + b + done, e - b - done,
                                static_cast<off_t>(sizeof(Header) + off + b + done));
      if (r <= 0) break;
      done += static_cast<size_t>(r);
    }
    got[static_cast<size_t>(k)] = done;
  };
  std::vector<std::thread> th;
  for (int k = 1; k < static_cast<int>(got.size()); ++k) th.emplace_back(work, k);
  work(0);
  for (std::thread& t : th) t.join();
  size_t total = 0;
  for (const size_t g : got) total += g;
  return total;
}

BinaryFile::~BinaryFile() {
  if (f) std::fclose(f);
}

}  // namespace psg
