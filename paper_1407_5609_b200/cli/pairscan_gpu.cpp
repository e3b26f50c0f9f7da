// pairscan-gpu — the reference front end's series/point scans
// with every engine on the B200 library (libpairscan_b200.so, C ABI only).
//
// Mirrors /root/reference/proj/tools/src/main.cpp for the commands on the
// north_star path, with the same options, defaults, report schema and
// replay contract:
//   gen-walk   main.cpp:200-214  (cmd_gen_walk)
//   motif      main.cpp:262-382  (MotifOpts, add_series_input, cmd_motif)
//   frnn       main.cpp:384-491  (FrnnOpts, cmd_frnn, --pairs-out)
//   sweep      main.cpp:792-897  (cmd_sweep: aggregate + raw CSV)
//   verify     main.cpp:899-1013 (replay each report's params line, compare fields)
// plus the point-cloud input format the survey asks for (G5):
//   closest    exact closest pair of the rows of a .psgb point file
//   neighbors  fixed-radius neighbour pairs of a .psgb point file
//
// Engines: mpr (the default, as in the reference), mk (f = 1) and brute, all
// executed on the GPU; `gpu` is accepted as a synonym of mpr.  Reports are the
// reference's Report (io.hpp:24-40) rendered by the same JSON writer
// (nlohmann::json dump(2), io.cpp:140-185) and CSV layout (io.cpp:187-225), so
// a reference report and a GPU report of the same run differ only in
// pairs_examined (the engines examine different pairs) and
// wall_seconds.
//
// Argument parsing is a small hand-written parser (CLI11 is not available in
// this image): `--opt value`, `--opt=value`, flags, positionals; errors print
// "error: ..." to stderr and exit 2 (the reference's CLI11 uses its own exit
// codes for parse errors; run errors are 2 in both).
#include <algorithm>
#include <cerrno>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <iomanip>
#include <functional>
#include <iostream>
#include <map>
#include <memory>
#include <optional>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include <json.hpp>

#include "pairscan_b200.h"

namespace {

constexpr const char* kVersion = "0.1.0";

struct usage_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ---------------------------------------------------------------------------
// the library boundary

void check(int rc) {
  if (rc == PSG_OK) return;
  const std::string msg = psg_last_error();
  if (rc == PSG_ERR_INVALID) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

struct PointsetDel {
  void operator()(psg_pointset* p) const { psg_pointset_free(p); }
};
using Points = std::unique_ptr<psg_pointset, PointsetDel>;

struct Lists {  // CSR neighbour lists (psg_neighbor_result)
  uint64_t n = 0;
  std::vector<uint64_t> offsets, neighbors;
  uint64_t examined = 0;
  bool operator==(const Lists& o) const { return offsets == o.offsets && neighbors == o.neighbors; }
};

Lists take(psg_neighbor_result& r) {
  Lists l;
  l.n = r.n;
  l.offsets.assign(r.offsets, r.offsets + r.n + 1);
  l.neighbors.assign(r.neighbors, r.neighbors + r.offsets[r.n]);
  l.examined = r.stats.pairs_examined;
  psg_neighbor_result_free(&r);
  return l;
}

// ---------------------------------------------------------------------------
// report rendering (io.hpp:24-40, io.cpp:140-225)

std::string fmt_num(double v) { return nlohmann::json(v).dump(); }  // main.cpp:44-46

struct Report {
  std::string algorithm, params, dataset;
  uint64_t pair_index_1 = 0, pair_index_2 = 0;
  double distance_or_matches = 0.0;
  uint64_t pairs_examined = 0, iterations = 0;
  double wall_seconds = 0.0;
  uint64_t seed = 0;
};

// The report schema as one table: the JSON object, the CSV header and row,
// and verify's field comparison all walk it in this (the reference's
// io.cpp:140-155) order.
struct Field {
  const char* name;
  nlohmann::json (*get)(const Report&);
  bool replayed;  // compared by verify (params and wall time are not)
};
const Field kFields[] = {
    {"algorithm", [](const Report& r) { return nlohmann::json(r.algorithm); }, true},
    {"params", [](const Report& r) { return nlohmann::json(r.params); }, false},
    {"dataset", [](const Report& r) { return nlohmann::json(r.dataset); }, true},
    {"pair_index_1", [](const Report& r) { return nlohmann::json(r.pair_index_1); }, true},
    {"pair_index_2", [](const Report& r) { return nlohmann::json(r.pair_index_2); }, true},
    {"distance_or_matches", [](const Report& r) { return nlohmann::json(r.distance_or_matches); }, true},
    {"pairs_examined", [](const Report& r) { return nlohmann::json(r.pairs_examined); }, true},
    {"iterations", [](const Report& r) { return nlohmann::json(r.iterations); }, true},
    {"wall_seconds", [](const Report& r) { return nlohmann::json(r.wall_seconds); }, false},
    {"seed", [](const Report& r) { return nlohmann::json(r.seed); }, true},
};

nlohmann::json to_json(const Report& r) {
  nlohmann::json j = nlohmann::json::object();
  for (const Field& f : kFields) j[f.name] = f.get(r);
  return j;
}

// RFC 4180 cell from the JSON scalar text, so a value has the same bytes in
// both formats; std::quoted with '"' as its own escape doubles inner quotes.
std::string csv_cell(const nlohmann::json& v) {
  const std::string text = v.is_string() ? v.get<std::string>() : v.dump();
  if (text.find_first_of(",\"\n") == std::string::npos) return text;
  std::ostringstream q;
  q << std::quoted(text, '"', '"');
  return q.str();
}

std::string reports_to_csv(const std::vector<Report>& reports) {
  std::ostringstream csv;
  const char* sep = "";
  for (const Field& f : kFields) csv << std::exchange(sep, ",") << f.name;
  csv << '\n';
  for (const Report& r : reports) {
    sep = "";
    for (const Field& f : kFields) csv << std::exchange(sep, ",") << csv_cell(f.get(r));
    csv << '\n';
  }
  return csv.str();
}

// Whole-file text I/O (stdio); failures are the reference's messages.
void write_text_file(const std::string& path, const std::string& content) {
  std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(path.c_str(), "wb"), &std::fclose);
  if (!f) throw std::runtime_error("cannot open " + path + " for writing");
  if (std::fwrite(content.data(), 1, content.size(), f.get()) != content.size() || std::fflush(f.get()) != 0)
    throw std::runtime_error("write failed for " + path);
}

std::string read_text_file(const std::string& path) {
  std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(path.c_str(), "rb"), &std::fclose);
  if (!f) throw std::runtime_error("cannot open " + path + " for reading");
  std::string text;
  char buf[1 << 16];
  for (size_t got; (got = std::fread(buf, 1, sizeof buf, f.get())) > 0;) text.append(buf, got);
  return text;
}

// "--out dir/name.ext" -> "dir/name": the last '.' of the file-name part.
std::string strip_extension(const std::string& p) {
  const size_t name = p.find_last_of('/') + 1;  // npos + 1 == 0
  const size_t dot = p.find_last_of('.');
  return dot != std::string::npos && dot >= name ? p.substr(0, dot) : p;
}

// ---------------------------------------------------------------------------
// params lines: the report's replayable command line, kept as tokens and
// rendered once; a token that is empty or holds a blank or a quote is
// double-quoted (split_params below takes it apart again).

struct ParamLine {
  std::vector<std::string> toks;
  explicit ParamLine(std::string cmd) { toks.push_back(std::move(cmd)); }
  void value(std::string v) { toks.push_back(std::move(v)); }
  void flag(const char* name) { toks.emplace_back(name); }
  void option(const char* name, std::string v) {
    flag(name);
    value(std::move(v));
  }
  void option(const char* name, uint64_t v) { option(name, std::to_string(v)); }
  void option(const char* name, double v) { option(name, fmt_num(v)); }
  std::string render() const {
    std::string line;
    for (const std::string& t : toks) {
      if (!line.empty()) line += ' ';
      const bool bare = !t.empty() && t.find_first_of(" \t\"'") == std::string::npos;
      line += bare ? t : '"' + t + '"';
    }
    return line;
  }
};

// Whitespace split honouring "..." and '...' quoting (what CLI11's split_up
// does for the reference's verify).
std::vector<std::string> split_params(const std::string& s) {
  std::vector<std::string> out;
  size_t i = 0;
  while (i < s.size()) {
    while (i < s.size() && (s[i] == ' ' || s[i] == '\t')) ++i;
    if (i >= s.size()) break;
    std::string tok;
    if (s[i] == '"' || s[i] == '\'') {
      const char q = s[i++];
      const size_t e = s.find(q, i);
      tok = s.substr(i, e == std::string::npos ? std::string::npos : e - i);
      i = e == std::string::npos ? s.size() : e + 1;
    } else {
      while (i < s.size() && s[i] != ' ' && s[i] != '\t') tok += s[i++];
    }
    out.push_back(tok);
  }
  return out;
}

// ---------------------------------------------------------------------------
// argument parsing

struct Spec {
  std::set<std::string> options, flags;
  std::vector<std::string> positionals;  // names, in order (all optional here)
};

struct Parsed {
  std::map<std::string, std::string> opt;
  std::set<std::string> flags;
  std::vector<std::string> pos;
  bool has(const std::string& k) const { return opt.count(k) != 0; }
  std::string str(const std::string& k, const std::string& def = "") const {
    auto it = opt.find(k);
    return it == opt.end() ? def : it->second;
  }
};

Parsed parse(const std::vector<std::string>& args, size_t from, const Spec& spec) {
  Parsed p;
  for (size_t i = from; i < args.size(); ++i) {
    const std::string& a = args[i];
    if (a.size() > 2 && a.compare(0, 2, "--") == 0) {
      std::string key = a, val;
      bool inline_val = false;
      if (const auto eq = a.find('='); eq != std::string::npos) {
        key = a.substr(0, eq);
        val = a.substr(eq + 1);
        inline_val = true;
      }
      if (spec.flags.count(key)) {
        if (inline_val) throw usage_error(key + " is a flag and takes no value");
        p.flags.insert(key);
      } else if (spec.options.count(key)) {
        if (!inline_val) {
          if (i + 1 >= args.size()) throw usage_error(key + " requires a value");
          val = args[++i];
        }
        p.opt[key] = val;
      } else {
        throw usage_error("the following argument was not expected: " + a);
      }
    } else {
      if (p.pos.size() >= spec.positionals.size()) throw usage_error("the following argument was not expected: " + a);
      p.pos.push_back(a);
    }
  }
  return p;
}

uint64_t to_u64(const std::string& key, const std::string& v) {
  char* e = nullptr;
  errno = 0;
  if (v.empty() || v[0] == '-') throw usage_error(key + ": expected a non-negative integer, got '" + v + "'");
  const unsigned long long x = std::strtoull(v.c_str(), &e, 10);
  if (*e != '\0' || errno == ERANGE) throw usage_error(key + ": expected a non-negative integer, got '" + v + "'");
  return x;
}

int64_t to_i64(const std::string& key, const std::string& v) {
  char* e = nullptr;
  errno = 0;
  const long long x = std::strtoll(v.c_str(), &e, 10);
  if (v.empty() || *e != '\0' || errno == ERANGE) throw usage_error(key + ": expected an integer, got '" + v + "'");
  return x;
}

double to_f64(const std::string& key, const std::string& v) {
  char* e = nullptr;
  errno = 0;
  const double x = std::strtod(v.c_str(), &e);
  if (v.empty() || *e != '\0' || errno == ERANGE) throw usage_error(key + ": expected a number, got '" + v + "'");
  return x;
}

std::vector<std::string> split_list(const std::string& v) {
  std::vector<std::string> out;
  size_t b = 0;
  for (;;) {
    const size_t e = v.find(',', b);
    out.push_back(v.substr(b, e == std::string::npos ? std::string::npos : e - b));
    if (e == std::string::npos) break;
    b = e + 1;
  }
  return out;
}

const std::set<std::string> kEngines{"mpr", "mk", "brute", "gpu"};

std::string engine_of(const Parsed& p, const char* key, const std::string& def) {
  const std::string e = p.str(key, def);
  if (!kEngines.count(e)) throw usage_error(std::string(key) + ": " + e + " not in {brute, gpu, mk, mpr}");
  return e;
}

struct Timer {
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  double seconds() const { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); }
};

// ---------------------------------------------------------------------------
// shared options (main.cpp:86-108)

struct CommonOpts {
  std::string out;
  bool deterministic = false;
  std::string version_tag = kVersion;
};

void add_common(Spec& s) {
  s.options.insert({"--out", "--version-tag"});
  s.flags.insert("--deterministic");
}

CommonOpts common_of(const Parsed& p) {
  CommonOpts c;
  c.out = p.str("--out");
  c.deterministic = p.flags.count("--deterministic") != 0;
  c.version_tag = p.str("--version-tag", kVersion);
  return c;
}

void finish_params(ParamLine& pb, const CommonOpts& c) {
  pb.option("--version-tag", c.version_tag);
  if (c.deterministic) pb.flag("--deterministic");
}

int emit(std::vector<Report> reports, const CommonOpts& c, std::vector<Report>* capture) {  // main.cpp:176-191
  if (capture) {
    for (auto& r : reports) capture->push_back(std::move(r));
    return 0;
  }
  std::string json;
  if (reports.size() == 1) {
    json = to_json(reports[0]).dump(2) + "\n";
  } else {
    nlohmann::json arr = nlohmann::json::array();
    for (const Report& r : reports) arr.push_back(to_json(r));
    json = arr.dump(2) + "\n";
  }
  std::cout << json;
  if (!c.out.empty()) {
    const std::string base = strip_extension(c.out);
    write_text_file(base + ".json", json);
    write_text_file(base + ".csv", reports_to_csv(reports));
  }
  return 0;
}

int not_a_report_command(std::vector<Report>* capture, const char* name) {
  if (!capture) return 0;
  std::cerr << "error: " << name << " does not produce a report to verify\n";
  return 2;
}

// ---------------------------------------------------------------------------
// inputs

std::vector<double> load_series(const std::string& path) {  // io.cpp:44-60 via the library's parser
  double* v = nullptr;
  uint64_t n = 0;
  check(psg_load_series_text(path.c_str(), &v, &n));
  std::vector<double> out(v, v + n);
  psg_free(v);
  return out;
}

std::vector<double> gen_walk(uint64_t n, uint64_t seed, double stddev) {  // datagen.cpp:10-23
  std::vector<double> v(n);
  check(psg_gen_random_walk(n, seed, stddev, v.data()));
  return v;
}

Points windows_of(const std::vector<double>& s, uint64_t len) {  // series.cpp:34-42 (raw windows)
  psg_pointset* ps = nullptr;
  check(psg_pointset_windows_f64(s.data(), s.size(), len, 0, 0, &ps));
  return Points(ps);
}

uint64_t admissible_pair_count(uint64_t n, uint64_t zone) {  // main.cpp:384-393
  if (zone == 0) return n * (n - 1) / 2;
  uint64_t c = 0;
  for (uint64_t i = 0; i < n; ++i)
    if (n > i + zone) c += n - i - zone;
  return c;
}

struct PairRun {
  psg_pair_result r{};
  double wall = 0.0;
};

PairRun run_pair(psg_pointset* ps, const std::string& eng, uint64_t q, double f, uint64_t seed, uint64_t zone) {
  if (psg_pointset_size(ps) < 2) throw std::invalid_argument("closest_pair needs at least 2 points");
  Timer t;
  PairRun pr;
  if (eng == "brute")
    check(psg_brute_force_closest_pair_ps(ps, zone, &pr.r));
  else
    check(psg_closest_pair_ps(ps, q, eng == "mk" ? 1.0 : f, seed, zone, &pr.r));
  pr.wall = t.seconds();
  return pr;
}

struct FrnnRun {
  Lists lists;
  double wall = 0.0;
};

FrnnRun run_frnn(psg_pointset* ps, const std::string& eng, double radius, uint64_t q, double f, uint64_t seed,
                 uint64_t zone) {
  const uint64_t n = psg_pointset_size(ps);
  if (n == 0) throw std::invalid_argument("empty input");
  Timer t;
  FrnnRun fr;
  psg_neighbor_result r{};
  if (eng == "brute") {
    // the device all-pairs engine over the same points (refscan.cpp:211-227)
    check(psg_brute_force_neighbors_ps(ps, radius, zone, 1, &r));
    fr.lists = take(r);
    fr.lists.examined = admissible_pair_count(n, zone);
  } else {
    check(psg_fixed_radius_neighbors_ps(ps, radius, q, eng == "mk" ? 1.0 : f, seed, zone, 1, &r));
    fr.lists = take(r);
  }
  fr.wall = t.seconds();
  return fr;
}

// ---------------------------------------------------------------------------
// gen-walk (main.cpp:200-214)

int cmd_gen_walk(const std::vector<std::string>& args, std::vector<Report>* capture) {
  Spec s;
  s.options = {"--n", "--seed", "--stddev", "--out"};
  const Parsed p = parse(args, 1, s);
  if (!p.has("--n")) throw usage_error("--n is required");
  if (!p.has("--out")) throw usage_error("--out is required");
  if (const int rc = not_a_report_command(capture, "gen-walk")) return rc;
  const uint64_t n = to_u64("--n", p.str("--n"));
  const std::vector<double> v = gen_walk(n, to_u64("--seed", p.str("--seed", "1")),
                                         to_f64("--stddev", p.str("--stddev", "1")));
  check(psg_save_series_text(p.str("--out").c_str(), v.data(), v.size()));
  std::cout << "wrote " << n << " values to " << p.str("--out") << "\n";
  return 0;
}

// ---------------------------------------------------------------------------
// series scans: motif (main.cpp:262-382) and frnn (main.cpp:396-491)

struct SeriesOpts {
  std::string series;
  uint64_t gen_n = 0;
  double stddev = 1.0;
  uint64_t len = 0, refs = 10, seed = 1;
  double factor = 10.0;
  int64_t exclusion = -1;
  std::string engine = "mpr", verify_engine;
  CommonOpts common;
};

Spec series_spec() {
  Spec s;
  s.positionals = {"series"};
  s.options = {"--gen-walk", "--walk-stddev", "--len", "--refs", "--factor", "--seed", "--exclusion", "--engine",
               "--verify"};
  add_common(s);
  return s;
}

SeriesOpts series_opts(const Parsed& p) {
  SeriesOpts o;
  if (!p.pos.empty()) o.series = p.pos[0];
  if (p.has("--gen-walk")) {
    if (!o.series.empty()) throw usage_error("series excludes --gen-walk");
    o.gen_n = to_u64("--gen-walk", p.str("--gen-walk"));
  }
  if (p.has("--walk-stddev")) {
    if (!p.has("--gen-walk")) throw usage_error("--walk-stddev requires --gen-walk");
    o.stddev = to_f64("--walk-stddev", p.str("--walk-stddev"));
  }
  if (!p.has("--len")) throw usage_error("--len is required");
  o.len = to_u64("--len", p.str("--len"));
  o.refs = to_u64("--refs", p.str("--refs", "10"));
  o.factor = to_f64("--factor", p.str("--factor", "10"));
  o.seed = to_u64("--seed", p.str("--seed", "1"));
  o.exclusion = to_i64("--exclusion", p.str("--exclusion", "-1"));
  o.engine = engine_of(p, "--engine", "mpr");
  if (p.has("--verify")) o.verify_engine = engine_of(p, "--verify", "");
  o.common = common_of(p);
  return o;
}

std::pair<std::vector<double>, std::string> series_input(const SeriesOpts& o) {  // main.cpp:300-317
  if (o.series.empty() == (o.gen_n == 0)) throw std::invalid_argument("pass a series file or --gen-walk, not both");
  if (o.series.empty())
    return {gen_walk(o.gen_n, o.seed, o.stddev), "gen-walk:n=" + std::to_string(o.gen_n) + ",seed=" +
                                                     std::to_string(o.seed) + ",stddev=" + fmt_num(o.stddev)};
  return {load_series(o.series), o.series};
}

void series_params(ParamLine& pb, const SeriesOpts& o, uint64_t zone, double f_eff) {  // main.cpp:319-331
  if (!o.series.empty()) {
    pb.value(o.series);
  } else {
    pb.option("--gen-walk", o.gen_n);
    pb.option("--walk-stddev", o.stddev);
  }
  pb.option("--len", o.len);
  pb.option("--refs", o.refs);
  pb.option("--factor", f_eff);
  pb.option("--seed", o.seed);
  pb.option("--exclusion", zone);
  pb.option("--engine", o.engine);
}

int pair_report(const std::string& cmd, psg_pointset* ps, const std::string& dataset, uint64_t q, double factor,
                uint64_t seed, uint64_t zone, const std::string& engine, const std::string& verify_engine,
                const CommonOpts& common, const std::function<void(ParamLine&, double)>& input_params,
                std::vector<Report>* capture) {
  const PairRun res = run_pair(ps, engine, q, factor, seed, zone);
  const double f_eff = engine == "mk" ? 1.0 : factor;
  ParamLine pb(cmd);
  input_params(pb, f_eff);
  finish_params(pb, common);
  Report r;
  r.algorithm = engine;
  r.params = pb.render();
  r.dataset = dataset;
  r.pair_index_1 = res.r.index_i + 1;
  r.pair_index_2 = res.r.index_j + 1;
  r.distance_or_matches = res.r.distance;
  r.pairs_examined = res.r.stats.pairs_examined;
  r.wall_seconds = common.deterministic ? 0.0 : res.wall;
  r.seed = seed;
  if (const int rc = emit({r}, common, capture)) return rc;
  if (!verify_engine.empty() && !capture) {  // main.cpp:368-381
    const PairRun other = run_pair(ps, verify_engine, q, factor, seed, zone);
    if (other.r.distance != res.r.distance) {
      std::cerr << "verify: MISMATCH " << verify_engine << " found distance " << fmt_num(other.r.distance) << " at ("
                << other.r.index_i + 1 << ", " << other.r.index_j + 1 << "), " << engine << " found "
                << fmt_num(res.r.distance) << "\n";
      return 3;
    }
    std::cerr << "verify: " << verify_engine << " agrees, distance " << fmt_num(res.r.distance);
    if (other.r.index_i != res.r.index_i || other.r.index_j != res.r.index_j)
      std::cerr << " (tie, different pair: " << other.r.index_i + 1 << ", " << other.r.index_j + 1 << ")";
    std::cerr << "\n";
  }
  return 0;
}

int frnn_report(const std::string& cmd, psg_pointset* ps, const std::string& dataset, double radius, uint64_t q,
                double factor, uint64_t seed, uint64_t zone, const std::string& engine,
                const std::string& verify_engine, const std::string& pairs_out, const CommonOpts& common,
                const std::function<void(ParamLine&, double)>& input_params, std::vector<Report>* capture) {
  const FrnnRun res = run_frnn(ps, engine, radius, q, factor, seed, zone);
  const Lists& L = res.lists;
  const uint64_t pair_count = L.neighbors.size() / 2;
  uint64_t first_a = 0, first_b = 0;
  for (uint64_t i = 0; i < L.n && first_a == 0; ++i)
    for (uint64_t k = L.offsets[i]; k < L.offsets[i + 1]; ++k)
      if (L.neighbors[k] > i) {
        first_a = i + 1;
        first_b = L.neighbors[k] + 1;
        break;
      }
  const double f_eff = engine == "mk" ? 1.0 : factor;
  ParamLine pb(cmd);
  input_params(pb, f_eff);
  pb.option("--radius", radius);
  finish_params(pb, common);
  Report r;
  r.algorithm = engine;
  r.params = pb.render();
  r.dataset = dataset;
  r.pair_index_1 = first_a;
  r.pair_index_2 = first_b;
  r.distance_or_matches = static_cast<double>(pair_count);
  r.pairs_examined = L.examined;
  r.wall_seconds = common.deterministic ? 0.0 : res.wall;
  r.seed = seed;
  if (const int rc = emit({r}, common, capture)) return rc;
  if (!pairs_out.empty() && !capture) {  // main.cpp:465-478
    std::string out;
    for (uint64_t i = 0; i < L.n; ++i)
      for (uint64_t k = L.offsets[i]; k < L.offsets[i + 1]; ++k)
        if (L.neighbors[k] > i) {
          out += std::to_string(i + 1);
          out += ',';
          out += std::to_string(L.neighbors[k] + 1);
          out += '\n';
        }
    write_text_file(pairs_out, out);
  }
  if (!verify_engine.empty() && !capture) {  // main.cpp:480-489
    const FrnnRun other = run_frnn(ps, verify_engine, radius, q, factor, seed, zone);
    if (!(other.lists == L)) {
      std::cerr << "verify: MISMATCH neighbor lists differ between " << engine << " and " << verify_engine << "\n";
      return 3;
    }
    std::cerr << "verify: " << verify_engine << " agrees, " << pair_count << " neighbor pairs\n";
  }
  return 0;
}

int cmd_motif(const std::vector<std::string>& args, std::vector<Report>* capture) {
  const SeriesOpts o = series_opts(parse(args, 1, series_spec()));
  const auto [series, dataset] = series_input(o);
  Points ps = windows_of(series, o.len);
  const uint64_t zone = o.exclusion < 0 ? o.len : static_cast<uint64_t>(o.exclusion);
  return pair_report(
      "motif", ps.get(), dataset, o.refs, o.factor, o.seed, zone, o.engine, o.verify_engine, o.common,
      [&](ParamLine& pb, double f_eff) { series_params(pb, o, zone, f_eff); }, capture);
}

int cmd_frnn(const std::vector<std::string>& args, std::vector<Report>* capture) {
  Spec s = series_spec();
  s.options.insert({"--radius", "--pairs-out"});
  const Parsed p = parse(args, 1, s);
  const SeriesOpts o = series_opts(p);
  if (!p.has("--radius")) throw usage_error("--radius is required");
  const double radius = to_f64("--radius", p.str("--radius"));
  const auto [series, dataset] = series_input(o);
  Points ps = windows_of(series, o.len);
  const uint64_t zone = o.exclusion < 0 ? o.len : static_cast<uint64_t>(o.exclusion);
  return frnn_report(
      "frnn", ps.get(), dataset, radius, o.refs, o.factor, o.seed, zone, o.engine, o.verify_engine,
      p.str("--pairs-out"), o.common, [&](ParamLine& pb, double f_eff) { series_params(pb, o, zone, f_eff); },
      capture);
}

// ---------------------------------------------------------------------------
// point clouds (G5): closest / neighbors over the rows of a .psgb file

struct CloudOpts {
  std::string path;
  uint64_t refs = 10, seed = 1, zone = 0;
  double factor = 10.0;
  std::string engine = "mpr", verify_engine;
  CommonOpts common;
};

Spec cloud_spec() {
  Spec s;
  s.positionals = {"points"};
  s.options = {"--refs", "--factor", "--seed", "--exclusion", "--engine", "--verify"};
  add_common(s);
  return s;
}

CloudOpts cloud_opts(const Parsed& p) {
  CloudOpts o;
  if (p.pos.empty()) throw usage_error("points is required");
  o.path = p.pos[0];
  o.refs = to_u64("--refs", p.str("--refs", "10"));
  o.factor = to_f64("--factor", p.str("--factor", "10"));
  o.seed = to_u64("--seed", p.str("--seed", "1"));
  o.zone = to_u64("--exclusion", p.str("--exclusion", "0"));
  o.engine = engine_of(p, "--engine", "mpr");
  if (p.has("--verify")) o.verify_engine = engine_of(p, "--verify", "");
  o.common = common_of(p);
  return o;
}

void cloud_params(ParamLine& pb, const CloudOpts& o, double f_eff) {
  pb.value(o.path);
  pb.option("--refs", o.refs);
  pb.option("--factor", f_eff);
  pb.option("--seed", o.seed);
  pb.option("--exclusion", o.zone);
  pb.option("--engine", o.engine);
}

Points cloud_points(const std::string& path) {
  psg_pointset* ps = nullptr;
  check(psg_pointset_from_file(path.c_str(), &ps));
  return Points(ps);
}

int cmd_closest(const std::vector<std::string>& args, std::vector<Report>* capture) {
  const CloudOpts o = cloud_opts(parse(args, 1, cloud_spec()));
  Points ps = cloud_points(o.path);
  return pair_report(
      "closest", ps.get(), o.path, o.refs, o.factor, o.seed, o.zone, o.engine, o.verify_engine, o.common,
      [&](ParamLine& pb, double f_eff) { cloud_params(pb, o, f_eff); }, capture);
}

int cmd_neighbors(const std::vector<std::string>& args, std::vector<Report>* capture) {
  Spec s = cloud_spec();
  s.options.insert({"--radius", "--pairs-out"});
  const Parsed p = parse(args, 1, s);
  const CloudOpts o = cloud_opts(p);
  if (!p.has("--radius")) throw usage_error("--radius is required");
  const double radius = to_f64("--radius", p.str("--radius"));
  Points ps = cloud_points(o.path);
  return frnn_report(
      "neighbors", ps.get(), o.path, radius, o.refs, o.factor, o.seed, o.zone, o.engine, o.verify_engine,
      p.str("--pairs-out"), o.common, [&](ParamLine& pb, double f_eff) { cloud_params(pb, o, f_eff); }, capture);
}

// ---------------------------------------------------------------------------
// sweep (main.cpp:806-897)

int cmd_sweep(const std::vector<std::string>& args, std::vector<Report>* capture) {
  Spec s;
  s.options = {"--n-list", "--len-list", "--q-list", "--f-list", "--engines", "--reps", "--seed", "--out", "--raw-out"};
  s.flags = {"--deterministic"};
  const Parsed p = parse(args, 1, s);
  if (!p.has("--n-list")) throw usage_error("--n-list is required");
  if (!p.has("--len-list")) throw usage_error("--len-list is required");
  if (const int rc = not_a_report_command(capture, "sweep")) return rc;
  std::vector<uint64_t> ns, lens, qs{10};
  std::vector<double> fs{10.0};
  std::vector<std::string> engines{"mk", "mpr"};
  for (const auto& v : split_list(p.str("--n-list"))) ns.push_back(to_u64("--n-list", v));
  for (const auto& v : split_list(p.str("--len-list"))) lens.push_back(to_u64("--len-list", v));
  if (p.has("--q-list")) {
    qs.clear();
    for (const auto& v : split_list(p.str("--q-list"))) qs.push_back(to_u64("--q-list", v));
  }
  if (p.has("--f-list")) {
    fs.clear();
    for (const auto& v : split_list(p.str("--f-list"))) fs.push_back(to_f64("--f-list", v));
  }
  if (p.has("--engines")) {
    engines = split_list(p.str("--engines"));
    for (const auto& e : engines)
      if (!kEngines.count(e)) throw usage_error("--engines: " + e + " not in {brute, gpu, mk, mpr}");
  }
  const uint64_t reps = to_u64("--reps", p.str("--reps", "10"));
  const uint64_t seed = to_u64("--seed", p.str("--seed", "1"));
  const bool deterministic = p.flags.count("--deterministic") != 0;
  if (reps < 1) throw std::invalid_argument("--reps must be at least 1");

  struct Agg {
    double pairs = 0.0, wall = 0.0;
    uint64_t count = 0;
  };
  std::vector<std::string> agg_keys;
  std::vector<Agg> agg;
  auto agg_index = [&](const std::string& key) {
    for (size_t i = 0; i < agg_keys.size(); ++i)
      if (agg_keys[i] == key) return i;
    agg_keys.push_back(key);
    agg.emplace_back();
    return agg.size() - 1;
  };
  std::string raw = "n,len,q,f,engine,rep,seed,pair_index_1,pair_index_2,distance,pairs_examined,wall_seconds\n";
  for (size_t ni = 0; ni < ns.size(); ++ni) {
    for (size_t li = 0; li < lens.size(); ++li) {
      const uint64_t n = ns[ni], len = lens[li], cell = ni * lens.size() + li;
      for (uint64_t rep = 0; rep < reps; ++rep) {
        const uint64_t dseed = psg_derive_seed(psg_derive_seed(seed, cell), rep);  // rng.cpp:57-59
        const std::vector<double> walk = gen_walk(n, dseed, 1.0);
        Points ps = windows_of(walk, len);
        const uint64_t zone = len;
        double cell_distance = 0.0;
        bool have = false;
        for (const std::string& eng : engines) {
          const bool brute = eng == "brute";
          const std::vector<uint64_t> ql = brute ? std::vector<uint64_t>{0} : qs;
          const std::vector<double> fl = brute || eng == "mk" ? std::vector<double>{1.0} : fs;
          for (const uint64_t q : ql) {
            for (const double f : fl) {
              const PairRun r = run_pair(ps.get(), brute ? "brute" : "mpr", q, f, dseed, zone);
              const double wall = deterministic ? 0.0 : r.wall;
              if (!have) {
                cell_distance = r.r.distance;
                have = true;
              } else if (r.r.distance != cell_distance) {
                std::cerr << "sweep: engines disagree on n=" << n << " len=" << len << " rep=" << rep + 1 << ": "
                          << fmt_num(r.r.distance) << " vs " << fmt_num(cell_distance) << "\n";
                return 3;
              }
              raw += std::to_string(n) + "," + std::to_string(len) + "," + std::to_string(q) + "," + fmt_num(f) +
                     "," + eng + "," + std::to_string(rep + 1) + "," + std::to_string(dseed) + "," +
                     std::to_string(r.r.index_i + 1) + "," + std::to_string(r.r.index_j + 1) + "," +
                     fmt_num(r.r.distance) + "," + std::to_string(r.r.stats.pairs_examined) + "," + fmt_num(wall) +
                     "\n";
              const size_t ai = agg_index(std::to_string(n) + "," + std::to_string(len) + "," + std::to_string(q) +
                                          "," + fmt_num(f) + "," + eng);
              agg[ai].pairs += static_cast<double>(r.r.stats.pairs_examined);
              agg[ai].wall += wall;
              agg[ai].count += 1;
            }
          }
        }
      }
    }
  }
  std::string table = "n,len,q,f,engine,reps,mean_pairs_examined,mean_wall_seconds\n";
  for (size_t i = 0; i < agg_keys.size(); ++i) {
    const double c = static_cast<double>(agg[i].count);
    table += agg_keys[i] + "," + std::to_string(agg[i].count) + "," + fmt_num(agg[i].pairs / c) + "," +
             fmt_num(agg[i].wall / c) + "\n";
  }
  std::cout << table;
  const std::string out = p.str("--out"), raw_out = p.str("--raw-out");
  if (!out.empty()) {
    write_text_file(out, table);
    write_text_file(raw_out.empty() ? strip_extension(out) + ".raw.csv" : raw_out, raw);
  } else if (!raw_out.empty()) {
    write_text_file(raw_out, raw);
  }
  return 0;
}

// ---------------------------------------------------------------------------
// verify (main.cpp:899-1013)

int run_cli(const std::vector<std::string>& args, std::vector<Report>* capture);

// First replayed field where the stored row and the re-run differ, as
// "<field> expected <stored> got <re-run>" (empty when they agree).
std::string first_difference(const nlohmann::json& stored, const Report& rerun) {
  for (const Field& f : kFields) {
    if (!f.replayed) continue;
    const auto it = stored.find(f.name);
    if (it == stored.end()) return std::string(f.name) + " missing from report";
    const nlohmann::json now = f.get(rerun);
    if (*it != now) return std::string(f.name) + " expected " + it->dump() + " got " + now.dump();
  }
  return {};
}

// One params line and the stored rows it produced, in file order.
struct ReplayGroup {
  std::string params;
  std::vector<const nlohmann::json*> rows;
};

// Replays one group; returns the line verify prints for it.
std::string replay(const ReplayGroup& g) {
  if (g.params.empty()) return "MISMATCH report has no params line";
  const std::vector<std::string> argv = split_params(g.params);
  if (argv.empty() || argv[0] == "verify") return "MISMATCH params line is not replayable: " + g.params;
  std::vector<Report> rerun;
  if (const int rc = run_cli(argv, &rerun); rc != 0)
    return "MISMATCH re-run exited with code " + std::to_string(rc) + ": " + g.params;
  if (rerun.size() != g.rows.size())
    return "MISMATCH re-run produced " + std::to_string(rerun.size()) + " reports, file holds " +
           std::to_string(g.rows.size()) + ": " + g.params;
  for (size_t k = 0; k < rerun.size(); ++k)
    if (std::string why = first_difference(*g.rows[k], rerun[k]); !why.empty())
      return "MISMATCH row " + std::to_string(k + 1) + ": " + why + ": " + g.params;
  return "OK " + g.params;
}

int cmd_verify(const std::vector<std::string>& args, std::vector<Report>* capture) {
  Spec s;
  s.positionals = {"report"};
  const Parsed p = parse(args, 1, s);
  if (p.pos.empty()) throw usage_error("report is required");
  if (capture) {
    std::cerr << "error: verify cannot replay a verify run\n";
    return 2;
  }
  nlohmann::json doc = nlohmann::json::parse(read_text_file(p.pos[0]));
  if (!doc.is_array()) doc = nlohmann::json::array({std::move(doc)});
  if (doc.empty()) {
    std::cerr << "error: report file holds no reports\n";
    return 2;
  }
  // rows sharing a params line came from one run: group them, first-seen order
  std::vector<ReplayGroup> groups;
  std::map<std::string, size_t> group_of;
  for (const nlohmann::json& row : doc) {
    const std::string params = row.value("params", "");
    const auto [it, fresh] = group_of.try_emplace(params, groups.size());
    if (fresh) groups.push_back({params, {}});
    groups[it->second].rows.push_back(&row);
  }
  int failed = 0;
  for (const ReplayGroup& g : groups) {
    const std::string line = replay(g);
    failed += line.rfind("OK ", 0) != 0;
    std::cout << "verify: " << line << "\n";
  }
  return failed ? 3 : 0;
}

// ---------------------------------------------------------------------------

const char* kUsage =
    "pairscan-gpu: exact pair scans over series and point clouds on B200\n"
    "usage: pairscan-gpu <command> [options]\n"
    "  gen-walk  --n N --out PATH [--seed S] [--stddev X]\n"
    "  motif     [SERIES | --gen-walk N [--walk-stddev X]] --len L [--refs Q] [--factor F] [--seed S]\n"
    "            [--exclusion Z] [--engine mpr|mk|brute|gpu] [--verify ENGINE] [--out P] [--deterministic]\n"
    "  frnn      same inputs as motif + --radius R [--pairs-out PATH]\n"
    "  closest   POINTS.psgb [--refs Q] [--factor F] [--seed S] [--exclusion Z] [--engine E] [--verify E] ...\n"
    "  neighbors POINTS.psgb --radius R [--pairs-out PATH] (options as closest)\n"
    "  sweep     --n-list N,.. --len-list L,.. [--q-list] [--f-list] [--engines] [--reps] [--seed] [--out]\n"
    "            [--raw-out] [--deterministic]\n"
    "  verify    REPORT.json\n";

int run_cli(const std::vector<std::string>& args, std::vector<Report>* capture) {
  try {
    if (args.empty()) throw usage_error("a subcommand is required");
    const std::string& sub = args[0];
    if (sub == "--version") {
      std::cout << kVersion << "\n";
      return 0;
    }
    if (sub == "--help" || sub == "-h") {
      std::cout << kUsage;
      return 0;
    }
    if (sub == "gen-walk") return cmd_gen_walk(args, capture);
    if (sub == "motif") return cmd_motif(args, capture);
    if (sub == "frnn") return cmd_frnn(args, capture);
    if (sub == "closest") return cmd_closest(args, capture);
    if (sub == "neighbors") return cmd_neighbors(args, capture);
    if (sub == "sweep") return cmd_sweep(args, capture);
    if (sub == "verify") return cmd_verify(args, capture);
    throw usage_error("unknown subcommand: " + sub);
  } catch (const usage_error& e) {
    std::cerr << "error: " << e.what() << "\n" << (capture ? "" : kUsage);
    return 2;
  } catch (const std::exception& e) {  // main.cpp:1202-1205
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  }
}

}  // namespace

int main(int argc, char** argv) { return run_cli(std::vector<std::string>(argv + 1, argv + argc), nullptr); }
