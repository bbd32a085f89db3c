// On-disk datasets: reference text layout + binary twin (see dataset_io.hpp).
// Reference: src/dataset_io.cpp:40-165.
#include "dataset_io.hpp"

#include <algorithm>
#include <cerrno>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <thread>

namespace dgnn {
namespace fs = std::filesystem;

namespace {

[[noreturn]] void fail(const std::string& msg) { throw std::invalid_argument(msg); }
void check(bool ok, const std::string& msg) {
  if (!ok) fail(msg);
}

int pick_threads(int requested, int64_t work, int64_t grain) {
  int hw = static_cast<int>(std::thread::hardware_concurrency());
  int t = requested > 0 ? requested : std::max(1, std::min(hw, 16));
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(t, work / grain + 1)));
}

template <class F>
void parallel_for(int threads, int64_t n, F&& f) {  // f(begin, end, part)
  if (threads <= 1 || n < 2) {
    f(int64_t{0}, n, 0);
    return;
  }
  std::vector<std::thread> pool;
  for (int p = 0; p < threads; ++p) {
    const int64_t b = n * p / threads, e = n * (p + 1) / threads;
    pool.emplace_back([&, b, e, p] { f(b, e, p); });
  }
  for (auto& th : pool) th.join();
}

// read_file (src/dataset_io.cpp:30-36): whole file, NUL-terminated.
std::string read_file(const fs::path& p) {
  std::ifstream in(p, std::ios::binary | std::ios::ate);
  check(in.good(), "cannot open for reading: " + p.string());
  const std::streamoff n = in.tellg();
  std::string s(static_cast<size_t>(std::max<std::streamoff>(n, 0)), '\0');
  in.seekg(0);
  if (n > 0) in.read(s.data(), n);
  return s;
}

// write_file (src/dataset_io.cpp:24-28)
struct Out {
  std::ofstream f;
  explicit Out(const fs::path& p) : f(p, std::ios::binary | std::ios::trunc) {
    check(f.good(), "cannot open for writing: " + p.string());
  }
  void put(const void* d, size_t n) {
    if (n) f.write(static_cast<const char*>(d), static_cast<std::streamsize>(n));
  }
  void put(const std::string& s) { put(s.data(), s.size()); }
};

inline bool is_space(char c) { return c == ' ' || (c >= '\t' && c <= '\r'); }

// `stream >> long long` (num_get): skip whitespace, optional sign, decimal
// digits; no digits or overflow = failure.
inline bool extract_ll(const char*& p, const char* end, long long& v) {
  while (p < end && is_space(*p)) ++p;
  const char* q = p;
  bool neg = false;
  if (q < end && (*q == '+' || *q == '-')) neg = *q++ == '-';
  if (q >= end || *q < '0' || *q > '9') return false;
  unsigned long long acc = 0;
  const unsigned long long lim = neg ? 9223372036854775808ull : 9223372036854775807ull;
  for (; q < end && *q >= '0' && *q <= '9'; ++q) {
    const unsigned dig = static_cast<unsigned>(*q - '0');
    if (acc > (lim - dig) / 10) return false;
    acc = acc * 10 + dig;
  }
  v = neg ? static_cast<long long>(0ull - acc) : static_cast<long long>(acc);
  p = q;
  return true;
}

// `stream >> std::string`: one whitespace-delimited token.
inline bool extract_token(const char*& p, const char* end, const char*& b, const char*& e) {
  while (p < end && is_space(*p)) ++p;
  if (p >= end) return false;
  b = p;
  while (p < end && !is_space(*p)) ++p;
  e = p;
  return true;
}

bool all_space(const char* b, const char* e) {
  for (; b < e; ++b)
    if (!is_space(*b)) return false;
  return true;
}

// std::stod on one CSV cell [b, e) of a NUL-terminated buffer (strtod
// semantics: leading whitespace, trailing junk ignored; no conversion ->
// invalid_argument("stod"), ERANGE -> out_of_range("stod")).
double stod_cell(const char* b, const char* e) {
  if (all_space(b, e)) throw std::invalid_argument("stod");
  char* endp = nullptr;
  errno = 0;
  const double v = std::strtod(b, &endp);
  if (endp == b || endp > e) throw std::invalid_argument("stod");
  if (errno == ERANGE) throw std::out_of_range("stod");
  return v;
}

long stol_cell(const char* b, const char* e) {
  if (all_space(b, e)) throw std::invalid_argument("stol");
  char* endp = nullptr;
  errno = 0;
  const long v = std::strtol(b, &endp, 10);
  if (endp == b || endp > e) throw std::invalid_argument("stol");
  if (errno == ERANGE) throw std::out_of_range("stol");
  return v;
}

// Repeated std::getline(row, cell, ','): an empty line has no cells, a
// trailing delimiter does not start an empty cell.
template <class F>
void for_cells(const char* b, const char* e, F&& f) {  // f(cb, ce) -> false stops
  const char* p = b;
  while (p < e) {
    const char* q = static_cast<const char*>(std::memchr(p, ',', static_cast<size_t>(e - p)));
    const char* ce = q ? q : e;
    if (!f(p, ce)) return;
    p = q ? q + 1 : e;
  }
}

// Line starts of the first `want` lines (std::getline on '\n').
std::vector<std::pair<const char*, const char*>> split_lines(const std::string& s, int64_t want) {
  std::vector<std::pair<const char*, const char*>> lines;
  const char* p = s.data();
  const char* end = p + s.size();
  while (p < end && (want < 0 || static_cast<int64_t>(lines.size()) < want)) {
    const char* q = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(end - p)));
    const char* le = q ? q : end;
    lines.emplace_back(p, le);
    p = q ? q + 1 : end;
  }
  return lines;
}

struct ErrSlot {  // first failure in file order across parallel parts
  int64_t at = INT64_MAX;
  int kind = 0;  // 1 invalid_argument, 2 out_of_range
  std::string msg;
  void set(int64_t i, int k, const std::string& m) {
    if (i < at) {
      at = i;
      kind = k;
      msg = m;
    }
  }
  void raise() const {
    if (kind == 1) throw std::invalid_argument(msg);
    if (kind == 2) throw std::out_of_range(msg);
  }
};

// ---- binary twin
constexpr char kMagic[8] = {'D', 'G', 'N', 'N', 'B', '2', '0', '0'};
struct BinBase {
  char magic[8];
  uint32_t version, kind;
  int64_t num_edges;
  int32_t num_nodes, dim;
};
struct BinStep {
  char magic[8];
  uint32_t version, kind;
  int64_t n_del, n_ins, n_changed;
  int32_t t, dim;
};
static_assert(sizeof(BinBase) == 32 && sizeof(BinStep) == 48, "binary header layout");

fs::path step_path(const fs::path& dir, int32_t t, const char* ext) {
  return dir / ("delta_" + std::to_string(t) + ext);
}

// Flat JSON object with integer / string values (the manifest).
std::vector<std::pair<std::string, std::string>> parse_flat_json(const std::string& s) {
  std::vector<std::pair<std::string, std::string>> kv;
  size_t i = 0;
  auto ws = [&] {
    while (i < s.size() && is_space(s[i])) ++i;
  };
  auto str = [&] {
    check(i < s.size() && s[i] == '"', "malformed manifest");
    const size_t b = ++i;
    while (i < s.size() && s[i] != '"') ++i;
    check(i < s.size(), "malformed manifest");
    return s.substr(b, i++ - b);
  };
  ws();
  check(i < s.size() && s[i] == '{', "malformed manifest");
  ++i;
  ws();
  if (i < s.size() && s[i] == '}') return kv;
  for (;;) {
    ws();
    std::string k = str();
    ws();
    check(i < s.size() && s[i] == ':', "malformed manifest");
    ++i;
    ws();
    std::string v;
    if (i < s.size() && s[i] == '"') {
      v = "\"" + str() + "\"";
    } else {
      const size_t b = i;
      while (i < s.size() && s[i] != ',' && s[i] != '}' && !is_space(s[i])) ++i;
      v = s.substr(b, i - b);
    }
    kv.emplace_back(std::move(k), std::move(v));
    ws();
    check(i < s.size(), "malformed manifest");
    if (s[i] == '}') break;
    check(s[i] == ',', "malformed manifest");
    ++i;
  }
  return kv;
}

}  // namespace

void append_value(std::string& out, double v) {
  char buf[64];
  const int n = std::snprintf(buf, sizeof(buf), "%.9g", v);
  out.append(buf, static_cast<size_t>(n));
}

// ---------------------------------------------------------------- reader
DatasetReader::DatasetReader(fs::path dir, int threads) : dir_(std::move(dir)), threads_(threads) {
  // src/dataset_io.cpp:98-104
  const auto kv = parse_flat_json(read_file(dir_ / "manifest.json"));
  auto at = [&](const char* key) -> const std::string& {
    for (const auto& p : kv)
      if (p.first == key) return p.second;
    throw std::out_of_range(std::string("manifest key not found: ") + key);
  };
  auto as_int = [&](const char* key) -> long long {
    const std::string& v = at(key);
    const char* p = v.c_str();
    long long x = 0;
    check(extract_ll(p, v.c_str() + v.size(), x) && *p == '\0', "malformed manifest");
    return x;
  };
  m_.num_nodes = static_cast<int32_t>(as_int("num_nodes"));
  m_.feature_dim = static_cast<int32_t>(as_int("feature_dim"));
  m_.T = static_cast<int32_t>(as_int("T"));
  const long long ver = as_int("format_version");
  check(ver == 1 || ver == 2, "unsupported dataset format version");
  m_.format = static_cast<int32_t>(ver);
  if (ver == 2) check(at("encoding") == "\"b200-le\"", "unsupported dataset encoding");
  check(m_.num_nodes > 0 && m_.feature_dim > 0 && m_.T > 0, "malformed manifest");
}

void DatasetReader::read_base(std::vector<int32_t>& src, std::vector<int32_t>& dst,
                              std::vector<float>& feats) const {
  const int64_t N = m_.num_nodes, d = m_.feature_dim;
  if (m_.format == 2) {
    const fs::path p = dir_ / "snapshot_0.bin";
    std::ifstream in(p, std::ios::binary);
    check(in.good(), "cannot open for reading: " + p.string());
    BinBase h{};
    in.read(reinterpret_cast<char*>(&h), sizeof(h));
    check(in.good() && std::memcmp(h.magic, kMagic, 8) == 0 && h.version == 1 && h.kind == 0,
          "not a binary snapshot file: " + p.string());
    check(h.num_nodes == m_.num_nodes && h.dim == m_.feature_dim && h.num_edges >= 0,
          "binary snapshot does not match the manifest");
    src.resize(static_cast<size_t>(h.num_edges));
    dst.resize(static_cast<size_t>(h.num_edges));
    feats.resize(static_cast<size_t>(N * d));
    in.read(reinterpret_cast<char*>(src.data()), static_cast<std::streamsize>(4 * h.num_edges));
    in.read(reinterpret_cast<char*>(dst.data()), static_cast<std::streamsize>(4 * h.num_edges));
    in.read(reinterpret_cast<char*>(feats.data()), static_cast<std::streamsize>(4 * N * d));
    check(in.good(), "binary dataset file truncated: " + p.string());
    return;
  }
  // snapshot_0.edges: while (in >> src >> dst) (src/dataset_io.cpp:106-110).
  // Parallel over chunks cut at line boundaries; the extracted integers are
  // concatenated up to the first failing extraction, then paired, which is
  // exactly the sequential loop's result.
  {
    const std::string s = read_file(dir_ / "snapshot_0.edges");
    const int nt = pick_threads(threads_, static_cast<int64_t>(s.size()), 1 << 22);
    std::vector<size_t> cut(nt + 1, s.size());
    cut[0] = 0;
    for (int p = 1; p < nt; ++p) {
      size_t c = s.size() * p / nt;
      c = std::max(c, cut[p - 1]);
      while (c < s.size() && s[c] != '\n') ++c;
      cut[p] = std::min(s.size(), c + (c < s.size() ? 1 : 0));
    }
    std::vector<std::vector<long long>> vals(nt);
    std::vector<char> stopped(nt, 0);
    parallel_for(nt, nt, [&](int64_t b, int64_t e, int) {
      for (int64_t part = b; part < e; ++part) {
        const char* p = s.data() + cut[part];
        const char* end = s.data() + cut[part + 1];
        auto& v = vals[part];
        v.reserve(static_cast<size_t>((end - p) / 6));
        long long x;
        while (extract_ll(p, end, x)) v.push_back(x);
        // a stop before the chunk end (non-space left) is a failed extraction
        while (p < end && is_space(*p)) ++p;
        if (p < end) stopped[part] = 1;
      }
    });
    int64_t total = 0;
    for (int p = 0; p < nt; ++p) {
      total += static_cast<int64_t>(vals[p].size());
      if (stopped[p]) break;
    }
    const int64_t E = total / 2;
    src.resize(static_cast<size_t>(E));
    dst.resize(static_cast<size_t>(E));
    int64_t k = 0;
    for (int p = 0; p < nt && k < 2 * E; ++p) {
      for (long long x : vals[p]) {
        if (k >= 2 * E) break;
        (k & 1 ? dst : src)[static_cast<size_t>(k >> 1)] = static_cast<int32_t>(x);
        ++k;
      }
      if (stopped[p]) break;
    }
  }
  // snapshot_0.feats (src/dataset_io.cpp:111-123)
  {
    const std::string s = read_file(dir_ / "snapshot_0.feats");
    const auto lines = split_lines(s, N);
    feats.resize(static_cast<size_t>(N * d));
    ErrSlot err;
    if (static_cast<int64_t>(lines.size()) < N) err.set(static_cast<int64_t>(lines.size()), 1, "snapshot_0.feats truncated");
    const int64_t nl = static_cast<int64_t>(lines.size());
    const int nt = pick_threads(threads_, nl * d, 1 << 16);
    std::vector<ErrSlot> errs(nt);
    parallel_for(nt, nl, [&](int64_t b, int64_t e, int part) {
      for (int64_t i = b; i < e; ++i) {
        int64_t j = 0;
        float* row = feats.data() + i * d;
        try {
          for_cells(lines[i].first, lines[i].second, [&](const char* cb, const char* ce) {
            row[j++] = static_cast<float>(stod_cell(cb, ce));
            return j < d;
          });
        } catch (const std::out_of_range& x) {
          errs[part].set(i, 2, x.what());
          return;
        } catch (const std::invalid_argument& x) {
          errs[part].set(i, 1, x.what());
          return;
        }
        if (j < d) {
          errs[part].set(i, 1, "snapshot_0.feats row truncated");
          return;
        }
      }
    });
    for (const auto& e : errs) err.set(e.at, e.kind, e.msg);
    err.raise();
  }
}

void DatasetReader::read_step(int32_t t, CompactStep& out) const {
  check(t >= 1 && t < m_.T, "delta index out of range");
  const int64_t d = m_.feature_dim;
  out.del_src.clear();
  out.del_dst.clear();
  out.ins_src.clear();
  out.ins_dst.clear();
  out.changed.clear();
  out.changed_feats.clear();
  if (m_.format == 2) {
    const fs::path p = step_path(dir_, t, ".bin");
    std::ifstream in(p, std::ios::binary);
    check(in.good(), "cannot open for reading: " + p.string());
    BinStep h{};
    in.read(reinterpret_cast<char*>(&h), sizeof(h));
    check(in.good() && std::memcmp(h.magic, kMagic, 8) == 0 && h.version == 1 && h.kind == 1,
          "not a binary delta file: " + p.string());
    check(h.t == t && h.dim == m_.feature_dim && h.n_del >= 0 && h.n_ins >= 0 && h.n_changed >= 0,
          "binary delta does not match the manifest");
    auto rd = [&](auto& v, int64_t n) {
      v.resize(static_cast<size_t>(n));
      in.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(4 * n));
    };
    rd(out.del_src, h.n_del);
    rd(out.del_dst, h.n_del);
    rd(out.ins_src, h.n_ins);
    rd(out.ins_dst, h.n_ins);
    rd(out.changed, h.n_changed);
    rd(out.changed_feats, h.n_changed * d);
    check(in.good(), "binary dataset file truncated: " + p.string());
    return;
  }
  // delta_t.edges: while (in >> kind >> src >> dst) (src/dataset_io.cpp:131-145)
  {
    const std::string s = read_file(step_path(dir_, t, ".edges"));
    const char* p = s.data();
    const char* end = p + s.size();
    const char *kb, *ke;
    long long a, b;
    while (extract_token(p, end, kb, ke) && extract_ll(p, end, a) && extract_ll(p, end, b)) {
      const std::string_view kind(kb, static_cast<size_t>(ke - kb));
      if (kind == "D") {
        out.del_src.push_back(static_cast<int32_t>(a));
        out.del_dst.push_back(static_cast<int32_t>(b));
      } else if (kind == "I") {
        out.ins_src.push_back(static_cast<int32_t>(a));
        out.ins_dst.push_back(static_cast<int32_t>(b));
      } else {
        fail("bad delta edge tag: " + std::string(kind));
      }
    }
  }
  // delta_t.feats (src/dataset_io.cpp:146-162)
  {
    const std::string s = read_file(step_path(dir_, t, ".feats"));
    for (const auto& [lb, le] : split_lines(s, -1)) {
      if (lb == le) continue;
      bool first = true;
      int64_t arity = 0;
      const size_t base = out.changed_feats.size();
      for_cells(lb, le, [&](const char* cb, const char* ce) {
        if (first) {
          out.changed.push_back(static_cast<int32_t>(stol_cell(cb, ce)));
          first = false;
        } else {
          out.changed_feats.push_back(static_cast<float>(stod_cell(cb, ce)));
          ++arity;
        }
        return true;
      });
      check(!first, "delta feats row truncated");
      check(arity == d, "delta feats row has wrong arity");
      (void)base;
    }
  }
}

// ---------------------------------------------------------------- writer
void write_manifest(const fs::path& dir, const DatasetManifest& m) {
  fs::create_directories(dir);
  // nlohmann::json object keys are ordered ("T" < "encoding" < "feature_dim" < ...)
  std::string s = "{\"T\":" + std::to_string(m.T);
  if (m.format == 2) s += ",\"encoding\":\"b200-le\"";
  s += ",\"feature_dim\":" + std::to_string(m.feature_dim) +
       ",\"format_version\":" + std::to_string(m.format) +
       ",\"num_nodes\":" + std::to_string(m.num_nodes) + "}\n";
  Out(dir / "manifest.json").put(s);
}

void write_base(const fs::path& dir, const DatasetManifest& m, const int32_t* src,
                const int32_t* dst, int64_t num_edges, const float* feats, int threads) {
  const int64_t N = m.num_nodes, d = m.feature_dim;
  if (m.format == 2) {
    Out o(dir / "snapshot_0.bin");
    BinBase h{};
    std::memcpy(h.magic, kMagic, 8);
    h.version = 1;
    h.kind = 0;
    h.num_edges = num_edges;
    h.num_nodes = m.num_nodes;
    h.dim = m.feature_dim;
    o.put(&h, sizeof(h));
    o.put(src, 4 * static_cast<size_t>(num_edges));
    o.put(dst, 4 * static_cast<size_t>(num_edges));
    o.put(feats, 4 * static_cast<size_t>(N * d));
    return;
  }
  // src/dataset_io.cpp:50-67, formatted in parallel row blocks
  const int nt = pick_threads(threads, std::max<int64_t>(num_edges, N * d), 1 << 18);
  std::vector<std::string> parts(nt);
  {
    parallel_for(nt, num_edges, [&](int64_t b, int64_t e, int part) {
      std::string& s = parts[part];
      s.reserve(static_cast<size_t>((e - b) * 16));
      char buf[32];
      for (int64_t i = b; i < e; ++i) {
        int n = std::snprintf(buf, sizeof(buf), "%d\t%d\n", src[i], dst[i]);
        s.append(buf, static_cast<size_t>(n));
      }
    });
    Out o(dir / "snapshot_0.edges");
    for (auto& s : parts) {
      o.put(s);
      std::string().swap(s);
    }
  }
  {
    parallel_for(nt, N, [&](int64_t b, int64_t e, int part) {
      std::string& s = parts[part];
      s.reserve(static_cast<size_t>((e - b) * d * 13));
      for (int64_t i = b; i < e; ++i) {
        for (int64_t j = 0; j < d; ++j) {
          if (j) s += ',';
          append_value(s, static_cast<double>(feats[i * d + j]));
        }
        s += '\n';
      }
    });
    Out o(dir / "snapshot_0.feats");
    for (auto& s : parts) o.put(s);
  }
}

void write_step(const fs::path& dir, const DatasetManifest& m, int32_t t, const StepView& v) {
  const int64_t d = m.feature_dim;
  if (m.format == 2) {
    Out o(step_path(dir, t, ".bin"));
    BinStep h{};
    std::memcpy(h.magic, kMagic, 8);
    h.version = 1;
    h.kind = 1;
    h.n_del = v.n_del;
    h.n_ins = v.n_ins;
    h.n_changed = v.n_changed;
    h.t = t;
    h.dim = m.feature_dim;
    o.put(&h, sizeof(h));
    o.put(v.del_src, 4 * static_cast<size_t>(v.n_del));
    o.put(v.del_dst, 4 * static_cast<size_t>(v.n_del));
    o.put(v.ins_src, 4 * static_cast<size_t>(v.n_ins));
    o.put(v.ins_dst, 4 * static_cast<size_t>(v.n_ins));
    o.put(v.changed, 4 * static_cast<size_t>(v.n_changed));
    o.put(v.changed_feats, 4 * static_cast<size_t>(v.n_changed * d));
    return;
  }
  // src/dataset_io.cpp:69-94
  std::string s;
  s.reserve(static_cast<size_t>((v.n_del + v.n_ins) * 18));
  char buf[48];
  for (int64_t i = 0; i < v.n_del; ++i) {
    int n = std::snprintf(buf, sizeof(buf), "D %d %d\n", v.del_src[i], v.del_dst[i]);
    s.append(buf, static_cast<size_t>(n));
  }
  for (int64_t i = 0; i < v.n_ins; ++i) {
    int n = std::snprintf(buf, sizeof(buf), "I %d %d\n", v.ins_src[i], v.ins_dst[i]);
    s.append(buf, static_cast<size_t>(n));
  }
  Out(step_path(dir, t, ".edges")).put(s);
  s.clear();
  for (int64_t i = 0; i < v.n_changed; ++i) {
    s += std::to_string(v.changed[i]);
    for (int64_t j = 0; j < d; ++j) {
      s += ',';
      append_value(s, static_cast<double>(v.changed_feats[i * d + j]));
    }
    s += '\n';
  }
  Out(step_path(dir, t, ".feats")).put(s);
}

void save_compact(const CompactGraph& g, const fs::path& dir, int32_t format) {
  check(format == 1 || format == 2, "unsupported dataset format version");
  DatasetManifest m{g.num_nodes, g.feature_dim, g.num_snapshots, format};
  write_manifest(dir, m);
  write_base(dir, m, g.base_src.data(), g.base_dst.data(), static_cast<int64_t>(g.base_src.size()),
             g.base_feats.data());
  for (size_t i = 0; i < g.steps.size(); ++i) {
    const CompactStep& st = g.steps[i];
    StepView v;
    v.n_del = static_cast<int64_t>(st.del_src.size());
    v.n_ins = static_cast<int64_t>(st.ins_src.size());
    v.n_changed = static_cast<int64_t>(st.changed.size());
    v.del_src = st.del_src.data();
    v.del_dst = st.del_dst.data();
    v.ins_src = st.ins_src.data();
    v.ins_dst = st.ins_dst.data();
    v.changed = st.changed.data();
    v.changed_feats = st.changed_feats.data();
    write_step(dir, m, static_cast<int32_t>(i + 1), v);
  }
}

}  // namespace dgnn
