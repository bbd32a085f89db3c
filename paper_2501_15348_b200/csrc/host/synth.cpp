// Bit-exact streaming synthesize (see synth.hpp).
#include "synth.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <random>
#include <stdexcept>
#include <type_traits>
#include <cstdlib>
#include <new>
#include <sys/mman.h>

#include "aggregate.hpp"

namespace dgnn {
namespace {

inline uint64_t key_of(int32_t s, int32_t d) {
  return (static_cast<uint64_t>(static_cast<uint32_t>(s)) << 32) | static_cast<uint32_t>(d);
}

// 2 MB-page backed storage for the multi-GB random-access arrays (edge hash
// set, shuffle pool): with 4 KB pages every random probe is also a TLB miss.
template <class T>
struct HugeAlloc {
  using value_type = T;
  HugeAlloc() = default;
  template <class U>
  HugeAlloc(const HugeAlloc<U>&) {}
  T* allocate(size_t n) {
    const size_t bytes = n * sizeof(T);
    if (bytes < (size_t{8} << 20)) return static_cast<T*>(::operator new(bytes));
    const size_t huge = size_t{2} << 20;
    void* p = std::aligned_alloc(huge, (bytes + huge - 1) / huge * huge);
    if (!p) throw std::bad_alloc();
    madvise(p, (bytes + huge - 1) / huge * huge, MADV_HUGEPAGE);
    return static_cast<T*>(p);
  }
  void deallocate(T* p, size_t n) {
    if (n * sizeof(T) < (size_t{8} << 20)) ::operator delete(p);
    else std::free(p);
  }
  template <class U>
  bool operator==(const HugeAlloc<U>&) const { return true; }
};
template <class T>
using HugeVec = std::vector<T, HugeAlloc<T>>;

// Linear-probing set of edge keys with backward-shift deletion (no tombstones).
class EdgeSet {
 public:
  explicit EdgeSet(size_t expected) {
    size_t cap = 16;
    while (cap < expected * 2 + 16) cap <<= 1;
    slots_.assign(cap, kEmpty);
    mask_ = cap - 1;
  }
  bool contains(uint64_t k) const {
    for (size_t i = hash(k);; i = (i + 1) & mask_) {
      if (slots_[i] == kEmpty) return false;
      if (slots_[i] == k) return true;
    }
  }
  bool insert(uint64_t k) {
    for (size_t i = hash(k);; i = (i + 1) & mask_) {
      if (slots_[i] == kEmpty) {
        slots_[i] = k;
        ++size_;
        return true;
      }
      if (slots_[i] == k) return false;
    }
  }
  void erase(uint64_t k) {
    size_t i = hash(k);
    for (;; i = (i + 1) & mask_) {
      if (slots_[i] == kEmpty) return;
      if (slots_[i] == k) break;
    }
    size_t j = i;
    for (;;) {
      j = (j + 1) & mask_;
      if (slots_[j] == kEmpty) break;
      const size_t h = hash(slots_[j]);
      // move slots_[j] back to i if its home is not cyclically in (i, j]
      const bool in_range = (i <= j) ? (h > i && h <= j) : (h > i || h <= j);
      if (!in_range) {
        slots_[i] = slots_[j];
        i = j;
      }
    }
    slots_[i] = kEmpty;
    --size_;
  }
  size_t size() const { return size_; }
  void prefetch(uint64_t k) const { __builtin_prefetch(&slots_[hash(k)], 1); }

 private:
  static constexpr uint64_t kEmpty = ~0ull;  // never a valid (src,dst) key
  size_t hash(uint64_t k) const { return static_cast<size_t>(mix64(k)) & mask_; }
  HugeVec<uint64_t> slots_;
  size_t mask_ = 0;
  size_t size_ = 0;
};

// ref random_non_edge (src/synth.cpp:23-33): Edge e{pick(rng), pick(rng)}
// draws src then dst, retrying until the edge is new. The draws do not depend
// on the set, so a copy of the generator running kAhead attempts in front
// prefetches the hash slots the real attempts will probe (the real generator
// consumes exactly the reference's sequence).
class NonEdgeSampler {
 public:
  static constexpr int kAhead = 24;
  NonEdgeSampler(int32_t n, std::mt19937_64& rng, const EdgeSet& present, const EdgeSet* banned)
      : pick_(0, n - 1), ahead_pick_(0, n - 1), rng_(rng), ahead_(rng), present_(present),
        banned_(banned) {
    for (int i = 0; i < kAhead; ++i) advance_ahead();
  }
  uint64_t next() {
    while (true) {
      advance_ahead();
      const int32_t s = pick_(rng_);
      const int32_t d = pick_(rng_);
      if (s == d) continue;
      const uint64_t k = key_of(s, d);
      if (present_.contains(k) || (banned_ && banned_->contains(k))) continue;
      return k;
    }
  }

 private:
  void advance_ahead() {
    const int32_t s = ahead_pick_(ahead_);
    const int32_t d = ahead_pick_(ahead_);
    present_.prefetch(key_of(s, d));
  }
  std::uniform_int_distribution<int32_t> pick_, ahead_pick_;
  std::mt19937_64& rng_;
  std::mt19937_64 ahead_;
  const EdgeSet& present_;
  const EdgeSet* banned_;
};

// std::uniform_real_distribution<double>(a, b)(g) for mt19937_64, bit-exact
// with libstdc++: generate_canonical<double, 53> takes one 64-bit draw,
// u = double(x) / 2^64 (clamped below 1), and the value is u * (b - a) + a.
// The library recomputes log(range) / log(2) in long double on every call;
// this is the same arithmetic without it.
struct UniformReal {
  double a, span;
  UniformReal(double lo, double hi) : a(lo), span(hi - lo) {}
  double operator()(std::mt19937_64& g) const {
    double u = static_cast<double>(g() - std::mt19937_64::min()) * 0x1p-64;
    if (__builtin_expect(u >= 1.0, 0)) u = std::nextafter(1.0, 0.0);
    return u * span + a;
  }
};

// LSD radix sort of 64-bit keys (4 passes of 16 bits); same result as std::sort.
void radix_sort_u64(HugeVec<uint64_t>& v) {
  HugeVec<uint64_t> tmp(v.size());
  std::vector<size_t> cnt(65536);
  for (int pass = 0; pass < 4; ++pass) {
    const int sh = pass * 16;
    std::fill(cnt.begin(), cnt.end(), 0);
    for (uint64_t x : v) ++cnt[(x >> sh) & 0xffff];
    size_t s = 0;
    for (auto& c : cnt) {
      const size_t k = c;
      c = s;
      s += k;
    }
    for (uint64_t x : v) tmp[cnt[(x >> sh) & 0xffff]++] = x;
    v.swap(tmp);
  }
}

// The first `take` elements of std::shuffle(copy of src, g), without
// materialising the shuffle. libstdc++'s shuffle does, for i = 1 .. n-1,
// swap(v[i], v[r_i]) with r_i in [0, i] (drawn as above). Position i is
// untouched before step i, so a later step j > x with r_j = x writes src[j]
// into x; otherwise x last received, at its own step x, the value position
// r_x held after step x-1 — a chain over strictly smaller positions, all
// < take. So only the steps hitting positions < take (~take * ln(n / take))
// are recorded; every draw is still consumed in order.
template <class V>
std::vector<typename V::value_type> shuffled_prefix(const V& src, size_t take, std::mt19937_64& g) {
  using T = typename V::value_type;
  using uc = unsigned long;
  const size_t n = src.size();
  std::vector<T> out;
  if (n == 0) return out;
  take = std::min(take, n);
  if ((g.max() - g.min()) / uc(n) < uc(n)) {  // n > 2^32: the one-draw-per-swap path
    HugeVec<T> v(src.begin(), src.end());
    std::shuffle(v.begin(), v.end(), g);
    out.assign(v.begin(), v.begin() + take);
    return out;
  }
  std::vector<uint32_t> r_small(take);
  std::vector<std::pair<uint32_t, uint32_t>> hits;  // (position < take, step), steps ascending
  hits.reserve(static_cast<size_t>(take * (std::log(double(n) / double(take + 1)) + 2.0)) + 16);
  auto record = [&](size_t j, uc r) {
    if (j < take) r_small[j] = static_cast<uint32_t>(r);
    if (r < take) hits.emplace_back(static_cast<uint32_t>(r), static_cast<uint32_t>(j));
  };
  size_t i = 1;
  if (n % 2 == 0) {
    std::uniform_int_distribution<uc> d{0, 1};
    record(1, d(g));
    i = 2;
  }
  for (; i < n; i += 2) {
    const uc r = static_cast<uc>(i) + 1;
    const uc x = std::uniform_int_distribution<uc>{0, r * (r + 1) - 1}(g);
    record(i, x / (r + 1));
    record(i + 1, x % (r + 1));
  }
  // steps per position (counting sort, stable: ascending within a position)
  std::vector<uint32_t> start(take + 1, 0), js(hits.size());
  for (const auto& h : hits) ++start[h.first + 1];
  for (size_t x = 0; x < take; ++x) start[x + 1] += start[x];
  {
    std::vector<uint32_t> fill(start.begin(), start.end() - 1);
    for (const auto& h : hits) js[fill[h.first]++] = h.second;
  }
  auto value = [&](size_t x, size_t t) -> T {  // content of position x after steps 1..t
    while (true) {
      const auto b = js.begin() + start[x], e = js.begin() + start[x + 1];
      const auto it = std::upper_bound(b, e, static_cast<uint32_t>(t));
      if (it != b && *(it - 1) > x) return src[*(it - 1)];
      if (x == 0) return src[0];
      const size_t rx = r_small[x];
      if (rx == x) return src[x];
      t = x - 1;
      x = rx;
    }
  };
  out.resize(take);
  for (size_t q = 0; q < take; ++q) out[q] = value(q, n - 1);
  return out;
}

}  // namespace

CompactGraph synthesize_compact(const SynthParams& p) {
  check(p.num_nodes > 0, "synthesize: num_nodes must be positive");
  check(p.num_snapshots > 0, "synthesize: T must be positive");
  check(p.avg_degree >= 1.0, "synthesize: avg_degree must be >= 1");
  check(p.feature_dim > 0, "synthesize: feature_dim must be positive");
  auto ratio_ok = [](bool uni, double v) { return uni || (v >= 0.0 && v <= 1.0); };
  check(ratio_ok(p.edge_change_uniform, p.edge_change) &&
            ratio_ok(p.feature_change_uniform, p.feature_change),
        "synthesize: change ratios must lie in [0, 1]");
  std::mt19937_64 rng(derive_seed(p.seed, 0x5eed));
  const auto target = static_cast<int64_t>(std::llround(p.avg_degree * p.num_nodes));
  check(target <= static_cast<int64_t>(p.num_nodes) * (p.num_nodes - 1),
        "synthesize: avg_degree too large for a simple digraph");

  CompactGraph g;
  g.num_nodes = p.num_nodes;
  g.feature_dim = p.feature_dim;
  g.num_snapshots = p.num_snapshots;
  EdgeSet edges(static_cast<size_t>(target) + 16);
  HugeVec<uint64_t> sorted;
  sorted.reserve(target);
  {
    NonEdgeSampler sampler(p.num_nodes, rng, edges, nullptr);
    while (static_cast<int64_t>(edges.size()) < target) {
      const uint64_t k = sampler.next();
      edges.insert(k);
      sorted.push_back(k);
    }
  }
  radix_sort_u64(sorted);
  const int64_t nd = static_cast<int64_t>(p.num_nodes) * p.feature_dim;
  HugeVec<double> feats(nd);
  {
    const UniformReal unit(-1.0, 1.0);
    for (int64_t i = 0; i < nd; ++i) feats[i] = unit(rng);  // random_features, row-major
  }
  g.base_src.resize(sorted.size());
  g.base_dst.resize(sorted.size());
  for (size_t i = 0; i < sorted.size(); ++i) {
    g.base_src[i] = static_cast<int32_t>(sorted[i] >> 32);
    g.base_dst[i] = static_cast<int32_t>(sorted[i] & 0xffffffffu);
  }
  g.base_feats.assign(feats.begin(), feats.end());

  const UniformReal unit01(0.0, 1.0);
  HugeVec<uint64_t> pool;
  HugeVec<int32_t> nodes(p.num_nodes);  // the reference shuffles iota(N) each step
  std::iota(nodes.begin(), nodes.end(), 0);
  for (int32_t t = 1; t < p.num_snapshots; ++t) {
    const double edge_ratio = p.edge_change_uniform ? unit01(rng) : p.edge_change;
    const double feat_ratio = p.feature_change_uniform ? unit01(rng) : p.feature_change;
    const auto changes = static_cast<int64_t>(std::ceil(edge_ratio * static_cast<double>(edges.size())));
    const int64_t n_del = changes / 2;
    const int64_t n_ins = changes - n_del;
    // the reference shuffles a copy of the edge list and removes its first n_del
    const int64_t take = std::min<int64_t>(n_del, static_cast<int64_t>(sorted.size()));
    std::vector<uint64_t> removed = shuffled_prefix(sorted, static_cast<size_t>(take), rng);
    std::sort(removed.begin(), removed.end());
    EdgeSet banned(removed.size() + 16);
    for (uint64_t k : removed) {
      banned.insert(k);
      edges.erase(k);
    }
    std::vector<uint64_t> inserted;
    inserted.reserve(n_ins);
    if (n_ins > 0) {
      NonEdgeSampler sampler(p.num_nodes, rng, edges, &banned);
      for (int64_t i = 0; i < n_ins; ++i) {
        const uint64_t k = sampler.next();
        edges.insert(k);
        inserted.push_back(k);
      }
    }
    std::sort(inserted.begin(), inserted.end());
    const auto n_feat = static_cast<int32_t>(std::ceil(feat_ratio * static_cast<double>(p.num_nodes)));
    const std::vector<int32_t> picked = shuffled_prefix(nodes, static_cast<size_t>(n_feat), rng);
    const UniformReal unit(-1.0, 1.0);
    for (int32_t i = 0; i < n_feat; ++i) {
      double* row = feats.data() + static_cast<int64_t>(picked[i]) * p.feature_dim;
      for (int32_t j = 0; j < p.feature_dim; ++j) row[j] = unit(rng);
    }
    CompactStep s;
    for (uint64_t k : removed) {
      s.del_src.push_back(static_cast<int32_t>(k >> 32));
      s.del_dst.push_back(static_cast<int32_t>(k & 0xffffffffu));
    }
    for (uint64_t k : inserted) {
      s.ins_src.push_back(static_cast<int32_t>(k >> 32));
      s.ins_dst.push_back(static_cast<int32_t>(k & 0xffffffffu));
    }
    s.changed.assign(picked.begin(), picked.end());
    std::sort(s.changed.begin(), s.changed.end());
    s.changed_feats.resize(static_cast<size_t>(n_feat) * p.feature_dim);
    for (int32_t i = 0; i < n_feat; ++i) {
      const double* row = feats.data() + static_cast<int64_t>(s.changed[i]) * p.feature_dim;
      std::copy(row, row + p.feature_dim, s.changed_feats.begin() + static_cast<int64_t>(i) * p.feature_dim);
    }
    g.steps.push_back(std::move(s));
    // sorted edge list of snapshot t = merge((sorted \ removed), inserted), one
    // pass into the (already sized) pool buffer; removed is a sorted subset of
    // sorted and inserted is disjoint from it
    pool.resize(sorted.size() - removed.size() + inserted.size());
    {
      size_t a = 0, r = 0, b = 0, o = 0;
      const size_t na = sorted.size(), nr = removed.size(), nb = inserted.size();
      while (a < na) {
        const uint64_t x = sorted[a];
        if (r < nr && removed[r] == x) {
          ++a;
          ++r;
          continue;
        }
        while (b < nb && inserted[b] < x) pool[o++] = inserted[b++];
        pool[o++] = x;
        ++a;
      }
      while (b < nb) pool[o++] = inserted[b++];
    }
    sorted.swap(pool);
  }
  return g;
}

}  // namespace dgnn
