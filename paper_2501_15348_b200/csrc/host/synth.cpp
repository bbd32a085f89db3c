// Bit-exact streaming synthesize (see synth.hpp).
#include "synth.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <random>
#include <stdexcept>
#include <type_traits>

#include "aggregate.hpp"

namespace dgnn {
namespace {

inline uint64_t key_of(int32_t s, int32_t d) {
  return (static_cast<uint64_t>(static_cast<uint32_t>(s)) << 32) | static_cast<uint32_t>(d);
}

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
  std::vector<uint64_t> slots_;
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

// std::shuffle, bit-exact with libstdc++'s algorithm (stl_algo.h: for a range
// n with n*n <= the generator range, positions for two successive elements
// come from one draw, x in [0, b0*b1) -> (x / b1, x % b1); for even n the
// first swap is drawn alone from {0, 1}). The positions of a block of swaps
// are drawn first and the swaps then applied in order with the random slots
// prefetched — same draws, same swap order, a fraction of the miss latency.
template <class T>
void shuffle_exact(std::vector<T>& v, std::mt19937_64& g) {
#if defined(__GLIBCXX__)
  using uc = unsigned long;
  static_assert(std::is_same_v<std::mt19937_64::result_type, uc>, "generator width");
  const size_t n = v.size();
  if (n == 0) return;
  const uc urngrange = g.max() - g.min();
  const uc urange = n;
  if (urngrange / urange < urange) {
    std::shuffle(v.begin(), v.end(), g);
    return;
  }
  size_t i = 1;
  if (urange % 2 == 0) {
    std::uniform_int_distribution<uc> d{0, 1};
    std::swap(v[i], v[d(g)]);
    ++i;
  }
  constexpr size_t kBlock = 8192, kDist = 32;
  static thread_local std::vector<uc> pos(kBlock);
  while (i < n) {
    size_t cnt = 0;
    for (size_t j = i; j < n && cnt < kBlock; j += 2) {
      const uc r = static_cast<uc>(j) + 1;  // swap range of element j: [0, j]
      const uc x = std::uniform_int_distribution<uc>{0, r * (r + 1) - 1}(g);
      pos[cnt++] = x / (r + 1);
      pos[cnt++] = x % (r + 1);
    }
    for (size_t k = 0; k < cnt; ++k) {
      if (k + kDist < cnt) __builtin_prefetch(&v[pos[k + kDist]], 1);
      std::swap(v[i + k], v[pos[k]]);
    }
    i += cnt;
  }
#else
  std::shuffle(v.begin(), v.end(), g);
#endif
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
  std::vector<uint64_t> sorted;
  sorted.reserve(target);
  {
    NonEdgeSampler sampler(p.num_nodes, rng, edges, nullptr);
    while (static_cast<int64_t>(edges.size()) < target) {
      const uint64_t k = sampler.next();
      edges.insert(k);
      sorted.push_back(k);
    }
  }
  std::sort(sorted.begin(), sorted.end());
  const int64_t nd = static_cast<int64_t>(p.num_nodes) * p.feature_dim;
  std::vector<double> feats(nd);
  {
    std::uniform_real_distribution<double> unit(-1.0, 1.0);
    for (int64_t i = 0; i < nd; ++i) feats[i] = unit(rng);  // random_features, row-major
  }
  g.base_src.resize(sorted.size());
  g.base_dst.resize(sorted.size());
  for (size_t i = 0; i < sorted.size(); ++i) {
    g.base_src[i] = static_cast<int32_t>(sorted[i] >> 32);
    g.base_dst[i] = static_cast<int32_t>(sorted[i] & 0xffffffffu);
  }
  g.base_feats.assign(feats.begin(), feats.end());

  std::uniform_real_distribution<double> unit01(0.0, 1.0);
  std::vector<uint64_t> pool;
  std::vector<int32_t> nodes(p.num_nodes);
  for (int32_t t = 1; t < p.num_snapshots; ++t) {
    const double edge_ratio = p.edge_change_uniform ? unit01(rng) : p.edge_change;
    const double feat_ratio = p.feature_change_uniform ? unit01(rng) : p.feature_change;
    const auto changes = static_cast<int64_t>(std::ceil(edge_ratio * static_cast<double>(edges.size())));
    const int64_t n_del = changes / 2;
    const int64_t n_ins = changes - n_del;
    pool = sorted;
    shuffle_exact(pool, rng);
    const int64_t take = std::min<int64_t>(n_del, static_cast<int64_t>(pool.size()));
    std::vector<uint64_t> removed(pool.begin(), pool.begin() + take);
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
    std::iota(nodes.begin(), nodes.end(), 0);
    shuffle_exact(nodes, rng);
    std::uniform_real_distribution<double> unit(-1.0, 1.0);
    for (int32_t i = 0; i < n_feat; ++i) {
      double* row = feats.data() + static_cast<int64_t>(nodes[i]) * p.feature_dim;
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
    s.changed.assign(nodes.begin(), nodes.begin() + n_feat);
    std::sort(s.changed.begin(), s.changed.end());
    s.changed_feats.resize(static_cast<size_t>(n_feat) * p.feature_dim);
    for (int32_t i = 0; i < n_feat; ++i) {
      const double* row = feats.data() + static_cast<int64_t>(s.changed[i]) * p.feature_dim;
      std::copy(row, row + p.feature_dim, s.changed_feats.begin() + static_cast<int64_t>(i) * p.feature_dim);
    }
    g.steps.push_back(std::move(s));
    // sorted edge list of snapshot t = merge((sorted \ removed), inserted)
    std::vector<uint64_t> kept;
    kept.reserve(sorted.size());
    std::set_difference(sorted.begin(), sorted.end(), removed.begin(), removed.end(),
                        std::back_inserter(kept));
    sorted.clear();
    std::merge(kept.begin(), kept.end(), inserted.begin(), inserted.end(), std::back_inserter(sorted));
  }
  return g;
}

}  // namespace dgnn
