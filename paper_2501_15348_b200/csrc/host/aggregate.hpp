// B200 mirror of dgnn/aggregate.hpp (ref proj/include/dgnn/aggregate.hpp).
//
// Same names, argument meaning and error messages as the reference; matrices
// are fp32 device buffers, AggResult payloads live in HBM and are co-owned by
// the cache, the engine's chain register and the autograd tape through
// shared_ptr exactly like the reference's std::shared_ptr<const AggResult>.
#pragma once

#include <memory>
#include <string>

#include "../agg_kernels.h"
#include "../graph_store.h"
#include "../memory.h"

namespace dgnn {

using NodeId = int32_t;
using Timestep = int32_t;
using EdgeIdx = int64_t;

[[noreturn]] inline void fail(const std::string& msg) { throw std::invalid_argument(msg); }
inline void check(bool cond, const std::string& msg) {
  if (!cond) fail(msg);
}

// splitmix64 / derive_seed, bit-identical to ref inc/common.hpp:43-52.
inline uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
inline uint64_t derive_seed(uint64_t seed, uint64_t a, uint64_t b = 0, uint64_t c = 0) {
  return mix64(mix64(mix64(seed ^ mix64(a)) ^ mix64(b)) ^ mix64(c));
}

enum class AggrKind { kSum, kMean, kMax, kMin };
const char* to_string(AggrKind kind);
AggrKind aggr_kind_from_string(const std::string& s);

struct AggrFn {
  AggrKind kind = AggrKind::kSum;
  bool edge_weighted = false;  // unsupported on device (no model path uses it)
};

// Non-owning device view of one snapshot's adjacency (ref GraphView,
// inc/snapshot.hpp:20-35) plus the out-CSR the transposed SpMM pulls over.
struct GraphView {
  NodeId num_nodes = 0;
  EdgeIdx num_edges = 0;
  const int64_t* in_ptr = nullptr;
  const int32_t* in_src = nullptr;
  const int64_t* out_ptr = nullptr;
  const int32_t* out_dst = nullptr;
  Timestep t = 0;
  static GraphView of(const DeviceGraph& g, Timestep t);
};

// Device AggResult (ref inc/aggregate.hpp:31-47).
struct AggResult {
  cuda::DevArray<float> values;      // num_nodes x dim
  AggrKind kind = AggrKind::kSum;
  cuda::DevArray<float> degree;      // mean only
  cuda::DevArray<float> mean_sums;   // mean only
  cuda::DevArray<int32_t> argext;    // max/min only
  cuda::DevArray<float> dense;       // max/min: dense_values() cache
  Timestep t = 0;
  EdgeIdx num_edges = 0;
  int incremental_depth = 0;
  NodeId rows = 0;
  int32_t dim = 0;

  double size_units() const { return static_cast<double>(rows) * dim; }
  bool extremal() const { return kind == AggrKind::kMax || kind == AggrKind::kMin; }
  // values with max/min empty-row sentinels replaced by zero (device pointer).
  const float* dense_values() const { return extremal() ? dense.get() : values.get(); }
};
using AggPtr = std::shared_ptr<const AggResult>;

struct IncrementalOptions {
  double fallback_threshold = 0.5;
  int rescratch_period = 64;
};

enum class FallbackReason { kNone, kChangeRatio, kDeletedContributor, kRescratchPeriod };

struct IncrementalResult {
  std::shared_ptr<AggResult> result;
  bool used_fallback = false;
  FallbackReason reason = FallbackReason::kNone;
};

// (|deletions| + |insertions|) / (2 |E(base)|); +inf when base has no edges.
double change_ratio(const DevDelta& delta, EdgeIdx base_edges);

// values[v] = fn over {feats[u] : edge u->v} (ref src/aggregate.cpp:55-115).
std::shared_ptr<AggResult> aggregate_scratch(const GraphView& graph, const float* feats,
                                             int32_t dim, const AggrFn& fn, cudaStream_t stream);

// Agg_{G_t}(H) from base = Agg_{G_{t-1}}(H) of the SAME matrix H: a copy
// plus the structural part of delta t (removed edges subtract H[src], added
// edges add it). Same values as aggregate_scratch(graph, H) up to fp32
// summation order. Sum / mean only; graph must be the full snapshot t.
// Whether aggregate_rebase handles (fn, dim, feats); otherwise aggregate from
// scratch.
bool rebase_supported(const AggrFn& fn, int32_t dim, const float* feats);
std::shared_ptr<AggResult> aggregate_rebase(const AggResult& base, const GraphView& graph,
                                            const float* feats, int32_t dim, const DevDelta& delta,
                                            const AggrFn& fn, cudaStream_t stream);

// aggregate_scratch of an all-zero feature matrix under sum: zero values
// without the SpMM (a GraphRNN's initial hidden state); false = not handled.
std::shared_ptr<AggResult> aggregate_zero_sum(const GraphView& graph, int32_t dim, cudaStream_t stream);

// Eq. 2 incremental update from prev (ref src/aggregate.cpp:117-207): the
// new result is out of place (prev stays valid for its co-owners).
IncrementalResult aggregate_incremental(const AggResult& prev, const GraphView& prev_graph,
                                        const GraphView& curr_graph, const float* prev_feats,
                                        const float* curr_feats, const DevDelta& delta,
                                        Timestep delta_t, const AggrFn& fn,
                                        const IncrementalOptions& opts, cudaStream_t stream);

// grad (num_nodes x dim, caller-allocated) = scatter of upstream to sources
// (ref src/aggregate.cpp:209-246).
void aggregate_backward(const GraphView& graph, const float* upstream, int32_t dim,
                        const AggrFn& fn, const AggResult& forward, float* grad,
                        cudaStream_t stream, const float* addend = nullptr);

// grad[u] += sum over the structural part of delta t (source-grouped,
// DevDelta::rows_t) of +-upstream[v], in place: turns A_{t-1}^T upstream into
// A_t^T upstream (sum aggregation over full snapshots). Returns false, doing
// nothing, when the shape is unsupported.
bool aggregate_backward_delta(const DevDelta& delta, int32_t num_nodes, const float* upstream,
                              int32_t dim, float* grad, cudaStream_t stream);

// Per-kernel-class device timing (bench.py roofline): when enabled, the
// wrappers bracket kernels with CUDA events and accumulate durations and
// algorithmic bytes per class.
enum ProfClass { kProfAggScratch = 0, kProfAggDelta = 1, kProfAggBackward = 2, kProfCellFwd = 3,
                 kProfCellBwd = 4, kProfWeightGrad = 5, kProfOther = 6, kProfCellBwdGemm = 7,
                 kProfAggRebase = 8,   // hidden aggregation rebased across a structural delta
                 kProfSample = 9,      // one whole (window, batch) sample, first to last op
                 kProfSampleHost = 10, // host time to issue one sample (no events)
                 kProfHostBuild = 11, kProfHostFwd = 12, kProfHostBwd = 13,  // its phases
                 kProfHostAlloc = 14,  // host time inside device allocations
                 kProfCount = 15 };
struct ProfStat {
  int64_t launches = 0;
  double ms = 0.0;
  double bytes = 0.0;
  double flops = 0.0;
  double max_ms = 0.0;
};
void prof_enable(bool on);
bool prof_enabled();
void prof_reset();
void prof_flush();  // resolves pending events (synchronises them)
ProfStat prof_get(int cls);
void prof_add_host(int cls, double ms);  // a host-timed scope
class ProfScope {
 public:
  ProfScope(int cls, cudaStream_t s, double bytes, double flops = 0.0);
  ~ProfScope();

 private:
  int cls_;
  cudaStream_t s_;
  double bytes_, flops_;
  cudaEvent_t a_ = nullptr, b_ = nullptr;
};

}  // namespace dgnn
