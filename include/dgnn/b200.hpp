// dgnn/b200.hpp — C++ face of the B200 library in the reference's own
// vocabulary (namespace dgnn; ref proj/include/dgnn/{snapshot,synth,model,
// train,distsim}.hpp), header-only over the C ABI in dgnn_b200.h. A caller of
// the reference's TrainSession / DistSession / synthesize / sliding_windows /
// plan switches by including this header and linking _dgnn_b200.so; the
// types keep the reference's names and field meanings, failures throw
// std::invalid_argument / std::out_of_range with the reference's messages
// (ref inc/common.hpp:36-40) and std::runtime_error for CUDA / NCCL errors.
//
// Differences a caller sees: graphs live in HBM (DynamicGraph is built from
// host edge lists and deltas, not from dgnn::Snapshot objects), matrices are
// fp32 on the device, and the distributed trainer is one process per GPU
// (DistSession takes this process's rank and an NCCL communicator) instead
// of the reference's sequentially interleaved workers.
#ifndef DGNN_B200_HPP
#define DGNN_B200_HPP

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../dgnn_b200.h"

namespace dgnn {

namespace detail {
inline void check_status(int rc) {
  if (rc == 0) return;
  const std::string msg = dgnn_last_error();
  if (rc == 1) throw std::invalid_argument(msg);
  if (rc == 2) throw std::out_of_range(msg);
  throw std::runtime_error(msg);
}
}  // namespace detail

using NodeId = int32_t;
using Timestep = int32_t;

// ref inc/model.hpp:21
enum class Architecture { kGcrnM1 = 0, kCdGcn = 1, kGcrnM2 = 2, kTgcn = 3 };
// ref inc/aggregate.hpp:21
enum class AggrKind { kSum = 0, kMean = 1, kMax = 2, kMin = 3 };
// ref inc/cache.hpp (CachePolicy); nullopt in the reference = no cache
enum class CachePolicy { kNone = -1, kReinc = 0, kLru = 1, kLfu = 2 };
// ref inc/train.hpp:17-18
enum class IterationOrder { kSeqFirst = 0, kNodeFirst = 1 };
enum class OptimizerKind { kSgd = 0, kAdam = 1 };

// ref inc/model.hpp:28-40 (defaults as the reference's)
struct ModelConfig {
  Architecture arch = Architecture::kGcrnM2;
  int layers = 2;
  int hidden_dim = 64;
  Timestep seq_len = 8;
  Timestep horizon = 1;
  bool teacher_forcing = true;
  AggrKind aggregation = AggrKind::kSum;
  std::vector<int32_t> fanouts;  // empty or all -1: whole snapshots
};

// ref inc/train.hpp:20-40
struct TrainConfig {
  int batch_size = 0;
  int epochs = 1;
  double lr = 0.01;
  OptimizerKind optimizer = OptimizerKind::kAdam;
  IterationOrder iteration = IterationOrder::kSeqFirst;
  Timestep stride = 1;
  uint64_t seed = 1;
  double fallback_threshold = 0.5;
  int rescratch_period = 64;
  bool incremental = true;
  CachePolicy cache_policy = CachePolicy::kReinc;
  double cache_capacity_frac = 1.0;
  int64_t hbm_cache_budget_bytes = 0;  // B200: second cache level (0 = HBM only)
};

// ref inc/train.hpp:42-58 (seconds are device-timed)
struct EpochReport {
  std::vector<double> sample_losses;
  double loss = 0.0;
  double seconds = 0.0;
  int64_t hits = 0, misses = 0, evictions = 0, expirations = 0, invalidations = 0, rejected = 0;
  int64_t scratch_calls = 0, incremental_calls = 0, fallbacks = 0, skipped_steps = 0;
  int64_t spills = 0, refills = 0;
};

// ref inc/windows.hpp / src/windows.cpp:5-15
struct SequenceWindow {
  Timestep start = 0, length = 0, stride = 1, horizon = 0;
};
inline std::vector<SequenceWindow> sliding_windows(Timestep total, Timestep seq_len, Timestep stride,
                                                   Timestep horizon) {
  const int64_t n = dgnn_sliding_windows(total, seq_len, stride, horizon, nullptr, 0);
  std::vector<int32_t> starts(static_cast<size_t>(n));
  dgnn_sliding_windows(total, seq_len, stride, horizon, starts.data(), n);
  std::vector<SequenceWindow> out;
  for (int32_t s : starts) out.push_back({s, seq_len, stride, horizon});
  return out;
}

// ref inc/distsim.hpp:32-54, consecutive_block
struct WorkerAssignment {
  Timestep block_begin = 0, block_end = 0;
  int64_t window_begin = 0, window_end = 0;
};
inline std::vector<WorkerAssignment> plan(Timestep total, int num_workers, Timestep seq_len,
                                          Timestep stride, Timestep horizon) {
  std::vector<int64_t> raw(4 * static_cast<size_t>(num_workers));
  detail::check_status(dgnn_plan(total, num_workers, seq_len, stride, horizon, raw.data()));
  std::vector<WorkerAssignment> out(static_cast<size_t>(num_workers));
  for (int m = 0; m < num_workers; ++m)
    out[m] = {static_cast<Timestep>(raw[4 * m]), static_cast<Timestep>(raw[4 * m + 1]), raw[4 * m + 2],
              raw[4 * m + 3]};
  return out;
}

// A dynamic graph resident in HBM (ref DynamicGraph, inc/snapshot.hpp:95-110).
class DynamicGraph {
 public:
  DynamicGraph(NodeId num_nodes, int32_t feature_dim, void* stream = nullptr) {
    detail::check_status(dgnn_graph_create(num_nodes, feature_dim, stream, &g_));
  }
  explicit DynamicGraph(dgnn_graph* adopt) : g_(adopt) {}
  ~DynamicGraph() { dgnn_graph_free(g_); }
  DynamicGraph(const DynamicGraph&) = delete;
  DynamicGraph& operator=(const DynamicGraph&) = delete;
  DynamicGraph(DynamicGraph&& o) noexcept : g_(std::exchange(o.g_, nullptr)) {}

  // Snapshot ctor (src/snapshot.cpp:20-69): host edge list + features
  void add_snapshot(const std::vector<std::pair<NodeId, NodeId>>& edges, const std::vector<float>& feats) {
    std::vector<int32_t> s, d;
    split(edges, s, d);
    detail::check_status(dgnn_graph_add_snapshot(g_, s.data(), d.data(), static_cast<int64_t>(s.size()),
                                                 feats.data()));
  }
  // apply_delta (src/snapshot.cpp:142-154)
  void add_delta(const std::vector<std::pair<NodeId, NodeId>>& deletions,
                 const std::vector<std::pair<NodeId, NodeId>>& insertions,
                 const std::vector<NodeId>& changed_nodes, const std::vector<float>& changed_feats) {
    std::vector<int32_t> ds, dd, is, id;
    split(deletions, ds, dd);
    split(insertions, is, id);
    detail::check_status(dgnn_graph_add_delta(g_, ds.data(), dd.data(), static_cast<int64_t>(ds.size()),
                                              is.data(), id.data(), static_cast<int64_t>(is.size()),
                                              changed_nodes.data(),
                                              static_cast<int64_t>(changed_nodes.size()),
                                              changed_feats.data()));
  }
  Timestep length() const { return dgnn_graph_length(g_); }
  int64_t num_edges(Timestep t) const { return dgnn_graph_num_edges(g_, t); }
  double change_ratio(Timestep t) const { return dgnn_graph_change_ratio(g_, t); }
  dgnn_graph* handle() const { return g_; }

 private:
  static void split(const std::vector<std::pair<NodeId, NodeId>>& e, std::vector<int32_t>& s,
                    std::vector<int32_t>& d) {
    s.reserve(e.size());
    d.reserve(e.size());
    for (const auto& p : e) {
      s.push_back(p.first);
      d.push_back(p.second);
    }
  }
  dgnn_graph* g_ = nullptr;
};

// synthesize (ref inc/synth.hpp:25-39, src/synth.cpp:36-91): bit-exact
// generator, built straight into the device graph store.
struct SynthParams {
  NodeId num_nodes = 1000;
  double avg_degree = 8.0;
  int32_t feature_dim = 16;
  Timestep num_snapshots = 10;
  double edge_change_rate = 0.01;
  double feature_change_rate = 0.01;
  uint64_t seed = 1;
};
inline DynamicGraph synthesize(const SynthParams& p, void* stream = nullptr) {
  dgnn_synth* s = nullptr;
  detail::check_status(dgnn_synth_create(p.num_nodes, p.avg_degree, p.feature_dim, p.num_snapshots,
                                         p.edge_change_rate, p.feature_change_rate, p.seed, &s));
  dgnn_graph* g = nullptr;
  const int rc = dgnn_synth_to_graph(s, stream, &g);
  dgnn_synth_free(s);
  detail::check_status(rc);
  return DynamicGraph(g);
}

namespace detail {
inline dgnn_run_cfg run_cfg(const ModelConfig& m, const TrainConfig& t, int workers) {
  dgnn_run_cfg c{};
  c.arch = static_cast<int32_t>(m.arch);
  c.layers = m.layers;
  c.hidden = m.hidden_dim;
  c.seq_len = m.seq_len;
  c.horizon = m.horizon;
  c.teacher_forcing = m.teacher_forcing ? 1 : 0;
  c.aggr = static_cast<int32_t>(m.aggregation);
  c.batch_size = t.batch_size;
  c.seed = t.seed;
  c.lr = t.lr;
  c.optimizer = static_cast<int32_t>(t.optimizer);
  c.stride = t.stride;
  c.fallback_threshold = t.fallback_threshold;
  c.rescratch_period = t.rescratch_period;
  c.incremental = t.incremental ? 1 : 0;
  c.cache_policy = static_cast<int32_t>(t.cache_policy);
  c.cache_frac = t.cache_capacity_frac;
  c.workers = workers;
  c.epochs = t.epochs;
  c.hbm_cache_budget_bytes = t.hbm_cache_budget_bytes;
  c.n_fanouts = static_cast<int32_t>(m.fanouts.size());
  for (size_t i = 0; i < m.fanouts.size() && i < 8; ++i) c.fanouts[i] = m.fanouts[i];
  c.iteration = static_cast<int32_t>(t.iteration);
  return c;
}
inline EpochReport report(dgnn_session* s, const dgnn_epoch_report& r) {
  EpochReport e;
  e.loss = r.loss;
  e.seconds = r.seconds;
  e.hits = r.hits;
  e.misses = r.misses;
  e.evictions = r.evictions;
  e.expirations = r.expirations;
  e.invalidations = r.invalidations;
  e.rejected = r.rejected;
  e.scratch_calls = r.scratch_calls;
  e.incremental_calls = r.incremental_calls;
  e.fallbacks = r.fallbacks;
  e.skipped_steps = r.skipped_steps;
  e.spills = r.spills;
  e.refills = r.refills;
  int64_t n = 0;
  check_status(dgnn_session_losses(s, nullptr, &n));
  e.sample_losses.resize(static_cast<size_t>(n));
  check_status(dgnn_session_losses(s, e.sample_losses.data(), &n));
  return e;
}
}  // namespace detail

class SessionBase {
 public:
  SessionBase(const SessionBase&) = delete;
  SessionBase& operator=(const SessionBase&) = delete;
  ~SessionBase() { dgnn_session_free(s_); }
  int64_t num_params() const { return dgnn_session_num_params(s_); }
  // DgnnModel::flatten_params / unflatten_params (src/model.cpp:91-107), fp64
  std::vector<double> flatten_params() const {
    std::vector<double> p(static_cast<size_t>(num_params()));
    detail::check_status(dgnn_session_get_params(s_, p.data()));
    return p;
  }
  void unflatten_params(const std::vector<double>& p) {
    detail::check_status(dgnn_session_set_params(s_, p.data()));
  }
  dgnn_session* handle() const { return s_; }

 protected:
  SessionBase(const DynamicGraph& g, const dgnn_run_cfg& c, int rank, void* stream) {
    detail::check_status(dgnn_session_create(g.handle(), &c, rank, stream, &s_));
  }
  dgnn_session* s_ = nullptr;
};

// ref TrainSession (inc/train.hpp:92-114): seq-first epochs on one GPU.
class TrainSession : public SessionBase {
 public:
  TrainSession(const DynamicGraph& graph, const ModelConfig& mcfg, const TrainConfig& tcfg,
               void* stream = nullptr)
      : SessionBase(graph, detail::run_cfg(mcfg, tcfg, 0), 0, stream), epochs_(tcfg.epochs) {}
  EpochReport run_epoch() {
    dgnn_epoch_report r{};
    detail::check_status(dgnn_session_run_epoch(s_, &r));
    return detail::report(s_, r);
  }
  std::vector<EpochReport> run() {
    std::vector<EpochReport> out;
    for (int e = 0; e < epochs_; ++e) out.push_back(run_epoch());
    return out;
  }

 private:
  int epochs_;
};

// The NCCL gradient all-reduce of the sharded trainer (one per process).
class Communicator {
 public:
  static std::vector<uint8_t> unique_id() {
    std::vector<uint8_t> id(128);
    detail::check_status(dgnn_comm_unique_id(id.data()));
    return id;
  }
  Communicator(const std::vector<uint8_t>& id, int world, int rank) : world_(world), rank_(rank) {
    if (id.size() != 128) throw std::invalid_argument("communicator id must be 128 bytes");
    detail::check_status(dgnn_comm_create(id.data(), world, rank, &c_));
  }
  ~Communicator() { dgnn_comm_free(c_); }
  Communicator(const Communicator&) = delete;
  Communicator& operator=(const Communicator&) = delete;
  void allreduce_sum(float* device_data, int64_t n, void* stream = nullptr) {
    detail::check_status(dgnn_grad_allreduce(c_, device_data, n, stream));
  }
  int world() const { return world_; }
  int rank() const { return rank_; }
  dgnn_comm* handle() const { return c_; }

 private:
  dgnn_comm* c_ = nullptr;
  int world_, rank_;
};

// ref DistSession (inc/distsim.hpp:82-102) under consecutive_block /
// replicate_overlap, one rank per process: run_epoch() is this rank's part of
// run_distributed_epoch (src/distsim.cpp:186-281) — per batch its window
// block's gradient sum, the NCCL sum over ranks, one identical Adam / SGD step
// on every rank (normalised by the global window count).
class DistSession : public SessionBase {
 public:
  DistSession(const DynamicGraph& graph, const ModelConfig& mcfg, const TrainConfig& tcfg, int world,
              int rank, Communicator* comm, void* stream = nullptr)
      : SessionBase(graph, detail::run_cfg(mcfg, tcfg, world), rank, stream), comm_(comm) {}
  EpochReport run_epoch() {
    dgnn_epoch_report r{};
    detail::check_status(dgnn_session_run_dist_epoch(s_, comm_ ? comm_->handle() : nullptr, &r));
    return detail::report(s_, r);
  }
  // [window_begin, window_end) of this rank and the global window count
  std::pair<int64_t, int64_t> local_windows(int64_t* total = nullptr) const {
    int64_t t = 0, b = 0, e = 0;
    detail::check_status(dgnn_session_num_windows(s_, &t, &b, &e));
    if (total) *total = t;
    return {b, e};
  }

 private:
  Communicator* comm_;
};

}  // namespace dgnn

#endif  // DGNN_B200_HPP
