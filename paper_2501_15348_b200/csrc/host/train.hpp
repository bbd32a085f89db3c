// B200 mirror of dgnn/train.hpp and the consecutive-block part of
// dgnn/distsim.hpp (ref proj/include/dgnn/{train,distsim}.hpp).
#pragma once

#include <memory>
#include <optional>
#include <utility>
#include <vector>

#include "comm.hpp"
#include "model.hpp"

namespace dgnn {

enum class IterationOrder { kSeqFirst, kNodeFirst };
enum class OptimizerKind { kSgd, kAdam };

struct TrainConfig {
  int batch_size = 0;
  int epochs = 1;
  double lr = 0.01;
  OptimizerKind optimizer = OptimizerKind::kAdam;
  double beta1 = 0.9;
  double beta2 = 0.999;
  double adam_eps = 1e-8;
  IterationOrder iteration = IterationOrder::kSeqFirst;
  Timestep stride = 1;
  uint64_t seed = 1;
  double fallback_threshold = 0.5;
  int rescratch_period = 64;
  bool incremental = true;
  std::optional<CachePolicy> cache_policy = CachePolicy::kReinc;
  double cache_capacity_frac = 1.0;
  int64_t hbm_cache_budget_bytes = 0;  // B200: 0 = all cached payloads stay in HBM
};

struct EpochReport {
  std::vector<double> sample_losses;
  double loss = 0.0;
  double mae = 0.0;
  CacheStats cache;
  int64_t kernel_invocations = 0;
  int64_t scratch_calls = 0;
  int64_t incremental_calls = 0;
  int64_t fallbacks = 0;
  int64_t skipped_steps = 0;
  double seconds = 0.0;  // device-timed (CUDA events around the epoch)
  std::vector<std::pair<int64_t, int64_t>> visitation;
};

struct OptimizerState {
  cuda::DevArray<float> m, v;
  int64_t step_count = 0;
};

std::vector<std::pair<NodeId, NodeId>> make_batches(NodeId num_nodes, int batch_size, uint64_t seed,
                                                    int64_t epoch_index);
double cache_data_size_units(const DeviceGraph& graph, const ModelConfig& mcfg);

// One parameter update from `grads` * gscale (flat, device). Non-finite
// gradients skip the step; an applied step refreshes the packed weights and
// invalidates weight-dependent cache entries (ref src/train.cpp:26-52).
bool optimizer_step(DgnnModel& model, const float* grads, float gscale, OptimizerState& state,
                    const TrainConfig& cfg, CacheStore* store, cudaStream_t stream);

// Per-GPU execution resources: cache store, provider, scratch buffers.
class Worker {
 public:
  Worker(const DeviceGraph& graph, DgnnModel& model, const TrainConfig& cfg, cudaStream_t stream);
  ~Worker();
  AggProvider& provider() { return *provider_; }
  CacheStore* store() { return store_.get(); }
  DgnnModel& model() { return model_; }
  const DeviceGraph& graph() const { return graph_; }
  cudaStream_t stream() const { return stream_; }
  // forward + loss + backward; grads accumulated into `grad`, loss added to *loss_slot.
  void run_sample(const SequenceWindow& window, Timestep windows_remaining, int64_t batch_id,
                  std::pair<NodeId, NodeId> node_range, float* grad, double* loss_slot);

 private:
  const DeviceGraph& graph_;
  DgnnModel& model_;
  TrainConfig cfg_;
  cudaStream_t stream_;
  cudaStream_t aux_ = nullptr;  // second layer lane (null: single-stream)
  std::unique_ptr<CacheStore> store_;
  std::unique_ptr<AggProvider> provider_;
  cuda::DevArray<double> loss_ws_;
};

// Outer loop over node mini-batches, inner loop over all windows; one
// optimizer step per sample (ref src/train.cpp:146-210).
EpochReport seq_first_epoch(DgnnModel& model, const DeviceGraph& graph,
                            const std::vector<SequenceWindow>& windows, const TrainConfig& cfg,
                            Worker& worker, OptimizerState& opt, int64_t epoch_index);
// node-first order (ref src/train.cpp:216-220): window outer, batch inner.
EpochReport node_first_epoch(DgnnModel& model, const DeviceGraph& graph,
                             const std::vector<SequenceWindow>& windows, const TrainConfig& cfg,
                             Worker& worker, OptimizerState& opt, int64_t epoch_index);

class TrainSession {
 public:
  // windows = sliding_windows(window_total, L, S, H); window_total <= 0 means
  // graph.length() - 1, the executable set.
  TrainSession(const DeviceGraph& graph, const ModelConfig& mcfg, const TrainConfig& tcfg,
               cudaStream_t stream, Timestep window_total = 0);
  EpochReport run_epoch();
  DgnnModel& model() { return *model_; }
  Worker& worker() { return *worker_; }
  const std::vector<SequenceWindow>& windows() const { return windows_; }
  OptimizerState& opt() { return opt_; }

 private:
  const DeviceGraph& graph_;
  TrainConfig tcfg_;
  std::unique_ptr<DgnnModel> model_;
  std::unique_ptr<Worker> worker_;
  std::vector<SequenceWindow> windows_;
  OptimizerState opt_;
  int64_t epoch_index_ = 0;
};

// Consecutive-block placement (ref src/distsim.cpp:35-81).
struct WorkerAssignment {
  Timestep block_begin = 0, block_end = 0;
  int64_t window_begin = 0, window_end = 0;
};
std::vector<WorkerAssignment> plan_consecutive_block(Timestep total, int num_workers,
                                                     Timestep seq_len, Timestep stride,
                                                     Timestep horizon);

// Communication ledger of one distributed epoch (ref CommVolume / CommLedger,
// inc/distsim.hpp:58-80; accounting src/distsim.cpp:101-182 and the per-step
// ring all-reduce volume, :262-268). Byte counts follow the reference's fp64
// storage (8 B per value), so they compare placements the way Table 1 does.
enum class PlacementScheme { kConsecutiveBlock, kNodePartition, kSequencePartition };
enum class OverlapMode { kReplicateOverlap, kRemoteFetch };
struct CommVolume {
  uint64_t remote_features = 0, intermediate_redistribution = 0, gradient_sync = 0,
           snapshot_fetch = 0;
};
struct CommLedger {
  CommVolume total;
  std::vector<CommVolume> per_worker;
};
CommLedger comm_ledger(const DeviceGraph& graph, PlacementScheme scheme, OverlapMode overlap,
                       int num_workers, Timestep seq_len, Timestep stride, Timestep horizon,
                       int hidden_dim, int64_t num_params, int64_t num_batches, cudaStream_t stream);

// One rank of the snapshot-window-sharded trainer (distsim semantics, ref
// src/distsim.cpp:197-272): per batch every rank sums the gradients of its
// own window block in window order; the caller all-reduces the flat buffer
// (NCCL) and every rank applies the identical step with gscale = 1/W.
class DistWorker {
 public:
  DistWorker(const DeviceGraph& graph, const ModelConfig& mcfg, const TrainConfig& tcfg,
             cudaStream_t stream, int rank, int world, Timestep window_total = 0);
  int64_t num_batches() const { return static_cast<int64_t>(batches_.size()); }
  int64_t total_windows() const { return static_cast<int64_t>(windows_.size()); }
  const WorkerAssignment& assignment() const { return assign_; }
  void begin_epoch();
  // grad_sum (flat, device) = sum over local windows of batch b of window grads.
  void local_grads(int64_t b, float* grad_sum);
  // applies the (all-reduced) gradient sum; returns false if skipped.
  bool apply(const float* grad_sum);
  void end_epoch();
  DgnnModel& model() { return *model_; }
  Worker& worker() { return *worker_; }
  OptimizerState& opt() { return opt_; }
  std::vector<double> take_losses();  // per local sample of the epoch (visit order)
  // The whole epoch natively (ref run_distributed_epoch, src/distsim.cpp:
  // 197-272): per batch local_grads -> NCCL sum over ranks (comm null: this
  // rank alone) -> apply. Device-timed with CUDA events; `seconds` is the max
  // over ranks. Sample losses via take_losses().
  struct EpochResult {
    int64_t batches = 0, skipped = 0;
    double seconds = 0.0;
  };
  EpochResult run_epoch(NcclComm* comm);
  int64_t epoch_index() const { return epoch_index_; }

 private:
  const DeviceGraph& graph_;
  TrainConfig tcfg_;
  std::unique_ptr<DgnnModel> model_;
  std::unique_ptr<Worker> worker_;
  std::vector<SequenceWindow> windows_;
  WorkerAssignment assign_;
  OptimizerState opt_;
  std::vector<std::pair<NodeId, NodeId>> batches_;
  int64_t epoch_index_ = 0;
  cuda::DevArray<float> grad_w_, grad_sum_;
  cuda::DevArray<double> losses_;
  int64_t n_loss_ = 0;
};

}  // namespace dgnn
