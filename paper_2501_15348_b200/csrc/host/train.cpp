// Trainers: seq-first (ref src/train.cpp) and consecutive-block sharded
// (ref src/distsim.cpp) over the device model.
#include "train.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <random>

namespace dgnn {

std::vector<std::pair<NodeId, NodeId>> make_batches(NodeId num_nodes, int batch_size, uint64_t seed,
                                                    int64_t epoch_index) {
  if (batch_size <= 0 || batch_size >= num_nodes) return {{0, num_nodes}};
  std::vector<std::pair<NodeId, NodeId>> ranges;
  for (NodeId begin = 0; begin < num_nodes; begin += batch_size) {
    ranges.push_back({begin, std::min<NodeId>(begin + batch_size, num_nodes)});
  }
  std::mt19937_64 rng(derive_seed(seed, 0xba7c4, static_cast<uint64_t>(epoch_index)));
  std::shuffle(ranges.begin(), ranges.end(), rng);
  return ranges;
}

double cache_data_size_units(const DeviceGraph& graph, const ModelConfig& mcfg) {
  return 2.0 * static_cast<double>(mcfg.seq_len) * static_cast<double>(graph.num_nodes()) *
         static_cast<double>(graph.feature_dim());
}

bool optimizer_step(DgnnModel& model, const float* grads, float gscale, OptimizerState& state,
                    const TrainConfig& cfg, CacheStore* store, cudaStream_t stream) {
  const int64_t P = model.num_params();
  cuda::DevArray<int32_t> flag(1, stream);
  flag.zero(stream);
  cuda::nonfinite_check(P, grads, flag.get(), stream);
  int32_t bad = 0;
  copy_to_host(&bad, flag.get(), sizeof(bad), stream);
  if (bad) return false;
  state.step_count += 1;
  if (!state.m) {
    state.m = cuda::DevArray<float>(P, stream);
    state.v = cuda::DevArray<float>(P, stream);
    state.m.zero(stream);
    state.v.zero(stream);
  }
  const double bc1 = 1.0 - std::pow(cfg.beta1, static_cast<double>(state.step_count));
  const double bc2 = 1.0 - std::pow(cfg.beta2, static_cast<double>(state.step_count));
  {
    ProfScope ps(kProfOther, stream, 4.0 * P * 5);
    cuda::adam_step(P, model.params(), state.m.get(), state.v.get(), grads, gscale,
                    static_cast<float>(cfg.lr), static_cast<float>(cfg.beta1),
                    static_cast<float>(cfg.beta2), static_cast<float>(cfg.adam_eps),
                    static_cast<float>(bc1), static_cast<float>(bc2),
                    cfg.optimizer == OptimizerKind::kSgd, nullptr, stream);
  }
  model.refresh_packed();
  if (store != nullptr) store->bump_epoch();
  return true;
}

// ---------------------------------------------------------------- Worker
Worker::Worker(const DeviceGraph& graph, DgnnModel& model, const TrainConfig& cfg, cudaStream_t stream)
    : graph_(graph), model_(model), cfg_(cfg), stream_(stream) {
  if (cfg.cache_policy) {
    const double capacity = cfg.cache_capacity_frac * cache_data_size_units(graph, model.cfg_);
    store_ = std::make_unique<CacheStore>(*cfg.cache_policy, capacity);
    if (cfg.hbm_cache_budget_bytes > 0) {
      store_->set_hbm_budget(cfg.hbm_cache_budget_bytes, stream,
                             model.cfg_.seq_len + model.cfg_.horizon);
    }
  }
  IncrementalOptions inc{cfg.fallback_threshold, cfg.rescratch_period};
  provider_ = std::make_unique<AggProvider>(store_.get(), &graph, model.cfg_.aggr, cfg.incremental,
                                            inc, stream);
  loss_ws_ = cuda::DevArray<double>(512, stream);
  model.set_gate_recompute(gate_recompute_policy(model.cfg_, graph.num_nodes()));
  // Layer lanes for multi-layer integrated models (opt-in: DGNN_LAYER_STREAMS=1).
  // Measured at C3 they lose ~7% to the single lane — both lanes are HBM-bound
  // and the part is power-capped, so overlap only adds L2 contention. The
  // HBM-spill level orders its copies against one compute stream, so it keeps
  // a single lane.
  const char* env = std::getenv("DGNN_LAYER_STREAMS");
  const bool lanes_on = env && std::string(env) == "1";
  if (lanes_on && !is_stacked(model.cfg_.arch) && model.cfg_.layers > 1 &&
      cfg.hbm_cache_budget_bytes <= 0) {
    DGNN_CUDA(cudaStreamCreateWithFlags(&aux_, cudaStreamNonBlocking));
  }
}

Worker::~Worker() {
  if (aux_) {
    cudaStreamSynchronize(aux_);
    cuda::release_stream_blocks(aux_);
    cudaStreamSynchronize(aux_);
    cudaStreamDestroy(aux_);
  }
}

void Worker::run_sample(const SequenceWindow& window, Timestep windows_remaining, int64_t batch_id,
                        std::pair<NodeId, NodeId> node_range, float* grad, double* loss_slot) {
  using clk = std::chrono::steady_clock;
  auto since = [](clk::time_point t) {
    return std::chrono::duration<double, std::milli>(clk::now() - t).count();
  };
  const auto h0 = clk::now();
  {
    ProfScope whole(kProfSample, stream_, 0.0);
    SeqSample sample =
        build_sample(graph_, model_.cfg_, window, windows_remaining, batch_id, node_range,
                     cfg_.seed, stream_);
    // from-scratch runs (incremental = false, the ablation baseline) take no
    // delta-based shortcut in the backward either
    if (!cfg_.incremental) sample.graph = nullptr;
    prof_add_host(kProfHostBuild, since(h0));
    const auto h1 = clk::now();
    Lanes lanes(stream_, aux_);
    ForwardArtifacts fwd = model_forward(model_, sample, *provider_, lanes);
    std::vector<Buf> dpred = seed_loss(sample, fwd, model_.cfg_.feature_dim, loss_slot,
                                       loss_ws_.get(), lanes.of(model_.cfg_.layers));
    prof_add_host(kProfHostFwd, since(h1));
    const auto h2 = clk::now();
    model_backward(model_, sample, fwd, dpred, grad, lanes);
    prof_add_host(kProfHostBwd, since(h2));
  }
  // the sample's tape has released its aggregations: re-apply the HBM budget
  if (store_) store_->rebalance();
  prof_add_host(kProfSampleHost, since(h0));
}

// ---------------------------------------------------------------- seq-first
namespace {

// run_epoch_impl (ref src/train.cpp:146-206): seq-first visits (batch outer,
// window inner), node-first (window outer, batch inner).
EpochReport run_epoch_impl(DgnnModel& model, const DeviceGraph& graph,
                           const std::vector<SequenceWindow>& windows, const TrainConfig& cfg,
                           Worker& worker, OptimizerState& opt, int64_t epoch_index,
                           bool seq_first) {
  check(!windows.empty(), "epoch needs at least one window");
  cudaStream_t st = worker.stream();
  AggProvider& provider = worker.provider();
  const CacheStats stats0 = provider.store() ? provider.store()->stats() : CacheStats{};
  const ExecutionStats exec0 = provider.stats();
  cudaEvent_t e0, e1;
  DGNN_CUDA(cudaEventCreate(&e0));
  DGNN_CUDA(cudaEventCreate(&e1));
  DGNN_CUDA(cudaEventRecord(e0, st));
  provider.reset_plan_state();
  EpochReport report;
  auto batches = make_batches(graph.num_nodes(), cfg.batch_size, cfg.seed, epoch_index);
  const int64_t nsamples = static_cast<int64_t>(batches.size() * windows.size());
  cuda::DevArray<double> losses(nsamples, st);
  losses.zero(st);
  cuda::DevArray<float> grad(model.num_params(), st);
  int64_t k = 0;
  auto run = [&](int64_t b, int64_t w) {
    grad.zero(st);
    worker.run_sample(windows[w], static_cast<Timestep>(windows.size() - 1 - w), b, batches[b],
                      grad.get(), losses.get() + k);
    if (!optimizer_step(model, grad.get(), 1.f, opt, cfg, provider.store(), st)) ++report.skipped_steps;
    report.visitation.push_back({b, w});
    ++k;
  };
  const int64_t nb = static_cast<int64_t>(batches.size()), nw = static_cast<int64_t>(windows.size());
  if (seq_first) {
    for (int64_t b = 0; b < nb; ++b)
      for (int64_t w = 0; w < nw; ++w) run(b, w);
  } else {
    for (int64_t w = 0; w < nw; ++w)
      for (int64_t b = 0; b < nb; ++b) run(b, w);
  }
  DGNN_CUDA(cudaEventRecord(e1, st));
  report.sample_losses.resize(nsamples);
  copy_to_host(report.sample_losses.data(), losses.get(), sizeof(double) * nsamples, st);
  float ms = 0.f;
  DGNN_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  DGNN_CUDA(cudaEventDestroy(e0));
  DGNN_CUDA(cudaEventDestroy(e1));
  double total = 0.0;
  for (double l : report.sample_losses) total += l;
  report.loss = report.sample_losses.empty() ? 0.0 : total / report.sample_losses.size();
  report.mae = report.loss;
  if (provider.store()) {
    const CacheStats& s1 = provider.store()->stats();
    report.cache = s1;
    report.cache.hits = s1.hits - stats0.hits;
    report.cache.misses = s1.misses - stats0.misses;
    report.cache.evictions = s1.evictions - stats0.evictions;
    report.cache.expirations = s1.expirations - stats0.expirations;
    report.cache.invalidations = s1.invalidations - stats0.invalidations;
    report.cache.rejected = s1.rejected - stats0.rejected;
  }
  const ExecutionStats& e = provider.stats();
  report.scratch_calls = e.scratch_calls - exec0.scratch_calls;
  report.incremental_calls = e.incremental_calls - exec0.incremental_calls;
  report.fallbacks = e.fallbacks - exec0.fallbacks;
  report.kernel_invocations = report.scratch_calls + report.incremental_calls;
  report.seconds = ms / 1000.0;
  return report;
}

}  // namespace

EpochReport seq_first_epoch(DgnnModel& model, const DeviceGraph& graph,
                            const std::vector<SequenceWindow>& windows, const TrainConfig& cfg,
                            Worker& worker, OptimizerState& opt, int64_t epoch_index) {
  return run_epoch_impl(model, graph, windows, cfg, worker, opt, epoch_index, true);
}

EpochReport node_first_epoch(DgnnModel& model, const DeviceGraph& graph,
                             const std::vector<SequenceWindow>& windows, const TrainConfig& cfg,
                             Worker& worker, OptimizerState& opt, int64_t epoch_index) {
  return run_epoch_impl(model, graph, windows, cfg, worker, opt, epoch_index, false);
}

TrainSession::TrainSession(const DeviceGraph& graph, const ModelConfig& mcfg,
                           const TrainConfig& tcfg, cudaStream_t stream, Timestep window_total)
    : graph_(graph), tcfg_(tcfg) {
  model_ = DgnnModel::create(mcfg, stream);
  windows_ = sliding_windows(window_total > 0 ? window_total : graph.length() - 1, mcfg.seq_len,
                             tcfg.stride, mcfg.horizon);
  check(!windows_.empty(), "dataset too short for the requested windows");
  worker_ = std::make_unique<Worker>(graph, *model_, tcfg, stream);
}

EpochReport TrainSession::run_epoch() {
  EpochReport r =
      tcfg_.iteration == IterationOrder::kSeqFirst
          ? seq_first_epoch(*model_, graph_, windows_, tcfg_, *worker_, opt_, epoch_index_)
          : node_first_epoch(*model_, graph_, windows_, tcfg_, *worker_, opt_, epoch_index_);
  ++epoch_index_;
  return r;
}

// ---------------------------------------------------------------- distributed
std::vector<WorkerAssignment> plan_consecutive_block(Timestep total, int num_workers,
                                                     Timestep seq_len, Timestep stride,
                                                     Timestep horizon) {
  check(num_workers >= 1, "plan needs at least one worker");
  check(total >= num_workers, "fewer snapshots than workers");
  const auto windows = sliding_windows(total, seq_len, stride, horizon);
  const auto W = static_cast<int64_t>(windows.size());
  std::vector<WorkerAssignment> out(num_workers);
  const int64_t base = W / num_workers, extra = W % num_workers;
  int64_t cursor = 0;
  for (int m = 0; m < num_workers; ++m) {
    WorkerAssignment& a = out[m];
    a.window_begin = cursor;
    a.window_end = cursor + base + (m < extra ? 1 : 0);
    cursor = a.window_end;
    a.block_begin = a.window_begin < W ? windows[a.window_begin].start : total;
    a.block_end = m + 1 < num_workers ? (a.window_end < W ? windows[a.window_end].start : total) : total;
    if (a.block_begin > a.block_end) a.block_begin = a.block_end;
  }
  if (!out.empty()) out.front().block_begin = 0;
  return out;
}

CommLedger comm_ledger(const DeviceGraph& graph, PlacementScheme scheme, OverlapMode overlap,
                       int M, Timestep seq_len, Timestep stride, Timestep horizon, int hidden_dim,
                       int64_t num_params, int64_t num_batches, cudaStream_t stream) {
  const Timestep T = graph.length();
  // the reference's distributed epoch windows the full length (src/distsim.cpp:190)
  const auto windows = sliding_windows(T, seq_len, stride, horizon);
  check(!windows.empty(), "distributed epoch needs at least one window");
  check(M >= 1, "plan needs at least one worker");
  check(T >= M, "fewer snapshots than workers");
  CommLedger L;
  L.per_worker.resize(M);
  auto add = [&](int m, uint64_t CommVolume::*f, uint64_t b) {
    L.per_worker[m].*f += b;
    L.total.*f += b;
  };
  // ring all-reduce per optimizer step (src/distsim.cpp:262-268)
  const uint64_t param_bytes = static_cast<uint64_t>(num_params) * 8;
  const auto sync = static_cast<uint64_t>(
      std::llround(2.0 * (M - 1) / std::max(M, 1) * static_cast<double>(param_bytes)));
  for (int64_t b = 0; b < num_batches; ++b)
    for (int m = 0; m < M; ++m) add(m, &CommVolume::gradient_sync, sync);
  const NodeId N = graph.num_nodes();
  std::vector<std::pair<NodeId, NodeId>> ranges;  // node_ranges (src/distsim.cpp:108-117)
  {
    NodeId base = N / M, extra = N % M, cur = 0;
    for (int m = 0; m < M; ++m) {
      const NodeId len = base + (m < extra ? 1 : 0);
      ranges.push_back({cur, cur + len});
      cur += len;
    }
  }
  const uint64_t d = static_cast<uint64_t>(graph.feature_dim());
  if (scheme == PlacementScheme::kConsecutiveBlock && overlap == OverlapMode::kRemoteFetch) {
    // account_snapshot_fetch (src/distsim.cpp:163-178)
    const auto plan = plan_consecutive_block(T, M, seq_len, stride, horizon);
    for (int m = 0; m < M; ++m) {
      const WorkerAssignment& a = plan[m];
      if (a.window_begin == a.window_end) continue;
      const Timestep end = std::min<Timestep>(a.block_end + seq_len + horizon - 1, T);
      for (Timestep t = a.block_end; t < end; ++t)
        add(m, &CommVolume::snapshot_fetch,
            static_cast<uint64_t>(graph.snapshot(t).num_edges) * 8 + static_cast<uint64_t>(N) * d * 8);
    }
  } else if (scheme == PlacementScheme::kNodePartition) {
    // account_node_partition (src/distsim.cpp:121-147), counts on the device
    std::vector<uint64_t> cover(T, 0);
    for (const auto& w : windows)
      for (Timestep t = w.start; t < w.start + w.length + w.horizon; ++t) ++cover[t];
    for (Timestep t = 0; t < T; ++t) {
      if (!cover[t]) continue;
      for (int m = 0; m < M; ++m) {
        const uint64_t uniq = remote_source_count(graph.snapshot(t), N, ranges[m].first, ranges[m].second, stream);
        add(m, &CommVolume::remote_features, uniq * d * 8 * cover[t]);
      }
    }
  } else if (scheme == PlacementScheme::kSequencePartition) {
    // account_sequence_partition (src/distsim.cpp:149-161)
    const uint64_t row = static_cast<uint64_t>(hidden_dim) * 8;
    for (const auto& w : windows)
      for (Timestep idx = 0; idx < w.length; ++idx) {
        const int owner = static_cast<int>(idx % M);
        const uint64_t resident = static_cast<uint64_t>(ranges[owner].second - ranges[owner].first);
        add(owner, &CommVolume::intermediate_redistribution, (static_cast<uint64_t>(N) - resident) * row);
      }
  }
  return L;
}

DistWorker::DistWorker(const DeviceGraph& graph, const ModelConfig& mcfg, const TrainConfig& tcfg,
                       cudaStream_t stream, int rank, int world, Timestep window_total)
    : graph_(graph), tcfg_(tcfg) {
  const Timestep total = window_total > 0 ? window_total : graph.length() - 1;
  model_ = DgnnModel::create(mcfg, stream);
  windows_ = sliding_windows(total, mcfg.seq_len, tcfg.stride, mcfg.horizon);
  check(!windows_.empty(), "distributed epoch needs at least one window");
  assign_ = plan_consecutive_block(total, world, mcfg.seq_len, tcfg.stride, mcfg.horizon).at(rank);
  worker_ = std::make_unique<Worker>(graph, *model_, tcfg, stream);
  grad_w_ = cuda::DevArray<float>(model_->num_params(), stream);
}

void DistWorker::begin_epoch() {
  worker_->provider().reset_plan_state();
  batches_ = make_batches(graph_.num_nodes(), tcfg_.batch_size, tcfg_.seed, epoch_index_);
  const int64_t local = (assign_.window_end - assign_.window_begin) * num_batches();
  losses_ = cuda::DevArray<double>(std::max<int64_t>(local, 1), worker_->stream());
  losses_.zero(worker_->stream());
  n_loss_ = 0;
}

void DistWorker::local_grads(int64_t b, float* grad_sum) {
  cudaStream_t st = worker_->stream();
  DGNN_CUDA(cudaMemsetAsync(grad_sum, 0, sizeof(float) * model_->num_params(), st));
  for (int64_t w = assign_.window_begin; w < assign_.window_end; ++w) {
    grad_w_.zero(st);
    worker_->run_sample(windows_[w], static_cast<Timestep>(assign_.window_end - 1 - w), b,
                        batches_[b], grad_w_.get(), losses_.get() + n_loss_);
    ++n_loss_;
    cuda::axpy(model_->num_params(), 1.f, grad_w_.get(), grad_sum, st);
  }
}

bool DistWorker::apply(const float* grad_sum) {
  const float inv = static_cast<float>(1.0 / static_cast<double>(windows_.size()));
  return optimizer_step(*model_, grad_sum, inv, opt_, tcfg_, worker_->store(), worker_->stream());
}

void DistWorker::end_epoch() { ++epoch_index_; }

DistWorker::EpochResult DistWorker::run_epoch(NcclComm* comm) {
  cudaStream_t st = worker_->stream();
  if (grad_sum_.size() == 0) grad_sum_ = cuda::DevArray<float>(model_->num_params(), st);
  cudaEvent_t ev[2];
  for (auto& e : ev) DGNN_CUDA(cudaEventCreate(&e));
  EpochResult r;
  DGNN_CUDA(cudaEventRecord(ev[0], st));
  begin_epoch();
  r.batches = num_batches();
  for (int64_t b = 0; b < r.batches; ++b) {
    local_grads(b, grad_sum_.get());
    if (comm != nullptr && comm->world() > 1) comm->allreduce_sum(grad_sum_.get(), model_->num_params(), st);
    if (!apply(grad_sum_.get())) ++r.skipped;
  }
  DGNN_CUDA(cudaEventRecord(ev[1], st));
  DGNN_CUDA(cudaEventSynchronize(ev[1]));
  float ms = 0.f;
  DGNN_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[1]));
  for (auto& e : ev) cudaEventDestroy(e);
  r.seconds = ms / 1e3;
  if (comm != nullptr && comm->world() > 1) r.seconds = comm->allreduce_max(r.seconds, st);
  end_epoch();
  return r;
}

std::vector<double> DistWorker::take_losses() {
  std::vector<double> out(n_loss_);
  copy_to_host(out.data(), losses_.get(), sizeof(double) * n_loss_, worker_->stream());
  return out;
}

}  // namespace dgnn
