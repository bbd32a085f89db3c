// B200 aggregation host layer: reference control flow (fallback decisions,
// checks, messages) around the K1/K2/K3 device kernels.
#include "aggregate.hpp"

#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <mutex>
#include <unordered_map>
#include <vector>

namespace dgnn {

namespace cuda {

int64_t& launch_counter() {
  static int64_t c = 0;
  return c;
}

void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
  throw std::runtime_error(std::string("CUDA error ") + cudaGetErrorName(e) + " (" +
                           cudaGetErrorString(e) + ") in " + what + " at " + file + ":" +
                           std::to_string(line));
}

int64_t& dev_bytes_live() {
  static int64_t b = 0;
  return b;
}

namespace {
std::once_flag g_pool_once;
void init_pool() {
  int dev = 0;
  DGNN_CUDA(cudaGetDevice(&dev));
  cudaMemPool_t pool;
  DGNN_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t threshold = UINT64_MAX;  // keep freed blocks cached in the pool
  DGNN_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
}
}  // namespace

void pool_stats(int64_t* reserved, int64_t* used, int64_t* reserved_high, int64_t* used_high) {
  std::call_once(g_pool_once, init_pool);
  int dev = 0;
  DGNN_CUDA(cudaGetDevice(&dev));
  cudaMemPool_t pool;
  DGNN_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  auto get = [&](cudaMemPoolAttr a, int64_t* out) {
    uint64_t v = 0;
    DGNN_CUDA(cudaMemPoolGetAttribute(pool, a, &v));
    if (out) *out = static_cast<int64_t>(v);
  };
  get(cudaMemPoolAttrReservedMemCurrent, reserved);
  get(cudaMemPoolAttrUsedMemCurrent, used);
  get(cudaMemPoolAttrReservedMemHigh, reserved_high);
  get(cudaMemPoolAttrUsedMemHigh, used_high);
}

// Per-stream exact-size block cache over the stream-ordered pool. A training
// sample allocates the same few shapes every time (n x w activations, tapes,
// aggregations); serving them from free lists keeps the driver out of the hot
// loop — cudaMallocAsync was measured to block the host for up to 1.4 s at
// the start of an epoch (the GPU then idles). A block is only reused on the
// stream that freed it, so stream order makes the reuse safe without events.
// On allocation failure every cached block goes back to the pool and the
// allocation is retried once.
namespace {
struct BlockCache {
  std::mutex mu;
  std::unordered_map<cudaStream_t, std::unordered_map<size_t, std::vector<void*>>> free;
  int64_t cached_bytes = 0;
};
BlockCache& block_cache() {
  static BlockCache* c = new BlockCache();  // never destroyed: frees may run at exit
  return *c;
}
// Size classes: 4 KB granules below 1 MB, then 8 classes per octave (at most
// 12.5% slack), so buffers whose sizes drift slightly (per-snapshot edge
// counts) still share a class.
size_t round_block(size_t bytes) {
  constexpr size_t kSmall = size_t{1} << 20;
  if (bytes < kSmall) return (bytes + 4095) / 4096 * 4096;
  int top = 63 - __builtin_clzll(static_cast<unsigned long long>(bytes));
  const size_t step = size_t{1} << (top - 3);
  return (bytes + step - 1) / step * step;
}
void release_cached_locked(BlockCache& c) {
  for (auto& [st, lists] : c.free)
    for (auto& [sz, v] : lists)
      for (void* p : v) cudaFreeAsync(p, st);
  c.free.clear();
  c.cached_bytes = 0;
}
}  // namespace

int64_t cached_block_bytes() {
  BlockCache& c = block_cache();
  std::lock_guard<std::mutex> lk(c.mu);
  return c.cached_bytes;
}

void release_cached_blocks() {
  BlockCache& c = block_cache();
  std::lock_guard<std::mutex> lk(c.mu);
  release_cached_locked(c);
}

void release_stream_blocks(cudaStream_t stream) {
  BlockCache& c = block_cache();
  std::lock_guard<std::mutex> lk(c.mu);
  auto it = c.free.find(stream);
  if (it == c.free.end()) return;
  for (auto& [sz, v] : it->second) {
    for (void* p : v) cudaFreeAsync(p, stream);
    c.cached_bytes -= static_cast<int64_t>(sz * v.size());
  }
  c.free.erase(it);
}

void* dev_alloc(size_t bytes, cudaStream_t stream) {
  std::call_once(g_pool_once, init_pool);
  const size_t r = round_block(bytes);
  BlockCache& c = block_cache();
  std::lock_guard<std::mutex> lk(c.mu);
  auto sit = c.free.find(stream);
  if (sit != c.free.end()) {
    auto it = sit->second.find(r);
    if (it != sit->second.end() && !it->second.empty()) {
      void* p = it->second.back();
      it->second.pop_back();
      c.cached_bytes -= static_cast<int64_t>(r);
      dev_bytes_live() += static_cast<int64_t>(r);
      return p;
    }
  }
  void* p = nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  cudaError_t e = cudaMallocAsync(&p, r, stream);
  if (e != cudaSuccess && c.cached_bytes > 0) {
    (void)cudaGetLastError();
    release_cached_locked(c);
    DGNN_CUDA(cudaDeviceSynchronize());
    e = cudaMallocAsync(&p, r, stream);
  }
  prof_add_host(kProfHostAlloc,
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    throw std::runtime_error("device allocation of " + std::to_string(bytes) + " bytes failed: " +
                             cudaGetErrorString(e) + " (live " + std::to_string(dev_bytes_live() >> 20) +
                             " MiB in buffers, device free " + std::to_string(free_b >> 20) + " of " +
                             std::to_string(total_b >> 20) + " MiB)");
  }
  dev_bytes_live() += static_cast<int64_t>(r);
  return p;
}

void dev_free(void* p, size_t bytes, cudaStream_t stream) {
  if (!p) return;
  const size_t r = round_block(bytes);
  BlockCache& c = block_cache();
  std::lock_guard<std::mutex> lk(c.mu);
  c.free[stream][r].push_back(p);
  c.cached_bytes += static_cast<int64_t>(r);
  dev_bytes_live() -= static_cast<int64_t>(r);
}

}  // namespace cuda

const char* to_string(AggrKind kind) {
  switch (kind) {
    case AggrKind::kSum: return "sum";
    case AggrKind::kMean: return "mean";
    case AggrKind::kMax: return "max";
    case AggrKind::kMin: return "min";
  }
  return "?";
}

AggrKind aggr_kind_from_string(const std::string& s) {
  if (s == "sum") return AggrKind::kSum;
  if (s == "mean") return AggrKind::kMean;
  if (s == "max") return AggrKind::kMax;
  if (s == "min") return AggrKind::kMin;
  fail("unknown aggregation kind: " + s);
}

GraphView GraphView::of(const DeviceGraph& g, Timestep t) {
  const DevSnapshot& s = g.snapshot(t);
  GraphView v;
  v.num_nodes = g.num_nodes();
  v.num_edges = s.num_edges;
  v.in_ptr = s.in_ptr.get();
  v.in_src = s.in_src.get();
  v.out_ptr = s.out_ptr.get();
  v.out_dst = s.out_dst.get();
  v.t = t;
  return v;
}

double change_ratio(const DevDelta& delta, EdgeIdx base_edges) {
  if (base_edges <= 0) return std::numeric_limits<double>::infinity();
  return static_cast<double>(delta.change_count()) / (2.0 * static_cast<double>(base_edges));
}

// ---------------------------------------------------------------- profiling
namespace {
struct Pending {
  int cls;
  cudaEvent_t a, b;
  double bytes, flops;
};
bool g_prof = false;
std::vector<Pending> g_pending;
ProfStat g_stats[kProfCount];
std::vector<cudaEvent_t> g_event_pool;

cudaEvent_t take_event() {
  if (!g_event_pool.empty()) {
    cudaEvent_t e = g_event_pool.back();
    g_event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  DGNN_CUDA(cudaEventCreate(&e));
  return e;
}
}  // namespace

void prof_enable(bool on) { g_prof = on; }
bool prof_enabled() { return g_prof; }
void prof_reset() {
  prof_flush();
  for (auto& s : g_stats) s = ProfStat{};
}
void prof_flush() {
  for (auto& p : g_pending) {
    DGNN_CUDA(cudaEventSynchronize(p.b));
    float ms = 0.f;
    DGNN_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
    g_stats[p.cls].launches += 1;
    g_stats[p.cls].ms += ms;
    g_stats[p.cls].max_ms = std::max(g_stats[p.cls].max_ms, static_cast<double>(ms));
    g_stats[p.cls].bytes += p.bytes;
    g_stats[p.cls].flops += p.flops;
    g_event_pool.push_back(p.a);
    g_event_pool.push_back(p.b);
  }
  g_pending.clear();
}
ProfStat prof_get(int cls) { return (cls >= 0 && cls < kProfCount) ? g_stats[cls] : ProfStat{}; }
void prof_add_host(int cls, double ms) {
  if (!g_prof || cls < 0 || cls >= kProfCount) return;
  g_stats[cls].launches += 1;
  g_stats[cls].ms += ms;
  if (ms > g_stats[cls].max_ms) {
    g_stats[cls].max_ms = ms;
    g_stats[cls].flops = static_cast<double>(g_stats[cls].launches - 1);  // index of the longest
  }
}

ProfScope::ProfScope(int cls, cudaStream_t s, double bytes, double flops)
    : cls_(cls), s_(s), bytes_(bytes), flops_(flops) {
  if (!g_prof) return;
  a_ = take_event();
  b_ = take_event();
  DGNN_CUDA(cudaEventRecord(a_, s_));
}
ProfScope::~ProfScope() {
  if (!a_) return;
  // queued only once both ends are recorded: a flush triggered by an inner
  // scope must never see an open (unrecorded) outer scope
  cudaEventRecord(b_, s_);
  g_pending.push_back({cls_, a_, b_, bytes_, flops_});
  if (g_pending.size() > 4096) {
    try {
      prof_flush();
    } catch (...) {
      g_pending.clear();
    }
  }
}

// ---------------------------------------------------------------- helpers
namespace {

int kind_i(AggrKind k) { return static_cast<int>(k); }

std::shared_ptr<AggResult> alloc_result(AggrKind kind, NodeId n, int32_t dim, cudaStream_t st) {
  auto r = std::make_shared<AggResult>();
  r->kind = kind;
  r->rows = n;
  r->dim = dim;
  const size_t nw = static_cast<size_t>(n) * dim;
  r->values = cuda::DevArray<float>(nw, st);
  if (kind == AggrKind::kMean) {
    r->degree = cuda::DevArray<float>(n, st);
    r->mean_sums = cuda::DevArray<float>(nw, st);
  }
  if (kind == AggrKind::kMax || kind == AggrKind::kMin) {
    r->argext = cuda::DevArray<int32_t>(nw, st);
    r->dense = cuda::DevArray<float>(nw, st);
  }
  return r;
}

void refresh_dense(AggResult& r, cudaStream_t st) {
  if (!r.extremal()) return;
  cuda::mask_empty_rows(r.rows, r.dim, r.argext.get(), r.values.get(), r.dense.get(), st);
}

void copy_dev(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes) DGNN_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st));
}

}  // namespace

std::shared_ptr<AggResult> aggregate_scratch(const GraphView& graph, const float* feats,
                                             int32_t dim, const AggrFn& fn, cudaStream_t stream) {
  check(feats != nullptr, "feature rows must cover all node ids");
  check(!fn.edge_weighted, "edge-weighted aggregation over an unweighted view");
  auto r = alloc_result(fn.kind, graph.num_nodes, dim, stream);
  r->num_edges = graph.num_edges;
  r->t = graph.t;
  {
    // per-edge gather of a w-wide row + CSR + one output write
    const double bytes = 8.0 * (graph.num_nodes + 1) + 4.0 * graph.num_edges +
                         4.0 * dim * graph.num_edges + 4.0 * dim * graph.num_nodes;
    ProfScope ps(kProfAggScratch, stream, bytes);
    cuda::agg_scratch(kind_i(fn.kind), graph.num_nodes, dim, graph.in_ptr, graph.in_src, feats,
                      r->values.get(), r->degree.get(), r->mean_sums.get(), r->argext.get(), stream);
  }
  refresh_dense(*r, stream);
  return r;
}

std::shared_ptr<AggResult> aggregate_zero_sum(const GraphView& graph, int32_t dim, cudaStream_t stream) {
  auto r = alloc_result(AggrKind::kSum, graph.num_nodes, dim, stream);
  r->num_edges = graph.num_edges;
  r->t = graph.t;
  const size_t nw = static_cast<size_t>(graph.num_nodes) * dim;
  ProfScope ps(kProfAggScratch, stream, 4.0 * nw);
  if (nw) DGNN_CUDA(cudaMemsetAsync(r->values.get(), 0, nw * sizeof(float), stream));
  return r;
}

bool rebase_supported(const AggrFn& fn, int32_t dim, const float* feats) {
  return cuda::agg_delta_struct_supported(kind_i(fn.kind), dim, feats);
}

std::shared_ptr<AggResult> aggregate_rebase(const AggResult& base, const GraphView& graph,
                                            const float* feats, int32_t dim, const DevDelta& delta,
                                            const AggrFn& fn, cudaStream_t stream) {
  check(fn.kind == AggrKind::kSum || fn.kind == AggrKind::kMean, "rebase: sum / mean only");
  check(base.rows == graph.num_nodes, "rebase: base rows differ from the view");
  auto r = alloc_result(fn.kind, graph.num_nodes, dim, stream);
  r->num_edges = graph.num_edges;
  r->t = graph.t;
  const size_t nw = static_cast<size_t>(graph.num_nodes) * dim;
  // copy of the base + the structural delta's gathers and row read-modify-writes
  const double bytes = 8.0 * nw + 8.0 * delta.n_ent_c + 4.0 * dim * delta.n_ent_c +
                       8.0 * dim * delta.n_rows;
  ProfScope ps(kProfAggRebase, stream, bytes);
  copy_dev(r->values.get(), base.values.get(), nw * sizeof(float), stream);
  if (fn.kind == AggrKind::kMean) {
    copy_dev(r->degree.get(), base.degree.get(), graph.num_nodes * sizeof(float), stream);
    copy_dev(r->mean_sums.get(), base.mean_sums.get(), nw * sizeof(float), stream);
  }
  const bool ok = cuda::agg_delta_struct(kind_i(fn.kind), delta.n_rows, dim, delta.rows.get(),
                                         delta.row_ptr_c.get(), delta.ent_c.get(), graph.num_nodes,
                                         delta.changed.get(), feats, r->values.get(),
                                         r->degree.get(), r->mean_sums.get(), stream);
  check(ok, "rebase: unsupported aggregation shape");
  return r;
}

bool aggregate_backward_delta(const DevDelta& delta, int32_t num_nodes, const float* upstream,
                              int32_t dim, float* grad, cudaStream_t stream) {
  if (!cuda::agg_delta_struct_supported(kind_i(AggrKind::kSum), dim, upstream) ||
      !cuda::agg_delta_struct_supported(kind_i(AggrKind::kSum), dim, grad))
    return false;
  const double bytes = 8.0 * delta.n_ent_t + 4.0 * dim * delta.n_ent_t + 8.0 * dim * delta.n_rows_t;
  ProfScope ps(kProfAggRebase, stream, bytes);
  return cuda::agg_delta_struct(kind_i(AggrKind::kSum), delta.n_rows_t, dim, delta.rows_t.get(),
                                delta.row_ptr_t.get(), delta.ent_t.get(), num_nodes, nullptr, upstream,
                                grad, nullptr, nullptr, stream);
}

IncrementalResult aggregate_incremental(const AggResult& prev, const GraphView& prev_graph,
                                        const GraphView& curr_graph, const float* prev_feats,
                                        const float* curr_feats, const DevDelta& delta,
                                        Timestep delta_t, const AggrFn& fn,
                                        const IncrementalOptions& opts, cudaStream_t stream) {
  (void)prev_graph;
  check(prev.kind == fn.kind, "incremental update must keep the aggregation kind");
  check(prev.t + 1 == delta_t, "incremental update needs the delta for t = prev.t + 1");
  if (fn.kind == AggrKind::kMean) {
    check(prev.degree.size() > 0, "mean update needs the stored degree vector");
  }
  if (fn.kind == AggrKind::kMax || fn.kind == AggrKind::kMin) {
    check(prev.argext.size() > 0, "max/min update needs stored contributor ids");
  }
  const int32_t dim = prev.dim;
  auto fallback = [&](FallbackReason why) {
    IncrementalResult out{aggregate_scratch(curr_graph, curr_feats, dim, fn, stream), true, why};
    out.result->t = delta_t;
    return out;
  };
  if (change_ratio(delta, prev.num_edges) > opts.fallback_threshold) {
    return fallback(FallbackReason::kChangeRatio);
  }
  if (opts.rescratch_period > 0 && prev.incremental_depth + 1 >= opts.rescratch_period) {
    return fallback(FallbackReason::kRescratchPeriod);
  }
  const bool extremal = fn.kind == AggrKind::kMax || fn.kind == AggrKind::kMin;
  if (extremal && delta.n_del > 0) {
    // A deleted edge that supplied any recorded extremum invalidates the row.
    cuda::DevArray<int32_t> flag(1, stream);
    flag.zero(stream);
    cuda::agg_deleted_contributor(delta.n_del, dim, delta.del.get(), prev.argext.get(), flag.get(), stream);
    int32_t h = 0;
    copy_to_host(&h, flag.get(), sizeof(h), stream);
    if (h) return fallback(FallbackReason::kDeletedContributor);
  }
  auto r = alloc_result(fn.kind, prev.rows, dim, stream);
  r->t = delta_t;
  r->num_edges = curr_graph.num_edges;
  r->incremental_depth = prev.incremental_depth + 1;
  const size_t nw = static_cast<size_t>(prev.rows) * dim;
  copy_dev(r->values.get(), prev.values.get(), nw * sizeof(float), stream);
  if (fn.kind == AggrKind::kMean) {
    copy_dev(r->degree.get(), prev.degree.get(), prev.rows * sizeof(float), stream);
    copy_dev(r->mean_sums.get(), prev.mean_sums.get(), nw * sizeof(float), stream);
  }
  if (extremal) copy_dev(r->argext.get(), prev.argext.get(), nw * sizeof(int32_t), stream);
  {
    // graded delta-SpMM bytes: 8|D| + 4d(U- + U+) + 8d U_dst
    double bytes = 8.0 * delta.n_ent + 4.0 * dim * (delta.u_minus + delta.u_plus) +
                   8.0 * dim * delta.n_rows;
    if (fn.kind == AggrKind::kMean) bytes += 8.0 * delta.n_rows;
    ProfScope ps(kProfAggDelta, stream, bytes);
    cuda::agg_delta(kind_i(fn.kind), delta.n_rows, dim, delta.rows.get(), delta.row_ptr.get(),
                    delta.ent.get(), prev_feats, curr_feats, r->values.get(), r->degree.get(),
                    r->mean_sums.get(), r->argext.get(), stream, delta.ent_c.get(),
                    curr_graph.num_nodes, delta.n_changed, delta.compact.get(),
                    delta.row_ptr_c.get());
  }
  refresh_dense(*r, stream);
  return {std::move(r), false, FallbackReason::kNone};
}

void aggregate_backward(const GraphView& graph, const float* upstream, int32_t dim,
                        const AggrFn& fn, const AggResult& forward, float* grad,
                        cudaStream_t stream, const float* addend) {
  check(!fn.edge_weighted, "edge-weighted aggregation over an unweighted view");
  if (fn.kind == AggrKind::kMean) {
    check(forward.degree.size() == static_cast<size_t>(graph.num_nodes),
          "mean backward needs forward degree");
  }
  if (fn.kind == AggrKind::kMax || fn.kind == AggrKind::kMin) {
    check(forward.argext.size() == static_cast<size_t>(graph.num_nodes) * dim,
          "max/min backward needs forward argext");
  }
  const double bytes = 8.0 * (graph.num_nodes + 1) + 4.0 * graph.num_edges +
                       4.0 * dim * graph.num_edges + 4.0 * dim * graph.num_nodes +
                       (addend ? 4.0 * dim * graph.num_nodes : 0.0);
  ProfScope ps(kProfAggBackward, stream, bytes);
  cuda::agg_backward(kind_i(fn.kind), graph.num_nodes, dim, graph.out_ptr, graph.out_dst, upstream,
                     forward.degree.get(), forward.argext.get(), grad, stream, addend);
}

}  // namespace dgnn
