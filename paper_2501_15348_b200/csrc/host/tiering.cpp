// HBM <-> pinned-host placement of cached aggregations (see tiering.hpp).
#include "tiering.hpp"

#include <algorithm>
#include <cstdlib>
#include <utility>

namespace dgnn {

// ---------------------------------------------------------------- PinnedPool
PinnedPool::~PinnedPool() {
  for (auto& [sz, v] : free_)
    for (auto& [p, e] : v)
      if (e) cudaEventDestroy(e);
  for (void* p : all_) cudaFreeHost(p);
}

void* PinnedPool::take(size_t bytes, cudaEvent_t* last_use) {
  auto it = free_.find(bytes);
  if (it != free_.end() && !it->second.empty()) {
    auto [p, e] = it->second.back();
    it->second.pop_back();
    *last_use = e;
    return p;
  }
  void* p = nullptr;
  DGNN_CUDA(cudaHostAlloc(&p, bytes, cudaHostAllocPortable));
  all_.push_back(p);
  reserved_ += static_cast<int64_t>(bytes);
  *last_use = nullptr;
  return p;
}

void PinnedPool::give(void* p, size_t bytes, cudaEvent_t last_use) {
  if (p) free_[bytes].emplace_back(p, last_use);
}

// ---------------------------------------------------------------- HbmTier
namespace {

// The payload's device arrays in one fixed order; the host block is their
// concatenation. Sizes follow from (kind, rows, dim), so a refill re-creates
// exactly the arrays alloc_result made.
template <typename F, typename I>
void each_array(AggResult& r, F&& on_float, I&& on_int) {
  on_float(r.values);
  on_float(r.degree);
  on_float(r.mean_sums);
  on_float(r.dense);
  on_int(r.argext);
}

struct Shape {
  size_t values = 0, degree = 0, mean_sums = 0, dense = 0, argext = 0;
  size_t bytes() const { return 4 * (values + degree + mean_sums + dense + argext); }
};

Shape shape_of(const AggResult& r) {
  Shape s;
  const size_t nw = static_cast<size_t>(r.rows) * r.dim;
  s.values = nw;
  if (r.kind == AggrKind::kMean) {
    s.degree = static_cast<size_t>(r.rows);
    s.mean_sums = nw;
  }
  if (r.extremal()) {
    s.dense = nw;
    s.argext = nw;
  }
  return s;
}

}  // namespace

namespace {
// device bytes of spills in flight before the host waits: max(budget, 4 GB),
// or DGNN_TIER_INFLIGHT_MB (tests force the backpressure path with it)
int64_t inflight_cap(int64_t budget) {
  if (const char* e = std::getenv("DGNN_TIER_INFLIGHT_MB")) return std::max<int64_t>(1, std::atoll(e)) << 20;
  return std::max<int64_t>(budget, int64_t{4} << 30);
}
}  // namespace

HbmTier::HbmTier(int64_t budget_bytes, cudaStream_t compute)
    : budget_(budget_bytes), retiring_cap_(inflight_cap(budget_bytes)), compute_(compute) {
  DGNN_CUDA(cudaStreamCreateWithFlags(&d2h_, cudaStreamNonBlocking));
  DGNN_CUDA(cudaStreamCreateWithFlags(&h2d_, cudaStreamNonBlocking));
}

HbmTier::~HbmTier() {
  if (d2h_) cudaStreamSynchronize(d2h_);
  if (h2d_) cudaStreamSynchronize(h2d_);
  reap(true);
  for (cudaEvent_t e : events_) cudaEventDestroy(e);
  if (d2h_) cudaStreamDestroy(d2h_);
  if (h2d_) cudaStreamDestroy(h2d_);
}

cudaEvent_t HbmTier::take_event() {
  if (!events_.empty()) {
    cudaEvent_t e = events_.back();
    events_.pop_back();
    return e;
  }
  cudaEvent_t e;
  DGNN_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return e;
}

int64_t HbmTier::device_bytes(const AggResult& r) {
  return static_cast<int64_t>(shape_of(r).bytes());
}

void HbmTier::spill(AggResult& r, Placement& p) {
  const Shape s = shape_of(r);
  // backpressure: bound the device bytes held by spills still in flight
  reap();
  while (retiring_bytes_ + static_cast<int64_t>(s.bytes()) > retiring_cap_ && !retiring_.empty()) {
    DGNN_CUDA(cudaEventSynchronize(retiring_.front().done));
    reap();
  }
  p.host_bytes = s.bytes();
  cudaEvent_t last_read = nullptr;
  p.host = pool_.take(p.host_bytes, &last_read);
  // the block's previous refill must have read it before this spill writes it
  if (last_read) {
    DGNN_CUDA(cudaStreamWaitEvent(d2h_, last_read, 0));
    give_event(last_read);
  }
  // the copy starts after everything the compute stream has queued so far
  // (the payload's producer and every reader issued before the spill)
  cudaEvent_t produced = take_event();
  DGNN_CUDA(cudaEventRecord(produced, compute_));
  DGNN_CUDA(cudaStreamWaitEvent(d2h_, produced, 0));
  give_event(produced);
  Retiring ret;
  ret.done = take_event();
  ret.bytes = static_cast<int64_t>(s.bytes());
  char* dst = static_cast<char*>(p.host);
  auto out = [&](auto& arr, auto& keep) {
    if (arr.size() == 0) return;
    DGNN_CUDA(cudaMemcpyAsync(dst, arr.get(), arr.bytes(), cudaMemcpyDeviceToHost, d2h_));
    dst += arr.bytes();
    keep.push_back(std::move(arr));
  };
  each_array(r, [&](cuda::DevArray<float>& a) { out(a, ret.f); },
             [&](cuda::DevArray<int32_t>& a) { out(a, ret.i); });
  DGNN_CUDA(cudaEventRecord(ret.done, d2h_));
  // the refill of this payload reads the block after this write
  p.host_written = take_event();
  DGNN_CUDA(cudaEventRecord(p.host_written, d2h_));
  retiring_bytes_ += ret.bytes;
  retiring_.push_back(std::move(ret));
  p.where = Placement::Where::kHost;
  ++stats_.spills;
  stats_.spill_bytes += static_cast<int64_t>(p.host_bytes);
}

void HbmTier::fetch(AggResult& r, Placement& p, bool ahead) {
  const Shape s = shape_of(r);
  // device arrays come from the compute stream's allocator; the copy stream
  // writes them only after the compute stream has reached this point
  r.values = cuda::DevArray<float>(s.values, compute_);
  r.degree = cuda::DevArray<float>(s.degree, compute_);
  r.mean_sums = cuda::DevArray<float>(s.mean_sums, compute_);
  r.dense = cuda::DevArray<float>(s.dense, compute_);
  r.argext = cuda::DevArray<int32_t>(s.argext, compute_);
  cudaEvent_t allocated = take_event();
  DGNN_CUDA(cudaEventRecord(allocated, compute_));
  DGNN_CUDA(cudaStreamWaitEvent(h2d_, allocated, 0));
  give_event(allocated);
  // the spill that wrote the block has completed before it is read
  if (p.host_written) {
    DGNN_CUDA(cudaStreamWaitEvent(h2d_, p.host_written, 0));
    give_event(p.host_written);
    p.host_written = nullptr;
  }
  const char* src = static_cast<const char*>(p.host);
  auto in = [&](auto& arr) {
    if (arr.size() == 0) return;
    DGNN_CUDA(cudaMemcpyAsync(arr.get(), src, arr.bytes(), cudaMemcpyHostToDevice, h2d_));
    src += arr.bytes();
  };
  each_array(r, in, in);
  p.inbound = take_event();
  DGNN_CUDA(cudaEventRecord(p.inbound, h2d_));
  // the next spill into this block waits for this read of it
  cudaEvent_t read_done = take_event();
  DGNN_CUDA(cudaEventRecord(read_done, h2d_));
  pool_.give(p.host, p.host_bytes, read_done);
  p.host = nullptr;
  p.where = Placement::Where::kInbound;
  ++stats_.refills;
  ++(ahead ? stats_.prefetches : stats_.demand_refills);
  stats_.refill_bytes += static_cast<int64_t>(p.host_bytes);
}

void HbmTier::settle(Placement& p) {
  if (p.where != Placement::Where::kInbound) return;
  DGNN_CUDA(cudaStreamWaitEvent(compute_, p.inbound, 0));
  give_event(p.inbound);
  p.inbound = nullptr;
  p.where = Placement::Where::kHbm;
}

void HbmTier::drop(AggResult& r, Placement& p) {
  (void)r;
  if (p.where == Placement::Where::kHost) {
    // its last use is the spill that wrote it
    pool_.give(p.host, p.host_bytes, p.host_written);
    p.host_written = nullptr;
    p.host = nullptr;
  } else if (p.where == Placement::Where::kInbound) {
    // the arrays are released in compute-stream order: order that after the
    // copy that fills them
    settle(p);
  }
  p.where = Placement::Where::kHbm;
}

void HbmTier::reap(bool wait) {
  size_t keep = 0;
  for (size_t k = 0; k < retiring_.size(); ++k) {
    Retiring& r = retiring_[k];
    const cudaError_t q = wait ? cudaEventSynchronize(r.done) : cudaEventQuery(r.done);
    if (q == cudaSuccess) {
      give_event(r.done);
      r.f.clear();  // back to the compute stream's free lists
      r.i.clear();
      retiring_bytes_ -= r.bytes;
      continue;
    }
    if (q != cudaErrorNotReady) DGNN_CUDA(q);
    if (keep != k) retiring_[keep] = std::move(r);
    ++keep;
  }
  retiring_.resize(keep);
}

}  // namespace dgnn
