// Second cache level (B200 addition): HBM <-> pinned host DRAM placement of
// cached aggregation payloads.
//
// The logical cache (CacheStore: what is resident, F / I / priority, hits,
// evictions) never changes because of placement; this layer only decides
// where a resident payload's bytes live:
//   kHbm     device arrays present, usable by kernels
//   kHost    bytes in a pinned host block, device arrays released
//   kInbound host->device copy issued on the copy stream, not yet waited on
// Spills (device -> host) and refills (host -> device) run on two copy
// streams, so PCIe carries both directions at once. A pinned block carries
// the event of its last use: a refill reading it waits for the spill that
// wrote it, a later spill into it waits for that refill. Device buffers a
// spill reads are released to the compute stream's allocator only after the
// spill copy has completed (polled); when the spills in flight exceed the
// in-flight cap the host waits for the oldest (backpressure: a saturated
// link must not turn into unbounded HBM held by retiring buffers). The
// compute stream waits on an inbound payload's event only when the payload
// is handed out (get / peek).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <vector>

#include "aggregate.hpp"

namespace dgnn {

// Exact-size free lists of cudaHostAlloc blocks (every cached aggregation of a
// run has one of a handful of sizes), kept until the pool is destroyed.
class PinnedPool {
 public:
  PinnedPool() = default;
  ~PinnedPool();
  PinnedPool(const PinnedPool&) = delete;
  PinnedPool& operator=(const PinnedPool&) = delete;
  // a block and the event of its last copy (null: never used)
  void* take(size_t bytes, cudaEvent_t* last_use);
  void give(void* p, size_t bytes, cudaEvent_t last_use);
  int64_t reserved_bytes() const { return reserved_; }

 private:
  std::map<size_t, std::vector<std::pair<void*, cudaEvent_t>>> free_;
  std::vector<void*> all_;
  int64_t reserved_ = 0;
};

struct Placement {
  enum class Where : uint8_t { kHbm, kHost, kInbound };
  Where where = Where::kHbm;
  void* host = nullptr;
  size_t host_bytes = 0;
  cudaEvent_t host_written = nullptr;  // D2H completion into `host` while kHost
  cudaEvent_t inbound = nullptr;       // H2D completion while kInbound
};

struct TierStats {
  int64_t spills = 0;
  int64_t refills = 0;         // payloads brought back to HBM (prefetched or on demand)
  int64_t prefetches = 0;      // refills issued ahead of the access
  int64_t demand_refills = 0;  // refills issued at the access itself
  int64_t spill_bytes = 0;
  int64_t refill_bytes = 0;
};

class HbmTier {
 public:
  HbmTier(int64_t budget_bytes, cudaStream_t compute);
  ~HbmTier();
  HbmTier(const HbmTier&) = delete;
  HbmTier& operator=(const HbmTier&) = delete;

  int64_t budget() const { return budget_; }
  cudaStream_t compute() const { return compute_; }
  cudaStream_t copy() const { return d2h_; }
  const TierStats& stats() const { return stats_; }
  int64_t pinned_bytes() const { return pool_.reserved_bytes(); }

  static int64_t device_bytes(const AggResult& r);
  // device -> host; the payload's arrays are released once the copy is done
  void spill(AggResult& r, Placement& p);
  // host -> device on the copy stream (kHost -> kInbound)
  void fetch(AggResult& r, Placement& p, bool ahead);
  // compute stream waits for an inbound payload (kInbound -> kHbm)
  void settle(Placement& p);
  // the entry leaves the cache: return its host block / order its buffers
  void drop(AggResult& r, Placement& p);
  // release device buffers whose spill copies have completed
  void reap(bool wait = false);

 private:
  struct Retiring {
    cudaEvent_t done;
    int64_t bytes = 0;
    std::vector<cuda::DevArray<float>> f;
    std::vector<cuda::DevArray<int32_t>> i;
  };
  cudaEvent_t take_event();
  void give_event(cudaEvent_t e) {
    if (e) events_.push_back(e);
  }

  int64_t budget_;
  int64_t retiring_cap_;  // device bytes of spills in flight before the host waits
  int64_t retiring_bytes_ = 0;
  cudaStream_t compute_;
  cudaStream_t d2h_ = nullptr, h2d_ = nullptr;
  PinnedPool pool_;
  std::vector<Retiring> retiring_;
  std::vector<cudaEvent_t> events_;
  TierStats stats_;
};

}  // namespace dgnn
