// Device memory: stream-ordered allocations from the device's default memory
// pool with an unbounded release threshold, i.e. a caching allocator whose
// frees are ordered on the owning stream (no device-wide synchronisation on the
// hot path).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <memory>
#include <utility>

#include "common.cuh"

namespace dgnn {
namespace cuda {

void* dev_alloc(size_t bytes, cudaStream_t stream);
void dev_free(void* p, size_t bytes, cudaStream_t stream);
// Blocks held by the per-stream free lists (see aggregate.cpp) / return them
// to the pool (callers must not have work pending that uses them).
int64_t cached_block_bytes();
void release_cached_blocks();
void release_stream_blocks(cudaStream_t stream);  // before destroying `stream`
// Stream-ordered pool occupancy: bytes reserved from the device / in live
// allocations, current and high-water.
void pool_stats(int64_t* reserved, int64_t* used, int64_t* reserved_high, int64_t* used_high);
// Bytes currently held by live DevArray allocations (for memory reporting).
int64_t& dev_bytes_live();

template <typename T>
class DevArray {
 public:
  DevArray() = default;
  DevArray(size_t n, cudaStream_t stream) : n_(n), stream_(stream) {
    if (n > 0) p_ = static_cast<T*>(dev_alloc(n * sizeof(T), stream));
  }
  ~DevArray() { reset(); }
  DevArray(const DevArray&) = delete;
  DevArray& operator=(const DevArray&) = delete;
  DevArray(DevArray&& o) noexcept { *this = std::move(o); }
  DevArray& operator=(DevArray&& o) noexcept {
    if (this != &o) {
      reset();
      p_ = o.p_;
      n_ = o.n_;
      stream_ = o.stream_;
      o.p_ = nullptr;
      o.n_ = 0;
    }
    return *this;
  }
  void reset() {
    if (p_) dev_free(p_, n_ * sizeof(T), stream_);
    p_ = nullptr;
    n_ = 0;
  }
  void zero(cudaStream_t s) {
    if (n_) DGNN_CUDA(cudaMemsetAsync(p_, 0, n_ * sizeof(T), s));
  }
  T* get() const { return p_; }
  size_t size() const { return n_; }
  size_t bytes() const { return n_ * sizeof(T); }
  explicit operator bool() const { return p_ != nullptr; }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
  cudaStream_t stream_ = nullptr;
};

}  // namespace cuda
}  // namespace dgnn
