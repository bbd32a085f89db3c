// Shared device/host helpers for the B200 dynamic-GNN hot path.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

namespace dgnn {
namespace cuda {

// Every kernel launch goes through DGNN_LAUNCH so the library can report how
// many of its own kernels ran inside a timed region (bench.py gpu_launches).
int64_t& launch_counter();

[[noreturn]] void throw_cuda(cudaError_t e, const char* what, const char* file, int line);

inline void check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) throw_cuda(e, what, file, line);
}

#define DGNN_CUDA(call) ::dgnn::cuda::check((call), #call, __FILE__, __LINE__)

// Device-side invariant checks of the checked build (DGNN_CHECKED=1, see
// build.py): a failed check prints its condition and traps the kernel.
#if defined(DGNN_CHECKED) && DGNN_CHECKED
#define DGNN_DCHECK(cond)                                                                  \
  do {                                                                                     \
    if (!(cond)) {                                                                         \
      printf("DGNN_DCHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);                \
      __trap();                                                                            \
    }                                                                                      \
  } while (0)
#else
#define DGNN_DCHECK(cond) \
  do {                    \
  } while (0)
#endif

#define DGNN_LAUNCH(kernel, grid, block, smem, stream, ...)                                \
  do {                                                                                      \
    ++::dgnn::cuda::launch_counter();                                                       \
    kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);                             \
    ::dgnn::cuda::check(cudaGetLastError(), #kernel, __FILE__, __LINE__);                  \
  } while (0)

constexpr int kNumSMs = 148;  // B200: 2 dies x 74 SMs

inline int ceil_div(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

// Grid for a grid-stride loop: enough CTAs to cover `work` items, capped at a
// whole number of waves of `per_sm` resident CTAs on all SMs.
inline int wave_grid(int64_t work, int threads, int per_sm) {
  int64_t need = (work + threads - 1) / threads;
  int64_t cap = static_cast<int64_t>(kNumSMs) * per_sm;
  if (need < 1) need = 1;
  return static_cast<int>(need < cap ? need : cap);
}

}  // namespace cuda
}  // namespace dgnn
