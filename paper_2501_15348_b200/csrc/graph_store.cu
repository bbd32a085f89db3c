// Device graph store build: snapshot CSRs (K12) and extract_delta (K11).
// Integer work only; every output is bit-exact with the reference
// (src/snapshot.cpp:20-154). Sorting/selection/scans use CUB (CUDA toolkit
// library primitives); the graph-specific passes are the kernels below.
#include <chrono>
#include <map>
#include <cub/cub.cuh>
#include <cub/device/device_merge.cuh>

#include <algorithm>
#include <cstdlib>
#include <stdexcept>

#include "common.cuh"
#include "graph_store.h"

namespace dgnn {

using cuda::DevArray;

namespace {

constexpr int kT = 256;

__global__ void k_make_keys(int64_t n, const int32_t* __restrict__ src,
                            const int32_t* __restrict__ dst, int32_t num_nodes,
                            uint64_t* __restrict__ keys, int32_t* __restrict__ flag) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t s = src[i], d = dst[i];
    if (s < 0 || s >= num_nodes || d < 0 || d >= num_nodes) atomicOr(flag, 1);
    keys[i] = (static_cast<uint64_t>(static_cast<uint32_t>(s)) << 32) | static_cast<uint32_t>(d);
  }
}

__global__ void k_adjacent_dup(int64_t n, const uint64_t* __restrict__ keys, int32_t* flag) {
  for (int64_t i = 1 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (keys[i] == keys[i - 1]) atomicOr(flag, 2);
}

__device__ __forceinline__ bool bsearch_u64(const uint64_t* __restrict__ a, int64_t n, uint64_t k) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < k) lo = mid + 1; else hi = mid;
  }
  return lo < n && a[lo] == k;
}

// keep[i] = (a[i] found in b) == want_found
__global__ void k_mark(int64_t na, const uint64_t* __restrict__ a, int64_t nb,
                       const uint64_t* __restrict__ b, int want_found, uint8_t* __restrict__ keep) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < na;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    keep[i] = bsearch_u64(b, nb, a[i]) == (want_found != 0);
}

// keep[pos] = 0 for every key of `d` present in the sorted array `a`
// (binary search per key of the small array, not per key of the big one)
__global__ void k_unmark_present(int64_t nd, const uint64_t* __restrict__ d, int64_t na,
                                 const uint64_t* __restrict__ a, int swap, uint8_t* __restrict__ keep) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nd;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t k = swap ? (d[i] << 32) | (d[i] >> 32) : d[i];
    int64_t lo = 0, hi = na;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (a[mid] < k) lo = mid + 1;
      else hi = mid;
    }
    if (lo < na && a[lo] == k) keep[lo] = 0;
  }
}

__global__ void k_low32(int64_t n, const uint64_t* __restrict__ keys, int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<int32_t>(keys[i] & 0xffffffffu);
}

// CSR of keys sorted by their high half in one pass: idx[i] = low half, and
// each row boundary writes the row pointers of the rows it closes (every
// ptr[v], v in [0, n], written exactly once; no atomics, no scan).
__global__ void k_csr_from_sorted(int64_t E, int32_t n, const uint64_t* __restrict__ keys,
                                  int64_t* __restrict__ ptr, int32_t* __restrict__ idx) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i <= E;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t cur = i < E ? static_cast<int64_t>(keys[i] >> 32) : n;
    const int64_t prev = i > 0 ? static_cast<int64_t>(keys[i - 1] >> 32) : -1;
    for (int64_t v = prev + 1; v <= cur; ++v) ptr[v] = i;
    if (i < E) idx[i] = static_cast<int32_t>(keys[i] & 0xffffffffu);
  }
}

__global__ void k_swap_halves(int64_t n, const uint64_t* __restrict__ in, uint64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = (in[i] << 32) | (in[i] >> 32);
}

// changed[u] = any component of row u differs exactly (ref src/snapshot.cpp:113-115)
__global__ void k_row_differs(int32_t n, int32_t d, const float* __restrict__ a,
                              const float* __restrict__ b, uint8_t* __restrict__ flags) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t u = warp; u < n; u += nwarps) {
    int diff = 0;
    for (int j = lane; j < d; j += 32) diff |= a[u * d + j] != b[u * d + j];
    diff = __any_sync(0xffffffffu, diff);
    if (lane == 0) flags[u] = diff ? 1 : 0;
  }
}

__global__ void k_iota(int32_t n, int32_t* out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<int32_t>(i);
}

__global__ void k_out_degree_of(int64_t m, const int32_t* __restrict__ nodes,
                                const int64_t* __restrict__ out_ptr, int64_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    cnt[i] = out_ptr[nodes[i] + 1] - out_ptr[nodes[i]];
}

// out-edges of the listed nodes, appended at offsets (exclusive scan of degrees)
__global__ void k_expand(int64_t m, const int32_t* __restrict__ nodes,
                         const int64_t* __restrict__ out_ptr, const int32_t* __restrict__ out_dst,
                         const int64_t* __restrict__ offs, uint64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t u = nodes[i];
    const uint64_t hi = static_cast<uint64_t>(static_cast<uint32_t>(u)) << 32;
    int64_t o = offs[i];
    for (int64_t e = out_ptr[u]; e < out_ptr[u + 1]; ++e) out[o++] = hi | static_cast<uint32_t>(out_dst[e]);
  }
}

// composite key for the dst-grouped layout: dst << 33 | is_ins << 32 | src
__global__ void k_composite(int64_t n, const uint64_t* __restrict__ keys, uint64_t is_ins,
                            uint64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t s = keys[i] >> 32, d = keys[i] & 0xffffffffu;
    out[i] = (d << 33) | (is_ins << 32) | s;
  }
}

// Checked build: CSR invariants of one direction (row pointers from 0 to E,
// non-decreasing; indices in range and strictly ascending within a row).
__global__ void k_check_csr(int32_t n, int64_t E, const int64_t* __restrict__ ptr,
                            const int32_t* __restrict__ idx, int32_t* __restrict__ bad) {
  for (int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; v < n;
       v += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = ptr[v], e = ptr[v + 1];
    if (v == 0 && b != 0) atomicOr(bad, 1);
    if (v == n - 1 && e != E) atomicOr(bad, 2);
    if (e < b) atomicOr(bad, 4);
    for (int64_t i = b; i < e && i < E; ++i) {
      if (idx[i] < 0 || idx[i] >= n) atomicOr(bad, 8);
      if (i > b && idx[i] <= idx[i - 1]) atomicOr(bad, 16);
    }
  }
}

// source-grouped twin of k_composite: source, then deletions before
// insertions, then destination
__global__ void k_composite_t(int64_t n, const uint64_t* __restrict__ keys, uint64_t is_ins,
                              uint64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t s = keys[i] >> 32, d = keys[i] & 0xffffffffu;
    out[i] = (s << 33) | (is_ins << 32) | d;
  }
}

__global__ void k_split_composite(int64_t n, const uint64_t* __restrict__ comp,
                                  int32_t* __restrict__ dsts, int32_t* __restrict__ ent) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t c = comp[i];
    dsts[i] = static_cast<int32_t>(c >> 33);
    const int32_t s = static_cast<int32_t>(c & 0xffffffffu);
    ent[i] = (c >> 32) & 1u ? s : ~s;
  }
}

__global__ void k_count_heads(int64_t n, const uint64_t* __restrict__ keys,
                              unsigned long long* __restrict__ out) {
  unsigned long long c = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    c += (i == 0 || (keys[i] >> 32) != (keys[i - 1] >> 32)) ? 1 : 0;
  if (c) atomicAdd(out, c);
}

__global__ void k_scatter_rows(int64_t m, int32_t d, const int32_t* __restrict__ nodes,
                               const float* __restrict__ rows, float* __restrict__ feats) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m * d;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / d;
    feats[static_cast<int64_t>(nodes[r]) * d + (i - r * d)] = rows[i];
  }
}

__global__ void k_gather_rows(int64_t m, int32_t d, const int32_t* __restrict__ nodes,
                              const float* __restrict__ feats, float* __restrict__ rows) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m * d;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / d;
    rows[i] = feats[static_cast<int64_t>(nodes[r]) * d + (i - r * d)];
  }
}

__device__ __forceinline__ int64_t find_sorted(const int32_t* a, int64_t n, int32_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo < n && a[lo] == x ? lo : -1;
}

// Per delta-SpMM entry (one thread; a hub destination can hold 10^4+
// entries, so rows are not serialised): ent_c = ent re-indexed for the
// compact block [F_{t-1}[changed] - F_t[changed] | F_t[changed]]. A
// feature-changed source u present as a deletion AND an insertion of the same
// destination (a persisting out-edge of a changed node — most of a feature
// delta's entries) becomes ONE deletion of its negated difference row
// (~(N + pos)): the row gains F_t[u] - F_{t-1}[u] from one gather instead of
// two, and the insertion entry is dropped (keep = 0). An unpaired changed
// insertion reads F_t[u] from the compact block (N + pos); an unpaired
// changed deletion keeps its plain index (F_{t-1} matrix). Row order is
// unchanged: deletions, then insertions, each ascending by source.
__global__ void k_remap_compact_ent(int64_t ne, int32_t n_rows, const int32_t* __restrict__ row_ptr,
                                    const int32_t* __restrict__ ent, int64_t n_changed,
                                    const int32_t* __restrict__ changed, int32_t num_nodes,
                                    int32_t* __restrict__ ent_c, int32_t* __restrict__ keep) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < ne;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t x = ent[i];
    const bool del = x < 0;
    const int32_t s = del ? ~x : x;
    const int64_t pos = find_sorted(changed, n_changed, s);
    int32_t out = x, k1 = 1;
    if (pos >= 0) {
      // row of entry i: last r with row_ptr[r] <= i
      int32_t lo = 0, hi = n_rows;
      while (hi - lo > 1) {
        const int32_t mid = (lo + hi) >> 1;
        if (row_ptr[mid] <= i) lo = mid; else hi = mid;
      }
      const int32_t b = row_ptr[lo], e = row_ptr[lo + 1];
      // first insertion of the row (deletions < 0 come first)
      int32_t kl = b, kh = e;
      while (kl < kh) {
        const int32_t mid = (kl + kh) >> 1;
        if (ent[mid] < 0) kl = mid + 1; else kh = mid;
      }
      // the opposite side, ascending by source
      int32_t l2 = del ? kl : b, h2 = del ? e : kl;
      const int32_t end = h2;
      while (l2 < h2) {
        const int32_t mid = (l2 + h2) >> 1;
        const int32_t v = del ? ent[mid] : ~ent[mid];
        if (v < s) l2 = mid + 1; else h2 = mid;
      }
      const bool paired = l2 < end && (del ? ent[l2] : ~ent[l2]) == s;
      const int32_t ci = num_nodes + static_cast<int32_t>(pos);
      if (del) {
        if (paired) out = ~ci;  // negated difference row
      } else if (paired) {
        k1 = 0;  // folded into the deletion entry
      } else {
        out = ci;
      }
    }
    ent_c[i] = out;
    keep[i] = k1;
  }
}

// row_ptr_c[r] = kept entries before row r (scan of keep at the row start)
__global__ void k_row_ptr_c(int32_t n_rows, const int32_t* __restrict__ row_ptr,
                            const int32_t* __restrict__ scan, int32_t* __restrict__ row_ptr_c) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r <= n_rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x)
    row_ptr_c[r] = scan[row_ptr[r]];
}

__global__ void k_nonzero_u8(int64_t n, const int32_t* __restrict__ x, uint8_t* __restrict__ f) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    f[i] = x[i] != 0;
}

// dst[i] -= src[i]
__global__ void k_sub_inplace(int64_t n, float* __restrict__ dst, const float* __restrict__ src) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] -= src[i];
}

int grid_for(int64_t n) { return cuda::wave_grid(n, kT, 8); }

// DGNN_BUILD_PROF=1: host-side phase timing of the device graph build (each
// mark synchronises the build stream), printed by release_build_state
struct BuildProf {
  bool on = std::getenv("DGNN_BUILD_PROF") != nullptr;
  std::map<std::string, double> ms;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* phase, cudaStream_t st) {
    if (!on) return;
    cudaStreamSynchronize(st);
    const auto now = std::chrono::steady_clock::now();
    ms[phase] += std::chrono::duration<double, std::milli>(now - t).count();
    t = now;
  }
  void restart() { t = std::chrono::steady_clock::now(); }
};
BuildProf& build_prof() {
  static BuildProf p;
  return p;
}

// Thin CUB wrappers with a growable temp buffer.
struct Cub {
  cudaStream_t st;
  DevArray<uint8_t> tmp;
  explicit Cub(cudaStream_t s) : st(s) {}
  void* get(size_t bytes) {
    if (bytes > tmp.size()) tmp = DevArray<uint8_t>(bytes + (bytes >> 2) + 256, st);
    return tmp.get();
  }
  void sort(const uint64_t* in, uint64_t* out, int64_t n, int end_bit = 64) {
    if (n == 0) return;
    size_t b = 0;
    DGNN_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, b, in, out, n, 0, end_bit, st));
    DGNN_CUDA(cub::DeviceRadixSort::SortKeys(get(b), b, in, out, n, 0, end_bit, st));
  }
  template <typename T>
  int64_t select_flagged(const T* in, const uint8_t* flags, T* out, int64_t n) {
    if (n == 0) return 0;
    DevArray<int64_t> cnt(1, st);
    size_t b = 0;
    DGNN_CUDA(cub::DeviceSelect::Flagged(nullptr, b, in, flags, out, cnt.get(), n, st));
    DGNN_CUDA(cub::DeviceSelect::Flagged(get(b), b, in, flags, out, cnt.get(), n, st));
    return read(cnt.get());
  }
  int64_t unique(const uint64_t* in, uint64_t* out, int64_t n) {
    if (n == 0) return 0;
    DevArray<int64_t> cnt(1, st);
    size_t b = 0;
    DGNN_CUDA(cub::DeviceSelect::Unique(nullptr, b, in, out, cnt.get(), n, st));
    DGNN_CUDA(cub::DeviceSelect::Unique(get(b), b, in, out, cnt.get(), n, st));
    return read(cnt.get());
  }
  template <typename TI, typename TO>
  void exclusive_sum(const TI* in, TO* out, int64_t n) {
    if (n == 0) return;
    size_t b = 0;
    DGNN_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, b, in, out, n, st));
    DGNN_CUDA(cub::DeviceScan::ExclusiveSum(get(b), b, in, out, n, st));
  }
  void merge(const uint64_t* a, int64_t na, const uint64_t* b, int64_t nb, uint64_t* out) {
    if (na + nb == 0) return;
    if (na == 0 || nb == 0) {
      DGNN_CUDA(cudaMemcpyAsync(out, na ? a : b, sizeof(uint64_t) * (na + nb), cudaMemcpyDeviceToDevice, st));
      return;
    }
    // DeviceMerge counts in int: refuse rather than truncate
    if (na + nb > static_cast<int64_t>(INT32_MAX))
      throw std::invalid_argument("incremental snapshot build supports up to 2^31-1 edges");
    size_t bytes = 0;
    DGNN_CUDA(cub::DeviceMerge::MergeKeys(nullptr, bytes, a, static_cast<int>(na), b,
                                          static_cast<int>(nb), out, ::cuda::std::less<>{}, st));
    DGNN_CUDA(cub::DeviceMerge::MergeKeys(get(bytes), bytes, a, static_cast<int>(na), b,
                                          static_cast<int>(nb), out, ::cuda::std::less<>{}, st));
  }
  int64_t rle(const int32_t* in, int32_t* uniq, int32_t* counts, int64_t n) {
    if (n == 0) return 0;
    DevArray<int64_t> cnt(1, st);
    size_t b = 0;
    DGNN_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, b, in, uniq, counts, cnt.get(), n, st));
    DGNN_CUDA(cub::DeviceRunLengthEncode::Encode(get(b), b, in, uniq, counts, cnt.get(), n, st));
    return read(cnt.get());
  }
  int64_t read(const int64_t* d) {
    int64_t h = 0;
    DGNN_CUDA(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, st));
    DGNN_CUDA(cudaStreamSynchronize(st));
    return h;
  }
};

template <typename T>
DevArray<T> upload(const T* host, int64_t n, cudaStream_t st) {
  DevArray<T> d(static_cast<size_t>(n), st);
  if (n > 0) DGNN_CUDA(cudaMemcpyAsync(d.get(), host, sizeof(T) * n, cudaMemcpyHostToDevice, st));
  return d;
}

int32_t read_flag(DevArray<int32_t>& f, cudaStream_t st) {
  int32_t h = 0;
  DGNN_CUDA(cudaMemcpyAsync(&h, f.get(), sizeof(h), cudaMemcpyDeviceToHost, st));
  DGNN_CUDA(cudaStreamSynchronize(st));
  return h;
}

// Sorted unique keys from an edge list; reference Snapshot ctor checks.
DevArray<uint64_t> sorted_edge_keys(const int32_t* src_h, const int32_t* dst_h, int64_t n,
                                    int32_t num_nodes, Cub& cub, bool reject_dups) {
  cudaStream_t st = cub.st;
  DevArray<int32_t> s = upload(src_h, n, st), d = upload(dst_h, n, st);
  DevArray<uint64_t> raw(n, st), keys(n, st);
  DevArray<int32_t> flag(1, st);
  flag.zero(st);
  if (n > 0) {
    DGNN_LAUNCH(k_make_keys, grid_for(n), kT, 0, st, n, s.get(), d.get(), num_nodes, raw.get(), flag.get());
    cub.sort(raw.get(), keys.get(), n);
    if (reject_dups) DGNN_LAUNCH(k_adjacent_dup, grid_for(n), kT, 0, st, n, keys.get(), flag.get());
  }
  const int32_t f = read_flag(flag, st);
  if (f & 1) throw std::invalid_argument("edge endpoint out of range");
  if (f & 2) throw std::invalid_argument("duplicate edge in snapshot");
  return keys;
}

}  // namespace

void copy_to_host(void* dst, const void* src, size_t bytes, cudaStream_t stream) {
  if (bytes == 0) return;
  DGNN_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, stream));
  DGNN_CUDA(cudaStreamSynchronize(stream));
}

DeviceGraph::DeviceGraph(int32_t num_nodes, int32_t feature_dim, cudaStream_t stream)
    : n_(num_nodes), d_(feature_dim), stream_(stream) {
  if (num_nodes <= 0) throw std::invalid_argument("snapshot needs at least one node");
  if (feature_dim <= 0) throw std::invalid_argument("feature_dim must be positive");
  double gb = 24.0;
  if (const char* e = std::getenv("DGNN_FEATURE_BUDGET_GB")) gb = std::atof(e);
  const double per = 4.0 * num_nodes * feature_dim;
  const double slots = gb * 1e9 / per;
  max_slots_ = slots >= 1e6 ? 1000000 : (slots < 2 ? 2 : static_cast<int32_t>(slots));
}

DeviceGraph::~DeviceGraph() {
  // slot buffers are freed on the graph stream: let readers on other streams finish
  cudaDeviceSynchronize();
}

// ---------------------------------------------------------------- feature versions
FeatSlot::~FeatSlot() {
  if (ready) cudaEventDestroy(ready);
  for (auto& r : readers) cudaEventDestroy(r.second);
}

FeatLease::FeatLease(std::shared_ptr<FeatSlot> slot, cudaStream_t stream)
    : slot_(std::move(slot)), stream_(stream) {}

FeatLease::~FeatLease() {
  // the slot may be rewritten once this stream's reads are done
  for (auto& r : slot_->readers) {
    if (r.first == stream_) {
      cudaEventRecord(r.second, stream_);
      return;
    }
  }
  cudaEvent_t e;
  if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess) {
    cudaEventRecord(e, stream_);
    slot_->readers.emplace_back(stream_, e);
  }
}

void DeviceGraph::order_after_write(const FeatSlot& s, cudaStream_t stream) const {
  if (s.ready && s.writer != stream) DGNN_CUDA(cudaStreamWaitEvent(stream, s.ready, 0));
}

std::shared_ptr<FeatSlot> DeviceGraph::free_slot(cudaStream_t stream) const {
  const int32_t resident = static_cast<int32_t>(slots_.size()) - 1;  // slots_[0] is snapshot 0
  std::shared_ptr<FeatSlot> victim;
  if (resident >= max_slots_) {
    for (size_t i = 1; i < slots_.size(); ++i) {
      const auto& s = slots_[i];
      if (s.use_count() != 1) continue;  // leased
      if (!victim || s->stamp < victim->stamp) victim = s;
    }
  }
  if (!victim) {  // below the budget, or every slot leased: grow
    victim = std::make_shared<FeatSlot>();
    victim->buf = DevArray<float>(static_cast<size_t>(n_) * d_, stream_);
    DGNN_CUDA(cudaEventCreateWithFlags(&victim->ready, cudaEventDisableTiming));
    slots_.push_back(victim);
    // the allocation is ordered on the graph stream
    DGNN_CUDA(cudaEventRecord(victim->ready, stream_));
    victim->writer = stream_;
  }
  order_after_write(*victim, stream);
  for (auto& r : victim->readers) DGNN_CUDA(cudaStreamWaitEvent(stream, r.second, 0));
  victim->t = -1;
  return victim;
}

FeatRef DeviceGraph::features(int32_t t, cudaStream_t stream) const {
  if (t < 0 || t >= length()) throw std::out_of_range("snapshot index out of range");
  if (t < first_ || t > last_) throw std::out_of_range("snapshot not retained in this graph store");
  std::shared_ptr<FeatSlot> hit, base;
  for (const auto& s : slots_) {
    if (s->t == t) hit = s;
    if (s->t >= 0 && s->t <= t && (!base || s->t > base->t)) base = s;
  }
  if (!hit) {
    // nearest version <= t, then the row patches of base.t+1 .. t in order
    auto src = std::make_shared<const FeatLease>(base, stream);  // pinned while copying
    hit = free_slot(stream);
    order_after_write(*base, stream);
    const int64_t nf = static_cast<int64_t>(n_) * d_;
    DGNN_CUDA(cudaMemcpyAsync(hit->buf.get(), base->buf.get(), sizeof(float) * nf,
                              cudaMemcpyDeviceToDevice, stream));
    for (int32_t k = base->t + 1; k <= t; ++k) {
      const DevDelta& dd = deltas_[k];
      if (dd.n_changed > 0)
        DGNN_LAUNCH(k_scatter_rows, grid_for(dd.n_changed * d_), kT, 0, stream, dd.n_changed, d_,
                    dd.changed.get(), dd.compact.get() + dd.n_changed * d_, hit->buf.get());
    }
    hit->t = t;
    hit->writer = stream;
    DGNN_CUDA(cudaEventRecord(hit->ready, stream));
    ++materialisations_;
  } else {
    order_after_write(*hit, stream);
  }
  hit->stamp = ++clock_;
  return std::make_shared<const FeatLease>(hit, stream);
}

const DevSnapshot& DeviceGraph::snapshot(int32_t t) const {
  if (t < 0 || t >= length()) throw std::out_of_range("snapshot index out of range");
  if (t < first_ || t > last_) throw std::out_of_range("snapshot not retained in this graph store");
  return snaps_[t];
}

const DevDelta& DeviceGraph::delta(int32_t t) const {
  if (!(t >= 1 && t < length())) throw std::invalid_argument("delta index out of range");
  if (t < first_ || t > last_) throw std::out_of_range("delta not retained in this graph store");
  return deltas_[t];
}

void DeviceGraph::retain(int32_t t_first, int32_t t_last) {
  if (!(t_first >= first_ && t_first <= t_last && t_last <= last_ && t_last < length()))
    throw std::invalid_argument("retain: range outside the retained snapshots");
  if (t_first > first_) {
    // the features of t_first as a resident base version (leased: never evicted)
    retained_base_ = features(t_first, stream_);
    DGNN_CUDA(cudaStreamSynchronize(stream_));
    for (const auto& sl : slots_) {
      if (sl->t >= 0 && sl->t < t_first && sl.use_count() == 1) {  // versions before the range
        sl->t = -1;
        if (sl == slots_[0]) sl->buf.reset();  // snapshot 0's matrix is no base any more
      }
    }
  }
  for (int32_t t = 0; t < length(); ++t) {
    if (t >= t_first && t <= t_last) continue;
    snaps_[t] = DevSnapshot{};
    if (t >= 1) deltas_[t] = DevDelta{};
  }
  first_ = t_first;
  last_ = t_last;
  DGNN_CUDA(cudaStreamSynchronize(stream_));
  cuda::release_stream_blocks(stream_);
}

int64_t DeviceGraph::device_bytes() const {
  int64_t b = 0;
  for (const auto& s : snaps_)
    b += s.in_ptr.bytes() + s.out_ptr.bytes() + s.in_src.bytes() + s.out_dst.bytes();
  for (const auto& d : deltas_)
    b += d.del.bytes() + d.ins.bytes() + d.changed.bytes() + d.rows.bytes() + d.row_ptr.bytes() +
         d.ent.bytes() + d.ent_c.bytes() + d.row_ptr_c.bytes() + d.compact.bytes();
  for (const auto& s : slots_) b += s->buf.bytes();
  return b;
}

void DeviceGraph::add_snapshot(const int32_t* src, const int32_t* dst, int64_t num_edges,
                               const float* feats) {
  cuda::release_stream_blocks(stream_);
  ensure_build_keys();  // previous snapshot's keys for extract_delta
  Cub cub(stream_);
  DevArray<uint64_t> keys = sorted_edge_keys(src, dst, num_edges, n_, cub, true);
  const int64_t nf = static_cast<int64_t>(n_) * d_;
  if (snaps_.empty()) {
    auto s0 = std::make_shared<FeatSlot>();
    s0->buf = upload(feats, nf, stream_);
    DGNN_CUDA(cudaEventCreateWithFlags(&s0->ready, cudaEventDisableTiming));
    DGNN_CUDA(cudaEventRecord(s0->ready, stream_));
    s0->writer = stream_;
    s0->t = 0;
    slots_.push_back(s0);
    finish_snapshot(std::move(keys), nullptr, s0->buf.get());
    return;
  }
  // a full snapshot t >= 1 (Snapshot ctor per step): its features become the
  // exact row patch against t-1
  const int32_t t = length();
  FeatRef prev = features(t - 1, stream_);
  std::shared_ptr<FeatSlot> cur = free_slot(stream_);
  DGNN_CUDA(cudaMemcpyAsync(cur->buf.get(), feats, sizeof(float) * nf, cudaMemcpyHostToDevice, stream_));
  finish_snapshot(std::move(keys), prev->get(), cur->buf.get());
  cur->t = t;
  cur->writer = stream_;
  cur->stamp = ++clock_;
  DGNN_CUDA(cudaEventRecord(cur->ready, stream_));
}

void DeviceGraph::add_delta(const int32_t* del_src, const int32_t* del_dst, int64_t n_del,
                            const int32_t* ins_src, const int32_t* ins_dst, int64_t n_ins,
                            const int32_t* changed_nodes, int64_t n_changed,
                            const float* changed_feats) {
  if (snaps_.empty()) throw std::invalid_argument("add_delta needs a previous snapshot");
  cudaStream_t st = stream_;
  // the previous build step's temporaries (sizes drift per snapshot) go back
  // to the pool instead of accumulating in the per-size free lists
  build_prof().restart();
  cuda::release_stream_blocks(st);
  ensure_build_keys();
  Cub cub(st);
  DevArray<uint64_t> del = sorted_edge_keys(del_src, del_dst, n_del, n_, cub, false);
  DevArray<uint64_t> ins = sorted_edge_keys(ins_src, ins_dst, n_ins, n_, cub, true);
  build_prof().mark("upload+sort delta keys", st);
  const int64_t E0 = static_cast<int64_t>(curr_keys_.size());
  // Incremental snapshot build: the work scales with |D| + |I| plus two
  // linear select / merge passes, not with sorts or searches over E.
  // kept = prev \ D: one binary search per deletion into prev
  DevArray<uint8_t> keep(E0, st);
  DevArray<uint64_t> kept(E0, st);
  int64_t nk = E0;
  if (E0 > 0) {
    DGNN_CUDA(cudaMemsetAsync(keep.get(), 1, E0, st));
    if (n_del) DGNN_LAUNCH(k_unmark_present, grid_for(n_del), kT, 0, st, n_del, del.get(), E0, curr_keys_.get(), 0, keep.get());
    nk = cub.select_flagged(curr_keys_.get(), keep.get(), kept.get(), E0);
  }
  // I' = I \ kept, so that merge(kept, I') is the set union (src/snapshot.cpp:145-148)
  DevArray<uint64_t> ins_new(n_ins, st);
  int64_t ni = 0;
  if (n_ins) {
    DevArray<uint8_t> f(n_ins, st);
    DGNN_LAUNCH(k_mark, grid_for(n_ins), kT, 0, st, n_ins, ins.get(), nk, kept.get(), 0, f.get());
    ni = cub.select_flagged(ins.get(), f.get(), ins_new.get(), n_ins);
  }
  const int64_t E1 = nk + ni;
  DevArray<uint64_t> exact(E1, st);
  cub.merge(kept.get(), nk, ins_new.get(), ni, exact.get());
  kept.reset();
  // (dst, src) order: prev's swapped keys minus D, merged with sorted swap(I')
  DevArray<uint64_t> sw_new(E1, st);
  {
    DevArray<uint64_t> sw_kept(E0, st);
    int64_t nsk = E0;
    if (E0 > 0) {
      DGNN_CUDA(cudaMemsetAsync(keep.get(), 1, E0, st));
      if (n_del) DGNN_LAUNCH(k_unmark_present, grid_for(n_del), kT, 0, st, n_del, del.get(), E0, curr_swapped_.get(), 1, keep.get());
      nsk = cub.select_flagged(curr_swapped_.get(), keep.get(), sw_kept.get(), E0);
    }
    DevArray<uint64_t> swi(ni, st), swi_sorted(ni, st);
    if (ni) {
      DGNN_LAUNCH(k_swap_halves, grid_for(ni), kT, 0, st, ni, ins_new.get(), swi.get());
      cub.sort(swi.get(), swi_sorted.get(), ni);
    }
    if (nsk + ni != E1) throw std::runtime_error("graph store: inconsistent incremental build");
    cub.merge(sw_kept.get(), nsk, swi_sorted.get(), ni, sw_new.get());
  }
  keep.reset();
  build_prof().mark("merge (src,dst) and (dst,src) keys", st);
  // exact structural change for extract_delta: removed = (prev ∩ D) \ I, added = I \ prev
  StructDiff diff;
  {
    diff.removed = DevArray<uint64_t>(n_del, st);
    if (n_del) {
      DevArray<uint8_t> in_prev(n_del, st), not_ins(n_del, st);
      DevArray<uint64_t> tmp(n_del, st), tmp2(n_del, st);
      DGNN_LAUNCH(k_mark, grid_for(n_del), kT, 0, st, n_del, del.get(), E0, curr_keys_.get(), 1, in_prev.get());
      const int64_t np = cub.select_flagged(del.get(), in_prev.get(), tmp.get(), n_del);
      if (np) {
        DGNN_LAUNCH(k_mark, grid_for(np), kT, 0, st, np, tmp.get(), n_ins, ins.get(), 0, not_ins.get());
        const int64_t nr = cub.select_flagged(tmp.get(), not_ins.get(), tmp2.get(), np);
        diff.n_removed = cub.unique(tmp2.get(), diff.removed.get(), nr);  // D may repeat keys
      }
    }
    diff.added = DevArray<uint64_t>(n_ins, st);
    if (n_ins) {
      DevArray<uint8_t> f(n_ins, st);
      DGNN_LAUNCH(k_mark, grid_for(n_ins), kT, 0, st, n_ins, ins.get(), E0, curr_keys_.get(), 0, f.get());
      diff.n_added = cub.select_flagged(ins.get(), f.get(), diff.added.get(), n_ins);
    }
  }
  build_prof().mark("structural diff", st);
  // features: prev rows with the changed rows replaced
  const int64_t nf = static_cast<int64_t>(n_) * d_;
  const int32_t t = length();
  FeatRef prev = features(t - 1, st);
  std::shared_ptr<FeatSlot> cur = free_slot(st);
  DGNN_CUDA(cudaMemcpyAsync(cur->buf.get(), prev->get(), sizeof(float) * nf, cudaMemcpyDeviceToDevice, st));
  if (n_changed > 0) {
    DevArray<int32_t> nodes = upload(changed_nodes, n_changed, st);
    DevArray<float> rows = upload(changed_feats, n_changed * d_, st);
    DGNN_LAUNCH(k_scatter_rows, grid_for(n_changed * d_), kT, 0, st, n_changed, d_, nodes.get(),
                rows.get(), cur->buf.get());
  }
  build_prof().mark("features", st);
  finish_snapshot(std::move(exact), prev->get(), cur->buf.get(), std::move(sw_new), &diff);
  cur->t = t;
  cur->writer = st;
  cur->stamp = ++clock_;
  DGNN_CUDA(cudaEventRecord(cur->ready, st));
}

namespace {
// (src,dst) keys of a snapshot from its out-CSR, (dst,src) keys from its in-CSR
__global__ void k_csr_keys(int32_t n, const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                           uint64_t* __restrict__ out) {
  const int64_t warp = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t u = warp; u < n; u += nw)
    for (int64_t e = ptr[u] + lane; e < ptr[u + 1]; e += 32)
      out[e] = (static_cast<uint64_t>(u) << 32) | static_cast<uint32_t>(idx[e]);
}
}  // namespace

void DeviceGraph::ensure_build_keys() {
  if (snaps_.empty()) return;
  const DevSnapshot& s = snaps_.back();
  const int64_t E = s.num_edges;
  if (static_cast<int64_t>(curr_keys_.size()) == E && static_cast<int64_t>(curr_swapped_.size()) == E) return;
  curr_keys_ = DevArray<uint64_t>(E, stream_);
  curr_swapped_ = DevArray<uint64_t>(E, stream_);
  if (E > 0) {
    DGNN_LAUNCH(k_csr_keys, cuda::wave_grid(static_cast<int64_t>(n_) * 32, kT, 8), kT, 0, stream_, n_,
                s.out_ptr.get(), s.out_dst.get(), curr_keys_.get());
    DGNN_LAUNCH(k_csr_keys, cuda::wave_grid(static_cast<int64_t>(n_) * 32, kT, 8), kT, 0, stream_, n_,
                s.in_ptr.get(), s.in_src.get(), curr_swapped_.get());
  }
}

void DeviceGraph::release_build_state() {
  DGNN_CUDA(cudaStreamSynchronize(stream_));
  if (build_prof().on) {
    for (const auto& [k, v] : build_prof().ms) std::fprintf(stderr, "[dgnn build] %-40s %9.1f ms\n", k.c_str(), v);
    build_prof().ms.clear();
  }
  curr_keys_.reset();
  curr_swapped_.reset();
  prev_keys_.reset();
  cuda::release_stream_blocks(stream_);
}

DevSnapshot csr_from_keys(const uint64_t* keys, int64_t E, int32_t n, cudaStream_t st,
                          const uint64_t* swapped_sorted, DevArray<uint64_t>* swapped_out) {
  Cub cub(st);
  DevSnapshot s;
  s.num_edges = E;
  // out-CSR: keys already sorted by (src, dst)
  s.out_ptr = DevArray<int64_t>(n + 1, st);
  s.out_dst = DevArray<int32_t>(E, st);
  DGNN_LAUNCH(k_csr_from_sorted, grid_for(E + 1), kT, 0, st, E, n, keys, s.out_ptr.get(), s.out_dst.get());
  // in-CSR: sort by (dst, src)
  s.in_ptr = DevArray<int64_t>(n + 1, st);
  s.in_src = DevArray<int32_t>(E, st);
  if (E > 0) {
    DevArray<uint64_t> sw_sorted;
    const uint64_t* swk = swapped_sorted;
    if (swk == nullptr) {
      DevArray<uint64_t> sw(E, st);
      sw_sorted = DevArray<uint64_t>(E, st);
      DGNN_LAUNCH(k_swap_halves, grid_for(E), kT, 0, st, E, keys, sw.get());
      cub.sort(sw.get(), sw_sorted.get(), E);
      swk = sw_sorted.get();
    }
    DGNN_LAUNCH(k_csr_from_sorted, grid_for(E + 1), kT, 0, st, E, n, swk, s.in_ptr.get(), s.in_src.get());
    if (swapped_out && swapped_sorted == nullptr) *swapped_out = std::move(sw_sorted);
  } else {
    DGNN_LAUNCH(k_csr_from_sorted, 1, kT, 0, st, int64_t{0}, n, static_cast<const uint64_t*>(nullptr), s.in_ptr.get(), s.in_src.get());
  }
  return s;
}

void DeviceGraph::finish_snapshot(DevArray<uint64_t> keys, const float* prev_feats,
                                  const float* feats, DevArray<uint64_t> swapped,
                                  const StructDiff* diff) {
  const int64_t E = static_cast<int64_t>(keys.size());
  if (static_cast<int64_t>(swapped.size()) == E && E > 0) {
    snaps_.push_back(csr_from_keys(keys.get(), E, n_, stream_, swapped.get()));
  } else {
    swapped.reset();
    snaps_.push_back(csr_from_keys(keys.get(), E, n_, stream_, nullptr, &swapped));
  }
  build_prof().mark("CSRs", stream_);
  deltas_.emplace_back();
  prev_keys_ = std::move(curr_keys_);
  curr_keys_ = std::move(keys);
  curr_swapped_ = std::move(swapped);
  if (snaps_.size() >= 2) build_delta(static_cast<int32_t>(snaps_.size()) - 1, prev_feats, feats, diff);
  build_prof().mark("extract_delta + delta layouts", stream_);
  prev_keys_.reset();
#if defined(DGNN_CHECKED) && DGNN_CHECKED
  {
    const DevSnapshot& S = snaps_.back();
    DevArray<int32_t> bad(1, stream_);
    bad.zero(stream_);
    if (n_ > 0) {
      DGNN_LAUNCH(k_check_csr, grid_for(n_), kT, 0, stream_, n_, S.num_edges, S.in_ptr.get(), S.in_src.get(),
                  bad.get());
      DGNN_LAUNCH(k_check_csr, grid_for(n_), kT, 0, stream_, n_, S.num_edges, S.out_ptr.get(),
                  S.out_dst.get(), bad.get());
    }
    const int32_t f = read_flag(bad, stream_);
    if (f) throw std::runtime_error("checked build: CSR invariant violated (flags " + std::to_string(f) + ")");
  }
#endif
}

void DeviceGraph::build_delta(int32_t t, const float* prev_feats, const float* feats,
                              const StructDiff* diff) {
  cudaStream_t st = stream_;
  Cub cub(st);
  const DevSnapshot& P = snaps_[t - 1];
  const DevSnapshot& Cs = snaps_[t];
  const int64_t Ep = P.num_edges, Ec = Cs.num_edges;
  DevDelta dd;
  // changed nodes (exact row inequality), ascending
  DevArray<uint8_t> fl(n_, st);
  DGNN_LAUNCH(k_row_differs, cuda::wave_grid(static_cast<int64_t>(n_) * 32, kT, 8), kT, 0, st, n_,
              d_, prev_feats, feats, fl.get());
  DevArray<int32_t> iota(n_, st);
  DGNN_LAUNCH(k_iota, grid_for(n_), kT, 0, st, n_, iota.get());
  DevArray<int32_t> changed(n_, st);
  dd.n_changed = cub.select_flagged(iota.get(), fl.get(), changed.get(), n_);
  dd.changed = DevArray<int32_t>(dd.n_changed, st);
  if (dd.n_changed) {
    DGNN_CUDA(cudaMemcpyAsync(dd.changed.get(), changed.get(), sizeof(int32_t) * dd.n_changed,
                              cudaMemcpyDeviceToDevice, st));
    // [F_{t-1}[changed] - F_t[changed] | F_t[changed]]; the second half is the
    // version patch of t
    dd.compact = DevArray<float>(2 * dd.n_changed * d_, st);
    DGNN_LAUNCH(k_gather_rows, grid_for(dd.n_changed * d_), kT, 0, st, dd.n_changed, d_,
                dd.changed.get(), prev_feats, dd.compact.get());
    DGNN_LAUNCH(k_gather_rows, grid_for(dd.n_changed * d_), kT, 0, st, dd.n_changed, d_,
                dd.changed.get(), feats, dd.compact.get() + dd.n_changed * d_);
    DGNN_LAUNCH(k_sub_inplace, grid_for(dd.n_changed * d_), kT, 0, st, dd.n_changed * d_,
                dd.compact.get(), dd.compact.get() + dd.n_changed * d_);
  }
  // expansion sizes
  auto expansion = [&](const DevSnapshot& S, int64_t* total) {
    DevArray<int64_t> deg(dd.n_changed + 1, st), off(dd.n_changed + 1, st);
    deg.zero(st);
    if (dd.n_changed)
      DGNN_LAUNCH(k_out_degree_of, grid_for(dd.n_changed), kT, 0, st, dd.n_changed,
                  dd.changed.get(), S.out_ptr.get(), deg.get());
    cub.exclusive_sum(deg.get(), off.get(), dd.n_changed + 1);
    *total = cub.read(off.get() + dd.n_changed);
    return off;
  };
  // a \ b (or, from an incremental build, the given exact difference) plus
  // the out-edges of the changed nodes in S
  auto side = [&](const uint64_t* a, int64_t na, const uint64_t* b, int64_t nb,
                  const DevSnapshot& S, int64_t* out_n, const uint64_t* exact_diff, int64_t n_exact) {
    int64_t nexp = 0;
    DevArray<int64_t> off = expansion(S, &nexp);
    const int64_t cap = exact_diff ? n_exact : na;
    DevArray<uint64_t> cat(cap + nexp, st);
    int64_t nd = 0;
    if (exact_diff) {
      nd = n_exact;
      if (nd) DGNN_CUDA(cudaMemcpyAsync(cat.get(), exact_diff, 8 * nd, cudaMemcpyDeviceToDevice, st));
    } else if (na > 0) {
      DevArray<uint8_t> keep(na, st);
      DGNN_LAUNCH(k_mark, grid_for(na), kT, 0, st, na, a, nb, b, 0, keep.get());
      nd = cub.select_flagged(a, keep.get(), cat.get(), na);
    }
    if (nexp > 0)
      DGNN_LAUNCH(k_expand, grid_for(dd.n_changed), kT, 0, st, dd.n_changed, dd.changed.get(),
                  S.out_ptr.get(), S.out_dst.get(), off.get(), cat.get() + nd);
    const int64_t m = nd + nexp;
    DevArray<uint64_t> sorted(m, st), uniq(m, st);
    cub.sort(cat.get(), sorted.get(), m);
    *out_n = cub.unique(sorted.get(), uniq.get(), m);
    DevArray<uint64_t> out(*out_n, st);
    if (*out_n)
      DGNN_CUDA(cudaMemcpyAsync(out.get(), uniq.get(), sizeof(uint64_t) * *out_n,
                                cudaMemcpyDeviceToDevice, st));
    return out;
  };
  dd.del = side(prev_keys_.get(), Ep, curr_keys_.get(), Ec, P, &dd.n_del,
                diff ? diff->removed.get() : nullptr, diff ? diff->n_removed : 0);
  dd.ins = side(curr_keys_.get(), Ec, prev_keys_.get(), Ep, Cs, &dd.n_ins,
                diff ? diff->added.get() : nullptr, diff ? diff->n_added : 0);
  // distinct sources per side
  DevArray<unsigned long long> heads(2, st);
  heads.zero(st);
  if (dd.n_del) DGNN_LAUNCH(k_count_heads, grid_for(dd.n_del), kT, 0, st, dd.n_del, dd.del.get(), heads.get());
  if (dd.n_ins) DGNN_LAUNCH(k_count_heads, grid_for(dd.n_ins), kT, 0, st, dd.n_ins, dd.ins.get(), heads.get() + 1);
  unsigned long long hh[2];
  copy_to_host(hh, heads.get(), sizeof(hh), st);
  dd.u_minus = static_cast<int64_t>(hh[0]);
  dd.u_plus = static_cast<int64_t>(hh[1]);
  // dst-grouped signed layout: deletions then insertions per destination
  const int64_t ne = dd.n_del + dd.n_ins;
  dd.n_ent = ne;
  DevArray<uint64_t> comp(ne, st), comp_sorted(ne, st);
  if (dd.n_del) DGNN_LAUNCH(k_composite, grid_for(dd.n_del), kT, 0, st, dd.n_del, dd.del.get(), 0ull, comp.get());
  if (dd.n_ins)
    DGNN_LAUNCH(k_composite, grid_for(dd.n_ins), kT, 0, st, dd.n_ins, dd.ins.get(), 1ull,
                comp.get() + dd.n_del);
  cub.sort(comp.get(), comp_sorted.get(), ne);
  DevArray<int32_t> dsts(ne, st);
  dd.ent = DevArray<int32_t>(ne, st);
  if (ne) DGNN_LAUNCH(k_split_composite, grid_for(ne), kT, 0, st, ne, comp_sorted.get(), dsts.get(), dd.ent.get());
  DevArray<int32_t> uniq(ne, st), counts(ne + 1, st);
  const int64_t nr = cub.rle(dsts.get(), uniq.get(), counts.get(), ne);
  dd.n_rows = static_cast<int32_t>(nr);
  dd.rows = DevArray<int32_t>(nr, st);
  dd.row_ptr = DevArray<int32_t>(nr + 1, st);
  if (nr) {
    DGNN_CUDA(cudaMemcpyAsync(dd.rows.get(), uniq.get(), sizeof(int32_t) * nr, cudaMemcpyDeviceToDevice, st));
    DGNN_CUDA(cudaMemsetAsync(counts.get() + nr, 0, sizeof(int32_t), st));
  }
  cub.exclusive_sum(counts.get(), dd.row_ptr.get(), nr + 1);
  // sources re-indexed into the compact changed-row block, persisting
  // changed-source pairs folded into one difference-row entry
  {
    DevArray<int32_t> ent_all(ne, st), keep(ne + 1, st), scan(ne + 1, st);
    DGNN_CUDA(cudaMemsetAsync(keep.get() + ne, 0, sizeof(int32_t), st));
    if (ne)
      DGNN_LAUNCH(k_remap_compact_ent, grid_for(ne), kT, 0, st, ne, static_cast<int32_t>(nr),
                  dd.row_ptr.get(), dd.ent.get(), dd.n_changed, dd.changed.get(), n_,
                  ent_all.get(), keep.get());
    cub.exclusive_sum(keep.get(), scan.get(), ne + 1);
    dd.row_ptr_c = DevArray<int32_t>(nr + 1, st);
    DGNN_LAUNCH(k_row_ptr_c, grid_for(nr + 1), kT, 0, st, static_cast<int32_t>(nr),
                dd.row_ptr.get(), scan.get(), dd.row_ptr_c.get());
    DevArray<uint8_t> flag(ne, st);
    if (ne) DGNN_LAUNCH(k_nonzero_u8, grid_for(ne), kT, 0, st, ne, keep.get(), flag.get());
    DevArray<int32_t> tmp(ne, st);
    dd.n_ent_c = cub.select_flagged(ent_all.get(), flag.get(), tmp.get(), ne);
    dd.ent_c = DevArray<int32_t>(dd.n_ent_c, st);
    if (dd.n_ent_c)
      DGNN_CUDA(cudaMemcpyAsync(dd.ent_c.get(), tmp.get(), sizeof(int32_t) * dd.n_ent_c,
                                cudaMemcpyDeviceToDevice, st));
  }
  // source-grouped structural delta (DevDelta::rows_t)
  {
    DevArray<uint8_t> keep_d(dd.n_del, st), keep_i(dd.n_ins, st);
    DevArray<uint64_t> rem(dd.n_del, st), add(dd.n_ins, st);
    if (dd.n_del)
      DGNN_LAUNCH(k_mark, grid_for(dd.n_del), kT, 0, st, dd.n_del, dd.del.get(), dd.n_ins,
                  dd.ins.get(), 0, keep_d.get());
    if (dd.n_ins)
      DGNN_LAUNCH(k_mark, grid_for(dd.n_ins), kT, 0, st, dd.n_ins, dd.ins.get(), dd.n_del,
                  dd.del.get(), 0, keep_i.get());
    const int64_t nr_ = cub.select_flagged(dd.del.get(), keep_d.get(), rem.get(), dd.n_del);
    const int64_t na_ = cub.select_flagged(dd.ins.get(), keep_i.get(), add.get(), dd.n_ins);
    const int64_t nt = nr_ + na_;
    dd.n_ent_t = nt;
    DevArray<uint64_t> ct(nt, st), ct_sorted(nt, st);
    if (nr_) DGNN_LAUNCH(k_composite_t, grid_for(nr_), kT, 0, st, nr_, rem.get(), 0ull, ct.get());
    if (na_) DGNN_LAUNCH(k_composite_t, grid_for(na_), kT, 0, st, na_, add.get(), 1ull, ct.get() + nr_);
    cub.sort(ct.get(), ct_sorted.get(), nt);
    DevArray<int32_t> srcs(nt, st), uq(nt, st), cn(nt + 1, st);
    dd.ent_t = DevArray<int32_t>(nt, st);
    if (nt) DGNN_LAUNCH(k_split_composite, grid_for(nt), kT, 0, st, nt, ct_sorted.get(), srcs.get(), dd.ent_t.get());
    const int64_t nrt = cub.rle(srcs.get(), uq.get(), cn.get(), nt);
    dd.n_rows_t = static_cast<int32_t>(nrt);
    dd.rows_t = DevArray<int32_t>(nrt, st);
    dd.row_ptr_t = DevArray<int32_t>(nrt + 1, st);
    if (nrt) {
      DGNN_CUDA(cudaMemcpyAsync(dd.rows_t.get(), uq.get(), sizeof(int32_t) * nrt, cudaMemcpyDeviceToDevice, st));
      DGNN_CUDA(cudaMemsetAsync(cn.get() + nrt, 0, sizeof(int32_t), st));
    }
    cub.exclusive_sum(cn.get(), dd.row_ptr_t.get(), nrt + 1);
  }
  DGNN_CUDA(cudaStreamSynchronize(st));
  deltas_[t] = std::move(dd);
}

// ---------------------------------------------------------------- k-hop
namespace {

// std::mt19937_64 (libstdc++), full state in local memory.
struct Mt64 {
  static constexpr int kN = 312, kM = 156;
  uint64_t mt[kN];
  int idx;
  __device__ explicit Mt64(uint64_t s) {
    mt[0] = s;
    for (int i = 1; i < kN; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i;
    idx = kN;
  }
  __device__ void twist() {
    for (int i = 0; i < kN; ++i) {
      const uint64_t y = (mt[i] & 0xFFFFFFFF80000000ULL) | (mt[i + 1 < kN ? i + 1 : 0] & 0x7FFFFFFFULL);
      mt[i] = mt[i + kM < kN ? i + kM : i + kM - kN] ^ (y >> 1) ^ ((y & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
    }
    idx = 0;
  }
  __device__ uint64_t operator()() {
    if (idx >= kN) twist();
    uint64_t z = mt[idx++];
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= z >> 43;
    return z;
  }
};

__device__ __forceinline__ uint64_t d_mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
// derive_seed (ref inc/common.hpp:50-52)
__device__ __forceinline__ uint64_t d_derive_seed(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  return d_mix64(d_mix64(d_mix64(seed ^ d_mix64(a)) ^ d_mix64(b)) ^ d_mix64(c));
}

// uniform_int_distribution<size_t>(a, b) on a 64-bit engine: Lemire's
// nearly-divisionless reduction (libstdc++ bits/uniform_int_dist.h, _S_nd).
__device__ __forceinline__ uint64_t d_uniform(Mt64& g, uint64_t a, uint64_t b) {
  const uint64_t range = b - a + 1;
  uint64_t x = g();
  uint64_t hi = __umul64hi(x, range), lo = x * range;
  if (lo < range) {
    const uint64_t threshold = (0ULL - range) % range;
    while (lo < threshold) {
      x = g();
      hi = __umul64hi(x, range);
      lo = x * range;
    }
  }
  return a + hi;
}

__global__ void k_hop_counts(int64_t nd, const int32_t* __restrict__ dests,
                             const int64_t* __restrict__ in_ptr, int32_t fanout,
                             int64_t* __restrict__ cnt, int64_t* __restrict__ pool_cnt) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nd;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t v = dests[i];
    const int64_t deg = in_ptr[v + 1] - in_ptr[v];
    const bool all = fanout < 0 || deg <= fanout;
    cnt[i] = all ? deg : fanout;
    pool_cnt[i] = all ? 0 : deg;
  }
}

// sample_in_edges (ref src/khop.cpp:38-55), one destination per thread.
__global__ void __launch_bounds__(128)
k_hop_sample(int64_t nd, const int32_t* __restrict__ dests, const int64_t* __restrict__ in_ptr,
             const int32_t* __restrict__ in_src, int32_t fanout, uint64_t seed, int hop,
             const int64_t* __restrict__ off, const int64_t* __restrict__ pool_off,
             int32_t* __restrict__ pool, uint64_t* __restrict__ keys) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nd;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t v = dests[i];
    const int64_t b = in_ptr[v], deg = in_ptr[v + 1] - b;
    uint64_t* out = keys + off[i];
    if (fanout < 0 || deg <= fanout) {
      for (int64_t j = 0; j < deg; ++j)
        out[j] = (static_cast<uint64_t>(static_cast<uint32_t>(in_src[b + j])) << 32) | static_cast<uint32_t>(v);
      continue;
    }
    int32_t* p = pool + pool_off[i];
    for (int64_t j = 0; j < deg; ++j) p[j] = in_src[b + j];
    Mt64 g(d_derive_seed(seed, static_cast<uint64_t>(v), static_cast<uint64_t>(hop), 0));
    for (int32_t j = 0; j < fanout; ++j) {  // partial Fisher-Yates
      const uint64_t k = d_uniform(g, static_cast<uint64_t>(j), static_cast<uint64_t>(deg - 1));
      const int32_t t = p[j];
      p[j] = p[k];
      p[k] = t;
      out[j] = (static_cast<uint64_t>(static_cast<uint32_t>(p[j])) << 32) | static_cast<uint32_t>(v);
    }
  }
}

__global__ void k_nodes_to_keys(int64_t n, const int32_t* __restrict__ nodes, uint64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<uint32_t>(nodes[i]);
}

__global__ void k_src_to_keys(int64_t n, const uint64_t* __restrict__ edges, uint64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = edges[i] >> 32;
}

DevArray<uint64_t> copy_keys(const uint64_t* src, int64_t n, cudaStream_t st) {
  DevArray<uint64_t> out(n, st);
  if (n) DGNN_CUDA(cudaMemcpyAsync(out.get(), src, sizeof(uint64_t) * n, cudaMemcpyDeviceToDevice, st));
  return out;
}

// closure: sorted unique (dests U sources of edges) (ref src/khop.cpp:88-93)
DevArray<int32_t> closure(const DevArray<int32_t>& dests, int64_t nd, const DevArray<uint64_t>& edges,
                          int64_t ne, int64_t* n_out, Cub& cub) {
  cudaStream_t st = cub.st;
  const int64_t m = nd + ne;
  DevArray<uint64_t> cat(m, st), sorted(m, st), uniq(m, st);
  if (nd) DGNN_LAUNCH(k_nodes_to_keys, grid_for(nd), kT, 0, st, nd, dests.get(), cat.get());
  if (ne) DGNN_LAUNCH(k_src_to_keys, grid_for(ne), kT, 0, st, ne, edges.get(), cat.get() + nd);
  cub.sort(cat.get(), sorted.get(), m, 32);
  *n_out = cub.unique(sorted.get(), uniq.get(), m);
  DevArray<int32_t> out(*n_out, st);
  if (*n_out) DGNN_LAUNCH(k_low32, grid_for(*n_out), kT, 0, st, *n_out, uniq.get(), out.get());
  return out;
}

// a \ b over sorted unique keys
DevArray<uint64_t> set_minus(const DevArray<uint64_t>& a, int64_t na, const DevArray<uint64_t>& b,
                             int64_t nb, int64_t* n_out, Cub& cub) {
  cudaStream_t st = cub.st;
  if (na == 0) {
    *n_out = 0;
    return DevArray<uint64_t>(0, st);
  }
  DevArray<uint8_t> keep(na, st);
  DevArray<uint64_t> tmp(na, st);
  DGNN_LAUNCH(k_mark, grid_for(na), kT, 0, st, na, a.get(), nb, b.get(), 0, keep.get());
  *n_out = cub.select_flagged(a.get(), keep.get(), tmp.get(), na);
  return copy_keys(tmp.get(), *n_out, st);
}

}  // namespace

DevCompGraph khop(const DevSnapshot& snap, int32_t num_nodes, std::vector<int32_t> seeds,
                  std::vector<int32_t> fanouts, uint64_t seed, cudaStream_t st) {
  // ref src/khop.cpp:66-80 (checks and messages)
  if (seeds.empty()) throw std::invalid_argument("khop: seeds must be non-empty");
  if (fanouts.empty()) throw std::invalid_argument("khop: fanouts must name at least one hop");
  std::sort(seeds.begin(), seeds.end());
  seeds.erase(std::unique(seeds.begin(), seeds.end()), seeds.end());
  for (int32_t s : seeds)
    if (s < 0 || s >= num_nodes) throw std::invalid_argument("khop: seed node out of range");
  for (int32_t f : fanouts)
    if (!(f == -1 || f >= 1)) throw std::invalid_argument("khop: fanout must be positive or full");
  Cub cub(st);
  DevCompGraph cg;
  cg.seeds = seeds;
  cg.fanouts = fanouts;
  cg.sample_seed = seed;
  int64_t nd = static_cast<int64_t>(seeds.size());
  DevArray<int32_t> dests = upload(seeds.data(), nd, st);
  for (size_t k = 0; k < fanouts.size(); ++k) {
    DevHop h;
    h.n_dest = nd;
    DevArray<int64_t> cnt(nd + 1, st), off(nd + 1, st), pcnt(nd + 1, st), poff(nd + 1, st);
    cnt.zero(st);
    pcnt.zero(st);
    DGNN_LAUNCH(k_hop_counts, grid_for(nd), kT, 0, st, nd, dests.get(), snap.in_ptr.get(),
                fanouts[k], cnt.get(), pcnt.get());
    cub.exclusive_sum(cnt.get(), off.get(), nd + 1);
    cub.exclusive_sum(pcnt.get(), poff.get(), nd + 1);
    const int64_t ne = cub.read(off.get() + nd), np = cub.read(poff.get() + nd);
    DevArray<uint64_t> raw(ne, st);
    DevArray<int32_t> pool(np, st);
    DGNN_LAUNCH(k_hop_sample, cuda::wave_grid(nd, 128, 4), 128, 0, st, nd, dests.get(),
                snap.in_ptr.get(), snap.in_src.get(), fanouts[k], seed, static_cast<int>(k),
                off.get(), poff.get(), pool.get(), raw.get());
    h.edges = DevArray<uint64_t>(ne, st);
    cub.sort(raw.get(), h.edges.get(), ne);
    h.n_edges = ne;
    int64_t nn = 0;
    DevArray<int32_t> next = closure(dests, nd, h.edges, ne, &nn, cub);
    h.dests = std::move(dests);
    cg.hops.push_back(std::move(h));
    dests = std::move(next);
    nd = nn;
  }
  DGNN_CUDA(cudaStreamSynchronize(st));
  return cg;
}

DevCgUpdate khop_delta(const DevCompGraph& prev, const DevSnapshot& curr, int32_t num_nodes,
                       cudaStream_t st) {
  DevCompGraph fresh = khop(curr, num_nodes, prev.seeds, prev.fanouts, prev.sample_seed, st);
  if (prev.hops.size() != fresh.hops.size())
    throw std::invalid_argument("khop_delta: hop count mismatch");
  Cub cub(st);
  DevCgUpdate up;
  up.hops.resize(fresh.hops.size());
  for (size_t k = 0; k < fresh.hops.size(); ++k) {
    const DevHop &a = prev.hops[k], &b = fresh.hops[k];
    up.hops[k].added = set_minus(b.edges, b.n_edges, a.edges, a.n_edges, &up.hops[k].n_added, cub);
    up.hops[k].removed = set_minus(a.edges, a.n_edges, b.edges, b.n_edges, &up.hops[k].n_removed, cub);
  }
  DGNN_CUDA(cudaStreamSynchronize(st));
  return up;
}

DevCompGraph apply_cg_update(const DevCompGraph& prev, const DevCgUpdate& update, cudaStream_t st) {
  if (update.hops.size() != prev.hops.size())
    throw std::invalid_argument("apply_cg_update: hop count mismatch");
  Cub cub(st);
  DevCompGraph out;
  out.seeds = prev.seeds;
  out.fanouts = prev.fanouts;
  out.sample_seed = prev.sample_seed;
  int64_t nd = static_cast<int64_t>(prev.seeds.size());
  DevArray<int32_t> dests = upload(prev.seeds.data(), nd, st);
  for (size_t k = 0; k < prev.hops.size(); ++k) {
    const DevHop& p = prev.hops[k];
    const auto& diff = update.hops[k];
    int64_t nk = 0;
    DevArray<uint64_t> kept = set_minus(p.edges, p.n_edges, diff.removed, diff.n_removed, &nk, cub);
    // set_union of two sorted unique ranges = sort + unique of the concatenation
    const int64_t m = nk + diff.n_added;
    DevArray<uint64_t> cat(m, st), sorted(m, st), uniq(m, st);
    if (nk) DGNN_CUDA(cudaMemcpyAsync(cat.get(), kept.get(), 8 * nk, cudaMemcpyDeviceToDevice, st));
    if (diff.n_added)
      DGNN_CUDA(cudaMemcpyAsync(cat.get() + nk, diff.added.get(), 8 * diff.n_added, cudaMemcpyDeviceToDevice, st));
    cub.sort(cat.get(), sorted.get(), m);
    DevHop h;
    h.n_edges = cub.unique(sorted.get(), uniq.get(), m);
    h.edges = copy_keys(uniq.get(), h.n_edges, st);
    h.n_dest = nd;
    int64_t nn = 0;
    DevArray<int32_t> next = closure(dests, nd, h.edges, h.n_edges, &nn, cub);
    h.dests = std::move(dests);
    out.hops.push_back(std::move(h));
    dests = std::move(next);
    nd = nn;
  }
  DGNN_CUDA(cudaStreamSynchronize(st));
  return out;
}

// ---------------------------------------------------------------- ledgers
namespace {

__global__ void k_mark_remote_sources(int32_t nb, int32_t ne, const int64_t* __restrict__ in_ptr,
                                      const int32_t* __restrict__ in_src, uint8_t* __restrict__ flag) {
  const int64_t b = in_ptr[nb], e = in_ptr[ne];
  for (int64_t i = b + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < e;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t u = in_src[i];
    if (u < nb || u >= ne) flag[u] = 1;
  }
}

__global__ void k_count_flags(int32_t n, const uint8_t* __restrict__ flag, unsigned long long* out) {
  unsigned long long c = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    c += flag[i];
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

}  // namespace

uint64_t remote_source_count(const DevSnapshot& snap, int32_t num_nodes, int32_t nb, int32_t ne,
                             cudaStream_t st) {
  DevArray<uint8_t> flag(num_nodes, st);
  DevArray<unsigned long long> cnt(1, st);
  DGNN_CUDA(cudaMemsetAsync(flag.get(), 0, num_nodes, st));
  cnt.zero(st);
  // the in-CSR rows of [nb, ne) are one contiguous edge range
  DGNN_LAUNCH(k_mark_remote_sources, cuda::wave_grid(snap.num_edges + 1, kT, 4), kT, 0, st, nb, ne,
              snap.in_ptr.get(), snap.in_src.get(), flag.get());
  DGNN_LAUNCH(k_count_flags, grid_for(num_nodes), kT, 0, st, num_nodes, flag.get(), cnt.get());
  unsigned long long h = 0;
  copy_to_host(&h, cnt.get(), sizeof(h), st);
  return h;
}

}  // namespace dgnn
