// Device-resident dynamic graph store (kernels K11/K12).
//
// Mirrors dgnn::DynamicGraph / Snapshot / DeltaGraph (ref inc/snapshot.hpp:39-107)
// with everything built and kept in HBM:
//   per snapshot t : in-CSR (in_ptr int64[N+1], in_src int32[E], sources
//                    ascending per destination), out-CSR (out_ptr, out_dst,
//                    destinations ascending per source), features fp32 N x d;
//   per t >= 1     : the reference's extract_delta (src/snapshot.cpp:102-130),
//                    bit-exact: deletions / insertions (sorted unique (src,dst)
//                    keys incl. the feature-change out-edge expansion), changed
//                    nodes ascending, plus the dst-grouped signed layout the
//                    delta-SpMM consumes (rows, row_ptr, ent = ~src | src).
// Snapshots are built on the device from snapshot 0 plus per-step structural
// deltas (the reference's apply_delta semantics, src/snapshot.cpp:142-154) or
// from full per-step edge lists (Snapshot ctor semantics, src/snapshot.cpp:20-69).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "memory.h"

namespace dgnn {

struct DevSnapshot {
  int64_t num_edges = 0;
  cuda::DevArray<int64_t> in_ptr, out_ptr;
  cuda::DevArray<int32_t> in_src, out_dst;
  cuda::DevArray<float> feats;  // N x d (may alias the previous snapshot's rows? no: owned)
};

struct DevDelta {
  int64_t n_del = 0, n_ins = 0, n_changed = 0;
  cuda::DevArray<uint64_t> del, ins;  // sorted (src << 32 | dst)
  cuda::DevArray<int32_t> changed;    // ascending
  // delta-SpMM layout
  int32_t n_rows = 0;
  int64_t n_ent = 0;
  cuda::DevArray<int32_t> rows, row_ptr, ent;
  // distinct deletion / insertion sources (algorithmic-byte accounting)
  int64_t u_minus = 0, u_plus = 0;
  int64_t change_count() const { return n_del + n_ins; }
};

class DeviceGraph {
 public:
  DeviceGraph(int32_t num_nodes, int32_t feature_dim, cudaStream_t stream);
  ~DeviceGraph();

  // Snapshot 0 (unsorted edges allowed; duplicates / out-of-range endpoints
  // rejected with the reference's messages). Host pointers.
  void add_snapshot(const int32_t* src, const int32_t* dst, int64_t num_edges, const float* feats);
  // Next snapshot from the previous one: (prev \ deletions) U insertions, with
  // feature rows `changed_nodes` replaced (apply_delta). Host pointers.
  void add_delta(const int32_t* del_src, const int32_t* del_dst, int64_t n_del,
                 const int32_t* ins_src, const int32_t* ins_dst, int64_t n_ins,
                 const int32_t* changed_nodes, int64_t n_changed, const float* changed_feats);

  int32_t length() const { return static_cast<int32_t>(snaps_.size()); }
  int32_t num_nodes() const { return n_; }
  int32_t feature_dim() const { return d_; }
  const DevSnapshot& snapshot(int32_t t) const;
  // Delta producing snapshot t from t-1 (t >= 1), computed at build time.
  const DevDelta& delta(int32_t t) const;
  cudaStream_t stream() const { return stream_; }

  // Drops the device features of snapshots < t_keep (memory at C4 scale).
  int64_t device_bytes() const;

 private:
  void finish_snapshot(cuda::DevArray<uint64_t> keys, cuda::DevArray<float> feats);
  void build_delta(int32_t t);

  int32_t n_, d_;
  cudaStream_t stream_;
  std::vector<DevSnapshot> snaps_;
  std::vector<DevDelta> deltas_;  // deltas_[t], t >= 1; deltas_[0] unused
  cuda::DevArray<uint64_t> prev_keys_, curr_keys_;  // sorted (src,dst) of the last two snapshots
};

// Host copies (tests / C-ABI getters).
void copy_to_host(void* dst, const void* src, size_t bytes, cudaStream_t stream);

}  // namespace dgnn
