// Device-resident dynamic graph store (kernels K11/K12).
//
// Mirrors dgnn::DynamicGraph / Snapshot / DeltaGraph (ref inc/snapshot.hpp:39-107)
// with everything built and kept in HBM:
//   per snapshot t : in-CSR (in_ptr int64[N+1], in_src int32[E], sources
//                    ascending per destination), out-CSR (out_ptr, out_dst,
//                    destinations ascending per source); features as
//                    versions (snapshot 0 whole + exact per-t row patches,
//                    see FeatSlot below);
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

#include <climits>
#include <cstdint>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "memory.h"

namespace dgnn {

struct DevSnapshot {
  int64_t num_edges = 0;
  cuda::DevArray<int64_t> in_ptr, out_ptr;
  cuda::DevArray<int32_t> in_src, out_dst;
};

// Versioned node features. Snapshot 0's N x d matrix is kept whole; every
// t >= 1 keeps only its exact changed rows (DevDelta::changed, values at t) —
// 2% of N at C4 instead of 2 GB per snapshot. Versions are materialised on
// demand (nearest resident version <= t, then the row patches in t order)
// into a bounded set of HBM slots, least-recently-used unpinned slot first.
// A lease pins its slot; cross-stream use is ordered by events (the slot's
// materialisation, and each reader stream's last use before a slot is reused).
struct FeatSlot {
  int32_t t = -1;
  uint64_t stamp = 0;
  cuda::DevArray<float> buf;
  cudaStream_t writer = nullptr;
  cudaEvent_t ready = nullptr;
  std::vector<std::pair<cudaStream_t, cudaEvent_t>> readers;
  ~FeatSlot();
};

class FeatLease {
 public:
  FeatLease(std::shared_ptr<FeatSlot> slot, cudaStream_t stream);
  ~FeatLease();
  FeatLease(const FeatLease&) = delete;
  FeatLease& operator=(const FeatLease&) = delete;
  const float* get() const { return slot_->buf.get(); }
  int32_t t() const { return slot_->t; }

 private:
  std::shared_ptr<FeatSlot> slot_;
  cudaStream_t stream_;
};
using FeatRef = std::shared_ptr<const FeatLease>;

struct DevDelta {
  int64_t n_del = 0, n_ins = 0, n_changed = 0;
  cuda::DevArray<uint64_t> del, ins;  // sorted (src << 32 | dst)
  cuda::DevArray<int32_t> changed;    // ascending
  // delta-SpMM layout
  int32_t n_rows = 0;
  int64_t n_ent = 0;
  cuda::DevArray<int32_t> rows, row_ptr, ent;
  // Feature-changed sources, compacted: compact = [F_{t-1}[changed] -
  // F_t[changed] | F_t[changed]] (2 x n_changed x d; the second half is also
  // the version patch of t). A changed node contributes all its out-edges to
  // both G- and G+ (~2/3 of the delta's entries at C4); ent_c / row_ptr_c fold
  // each such persisting pair into ONE entry ~(N + pos) that subtracts the
  // negated difference row, so those gathers halve and hit a 41 MB
  // L2-resident block instead of random rows of two 2 GB matrices. Unpaired
  // changed insertions read N + pos (F_t half); unpaired deletions keep
  // their plain index.
  int64_t n_ent_c = 0;
  cuda::DevArray<int32_t> ent_c, row_ptr_c;
  cuda::DevArray<float> compact;
  // Source-grouped structural delta (the transposed structural part of G_t vs
  // G_{t-1}: edges removed = del \ ins, added = ins \ del; persisting
  // feature-changed pairs cancel): rows_t = sources, entries ~dst (removed) /
  // dst (added). A_t^T y = A_{t-1}^T y + (this layout) y — used by the
  // backward to push a hidden gradient through A_{t-1}^T together with the
  // layer above's input gradient (one transposed SpMM instead of two).
  int32_t n_rows_t = 0;
  int64_t n_ent_t = 0;
  cuda::DevArray<int32_t> rows_t, row_ptr_t, ent_t;
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

  // Features of snapshot t, resident for the lifetime of the returned lease
  // and ordered before work later issued on `stream`.
  FeatRef features(int32_t t, cudaStream_t stream) const;
  // HBM slots for materialised feature versions (snapshot 0 is always
  // resident and not counted). Default: every version if they fit
  // DGNN_FEATURE_BUDGET_GB (default 24), else as many as fit, at least 2.
  void set_feature_slots(int32_t slots) { max_slots_ = slots < 2 ? 2 : slots; }
  int32_t feature_slots() const { return max_slots_; }
  int64_t feature_materialisations() const { return materialisations_; }

  int64_t device_bytes() const;
  // Keep only snapshots / deltas / feature versions [t_first, t_last]: a rank
  // of the window-sharded trainer needs its window block plus the L + H
  // overlap (replicate_overlap, ref inc/distsim.hpp:49-54). The features of
  // t_first become a resident base version (so earlier patches can go); the
  // snapshot indices and length() stay global, anything outside the range
  // throws std::out_of_range. Call it before sessions read the graph (it
  // frees device arrays without waiting for other streams' readers).
  void retain(int32_t t_first, int32_t t_last);
  int32_t retained_first() const { return first_; }
  int32_t retained_last() const { return last_; }
  // Frees the build-time key arrays of the last snapshot (2 x 8 B per edge);
  // a later add_delta rebuilds them from the snapshot's CSRs.
  void release_build_state();

 private:
  // Structural edge change of an apply_delta step, known exactly from its
  // inputs: removed = (prev ∩ D) \ I, added = I \ prev (sorted unique).
  struct StructDiff {
    cuda::DevArray<uint64_t> removed, added;
    int64_t n_removed = 0, n_added = 0;
  };
  void finish_snapshot(cuda::DevArray<uint64_t> keys, const float* prev_feats, const float* feats,
                       cuda::DevArray<uint64_t> swapped = {}, const StructDiff* diff = nullptr);
  void build_delta(int32_t t, const float* prev_feats, const float* feats, const StructDiff* diff);
  void ensure_build_keys();
  std::shared_ptr<FeatSlot> free_slot(cudaStream_t stream) const;
  void order_after_write(const FeatSlot& s, cudaStream_t stream) const;

  int32_t n_, d_;
  cudaStream_t stream_;
  std::vector<DevSnapshot> snaps_;
  std::vector<DevDelta> deltas_;  // deltas_[t], t >= 1; deltas_[0] unused
  cuda::DevArray<uint64_t> prev_keys_, curr_keys_;  // sorted (src,dst) of the last two snapshots
  cuda::DevArray<uint64_t> curr_swapped_;           // last snapshot's (dst,src) keys, sorted
  // feature versions (the per-t patch is the second half of delta(t).compact)
  mutable std::vector<std::shared_ptr<FeatSlot>> slots_;  // slots_[0] = snapshot 0
  std::shared_ptr<const FeatLease> retained_base_;          // features(first_) after retain()
  int32_t first_ = 0, last_ = INT32_MAX;
  mutable uint64_t clock_ = 0;
  mutable int64_t materialisations_ = 0;
  int32_t max_slots_ = 0;
};

// Host copies (tests / C-ABI getters).
void copy_to_host(void* dst, const void* src, size_t bytes, cudaStream_t stream);

// In-CSR (sources ascending per destination) + out-CSR over num_nodes from
// sorted unique (src << 32 | dst) keys (ref Snapshot ctor CSR build,
// src/snapshot.cpp:46-69, and ComputationalGraph::to_view, src/khop.cpp:22-33).
DevSnapshot csr_from_keys(const uint64_t* keys, int64_t num_edges, int32_t num_nodes,
                          cudaStream_t stream, const uint64_t* swapped_sorted = nullptr,
                          cuda::DevArray<uint64_t>* swapped_out = nullptr);

// Distinct sources outside [nb, ne) with an in-edge into [nb, ne) in one
// snapshot (the node-partition remote-feature count, src/distsim.cpp:121-139).
uint64_t remote_source_count(const DevSnapshot& snap, int32_t num_nodes, int32_t nb, int32_t ne,
                             cudaStream_t stream);

// ---------------------------------------------------------------- k-hop
// Sampled k-hop computational graphs (ref inc/khop.hpp:35-88, src/khop.cpp),
// built on the device from a resident snapshot. Sampling is bit-exact with the
// reference: per (destination, hop) an mt19937_64 seeded with
// derive_seed(seed, dst, hop) drives a partial Fisher-Yates over the
// destination's ascending in-neighbours with libstdc++'s
// uniform_int_distribution<size_t> (Lemire's nearly-divisionless method).
struct DevHop {
  int64_t n_dest = 0, n_edges = 0;
  cuda::DevArray<int32_t> dests;   // sorted
  cuda::DevArray<uint64_t> edges;  // sorted (src << 32 | dst), dst in dests
};

struct DevCompGraph {
  std::vector<int32_t> seeds;    // sorted unique (host)
  std::vector<int32_t> fanouts;  // -1 = full
  uint64_t sample_seed = 0;
  std::vector<DevHop> hops;
};

struct DevCgUpdate {
  struct Diff {
    int64_t n_added = 0, n_removed = 0;
    cuda::DevArray<uint64_t> added, removed;  // sorted keys
  };
  std::vector<Diff> hops;
  bool empty() const {
    for (const auto& h : hops)
      if (h.n_added || h.n_removed) return false;
    return true;
  }
};

// khop (src/khop.cpp:66-96): reference checks and messages.
DevCompGraph khop(const DevSnapshot& snap, int32_t num_nodes, std::vector<int32_t> seeds,
                  std::vector<int32_t> fanouts, uint64_t seed, cudaStream_t stream);
// khop_delta (src/khop.cpp:105-121): fresh k-hop graph of `curr`, per-hop set
// differences against prev.
DevCgUpdate khop_delta(const DevCompGraph& prev, const DevSnapshot& curr, int32_t num_nodes,
                       cudaStream_t stream);
// apply_cg_update (src/khop.cpp:123-150).
DevCompGraph apply_cg_update(const DevCompGraph& prev, const DevCgUpdate& update,
                             cudaStream_t stream);

}  // namespace dgnn
