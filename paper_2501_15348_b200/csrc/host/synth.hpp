// Streaming, bit-exact equivalent of dgnn::synthesize (ref src/synth.cpp:36-91).
//
// Same libstdc++ engines and distributions in the same call order (edge
// draws, feature draws, per-step shuffles), so the generated dynamic graph is
// identical to the reference's. Differences are representational only: edges
// live in an open-addressing hash set plus one sorted vector instead of a
// std::set, and the output is snapshot 0 plus per-step structural deltas
// (removed / inserted edges, redrawn feature rows as fp32) instead of T fully
// materialised fp64 snapshots, which keeps the 80M-edge C4 graph in a few GB
// of host memory.
#pragma once

#include <cstdint>
#include <vector>

namespace dgnn {

struct SynthParams {
  int32_t num_nodes = 0;
  double avg_degree = 1.0;
  int32_t feature_dim = 1;
  int32_t num_snapshots = 1;
  double edge_change = 0.0;
  bool edge_change_uniform = false;
  double feature_change = 0.0;
  bool feature_change_uniform = false;
  uint64_t seed = 0;
};

struct CompactStep {
  std::vector<int32_t> del_src, del_dst;  // removed edges, sorted (src,dst)
  std::vector<int32_t> ins_src, ins_dst;  // inserted edges, sorted (src,dst)
  std::vector<int32_t> changed;           // redrawn nodes, ascending
  std::vector<float> changed_feats;       // rows aligned with `changed`
};

struct CompactGraph {
  int32_t num_nodes = 0, feature_dim = 0, num_snapshots = 0;
  std::vector<int32_t> base_src, base_dst;  // snapshot 0, sorted (src,dst)
  std::vector<float> base_feats;            // n x d
  std::vector<CompactStep> steps;           // steps[t-1] produces snapshot t
};

CompactGraph synthesize_compact(const SynthParams& p);

}  // namespace dgnn
