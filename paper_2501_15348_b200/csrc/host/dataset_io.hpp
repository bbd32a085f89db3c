// On-disk dynamic-graph datasets: the reference's bit-exact
// text layout plus a binary twin, read step by step so a graph can stream into
// the HBM graph store without materialising snapshots on the host.
//
// Reference: save_dataset / load_dataset (inc/dataset_io.hpp:6-11,
// src/dataset_io.cpp:40-165). Text layout (format_version 1), byte-identical
// to the reference writer for the same values:
//   manifest.json        {"T":T,"feature_dim":d,"format_version":1,"num_nodes":N}
//   snapshot_0.edges     "src\tdst" per line, ascending (src,dst)
//   snapshot_0.feats     CSV, row i = node i, "%.9g"
//   delta_{t}.edges      "D src dst" lines then "I src dst" lines
//   delta_{t}.feats      CSV "node_id,f0,f1,..." for feature-changed nodes
// The reader follows the reference parser's acceptance rules and messages
// (stream extraction for edges, getline/stod for CSV cells, the arity and
// truncation checks). Device features are fp32, so a loaded value is the fp32
// rounding of the reference's stod(); "%.9g" of an fp32 value round-trips it
// exactly, so save -> load of a device graph is bit-exact.
//
// Binary twin (format_version 2, "encoding":"b200-le", little-endian):
//   snapshot_0.bin  header{magic "DGNNB200", u32 1, u32 kind 0, i64 E, i32 N, i32 d}
//                   i32 src[E], i32 dst[E], f32 feats[N*d]
//   delta_{t}.bin   header{magic, u32 1, u32 kind 1, i64 n_del, i64 n_ins,
//                   i64 n_changed, i32 t, i32 d}
//                   i32 del_src, del_dst, ins_src, ins_dst, changed; f32 rows
// A delta may be the structural change plus redrawn rows (what the generator
// produces) or the reference's expanded G-/G+ (what extract_delta produces):
// apply_delta gives the same snapshot for both (src/snapshot.cpp:142-154).
#pragma once

#include <cstdint>
#include <filesystem>
#include <string>
#include <vector>

#include "synth.hpp"

namespace dgnn {

struct DatasetManifest {
  int32_t num_nodes = 0, feature_dim = 0, T = 0;
  int32_t format = 1;  // 1 = reference text layout, 2 = binary twin
};

// Non-owning view of one step's change (host memory).
struct StepView {
  int64_t n_del = 0, n_ins = 0, n_changed = 0;
  const int32_t *del_src = nullptr, *del_dst = nullptr, *ins_src = nullptr, *ins_dst = nullptr;
  const int32_t* changed = nullptr;
  const float* changed_feats = nullptr;  // n_changed x d
};

// ---------------------------------------------------------------- reading
class DatasetReader {
 public:
  // Parses and validates the manifest (src/dataset_io.cpp:98-104).
  explicit DatasetReader(std::filesystem::path dir, int threads = 0);
  const DatasetManifest& manifest() const { return m_; }
  // snapshot 0: edges in file order (validated / sorted by the graph store,
  // as by the Snapshot ctor), features N x d.
  void read_base(std::vector<int32_t>& src, std::vector<int32_t>& dst, std::vector<float>& feats) const;
  // delta_t (1 <= t < T) into `out` (reused buffers).
  void read_step(int32_t t, CompactStep& out) const;

 private:
  std::filesystem::path dir_;
  DatasetManifest m_;
  int threads_;
};

// ---------------------------------------------------------------- writing
// Manifest + directory (src/dataset_io.cpp:40-48).
void write_manifest(const std::filesystem::path& dir, const DatasetManifest& m);
// snapshot 0; edges must be ascending (src,dst) for a reference-identical file.
void write_base(const std::filesystem::path& dir, const DatasetManifest& m, const int32_t* src,
                const int32_t* dst, int64_t num_edges, const float* feats, int threads = 0);
void write_step(const std::filesystem::path& dir, const DatasetManifest& m, int32_t t,
                const StepView& s);
// Whole compact graph (the generator's output).
void save_compact(const CompactGraph& g, const std::filesystem::path& dir, int32_t format);

// "%.9g" (src/dataset_io.cpp:17-21); appends to `out`.
void append_value(std::string& out, double v);

}  // namespace dgnn
