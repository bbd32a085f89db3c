// Host launchers for the aggregation kernels (agg_kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace dgnn {
namespace cuda {

// AggrKind order of the reference (inc/aggregate.hpp:21).
enum : int { kAggSum = 0, kAggMean = 1, kAggMax = 2, kAggMin = 3 };

// values[v] = fn over in-neighbours u of v of feats[u]; feats/values are
// row-major n x w. mean also writes degree (n) and mean_sums (n x w);
// max/min write argext (n x w, -1 for empty rows, +/-inf sentinel values).
void agg_scratch(int kind, int n, int w, const int64_t* in_ptr, const int32_t* in_src,
                 const float* feats, float* values, float* degree, float* mean_sums,
                 int32_t* argext, cudaStream_t stream);

// In-place delta update of an aggregation already holding Agg_{t-1}:
// for each listed destination rows[r], entries ent[row_ptr[r]..row_ptr[r+1])
// are deletions (~src, gathered from f_prev) then insertions (src, from f_curr).
// sum: values +=/-=; mean: mean_sums and degree updated, values renormalised;
// max/min: insertions only (deleted contributors must have been ruled out).
// With ent_c / row_ptr_c (sum / mean, 128-bit aligned rows, w <= 512) the
// pipelined kernel reads sources >= num_nodes from the compact changed-row
// block (DevDelta::compact): deletions ~(N + p) subtract the negated
// difference row compact[p * w] (a folded deletion + insertion pair: degree
// unchanged), insertions N + p add F_t[changed[p]] = compact[(n_changed + p) * w].
void agg_delta(int kind, int n_rows, int w, const int32_t* rows, const int32_t* row_ptr,
               const int32_t* ent, const float* f_prev, const float* f_curr, float* values,
               float* degree, float* mean_sums, int32_t* argext, cudaStream_t stream,
               const int32_t* ent_c = nullptr, int32_t num_nodes = 0, int64_t n_changed = 0,
               const float* compact = nullptr, const int32_t* row_ptr_c = nullptr);

// Structural update of one matrix's aggregation, in place: values (=
// Agg_{G_{t-1}}(H), sum / mean) becomes Agg_{G_t}(H) using delta t's folded
// layout (rows, row_ptr_c, ent_c; `changed` = DevDelta::changed): removed
// edges subtract H[src], added edges add it, persisting edges of
// feature-changed nodes are skipped. Returns false (nothing launched) when
// the shape / kind is not supported; the caller then aggregates from scratch.
// shape / alignment check for agg_delta_struct (callers fall back to scratch)
bool agg_delta_struct_supported(int kind, int w, const float* h);
bool agg_delta_struct(int kind, int n_rows, int w, const int32_t* rows, const int32_t* row_ptr_c,
                      const int32_t* ent_c, int32_t num_nodes, const int32_t* changed,
                      const float* h, float* values, float* degree, float* mean_sums,
                      cudaStream_t stream);

// flag |= 1 if any deleted edge (sorted src << 32 | dst keys) is a recorded
// max/min contributor.
void agg_deleted_contributor(int64_t n_del, int w, const uint64_t* del_keys,
                             const int32_t* argext, int32_t* flag, cudaStream_t stream);

// grad[u] = sum over out-neighbours v of u of s_v * up[v] (sum: s=1, mean:
// s=1/degree[v]); max/min scatter up[v,d] to argext[v,d]. With `addend`
// (may alias grad) the result is added to it: grad = addend + ... — the GRU
// skip gradient and the layer-input gradient accumulate without a separate
// read-modify-write pass.
void agg_backward(int kind, int n, int w, const int64_t* out_ptr, const int32_t* out_dst,
                  const float* up, const float* degree, const int32_t* argext, float* grad,
                  cudaStream_t stream, const float* addend = nullptr);

// out = in with rows whose argext[v,0] < 0 zeroed (AggResult::dense_values,
// ref src/aggregate.cpp:30-37, and the empty-row gradient stop, src/cells.cpp:222-229).
void mask_empty_rows(int n, int w, const int32_t* argext, const float* in, float* out,
                     cudaStream_t stream);

}  // namespace cuda
}  // namespace dgnn
