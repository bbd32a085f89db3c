/*
 * dgnn_b200.h — C ABI of the B200-native ReInc dynamic-GNN training hot path.
 *
 * This is the drop-in boundary. The reference is a C++
 * library (proj/include/dgnn/ headers) with no FFI of its own; every entry point
 * below names the reference interface it replaces (file:line into
 * /root/reference/proj). Plain pointers and sizes only: device pointers are
 * fp32 / int32 / int64 HBM buffers, `stream` is a cudaStream_t (NULL = the
 * library's own stream for sessions, the legacy default stream for ops).
 *
 * Error convention: every function returning int returns 0 on success,
 * 1 = std::invalid_argument (the reference's check()/fail() messages,
 * inc/common.hpp:36-40), 2 = std::out_of_range (the reference's .at()),
 * 3 = CUDA / runtime error. dgnn_last_error() returns the message of the last
 * failure on the calling thread.
 *
 * Aggregation kinds follow AggrKind (inc/aggregate.hpp:21): 0 sum, 1 mean,
 * 2 max, 3 min. Architectures follow Architecture (inc/model.hpp:21):
 * 0 gcrn_m1, 1 cd_gcn, 2 gcrn_m2, 3 tgcn.
 */
#ifndef DGNN_B200_H
#define DGNN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dgnn_graph dgnn_graph;
typedef struct dgnn_synth dgnn_synth;
typedef struct dgnn_session dgnn_session;
typedef struct dgnn_dataset dgnn_dataset;
typedef struct dgnn_cg dgnn_cg;
typedef struct dgnn_cg_update dgnn_cg_update;
typedef struct dgnn_comm dgnn_comm;

const char* dgnn_last_error(void);
const char* dgnn_version(void);
/* Number of this library's kernels launched so far (process-wide). */
int64_t dgnn_launch_count(void);
int dgnn_synchronize(void* stream);
/* cudaSetDevice for callers without their own CUDA runtime (one GPU per process). */
int dgnn_set_device(int32_t device);

/* ------------------------------------------------------------------ graph
 * Replaces dgnn::DynamicGraph / Snapshot / DeltaGraph / extract_delta /
 * apply_delta / change_ratio (inc/snapshot.hpp:39-119, src/snapshot.cpp:20-154).
 * Snapshots live in HBM (in-CSR, out-CSR, fp32 features); extract_delta is
 * evaluated on the device when each snapshot is added. Host input pointers. */
int dgnn_graph_create(int32_t num_nodes, int32_t feature_dim, void* stream, dgnn_graph** out);
void dgnn_graph_free(dgnn_graph* g);
/* Snapshot ctor (src/snapshot.cpp:20-69): edges in any order; duplicates and
 * out-of-range endpoints are rejected. feats: num_nodes x feature_dim. */
int dgnn_graph_add_snapshot(dgnn_graph* g, const int32_t* src, const int32_t* dst,
                            int64_t num_edges, const float* feats);
/* apply_delta (src/snapshot.cpp:142-154): next = (last \ deletions) U insertions,
 * feature rows of changed_nodes replaced by changed_feats (n_changed x dim). */
int dgnn_graph_add_delta(dgnn_graph* g, const int32_t* del_src, const int32_t* del_dst,
                         int64_t n_del, const int32_t* ins_src, const int32_t* ins_dst,
                         int64_t n_ins, const int32_t* changed_nodes, int64_t n_changed,
                         const float* changed_feats);
int32_t dgnn_graph_length(const dgnn_graph* g);
/* Keep only snapshots / deltas / feature versions [t_first, t_last] (a rank's
 * window block plus the L+H overlap: replicate_overlap, inc/distsim.hpp:49-54);
 * indices stay global, access outside the range is status 2 (out_of_range). */
int dgnn_graph_retain(dgnn_graph* g, int32_t t_first, int32_t t_last);
int64_t dgnn_graph_num_edges(const dgnn_graph* g, int32_t t);
/* HBM held by the graph store (CSRs, deltas, feature versions and patches);
 * the feature-version slot budget and how many versions were materialised. */
int64_t dgnn_graph_device_bytes(const dgnn_graph* g);
int dgnn_graph_feature_stats(const dgnn_graph* g, int32_t* slots, int64_t* materialisations);
/* Device pointers of snapshot t (GraphView, inc/snapshot.hpp:20-35, plus the out-CSR). */
int dgnn_graph_snapshot(const dgnn_graph* g, int32_t t, const int64_t** in_ptr,
                        const int32_t** in_src, const int64_t** out_ptr, const int32_t** out_dst,
                        const float** feats);
/* DynamicGraph::delta(t) sizes (inc/snapshot.hpp:79-104); n_rows = distinct
 * destinations, u_minus / u_plus = distinct deletion / insertion sources. */
int dgnn_graph_delta_sizes(const dgnn_graph* g, int32_t t, int64_t* n_del, int64_t* n_ins,
                           int64_t* n_changed, int64_t* n_rows, int64_t* u_minus,
                           int64_t* u_plus);
/* Host copies of DeltaGraph deletions / insertions (sorted (src,dst)) and
 * changed_nodes (ascending). */
int dgnn_graph_delta_copy(const dgnn_graph* g, int32_t t, int32_t* del_src, int32_t* del_dst,
                          int32_t* ins_src, int32_t* ins_dst, int32_t* changed_nodes);
/* Device pointers of the delta-SpMM layout: rows[r] destinations, entries
 * ent[row_ptr[r]..row_ptr[r+1]) = deletions (~src) then insertions (src). */
int dgnn_graph_delta_layout(const dgnn_graph* g, int32_t t, const int32_t** rows,
                            const int32_t** row_ptr, const int32_t** ent);
/* change_ratio(delta(t), snapshot(t-1)) (src/snapshot.cpp:132-140). */
double dgnn_graph_change_ratio(const dgnn_graph* g, int32_t t);

/* ------------------------------------------------------------------ synth
 * Replaces dgnn::synthesize (inc/synth.hpp:39, src/synth.cpp:36-91) with a
 * bit-exact streaming generator producing snapshot 0 + per-step deltas. */
int dgnn_synth_create(int32_t num_nodes, double avg_degree, int32_t feature_dim,
                      int32_t num_snapshots, double edge_change, double feature_change,
                      uint64_t seed, dgnn_synth** out);
void dgnn_synth_free(dgnn_synth* s);
/* sizes: [E0, then per step t=1..T-1: n_del, n_ins, n_changed] (1 + 3(T-1) int64). */
int dgnn_synth_sizes(const dgnn_synth* s, int64_t* sizes);
/* Host views (valid while s lives). */
int dgnn_synth_base(const dgnn_synth* s, const int32_t** src, const int32_t** dst,
                    const float** feats);
int dgnn_synth_step(const dgnn_synth* s, int32_t t, const int32_t** del_src,
                    const int32_t** del_dst, const int32_t** ins_src, const int32_t** ins_dst,
                    const int32_t** changed, const float** changed_feats);
/* Uploads the compact graph and builds every snapshot + delta on the device. */
int dgnn_synth_to_graph(const dgnn_synth* s, void* stream, dgnn_graph** out);

/* ---------------------------------------------------------------- dataset
 * Replaces dgnn::save_dataset / load_dataset (inc/dataset_io.hpp:6-24,
 * src/dataset_io.cpp:40-165). format 1 = the reference's text layout
 * (byte-identical writer, same parser rules and messages); format 2 = binary
 * twin (manifest "format_version":2, "encoding":"b200-le"; *.bin files).
 * Host-only reader (no GPU needed): open / info / read_base / read_step;
 * views stay valid until the next read on the same handle. */
int dgnn_dataset_open(const char* dir, int32_t threads, dgnn_dataset** out);
void dgnn_dataset_free(dgnn_dataset* d);
int dgnn_dataset_info(const dgnn_dataset* d, int32_t* num_nodes, int32_t* feature_dim,
                      int32_t* T, int32_t* format);
/* snapshot_0: edges in file order, features num_nodes x feature_dim (fp32). */
int dgnn_dataset_read_base(dgnn_dataset* d, int64_t* num_edges, const int32_t** src,
                           const int32_t** dst, const float** feats);
/* delta_t (1 <= t < T): sizes = [n_del, n_ins, n_changed]. */
int dgnn_dataset_read_step(dgnn_dataset* d, int32_t t, int64_t* sizes, const int32_t** del_src,
                           const int32_t** del_dst, const int32_t** ins_src,
                           const int32_t** ins_dst, const int32_t** changed,
                           const float** changed_feats);
/* load_dataset into the HBM graph store, streaming (parse t+1 while the
 * device builds t; host memory bounded by two steps). threads <= 0: auto. */
int dgnn_dataset_load(const char* dir, int32_t threads, void* stream, dgnn_graph** out);
/* save_dataset of a device graph (deltas = DynamicGraph::delta(t), expanded). */
int dgnn_dataset_save_graph(const dgnn_graph* g, const char* dir, int32_t format);
/* Generator output (structural deltas + redrawn rows; same snapshots on load). */
int dgnn_synth_save(const dgnn_synth* s, const char* dir, int32_t format);

/* ------------------------------------------------------------------ k-hop
 * Replaces dgnn::khop / ComputationalGraph / khop_delta / apply_cg_update
 * (inc/khop.hpp:35-88, src/khop.cpp:12-150), sampled on the device from
 * snapshot t, bit-exact (mt19937_64 per (destination, hop), derive_seed,
 * partial Fisher-Yates, libstdc++ uniform_int_distribution). Fanout -1 =
 * full. Hop k: sorted destinations (the (k)-hop closure) and sorted
 * (src, dst) edges. */
int dgnn_khop(const dgnn_graph* g, int32_t t, const int32_t* seeds, int64_t n_seeds,
              const int32_t* fanouts, int32_t n_hops, uint64_t seed, dgnn_cg** out);
void dgnn_cg_free(dgnn_cg* c);
int32_t dgnn_cg_num_hops(const dgnn_cg* c);
int dgnn_cg_hop_sizes(const dgnn_cg* c, int32_t k, int64_t* n_dest, int64_t* n_edges);
int dgnn_cg_hop_copy(const dgnn_cg* c, int32_t k, int32_t* dests, int32_t* src, int32_t* dst);
/* ComputationalGraph::to_view (src/khop.cpp:22-33): device in-CSR (+ out-CSR)
 * over the node universe of the deepest hop's edges; owned by c. */
int dgnn_cg_view(dgnn_cg* c, const int64_t** in_ptr, const int32_t** in_src,
                 const int64_t** out_ptr, const int32_t** out_dst, int64_t* num_edges);
/* khop_delta against snapshot t of g (t >= 1). */
int dgnn_khop_delta(const dgnn_cg* prev, const dgnn_graph* g, int32_t t, dgnn_cg_update** out);
void dgnn_cg_update_free(dgnn_cg_update* u);
int dgnn_cg_update_sizes(const dgnn_cg_update* u, int32_t k, int64_t* n_added, int64_t* n_removed);
int dgnn_cg_update_copy(const dgnn_cg_update* u, int32_t k, int32_t* add_src, int32_t* add_dst,
                        int32_t* rem_src, int32_t* rem_dst);
int32_t dgnn_cg_update_empty(const dgnn_cg_update* u);
int dgnn_apply_cg_update(const dgnn_cg* prev, const dgnn_cg_update* up, dgnn_cg** out);

/* ------------------------------------------------------------ aggregation
 * Kernels K1/K2/K3 over device buffers (src/aggregate.cpp:55-246). */
int dgnn_agg_scratch(int32_t kind, int32_t n, int32_t w, const int64_t* in_ptr,
                     const int32_t* in_src, const float* feats, float* values, float* degree,
                     float* mean_sums, int32_t* argext, void* stream);
int dgnn_agg_delta(int32_t kind, int32_t n_rows, int32_t w, const int32_t* rows,
                   const int32_t* row_ptr, const int32_t* ent, const float* f_prev,
                   const float* f_curr, float* values, float* degree, float* mean_sums,
                   int32_t* argext, void* stream);
/* K2 on the graph's own delta(t) (aggregate_incremental's update step,
 * src/aggregate.cpp:170-205, without the fallback checks): values (and mean /
 * extremal state) hold Agg_{t-1} of the graph features (w = feature_dim) and
 * become Agg_t in place; uses the compact changed-row block. */
int dgnn_graph_apply_delta(const dgnn_graph* g, int32_t t, int32_t kind, float* values,
                           float* degree, float* mean_sums, int32_t* argext, void* stream);
int dgnn_agg_backward(int32_t kind, int32_t n, int32_t w, const int64_t* out_ptr,
                      const int32_t* out_dst, const float* upstream, const float* degree,
                      const int32_t* argext, float* grad, void* stream);
/* aggregate_incremental with the reference's fallback logic
 * (src/aggregate.cpp:117-207) from a caller-held AggResult of snapshot t-1 of
 * graph g (features of the graph store). prev_* may alias nothing; out_* are
 * caller-allocated (n x w; degree n). info[0] used_fallback, info[1]
 * FallbackReason, info[2] incremental_depth of the result. */
int dgnn_agg_incremental(const dgnn_graph* g, int32_t t, int32_t kind, const float* prev_values,
                         const float* prev_degree, const float* prev_mean_sums,
                         const int32_t* prev_argext, int32_t prev_depth, int64_t prev_num_edges,
                         double fallback_threshold, int32_t rescratch_period, float* values,
                         float* degree, float* mean_sums, int32_t* argext, int32_t* info);

/* ------------------------------------------------------------------ cells
 * Fused GraphRNN cell (cell_core_forward / cell_core_backward,
 * src/cells.cpp:102-195). W: (in+H) x 4H packed gate weights, bias 4H. */
int dgnn_pack_cell(int32_t lstm, int32_t in, int32_t H, const float* flat, float* W, float* bias,
                   void* stream);
int dgnn_cell_forward(int32_t lstm, int32_t n, int32_t in, int32_t H, const float* X,
                      const float* Hm, const float* h_skip, const float* c_prev, const float* W,
                      const float* bias, float* gates, float* c, float* h, void* stream);
/* Grads: dX (n x in, may be NULL), dHm (n x H), dc_prev (LSTM) / dh_skip
 * (GRU), flat parameter grads accumulated into dflat ([wx_g, uh_g, b_g]_g). */
int dgnn_cell_backward(int32_t lstm, int32_t n, int32_t in, int32_t H, const float* X,
                       const float* Hm, const float* W, const float* gates, const float* c,
                       const float* c_prev, const float* h_skip, const float* dh, const float* dc,
                       float* dX, float* dHm, float* dc_prev, float* dh_skip, float* dflat,
                       void* stream);

/* ---------------------------------------------------------------- trainer
 * Replaces TrainSession / seq_first_epoch / optimizer_step
 * (inc/train.hpp:64-114) and the consecutive-block DistSession
 * (inc/distsim.hpp:55-108). Field order mirrors RunSettings
 * (inc/config.hpp:18-57). */
typedef struct dgnn_run_cfg {
  int32_t arch;
  int32_t layers;
  int32_t hidden;
  int32_t seq_len;
  int32_t horizon;
  int32_t teacher_forcing;
  int32_t aggr;
  int32_t batch_size;
  uint64_t seed;
  double lr;
  int32_t optimizer; /* 0 sgd, 1 adam */
  int32_t stride;
  double fallback_threshold;
  int32_t rescratch_period;
  int32_t incremental;
  int32_t cache_policy; /* -1 off, 0 reinc, 1 lru, 2 lfu */
  double cache_frac;
  int32_t workers;      /* 0: seq-first session; >= 1: world size of the sharded trainer */
  int32_t epochs;
  int32_t window_total; /* sliding_windows total T' (0 -> T-1) */
  int32_t record_events;
  int64_t hbm_cache_budget_bytes; /* 0 = no second cache level */
  /* ModelConfig::fanouts (inc/model.hpp:37): 0 hops or all -1 = whole-snapshot
   * views; otherwise sampled k-hop views per sample (src/train.cpp:86-98). */
  int32_t n_fanouts;
  int32_t fanouts[8];
  int32_t iteration; /* IterationOrder (inc/train.hpp:17): 0 seq-first, 1 node-first */
} dgnn_run_cfg;

typedef struct dgnn_epoch_report {
  double loss;
  double seconds; /* device-timed */
  int64_t samples;
  int64_t hits, misses, evictions, expirations, invalidations, rejected;
  int64_t scratch_calls, incremental_calls, fallbacks, skipped_steps;
  int64_t spills, refills;
} dgnn_epoch_report;

int dgnn_session_create(dgnn_graph* g, const dgnn_run_cfg* cfg, int32_t rank, void* stream,
                        dgnn_session** out);
void dgnn_session_free(dgnn_session* s);
int64_t dgnn_session_num_params(const dgnn_session* s);
int dgnn_session_num_windows(const dgnn_session* s, int64_t* total, int64_t* local_begin,
                             int64_t* local_end);
/* DgnnModel::flatten_params / unflatten_params (src/model.cpp:91-107). */
int dgnn_session_get_params(dgnn_session* s, double* out);
int dgnn_session_set_params(dgnn_session* s, const double* in);
int dgnn_session_initial_params(dgnn_session* s, double* out);
/* seq_first_epoch (src/train.cpp:146-210); sample losses via dgnn_session_losses. */
int dgnn_session_run_epoch(dgnn_session* s, dgnn_epoch_report* report);
/* Sharded trainer, one call sequence per epoch:
 *   begin_epoch; for b < num_batches: local_grads(b, g); <all-reduce g>; apply(g)
 *   end_epoch. g: device fp32 buffer of num_params floats. */
int dgnn_session_begin_epoch(dgnn_session* s, int64_t* num_batches);
int dgnn_session_local_grads(dgnn_session* s, int64_t batch, float* grad_sum);
int dgnn_session_apply(dgnn_session* s, const float* grad_sum, int32_t* applied);
int dgnn_session_end_epoch(dgnn_session* s);
/* The gradient all-reduce of the sharded trainer (allreduce_sim,
 * inc/distsim.hpp:75 / src/distsim.cpp:248-260) over NCCL: one communicator
 * per rank (NVLink / NVSwitch inside a box). Rank 0 calls dgnn_comm_unique_id
 * and hands the 128 bytes to every rank (file, socket, MPI, ...); each rank
 * then calls dgnn_comm_create with its cudaSetDevice already done. */
int dgnn_comm_unique_id(uint8_t* out128);
int dgnn_comm_create(const uint8_t* id128, int32_t world, int32_t rank, dgnn_comm** out);
void dgnn_comm_free(dgnn_comm* c);
/* In-place fp32 sum over ranks of n values (device pointer), stream-ordered. */
int dgnn_grad_allreduce(dgnn_comm* c, float* data, int64_t n, void* stream);
/* One whole sharded epoch natively (run_distributed_epoch, inc/distsim.hpp:
 * 104-108, src/distsim.cpp:197-272): per batch this rank's window-gradient
 * sum, dgnn_grad_allreduce, the identical optimizer step on every rank.
 * comm may be NULL when cfg.workers == 1. report->seconds is device-timed,
 * max over ranks; sample losses via dgnn_session_losses. */
int dgnn_session_run_dist_epoch(dgnn_session* s, dgnn_comm* comm, dgnn_epoch_report* report);
/* Sample losses of the last epoch (visit order). */
int dgnn_session_losses(dgnn_session* s, double* out, int64_t* n);
/* One sample's forward + backward at the current parameters with a fresh
 * cache/provider: loss, prediction of horizon step 0 (n x d) and flat grads. */
int dgnn_session_sample_grads(dgnn_session* s, int32_t window_index, double* loss, float* pred0,
                              double* grads);
/* Invocation log rows (layer, t, kind, incremental); pass NULL to size. */
int dgnn_session_invocations(dgnn_session* s, int32_t* out, int64_t* n);
/* Cache observer events rows (type, level, layer, t, kind, batch, serial,
 * hit, assigned_f, stored) when record_events; pass NULL to size. */
int dgnn_session_cache_events(dgnn_session* s, int64_t* out, int64_t* n);
/* Cumulative stats: hits misses evictions expirations invalidations rejected
 * scratch incremental fallbacks spills refills peak_units(as int64). */
int dgnn_session_stats(dgnn_session* s, int64_t* out12);
/* Second cache level (HBM <-> pinned host, B200 addition; no reference
 * counterpart): spills refills prefetches demand_refills spill_bytes
 * refill_bytes pinned_bytes hbm_resident_bytes. */
int dgnn_session_tier_stats(dgnn_session* s, int64_t* out8);

/* ------------------------------------------------------- host-side plan logic
 * Pure host functions (no device needed). */
/* sliding_windows (src/windows.cpp:5-15): writes up to cap starts, returns count. */
int64_t dgnn_sliding_windows(int32_t total, int32_t L, int32_t S, int32_t H, int32_t* starts,
                             int64_t cap);
/* plan, consecutive_block (src/distsim.cpp:35-81): out[4m..4m+3] =
 * block_begin, block_end, window_begin, window_end. */
int dgnn_plan(int32_t total, int32_t workers, int32_t L, int32_t S, int32_t H, int64_t* out);
/* Communication ledger of one distributed epoch (CommLedger, inc/distsim.hpp:58-80;
 * accounting of src/distsim.cpp:101-182 and the per-step ring all-reduce,
 * :262-268), placements compared the way the paper's Table 1 does: scheme 0
 * consecutive_block, 1 node_partition, 2 sequence_partition; overlap 0
 * replicate_overlap, 1 remote_fetch. Windows = sliding_windows(T, L, S, H) as in
 * the reference's distributed epoch. out: (workers + 1) x 4 uint64 rows
 * [remote_features, intermediate_redistribution, gradient_sync, snapshot_fetch],
 * per worker then the total; bytes at the reference's 8 B per value. */
int dgnn_comm_ledger(const dgnn_graph* g, int32_t scheme, int32_t overlap, int32_t workers,
                     int32_t seq_len, int32_t stride, int32_t horizon, int32_t hidden,
                     int64_t num_params, int64_t num_batches, uint64_t* out);
/* future_access_count / imminence (src/cache.cpp:27-62); ctx = num_layers,
 * gates, gate, L, S, idx, part, layer, teacher_forcing, H, windows_remaining, kind. */
int dgnn_cache_scores(const int32_t* ctx, int32_t* f, int32_t* imm);
/* AggKeyHash (inc/cache.hpp:54-61). */
uint64_t dgnn_key_hash(int32_t level, int32_t layer, int32_t t, int32_t kind, int64_t batch,
                       int64_t serial);
/* make_batches (src/train.cpp:54-64): out[2i], out[2i+1] = range; returns count. */
int64_t dgnn_make_batches(int32_t num_nodes, int32_t batch_size, uint64_t seed,
                          int64_t epoch_index, int32_t* out, int64_t cap);
/* DgnnModel::create parameter draws (src/model.cpp:41-70) without a device:
 * writes the fp64 flat init (visit order) when out != NULL; returns count. */
int64_t dgnn_init_params(const dgnn_run_cfg* cfg, int32_t feature_dim, double* out);

/* ---------------------------------------------------------------- profiling
 * Device timing per kernel class (0 agg_scratch, 1 agg_delta, 2 agg_backward,
 * 3 cell_fwd, 4 cell_bwd (pointwise), 5 weight_grad, 6 other, 7 cell_bwd_gemm
 * (the dX | dHm contraction), 8 agg_rebase (a hidden aggregation carried
 * across a structural delta), 9 sample = one whole (window, batch) sample)
 * with algorithmic bytes; dgnn_prof_get_max = the longest single scope. */
/* Device memory pool (stream-ordered allocations of every buffer above):
 * reserved / used bytes, current and high-water. */
int dgnn_mem_stats(int64_t* reserved, int64_t* used, int64_t* reserved_high, int64_t* used_high);
int dgnn_prof_enable(int32_t on);
int dgnn_prof_reset(void);
int dgnn_prof_get(int32_t cls, int64_t* launches, double* ms, double* bytes, double* flops);
int dgnn_prof_get_max(int32_t cls, double* max_ms);

#ifdef __cplusplus
}
#endif

#endif /* DGNN_B200_H */
