// Golden-dump / CPU-baseline harness over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY (oracle/). Linked with the reference sources into
// oracle/_ref/libdgnn_ref.so by oracle/Makefile. Exposes a plain C ABI so the
// Python test-suite, tests/golden/make_golden.py and bench.py's reference arm
// can drive the reference's own public API (proj/include/dgnn/*.hpp) without
// any of the product code. Nothing here re-implements reference maths except
// the distributed epoch loop, which the reference cannot execute at S=1
// (last window reads snapshot T, src/train.cpp:100-102) and is
// therefore re-driven from the reference's public pieces exactly as
// src/distsim.cpp:210-272 does.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "dgnn/dataset_io.hpp"
#include "dgnn/distsim.hpp"
#include "dgnn/khop.hpp"
#include "dgnn/synth.hpp"
#include "dgnn/train.hpp"

using namespace dgnn;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = std::string("invalid_argument: ") + e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_err = std::string("out_of_range: ") + e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

Matrix to_matrix(const double* p, int64_t rows, int64_t cols) {
  Matrix m(rows, cols);
  if (rows * cols > 0) std::memcpy(m.data(), p, sizeof(double) * rows * cols);
  return m;
}

void from_matrix(const Matrix& m, double* out) {
  if (m.size() > 0) std::memcpy(out, m.data(), sizeof(double) * m.size());
}

}  // namespace

extern "C" {

// Run configuration shared with python (ctypes mirror in oracle/refbind.py).
struct RefRunCfg {
  int32_t arch;            // Architecture enum order: gcrn_m1, cd_gcn, gcrn_m2, tgcn
  int32_t layers;
  int32_t hidden;
  int32_t seq_len;
  int32_t horizon;
  int32_t teacher_forcing;
  int32_t aggr;            // AggrKind order: sum, mean, max, min
  int32_t batch_size;
  uint64_t seed;
  double lr;
  int32_t optimizer;       // 0 sgd, 1 adam
  int32_t stride;
  double fallback_threshold;
  int32_t rescratch_period;
  int32_t incremental;
  int32_t cache_policy;    // -1 off, 0 reinc, 1 lru, 2 lfu
  double cache_frac;
  int32_t workers;         // 0: seq_first TrainSession semantics; >=1 distsim loop
  int32_t epochs;
  int32_t window_total;    // T' passed to sliding_windows (T-1)
  int32_t record_events;
  int32_t n_fanouts;       // ModelConfig::fanouts (inc/model.hpp:37)
  int32_t fanouts[8];
  int32_t iteration;       // 0 seq-first, 1 node-first
};

const char* ref_last_error() { return g_err.c_str(); }

// ----------------------------------------------------------------- graphs

void* ref_synth(int32_t n, double avg_degree, int32_t dim, int32_t T, double edge_ratio,
                double feat_ratio, uint64_t seed) {
  DynamicGraph* out = nullptr;
  int rc = guarded([&] {
    SynthParams p;
    p.num_nodes = n;
    p.avg_degree = avg_degree;
    p.feature_dim = dim;
    p.num_snapshots = T;
    p.edge_change = ChangeRatio::fixed(edge_ratio);
    p.feature_change = ChangeRatio::fixed(feat_ratio);
    p.seed = seed;
    out = new DynamicGraph(synthesize(p));
  });
  return rc == 0 ? out : nullptr;
}

// Builds a graph from per-snapshot edge lists (concatenated) and features.
void* ref_graph_from_arrays(int32_t n, int32_t dim, int32_t T, const int64_t* edge_counts,
                            const int32_t* src, const int32_t* dst, const double* feats) {
  DynamicGraph* out = nullptr;
  int rc = guarded([&] {
    std::vector<Snapshot> snaps;
    int64_t off = 0;
    for (int32_t t = 0; t < T; ++t) {
      std::vector<Edge> es(edge_counts[t]);
      for (int64_t i = 0; i < edge_counts[t]; ++i) es[i] = {src[off + i], dst[off + i]};
      off += edge_counts[t];
      snaps.emplace_back(t, n, std::move(es),
                         to_matrix(feats + static_cast<int64_t>(t) * n * dim, n, dim));
    }
    out = new DynamicGraph(std::move(snaps));
  });
  return rc == 0 ? out : nullptr;
}

void ref_graph_free(void* g) { delete static_cast<DynamicGraph*>(g); }

// khop / khop_delta / apply_cg_update (src/khop.cpp), unmodified.
void* ref_khop(void* g, int32_t t, const int32_t* seeds, int64_t n_seeds, const int32_t* fanouts,
               int32_t n_hops, uint64_t seed) {
  ComputationalGraph* out = nullptr;
  int rc = guarded([&] {
    const DynamicGraph& G = *static_cast<DynamicGraph*>(g);
    out = new ComputationalGraph(khop(G.snapshot(t), std::vector<NodeId>(seeds, seeds + n_seeds),
                                      std::vector<Fanout>(fanouts, fanouts + n_hops), seed));
  });
  return rc == 0 ? out : nullptr;
}
void ref_cg_free(void* c) { delete static_cast<ComputationalGraph*>(c); }
int32_t ref_cg_num_hops(void* c) { return static_cast<int32_t>(static_cast<ComputationalGraph*>(c)->hops.size()); }
void ref_cg_hop_sizes(void* c, int32_t k, int64_t* nd, int64_t* ne) {
  const HopBlock& h = static_cast<ComputationalGraph*>(c)->hops.at(k);
  *nd = static_cast<int64_t>(h.destinations.size());
  *ne = static_cast<int64_t>(h.edges.size());
}
void ref_cg_hop_copy(void* c, int32_t k, int32_t* dests, int32_t* src, int32_t* dst) {
  const HopBlock& h = static_cast<ComputationalGraph*>(c)->hops.at(k);
  for (size_t i = 0; i < h.destinations.size(); ++i) dests[i] = h.destinations[i];
  for (size_t i = 0; i < h.edges.size(); ++i) {
    src[i] = h.edges[i].src;
    dst[i] = h.edges[i].dst;
  }
}
void ref_cg_view(void* c, int32_t n, int64_t* in_ptr, int32_t* in_src) {
  OwnedView v = static_cast<ComputationalGraph*>(c)->to_view(n);
  std::memcpy(in_ptr, v.in_ptr.data(), sizeof(int64_t) * v.in_ptr.size());
  if (!v.in_src.empty()) std::memcpy(in_src, v.in_src.data(), sizeof(int32_t) * v.in_src.size());
}
void* ref_khop_delta(void* c, void* g, int32_t t) {
  CgUpdate* out = nullptr;
  int rc = guarded([&] {
    const DynamicGraph& G = *static_cast<DynamicGraph*>(g);
    out = new CgUpdate(khop_delta(*static_cast<ComputationalGraph*>(c), G.snapshot(t), G.delta(t)));
  });
  return rc == 0 ? out : nullptr;
}
void ref_cg_update_free(void* u) { delete static_cast<CgUpdate*>(u); }
void ref_cg_update_sizes(void* u, int32_t k, int64_t* na, int64_t* nr) {
  const auto& h = static_cast<CgUpdate*>(u)->hops.at(k);
  *na = static_cast<int64_t>(h.added.size());
  *nr = static_cast<int64_t>(h.removed.size());
}
void ref_cg_update_copy(void* u, int32_t k, int32_t* as, int32_t* ad, int32_t* rs, int32_t* rd) {
  const auto& h = static_cast<CgUpdate*>(u)->hops.at(k);
  for (size_t i = 0; i < h.added.size(); ++i) {
    as[i] = h.added[i].src;
    ad[i] = h.added[i].dst;
  }
  for (size_t i = 0; i < h.removed.size(); ++i) {
    rs[i] = h.removed[i].src;
    rd[i] = h.removed[i].dst;
  }
}
int32_t ref_cg_update_empty(void* u) { return static_cast<CgUpdate*>(u)->empty() ? 1 : 0; }
void* ref_apply_cg_update(void* c, void* u) {
  ComputationalGraph* out = nullptr;
  int rc = guarded([&] {
    out = new ComputationalGraph(
        apply_cg_update(*static_cast<ComputationalGraph*>(c), *static_cast<CgUpdate*>(u)));
  });
  return rc == 0 ? out : nullptr;
}

// save_dataset / load_dataset (src/dataset_io.cpp:40-165), unmodified.
int ref_save_dataset(void* g, const char* dir) {
  return guarded([&] { save_dataset(*static_cast<DynamicGraph*>(g), dir); });
}

void* ref_load_dataset(const char* dir) {
  DynamicGraph* out = nullptr;
  int rc = guarded([&] { out = new DynamicGraph(load_dataset(dir)); });
  return rc == 0 ? out : nullptr;
}

int32_t ref_graph_length(void* g) { return static_cast<DynamicGraph*>(g)->length(); }
int32_t ref_graph_num_nodes(void* g) { return static_cast<DynamicGraph*>(g)->num_nodes(); }
int32_t ref_graph_feature_dim(void* g) { return static_cast<DynamicGraph*>(g)->feature_dim(); }

int64_t ref_snapshot_num_edges(void* g, int32_t t) {
  return static_cast<DynamicGraph*>(g)->snapshot(t).num_edges();
}

// Sorted (src,dst) edge list of snapshot t.
void ref_snapshot_edges(void* g, int32_t t, int32_t* src, int32_t* dst) {
  const auto& es = static_cast<DynamicGraph*>(g)->snapshot(t).edges();
  for (size_t i = 0; i < es.size(); ++i) {
    src[i] = es[i].src;
    dst[i] = es[i].dst;
  }
}

void ref_snapshot_feats(void* g, int32_t t, double* out) {
  from_matrix(static_cast<DynamicGraph*>(g)->snapshot(t).feats(), out);
}

void ref_snapshot_in_csr(void* g, int32_t t, int64_t* ptr, int32_t* src) {
  GraphView v = static_cast<DynamicGraph*>(g)->snapshot(t).view();
  for (NodeId i = 0; i <= v.num_nodes; ++i) ptr[i] = v.in_ptr[i];
  for (EdgeIdx e = 0; e < v.num_edges; ++e) src[e] = v.in_src[e];
}

void ref_snapshot_out_csr(void* g, int32_t t, int64_t* ptr, int32_t* dst) {
  const Snapshot& s = static_cast<DynamicGraph*>(g)->snapshot(t);
  int64_t off = 0;
  for (NodeId u = 0; u < s.num_nodes(); ++u) {
    ptr[u] = off;
    for (NodeId v : s.out_neighbors(u)) dst[off++] = v;
  }
  ptr[s.num_nodes()] = off;
}

int ref_delta_sizes(void* g, int32_t t, int64_t* n_del, int64_t* n_ins, int64_t* n_changed) {
  return guarded([&] {
    const DeltaGraph& d = static_cast<DynamicGraph*>(g)->delta(t);
    *n_del = static_cast<int64_t>(d.deletions.size());
    *n_ins = static_cast<int64_t>(d.insertions.size());
    *n_changed = static_cast<int64_t>(d.changed_nodes.size());
  });
}

int ref_delta_get(void* g, int32_t t, int32_t* del_src, int32_t* del_dst, int32_t* ins_src,
                  int32_t* ins_dst, int32_t* changed, double* changed_feats) {
  return guarded([&] {
    const DeltaGraph& d = static_cast<DynamicGraph*>(g)->delta(t);
    for (size_t i = 0; i < d.deletions.size(); ++i) {
      del_src[i] = d.deletions[i].src;
      del_dst[i] = d.deletions[i].dst;
    }
    for (size_t i = 0; i < d.insertions.size(); ++i) {
      ins_src[i] = d.insertions[i].src;
      ins_dst[i] = d.insertions[i].dst;
    }
    for (size_t i = 0; i < d.changed_nodes.size(); ++i) changed[i] = d.changed_nodes[i];
    from_matrix(d.changed_feats, changed_feats);
  });
}

double ref_change_ratio(void* g, int32_t t) {
  auto* G = static_cast<DynamicGraph*>(g);
  return change_ratio(G->delta(t), G->snapshot(t - 1));
}

// ------------------------------------------------------------ aggregation

namespace {
void dump_agg(const AggResult& r, double* values, double* degree, double* mean_sums,
              int32_t* argext) {
  from_matrix(r.values, values);
  if (degree && r.degree.size() > 0) std::memcpy(degree, r.degree.data(), sizeof(double) * r.degree.size());
  if (mean_sums && r.mean_sums.size() > 0) from_matrix(r.mean_sums, mean_sums);
  if (argext && r.argext.size() > 0)
    std::memcpy(argext, r.argext.data(), sizeof(int32_t) * r.argext.size());
}
}  // namespace

// aggregate_scratch over snapshot t's view with caller-provided features (N x w).
int ref_agg_scratch(void* g, int32_t t, int32_t kind, const double* feats, int32_t w,
                    double* values, double* degree, double* mean_sums, int32_t* argext) {
  return guarded([&] {
    auto* G = static_cast<DynamicGraph*>(g);
    const Snapshot& s = G->snapshot(t);
    AggResult r = aggregate_scratch(s.view(), to_matrix(feats, s.num_nodes(), w),
                                    AggrFn{static_cast<AggrKind>(kind)});
    dump_agg(r, values, degree, mean_sums, argext);
  });
}

// Chain of input aggregations over snapshot features: scratch at t0, then
// aggregate_incremental for t0+1..t1 (each step from the previous result).
// Writes the final AggResult and, per step, (used_fallback, reason, depth).
int ref_agg_chain(void* g, int32_t t0, int32_t t1, int32_t kind, double threshold,
                  int32_t rescratch, double* values, double* degree, double* mean_sums,
                  int32_t* argext, int32_t* step_info) {
  return guarded([&] {
    auto* G = static_cast<DynamicGraph*>(g);
    AggrFn fn{static_cast<AggrKind>(kind)};
    IncrementalOptions opts{threshold, rescratch};
    AggResult cur = aggregate_scratch(G->snapshot(t0).view(), G->snapshot(t0).feats(), fn);
    cur.t = t0;
    for (int32_t t = t0 + 1; t <= t1; ++t) {
      const Snapshot& ps = G->snapshot(t - 1);
      const Snapshot& cs = G->snapshot(t);
      IncrementalResult inc = aggregate_incremental(cur, ps.view(), cs.view(), ps.feats(),
                                                    cs.feats(), G->delta(t), fn, opts);
      step_info[3 * (t - t0 - 1) + 0] = inc.used_fallback ? 1 : 0;
      step_info[3 * (t - t0 - 1) + 1] = static_cast<int32_t>(inc.reason);
      step_info[3 * (t - t0 - 1) + 2] = inc.result.incremental_depth;
      cur = std::move(inc.result);
    }
    dump_agg(cur, values, degree, mean_sums, argext);
  });
}

// aggregate_backward over snapshot t with the forward = scratch of `feats`.
int ref_agg_backward(void* g, int32_t t, int32_t kind, const double* feats, int32_t w,
                     const double* upstream, double* grad) {
  return guarded([&] {
    auto* G = static_cast<DynamicGraph*>(g);
    const Snapshot& s = G->snapshot(t);
    AggrFn fn{static_cast<AggrKind>(kind)};
    AggResult fwd = aggregate_scratch(s.view(), to_matrix(feats, s.num_nodes(), w), fn);
    Matrix gr = aggregate_backward(s.view(), to_matrix(upstream, s.num_nodes(), w), fn, fwd);
    from_matrix(gr, grad);
  });
}

// ------------------------------------------------------------------ cells

namespace {
CellParams cell_from_flat(int32_t kind, int32_t in, int32_t hidden, const double* flat) {
  CellParams p;
  p.kind = static_cast<CellKind>(kind);
  p.in_dim = in;
  p.hidden_dim = hidden;
  const int K = gate_count(p.kind);
  int64_t off = 0;
  for (int g = 0; g < K; ++g) {
    p.wx.push_back(to_matrix(flat + off, in, hidden));
    off += static_cast<int64_t>(in) * hidden;
    p.uh.push_back(to_matrix(flat + off, hidden, hidden));
    off += static_cast<int64_t>(hidden) * hidden;
    p.b.push_back(to_matrix(flat + off, 1, hidden));
    off += hidden;
  }
  return p;
}
}  // namespace

// Cell parameters drawn exactly as CellParams::init does (src/cells.cpp:75-90)
// from an mt19937_64 seeded with `seed`; flat layout [wx_g, uh_g, b_g]_g.
void ref_cell_init(int32_t kind, int32_t in, int32_t hidden, uint64_t seed, double* flat) {
  std::mt19937_64 rng(seed);
  CellParams p;
  p.init(static_cast<CellKind>(kind), in, hidden, rng);
  int64_t off = 0;
  for (size_t g = 0; g < p.wx.size(); ++g) {
    from_matrix(p.wx[g], flat + off);
    off += p.wx[g].size();
    from_matrix(p.uh[g], flat + off);
    off += p.uh[g].size();
    from_matrix(p.b[g], flat + off);
    off += p.b[g].size();
  }
}

// cell_core_forward + cell_core_backward on given operands. Outputs: gates
// (K x N x h, post-activation), hn (GRU), c (LSTM), h; and grads dX, dHm,
// dh_skip (GRU), dc_prev (LSTM), param grads flat (same layout as params).
int ref_cell_fwd_bwd(int32_t kind, int32_t in, int32_t hidden, int32_t n, const double* params,
                     const double* X, const double* Hm, const double* h_skip,
                     const double* c_prev, const double* dh, const double* dc, double* gates,
                     double* hn, double* c, double* h, double* dX, double* dHm,
                     double* dh_skip, double* dc_prev, double* dparams) {
  return guarded([&] {
    CellParams p = cell_from_flat(kind, in, hidden, params);
    Matrix Xm = to_matrix(X, n, in), Hmm = to_matrix(Hm, n, hidden);
    Matrix hs = to_matrix(h_skip, n, hidden);
    Matrix cp = c_prev ? to_matrix(c_prev, n, hidden) : Matrix();
    CellTape tape = cell_core_forward(p, Xm, Hmm, hs, c_prev ? &cp : nullptr);
    for (size_t g = 0; g < tape.gates.size(); ++g) from_matrix(tape.gates[g], gates + g * n * hidden);
    if (p.kind == CellKind::kGru) from_matrix(tape.hn, hn);
    if (p.kind == CellKind::kLstm) from_matrix(tape.c, c);
    from_matrix(tape.h, h);
    ParamMap grads;
    Matrix dhm = to_matrix(dh, n, hidden);
    Matrix dcm = dc ? to_matrix(dc, n, hidden) : Matrix();
    CellCoreGrads cg = cell_core_backward(p, tape, Xm, Hmm, dhm, dc ? &dcm : nullptr, "cell", &grads);
    from_matrix(cg.dX, dX);
    from_matrix(cg.dHm, dHm);
    if (p.kind == CellKind::kGru) from_matrix(cg.dh_skip, dh_skip);
    if (p.kind == CellKind::kLstm) from_matrix(cg.dc_prev, dc_prev);
    int64_t off = 0;
    const int K = gate_count(p.kind);
    for (int g = 0; g < K; ++g) {
      const std::string i = std::to_string(g);
      from_matrix(grads.at("cell/wx" + i), dparams + off);
      off += static_cast<int64_t>(in) * hidden;
      from_matrix(grads.at("cell/uh" + i), dparams + off);
      off += static_cast<int64_t>(hidden) * hidden;
      from_matrix(grads.at("cell/b" + i), dparams + off);
      off += hidden;
    }
  });
}

// ------------------------------------------------------------ model / train

namespace {

ModelConfig model_cfg(const RefRunCfg& c, Eigen::Index feature_dim) {
  ModelConfig m;
  m.arch = static_cast<Architecture>(c.arch);
  m.layers = c.layers;
  m.feature_dim = feature_dim;
  m.hidden_dim = c.hidden;
  m.seq_len = c.seq_len;
  m.horizon = c.horizon;
  m.teacher_forcing = c.teacher_forcing != 0;
  m.aggr = AggrFn{static_cast<AggrKind>(c.aggr)};
  m.fanouts = {kFullFanout, kFullFanout};
  m.seed = c.seed;
  m.fanouts.assign(c.fanouts, c.fanouts + c.n_fanouts);
  return m;
}

TrainConfig train_cfg(const RefRunCfg& c) {
  TrainConfig t;
  t.batch_size = c.batch_size;
  t.epochs = c.epochs;
  t.lr = c.lr;
  t.optimizer = c.optimizer == 0 ? OptimizerKind::kSgd : OptimizerKind::kAdam;
  t.stride = c.stride;
  t.seed = c.seed;
  t.fallback_threshold = c.fallback_threshold;
  t.rescratch_period = c.rescratch_period;
  t.incremental = c.incremental != 0;
  if (c.cache_policy < 0) {
    t.cache_policy = std::nullopt;
  } else {
    t.cache_policy = static_cast<CachePolicy>(c.cache_policy);
  }
  t.cache_capacity_frac = c.cache_frac;
  return t;
}

struct RunResult {
  std::vector<double> params0;
  std::vector<double> params;
  std::vector<double> losses;          // per sample in visit order (all workers)
  std::vector<int64_t> visitation;     // (worker, batch, window)
  std::vector<int32_t> invocations;    // (worker, layer, t, kind, incremental)
  std::vector<int64_t> events;         // (worker, type, level, layer, t, kind, batch, serial, hit, f, stored)
  std::vector<int64_t> stats;          // per worker: hits misses evictions expirations invalidations rejected scratch incr fallbacks skipped
  std::vector<double> peak_units;
  std::vector<double> grads0;          // flat grads of the first sample (seq-first) or the first step (dist)
  double seconds = 0.0;
  int64_t samples = 0;
};

std::vector<double> flatten_grads(DgnnModel& model, const ParamMap& grads) {
  std::vector<double> flat;
  model.visit_params([&](const std::string& name, Matrix* m) {
    auto it = grads.find(name);
    if (it == grads.end()) {
      flat.insert(flat.end(), m->size(), 0.0);
    } else {
      flat.insert(flat.end(), it->second.data(), it->second.data() + it->second.size());
    }
  });
  return flat;
}

void attach_observer(CacheStore* store, RunResult* res, int worker, bool on) {
  if (!store || !on) return;
  store->set_observer([res, worker](const CacheEvent& ev) {
    const AggKey& k = ev.key;
    int64_t row[11] = {worker,
                       static_cast<int64_t>(ev.type),
                       static_cast<int64_t>(k.level),
                       k.layer,
                       k.t,
                       static_cast<int64_t>(k.kind),
                       k.batch,
                       k.step_serial,
                       ev.hit ? 1 : 0,
                       ev.assigned_f,
                       ev.stored ? 1 : 0};
    res->events.insert(res->events.end(), row, row + 11);
  });
}

// MAE over the seed rows of every horizon step, mirroring the reference's
// private seed_loss (src/train.cpp:119-144) through the public loss_mae.
double sample_loss(const SeqSample& sample, const ForwardArtifacts& fwd,
                   std::vector<Matrix>* dpred) {
  const Timestep L = sample.window.length;
  const Timestep H = sample.window.horizon;
  const auto n_seeds = static_cast<Eigen::Index>(sample.seeds.size());
  double total = 0.0;
  for (Timestep j = 0; j < H; ++j) {
    const Matrix& pred = fwd.predictions[j];
    const Matrix& target_full = *sample.feats[L + j + 1];
    Matrix ps(n_seeds, pred.cols()), ts(n_seeds, pred.cols());
    for (Eigen::Index i = 0; i < n_seeds; ++i) {
      ps.row(i) = pred.row(sample.seeds[i]);
      ts.row(i) = target_full.row(sample.seeds[i]);
    }
    MaeLoss l = loss_mae(ps, ts);
    total += l.value;
    Matrix d = Matrix::Zero(pred.rows(), pred.cols());
    for (Eigen::Index i = 0; i < n_seeds; ++i) {
      d.row(sample.seeds[i]) = l.grad.row(i) / static_cast<double>(H);
    }
    dpred->push_back(std::move(d));
  }
  return H > 0 ? total / static_cast<double>(H) : 0.0;
}

std::unique_ptr<CacheStore> make_store(const RefRunCfg& c, const DynamicGraph& g,
                                       const ModelConfig& m) {
  TrainConfig t = train_cfg(c);
  if (!t.cache_policy) return nullptr;
  return std::make_unique<CacheStore>(*t.cache_policy,
                                      t.cache_capacity_frac * cache_data_size_units(g, m));
}

void record_provider(RunResult* res, int worker, AggProvider& prov, size_t inv_from) {
  const auto& inv = prov.stats().invocations;
  for (size_t i = inv_from; i < inv.size(); ++i) {
    int32_t row[5] = {worker, inv[i].layer, inv[i].t, static_cast<int32_t>(inv[i].kind),
                      inv[i].incremental ? 1 : 0};
    res->invocations.insert(res->invocations.end(), row, row + 5);
  }
}

void record_stats(RunResult* res, AggProvider& prov, int64_t skipped) {
  CacheStats cs = prov.store() ? prov.store()->stats() : CacheStats{};
  const ExecutionStats& es = prov.stats();
  int64_t row[10] = {cs.hits, cs.misses, cs.evictions, cs.expirations, cs.invalidations,
                     cs.rejected, es.scratch_calls, es.incremental_calls, es.fallbacks, skipped};
  res->stats.insert(res->stats.end(), row, row + 10);
  res->peak_units.push_back(cs.resident_peak_units);
}

}  // namespace

// Runs `epochs` epochs. workers == 0: seq_first_epoch (TrainSession semantics,
// src/train.cpp:146-206, one Adam step per sample). workers >= 1: the
// distributed consecutive-block loop of src/distsim.cpp:186-272 re-driven from
// public pieces (per-window grads, ordered sum / W, one step per batch).
// Windows are sliding_windows(window_total, L, S, H).
void* ref_run(void* g, const RefRunCfg* cfg) {
  RunResult* res = new RunResult();
  int rc = guarded([&] {
    const DynamicGraph& G = *static_cast<DynamicGraph*>(g);
    const RefRunCfg& c = *cfg;
    ModelConfig mcfg = model_cfg(c, G.feature_dim());
    TrainConfig tcfg = train_cfg(c);
    DgnnModel model = DgnnModel::create(mcfg);
    res->params0 = model.flatten_params();
    auto windows = sliding_windows(c.window_total, mcfg.seq_len, tcfg.stride, mcfg.horizon);
    check(!windows.empty(), "harness: no windows");
    IncrementalOptions inc{tcfg.fallback_threshold, tcfg.rescratch_period};
    OptimizerState opt;
    const int M = c.workers <= 0 ? 1 : c.workers;
    std::vector<std::unique_ptr<CacheStore>> stores;
    std::vector<std::unique_ptr<AggProvider>> provs;
    for (int m = 0; m < M; ++m) {
      stores.push_back(make_store(c, G, mcfg));
      attach_observer(stores.back().get(), res, m, c.record_events != 0);
      provs.push_back(std::make_unique<AggProvider>(stores.back().get(), &G, mcfg.aggr,
                                                    tcfg.incremental, inc));
    }
    std::vector<int64_t> skipped(M, 0);
    const auto t0 = std::chrono::steady_clock::now();
    for (int e = 0; e < c.epochs; ++e) {
      if (c.workers <= 0) {
        EpochReport r = c.iteration == 0
                            ? seq_first_epoch(model, G, windows, tcfg, *provs[0], opt, e)
                            : node_first_epoch(model, G, windows, tcfg, *provs[0], opt, e);
        res->losses.insert(res->losses.end(), r.sample_losses.begin(), r.sample_losses.end());
        for (auto [b, w] : r.visitation) {
          int64_t row[3] = {0, b, w};
          res->visitation.insert(res->visitation.end(), row, row + 3);
        }
        skipped[0] += r.skipped_steps;
        continue;
      }
      // Distributed loop (src/distsim.cpp:197-272) over executable windows.
      const auto W = static_cast<int64_t>(windows.size());
      WorkerPlan pl = plan(PlacementScheme::kConsecutiveBlock, c.window_total, M, mcfg.seq_len,
                           tcfg.stride, mcfg.horizon, OverlapMode::kReplicateOverlap);
      for (int m = 0; m < M; ++m) provs[m]->reset_plan_state();
      auto batches = make_batches(G.num_nodes(), tcfg.batch_size, tcfg.seed, e);
      for (int64_t b = 0; b < static_cast<int64_t>(batches.size()); ++b) {
        std::vector<ParamMap> window_grads(W);
        for (int m = 0; m < M; ++m) {
          const WorkerAssignment& a = pl.workers[m];
          for (int64_t w = a.window_begin; w < a.window_end; ++w) {
            SeqSample sample = build_sample(G, mcfg, windows[w],
                                            static_cast<Timestep>(a.window_end - 1 - w), b,
                                            batches[b], tcfg.seed);
            ForwardArtifacts fwd = model_forward(model, sample, *provs[m]);
            std::vector<Matrix> dpred;
            double mae = sample_loss(sample, fwd, &dpred);
            window_grads[w] = model_backward(model, sample, fwd, dpred);
            res->losses.push_back(mae);
            int64_t row[3] = {m, b, w};
            res->visitation.insert(res->visitation.end(), row, row + 3);
          }
        }
        ParamMap global;
        for (int64_t w = 0; w < W; ++w) {
          for (auto& [name, gm] : window_grads[w]) {
            auto it = global.find(name);
            if (it == global.end()) {
              global[name] = gm;
            } else {
              it->second += gm;
            }
          }
        }
        const double inv = 1.0 / static_cast<double>(W);
        for (auto& [name, gm] : global) gm *= inv;
        if (res->grads0.empty()) res->grads0 = flatten_grads(model, global);
        bool applied = false;
        for (int m = 0; m < M; ++m) {
          if (m == 0) {
            applied = optimizer_step(model, global, opt, tcfg, provs[m]->store());
          } else if (applied && provs[m]->store()) {
            provs[m]->store()->bump_epoch();
          }
        }
        if (!applied)
          for (auto& s : skipped) ++s;
      }
    }
    res->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    res->params = model.flatten_params();
    res->samples = static_cast<int64_t>(res->losses.size());
    for (int m = 0; m < M; ++m) {
      record_provider(res, m, *provs[m], 0);
      record_stats(res, *provs[m], skipped[m]);
    }
  });
  if (rc != 0) {
    delete res;
    return nullptr;
  }
  return res;
}

// One sample's forward + backward at the model's initial parameters (or at
// `params_in` when non-null) with a fresh provider/cache: loss, predictions
// of horizon step 0 and flat grads (visit order, src/model.cpp:72-89).
int ref_sample_grads(void* g, const RefRunCfg* cfg, int32_t window_index,
                     const double* params_in, double* loss, double* pred0, double* grads) {
  return guarded([&] {
    const DynamicGraph& G = *static_cast<DynamicGraph*>(g);
    const RefRunCfg& c = *cfg;
    ModelConfig mcfg = model_cfg(c, G.feature_dim());
    TrainConfig tcfg = train_cfg(c);
    DgnnModel model = DgnnModel::create(mcfg);
    if (params_in) {
      std::vector<double> flat(params_in, params_in + model.flatten_params().size());
      model.unflatten_params(flat);
    }
    auto windows = sliding_windows(c.window_total, mcfg.seq_len, tcfg.stride, mcfg.horizon);
    check(window_index >= 0 && window_index < static_cast<int32_t>(windows.size()),
          "harness: window index");
    auto store = make_store(c, G, mcfg);
    IncrementalOptions inc{tcfg.fallback_threshold, tcfg.rescratch_period};
    AggProvider prov(store.get(), &G, mcfg.aggr, tcfg.incremental, inc);
    auto batches = make_batches(G.num_nodes(), tcfg.batch_size, tcfg.seed, 0);
    SeqSample sample = build_sample(G, mcfg, windows[window_index],
                                    static_cast<Timestep>(windows.size() - 1 - window_index), 0,
                                    batches[0], tcfg.seed);
    ForwardArtifacts fwd = model_forward(model, sample, prov);
    std::vector<Matrix> dpred;
    *loss = sample_loss(sample, fwd, &dpred);
    if (pred0) from_matrix(fwd.predictions[0], pred0);
    ParamMap gm = model_backward(model, sample, fwd, dpred);
    auto flat = flatten_grads(model, gm);
    std::memcpy(grads, flat.data(), sizeof(double) * flat.size());
  });
}

int64_t ref_num_params(void* g, const RefRunCfg* cfg) {
  const DynamicGraph& G = *static_cast<DynamicGraph*>(g);
  DgnnModel model = DgnnModel::create(model_cfg(*cfg, G.feature_dim()));
  return static_cast<int64_t>(model.flatten_params().size());
}

void ref_init_params(void* g, const RefRunCfg* cfg, double* out) {
  const DynamicGraph& G = *static_cast<DynamicGraph*>(g);
  DgnnModel model = DgnnModel::create(model_cfg(*cfg, G.feature_dim()));
  auto flat = model.flatten_params();
  std::memcpy(out, flat.data(), sizeof(double) * flat.size());
}

// Accessors for RunResult: kind 0 params0, 1 params, 2 losses, 3 grads0,
// 4 peak_units (double); 10 visitation, 11 events, 12 stats (int64);
// 20 invocations (int32). Returns element count; copies when out != null.
int64_t ref_run_get(void* h, int32_t kind, void* out) {
  auto* r = static_cast<RunResult*>(h);
  auto put = [&](const auto& v) {
    using T = typename std::decay_t<decltype(v)>::value_type;
    if (out && !v.empty()) std::memcpy(out, v.data(), sizeof(T) * v.size());
    return static_cast<int64_t>(v.size());
  };
  switch (kind) {
    case 0: return put(r->params0);
    case 1: return put(r->params);
    case 2: return put(r->losses);
    case 3: return put(r->grads0);
    case 4: return put(r->peak_units);
    case 10: return put(r->visitation);
    case 11: return put(r->events);
    case 12: return put(r->stats);
    case 20: return put(r->invocations);
  }
  return -1;
}

double ref_run_seconds(void* h) { return static_cast<RunResult*>(h)->seconds; }
void ref_run_free(void* h) { delete static_cast<RunResult*>(h); }

// ---------------------------------------------------------------- misc KATs

void ref_sliding_windows(int32_t total, int32_t L, int32_t S, int32_t H, int32_t* starts,
                         int32_t* count) {
  auto ws = sliding_windows(total, L, S, H);
  *count = static_cast<int32_t>(ws.size());
  if (starts)
    for (size_t i = 0; i < ws.size(); ++i) starts[i] = ws[i].start;
}

int ref_plan(int32_t total, int32_t workers, int32_t L, int32_t S, int32_t H, int64_t* out) {
  return guarded([&] {
    WorkerPlan p = plan(PlacementScheme::kConsecutiveBlock, total, workers, L, S, H,
                        OverlapMode::kReplicateOverlap);
    for (int m = 0; m < workers; ++m) {
      out[4 * m + 0] = p.workers[m].block_begin;
      out[4 * m + 1] = p.workers[m].block_end;
      out[4 * m + 2] = p.workers[m].window_begin;
      out[4 * m + 3] = p.workers[m].window_end;
    }
  });
}

// future_access_count / imminence for an ExecContext given as ints.
int ref_cache_scores(const int32_t* ctx, int32_t* f, int32_t* imm) {
  return guarded([&] {
    ExecContext c;
    c.num_layers = ctx[0];
    c.gates = ctx[1];
    c.gate = ctx[2];
    c.seq_len = ctx[3];
    c.stride = ctx[4];
    c.idx = ctx[5];
    c.part = static_cast<ModelPart>(ctx[6]);
    c.layer = ctx[7];
    c.teacher_forcing = ctx[8] != 0;
    c.horizon = ctx[9];
    c.windows_remaining = ctx[10];
    c.kind = static_cast<AggKeyKind>(ctx[11]);
    *f = future_access_count(c);
    *imm = imminence(c);
  });
}

uint64_t ref_key_hash(int32_t level, int32_t layer, int32_t t, int32_t kind, int64_t batch,
                      int64_t serial) {
  AggKey k{static_cast<CacheLevel>(level), layer, t, static_cast<AggKeyKind>(kind), batch, serial};
  return static_cast<uint64_t>(AggKeyHash{}(k));
}

// run_distributed_epoch under plan(scheme, overlap) (src/distsim.cpp:35-81,
// 186-344), unmodified; returns its CommLedger as (M+1) x 4 rows.
int ref_comm_ledger(void* g, const RefRunCfg* cfg, int32_t scheme, int32_t overlap,
                    uint64_t* out, int64_t* num_params, int64_t* num_batches) {
  return guarded([&] {
    const DynamicGraph& G = *static_cast<DynamicGraph*>(g);
    ModelConfig m = model_cfg(*cfg, G.feature_dim());
    TrainConfig t = train_cfg(*cfg);
    WorkerPlan p = plan(static_cast<PlacementScheme>(scheme), G.length(), cfg->workers, m.seq_len,
                        t.stride, m.horizon, static_cast<OverlapMode>(overlap));
    DgnnModel model = DgnnModel::create(m);
    OptimizerState opt;
    DistributedResult r = run_distributed_epoch(model, G, p, m, t, opt, 0);
    auto put = [&](int row, const CommVolume& v) {
      out[4 * row + 0] = v.remote_features;
      out[4 * row + 1] = v.intermediate_redistribution;
      out[4 * row + 2] = v.gradient_sync;
      out[4 * row + 3] = v.snapshot_fetch;
    };
    for (int i = 0; i < cfg->workers; ++i) put(i, r.ledger.per_worker[i]);
    put(cfg->workers, r.ledger.total);
    *num_params = static_cast<int64_t>(model.flatten_params().size());
    *num_batches = static_cast<int64_t>(make_batches(G.num_nodes(), t.batch_size, t.seed, 0).size());
  });
}

}  // extern "C"
