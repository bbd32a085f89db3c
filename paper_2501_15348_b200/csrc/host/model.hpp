// B200 mirror of dgnn/model.hpp, dgnn/cells.hpp and dgnn/windows.hpp
// (ref proj/include/dgnn/{model,cells,windows}.hpp).
//
// Parameters live in one flat fp32 device buffer in the reference's
// visit_params order (src/model.cpp:72-89), which is also the gradient,
// Adam-state and NCCL all-reduce layout. Each GraphRNN cell additionally keeps
// a packed copy of its weights as one (in+H) x 4H matrix (+ transpose) so the
// gate contractions are single fused kernels; the pack is refreshed after every
// parameter update.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "../dense_kernels.h"
#include "../umma_kernels.h"
#include "engine.hpp"

namespace dgnn {

struct SequenceWindow {
  Timestep start = 0;
  Timestep length = 1;
  Timestep stride = 1;
  Timestep horizon = 0;
  Timestep snapshot_at(Timestep idx) const { return start + idx; }
  friend bool operator==(const SequenceWindow&, const SequenceWindow&) = default;
};

// Starts 0, S, 2S, ... while start + L + H <= T (ref src/windows.cpp:5-15).
std::vector<SequenceWindow> sliding_windows(Timestep total, Timestep length, Timestep stride,
                                            Timestep horizon);

enum class Architecture { kGcrnM1, kCdGcn, kGcrnM2, kTgcn };
enum class CellKind { kLstm, kGru };
inline int gate_count(CellKind k) { return k == CellKind::kLstm ? 4 : 3; }
Architecture architecture_from_string(const std::string& s);
const char* to_string(Architecture a);
bool is_stacked(Architecture a);
CellKind cell_kind_of(Architecture a);

struct ModelConfig {
  Architecture arch = Architecture::kGcrnM2;
  int layers = 2;
  int feature_dim = 0;
  int hidden_dim = 16;
  Timestep seq_len = 8;
  Timestep horizon = 1;
  bool teacher_forcing = true;
  AggrFn aggr;
  uint64_t seed = 1;
  std::vector<int32_t> fanouts;  // empty or all -1: whole-snapshot views (inc/model.hpp:37)
};

// Parameter names in visit_params order (src/model.cpp:72-89) and the fp64
// initial draws in that order (host only, no device needed).
std::vector<std::string> visit_order(const ModelConfig& cfg);
std::vector<double> initial_params_host(const ModelConfig& cfg);

// Whether umma cells drop the gates tape (recompute in the fused backward):
// env DGNN_GATE_TAPE=1 keeps it, =0 drops it, unset decides by tape size.
bool gate_recompute_policy(const ModelConfig& cfg, int64_t num_nodes);

using Buf = std::shared_ptr<cuda::DevArray<float>>;
Buf new_buf(size_t n, cudaStream_t stream);
Buf zero_buf(size_t n, cudaStream_t stream);

struct ParamSlot {
  std::string name;
  int64_t offset = 0;
  int64_t rows = 0, cols = 0;
  int64_t size() const { return rows * cols; }
};

// One GraphRNN / dense recurrent cell's slice of the flat buffer + packs.
struct CellSlot {
  std::string prefix;
  int64_t offset = 0;  // start of [wx_g, uh_g, b_g]_g in the flat buffer
  int in = 0, H = 0;
  bool lstm = true;
  cuda::DevArray<float> W, bias, WT;  // packed (in+H) x 4H, 4H, 4H x (in+H)
  cuda::DevArray<float> dW, db;       // per-sample gradient accumulators
  // tcgen05 B images (3xTF32 hi/lo, canonical UMMA layout): forward W^T,
  // backward W (dX | dHm) and its dHm-only rows.
  bool umma = false;
  // no gates tape: the backward recomputes them inside the fused tcgen05
  // backward kernel (umma cells; see gate_recompute_policy)
  bool recompute = false;
  cuda::DevArray<float> Bf, Bb, Bbh;
  int64_t flat_size() const {
    return static_cast<int64_t>(lstm ? 4 : 3) * (int64_t(in) * H + int64_t(H) * H + H);
  }
};

struct LinearSlot {
  std::string prefix;
  int64_t off_w = 0, off_b = 0;
  int in = 0, out = 0;
  cuda::DevArray<float> WT;  // out x in
  // tcgen05 path (the prediction head): B images of W^T (forward, bias in the
  // epilogue) and W (input gradient, accumulated in the epilogue); the
  // weight / bias gradient through the weight-gradient kernel
  bool umma = false, umma_wgrad = false;
  cuda::DevArray<float> Bf, Bb;
};

class DgnnModel {
 public:
  // Bit-exact with the reference initialisation (src/model.cpp:41-70): fp64
  // draws from mt19937_64(derive_seed(seed, 0x90de1)), uploaded as fp32.
  static std::unique_ptr<DgnnModel> create(const ModelConfig& cfg, cudaStream_t stream);

  const ModelConfig& config() const { return cfg_; }
  int gates() const { return gate_count(cell_kind_of(cfg_.arch)); }
  int64_t num_params() const { return num_params_; }
  const std::vector<ParamSlot>& slots() const { return slots_; }

  // fp64 host images of the parameters (initial draws / current device values).
  std::vector<double> flatten_params();
  void unflatten_params(const std::vector<double>& flat);
  const std::vector<double>& initial_params() const { return init_; }

  float* params() { return params_.get(); }
  void refresh_packed();  // after any parameter change
  // every cell's gradient accumulators (enc, dec, rnn) for one-launch
  // zeroing / unpacking per sample
  const cuda::CellGradDesc* cell_grad_table() const { return cell_grads_.get(); }
  int cell_grad_count() const { return n_cell_grads_; }
  int64_t cell_grad_max_elems() const { return cell_grad_max_; }
  void set_gate_recompute(bool on);

  ModelConfig cfg_;
  std::vector<CellSlot> enc_, dec_, rnn_;
  std::vector<LinearSlot> gcn_;
  LinearSlot head_;
  cudaStream_t stream_ = nullptr;

 private:
  std::vector<ParamSlot> slots_;
  std::vector<double> init_;
  int64_t num_params_ = 0;
  cuda::DevArray<float> params_;
  cuda::DevArray<cuda::CellGradDesc> cell_grads_;
  int n_cell_grads_ = 0;
  int64_t cell_grad_max_ = 0;
};

// One (batch, window) training sample (ref inc/model.hpp:65-73) over
// whole-snapshot device views.
struct SeqSample {
  SequenceWindow window;
  std::vector<GraphView> views;       // L+H views
  std::vector<std::shared_ptr<DevSnapshot>> owned;  // sampled k-hop views (to_view)
  std::vector<const float*> feats;    // L+H+1 feature matrices (device)
  std::vector<FeatRef> feat_refs;     // their version leases (resident while the sample lives)
  // the full snapshots the views are (null for sampled k-hop views): their
  // deltas let the backward merge transposed SpMMs across steps
  const DeviceGraph* graph = nullptr;
  NodeId seed_begin = 0, seed_end = 0;  // loss rows (contiguous node range)
  int64_t batch_id = 0;
  Timestep windows_remaining = 0;
};

SeqSample build_sample(const DeviceGraph& graph, const ModelConfig& mcfg,
                       const SequenceWindow& window, Timestep windows_remaining, int64_t batch_id,
                       std::pair<NodeId, NodeId> node_range, uint64_t seed, cudaStream_t stream);

struct CellTape {
  Buf gates;      // n x 4H (LSTM i,f,g,o; GRU r,z,n,hn)
  Buf c_prev, c;  // LSTM
  Buf h_skip;     // previous hidden state
  Buf h;
};

struct GraphStepTape {
  AggPtr agg_x, agg_h;
  CellTape core;
};

struct GcnTape {
  AggPtr agg;
  Buf out;
};

struct ForwardArtifacts {
  std::vector<Buf> predictions;  // H matrices n x d
  // integrated
  std::vector<std::vector<GraphStepTape>> enc_steps, dec_steps;
  std::vector<const float*> dec_inputs;
  Buf enc_final_pred;
  std::vector<Buf> feedback_keep;
  // stacked
  std::vector<std::vector<GcnTape>> gcn;
  std::vector<std::vector<CellTape>> rnn;
  std::vector<std::vector<Buf>> rnn_in, h_out;
};

// Layer pipelining of the integrated models: layer l of the GraphRNN stack
// runs on lane (l-1) % 2 — lane 0 is the sample's stream, lane 1 an auxiliary
// stream — so layer 2's neighbourhood SpMMs (HBM-bound) overlap layer 1's cell
// GEMMs (tensor-bound) of the next step, and vice versa in BPTT. Cross-layer
// data dependencies are CUDA events; buffers crossing lanes are kept alive
// until the final two-way join, after which every stream-ordered free is safe.
struct Lanes {
  cudaStream_t s[2] = {nullptr, nullptr};
  bool two = false;
  std::vector<cudaEvent_t> events;
  std::vector<Buf> keep;
  Lanes(cudaStream_t main, cudaStream_t aux) : s{main, aux ? aux : main}, two(aux != nullptr) {}
  ~Lanes();
  Lanes(const Lanes&) = delete;
  Lanes& operator=(const Lanes&) = delete;
  cudaStream_t main() const { return s[0]; }
  cudaStream_t of(int layer) const { return two ? s[(layer - 1) & 1] : s[0]; }
  // `to` waits for everything issued so far on `from`
  void dep(cudaStream_t from, cudaStream_t to);
  void join() {
    dep(s[1], s[0]);
    dep(s[0], s[1]);
  }
};

ForwardArtifacts model_forward(DgnnModel& model, const SeqSample& sample, AggProvider& provider);
ForwardArtifacts model_forward(DgnnModel& model, const SeqSample& sample, AggProvider& provider,
                               Lanes& lanes);

// grad (flat, num_params) += gradients of this sample given per-horizon dpred.
void model_backward(DgnnModel& model, const SeqSample& sample, const ForwardArtifacts& fwd,
                    const std::vector<Buf>& dpred, float* grad, cudaStream_t stream);
void model_backward(DgnnModel& model, const SeqSample& sample, const ForwardArtifacts& fwd,
                    const std::vector<Buf>& dpred, float* grad, Lanes& lanes);

// Per-sample MAE on the seed rows of every horizon step (ref src/train.cpp:119-144):
// writes dpred and adds the sample loss (mean over H) into *loss_slot (device).
std::vector<Buf> seed_loss(const SeqSample& sample, const ForwardArtifacts& fwd, int feature_dim,
                           double* loss_slot, double* ws, cudaStream_t stream);

}  // namespace dgnn
