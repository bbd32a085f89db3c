// DgnnModel init / forward / BPTT on device (ref src/model.cpp, src/cells.cpp,
// src/nn.cpp). Control flow, fetch order and gradient routing follow the
// reference; every matrix operation is a device kernel on the provider's stream.
#include "model.hpp"

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <random>

#include "../agg_kernels.h"

namespace dgnn {

std::vector<SequenceWindow> sliding_windows(Timestep total, Timestep length, Timestep stride,
                                            Timestep horizon) {
  check(length >= 1, "sliding_windows: L must be >= 1");
  check(stride >= 1, "sliding_windows: S must be >= 1");
  check(horizon >= 0, "sliding_windows: H must be >= 0");
  std::vector<SequenceWindow> out;
  for (Timestep start = 0; start + length + horizon <= total; start += stride) {
    out.push_back({start, length, stride, horizon});
  }
  return out;
}

Architecture architecture_from_string(const std::string& s) {
  if (s == "gcrn_m1") return Architecture::kGcrnM1;
  if (s == "cd_gcn") return Architecture::kCdGcn;
  if (s == "gcrn_m2") return Architecture::kGcrnM2;
  if (s == "tgcn") return Architecture::kTgcn;
  fail("unknown architecture: " + s);
}

const char* to_string(Architecture a) {
  switch (a) {
    case Architecture::kGcrnM1: return "gcrn_m1";
    case Architecture::kCdGcn: return "cd_gcn";
    case Architecture::kGcrnM2: return "gcrn_m2";
    case Architecture::kTgcn: return "tgcn";
  }
  return "?";
}

bool is_stacked(Architecture a) { return a == Architecture::kGcrnM1 || a == Architecture::kCdGcn; }

CellKind cell_kind_of(Architecture a) {
  return (a == Architecture::kGcrnM1 || a == Architecture::kGcrnM2) ? CellKind::kLstm
                                                                    : CellKind::kGru;
}

Buf new_buf(size_t n, cudaStream_t stream) {
  return std::make_shared<cuda::DevArray<float>>(n, stream);
}
Buf zero_buf(size_t n, cudaStream_t stream) {
  auto b = new_buf(n, stream);
  b->zero(stream);
  return b;
}

// ---------------------------------------------------------------- init
namespace {

struct HostMat {
  int64_t rows = 0, cols = 0;
  std::vector<double> v;
};

// make_linear (ref src/nn.cpp:43-53): weight row-major draws, then bias draws.
void make_linear(int64_t in, int64_t out, std::mt19937_64& rng, HostMat* w, HostMat* b) {
  const double bound = 1.0 / std::sqrt(static_cast<double>(in));
  std::uniform_real_distribution<double> dist(-bound, bound);
  w->rows = in;
  w->cols = out;
  w->v.resize(in * out);
  for (int64_t i = 0; i < in * out; ++i) w->v[i] = dist(rng);
  b->rows = 1;
  b->cols = out;
  b->v.resize(out);
  for (int64_t j = 0; j < out; ++j) b->v[j] = dist(rng);
}

// CellParams::init (ref src/cells.cpp:75-90): per gate make_linear(in,H) then
// make_linear(H,H) whose bias is drawn and discarded.
void cell_init(int gates, int64_t in, int64_t H, std::mt19937_64& rng,
               std::vector<std::pair<std::string, HostMat>>* out, const std::string& prefix) {
  for (int g = 0; g < gates; ++g) {
    HostMat wx, bx, uh, bh;
    make_linear(in, H, rng, &wx, &bx);
    make_linear(H, H, rng, &uh, &bh);
    const std::string i = std::to_string(g);
    out->push_back({prefix + "/wx" + i, std::move(wx)});
    out->push_back({prefix + "/uh" + i, std::move(uh)});
    out->push_back({prefix + "/b" + i, std::move(bx)});
  }
}

// Parameter draws in the reference's init order (src/model.cpp:41-70),
// keyed by visit_params name.
std::map<std::string, HostMat> draw_named(const ModelConfig& cfg) {
  std::mt19937_64 rng(derive_seed(cfg.seed, 0x90de1));
  const int K = gate_count(cell_kind_of(cfg.arch));
  const bool lstm = cell_kind_of(cfg.arch) == CellKind::kLstm;
  const int H = cfg.hidden_dim, d = cfg.feature_dim;
  // draw in the reference's init order, keyed by parameter name
  std::map<std::string, HostMat> named;
  auto take = [&](std::vector<std::pair<std::string, HostMat>>& v) {
    for (auto& kv : v) named[kv.first] = std::move(kv.second);
    v.clear();
  };
  std::vector<std::pair<std::string, HostMat>> tmp;
  if (is_stacked(cfg.arch)) {
    int in = d;
    for (int p = 0; p < cfg.layers; ++p) {
      HostMat w, b;
      make_linear(in, H, rng, &w, &b);
      named["gcn" + std::to_string(p + 1) + "/w"] = std::move(w);
      named["gcn" + std::to_string(p + 1) + "/b"] = std::move(b);
      cell_init(K, H, H, rng, &tmp, "rnn" + std::to_string(p + 1));
      take(tmp);
      in = H;
    }
  } else {
    for (int l = 0; l < cfg.layers; ++l) {
      const int in = l == 0 ? d : H;
      cell_init(K, in, H, rng, &tmp, "enc" + std::to_string(l + 1));
      take(tmp);
      cell_init(K, in, H, rng, &tmp, "dec" + std::to_string(l + 1));
      take(tmp);
    }
  }
  {
    HostMat w, b;
    make_linear(H, d, rng, &w, &b);
    named["head/w"] = std::move(w);
    named["head/b"] = std::move(b);
  }
  return named;
}

}  // namespace

std::vector<double> initial_params_host(const ModelConfig& cfg) {
  check(cfg.layers >= 1, "model needs at least one layer");
  check(cfg.feature_dim >= 1 && cfg.hidden_dim >= 1, "model dims must be positive");
  std::map<std::string, HostMat> named = draw_named(cfg);
  std::vector<double> flat;
  for (const std::string& name : visit_order(cfg)) {
    const HostMat& hm = named.at(name);
    flat.insert(flat.end(), hm.v.begin(), hm.v.end());
  }
  return flat;
}

std::vector<std::string> visit_order(const ModelConfig& cfg) {
  std::vector<std::string> out;
  const int K = gate_count(cell_kind_of(cfg.arch));
  auto cell = [&](const std::string& prefix) {
    for (int g = 0; g < K; ++g) {
      const std::string i = std::to_string(g);
      out.push_back(prefix + "/wx" + i);
      out.push_back(prefix + "/uh" + i);
      out.push_back(prefix + "/b" + i);
    }
  };
  if (!is_stacked(cfg.arch)) {
    for (int l = 0; l < cfg.layers; ++l) cell("enc" + std::to_string(l + 1));
    for (int l = 0; l < cfg.layers; ++l) cell("dec" + std::to_string(l + 1));
  } else {
    for (int p = 0; p < cfg.layers; ++p) {
      out.push_back("gcn" + std::to_string(p + 1) + "/w");
      out.push_back("gcn" + std::to_string(p + 1) + "/b");
    }
    for (int p = 0; p < cfg.layers; ++p) cell("rnn" + std::to_string(p + 1));
  }
  out.push_back("head/w");
  out.push_back("head/b");
  return out;
}

namespace {
// tcgen05 path of a linear layer (the GCN weight transforms and the head):
// y = x W + b (ReLU) and dx = dy W^T through the row GEMM, dW / db through
// the weight-gradient kernel with the output width padded to its 128 / 256
// row tile (linear_wgrad_h)
int linear_wgrad_h(const LinearSlot& l) { return l.out <= 128 ? 32 : 64; }
void set_linear_umma(LinearSlot& l, cudaStream_t stream) {
  // any width up to the row GEMM's N = 256 (narrow / odd widths, e.g. C2's
  // 2-feature head, take the element-copy producer and store epilogue)
  l.umma = cuda::umma_enabled() && l.in >= 1 && l.out >= 1 && l.out <= 256 && l.in <= 256;
  l.umma_wgrad = l.umma && l.out <= 256 && l.in + linear_wgrad_h(l) <= 192;
  if (l.umma) {
    l.Bf = cuda::DevArray<float>(cuda::umma_bimage_floats(l.out, l.in), stream);
    l.Bb = cuda::DevArray<float>(cuda::umma_bimage_floats(l.in, l.out), stream);
  }
}
}  // namespace

std::unique_ptr<DgnnModel> DgnnModel::create(const ModelConfig& cfg, cudaStream_t stream) {
  check(cfg.layers >= 1, "model needs at least one layer");
  check(cfg.feature_dim >= 1 && cfg.hidden_dim >= 1, "model dims must be positive");
  auto m = std::make_unique<DgnnModel>();
  m->cfg_ = cfg;
  m->stream_ = stream;
  const int K = gate_count(cell_kind_of(cfg.arch));
  const bool lstm = cell_kind_of(cfg.arch) == CellKind::kLstm;
  const int H = cfg.hidden_dim, d = cfg.feature_dim;
  std::map<std::string, HostMat> named = draw_named(cfg);
  // flat layout in visit order (ref src/model.cpp:72-89)
  int64_t off = 0;
  auto add_slot = [&](const std::string& name) {
    const HostMat& hm = named.at(name);
    m->slots_.push_back({name, off, hm.rows, hm.cols});
    m->init_.insert(m->init_.end(), hm.v.begin(), hm.v.end());
    off += hm.rows * hm.cols;
  };
  auto add_cell = [&](const std::string& prefix, int in, std::vector<CellSlot>* dst) {
    CellSlot c;
    c.prefix = prefix;
    c.offset = off;
    c.in = in;
    c.H = H;
    c.lstm = lstm;
    for (int g = 0; g < K; ++g) {
      const std::string i = std::to_string(g);
      add_slot(prefix + "/wx" + i);
      add_slot(prefix + "/uh" + i);
      add_slot(prefix + "/b" + i);
    }
    const int64_t KW = static_cast<int64_t>(in + H) * 4 * H;
    c.W = cuda::DevArray<float>(KW, stream);
    c.WT = cuda::DevArray<float>(KW, stream);
    c.bias = cuda::DevArray<float>(4 * H, stream);
    c.dW = cuda::DevArray<float>(KW, stream);
    c.db = cuda::DevArray<float>(4 * H, stream);
    c.umma = cuda::umma_cell_supported(in, H);
    if (c.umma) {
      c.Bf = cuda::DevArray<float>(cuda::umma_bimage_floats(4 * H, in + H), stream);
      c.Bb = cuda::DevArray<float>(cuda::umma_bimage_floats(in + H, 4 * H), stream);
      c.Bbh = cuda::DevArray<float>(cuda::umma_bimage_floats(H, 4 * H), stream);
    }
    dst->push_back(std::move(c));
  };
  if (!is_stacked(cfg.arch)) {
    for (int l = 0; l < cfg.layers; ++l) add_cell("enc" + std::to_string(l + 1), l == 0 ? d : H, &m->enc_);
    for (int l = 0; l < cfg.layers; ++l) add_cell("dec" + std::to_string(l + 1), l == 0 ? d : H, &m->dec_);
  } else {
    for (int p = 0; p < cfg.layers; ++p) {
      LinearSlot g;
      g.prefix = "gcn" + std::to_string(p + 1);
      g.in = p == 0 ? d : H;
      g.out = H;
      g.off_w = off;
      add_slot(g.prefix + "/w");
      g.off_b = off;
      add_slot(g.prefix + "/b");
      g.WT = cuda::DevArray<float>(static_cast<size_t>(g.in) * H, stream);
      set_linear_umma(g, stream);
      m->gcn_.push_back(std::move(g));
    }
    for (int p = 0; p < cfg.layers; ++p) add_cell("rnn" + std::to_string(p + 1), H, &m->rnn_);
  }
  m->head_.prefix = "head";
  m->head_.in = H;
  m->head_.out = d;
  m->head_.off_w = off;
  add_slot("head/w");
  m->head_.off_b = off;
  add_slot("head/b");
  m->head_.WT = cuda::DevArray<float>(static_cast<size_t>(H) * d, stream);
  set_linear_umma(m->head_, stream);
  m->num_params_ = off;
  m->params_ = cuda::DevArray<float>(off, stream);
  {
    std::vector<cuda::CellGradDesc> descs;
    for (auto* cells : {&m->enc_, &m->dec_, &m->rnn_})
      for (auto& c : *cells) {
        descs.push_back({c.dW.get(), c.db.get(), c.lstm ? 1 : 0, c.in, c.H, c.offset});
        m->cell_grad_max_ = std::max<int64_t>(m->cell_grad_max_, static_cast<int64_t>(c.in + c.H + 1) * 4 * c.H);
      }
    m->n_cell_grads_ = static_cast<int>(descs.size());
    m->cell_grads_ = cuda::DevArray<cuda::CellGradDesc>(std::max<size_t>(descs.size(), 1), stream);
    if (!descs.empty())
      DGNN_CUDA(cudaMemcpyAsync(m->cell_grads_.get(), descs.data(), sizeof(cuda::CellGradDesc) * descs.size(),
                                cudaMemcpyHostToDevice, stream));
  }
  m->unflatten_params(m->init_);
  return m;
}

std::vector<double> DgnnModel::flatten_params() {
  std::vector<float> f(num_params_);
  copy_to_host(f.data(), params_.get(), sizeof(float) * num_params_, stream_);
  return std::vector<double>(f.begin(), f.end());
}

void DgnnModel::unflatten_params(const std::vector<double>& flat) {
  check(static_cast<int64_t>(flat.size()) == num_params_, "parameter buffer size mismatch");
  std::vector<float> f(flat.begin(), flat.end());
  DGNN_CUDA(cudaMemcpyAsync(params_.get(), f.data(), sizeof(float) * num_params_,
                            cudaMemcpyHostToDevice, stream_));
  DGNN_CUDA(cudaStreamSynchronize(stream_));
  refresh_packed();
}

void DgnnModel::refresh_packed() {
  auto pack = [&](CellSlot& c) {
    cuda::pack_cell(c.lstm, c.in, c.H, params_.get() + c.offset, c.W.get(), c.bias.get(), stream_);
    cuda::transpose(c.in + c.H, 4 * c.H, c.W.get(), c.WT.get(), stream_);
    if (c.umma) {
      const int K = c.in + c.H, NC = 4 * c.H;
      cuda::umma_pack_cell_image(c.lstm, c.W.get(), c.in, c.H, c.Bf.get(), stream_);  // W^T
      cuda::umma_pack_b(c.W.get(), NC, false, 0, K, NC, c.Bb.get(), stream_);      // W
      cuda::umma_pack_b(c.W.get(), NC, false, c.in, c.H, NC, c.Bbh.get(), stream_);  // W[in:]
    }
  };
  for (auto& c : enc_) pack(c);
  for (auto& c : dec_) pack(c);
  for (auto& c : rnn_) pack(c);
  auto pack_linear = [&](LinearSlot& l) {
    cuda::transpose(l.in, l.out, params_.get() + l.off_w, l.WT.get(), stream_);
    if (l.umma) {
      const float* W = params_.get() + l.off_w;  // in x out, row-major
      cuda::umma_pack_b(W, l.out, true, 0, l.out, l.in, l.Bf.get(), stream_);   // W^T
      cuda::umma_pack_b(W, l.out, false, 0, l.in, l.out, l.Bb.get(), stream_);  // W
    }
  };
  for (auto& g : gcn_) pack_linear(g);
  pack_linear(head_);
}

SeqSample build_sample(const DeviceGraph& graph, const ModelConfig& mcfg,
                       const SequenceWindow& window, Timestep windows_remaining, int64_t batch_id,
                       std::pair<NodeId, NodeId> node_range, uint64_t seed, cudaStream_t stream) {
  SeqSample s;
  s.window = window;
  s.batch_id = batch_id;
  s.windows_remaining = windows_remaining;
  s.seed_begin = node_range.first;
  s.seed_end = node_range.second;
  const Timestep span = window.length + window.horizon;
  bool whole = true;  // full_fanouts (src/train.cpp:68-73)
  for (int32_t f : mcfg.fanouts)
    if (f != -1) whole = false;
  if (whole) s.graph = &graph;
  std::vector<int32_t> seeds;
  if (!whole)
    for (NodeId v = node_range.first; v < node_range.second; ++v) seeds.push_back(v);
  for (Timestep i = 0; i < span; ++i) {
    const Timestep t = window.start + i;
    if (whole) {
      s.views.push_back(GraphView::of(graph, t));
      continue;
    }
    // sampled k-hop view of snapshot t (src/train.cpp:93-97), built on the
    // device on the graph's stream, ordered before `stream`
    const DevSnapshot& snap = graph.snapshot(t);
    DevCompGraph cg = khop(snap, graph.num_nodes(), seeds, mcfg.fanouts,
                           derive_seed(seed, static_cast<uint64_t>(t)), stream);
    const DevHop& deep = cg.hops.back();
    s.owned.push_back(std::make_shared<DevSnapshot>(
        csr_from_keys(deep.edges.get(), deep.n_edges, graph.num_nodes(), stream)));
    const DevSnapshot& o = *s.owned.back();
    GraphView v;
    v.num_nodes = graph.num_nodes();
    v.num_edges = o.num_edges;
    v.in_ptr = o.in_ptr.get();
    v.in_src = o.in_src.get();
    v.out_ptr = o.out_ptr.get();
    v.out_dst = o.out_dst.get();
    v.t = t;
    s.views.push_back(v);
  }
  // snapshot(t) bound check reproduces the reference's .at()
  for (Timestep i = 0; i <= span; ++i) {
    s.feat_refs.push_back(graph.features(window.start + i, stream));
    s.feats.push_back(s.feat_refs.back()->get());
  }
  return s;
}

// ---------------------------------------------------------------- forward
namespace {

ExecContext make_ctx(const DgnnModel& model, const SeqSample& sample, ModelPart part, Timestep idx,
                     int layer, int gate, AggKeyKind kind) {
  ExecContext ctx;
  ctx.num_layers = model.cfg_.layers;
  ctx.gates = model.gates();
  ctx.gate = gate;
  ctx.seq_len = sample.window.length;
  ctx.stride = sample.window.stride;
  ctx.idx = idx;
  ctx.part = part;
  ctx.layer = layer;
  ctx.teacher_forcing = model.cfg_.teacher_forcing;
  ctx.horizon = sample.window.horizon;
  ctx.windows_remaining = sample.windows_remaining;
  ctx.kind = kind;
  return ctx;
}

double cell_flops(int64_t n, int in, int H) { return 2.0 * n * (in + H) * 4.0 * H; }

}  // namespace

// DGNN_UMMA_PARTS (experiments): bit 1 cell forward / recompute, 2 the dX|dHm
// contraction, 4 the weight gradient on tcgen05 (default all)
static int umma_parts() {
  static const int p = [] {
    const char* e = std::getenv("DGNN_UMMA_PARTS");
    return e ? std::atoi(e) : 7;
  }();
  return p;
}

bool gate_recompute_policy(const ModelConfig& cfg, int64_t num_nodes) {
  if (const char* e = std::getenv("DGNN_GATE_TAPE")) return e[0] == '0';
  // auto: drop the gates tape when it would take more than 24 GB per sample
  // (C4: 4M nodes x 4H x 9 steps x 2 layers = 74 GB; C3 keeps its 18 GB tape,
  // which measured ~2% faster than the recompute)
  const double tape = 4.0 * num_nodes * 4 * cfg.hidden_dim *
                      static_cast<double>(cfg.seq_len + cfg.horizon) * cfg.layers;
  return tape > 24e9;
}

void DgnnModel::set_gate_recompute(bool on) {
  for (auto* cells : {&enc_, &dec_, &rnn_})
    for (auto& c : *cells) c.recompute = c.umma && on && (umma_parts() & 1);
}

namespace {

// cell_core_forward on device operands (ref src/cells.cpp:102-132).
CellTape cell_forward(const CellSlot& c, NodeId n, const float* X, const float* Hm, const Buf& h_skip,
                      const Buf& c_prev, cudaStream_t st) {
  CellTape t;
  if (!c.recompute) t.gates = new_buf(static_cast<size_t>(n) * 4 * c.H, st);
  t.h = new_buf(static_cast<size_t>(n) * c.H, st);
  t.h_skip = h_skip;
  if (c.lstm) {
    t.c_prev = c_prev;
    t.c = new_buf(static_cast<size_t>(n) * c.H, st);
  }
  // X, Hm, W + (gates), h (c, c_prev) traffic
  const double bytes =
      4.0 * n * (c.in + c.H + (c.recompute ? 0 : 4 * c.H) + c.H + (c.lstm ? 2 * c.H : c.H));
  ProfScope ps(kProfCellFwd, st, bytes, cell_flops(n, c.in, c.H));
  if (c.umma && (umma_parts() & 1)) {
    cuda::umma_cell_forward(c.lstm, n, c.in, c.H, X, Hm, h_skip->get(),
                            c.lstm ? c_prev->get() : nullptr, c.Bf.get(), c.bias.get(),
                            t.gates ? t.gates->get() : nullptr, c.lstm ? t.c->get() : nullptr,
                            t.h->get(), st);
  } else {
    cuda::cell_forward(c.lstm, n, c.in, c.H, X, Hm, h_skip->get(), c.lstm ? c_prev->get() : nullptr,
                       c.W.get(), c.bias.get(), t.gates->get(), c.lstm ? t.c->get() : nullptr,
                       t.h->get(), st);
  }
  return t;
}

Buf linear_forward(DgnnModel& m, const LinearSlot& lin, NodeId n, const float* x, bool relu,
                   cudaStream_t st) {
  Buf y = new_buf(static_cast<size_t>(n) * lin.out, st);
  ProfScope ps(kProfOther, st, 4.0 * n * (lin.in + lin.out), 2.0 * n * lin.in * lin.out);
  if (lin.umma) {
    // split accumulators (RowGemmArgs::split_acc): the head's outputs are the
    // predictions the MAE sign reads
    cuda::umma_gemm_store2(n, lin.in, x, lin.Bf.get(), lin.out, 0, y->get(), nullptr, st,
                           m.params() + lin.off_b, false, 0, relu, true);
  } else {
    cuda::gemm_nn(n, lin.in, 0, lin.out, 0, x, nullptr, m.params() + lin.off_w, lin.out,
                  m.params() + lin.off_b, relu, false, y->get(), nullptr, st);
  }
  return y;
}

void run_stack_step(DgnnModel& model, std::vector<CellSlot>& cells, const SeqSample& sample,
                    AggProvider& provider, ModelPart part, Timestep pos, Timestep t,
                    const GraphView& view, const float* x, bool x_is_data, std::vector<Buf>* h,
                    std::vector<Buf>* c, std::vector<GraphStepTape>* tapes, Lanes& lanes) {
  const int D = model.cfg_.layers;
  const int K = model.gates();
  const NodeId n = view.num_nodes;
  for (int l = 1; l <= D; ++l) {
    cudaStream_t st = lanes.of(l);
    // layer l consumes layer l-1's output of this step (other lane)
    if (l > 1) lanes.dep(lanes.of(l - 1), st);
    provider.set_stream(st);
    provider.begin_cell_step();
    const CellSlot& cell = cells[l - 1];
    const float* x_src = l == 1 ? x : (*h)[l - 2]->get();
    const int x_dim = cell.in;
    GraphStepTape tape;
    for (int g = 1; g <= K; ++g) {
      if (l == 1 && x_is_data) {
        tape.agg_x = provider.fetch_input(sample.batch_id, t, view, x_src, x_dim,
                                          make_ctx(model, sample, part, pos, 1, g, AggKeyKind::kInput));
      } else {
        tape.agg_x = provider.fetch_hidden(
            sample.batch_id, t, l, AggKeyKind::kHiddenPrevLayer, view, x_src, x_dim,
            make_ctx(model, sample, part, pos, l, g, AggKeyKind::kHiddenPrevLayer));
      }
      tape.agg_h = provider.fetch_hidden(
          sample.batch_id, t, l, AggKeyKind::kHiddenPrevT, view, (*h)[l - 1]->get(), cell.H,
          make_ctx(model, sample, part, pos, l, g, AggKeyKind::kHiddenPrevT));
    }
    tape.core = cell_forward(cell, n, tape.agg_x->dense_values(), tape.agg_h->dense_values(),
                             (*h)[l - 1], cell.lstm ? (*c)[l - 1] : nullptr, st);
    (*h)[l - 1] = tape.core.h;
    if (cell.lstm) (*c)[l - 1] = tape.core.c;
    tapes->push_back(std::move(tape));
  }
  provider.set_stream(lanes.main());
}

ForwardArtifacts seq2seq_forward(DgnnModel& model, const SeqSample& sample, AggProvider& provider,
                                 Lanes& lanes) {
  const ModelConfig& cfg = model.cfg_;
  check(!is_stacked(cfg.arch), "seq2seq_forward needs an integrated model");
  const Timestep L = sample.window.length, H = sample.window.horizon;
  check(static_cast<Timestep>(sample.views.size()) == L + H, "sample views must cover L+H steps");
  check(static_cast<Timestep>(sample.feats.size()) == L + H + 1,
        "sample features must cover L+H+1 snapshots");
  cudaStream_t st = lanes.main();
  const NodeId n = sample.views[0].num_nodes;
  const int D = cfg.layers;
  const bool lstm = cell_kind_of(cfg.arch) == CellKind::kLstm;
  std::vector<Buf> h(D), c;
  for (int l = 0; l < D; ++l) {
    h[l] = zero_buf(static_cast<size_t>(n) * cfg.hidden_dim, st);
    provider.note_zero(h[l]->get());
  }
  if (lstm) {
    c.resize(D);
    for (int l = 0; l < D; ++l) c[l] = zero_buf(static_cast<size_t>(n) * cfg.hidden_dim, st);
  }
  lanes.dep(st, lanes.s[1]);  // initial states (and the caller's zeroed grads) visible to lane 1
  ForwardArtifacts out;
  out.enc_steps.resize(L);
  for (Timestep idx = 0; idx < L; ++idx) {
    run_stack_step(model, model.enc_, sample, provider, ModelPart::kEncoder, idx,
                   sample.window.snapshot_at(idx), sample.views[idx], sample.feats[idx], true, &h,
                   &c, &out.enc_steps[idx], lanes);
  }
  cudaStream_t top = lanes.of(D);  // head / feedback on the top layer's lane
  if (!cfg.teacher_forcing) out.enc_final_pred = linear_forward(model, model.head_, n, h[D - 1]->get(), false, top);
  out.dec_steps.resize(H);
  Buf feedback = out.enc_final_pred;
  for (Timestep j = 0; j < H; ++j) {
    const Timestep t = sample.window.start + L + j;
    const bool forced = cfg.teacher_forcing;
    if (!forced) lanes.dep(top, lanes.of(1));  // fed-back prediction -> layer 1
    const float* x = forced ? sample.feats[L + j] : feedback->get();
    out.dec_inputs.push_back(x);
    if (!forced) out.feedback_keep.push_back(feedback);
    run_stack_step(model, model.dec_, sample, provider, ModelPart::kDecoder, j, t,
                   sample.views[L + j], x, forced, &h, &c, &out.dec_steps[j], lanes);
    Buf pred = linear_forward(model, model.head_, n, h[D - 1]->get(), false, top);
    feedback = pred;
    out.predictions.push_back(pred);
  }
  return out;
}

ForwardArtifacts stacked_forward(DgnnModel& model, const SeqSample& sample, AggProvider& provider) {
  const ModelConfig& cfg = model.cfg_;
  check(is_stacked(cfg.arch), "stacked_forward needs a stacked model");
  const Timestep L = sample.window.length, H = sample.window.horizon;
  cudaStream_t st = provider.stream();
  const NodeId n = sample.views[0].num_nodes;
  const int P = cfg.layers;
  const bool lstm = cell_kind_of(cfg.arch) == CellKind::kLstm;
  ForwardArtifacts out;
  out.gcn.resize(P);
  out.rnn.resize(P);
  out.rnn_in.resize(P);
  out.h_out.resize(P);
  std::vector<const float*> inputs;
  std::vector<Buf> keep_inputs(L);
  for (Timestep idx = 0; idx < L; ++idx) inputs.push_back(sample.feats[idx]);
  Buf h_final;
  for (int p = 0; p < P; ++p) {
    const LinearSlot& gcn = model.gcn_[p];
    for (Timestep idx = 0; idx < L; ++idx) {
      const Timestep t = sample.window.snapshot_at(idx);
      const GraphView& view = sample.views[idx];
      AggPtr agg;
      if (p == 0) {
        ExecContext ctx = make_ctx(model, sample, ModelPart::kEncoder, idx, 1, 1, AggKeyKind::kInput);
        ctx.gates = 1;
        ctx.num_layers = 1;
        agg = provider.fetch_input(sample.batch_id, t, view, inputs[idx], gcn.in, ctx);
      } else {
        agg = provider.compute_uncached(p + 1, t, AggKeyKind::kHiddenPrevLayer, view, inputs[idx], gcn.in);
      }
      GcnTape gt;
      gt.agg = agg;
      gt.out = linear_forward(model, gcn, n, agg->dense_values(), true, st);  // ReLU, no norm
      out.gcn[p].push_back(std::move(gt));
    }
    Buf h = zero_buf(static_cast<size_t>(n) * cfg.hidden_dim, st);
    Buf c = lstm ? zero_buf(static_cast<size_t>(n) * cfg.hidden_dim, st) : nullptr;
    for (Timestep idx = 0; idx < L; ++idx) {
      const Buf& x = out.gcn[p][idx].out;
      out.rnn_in[p].push_back(x);
      CellTape tape = cell_forward(model.rnn_[p], n, x->get(), h->get(), h, c, st);
      h = tape.h;
      if (lstm) c = tape.c;
      out.rnn[p].push_back(tape);
      out.h_out[p].push_back(h);
      inputs[idx] = h->get();
      keep_inputs[idx] = h;
    }
    h_final = h;
  }
  Buf pred = linear_forward(model, model.head_, n, h_final->get(), false, st);
  for (Timestep j = 0; j < H; ++j) out.predictions.push_back(pred);
  return out;
}

// ---------------------------------------------------------------- backward
bool backward_merge_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("DGNN_BACKWARD_MERGE");
    return !(e && e[0] == '0');
  }();
  return on;
}

struct Grads {
  float* flat;
  float* ws;  // gemm_tn workspace
};

void linear_param_grads(DgnnModel& m, const LinearSlot& lin, NodeId n, const float* x,
                        const float* dy, Grads& g, cudaStream_t st) {
  ProfScope ps(kProfWeightGrad, st, 4.0 * n * (lin.in + lin.out), 2.0 * n * lin.in * lin.out);
  if (lin.umma_wgrad) {  // dW (in x out) += x^T dy, db += colsum(dy)
    cuda::umma_wgrad(n, lin.in, linear_wgrad_h(lin), dy, x, nullptr, g.flat + lin.off_w, lin.out,
                     g.flat + lin.off_b, g.ws, st, lin.out);
  } else {
    cuda::gemm_tn_acc(n, lin.in, 0, lin.out, x, nullptr, dy, g.flat + lin.off_w, lin.out,
                      g.flat + lin.off_b, g.ws, st);
  }
  (void)m;
}

struct StepGrads {
  Buf dx, dh_prev, dc_prev;
  Buf dHm_deferred;  // HmRoute::kDefer: dHm, still to go through A_{t-1}^T
};

// How a graph step's hidden gradient dHm reaches dh_prev.
//   kFull   dh_prev = A_t^T dHm (+ GRU skip)
//   kSkip   the step is the window's first: dh_prev is the gradient of the
//           zero initial state, which nothing reads — no transposed SpMM
//   kDefer  dh_prev = (GRU skip) + Delta_t^T dHm, dHm handed back: the layer
//           above folds it into its input gradient at step t-1, whose
//           transposed SpMM runs over A_{t-1} (A_t = A_{t-1} + Delta_t), so
//           two SpMMs over the snapshot become one plus the structural delta
struct HmRoute {
  enum Mode { kFull, kSkip, kDefer } mode = kFull;
  const DevDelta* delta = nullptr;  // kDefer: delta t (snapshot t from t-1)
};

// cell_core_backward + the graph-step scatter (ref src/cells.cpp:134-236).
// `X`/`Hm` are the operands the forward used; `agg_x`/`agg_h` (graph steps)
// route dX/dHm back through aggregate_backward; null for dense steps.
StepGrads cell_step_backward(CellSlot& c, const CellTape& tape, const float* X, const float* Hm,
                             const AggResult* agg_x, const AggResult* agg_h, const GraphView* view,
                             const Buf& dh, const Buf& dc, bool need_dx, Grads& g, cudaStream_t st,
                             float* dx_into = nullptr, const Buf& dx_fold = nullptr,
                             HmRoute hm_route = {}) {
  // dx_into (graph steps): accumulate the input gradient straight into the
  // layer below's running dh instead of returning dx
  // dx_fold: the layer below's deferred dHm of step t+1 (n x in), added to dX
  // before its transposed SpMM (over A_t; see HmRoute)
  const NodeId n = view ? view->num_nodes : static_cast<NodeId>(tape.h->size() / c.H);
  const int H = c.H, in = c.in;
  Buf G = new_buf(static_cast<size_t>(n) * 4 * H, st);
  StepGrads out;
  Buf dh_skip;
  if (c.recompute) {
    // X, Hm, state, dh (dc) in; G, dc_prev / dh_skip out
    ProfScope ps(kProfCellBwd, st, 4.0 * n * (in + H + H + H + (c.lstm && dc ? H : 0) + 4 * H + H),
                 cell_flops(n, in, H));
    Buf& dstate = c.lstm ? out.dc_prev : dh_skip;
    dstate = new_buf(static_cast<size_t>(n) * H, st);
    cuda::umma_cell_backward_recompute(c.lstm, n, in, H, X, Hm, tape.h_skip->get(),
                                       c.lstm ? tape.c_prev->get() : nullptr, c.Bf.get(),
                                       c.bias.get(), dh->get(), dc ? dc->get() : nullptr, G->get(),
                                       dstate->get(), st);
  } else {
    ProfScope ps(kProfCellBwd, st, 4.0 * n * (4 * H + 4 * H + 4 * H));
    if (c.lstm) {
      out.dc_prev = new_buf(static_cast<size_t>(n) * H, st);
      cuda::cell_backward_pointwise(true, n, H, tape.gates->get(), tape.c->get(), tape.c_prev->get(),
                                    nullptr, dh->get(), dc ? dc->get() : nullptr, G->get(),
                                    out.dc_prev->get(), nullptr, st);
    } else {
      dh_skip = new_buf(static_cast<size_t>(n) * H, st);
      cuda::cell_backward_pointwise(false, n, H, tape.gates->get(), nullptr, nullptr,
                                    tape.h_skip->get(), dh->get(), nullptr, G->get(), nullptr,
                                    dh_skip->get(), st);
    }
  }
  {
    ProfScope ps(kProfWeightGrad, st, 4.0 * n * (in + H + 4 * H), cell_flops(n, in, H));
    if (c.umma && (umma_parts() & 4)) {
      cuda::umma_wgrad(n, in, H, G->get(), X, Hm, c.dW.get(), c.lstm ? 4 * H : 3 * H, c.db.get(),
                       g.ws, st);
    } else {
      cuda::gemm_tn_acc(n, in, H, 4 * H, X, Hm, G->get(), c.dW.get(), c.lstm ? 4 * H : 3 * H,
                        c.db.get(), g.ws, st);
    }
  }
  // dX accumulates onto dx_fold in the GEMM epilogue where it can
  const bool fold_in_gemm = dx_fold && c.umma && (umma_parts() & 2) && in % 16 == 0 && H % 16 == 0;
  Buf dX = need_dx ? (fold_in_gemm ? dx_fold : new_buf(static_cast<size_t>(n) * in, st)) : nullptr;
  // the window's first step needs no dHm (HmRoute::kSkip); without dX either
  // the contraction is skipped
  const bool skip_gemm = view != nullptr && hm_route.mode == HmRoute::kSkip && !need_dx;
  Buf dHm = skip_gemm ? nullptr : new_buf(static_cast<size_t>(n) * H, st);
  if (!skip_gemm) {
    ProfScope ps(kProfCellBwdGemm, st,
                 4.0 * n * (4 * H + (need_dx ? in : 0) + H + (fold_in_gemm ? in : 0)),
                 2.0 * n * 4 * H * ((need_dx ? in : 0) + H));
    if (c.umma && (umma_parts() & 2)) {
      if (need_dx) {
        cuda::umma_gemm_store2(n, 4 * H, G->get(), c.Bb.get(), in, H, dX->get(), dHm->get(), st,
                               nullptr, fold_in_gemm, c.lstm ? 0 : H);
      } else {
        cuda::umma_gemm_store2(n, 4 * H, G->get(), c.Bbh.get(), H, 0, dHm->get(), nullptr, st,
                               nullptr, false, c.lstm ? 0 : H);
      }
    } else if (need_dx) {
      cuda::gemm_nn(n, 4 * H, 0, in, H, G->get(), nullptr, c.WT.get(), in + H, nullptr, false,
                    false, dX->get(), dHm->get(), st);
    } else {
      cuda::gemm_nn(n, 4 * H, 0, H, 0, G->get(), nullptr, c.WT.get() + in, in + H, nullptr, false,
                    false, dHm->get(), nullptr, st);
    }
  }
  if (need_dx && dx_fold && !fold_in_gemm)
    cuda::axpy(static_cast<int64_t>(n) * in, 1.f, dx_fold->get(), dX->get(), st);
  if (view == nullptr) {  // dense step (stacked RNN): dx = dX, dh_prev = dHm (+ skip)
    out.dx = dX;
    out.dh_prev = dHm;
    if (!c.lstm) cuda::axpy(static_cast<int64_t>(n) * H, 1.f, dh_skip->get(), out.dh_prev->get(), st);
    return out;
  }
  // empty max/min rows contributed zeros; their gradient stops (src/cells.cpp:222-230)
  if (agg_x->extremal() && need_dx)
    cuda::mask_empty_rows(n, in, agg_x->argext.get(), dX->get(), dX->get(), st);
  if (agg_h->extremal() && dHm) cuda::mask_empty_rows(n, H, agg_h->argext.get(), dHm->get(), dHm->get(), st);
  // GRU: dh_prev = A^T dHm + dh_skip, the skip term added inside the SpMM
  if (hm_route.mode == HmRoute::kSkip) {
    out.dh_prev = c.lstm ? nullptr : dh_skip;
  } else if (hm_route.mode == HmRoute::kDefer) {
    out.dh_prev = c.lstm ? zero_buf(static_cast<size_t>(n) * H, st) : dh_skip;
    check(aggregate_backward_delta(*hm_route.delta, n, dHm->get(), H, out.dh_prev->get(), st),
          "deferred hidden gradient: unsupported shape");
    out.dHm_deferred = dHm;
  } else {
    out.dh_prev = new_buf(static_cast<size_t>(n) * H, st);
    aggregate_backward(*view, dHm->get(), H, AggrFn{agg_h->kind}, *agg_h, out.dh_prev->get(), st,
                       c.lstm ? nullptr : dh_skip->get());
  }
  if (need_dx) {
    if (dx_into != nullptr) {
      aggregate_backward(*view, dX->get(), in, AggrFn{agg_x->kind}, *agg_x, dx_into, st, dx_into);
    } else {
      out.dx = new_buf(static_cast<size_t>(n) * in, st);
      aggregate_backward(*view, dX->get(), in, AggrFn{agg_x->kind}, *agg_x, out.dx->get(), st);
    }
  }
  return out;
}

void head_backward(DgnnModel& model, NodeId n, const float* h_top, const Buf& dpred, Buf& dh,
                   Grads& g, cudaStream_t st) {
  linear_param_grads(model, model.head_, n, h_top, dpred->get(), g, st);
  // dh += dpred * W_head^T
  ProfScope ps(kProfOther, st, 4.0 * n * (model.head_.out + 2 * model.head_.in));
  if (model.head_.umma) {
    cuda::umma_gemm_store2(n, model.head_.out, dpred->get(), model.head_.Bb.get(), model.head_.in, 0,
                           dh->get(), nullptr, st, nullptr, /*accumulate=*/true);
  } else {
    cuda::gemm_nn(n, model.head_.out, 0, model.head_.in, 0, dpred->get(), nullptr,
                  model.head_.WT.get(), model.head_.in, nullptr, false, true, dh->get(), nullptr, st);
  }
}

void integrated_backward(DgnnModel& model, const SeqSample& sample, const ForwardArtifacts& fwd,
                         const std::vector<Buf>& dpred, Grads* g, Lanes& lanes) {
  const ModelConfig& cfg = model.cfg_;
  const Timestep L = sample.window.length, H = sample.window.horizon;
  const NodeId n = sample.views[0].num_nodes;
  const int D = cfg.layers;
  const bool lstm = cell_kind_of(cfg.arch) == CellKind::kLstm;
  auto lane_of = [&](int l) { return lanes.two ? (l - 1) & 1 : 0; };
  std::vector<Buf> dh(D), dc(D);
  // layer l's dHm of the step after the current one, deferred to layer l+1's
  // input gradient (HmRoute::kDefer)
  std::vector<Buf> deferred(D);
  const bool merge = sample.graph != nullptr && backward_merge_enabled();
  for (int l = 0; l < D; ++l) {
    dh[l] = zero_buf(static_cast<size_t>(n) * cfg.hidden_dim, lanes.of(l + 1));
    if (lstm) dc[l] = zero_buf(static_cast<size_t>(n) * cfg.hidden_dim, lanes.of(l + 1));
  }
  auto step = [&](std::vector<CellSlot>& cells, const std::vector<GraphStepTape>& tapes,
                  const GraphView& view, Timestep pos) {
    for (int l = D; l >= 1; --l) {
      cudaStream_t st = lanes.of(l);
      const GraphStepTape& tape = tapes[l - 1];
      // layer l's input gradient accumulates straight into the layer below's
      // running dh inside the transposed SpMM (no dx buffer, no axpy); with
      // two lanes that buffer belongs to layer l-1's lane, so the SpMM is
      // ordered after its last write and before its next use
      float* dx_into = l > 1 ? dh[l - 2]->get() : nullptr;
      if (l > 1) lanes.dep(lanes.of(l - 1), st);
      HmRoute route;
      const bool sum_h = tape.agg_h->kind == AggrKind::kSum;
      if (pos == 0) {
        route.mode = HmRoute::kSkip;
      } else if (merge && l < D && sum_h && tapes[l].agg_x->kind == AggrKind::kSum &&
                 cells[l].in == cells[l - 1].H && view.t >= 1 && view.t < sample.graph->length()) {
        route.mode = HmRoute::kDefer;
        route.delta = &sample.graph->delta(view.t);
      }
      Buf fold = l > 1 ? std::move(deferred[l - 2]) : nullptr;
      StepGrads sg = cell_step_backward(cells[l - 1], tape.core, tape.agg_x->dense_values(),
                                        tape.agg_h->dense_values(), tape.agg_x.get(),
                                        tape.agg_h.get(), &view, dh[l - 1], lstm ? dc[l - 1] : nullptr,
                                        l > 1, g[lane_of(l)], st, dx_into, fold, route);
      if (l > 1) lanes.dep(st, lanes.of(l - 1));
      deferred[l - 1] = std::move(sg.dHm_deferred);
      dh[l - 1] = sg.dh_prev;
      if (lstm) dc[l - 1] = sg.dc_prev;
      // layer-1 inputs are data or stop-gradient feedback: dx is never formed
    }
  };
  cudaStream_t top = lanes.of(D);
  for (Timestep j = H - 1; j >= 0; --j) {
    const GraphStepTape& ts = fwd.dec_steps[j][D - 1];
    head_backward(model, n, ts.core.h->get(), dpred[j], dh[D - 1], g[lane_of(D)], top);
    step(model.dec_, fwd.dec_steps[j], sample.views[L + j], L + j);
  }
  for (Timestep idx = L - 1; idx >= 0; --idx) step(model.enc_, fwd.enc_steps[idx], sample.views[idx], idx);
  lanes.join();
}

void stacked_backward(DgnnModel& model, const SeqSample& sample, const ForwardArtifacts& fwd,
                      const std::vector<Buf>& dpred, Grads& g, cudaStream_t st) {
  const ModelConfig& cfg = model.cfg_;
  const Timestep L = sample.window.length;
  const NodeId n = sample.views[0].num_nodes;
  const int P = cfg.layers;
  const int Hd = cfg.hidden_dim;
  const bool lstm = cell_kind_of(cfg.arch) == CellKind::kLstm;
  Buf dh_final = zero_buf(static_cast<size_t>(n) * Hd, st);
  const Buf& h_final = fwd.h_out[P - 1][L - 1];
  for (const Buf& dp : dpred) head_backward(model, n, h_final->get(), dp, dh_final, g, st);
  std::vector<std::vector<Buf>> dh_extra(P, std::vector<Buf>(L));
  dh_extra[P - 1][L - 1] = dh_final;
  for (int p = P - 1; p >= 0; --p) {
    Buf dh = zero_buf(static_cast<size_t>(n) * Hd, st);
    Buf dc = lstm ? zero_buf(static_cast<size_t>(n) * Hd, st) : nullptr;
    const LinearSlot& gcn = model.gcn_[p];
    for (Timestep idx = L - 1; idx >= 0; --idx) {
      if (dh_extra[p][idx]) cuda::axpy(static_cast<int64_t>(n) * Hd, 1.f, dh_extra[p][idx]->get(), dh->get(), st);
      const CellTape& tape = fwd.rnn[p][idx];
      StepGrads sg = cell_step_backward(model.rnn_[p], tape, fwd.rnn_in[p][idx]->get(),
                                        tape.h_skip->get(), nullptr, nullptr, nullptr, dh,
                                        lstm ? dc : nullptr, true, g, st);
      dh = sg.dh_prev;
      if (lstm) dc = sg.dc_prev;
      // gcn_backward (ref src/cells.cpp:57-73)
      const GcnTape& gt = fwd.gcn[p][idx];
      Buf dpre = new_buf(static_cast<size_t>(n) * Hd, st);
      cuda::relu_backward(static_cast<int64_t>(n) * Hd, gt.out->get(), sg.dx->get(), dpre->get(), st);
      linear_param_grads(model, gcn, n, gt.agg->dense_values(), dpre->get(), g, st);
      if (p == 0) continue;  // pair-1 input gradient is discarded by the reference
      Buf dnormed = new_buf(static_cast<size_t>(n) * gcn.in, st);
      {
        ProfScope ps(kProfOther, st, 4.0 * n * (Hd + gcn.in), 2.0 * n * Hd * gcn.in);
        if (gcn.umma) {
          cuda::umma_gemm_store2(n, Hd, dpre->get(), gcn.Bb.get(), gcn.in, 0, dnormed->get(), nullptr, st);
        } else {
          cuda::gemm_nn(n, Hd, 0, gcn.in, 0, dpre->get(), nullptr, gcn.WT.get(), gcn.in, nullptr, false,
                        false, dnormed->get(), nullptr, st);
        }
      }
      if (gt.agg->extremal())
        cuda::mask_empty_rows(n, gcn.in, gt.agg->argext.get(), dnormed->get(), dnormed->get(), st);
      Buf dinput = new_buf(static_cast<size_t>(n) * gcn.in, st);
      aggregate_backward(sample.views[idx], dnormed->get(), gcn.in, AggrFn{gt.agg->kind}, *gt.agg,
                         dinput->get(), st);
      if (dh_extra[p - 1][idx]) {
        cuda::axpy(static_cast<int64_t>(n) * Hd, 1.f, dinput->get(), dh_extra[p - 1][idx]->get(), st);
      } else {
        dh_extra[p - 1][idx] = dinput;
      }
    }
  }
}

}  // namespace

Lanes::~Lanes() {
  for (cudaEvent_t e : events) cudaEventDestroy(e);
}

void Lanes::dep(cudaStream_t from, cudaStream_t to) {
  if (from == to) return;
  if (events.empty()) {
    cudaEvent_t e;
    DGNN_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    events.push_back(e);
  }
  // a wait binds to the record preceding it, so one event can be re-recorded
  cudaEvent_t e = events[0];
  DGNN_CUDA(cudaEventRecord(e, from));
  DGNN_CUDA(cudaStreamWaitEvent(to, e, 0));
}

ForwardArtifacts model_forward(DgnnModel& model, const SeqSample& sample, AggProvider& provider,
                               Lanes& lanes) {
  if (is_stacked(model.cfg_.arch)) {
    provider.begin_forward(false);
    ForwardArtifacts out = stacked_forward(model, sample, provider);
    provider.end_forward();
    return out;
  }
  cudaStream_t prev = provider.stream();
  provider.set_stream(lanes.main());
  provider.begin_forward(true);
  ForwardArtifacts out = seq2seq_forward(model, sample, provider, lanes);
  provider.end_forward();
  provider.set_stream(prev);
  return out;
}

ForwardArtifacts model_forward(DgnnModel& model, const SeqSample& sample, AggProvider& provider) {
  Lanes lanes(provider.stream(), nullptr);
  return model_forward(model, sample, provider, lanes);
}

void model_backward(DgnnModel& model, const SeqSample& sample, const ForwardArtifacts& fwd,
                    const std::vector<Buf>& dpred, float* grad, cudaStream_t stream) {
  Lanes lanes(stream, nullptr);
  model_backward(model, sample, fwd, dpred, grad, lanes);
}

void model_backward(DgnnModel& model, const SeqSample& sample, const ForwardArtifacts& fwd,
                    const std::vector<Buf>& dpred, float* grad, Lanes& lanes) {
  cudaStream_t stream = lanes.main();
  check(dpred.size() == fwd.predictions.size(), "model_backward: dpred arity mismatch");
  const NodeId n = sample.views[0].num_nodes;
  const int H = model.cfg_.hidden_dim;
  const int d = model.cfg_.feature_dim;
  int64_t ws_n = 0;
  for (int in : {d, H}) {
    ws_n = std::max(ws_n, cuda::gemm_tn_workspace(n, in + H, 4 * H));  // cells
    ws_n = std::max(ws_n, cuda::gemm_tn_workspace(n, in, H));          // gcn
  }
  ws_n = std::max(ws_n, cuda::gemm_tn_workspace(n, H, d));             // head
  for (int in : {d, H})
    if (cuda::umma_cell_supported(in, H)) ws_n = std::max(ws_n, cuda::umma_wgrad_workspace(n, in, H));
  if (model.head_.umma_wgrad)
    ws_n = std::max(ws_n, cuda::umma_wgrad_workspace(n, model.head_.in, linear_wgrad_h(model.head_)));
  for (const LinearSlot& gl : model.gcn_)
    if (gl.umma_wgrad) ws_n = std::max(ws_n, cuda::umma_wgrad_workspace(n, gl.in, linear_wgrad_h(gl)));
  cuda::DevArray<float> ws(ws_n, stream);
  cuda::zero_cell_grads(model.cell_grad_table(), model.cell_grad_count(), model.cell_grad_max_elems(), stream);
  if (is_stacked(model.cfg_.arch)) {
    Grads g{grad, ws.get()};
    stacked_backward(model, sample, fwd, dpred, g, stream);
  } else {
    // one gemm_tn workspace per lane; accumulator zeroing visible to lane 1
    cuda::DevArray<float> ws1(lanes.two ? ws_n : 0, lanes.s[1]);
    lanes.dep(stream, lanes.s[1]);
    Grads g[2] = {{grad, ws.get()}, {grad, lanes.two ? ws1.get() : ws.get()}};
    integrated_backward(model, sample, fwd, dpred, g, lanes);  // ends joined
  }
  cuda::unpack_cell_grads(model.cell_grad_table(), model.cell_grad_count(), model.cell_grad_max_elems(), grad,
                          stream);
}

std::vector<Buf> seed_loss(const SeqSample& sample, const ForwardArtifacts& fwd, int feature_dim,
                           double* loss_slot, double* ws, cudaStream_t stream) {
  const Timestep L = sample.window.length, H = sample.window.horizon;
  const NodeId n = sample.views[0].num_nodes;
  std::vector<Buf> dpred;
  for (Timestep j = 0; j < H; ++j) {
    Buf d = new_buf(static_cast<size_t>(n) * feature_dim, stream);
    cuda::mae_loss(n, feature_dim, sample.seed_begin, sample.seed_end, fwd.predictions[j]->get(),
                   sample.feats[L + j + 1], d->get(), 1.0 / static_cast<double>(H), loss_slot, ws,
                   stream);
    dpred.push_back(std::move(d));
  }
  return dpred;
}

}  // namespace dgnn
