// extern "C" boundary (include/dgnn_b200.h) over the B200 host layer.
#include "../../include/dgnn_b200.h"

#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "host/dataset_io.hpp"
#include "host/synth.hpp"
#include "umma_kernels.h"
#include "host/train.hpp"

using namespace dgnn;

struct dgnn_graph {
  std::unique_ptr<DeviceGraph> g;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  FeatRef last_feats;  // keeps the version returned by dgnn_graph_snapshot resident
};

struct dgnn_synth {
  CompactGraph cg;
  // Pinned-host mirror of the compact graph (built on first upload): the
  // per-epoch host->HBM upload then runs at DMA speed.
  struct Pinned {
    void* arena = nullptr;
    const int32_t *base_src = nullptr, *base_dst = nullptr;
    const float* base_feats = nullptr;
    struct Step {
      const int32_t *del_src, *del_dst, *ins_src, *ins_dst, *changed;
      const float* changed_feats;
    };
    std::vector<Step> steps;
  } pin;
  ~dgnn_synth() {
    if (pin.arena) cudaFreeHost(pin.arena);
  }
  void ensure_pinned() {
    if (pin.arena) return;
    size_t bytes = 0;
    auto add = [&](size_t b) { bytes += (b + 255) / 256 * 256; };
    add(cg.base_src.size() * 4);
    add(cg.base_dst.size() * 4);
    add(cg.base_feats.size() * 4);
    for (const auto& s : cg.steps) {
      add(s.del_src.size() * 4);
      add(s.del_dst.size() * 4);
      add(s.ins_src.size() * 4);
      add(s.ins_dst.size() * 4);
      add(s.changed.size() * 4);
      add(s.changed_feats.size() * 4);
    }
    DGNN_CUDA(cudaMallocHost(&pin.arena, bytes + 256));
    char* cur = static_cast<char*>(pin.arena);
    auto put = [&](const auto& v) {
      using T = typename std::decay_t<decltype(v)>::value_type;
      T* dst = reinterpret_cast<T*>(cur);
      if (!v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(T));
      cur += (v.size() * sizeof(T) + 255) / 256 * 256;
      return const_cast<const T*>(dst);
    };
    pin.base_src = put(cg.base_src);
    pin.base_dst = put(cg.base_dst);
    pin.base_feats = put(cg.base_feats);
    for (const auto& s : cg.steps) {
      Pinned::Step p;
      p.del_src = put(s.del_src);
      p.del_dst = put(s.del_dst);
      p.ins_src = put(s.ins_src);
      p.ins_dst = put(s.ins_dst);
      p.changed = put(s.changed);
      p.changed_feats = put(s.changed_feats);
      pin.steps.push_back(p);
    }
  }
};

struct dgnn_session {
  dgnn_graph* graph = nullptr;
  dgnn_run_cfg cfg{};
  ModelConfig mcfg;
  TrainConfig tcfg;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::unique_ptr<TrainSession> seq;
  std::unique_ptr<DistWorker> dist;
  std::vector<double> losses;
  std::vector<int64_t> events;
  DgnnModel& model() { return seq ? seq->model() : dist->model(); }
  Worker& worker() { return seq ? seq->worker() : dist->worker(); }
  Timestep window_total() const {
    return cfg.window_total > 0 ? cfg.window_total : graph->g->length() - 1;
  }
};

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// Pinned staging buffer reused across the loader's steps (grown on demand).
struct PinnedStage {
  void* p = nullptr;
  size_t cap = 0;
  ~PinnedStage() {
    if (p) cudaFreeHost(p);
  }
  template <class T>
  T* put(size_t& off, const std::vector<T>& v) {
    T* d = reinterpret_cast<T*>(static_cast<char*>(p) + off);
    if (!v.empty()) std::memcpy(d, v.data(), v.size() * sizeof(T));
    off += (v.size() * sizeof(T) + 255) / 256 * 256;
    return d;
  }
  void reserve(size_t bytes) {
    if (bytes <= cap) return;
    if (p) DGNN_CUDA(cudaFreeHost(p));
    p = nullptr;
    DGNN_CUDA(cudaMallocHost(&p, bytes));
    cap = bytes;
  }
};

size_t staged_bytes(const CompactStep& s) {
  auto r = [](size_t b) { return (b + 255) / 256 * 256; };
  return r(s.del_src.size() * 4) + r(s.del_dst.size() * 4) + r(s.ins_src.size() * 4) +
         r(s.ins_dst.size() * 4) + r(s.changed.size() * 4) + r(s.changed_feats.size() * 4);
}

}  // namespace

extern "C" {

const char* dgnn_last_error(void) { return g_err.c_str(); }
const char* dgnn_version(void) { return "paper_2501_15348_b200 0.1 (sm_100a)"; }
int64_t dgnn_launch_count(void) { return cuda::launch_counter(); }
int dgnn_synchronize(void* stream) {
  return guarded([&] { DGNN_CUDA(cudaStreamSynchronize(as_stream(stream))); });
}

int dgnn_set_device(int32_t device) {
  return guarded([&] { DGNN_CUDA(cudaSetDevice(device)); });
}

// ------------------------------------------------------------------ graph
int dgnn_graph_create(int32_t num_nodes, int32_t feature_dim, void* stream, dgnn_graph** out) {
  return guarded([&] {
    auto h = std::make_unique<dgnn_graph>();
    if (stream) {
      h->stream = as_stream(stream);
    } else {
      DGNN_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
      h->own_stream = true;
    }
    h->g = std::make_unique<DeviceGraph>(num_nodes, feature_dim, h->stream);
    *out = h.release();
  });
}

void dgnn_graph_free(dgnn_graph* g) {
  if (!g) return;
  cudaStream_t s = g->stream;
  bool own = g->own_stream;
  g->last_feats.reset();  // leases end before their slots and stream
  g->g.reset();
  cudaStreamSynchronize(s);
  if (own) {
    cuda::release_stream_blocks(s);
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
  }
  delete g;
}

int dgnn_graph_add_snapshot(dgnn_graph* g, const int32_t* src, const int32_t* dst,
                            int64_t num_edges, const float* feats) {
  return guarded([&] { g->g->add_snapshot(src, dst, num_edges, feats); });
}

int dgnn_graph_add_delta(dgnn_graph* g, const int32_t* del_src, const int32_t* del_dst,
                         int64_t n_del, const int32_t* ins_src, const int32_t* ins_dst,
                         int64_t n_ins, const int32_t* changed_nodes, int64_t n_changed,
                         const float* changed_feats) {
  return guarded([&] {
    g->g->add_delta(del_src, del_dst, n_del, ins_src, ins_dst, n_ins, changed_nodes, n_changed,
                    changed_feats);
  });
}

int dgnn_graph_retain(dgnn_graph* g, int32_t t_first, int32_t t_last) {
  return guarded([&] { g->g->retain(t_first, t_last); });
}

int32_t dgnn_graph_length(const dgnn_graph* g) { return g->g->length(); }

int64_t dgnn_graph_num_edges(const dgnn_graph* g, int32_t t) {
  try {
    return g->g->snapshot(t).num_edges;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int64_t dgnn_graph_device_bytes(const dgnn_graph* g) {
  try {
    return g->g->device_bytes();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int dgnn_graph_feature_stats(const dgnn_graph* g, int32_t* slots, int64_t* materialisations) {
  return guarded([&] {
    if (slots) *slots = g->g->feature_slots();
    if (materialisations) *materialisations = g->g->feature_materialisations();
  });
}

int dgnn_graph_snapshot(const dgnn_graph* g, int32_t t, const int64_t** in_ptr,
                        const int32_t** in_src, const int64_t** out_ptr, const int32_t** out_dst,
                        const float** feats) {
  return guarded([&] {
    const DevSnapshot& s = g->g->snapshot(t);
    if (in_ptr) *in_ptr = s.in_ptr.get();
    if (in_src) *in_src = s.in_src.get();
    if (out_ptr) *out_ptr = s.out_ptr.get();
    if (out_dst) *out_dst = s.out_dst.get();
    if (feats) {
      auto* mg = const_cast<dgnn_graph*>(g);
      mg->last_feats = g->g->features(t, g->stream);
      DGNN_CUDA(cudaStreamSynchronize(g->stream));
      *feats = mg->last_feats->get();
    }
  });
}

int dgnn_graph_delta_sizes(const dgnn_graph* g, int32_t t, int64_t* n_del, int64_t* n_ins,
                           int64_t* n_changed, int64_t* n_rows, int64_t* u_minus,
                           int64_t* u_plus) {
  return guarded([&] {
    const DevDelta& d = g->g->delta(t);
    if (n_del) *n_del = d.n_del;
    if (n_ins) *n_ins = d.n_ins;
    if (n_changed) *n_changed = d.n_changed;
    if (n_rows) *n_rows = d.n_rows;
    if (u_minus) *u_minus = d.u_minus;
    if (u_plus) *u_plus = d.u_plus;
  });
}

int dgnn_graph_delta_copy(const dgnn_graph* g, int32_t t, int32_t* del_src, int32_t* del_dst,
                          int32_t* ins_src, int32_t* ins_dst, int32_t* changed_nodes) {
  return guarded([&] {
    const DevDelta& d = g->g->delta(t);
    auto split = [&](const cuda::DevArray<uint64_t>& keys, int64_t n, int32_t* s, int32_t* dd) {
      std::vector<uint64_t> h(n);
      copy_to_host(h.data(), keys.get(), sizeof(uint64_t) * n, g->stream);
      for (int64_t i = 0; i < n; ++i) {
        if (s) s[i] = static_cast<int32_t>(h[i] >> 32);
        if (dd) dd[i] = static_cast<int32_t>(h[i] & 0xffffffffu);
      }
    };
    split(d.del, d.n_del, del_src, del_dst);
    split(d.ins, d.n_ins, ins_src, ins_dst);
    if (changed_nodes) copy_to_host(changed_nodes, d.changed.get(), sizeof(int32_t) * d.n_changed, g->stream);
  });
}

int dgnn_graph_delta_layout(const dgnn_graph* g, int32_t t, const int32_t** rows,
                            const int32_t** row_ptr, const int32_t** ent) {
  return guarded([&] {
    const DevDelta& d = g->g->delta(t);
    if (rows) *rows = d.rows.get();
    if (row_ptr) *row_ptr = d.row_ptr.get();
    if (ent) *ent = d.ent.get();
  });
}

double dgnn_graph_change_ratio(const dgnn_graph* g, int32_t t) {
  try {
    return change_ratio(g->g->delta(t), g->g->snapshot(t - 1).num_edges);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1.0;
  }
}

// ------------------------------------------------------------------ synth
int dgnn_synth_create(int32_t num_nodes, double avg_degree, int32_t feature_dim,
                      int32_t num_snapshots, double edge_change, double feature_change,
                      uint64_t seed, dgnn_synth** out) {
  return guarded([&] {
    SynthParams p;
    p.num_nodes = num_nodes;
    p.avg_degree = avg_degree;
    p.feature_dim = feature_dim;
    p.num_snapshots = num_snapshots;
    p.edge_change = edge_change;
    p.feature_change = feature_change;
    p.seed = seed;
    auto s = std::make_unique<dgnn_synth>();
    s->cg = synthesize_compact(p);
    *out = s.release();
  });
}

void dgnn_synth_free(dgnn_synth* s) { delete s; }

int dgnn_synth_sizes(const dgnn_synth* s, int64_t* sizes) {
  return guarded([&] {
    sizes[0] = static_cast<int64_t>(s->cg.base_src.size());
    for (size_t i = 0; i < s->cg.steps.size(); ++i) {
      sizes[1 + 3 * i] = static_cast<int64_t>(s->cg.steps[i].del_src.size());
      sizes[2 + 3 * i] = static_cast<int64_t>(s->cg.steps[i].ins_src.size());
      sizes[3 + 3 * i] = static_cast<int64_t>(s->cg.steps[i].changed.size());
    }
  });
}

int dgnn_synth_base(const dgnn_synth* s, const int32_t** src, const int32_t** dst,
                    const float** feats) {
  return guarded([&] {
    *src = s->cg.base_src.data();
    *dst = s->cg.base_dst.data();
    *feats = s->cg.base_feats.data();
  });
}

int dgnn_synth_step(const dgnn_synth* s, int32_t t, const int32_t** del_src,
                    const int32_t** del_dst, const int32_t** ins_src, const int32_t** ins_dst,
                    const int32_t** changed, const float** changed_feats) {
  return guarded([&] {
    const CompactStep& st = s->cg.steps.at(t - 1);
    *del_src = st.del_src.data();
    *del_dst = st.del_dst.data();
    *ins_src = st.ins_src.data();
    *ins_dst = st.ins_dst.data();
    *changed = st.changed.data();
    *changed_feats = st.changed_feats.data();
  });
}

int dgnn_synth_to_graph(const dgnn_synth* s, void* stream, dgnn_graph** out) {
  return guarded([&] {
    dgnn_graph* g = nullptr;
    if (dgnn_graph_create(s->cg.num_nodes, s->cg.feature_dim, stream, &g) != 0)
      throw std::runtime_error(g_err);
    std::unique_ptr<dgnn_graph, void (*)(dgnn_graph*)> guard(g, dgnn_graph_free);
    auto* ss = const_cast<dgnn_synth*>(s);
    ss->ensure_pinned();
    const CompactGraph& cg = s->cg;
    const auto& pin = ss->pin;
    g->g->add_snapshot(pin.base_src, pin.base_dst, static_cast<int64_t>(cg.base_src.size()),
                       pin.base_feats);
    for (size_t i = 0; i < cg.steps.size(); ++i) {
      const CompactStep& st = cg.steps[i];
      const auto& ps = pin.steps[i];
      g->g->add_delta(ps.del_src, ps.del_dst, static_cast<int64_t>(st.del_src.size()), ps.ins_src,
                      ps.ins_dst, static_cast<int64_t>(st.ins_src.size()), ps.changed,
                      static_cast<int64_t>(st.changed.size()), ps.changed_feats);
    }
    DGNN_CUDA(cudaStreamSynchronize(g->stream));
    // build temporaries (sort buffers, CUB scratch, the last snapshot's key
    // arrays) go back to the pool
    g->g->release_build_state();
    *out = guard.release();
  });
}

int dgnn_comm_ledger(const dgnn_graph* g, int32_t scheme, int32_t overlap, int32_t workers,
                     int32_t seq_len, int32_t stride, int32_t horizon, int32_t hidden,
                     int64_t num_params, int64_t num_batches, uint64_t* out) {
  return guarded([&] {
    check(scheme >= 0 && scheme <= 2, "unknown placement scheme");
    check(overlap == 0 || overlap == 1, "unknown overlap mode");
    CommLedger L = comm_ledger(*g->g, static_cast<PlacementScheme>(scheme),
                               static_cast<OverlapMode>(overlap), workers, seq_len, stride, horizon,
                               hidden, num_params, num_batches, g->stream);
    auto put = [&](int row, const CommVolume& v) {
      out[4 * row + 0] = v.remote_features;
      out[4 * row + 1] = v.intermediate_redistribution;
      out[4 * row + 2] = v.gradient_sync;
      out[4 * row + 3] = v.snapshot_fetch;
    };
    for (int m = 0; m < workers; ++m) put(m, L.per_worker[m]);
    put(workers, L.total);
  });
}

// ---------------------------------------------------------------- dataset
struct dgnn_dataset {
  std::unique_ptr<DatasetReader> r;
  std::vector<int32_t> src, dst;
  std::vector<float> feats;
  CompactStep step;
};

int dgnn_dataset_open(const char* dir, int32_t threads, dgnn_dataset** out) {
  return guarded([&] {
    auto d = std::make_unique<dgnn_dataset>();
    d->r = std::make_unique<DatasetReader>(dir, threads);
    *out = d.release();
  });
}

void dgnn_dataset_free(dgnn_dataset* d) { delete d; }

int dgnn_dataset_info(const dgnn_dataset* d, int32_t* num_nodes, int32_t* feature_dim,
                      int32_t* T, int32_t* format) {
  return guarded([&] {
    const DatasetManifest& m = d->r->manifest();
    if (num_nodes) *num_nodes = m.num_nodes;
    if (feature_dim) *feature_dim = m.feature_dim;
    if (T) *T = m.T;
    if (format) *format = m.format;
  });
}

int dgnn_dataset_read_base(dgnn_dataset* d, int64_t* num_edges, const int32_t** src,
                           const int32_t** dst, const float** feats) {
  return guarded([&] {
    d->r->read_base(d->src, d->dst, d->feats);
    *num_edges = static_cast<int64_t>(d->src.size());
    *src = d->src.data();
    *dst = d->dst.data();
    *feats = d->feats.data();
  });
}

int dgnn_dataset_read_step(dgnn_dataset* d, int32_t t, int64_t* sizes, const int32_t** del_src,
                           const int32_t** del_dst, const int32_t** ins_src,
                           const int32_t** ins_dst, const int32_t** changed,
                           const float** changed_feats) {
  return guarded([&] {
    d->r->read_step(t, d->step);
    const CompactStep& st = d->step;
    sizes[0] = static_cast<int64_t>(st.del_src.size());
    sizes[1] = static_cast<int64_t>(st.ins_src.size());
    sizes[2] = static_cast<int64_t>(st.changed.size());
    *del_src = st.del_src.data();
    *del_dst = st.del_dst.data();
    *ins_src = st.ins_src.data();
    *ins_dst = st.ins_dst.data();
    *changed = st.changed.data();
    *changed_feats = st.changed_feats.data();
  });
}

// load_dataset (src/dataset_io.cpp:98-165) into the HBM graph store, one step
// at a time: a parser thread reads step t+1 while the device builds step t
// (snapshot CSRs, extract_delta), so host memory holds two steps, never the
// materialised snapshots.
int dgnn_dataset_load(const char* dir, int32_t threads, void* stream, dgnn_graph** out) {
  return guarded([&] {
    DatasetReader r(dir, threads);
    const DatasetManifest& m = r.manifest();
    dgnn_graph* g = nullptr;
    if (dgnn_graph_create(m.num_nodes, m.feature_dim, stream, &g) != 0)
      throw std::invalid_argument(g_err);
    std::unique_ptr<dgnn_graph, void (*)(dgnn_graph*)> guard(g, dgnn_graph_free);
    {
      std::vector<int32_t> src, dst;
      std::vector<float> feats;
      r.read_base(src, dst, feats);
      g->g->add_snapshot(src.data(), dst.data(), static_cast<int64_t>(src.size()), feats.data());
    }
    CompactStep bufs[2];
    PinnedStage stage[2];
    std::exception_ptr perr;
    auto parse = [&](int32_t t, int slot) {
      try {
        r.read_step(t, bufs[slot]);
      } catch (...) {
        perr = std::current_exception();
      }
    };
    if (m.T > 1) parse(1, 0);
    for (int32_t t = 1; t < m.T; ++t) {
      if (perr) std::rethrow_exception(perr);
      const int cur = (t - 1) & 1;
      std::thread next;
      if (t + 1 < m.T) next = std::thread(parse, t + 1, cur ^ 1);
      try {
        const CompactStep& st = bufs[cur];
        // stage into pinned memory once the previous use of this slot is done
        DGNN_CUDA(cudaStreamSynchronize(g->stream));
        stage[cur].reserve(staged_bytes(st));
        size_t off = 0;
        const int32_t* ds = stage[cur].put(off, st.del_src);
        const int32_t* dd = stage[cur].put(off, st.del_dst);
        const int32_t* is = stage[cur].put(off, st.ins_src);
        const int32_t* id = stage[cur].put(off, st.ins_dst);
        const int32_t* ch = stage[cur].put(off, st.changed);
        const float* cf = stage[cur].put(off, st.changed_feats);
        g->g->add_delta(ds, dd, static_cast<int64_t>(st.del_src.size()), is, id,
                        static_cast<int64_t>(st.ins_src.size()), ch,
                        static_cast<int64_t>(st.changed.size()), cf);
      } catch (...) {
        if (next.joinable()) next.join();
        throw;
      }
      if (next.joinable()) next.join();
    }
    DGNN_CUDA(cudaStreamSynchronize(g->stream));
    g->g->release_build_state();
    *out = guard.release();
  });
}

// save_dataset (src/dataset_io.cpp:40-95) from the HBM graph store: snapshot 0
// from its out-CSR (ascending (src,dst)) and features, each delta as
// DynamicGraph::delta(t) (the expanded G- / G+, changed rows at t).
int dgnn_dataset_save_graph(const dgnn_graph* g, const char* dir, int32_t format) {
  return guarded([&] {
    check(format == 1 || format == 2, "unsupported dataset format version");
    const DeviceGraph& G = *g->g;
    check(G.length() > 0, "graph has no snapshots");
    DatasetManifest m{G.num_nodes(), G.feature_dim(), G.length(), format};
    write_manifest(dir, m);
    const int64_t N = m.num_nodes, d = m.feature_dim;
    {
      const DevSnapshot& s0 = G.snapshot(0);
      std::vector<int64_t> ptr(N + 1);
      std::vector<int32_t> dst(s0.num_edges), src(s0.num_edges);
      copy_to_host(ptr.data(), s0.out_ptr.get(), sizeof(int64_t) * (N + 1), g->stream);
      copy_to_host(dst.data(), s0.out_dst.get(), sizeof(int32_t) * s0.num_edges, g->stream);
      for (int64_t u = 0; u < N; ++u)
        for (int64_t e = ptr[u]; e < ptr[u + 1]; ++e) src[e] = static_cast<int32_t>(u);
      std::vector<float> feats(N * d);
      {
        FeatRef f0 = G.features(0, g->stream);
        copy_to_host(feats.data(), f0->get(), sizeof(float) * N * d, g->stream);
      }
      write_base(dir, m, src.data(), dst.data(), s0.num_edges, feats.data());
    }
    for (int32_t t = 1; t < G.length(); ++t) {
      const DevDelta& dd = G.delta(t);
      std::vector<uint64_t> del(dd.n_del), ins(dd.n_ins);
      copy_to_host(del.data(), dd.del.get(), sizeof(uint64_t) * dd.n_del, g->stream);
      copy_to_host(ins.data(), dd.ins.get(), sizeof(uint64_t) * dd.n_ins, g->stream);
      std::vector<int32_t> ds(dd.n_del), dt(dd.n_del), is(dd.n_ins), it(dd.n_ins), ch(dd.n_changed);
      for (int64_t i = 0; i < dd.n_del; ++i) {
        ds[i] = static_cast<int32_t>(del[i] >> 32);
        dt[i] = static_cast<int32_t>(del[i] & 0xffffffffu);
      }
      for (int64_t i = 0; i < dd.n_ins; ++i) {
        is[i] = static_cast<int32_t>(ins[i] >> 32);
        it[i] = static_cast<int32_t>(ins[i] & 0xffffffffu);
      }
      std::vector<float> rows(dd.n_changed * d);
      if (dd.n_changed) {
        copy_to_host(ch.data(), dd.changed.get(), sizeof(int32_t) * dd.n_changed, g->stream);
        // second half of the compact block = F_t[changed]
        copy_to_host(rows.data(), dd.compact.get() + dd.n_changed * d,
                     sizeof(float) * dd.n_changed * d, g->stream);
      }
      StepView v;
      v.n_del = dd.n_del;
      v.n_ins = dd.n_ins;
      v.n_changed = dd.n_changed;
      v.del_src = ds.data();
      v.del_dst = dt.data();
      v.ins_src = is.data();
      v.ins_dst = it.data();
      v.changed = ch.data();
      v.changed_feats = rows.data();
      write_step(dir, m, t, v);
    }
  });
}

int dgnn_synth_save(const dgnn_synth* s, const char* dir, int32_t format) {
  return guarded([&] { save_compact(s->cg, dir, format); });
}

// ------------------------------------------------------------------ k-hop
struct dgnn_cg {
  DevCompGraph cg;
  int32_t num_nodes = 0;
  cudaStream_t stream = nullptr;
  std::unique_ptr<DevSnapshot> view;  // to_view(), built on first request
};

struct dgnn_cg_update {
  DevCgUpdate up;
};

int dgnn_khop(const dgnn_graph* g, int32_t t, const int32_t* seeds, int64_t n_seeds,
              const int32_t* fanouts, int32_t n_hops, uint64_t seed, dgnn_cg** out) {
  return guarded([&] {
    auto c = std::make_unique<dgnn_cg>();
    c->num_nodes = g->g->num_nodes();
    c->stream = g->stream;
    std::vector<int32_t> s(seeds, seeds + (n_seeds > 0 ? n_seeds : 0));
    std::vector<int32_t> f(fanouts, fanouts + (n_hops > 0 ? n_hops : 0));
    c->cg = khop(g->g->snapshot(t), c->num_nodes, std::move(s), std::move(f), seed, g->stream);
    *out = c.release();
  });
}

void dgnn_cg_free(dgnn_cg* c) { delete c; }

int32_t dgnn_cg_num_hops(const dgnn_cg* c) { return static_cast<int32_t>(c->cg.hops.size()); }

int dgnn_cg_hop_sizes(const dgnn_cg* c, int32_t k, int64_t* n_dest, int64_t* n_edges) {
  return guarded([&] {
    const DevHop& h = c->cg.hops.at(k);
    *n_dest = h.n_dest;
    *n_edges = h.n_edges;
  });
}

int dgnn_cg_hop_copy(const dgnn_cg* c, int32_t k, int32_t* dests, int32_t* src, int32_t* dst) {
  return guarded([&] {
    const DevHop& h = c->cg.hops.at(k);
    if (dests) copy_to_host(dests, h.dests.get(), sizeof(int32_t) * h.n_dest, c->stream);
    std::vector<uint64_t> e(h.n_edges);
    copy_to_host(e.data(), h.edges.get(), sizeof(uint64_t) * h.n_edges, c->stream);
    for (int64_t i = 0; i < h.n_edges; ++i) {
      if (src) src[i] = static_cast<int32_t>(e[i] >> 32);
      if (dst) dst[i] = static_cast<int32_t>(e[i] & 0xffffffffu);
    }
  });
}

int dgnn_cg_view(dgnn_cg* c, const int64_t** in_ptr, const int32_t** in_src,
                 const int64_t** out_ptr, const int32_t** out_dst, int64_t* num_edges) {
  return guarded([&] {
    if (!c->view) {
      const DevHop& h = c->cg.hops.back();
      c->view = std::make_unique<DevSnapshot>(csr_from_keys(h.edges.get(), h.n_edges, c->num_nodes, c->stream));
      // callers read the view on other streams
      DGNN_CUDA(cudaStreamSynchronize(c->stream));
    }
    if (in_ptr) *in_ptr = c->view->in_ptr.get();
    if (in_src) *in_src = c->view->in_src.get();
    if (out_ptr) *out_ptr = c->view->out_ptr.get();
    if (out_dst) *out_dst = c->view->out_dst.get();
    if (num_edges) *num_edges = c->view->num_edges;
  });
}

int dgnn_khop_delta(const dgnn_cg* prev, const dgnn_graph* g, int32_t t, dgnn_cg_update** out) {
  return guarded([&] {
    check(t >= 1 && t < g->g->length(), "delta index out of range");
    auto u = std::make_unique<dgnn_cg_update>();
    u->up = khop_delta(prev->cg, g->g->snapshot(t), g->g->num_nodes(), g->stream);
    *out = u.release();
  });
}

void dgnn_cg_update_free(dgnn_cg_update* u) { delete u; }

int dgnn_cg_update_sizes(const dgnn_cg_update* u, int32_t k, int64_t* n_added, int64_t* n_removed) {
  return guarded([&] {
    const auto& h = u->up.hops.at(k);
    *n_added = h.n_added;
    *n_removed = h.n_removed;
  });
}

int dgnn_cg_update_copy(const dgnn_cg_update* u, int32_t k, int32_t* add_src, int32_t* add_dst,
                        int32_t* rem_src, int32_t* rem_dst) {
  return guarded([&] {
    const auto& h = u->up.hops.at(k);
    auto split = [](const cuda::DevArray<uint64_t>& keys, int64_t n, int32_t* s, int32_t* d) {
      std::vector<uint64_t> e(n);
      copy_to_host(e.data(), keys.get(), sizeof(uint64_t) * n, nullptr);
      for (int64_t i = 0; i < n; ++i) {
        if (s) s[i] = static_cast<int32_t>(e[i] >> 32);
        if (d) d[i] = static_cast<int32_t>(e[i] & 0xffffffffu);
      }
    };
    DGNN_CUDA(cudaDeviceSynchronize());
    split(h.added, h.n_added, add_src, add_dst);
    split(h.removed, h.n_removed, rem_src, rem_dst);
  });
}

int32_t dgnn_cg_update_empty(const dgnn_cg_update* u) { return u->up.empty() ? 1 : 0; }

int dgnn_apply_cg_update(const dgnn_cg* prev, const dgnn_cg_update* up, dgnn_cg** out) {
  return guarded([&] {
    auto c = std::make_unique<dgnn_cg>();
    c->num_nodes = prev->num_nodes;
    c->stream = prev->stream;
    c->cg = apply_cg_update(prev->cg, up->up, prev->stream);
    *out = c.release();
  });
}

// ------------------------------------------------------------ aggregation
int dgnn_agg_scratch(int32_t kind, int32_t n, int32_t w, const int64_t* in_ptr,
                     const int32_t* in_src, const float* feats, float* values, float* degree,
                     float* mean_sums, int32_t* argext, void* stream) {
  return guarded([&] {
    check(kind >= 0 && kind <= 3, "unknown aggregation kind");
    cuda::agg_scratch(kind, n, w, in_ptr, in_src, feats, values, degree, mean_sums, argext,
                      as_stream(stream));
  });
}

int dgnn_agg_delta(int32_t kind, int32_t n_rows, int32_t w, const int32_t* rows,
                   const int32_t* row_ptr, const int32_t* ent, const float* f_prev,
                   const float* f_curr, float* values, float* degree, float* mean_sums,
                   int32_t* argext, void* stream) {
  return guarded([&] {
    check(kind >= 0 && kind <= 3, "unknown aggregation kind");
    cuda::agg_delta(kind, n_rows, w, rows, row_ptr, ent, f_prev, f_curr, values, degree,
                    mean_sums, argext, as_stream(stream));
  });
}

int dgnn_graph_apply_delta(const dgnn_graph* g, int32_t t, int32_t kind, float* values,
                           float* degree, float* mean_sums, int32_t* argext, void* stream) {
  return guarded([&] {
    check(kind >= 0 && kind <= 3, "unknown aggregation kind");
    const DeviceGraph& G = *g->g;
    const DevDelta& dd = G.delta(t);
    cudaStream_t st = as_stream(stream);
    FeatRef fp = G.features(t - 1, st), fc = G.features(t, st);
    cuda::agg_delta(kind, dd.n_rows, G.feature_dim(), dd.rows.get(), dd.row_ptr.get(), dd.ent.get(),
                    fp->get(), fc->get(), values, degree, mean_sums, argext, st, dd.ent_c.get(),
                    G.num_nodes(), dd.n_changed, dd.compact.get(), dd.row_ptr_c.get());
  });
}

int dgnn_agg_backward(int32_t kind, int32_t n, int32_t w, const int64_t* out_ptr,
                      const int32_t* out_dst, const float* upstream, const float* degree,
                      const int32_t* argext, float* grad, void* stream) {
  return guarded([&] {
    check(kind >= 0 && kind <= 3, "unknown aggregation kind");
    cuda::agg_backward(kind, n, w, out_ptr, out_dst, upstream, degree, argext, grad,
                       as_stream(stream));
  });
}

int dgnn_agg_incremental(const dgnn_graph* g, int32_t t, int32_t kind, const float* prev_values,
                         const float* prev_degree, const float* prev_mean_sums,
                         const int32_t* prev_argext, int32_t prev_depth, int64_t prev_num_edges,
                         double fallback_threshold, int32_t rescratch_period, float* values,
                         float* degree, float* mean_sums, int32_t* argext, int32_t* info) {
  return guarded([&] {
    cudaStream_t st = g->stream;
    const DeviceGraph& G = *g->g;
    const int32_t n = G.num_nodes(), w = G.feature_dim();
    const size_t nw = static_cast<size_t>(n) * w;
    AggResult prev;
    prev.kind = static_cast<AggrKind>(kind);
    prev.rows = n;
    prev.dim = w;
    prev.t = t - 1;
    prev.num_edges = prev_num_edges;
    prev.incremental_depth = prev_depth;
    auto cp = [&](auto& arr, const auto* src, size_t cnt) {
      using T = std::remove_cv_t<std::remove_pointer_t<decltype(src)>>;
      arr = cuda::DevArray<T>(cnt, st);
      DGNN_CUDA(cudaMemcpyAsync(arr.get(), src, sizeof(T) * cnt, cudaMemcpyDeviceToDevice, st));
    };
    cp(prev.values, prev_values, nw);
    if (kind == 1) {
      cp(prev.degree, prev_degree, n);
      cp(prev.mean_sums, prev_mean_sums, nw);
    }
    if (kind >= 2) cp(prev.argext, prev_argext, nw);
    FeatRef f_prev = G.features(t - 1, st), f_cur = G.features(t, st);
    IncrementalResult r = aggregate_incremental(
        prev, GraphView::of(G, t - 1), GraphView::of(G, t), f_prev->get(),
        f_cur->get(), G.delta(t), t, AggrFn{static_cast<AggrKind>(kind)},
        IncrementalOptions{fallback_threshold, rescratch_period}, st);
    DGNN_CUDA(cudaMemcpyAsync(values, r.result->values.get(), sizeof(float) * nw, cudaMemcpyDeviceToDevice, st));
    if (kind == 1) {
      DGNN_CUDA(cudaMemcpyAsync(degree, r.result->degree.get(), sizeof(float) * n, cudaMemcpyDeviceToDevice, st));
      DGNN_CUDA(cudaMemcpyAsync(mean_sums, r.result->mean_sums.get(), sizeof(float) * nw, cudaMemcpyDeviceToDevice, st));
    }
    if (kind >= 2)
      DGNN_CUDA(cudaMemcpyAsync(argext, r.result->argext.get(), sizeof(int32_t) * nw, cudaMemcpyDeviceToDevice, st));
    DGNN_CUDA(cudaStreamSynchronize(st));
    info[0] = r.used_fallback ? 1 : 0;
    info[1] = static_cast<int32_t>(r.reason);
    info[2] = r.result->incremental_depth;
  });
}

// ------------------------------------------------------------------ cells
int dgnn_pack_cell(int32_t lstm, int32_t in, int32_t H, const float* flat, float* W, float* bias,
                   void* stream) {
  return guarded([&] { cuda::pack_cell(lstm != 0, in, H, flat, W, bias, as_stream(stream)); });
}

int dgnn_cell_forward(int32_t lstm, int32_t n, int32_t in, int32_t H, const float* X,
                      const float* Hm, const float* h_skip, const float* c_prev, const float* W,
                      const float* bias, float* gates, float* c, float* h, void* stream) {
  return guarded([&] {
    cudaStream_t st = as_stream(stream);
    if (cuda::umma_cell_supported(in, H)) {
      cuda::DevArray<float> img(cuda::umma_bimage_floats(4 * H, in + H), st);
      cuda::umma_pack_cell_image(lstm != 0, W, in, H, img.get(), st);
      cuda::umma_cell_forward(lstm != 0, n, in, H, X, Hm, h_skip, c_prev, img.get(), bias, gates,
                              c, h, st);
      DGNN_CUDA(cudaStreamSynchronize(st));
      return;
    }
    cuda::cell_forward(lstm != 0, n, in, H, X, Hm, h_skip, c_prev, W, bias, gates, c, h, st);
  });
}

int dgnn_cell_backward(int32_t lstm, int32_t n, int32_t in, int32_t H, const float* X,
                       const float* Hm, const float* W, const float* gates, const float* c,
                       const float* c_prev, const float* h_skip, const float* dh, const float* dc,
                       float* dX, float* dHm, float* dc_prev, float* dh_skip, float* dflat,
                       void* stream) {
  return guarded([&] {
    cudaStream_t st = as_stream(stream);
    const int K = in + H;
    cuda::DevArray<float> G(static_cast<size_t>(n) * 4 * H, st), WT(static_cast<size_t>(K) * 4 * H, st);
    cuda::DevArray<float> dW(static_cast<size_t>(K) * 4 * H, st), db(4 * H, st);
    const bool tc = cuda::umma_cell_supported(in, H);
    cuda::DevArray<float> ws(tc ? cuda::umma_wgrad_workspace(n, in, H) : cuda::gemm_tn_workspace(n, K, 4 * H), st);
    dW.zero(st);
    db.zero(st);
    cuda::transpose(K, 4 * H, W, WT.get(), st);
    cuda::cell_backward_pointwise(lstm != 0, n, H, gates, c, c_prev, h_skip, dh, dc, G.get(),
                                  dc_prev, dh_skip, st);
    if (tc) {
      cuda::umma_wgrad(n, in, H, G.get(), X, Hm, dW.get(), lstm ? 4 * H : 3 * H, db.get(), ws.get(), st);
      cuda::DevArray<float> img(cuda::umma_bimage_floats(K, 4 * H), st);
      if (dX) {
        cuda::umma_pack_b(W, 4 * H, false, 0, K, 4 * H, img.get(), st);
        cuda::umma_gemm_store2(n, 4 * H, G.get(), img.get(), in, H, dX, dHm, st, nullptr, false,
                               lstm ? 0 : H);
      } else {
        cuda::umma_pack_b(W, 4 * H, false, in, H, 4 * H, img.get(), st);
        cuda::umma_gemm_store2(n, 4 * H, G.get(), img.get(), H, 0, dHm, nullptr, st, nullptr, false,
                               lstm ? 0 : H);
      }
      cuda::unpack_cell_grad(lstm != 0, in, H, dW.get(), db.get(), dflat, st);
      DGNN_CUDA(cudaStreamSynchronize(st));
      return;
    }
    cuda::gemm_tn_acc(n, in, H, 4 * H, X, Hm, G.get(), dW.get(), lstm ? 4 * H : 3 * H, db.get(),
                      ws.get(), st);
    if (dX) {
      cuda::gemm_nn(n, 4 * H, 0, in, H, G.get(), nullptr, WT.get(), K, nullptr, false, false, dX,
                    dHm, st);
    } else {
      cuda::gemm_nn(n, 4 * H, 0, H, 0, G.get(), nullptr, WT.get() + in, K, nullptr, false, false,
                    dHm, nullptr, st);
    }
    cuda::unpack_cell_grad(lstm != 0, in, H, dW.get(), db.get(), dflat, st);
    DGNN_CUDA(cudaStreamSynchronize(st));
  });
}

// ---------------------------------------------------------------- trainer
namespace {

void fill_configs(dgnn_session* s) {
  const dgnn_run_cfg& c = s->cfg;
  ModelConfig& m = s->mcfg;
  m.arch = static_cast<Architecture>(c.arch);
  m.layers = c.layers;
  m.feature_dim = s->graph->g->feature_dim();
  m.hidden_dim = c.hidden;
  m.seq_len = c.seq_len;
  m.horizon = c.horizon;
  m.teacher_forcing = c.teacher_forcing != 0;
  check(c.aggr >= 0 && c.aggr <= 3, "unknown aggregation kind");
  m.aggr = AggrFn{static_cast<AggrKind>(c.aggr)};
  m.seed = c.seed;
  check(c.n_fanouts >= 0 && c.n_fanouts <= 8, "at most 8 fanout hops");
  m.fanouts.assign(c.fanouts, c.fanouts + c.n_fanouts);
  TrainConfig& t = s->tcfg;
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
    check(c.cache_policy <= 2, "unknown cache policy");
    t.cache_policy = static_cast<CachePolicy>(c.cache_policy);
  }
  t.cache_capacity_frac = c.cache_frac;
  t.hbm_cache_budget_bytes = c.hbm_cache_budget_bytes;
  check(c.iteration == 0 || c.iteration == 1, "unknown iteration order");
  t.iteration = c.iteration == 0 ? IterationOrder::kSeqFirst : IterationOrder::kNodeFirst;
}

void attach_observer(dgnn_session* s) {
  CacheStore* store = s->worker().store();
  if (!store || !s->cfg.record_events) return;
  store->set_observer([s](const CacheEvent& ev) {
    const AggKey& k = ev.key;
    const int64_t row[10] = {static_cast<int64_t>(ev.type), static_cast<int64_t>(k.level), k.layer, k.t,
                             static_cast<int64_t>(k.kind), k.batch, k.step_serial, ev.hit ? 1 : 0,
                             ev.assigned_f, ev.stored ? 1 : 0};
    s->events.insert(s->events.end(), row, row + 10);
  });
}

}  // namespace

int dgnn_session_create(dgnn_graph* g, const dgnn_run_cfg* cfg, int32_t rank, void* stream,
                        dgnn_session** out) {
  return guarded([&] {
    auto s = std::make_unique<dgnn_session>();
    s->graph = g;
    s->cfg = *cfg;
    if (stream) {
      s->stream = as_stream(stream);
    } else {
      s->stream = g->stream;
    }
    // the graph store may have been built on another stream
    DGNN_CUDA(cudaStreamSynchronize(g->stream));
    fill_configs(s.get());
    if (cfg->workers <= 0) {
      s->seq = std::make_unique<TrainSession>(*g->g, s->mcfg, s->tcfg, s->stream, cfg->window_total);
    } else {
      check(rank >= 0 && rank < cfg->workers, "rank must lie in [0, workers)");
      s->dist = std::make_unique<DistWorker>(*g->g, s->mcfg, s->tcfg, s->stream, rank,
                                             cfg->workers, cfg->window_total);
    }
    attach_observer(s.get());
    *out = s.release();
  });
}

void dgnn_session_free(dgnn_session* s) {
  if (!s) return;
  cudaStream_t st = s->stream;
  s->seq.reset();
  s->dist.reset();
  cudaStreamSynchronize(st);
  delete s;
}

int64_t dgnn_session_num_params(const dgnn_session* s) {
  return const_cast<dgnn_session*>(s)->model().num_params();
}

int dgnn_session_num_windows(const dgnn_session* s, int64_t* total, int64_t* local_begin,
                             int64_t* local_end) {
  return guarded([&] {
    if (s->seq) {
      *total = static_cast<int64_t>(s->seq->windows().size());
      *local_begin = 0;
      *local_end = *total;
    } else {
      *total = s->dist->total_windows();
      *local_begin = s->dist->assignment().window_begin;
      *local_end = s->dist->assignment().window_end;
    }
  });
}

int dgnn_session_get_params(dgnn_session* s, double* out) {
  return guarded([&] {
    auto v = s->model().flatten_params();
    std::memcpy(out, v.data(), sizeof(double) * v.size());
  });
}

int dgnn_session_set_params(dgnn_session* s, const double* in) {
  return guarded([&] {
    std::vector<double> v(in, in + s->model().num_params());
    s->model().unflatten_params(v);
  });
}

int dgnn_session_initial_params(dgnn_session* s, double* out) {
  return guarded([&] {
    const auto& v = s->model().initial_params();
    std::memcpy(out, v.data(), sizeof(double) * v.size());
  });
}

int dgnn_session_run_epoch(dgnn_session* s, dgnn_epoch_report* report) {
  return guarded([&] {
    check(s->seq != nullptr, "run_epoch needs a seq-first session (workers = 0)");
    EpochReport r = s->seq->run_epoch();
    s->losses = r.sample_losses;
    if (report) {
      report->loss = r.loss;
      report->seconds = r.seconds;
      report->samples = static_cast<int64_t>(r.sample_losses.size());
      report->hits = r.cache.hits;
      report->misses = r.cache.misses;
      report->evictions = r.cache.evictions;
      report->expirations = r.cache.expirations;
      report->invalidations = r.cache.invalidations;
      report->rejected = r.cache.rejected;
      report->scratch_calls = r.scratch_calls;
      report->incremental_calls = r.incremental_calls;
      report->fallbacks = r.fallbacks;
      report->skipped_steps = r.skipped_steps;
      report->spills = r.cache.spills;
      report->refills = r.cache.refills;
    }
  });
}

// ------------------------------------------------------- gradient all-reduce
struct dgnn_comm {
  std::unique_ptr<NcclComm> c;
};

int dgnn_comm_unique_id(uint8_t* out) {
  return guarded([&] { NcclComm::unique_id(out); });
}

int dgnn_comm_create(const uint8_t* id, int32_t world, int32_t rank, dgnn_comm** out) {
  return guarded([&] {
    auto c = std::make_unique<dgnn_comm>();
    c->c = std::make_unique<NcclComm>(id, world, rank);
    *out = c.release();
  });
}

void dgnn_comm_free(dgnn_comm* c) { delete c; }

int dgnn_grad_allreduce(dgnn_comm* c, float* data, int64_t n, void* stream) {
  return guarded([&] { c->c->allreduce_sum(data, n, static_cast<cudaStream_t>(stream)); });
}

int dgnn_session_run_dist_epoch(dgnn_session* s, dgnn_comm* comm, dgnn_epoch_report* report) {
  return guarded([&] {
    check(s->dist != nullptr, "sharded epochs need workers >= 1");
    check(comm != nullptr || s->cfg.workers <= 1, "a sharded epoch over several ranks needs a comm");
    if (comm) check(comm->c->world() == s->cfg.workers, "comm size differs from cfg.workers");
    const DistWorker::EpochResult r = s->dist->run_epoch(comm ? comm->c.get() : nullptr);
    s->losses = s->dist->take_losses();
    if (report) {
      std::memset(report, 0, sizeof(*report));
      double sum = 0.0;
      for (double v : s->losses) sum += v;
      report->loss = s->losses.empty() ? 0.0 : sum / static_cast<double>(s->losses.size());
      report->seconds = r.seconds;
      report->samples = static_cast<int64_t>(s->losses.size());
      CacheStore* store = s->worker().store();
      const CacheStats cs = store ? store->stats() : CacheStats{};
      const ExecutionStats& es = s->worker().provider().stats();
      report->hits = cs.hits;
      report->misses = cs.misses;
      report->evictions = cs.evictions;
      report->expirations = cs.expirations;
      report->invalidations = cs.invalidations;
      report->rejected = cs.rejected;
      report->scratch_calls = es.scratch_calls;
      report->incremental_calls = es.incremental_calls;
      report->fallbacks = es.fallbacks;
      report->skipped_steps = r.skipped;
      report->spills = cs.spills;
      report->refills = cs.refills;
    }
  });
}

int dgnn_session_begin_epoch(dgnn_session* s, int64_t* num_batches) {
  return guarded([&] {
    check(s->dist != nullptr, "sharded epochs need workers >= 1");
    s->dist->begin_epoch();
    if (num_batches) *num_batches = s->dist->num_batches();
  });
}

int dgnn_session_local_grads(dgnn_session* s, int64_t batch, float* grad_sum) {
  return guarded([&] {
    check(s->dist != nullptr, "sharded epochs need workers >= 1");
    check(batch >= 0 && batch < s->dist->num_batches(), "batch index out of range");
    s->dist->local_grads(batch, grad_sum);
  });
}

int dgnn_session_apply(dgnn_session* s, const float* grad_sum, int32_t* applied) {
  return guarded([&] {
    check(s->dist != nullptr, "sharded epochs need workers >= 1");
    const bool ok = s->dist->apply(grad_sum);
    if (applied) *applied = ok ? 1 : 0;
  });
}

int dgnn_session_end_epoch(dgnn_session* s) {
  return guarded([&] {
    check(s->dist != nullptr, "sharded epochs need workers >= 1");
    s->losses = s->dist->take_losses();
    s->dist->end_epoch();
  });
}

int dgnn_session_losses(dgnn_session* s, double* out, int64_t* n) {
  return guarded([&] {
    if (out) std::memcpy(out, s->losses.data(), sizeof(double) * s->losses.size());
    *n = static_cast<int64_t>(s->losses.size());
  });
}

int dgnn_session_sample_grads(dgnn_session* s, int32_t window_index, double* loss, float* pred0,
                              double* grads) {
  return guarded([&] {
    DgnnModel& model = s->model();
    const DeviceGraph& G = *s->graph->g;
    cudaStream_t st = s->stream;
    auto windows = sliding_windows(s->window_total(), s->mcfg.seq_len, s->tcfg.stride, s->mcfg.horizon);
    check(window_index >= 0 && window_index < static_cast<int32_t>(windows.size()),
          "window index out of range");
    Worker fresh(G, model, s->tcfg, st);
    auto batches = make_batches(G.num_nodes(), s->tcfg.batch_size, s->tcfg.seed, 0);
    SeqSample sample = build_sample(G, s->mcfg, windows[window_index],
                                    static_cast<Timestep>(windows.size() - 1 - window_index), 0,
                                    batches[0], s->tcfg.seed, st);
    ForwardArtifacts fwd = model_forward(model, sample, fresh.provider());
    cuda::DevArray<double> slot(1, st), ws(512, st);
    slot.zero(st);
    auto dpred = seed_loss(sample, fwd, s->mcfg.feature_dim, slot.get(), ws.get(), st);
    cuda::DevArray<float> grad(model.num_params(), st);
    grad.zero(st);
    model_backward(model, sample, fwd, dpred, grad.get(), st);
    copy_to_host(loss, slot.get(), sizeof(double), st);
    if (pred0) {
      copy_to_host(pred0, fwd.predictions[0]->get(),
                   sizeof(float) * static_cast<size_t>(G.num_nodes()) * s->mcfg.feature_dim, st);
    }
    std::vector<float> g(model.num_params());
    copy_to_host(g.data(), grad.get(), sizeof(float) * g.size(), st);
    for (size_t i = 0; i < g.size(); ++i) grads[i] = g[i];
  });
}

int dgnn_session_invocations(dgnn_session* s, int32_t* out, int64_t* n) {
  return guarded([&] {
    const auto& inv = s->worker().provider().stats().invocations;
    *n = static_cast<int64_t>(inv.size());
    if (!out) return;
    for (size_t i = 0; i < inv.size(); ++i) {
      out[4 * i + 0] = inv[i].layer;
      out[4 * i + 1] = inv[i].t;
      out[4 * i + 2] = static_cast<int32_t>(inv[i].kind);
      out[4 * i + 3] = inv[i].incremental ? 1 : 0;
    }
  });
}

int dgnn_session_cache_events(dgnn_session* s, int64_t* out, int64_t* n) {
  return guarded([&] {
    *n = static_cast<int64_t>(s->events.size() / 10);
    if (out) std::memcpy(out, s->events.data(), sizeof(int64_t) * s->events.size());
  });
}

int dgnn_session_stats(dgnn_session* s, int64_t* out12) {
  return guarded([&] {
    CacheStore* store = s->worker().store();
    CacheStats cs = store ? store->stats() : CacheStats{};
    const ExecutionStats& es = s->worker().provider().stats();
    const int64_t v[12] = {cs.hits, cs.misses, cs.evictions, cs.expirations, cs.invalidations,
                           cs.rejected, es.scratch_calls, es.incremental_calls, es.fallbacks,
                           cs.spills, cs.refills, static_cast<int64_t>(cs.resident_peak_units)};
    std::memcpy(out12, v, sizeof(v));
  });
}

int dgnn_session_tier_stats(dgnn_session* s, int64_t* out8) {
  return guarded([&] {
    CacheStore* store = s->worker().store();
    CacheStats cs = store ? store->stats() : CacheStats{};
    const int64_t v[8] = {cs.spills, cs.refills, cs.prefetches, cs.demand_refills, cs.spill_bytes,
                          cs.refill_bytes, store ? store->pinned_bytes() : 0,
                          store ? store->hbm_resident_bytes() : 0};
    std::memcpy(out8, v, sizeof(v));
  });
}

// ------------------------------------------------------- host-side plan logic
int64_t dgnn_sliding_windows(int32_t total, int32_t L, int32_t S, int32_t H, int32_t* starts,
                             int64_t cap) {
  try {
    auto w = sliding_windows(total, L, S, H);
    for (int64_t i = 0; i < static_cast<int64_t>(w.size()) && i < cap; ++i) starts[i] = w[i].start;
    return static_cast<int64_t>(w.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int dgnn_plan(int32_t total, int32_t workers, int32_t L, int32_t S, int32_t H, int64_t* out) {
  return guarded([&] {
    auto p = plan_consecutive_block(total, workers, L, S, H);
    for (int m = 0; m < workers; ++m) {
      out[4 * m + 0] = p[m].block_begin;
      out[4 * m + 1] = p[m].block_end;
      out[4 * m + 2] = p[m].window_begin;
      out[4 * m + 3] = p[m].window_end;
    }
  });
}

int dgnn_cache_scores(const int32_t* ctx, int32_t* f, int32_t* imm) {
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

uint64_t dgnn_key_hash(int32_t level, int32_t layer, int32_t t, int32_t kind, int64_t batch,
                       int64_t serial) {
  AggKey k{static_cast<CacheLevel>(level), layer, t, static_cast<AggKeyKind>(kind), batch, serial};
  return static_cast<uint64_t>(AggKeyHash{}(k));
}

int64_t dgnn_make_batches(int32_t num_nodes, int32_t batch_size, uint64_t seed,
                          int64_t epoch_index, int32_t* out, int64_t cap) {
  auto b = make_batches(num_nodes, batch_size, seed, epoch_index);
  for (int64_t i = 0; i < static_cast<int64_t>(b.size()) && i < cap; ++i) {
    out[2 * i] = b[i].first;
    out[2 * i + 1] = b[i].second;
  }
  return static_cast<int64_t>(b.size());
}

int64_t dgnn_init_params(const dgnn_run_cfg* cfg, int32_t feature_dim, double* out) {
  try {
    ModelConfig m;
    m.arch = static_cast<Architecture>(cfg->arch);
    m.layers = cfg->layers;
    m.feature_dim = feature_dim;
    m.hidden_dim = cfg->hidden;
    m.seed = cfg->seed;
    auto v = initial_params_host(m);
    if (out) std::memcpy(out, v.data(), sizeof(double) * v.size());
    return static_cast<int64_t>(v.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// ---------------------------------------------------------------- profiling
int dgnn_mem_stats(int64_t* reserved, int64_t* used, int64_t* reserved_high, int64_t* used_high) {
  return guarded([&] { cuda::pool_stats(reserved, used, reserved_high, used_high); });
}
int dgnn_prof_enable(int32_t on) {
  return guarded([&] { prof_enable(on != 0); });
}
int dgnn_prof_reset(void) {
  return guarded([&] { prof_reset(); });
}
int dgnn_prof_get(int32_t cls, int64_t* launches, double* ms, double* bytes, double* flops) {
  return guarded([&] {
    prof_flush();
    ProfStat p = prof_get(cls);
    if (launches) *launches = p.launches;
    if (ms) *ms = p.ms;
    if (bytes) *bytes = p.bytes;
    if (flops) *flops = p.flops;
  });
}

int dgnn_prof_get_max(int32_t cls, double* max_ms) {
  return guarded([&] {
    prof_flush();
    if (max_ms) *max_ms = prof_get(cls).max_ms;
  });
}

}  // extern "C"
