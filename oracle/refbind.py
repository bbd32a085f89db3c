"""ctypes binding to oracle/_ref/libdgnn_ref.so (the compiled CPU reference).

TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module. The library is the
reference's own proj/src compiled against oracle/eigen_shim (see oracle/Makefile)
plus oracle/ref_harness.cpp; every function below forwards to the reference's
public API named in the harness.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libdgnn_ref.so")

ARCH = {"gcrn_m1": 0, "cd_gcn": 1, "gcrn_m2": 2, "tgcn": 3}
AGGR = {"sum": 0, "mean": 1, "max": 2, "min": 3}
POLICY = {"off": -1, "reinc": 0, "lru": 1, "lfu": 2}


class RefRunCfg(C.Structure):
    _fields_ = [
        ("arch", C.c_int32), ("layers", C.c_int32), ("hidden", C.c_int32),
        ("seq_len", C.c_int32), ("horizon", C.c_int32), ("teacher_forcing", C.c_int32),
        ("aggr", C.c_int32), ("batch_size", C.c_int32), ("seed", C.c_uint64),
        ("lr", C.c_double), ("optimizer", C.c_int32), ("stride", C.c_int32),
        ("fallback_threshold", C.c_double), ("rescratch_period", C.c_int32),
        ("incremental", C.c_int32), ("cache_policy", C.c_int32), ("cache_frac", C.c_double),
        ("workers", C.c_int32), ("epochs", C.c_int32), ("window_total", C.c_int32),
        ("record_events", C.c_int32), ("n_fanouts", C.c_int32), ("fanouts", C.c_int32 * 8),
        ("iteration", C.c_int32),
    ]


@dataclass
class RunCfg:
    """Python-side run configuration (defaults = RunSettings, inc/config.hpp:18-57)."""
    arch: str = "gcrn_m2"
    layers: int = 2
    hidden: int = 16
    seq_len: int = 8
    horizon: int = 1
    teacher_forcing: bool = True
    aggr: str = "sum"
    batch_size: int = 0
    seed: int = 1
    lr: float = 0.01
    optimizer: str = "adam"
    stride: int = 1
    fallback_threshold: float = 0.5
    rescratch_period: int = 64
    incremental: bool = True
    cache: str = "reinc"
    cache_frac: float = 1.0
    workers: int = 0
    epochs: int = 1
    window_total: int = 0  # 0 -> T-1
    record_events: bool = True
    fanouts: tuple = ()
    iteration: str = "seq_first"

    def to_c(self, T: int) -> RefRunCfg:
        c = RefRunCfg()
        c.arch = ARCH[self.arch]
        c.layers = self.layers
        c.hidden = self.hidden
        c.seq_len = self.seq_len
        c.horizon = self.horizon
        c.teacher_forcing = int(self.teacher_forcing)
        c.aggr = AGGR[self.aggr]
        c.batch_size = self.batch_size
        c.seed = self.seed
        c.lr = self.lr
        c.optimizer = 0 if self.optimizer == "sgd" else 1
        c.stride = self.stride
        c.fallback_threshold = self.fallback_threshold
        c.rescratch_period = self.rescratch_period
        c.incremental = int(self.incremental)
        c.cache_policy = POLICY[self.cache]
        c.cache_frac = self.cache_frac
        c.workers = self.workers
        c.epochs = self.epochs
        c.window_total = self.window_total if self.window_total > 0 else T - 1
        c.record_events = int(self.record_events)
        c.n_fanouts = len(self.fanouts)
        for i, f in enumerate(self.fanouts):
            c.fanouts[i] = f
        c.iteration = {"seq_first": 0, "node_first": 1}[self.iteration]
        return c


_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not available():
        raise RuntimeError(f"reference oracle not built: {LIB_PATH} (run `make -C oracle`)")
    L = C.CDLL(LIB_PATH)
    P, I32, I64, U64, D = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double
    sig = {
        "ref_last_error": (C.c_char_p, []),
        "ref_synth": (P, [I32, D, I32, I32, D, D, U64]),
        "ref_graph_from_arrays": (P, [I32, I32, I32, P, P, P, P]),
        "ref_graph_free": (None, [P]),
        "ref_save_dataset": (C.c_int, [P, C.c_char_p]),
        "ref_khop": (P, [P, I32, P, I64, P, I32, U64]),
        "ref_comm_ledger": (C.c_int, [P, C.POINTER(RefRunCfg), I32, I32, P, P, P]),
        "ref_cg_free": (None, [P]),
        "ref_cg_num_hops": (I32, [P]),
        "ref_cg_hop_sizes": (None, [P, I32, P, P]),
        "ref_cg_hop_copy": (None, [P, I32, P, P, P]),
        "ref_cg_view": (None, [P, I32, P, P]),
        "ref_khop_delta": (P, [P, P, I32]),
        "ref_cg_update_free": (None, [P]),
        "ref_cg_update_sizes": (None, [P, I32, P, P]),
        "ref_cg_update_copy": (None, [P, I32, P, P, P, P]),
        "ref_cg_update_empty": (I32, [P]),
        "ref_apply_cg_update": (P, [P, P]),
        "ref_load_dataset": (P, [C.c_char_p]),
        "ref_graph_length": (I32, [P]),
        "ref_graph_num_nodes": (I32, [P]),
        "ref_graph_feature_dim": (I32, [P]),
        "ref_snapshot_num_edges": (I64, [P, I32]),
        "ref_snapshot_edges": (None, [P, I32, P, P]),
        "ref_snapshot_feats": (None, [P, I32, P]),
        "ref_snapshot_in_csr": (None, [P, I32, P, P]),
        "ref_snapshot_out_csr": (None, [P, I32, P, P]),
        "ref_delta_sizes": (C.c_int, [P, I32, P, P, P]),
        "ref_delta_get": (C.c_int, [P, I32, P, P, P, P, P, P]),
        "ref_change_ratio": (D, [P, I32]),
        "ref_agg_scratch": (C.c_int, [P, I32, I32, P, I32, P, P, P, P]),
        "ref_agg_chain": (C.c_int, [P, I32, I32, I32, D, I32, P, P, P, P, P]),
        "ref_agg_backward": (C.c_int, [P, I32, I32, P, I32, P, P]),
        "ref_cell_init": (None, [I32, I32, I32, U64, P]),
        "ref_cell_fwd_bwd": (C.c_int, [I32, I32, I32, I32] + [P] * 15),
        "ref_run": (P, [P, C.POINTER(RefRunCfg)]),
        "ref_sample_grads": (C.c_int, [P, C.POINTER(RefRunCfg), I32, P, P, P, P]),
        "ref_num_params": (I64, [P, C.POINTER(RefRunCfg)]),
        "ref_init_params": (None, [P, C.POINTER(RefRunCfg), P]),
        "ref_run_get": (I64, [P, I32, P]),
        "ref_run_seconds": (D, [P]),
        "ref_run_free": (None, [P]),
        "ref_sliding_windows": (None, [I32, I32, I32, I32, P, P]),
        "ref_plan": (C.c_int, [I32, I32, I32, I32, I32, P]),
        "ref_cache_scores": (C.c_int, [P, P, P]),
        "ref_key_hash": (U64, [I32, I32, I32, I32, I64, I64]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _check(rc: int):
    if rc != 0:
        msg = lib().ref_last_error().decode()
        if rc == 2:
            raise IndexError(msg)
        raise ValueError(msg)


class RefGraph:
    """Owns a reference dgnn::DynamicGraph."""

    def __init__(self, handle):
        if not handle:
            raise ValueError(lib().ref_last_error().decode())
        self.h = handle
        L = lib()
        self.T = L.ref_graph_length(self.h)
        self.n = L.ref_graph_num_nodes(self.h)
        self.dim = L.ref_graph_feature_dim(self.h)

    @classmethod
    def synth(cls, n, avg_degree, dim, T, edge_ratio, feat_ratio, seed=1):
        return cls(lib().ref_synth(n, avg_degree, dim, T, edge_ratio, feat_ratio, seed))

    @classmethod
    def from_snapshots(cls, n, dim, edges_per_t, feats_per_t):
        T = len(edges_per_t)
        counts = np.array([len(e) for e in edges_per_t], dtype=np.int64)
        allv = [np.asarray(e, dtype=np.int32).reshape(-1, 2) for e in edges_per_t]
        cat = np.concatenate(allv) if counts.sum() else np.zeros((0, 2), np.int32)
        src = np.ascontiguousarray(cat[:, 0])
        dst = np.ascontiguousarray(cat[:, 1])
        feats = np.ascontiguousarray(np.stack(feats_per_t).astype(np.float64))
        return cls(lib().ref_graph_from_arrays(n, dim, T, _p(counts), _p(src), _p(dst), _p(feats)))

    def comm_ledger(self, cfg: "RunCfg", scheme: int, overlap: int):
        """run_distributed_epoch's CommLedger -> ((M+1) x 4, num_params, num_batches)."""
        c = cfg.to_c(self.T)
        out = np.zeros((cfg.workers + 1, 4), np.uint64)
        npar, nb = np.zeros(1, np.int64), np.zeros(1, np.int64)
        _check(lib().ref_comm_ledger(self.h, C.byref(c), scheme, overlap, _p(out), _p(npar), _p(nb)))
        return out, int(npar[0]), int(nb[0])

    @classmethod
    def load_dataset(cls, path):
        """load_dataset (src/dataset_io.cpp:98-165)."""
        return cls(lib().ref_load_dataset(os.fsencode(path)))

    def save_dataset(self, path):
        """save_dataset (src/dataset_io.cpp:40-95)."""
        _check(lib().ref_save_dataset(self.h, os.fsencode(path)))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_graph_free(self.h)
            self.h = None

    def edges(self, t):
        m = lib().ref_snapshot_num_edges(self.h, t)
        s = np.empty(m, np.int32)
        d = np.empty(m, np.int32)
        lib().ref_snapshot_edges(self.h, t, _p(s), _p(d))
        return s, d

    def feats(self, t):
        out = np.empty((self.n, self.dim), np.float64)
        lib().ref_snapshot_feats(self.h, t, _p(out))
        return out

    def in_csr(self, t):
        m = lib().ref_snapshot_num_edges(self.h, t)
        ptr = np.empty(self.n + 1, np.int64)
        src = np.empty(m, np.int32)
        lib().ref_snapshot_in_csr(self.h, t, _p(ptr), _p(src))
        return ptr, src

    def out_csr(self, t):
        m = lib().ref_snapshot_num_edges(self.h, t)
        ptr = np.empty(self.n + 1, np.int64)
        dst = np.empty(m, np.int32)
        lib().ref_snapshot_out_csr(self.h, t, _p(ptr), _p(dst))
        return ptr, dst

    def delta(self, t):
        nd, ni, nc = C.c_int64(), C.c_int64(), C.c_int64()
        _check(lib().ref_delta_sizes(self.h, t, C.byref(nd), C.byref(ni), C.byref(nc)))
        ds, dd = np.empty(nd.value, np.int32), np.empty(nd.value, np.int32)
        is_, id_ = np.empty(ni.value, np.int32), np.empty(ni.value, np.int32)
        ch = np.empty(nc.value, np.int32)
        cf = np.empty((nc.value, self.dim), np.float64)
        _check(lib().ref_delta_get(self.h, t, _p(ds), _p(dd), _p(is_), _p(id_), _p(ch), _p(cf)))
        return {"del_src": ds, "del_dst": dd, "ins_src": is_, "ins_dst": id_,
                "changed": ch, "changed_feats": cf}

    def change_ratio(self, t):
        return lib().ref_change_ratio(self.h, t)

    def agg_scratch(self, t, kind, feats):
        feats = np.ascontiguousarray(feats, np.float64)
        n, w = feats.shape
        vals = np.empty((n, w), np.float64)
        deg = np.zeros(n, np.float64)
        ms = np.zeros((n, w), np.float64)
        arg = np.full((n, w), -1, np.int32)
        _check(lib().ref_agg_scratch(self.h, t, AGGR[kind], _p(feats), w, _p(vals), _p(deg), _p(ms), _p(arg)))
        return {"values": vals, "degree": deg, "mean_sums": ms, "argext": arg}

    def agg_chain(self, t0, t1, kind, threshold=0.5, rescratch=64):
        n, w = self.n, self.dim
        vals = np.empty((n, w), np.float64)
        deg = np.zeros(n, np.float64)
        ms = np.zeros((n, w), np.float64)
        arg = np.full((n, w), -1, np.int32)
        info = np.zeros((max(t1 - t0, 1), 3), np.int32)
        _check(lib().ref_agg_chain(self.h, t0, t1, AGGR[kind], threshold, rescratch,
                                   _p(vals), _p(deg), _p(ms), _p(arg), _p(info)))
        return {"values": vals, "degree": deg, "mean_sums": ms, "argext": arg,
                "steps": info[: t1 - t0]}

    def agg_backward(self, t, kind, feats, upstream):
        feats = np.ascontiguousarray(feats, np.float64)
        up = np.ascontiguousarray(upstream, np.float64)
        out = np.empty_like(up)
        _check(lib().ref_agg_backward(self.h, t, AGGR[kind], _p(feats), feats.shape[1], _p(up), _p(out)))
        return out

    # ---------------------------------------------------------- training
    def run(self, cfg: RunCfg) -> "RunResult":
        c = cfg.to_c(self.T)
        h = lib().ref_run(self.h, C.byref(c))
        if not h:
            raise ValueError(lib().ref_last_error().decode())
        try:
            return RunResult.collect(h)
        finally:
            lib().ref_run_free(h)

    def num_params(self, cfg: RunCfg) -> int:
        c = cfg.to_c(self.T)
        return lib().ref_num_params(self.h, C.byref(c))

    def init_params(self, cfg: RunCfg) -> np.ndarray:
        c = cfg.to_c(self.T)
        out = np.empty(self.num_params(cfg), np.float64)
        lib().ref_init_params(self.h, C.byref(c), _p(out))
        return out

    def sample_grads(self, cfg: RunCfg, window_index=0, params=None):
        c = cfg.to_c(self.T)
        P = self.num_params(cfg)
        loss = C.c_double()
        pred0 = np.empty((self.n, self.dim), np.float64)
        grads = np.empty(P, np.float64)
        pin = None if params is None else np.ascontiguousarray(params, np.float64)
        _check(lib().ref_sample_grads(self.h, C.byref(c), window_index, _p(pin), C.byref(loss), _p(pred0), _p(grads)))
        return loss.value, pred0, grads


class RefCompGraph:
    """Owns a reference dgnn::ComputationalGraph (inc/khop.hpp:42-51)."""

    def __init__(self, handle, n):
        if not handle:
            raise ValueError(lib().ref_last_error().decode())
        self.h, self.n = handle, n

    @classmethod
    def khop(cls, g: "RefGraph", t, seeds, fanouts, seed):
        s = np.ascontiguousarray(seeds, np.int32)
        f = np.ascontiguousarray(fanouts, np.int32)
        return cls(lib().ref_khop(g.h, t, _p(s), len(s), _p(f), len(f), seed), g.n)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_cg_free(self.h)
            self.h = None

    def hops(self):
        out = []
        for k in range(lib().ref_cg_num_hops(self.h)):
            nd, ne = C.c_int64(), C.c_int64()
            lib().ref_cg_hop_sizes(self.h, k, C.byref(nd), C.byref(ne))
            d = np.empty(nd.value, np.int32)
            s, t = np.empty(ne.value, np.int32), np.empty(ne.value, np.int32)
            lib().ref_cg_hop_copy(self.h, k, _p(d), _p(s), _p(t))
            out.append({"dests": d, "src": s, "dst": t})
        return out

    def view(self):
        ne = len(self.hops()[-1]["src"])
        ptr, src = np.empty(self.n + 1, np.int64), np.empty(ne, np.int32)
        lib().ref_cg_view(self.h, self.n, _p(ptr), _p(src))
        return ptr, src

    def delta(self, g: "RefGraph", t):
        u = lib().ref_khop_delta(self.h, g.h, t)
        if not u:
            raise ValueError(lib().ref_last_error().decode())
        try:
            hops = []
            for k in range(lib().ref_cg_num_hops(self.h)):
                na, nr = C.c_int64(), C.c_int64()
                lib().ref_cg_update_sizes(u, k, C.byref(na), C.byref(nr))
                a = [np.empty(na.value, np.int32) for _ in range(2)]
                r = [np.empty(nr.value, np.int32) for _ in range(2)]
                lib().ref_cg_update_copy(u, k, _p(a[0]), _p(a[1]), _p(r[0]), _p(r[1]))
                hops.append({"add_src": a[0], "add_dst": a[1], "rem_src": r[0], "rem_dst": r[1]})
            empty = bool(lib().ref_cg_update_empty(u))
            applied = RefCompGraph(lib().ref_apply_cg_update(self.h, u), self.n)
        finally:
            lib().ref_cg_update_free(u)
        return hops, empty, applied


@dataclass
class RunResult:
    params0: np.ndarray
    params: np.ndarray
    losses: np.ndarray
    grads0: np.ndarray
    peak_units: np.ndarray
    visitation: np.ndarray
    events: np.ndarray
    stats: np.ndarray
    invocations: np.ndarray
    seconds: float = 0.0
    extra: dict = field(default_factory=dict)

    @classmethod
    def collect(cls, h):
        L = lib()

        def get(kind, dtype, width=1):
            n = L.ref_run_get(h, kind, None)
            out = np.empty(n, dtype)
            L.ref_run_get(h, kind, _p(out))
            return out.reshape(-1, width) if width > 1 else out

        return cls(
            params0=get(0, np.float64), params=get(1, np.float64), losses=get(2, np.float64),
            grads0=get(3, np.float64), peak_units=get(4, np.float64),
            visitation=get(10, np.int64, 3), events=get(11, np.int64, 11),
            stats=get(12, np.int64, 10), invocations=get(20, np.int32, 5),
            seconds=L.ref_run_seconds(h),
        )


def sliding_windows(total, L, S, H):
    cnt = C.c_int32()
    lib().ref_sliding_windows(total, L, S, H, None, C.byref(cnt))
    out = np.empty(max(cnt.value, 1), np.int32)
    lib().ref_sliding_windows(total, L, S, H, _p(out), C.byref(cnt))
    return out[: cnt.value]


def plan(total, workers, L, S, H):
    out = np.empty((workers, 4), np.int64)
    _check(lib().ref_plan(total, workers, L, S, H, _p(out)))
    return out


def cache_scores(num_layers, gates, gate, L, S, idx, part, layer, tf, H, wrem, kind):
    ctx = np.array([num_layers, gates, gate, L, S, idx, part, layer, tf, H, wrem, kind], np.int32)
    f, imm = C.c_int32(), C.c_int32()
    _check(lib().ref_cache_scores(_p(ctx), C.byref(f), C.byref(imm)))
    return f.value, imm.value


def key_hash(level, layer, t, kind, batch, serial):
    return lib().ref_key_hash(level, layer, t, kind, batch, serial)


def cell_init(kind, n_in, hidden, seed):
    K = 4 if kind == 0 else 3
    out = np.empty(K * (n_in * hidden + hidden * hidden + hidden), np.float64)
    lib().ref_cell_init(kind, n_in, hidden, seed, _p(out))
    return out


def cell_fwd_bwd(kind, n_in, hidden, params, X, Hm, h_skip, c_prev, dh, dc):
    """kind 0 = LSTM, 1 = GRU. Returns dict of forward tape and gradients."""
    n = X.shape[0]
    K = 4 if kind == 0 else 3
    f64 = lambda a: None if a is None else np.ascontiguousarray(a, np.float64)
    params, X, Hm, h_skip, c_prev, dh, dc = map(f64, (params, X, Hm, h_skip, c_prev, dh, dc))
    o = {k: np.zeros(s, np.float64) for k, s in {
        "gates": (K, n, hidden), "hn": (n, hidden), "c": (n, hidden), "h": (n, hidden),
        "dX": (n, n_in), "dHm": (n, hidden), "dh_skip": (n, hidden), "dc_prev": (n, hidden),
        "dparams": params.shape}.items()}
    _check(lib().ref_cell_fwd_bwd(kind, n_in, hidden, n, _p(params), _p(X), _p(Hm), _p(h_skip),
                                  _p(c_prev), _p(dh), _p(dc), _p(o["gates"]), _p(o["hn"]), _p(o["c"]),
                                  _p(o["h"]), _p(o["dX"]), _p(o["dHm"]), _p(o["dh_skip"]),
                                  _p(o["dc_prev"]), _p(o["dparams"])))
    return o
