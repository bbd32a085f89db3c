"""Python mirror of the reference's public interface over the C ABI.

Names and argument meaning follow proj/include/dgnn (DynamicGraph, synthesize,
aggregate_scratch / aggregate_incremental / aggregate_backward, TrainSession,
the consecutive-block distributed session). Device buffers are torch CUDA
tensors (torch is used for allocation and streams only); all computation runs
in _dgnn_b200.so. Errors surface as ValueError (the reference's
std::invalid_argument), IndexError (std::out_of_range) or DgnnError (CUDA).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check, lib

AGGR = {"sum": 0, "mean": 1, "max": 2, "min": 3}
ARCH = {"gcrn_m1": 0, "cd_gcn": 1, "gcrn_m2": 2, "tgcn": 3}
POLICY = {"off": -1, "reinc": 0, "lru": 1, "lfu": 2}


def _torch():
    import torch
    return torch


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _np_ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


CUDA_STREAM_LEGACY = 1  # cudaStreamLegacy


def _stream_handle(stream):
    """cudaStream_t for the C ABI. torch's default stream has handle 0, which
    the C ABI would read as "library-owned stream"; pass cudaStreamLegacy so
    the library and torch share the same (synchronising) default stream."""
    if stream is None:
        return None
    h = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    return C.c_void_p(h if h else CUDA_STREAM_LEGACY)


def current_stream():
    torch = _torch()
    return torch.cuda.current_stream()


class _CudaArray:
    def __init__(self, ptr, shape, dtype):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": np.dtype(dtype).str,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


def device_view(ptr, shape, dtype):
    """Zero-copy torch view of a device buffer owned by the library."""
    torch = _torch()
    return torch.as_tensor(_CudaArray(ptr, shape, dtype), device="cuda")


def launch_count() -> int:
    return lib().dgnn_launch_count()


def sliding_windows(total: int, length: int, stride: int, horizon: int) -> list[int]:
    """Window starts 0, S, 2S, ... while start + L + H <= T (ref src/windows.cpp:5-15)."""
    if length < 1:
        raise ValueError("sliding_windows: L must be >= 1")
    if stride < 1:
        raise ValueError("sliding_windows: S must be >= 1")
    if horizon < 0:
        raise ValueError("sliding_windows: H must be >= 0")
    return list(range(0, max(total - length - horizon + 1, 0), stride))


def plan(total: int, workers: int, L: int, S: int, H: int):
    """Consecutive-block placement (ref src/distsim.cpp:35-81): per worker
    (block_begin, block_end, window_begin, window_end)."""
    if workers < 1:
        raise ValueError("plan needs at least one worker")
    if total < workers:
        raise ValueError("fewer snapshots than workers")
    starts = sliding_windows(total, L, S, H)
    W = len(starts)
    base, extra = divmod(W, workers)
    out, cur = [], 0
    for m in range(workers):
        wb, we = cur, cur + base + (1 if m < extra else 0)
        cur = we
        bb = starts[wb] if wb < W else total
        be = (starts[we] if we < W else total) if m + 1 < workers else total
        out.append([min(bb, be), be, wb, we])
    out[0][0] = 0
    return out


# ------------------------------------------------------------------ graphs
class Synth:
    """Bit-exact streaming synthesize (ref src/synth.cpp:36-91), host side."""

    def __init__(self, num_nodes, avg_degree, feature_dim, num_snapshots, edge_change,
                 feature_change, seed=1):
        h = C.c_void_p()
        check(lib().dgnn_synth_create(num_nodes, avg_degree, feature_dim, num_snapshots,
                                      edge_change, feature_change, seed, C.byref(h)))
        self.h = h
        self.n, self.dim, self.T = num_nodes, feature_dim, num_snapshots
        sizes = np.empty(1 + 3 * (num_snapshots - 1), np.int64)
        check(lib().dgnn_synth_sizes(self.h, _np_ptr(sizes)))
        self.sizes = sizes

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None and _lib._lib is not None:
            lib().dgnn_synth_free(self.h)
            self.h = None

    def base(self):
        s, d, f = C.c_void_p(), C.c_void_p(), C.c_void_p()
        check(lib().dgnn_synth_base(self.h, C.byref(s), C.byref(d), C.byref(f)))
        E = int(self.sizes[0])
        src = np.ctypeslib.as_array(C.cast(s, C.POINTER(C.c_int32)), (E,)).copy() if E else np.zeros(0, np.int32)
        dst = np.ctypeslib.as_array(C.cast(d, C.POINTER(C.c_int32)), (E,)).copy() if E else np.zeros(0, np.int32)
        feats = np.ctypeslib.as_array(C.cast(f, C.POINTER(C.c_float)), (self.n * self.dim,)).copy()
        return src, dst, feats.reshape(self.n, self.dim)

    def step(self, t):
        ptrs = [C.c_void_p() for _ in range(6)]
        check(lib().dgnn_synth_step(self.h, t, *[C.byref(p) for p in ptrs]))
        nd, ni, nc = (int(x) for x in self.sizes[1 + 3 * (t - 1): 4 + 3 * (t - 1)])

        def arr(p, n, ct=C.c_int32):
            if n == 0:
                return np.zeros(0, np.int32 if ct is C.c_int32 else np.float32)
            return np.ctypeslib.as_array(C.cast(p, C.POINTER(ct)), (n,)).copy()

        return {"del_src": arr(ptrs[0], nd), "del_dst": arr(ptrs[1], nd),
                "ins_src": arr(ptrs[2], ni), "ins_dst": arr(ptrs[3], ni),
                "changed": arr(ptrs[4], nc),
                "changed_feats": arr(ptrs[5], nc * self.dim, C.c_float).reshape(nc, self.dim)}

    def to_graph(self, stream=None) -> "DynamicGraph":
        h = C.c_void_p()
        check(lib().dgnn_synth_to_graph(self.h, _stream_handle(stream), C.byref(h)))
        return DynamicGraph._wrap(h, self.n, self.dim)


    def save(self, path, binary=True):
        """Writes the generator output as a dataset (format 2 binary by default;
        format 1 = the reference's text layout with structural deltas)."""
        check(lib().dgnn_synth_save(self.h, os.fsencode(path), 2 if binary else 1))


# ---------------------------------------------------------------- datasets
class Dataset:
    """Host-side reader of an on-disk dataset (ref load_dataset,
    src/dataset_io.cpp:98-165): the text layout (format 1) or the binary twin
    (format 2). Needs no GPU."""

    def __init__(self, path, threads=0):
        h = C.c_void_p()
        check(lib().dgnn_dataset_open(os.fsencode(path), threads, C.byref(h)))
        self.h = h
        n, d, T, fmt = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        check(lib().dgnn_dataset_info(self.h, C.byref(n), C.byref(d), C.byref(T), C.byref(fmt)))
        self.num_nodes, self.feature_dim, self.T, self.format = n.value, d.value, T.value, fmt.value

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None and _lib._lib is not None:
            lib().dgnn_dataset_free(self.h)
            self.h = None

    @staticmethod
    def _arr(p, n, ct=C.c_int32):
        if n == 0:
            return np.zeros(0, np.int32 if ct is C.c_int32 else np.float32)
        return np.ctypeslib.as_array(C.cast(p, C.POINTER(ct)), (n,)).copy()

    def base(self):
        E = C.c_int64()
        s, d, f = C.c_void_p(), C.c_void_p(), C.c_void_p()
        check(lib().dgnn_dataset_read_base(self.h, C.byref(E), C.byref(s), C.byref(d), C.byref(f)))
        n = self.num_nodes * self.feature_dim
        return (self._arr(s, E.value), self._arr(d, E.value),
                self._arr(f, n, C.c_float).reshape(self.num_nodes, self.feature_dim))

    def step(self, t):
        sizes = np.zeros(3, np.int64)
        ptrs = [C.c_void_p() for _ in range(6)]
        check(lib().dgnn_dataset_read_step(self.h, t, _np_ptr(sizes), *[C.byref(p) for p in ptrs]))
        nd, ni, nc = (int(x) for x in sizes)
        a = self._arr
        return {"del_src": a(ptrs[0], nd), "del_dst": a(ptrs[1], nd),
                "ins_src": a(ptrs[2], ni), "ins_dst": a(ptrs[3], ni), "changed": a(ptrs[4], nc),
                "changed_feats": a(ptrs[5], nc * self.feature_dim, C.c_float).reshape(nc, self.feature_dim)}


def load_dataset(path, stream=None, threads=0) -> "DynamicGraph":
    """load_dataset (src/dataset_io.cpp:98-165) straight into the HBM graph
    store, one step at a time."""
    info = Dataset(path)  # manifest only
    h = C.c_void_p()
    check(lib().dgnn_dataset_load(os.fsencode(path), threads, _stream_handle(stream), C.byref(h)))
    return DynamicGraph._wrap(h, info.num_nodes, info.feature_dim)


def save_dataset(graph: "DynamicGraph", path, binary=False):
    """save_dataset (src/dataset_io.cpp:40-95) of a device graph; format 1
    (reference text, default) or the binary twin."""
    check(lib().dgnn_dataset_save_graph(graph.h, os.fsencode(path), 2 if binary else 1))


# ------------------------------------------------------------------ ledgers
LEDGER_FIELDS = ("remote_features", "intermediate_redistribution", "gradient_sync", "snapshot_fetch")


def comm_ledger(graph: "DynamicGraph", scheme="consecutive_block", overlap="replicate_overlap",
                workers=1, seq_len=8, stride=1, horizon=1, hidden=16, num_params=0, num_batches=1):
    """CommLedger of one distributed epoch (ref inc/distsim.hpp:58-80,
    src/distsim.cpp:101-182): per-worker rows then the total, in bytes."""
    sch = {"consecutive_block": 0, "node_partition": 1, "sequence_partition": 2}[scheme]
    ov = {"replicate_overlap": 0, "remote_fetch": 1}[overlap]
    out = np.zeros((workers + 1, 4), np.uint64)
    check(lib().dgnn_comm_ledger(graph.h, sch, ov, workers, seq_len, stride, horizon, hidden,
                                 num_params, num_batches, _np_ptr(out)))
    return out


# ------------------------------------------------------------------ k-hop
class ComputationalGraph:
    """Sampled k-hop computational graph on the device (ref
    ComputationalGraph, inc/khop.hpp:42-51; khop, src/khop.cpp:66-96)."""

    def __init__(self, h, n):
        self.h, self.n = h, n

    @classmethod
    def khop(cls, graph: "DynamicGraph", t, seeds, fanouts, seed):
        s = np.ascontiguousarray(seeds, np.int32)
        f = np.ascontiguousarray(fanouts, np.int32)
        h = C.c_void_p()
        check(lib().dgnn_khop(graph.h, t, _np_ptr(s), len(s), _np_ptr(f), len(f), seed, C.byref(h)))
        return cls(h, graph.n)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None and _lib._lib is not None:
            lib().dgnn_cg_free(self.h)
            self.h = None

    def hops(self):
        out = []
        for k in range(lib().dgnn_cg_num_hops(self.h)):
            nd, ne = C.c_int64(), C.c_int64()
            check(lib().dgnn_cg_hop_sizes(self.h, k, C.byref(nd), C.byref(ne)))
            d = np.empty(nd.value, np.int32)
            s, t = np.empty(ne.value, np.int32), np.empty(ne.value, np.int32)
            check(lib().dgnn_cg_hop_copy(self.h, k, _np_ptr(d), _np_ptr(s), _np_ptr(t)))
            out.append({"dests": d, "src": s, "dst": t})
        return out

    def view(self):
        """to_view (src/khop.cpp:22-33): host copies of the device in-CSR."""
        ip, is_, op, od = (C.c_void_p() for _ in range(4))
        ne = C.c_int64()
        check(lib().dgnn_cg_view(self.h, C.byref(ip), C.byref(is_), C.byref(op), C.byref(od), C.byref(ne)))
        lib().dgnn_synchronize(None)
        ptr = device_view(ip.value, (self.n + 1,), np.int64).cpu().numpy()
        src = (device_view(is_.value, (ne.value,), np.int32).cpu().numpy() if ne.value
               else np.zeros(0, np.int32))
        return ptr, src

    def delta(self, graph: "DynamicGraph", t):
        """khop_delta (src/khop.cpp:105-121) -> (per-hop diffs, empty, apply_cg_update result)."""
        u = C.c_void_p()
        check(lib().dgnn_khop_delta(self.h, graph.h, t, C.byref(u)))
        try:
            hops = []
            for k in range(lib().dgnn_cg_num_hops(self.h)):
                na, nr = C.c_int64(), C.c_int64()
                check(lib().dgnn_cg_update_sizes(u, k, C.byref(na), C.byref(nr)))
                a = [np.empty(na.value, np.int32) for _ in range(2)]
                r = [np.empty(nr.value, np.int32) for _ in range(2)]
                check(lib().dgnn_cg_update_copy(u, k, *[_np_ptr(x) for x in a + r]))
                hops.append({"add_src": a[0], "add_dst": a[1], "rem_src": r[0], "rem_dst": r[1]})
            empty = bool(lib().dgnn_cg_update_empty(u))
            h = C.c_void_p()
            check(lib().dgnn_apply_cg_update(self.h, u, C.byref(h)))
            applied = ComputationalGraph(h, self.n)
        finally:
            lib().dgnn_cg_update_free(u)
        return hops, empty, applied


def synthesize(num_nodes, avg_degree, feature_dim, num_snapshots, edge_change, feature_change,
               seed=1, stream=None) -> "DynamicGraph":
    return Synth(num_nodes, avg_degree, feature_dim, num_snapshots, edge_change,
                 feature_change, seed).to_graph(stream)


class DynamicGraph:
    """Device-resident dynamic graph (ref DynamicGraph, inc/snapshot.hpp:92-107)."""

    def __init__(self, num_nodes: int, feature_dim: int, stream=None):
        h = C.c_void_p()
        check(lib().dgnn_graph_create(num_nodes, feature_dim, _stream_handle(stream), C.byref(h)))
        self.h, self.n, self.dim = h, num_nodes, feature_dim

    @classmethod
    def _wrap(cls, h, n, dim):
        g = cls.__new__(cls)
        g.h, g.n, g.dim = h, n, dim
        return g

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None and _lib._lib is not None:
            lib().dgnn_graph_free(self.h)
            self.h = None

    @classmethod
    def from_snapshots(cls, num_nodes, edges_per_t, feats_per_t, stream=None):
        """Snapshot ctor per step (src/snapshot.cpp:20-69)."""
        g = cls(num_nodes, np.asarray(feats_per_t[0]).shape[1], stream)
        for e, f in zip(edges_per_t, feats_per_t):
            g.add_snapshot(e, f)
        return g

    def add_snapshot(self, edges, feats):
        e = np.ascontiguousarray(np.asarray(edges, np.int32).reshape(-1, 2))
        src, dst = np.ascontiguousarray(e[:, 0]), np.ascontiguousarray(e[:, 1])
        f = np.ascontiguousarray(feats, np.float32)
        check(lib().dgnn_graph_add_snapshot(self.h, _np_ptr(src), _np_ptr(dst), len(src), _np_ptr(f)))

    def add_delta(self, deletions, insertions, changed_nodes=(), changed_feats=None):
        """apply_delta (src/snapshot.cpp:142-154)."""
        d = np.ascontiguousarray(np.asarray(deletions, np.int32).reshape(-1, 2))
        i = np.ascontiguousarray(np.asarray(insertions, np.int32).reshape(-1, 2))
        c = np.ascontiguousarray(np.asarray(changed_nodes, np.int32))
        cf = np.ascontiguousarray(np.zeros((0, self.dim), np.float32) if changed_feats is None
                                  else np.asarray(changed_feats, np.float32))
        ds, dd = np.ascontiguousarray(d[:, 0]), np.ascontiguousarray(d[:, 1])
        is_, id_ = np.ascontiguousarray(i[:, 0]), np.ascontiguousarray(i[:, 1])
        check(lib().dgnn_graph_add_delta(self.h, _np_ptr(ds), _np_ptr(dd), len(ds), _np_ptr(is_),
                                         _np_ptr(id_), len(is_), _np_ptr(c), len(c), _np_ptr(cf)))

    def length(self) -> int:
        return lib().dgnn_graph_length(self.h)

    def retain(self, t_first: int, t_last: int):
        """Keep only snapshots [t_first, t_last] in HBM (a rank's window block
        plus the L+H overlap); indices stay global."""
        check(lib().dgnn_graph_retain(self.h, t_first, t_last))

    def retain_for_rank(self, world: int, rank: int, L: int, S: int, H: int):
        """retain() the snapshots rank `rank` of a consecutive-block plan over
        sliding_windows(length - 1, L, S, H) reads (windows, their targets)."""
        row = plan(self.length() - 1, world, L, S, H)[rank]
        wb, we = int(row[2]), int(row[3])
        if we <= wb:  # no windows on this rank: keep everything
            return 0, self.length() - 1
        starts = sliding_windows(self.length() - 1, L, S, H)
        first, last = starts[wb], min(self.length() - 1, starts[we - 1] + L + H)
        self.retain(first, last)
        return first, last

    def device_bytes(self) -> int:
        return lib().dgnn_graph_device_bytes(self.h)

    def feature_stats(self) -> dict:
        s, m = C.c_int32(), C.c_int64()
        check(lib().dgnn_graph_feature_stats(self.h, C.byref(s), C.byref(m)))
        return {"slots": s.value, "materialisations": m.value}

    def num_edges(self, t) -> int:
        n = lib().dgnn_graph_num_edges(self.h, t)
        if n < 0:
            raise IndexError(lib().dgnn_last_error().decode())
        return n

    def snapshot_ptrs(self, t):
        ptrs = [C.c_void_p() for _ in range(5)]
        check(lib().dgnn_graph_snapshot(self.h, t, *[C.byref(p) for p in ptrs]))
        return [p.value for p in ptrs]

    def _dev_to_numpy(self, ptr, n, dtype):
        if n == 0:
            return np.zeros(0, dtype)
        lib().dgnn_synchronize(None)
        return device_view(ptr, (n,), dtype).cpu().numpy()

    def in_csr(self, t):
        ip, isrc, _, _, _ = self.snapshot_ptrs(t)
        E = self.num_edges(t)
        return self._dev_to_numpy(ip, self.n + 1, np.int64), self._dev_to_numpy(isrc, E, np.int32)

    def out_csr(self, t):
        _, _, op, od, _ = self.snapshot_ptrs(t)
        E = self.num_edges(t)
        return self._dev_to_numpy(op, self.n + 1, np.int64), self._dev_to_numpy(od, E, np.int32)

    def feats(self, t):
        f = self.snapshot_ptrs(t)[4]
        return self._dev_to_numpy(f, self.n * self.dim, np.float32).reshape(self.n, self.dim)

    def feats_tensor(self, t):
        """Zero-copy-free device copy of snapshot t's features as a torch tensor."""
        torch = _torch()
        return torch.from_numpy(self.feats(t)).cuda()

    def edges(self, t):
        ptr, dst = self.out_csr(t)
        src = np.repeat(np.arange(self.n, dtype=np.int32), np.diff(ptr))
        return src, dst

    def delta_sizes(self, t):
        vals = [C.c_int64() for _ in range(6)]
        check(lib().dgnn_graph_delta_sizes(self.h, t, *[C.byref(v) for v in vals]))
        keys = ["n_del", "n_ins", "n_changed", "n_rows", "u_minus", "u_plus"]
        return {k: v.value for k, v in zip(keys, vals)}

    def delta(self, t):
        s = self.delta_sizes(t)
        ds, dd = np.empty(s["n_del"], np.int32), np.empty(s["n_del"], np.int32)
        is_, id_ = np.empty(s["n_ins"], np.int32), np.empty(s["n_ins"], np.int32)
        ch = np.empty(s["n_changed"], np.int32)
        check(lib().dgnn_graph_delta_copy(self.h, t, _np_ptr(ds), _np_ptr(dd), _np_ptr(is_),
                                          _np_ptr(id_), _np_ptr(ch)))
        return {"del_src": ds, "del_dst": dd, "ins_src": is_, "ins_dst": id_, "changed": ch}

    def delta_layout(self, t):
        ptrs = [C.c_void_p() for _ in range(3)]
        check(lib().dgnn_graph_delta_layout(self.h, t, *[C.byref(p) for p in ptrs]))
        return [p.value for p in ptrs]

    def change_ratio(self, t) -> float:
        r = lib().dgnn_graph_change_ratio(self.h, t)
        if r < 0:
            raise ValueError(lib().dgnn_last_error().decode())
        return r


# ------------------------------------------------------------- aggregation
def aggregate_scratch(graph: DynamicGraph, t: int, feats, kind="sum", stream=None):
    """K1 over snapshot t's in-CSR; feats: (n, w) float32 CUDA tensor."""
    torch = _torch()
    n, w = feats.shape
    ip, isrc, _, _, _ = graph.snapshot_ptrs(t)
    out = {"values": torch.empty(n, w, device="cuda")}
    if kind == "mean":
        out["degree"] = torch.empty(n, device="cuda")
        out["mean_sums"] = torch.empty(n, w, device="cuda")
    if kind in ("max", "min"):
        out["argext"] = torch.empty(n, w, dtype=torch.int32, device="cuda")
    check(lib().dgnn_agg_scratch(AGGR[kind], n, w, C.c_void_p(ip), C.c_void_p(isrc), _ptr(feats),
                                 _ptr(out["values"]), _ptr(out.get("degree")),
                                 _ptr(out.get("mean_sums")), _ptr(out.get("argext")),
                                 _stream_handle(stream or current_stream())))
    return out


def aggregate_delta_inplace(graph: DynamicGraph, t: int, agg: dict, f_prev, f_curr, kind="sum",
                            stream=None):
    """K2: apply delta(t) in place to an aggregation holding Agg_{t-1}."""
    n, w = agg["values"].shape
    rows, row_ptr, ent = graph.delta_layout(t)
    nr = graph.delta_sizes(t)["n_rows"]
    check(lib().dgnn_agg_delta(AGGR[kind], nr, w, C.c_void_p(rows), C.c_void_p(row_ptr),
                               C.c_void_p(ent), _ptr(f_prev), _ptr(f_curr), _ptr(agg["values"]),
                               _ptr(agg.get("degree")), _ptr(agg.get("mean_sums")),
                               _ptr(agg.get("argext")), _stream_handle(stream or current_stream())))
    return agg


def apply_graph_delta(graph: DynamicGraph, t: int, agg: dict, kind="sum", stream=None):
    """K2 on the graph's own delta(t) and feature versions (compact changed-row
    block): agg holds Agg_{t-1} of the graph features and becomes Agg_t."""
    check(lib().dgnn_graph_apply_delta(graph.h, t, AGGR[kind], _ptr(agg["values"]),
                                       _ptr(agg.get("degree")), _ptr(agg.get("mean_sums")),
                                       _ptr(agg.get("argext")),
                                       _stream_handle(stream or current_stream())))
    return agg


def aggregate_incremental(graph: DynamicGraph, t: int, prev: dict, kind="sum", prev_depth=0,
                          prev_num_edges=None, fallback_threshold=0.5, rescratch_period=64):
    """aggregate_incremental with the reference's fallback logic (src/aggregate.cpp:117-207)."""
    torch = _torch()
    n, w = prev["values"].shape
    if prev_num_edges is None:
        prev_num_edges = graph.num_edges(t - 1)
    out = {"values": torch.empty(n, w, device="cuda")}
    if kind == "mean":
        out["degree"] = torch.empty(n, device="cuda")
        out["mean_sums"] = torch.empty(n, w, device="cuda")
    if kind in ("max", "min"):
        out["argext"] = torch.empty(n, w, dtype=torch.int32, device="cuda")
    info = np.zeros(3, np.int32)
    torch.cuda.synchronize()
    check(lib().dgnn_agg_incremental(graph.h, t, AGGR[kind], _ptr(prev["values"]),
                                     _ptr(prev.get("degree")), _ptr(prev.get("mean_sums")),
                                     _ptr(prev.get("argext")), prev_depth, prev_num_edges,
                                     fallback_threshold, rescratch_period, _ptr(out["values"]),
                                     _ptr(out.get("degree")), _ptr(out.get("mean_sums")),
                                     _ptr(out.get("argext")), _np_ptr(info)))
    out["used_fallback"], out["reason"], out["depth"] = bool(info[0]), int(info[1]), int(info[2])
    return out


def aggregate_backward(graph: DynamicGraph, t: int, upstream, kind="sum", forward=None,
                       stream=None):
    """K3: grad[u] = sum over out-edges of upstream (ref src/aggregate.cpp:209-246)."""
    torch = _torch()
    n, w = upstream.shape
    _, _, op, od, _ = graph.snapshot_ptrs(t)
    grad = torch.empty(n, w, device="cuda")
    forward = forward or {}
    check(lib().dgnn_agg_backward(AGGR[kind], n, w, C.c_void_p(op), C.c_void_p(od), _ptr(upstream),
                                  _ptr(forward.get("degree")), _ptr(forward.get("argext")),
                                  _ptr(grad), _stream_handle(stream or current_stream())))
    return grad


# ------------------------------------------------------------------ cells
def pack_cell(lstm: bool, n_in: int, H: int, flat):
    torch = _torch()
    W = torch.empty((n_in + H) * 4 * H, device="cuda")
    b = torch.empty(4 * H, device="cuda")
    check(lib().dgnn_pack_cell(int(lstm), n_in, H, _ptr(flat), _ptr(W), _ptr(b),
                               _stream_handle(current_stream())))
    return W, b


def cell_forward(lstm, X, Hm, h_skip, c_prev, flat):
    """Fused cell_core_forward (src/cells.cpp:102-132)."""
    torch = _torch()
    n, n_in = X.shape
    H = Hm.shape[1]
    W, b = pack_cell(lstm, n_in, H, flat)
    gates = torch.empty(n, 4 * H, device="cuda")
    c = torch.empty(n, H, device="cuda") if lstm else None
    h = torch.empty(n, H, device="cuda")
    check(lib().dgnn_cell_forward(int(lstm), n, n_in, H, _ptr(X), _ptr(Hm), _ptr(h_skip),
                                  _ptr(c_prev), _ptr(W), _ptr(b), _ptr(gates), _ptr(c), _ptr(h),
                                  _stream_handle(current_stream())))
    return {"gates": gates, "c": c, "h": h, "W": W, "b": b}


def cell_backward(lstm, X, Hm, fwd, h_skip, c_prev, dh, dc, need_dx=True):
    """cell_core_backward (src/cells.cpp:134-195): returns dX, dHm, dc_prev/dh_skip, dflat."""
    torch = _torch()
    n, n_in = X.shape
    H = Hm.shape[1]
    K = 4 if lstm else 3
    dX = torch.empty(n, n_in, device="cuda") if need_dx else None
    dHm = torch.empty(n, H, device="cuda")
    dcp = torch.empty(n, H, device="cuda") if lstm else None
    dhs = None if lstm else torch.empty(n, H, device="cuda")
    dflat = torch.zeros(K * (n_in * H + H * H + H), device="cuda")
    check(lib().dgnn_cell_backward(int(lstm), n, n_in, H, _ptr(X), _ptr(Hm), _ptr(fwd["W"]),
                                   _ptr(fwd["gates"]), _ptr(fwd["c"]), _ptr(c_prev), _ptr(h_skip),
                                   _ptr(dh), _ptr(dc), _ptr(dX), _ptr(dHm), _ptr(dcp), _ptr(dhs),
                                   _ptr(dflat), _stream_handle(current_stream())))
    return {"dX": dX, "dHm": dHm, "dc_prev": dcp, "dh_skip": dhs, "dflat": dflat}


# ------------------------------------------------------------------ training
@dataclass
class TrainConfig:
    """RunSettings defaults (ref inc/config.hpp:18-57) plus the B200 cache budget."""
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
    window_total: int = 0
    record_events: bool = False
    hbm_cache_budget_bytes: int = 0
    fanouts: tuple = ()  # () or all -1: whole-snapshot views; else sampled k-hop views
    iteration: str = "seq_first"  # or "node_first" (ref IterationOrder)

    def to_c(self) -> _lib.RunCfg:
        c = _lib.RunCfg()
        c.arch, c.layers, c.hidden = ARCH[self.arch], self.layers, self.hidden
        c.seq_len, c.horizon, c.teacher_forcing = self.seq_len, self.horizon, int(self.teacher_forcing)
        c.aggr, c.batch_size, c.seed = AGGR[self.aggr], self.batch_size, self.seed
        c.lr, c.optimizer, c.stride = self.lr, 0 if self.optimizer == "sgd" else 1, self.stride
        c.fallback_threshold, c.rescratch_period = self.fallback_threshold, self.rescratch_period
        c.incremental, c.cache_policy, c.cache_frac = int(self.incremental), POLICY[self.cache], self.cache_frac
        c.workers, c.epochs, c.window_total = self.workers, self.epochs, self.window_total
        c.record_events, c.hbm_cache_budget_bytes = int(self.record_events), self.hbm_cache_budget_bytes
        if len(self.fanouts) > 8:
            raise ValueError("at most 8 fanout hops")
        c.n_fanouts = len(self.fanouts)
        for i, f in enumerate(self.fanouts):
            c.fanouts[i] = f
        c.iteration = {"seq_first": 0, "node_first": 1}[self.iteration]
        return c


class Comm:
    """The sharded trainer's gradient all-reduce (NCCL, in the library).
    `Comm.unique_id()` on rank 0, the 128 bytes shared with every rank by the
    caller, then `Comm(uid, world, rank)` on each (device already selected)."""

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(lib().dgnn_comm_unique_id(buf))
        return bytes(buf)

    def __init__(self, uid: bytes, world: int, rank: int):
        assert len(uid) == 128
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        check(lib().dgnn_comm_create(buf, world, rank, C.byref(h)))
        self.h, self.world, self.rank = h, world, rank

    def allreduce(self, t, stream=None):
        """In-place fp32 sum over ranks of a CUDA tensor."""
        if stream is None:
            stream = current_stream()
        check(lib().dgnn_grad_allreduce(self.h, _ptr(t), t.numel(), _stream_handle(stream)))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None and _lib._lib is not None:
            lib().dgnn_comm_free(self.h)
            self.h = None


def comm_from_torch(world: int, rank: int) -> "Comm | None":
    """Build the library's communicator, exchanging the NCCL id over the
    default torch.distributed group (None for one rank)."""
    if world <= 1:
        return None
    import torch
    import torch.distributed as dist
    uid = Comm.unique_id() if rank == 0 else bytes(128)
    t = torch.tensor(list(uid), dtype=torch.uint8, device="cuda")
    dist.broadcast(t, 0)
    return Comm(bytes(t.cpu().tolist()), world, rank)


class TrainSession:
    """TrainSession / DistSession rank over a device graph (ref inc/train.hpp:92-114,
    inc/distsim.hpp:82-102). workers == 0: seq-first; workers >= 1: rank `rank` of
    the consecutive-block sharded trainer."""

    def __init__(self, graph: DynamicGraph, cfg: TrainConfig, rank: int = 0, stream=None):
        self.graph, self.cfg = graph, cfg
        self._c = cfg.to_c()
        if stream is None:  # run on the caller's torch stream: ordering with torch ops is implicit
            stream = current_stream()
        h = C.c_void_p()
        check(lib().dgnn_session_create(graph.h, C.byref(self._c), rank, _stream_handle(stream),
                                        C.byref(h)))
        self.h = h
        self.num_params = lib().dgnn_session_num_params(self.h)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None and _lib._lib is not None:
            lib().dgnn_session_free(self.h)
            self.h = None

    def windows(self):
        tot, b, e = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib().dgnn_session_num_windows(self.h, C.byref(tot), C.byref(b), C.byref(e)))
        return tot.value, b.value, e.value

    def params(self) -> np.ndarray:
        out = np.empty(self.num_params, np.float64)
        check(lib().dgnn_session_get_params(self.h, _np_ptr(out)))
        return out

    def set_params(self, p):
        p = np.ascontiguousarray(p, np.float64)
        check(lib().dgnn_session_set_params(self.h, _np_ptr(p)))

    def initial_params(self) -> np.ndarray:
        out = np.empty(self.num_params, np.float64)
        check(lib().dgnn_session_initial_params(self.h, _np_ptr(out)))
        return out

    def run_epoch(self) -> dict:
        r = _lib.EpochReport()
        check(lib().dgnn_session_run_epoch(self.h, C.byref(r)))
        out = {k: getattr(r, k) for k, _ in _lib.EpochReport._fields_}
        out["sample_losses"] = self.losses()
        return out

    def begin_epoch(self) -> int:
        nb = C.c_int64()
        check(lib().dgnn_session_begin_epoch(self.h, C.byref(nb)))
        return nb.value

    def local_grads(self, batch: int, grad_sum):
        check(lib().dgnn_session_local_grads(self.h, batch, _ptr(grad_sum)))

    def apply(self, grad_sum) -> bool:
        a = C.c_int32()
        check(lib().dgnn_session_apply(self.h, _ptr(grad_sum), C.byref(a)))
        return bool(a.value)

    def end_epoch(self):
        check(lib().dgnn_session_end_epoch(self.h))

    def run_dist_epoch(self, comm: "Comm | None" = None) -> dict:
        """One whole sharded epoch in the library (NCCL all-reduce through
        `comm`; None for a single rank). seconds = device time, max over ranks."""
        r = _lib.EpochReport()
        check(lib().dgnn_session_run_dist_epoch(self.h, comm.h if comm is not None else None,
                                                C.byref(r)))
        out = {k: getattr(r, k) for k, _ in _lib.EpochReport._fields_}
        out["sample_losses"] = self.losses()
        return out

    def run_sharded_epoch(self, allreduce=None) -> list[float]:
        """One distsim epoch on this rank; `allreduce(tensor)` sums over ranks."""
        from .sharding import run_sharded_epoch
        torch = _torch()
        g = torch.empty(self.num_params, device="cuda")
        run_sharded_epoch(self, g, allreduce)
        return self.losses()

    def losses(self) -> np.ndarray:
        n = C.c_int64()
        check(lib().dgnn_session_losses(self.h, None, C.byref(n)))
        out = np.empty(n.value, np.float64)
        check(lib().dgnn_session_losses(self.h, _np_ptr(out), C.byref(n)))
        return out

    def sample_grads(self, window_index=0):
        loss = C.c_double()
        pred0 = np.empty((self.graph.n, self.graph.dim), np.float32)
        grads = np.empty(self.num_params, np.float64)
        check(lib().dgnn_session_sample_grads(self.h, window_index, C.byref(loss), _np_ptr(pred0),
                                              _np_ptr(grads)))
        return loss.value, pred0, grads

    def invocations(self) -> np.ndarray:
        n = C.c_int64()
        check(lib().dgnn_session_invocations(self.h, None, C.byref(n)))
        out = np.empty((n.value, 4), np.int32)
        check(lib().dgnn_session_invocations(self.h, _np_ptr(out), C.byref(n)))
        return out

    def cache_events(self) -> np.ndarray:
        n = C.c_int64()
        check(lib().dgnn_session_cache_events(self.h, None, C.byref(n)))
        out = np.empty((n.value, 10), np.int64)
        check(lib().dgnn_session_cache_events(self.h, _np_ptr(out), C.byref(n)))
        return out

    def stats(self) -> dict:
        out = np.empty(12, np.int64)
        check(lib().dgnn_session_stats(self.h, _np_ptr(out)))
        keys = ["hits", "misses", "evictions", "expirations", "invalidations", "rejected",
                "scratch_calls", "incremental_calls", "fallbacks", "spills", "refills",
                "resident_peak_units"]
        return dict(zip(keys, out.tolist()))

    def tier_stats(self) -> dict:
        """Second cache level (HBM <-> pinned host placement) counters."""
        out = np.empty(8, np.int64)
        check(lib().dgnn_session_tier_stats(self.h, _np_ptr(out)))
        keys = ["spills", "refills", "prefetches", "demand_refills", "spill_bytes", "refill_bytes",
                "pinned_bytes", "hbm_resident_bytes"]
        return dict(zip(keys, out.tolist()))


# ------------------------------------------------------------------ profiling
PROF_CLASSES = ["agg_scratch", "agg_delta", "agg_backward", "cell_fwd", "cell_bwd",
                "weight_grad", "other", "cell_bwd_gemm", "agg_rebase"]
# non-kernel scopes (not part of kernel-time sums)
PROF_SCOPES = ["sample", "sample_host", "host_build", "host_fwd", "host_bwd", "host_alloc"]


def mem_stats() -> dict:
    """Device pool occupancy in bytes (reserved / used, current and high-water)."""
    v = [C.c_int64() for _ in range(4)]
    check(lib().dgnn_mem_stats(*[C.byref(x) for x in v]))
    return dict(zip(["reserved", "used", "reserved_high", "used_high"], [x.value for x in v]))


def prof_enable(on=True):
    check(lib().dgnn_prof_enable(int(on)))


def prof_reset():
    check(lib().dgnn_prof_reset())


def prof_get(scopes=False) -> dict:
    """Per kernel class: launches, device ms, algorithmic bytes / flops, longest
    launch. scopes=True returns the non-kernel scopes (whole samples) instead."""
    out = {}
    names = PROF_SCOPES if scopes else PROF_CLASSES
    base = len(PROF_CLASSES) if scopes else 0
    for i, name in enumerate(names):
        n, ms, b, f, mx = C.c_int64(), C.c_double(), C.c_double(), C.c_double(), C.c_double()
        check(lib().dgnn_prof_get(base + i, C.byref(n), C.byref(ms), C.byref(b), C.byref(f)))
        check(lib().dgnn_prof_get_max(base + i, C.byref(mx)))
        out[name] = {"launches": n.value, "ms": ms.value, "bytes": b.value, "flops": f.value,
                     "max_ms": mx.value}
    return out
