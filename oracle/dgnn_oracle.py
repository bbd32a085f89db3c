"""CPU restatement (numpy, fp64) of the reference's hot-path algorithm.

TEST INFRASTRUCTURE ONLY — the parity checker, never the product. Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline leg may import it.

Each function cites the reference file:line it restates (/root/reference/proj).
It is pinned in two ways (see tests/test_oracle_cpu.py):
  * against the reference itself, compiled from its unmodified sources with an
    Eigen-subset shim (oracle/_ref, oracle/Makefile), on random cases;
  * against golden fixtures under tests/golden/ generated from that compiled
    reference by tests/golden/make_golden.py, and against the SPEC's
    known-answer examples.
"""
from __future__ import annotations

import math

import numpy as np

MASK64 = (1 << 64) - 1
SUM, MEAN, MAX, MIN = 0, 1, 2, 3
KIND = {"sum": SUM, "mean": MEAN, "max": MAX, "min": MIN}


# ------------------------------------------------------------------ common
def mix64(x: int) -> int:
    """splitmix64 finaliser (inc/common.hpp:43-48)."""
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK64
    return x ^ (x >> 31)


def derive_seed(seed: int, a: int, b: int = 0, c: int = 0) -> int:
    """inc/common.hpp:50-52."""
    u = lambda v: v & MASK64
    return mix64(mix64(mix64(u(seed) ^ mix64(u(a))) ^ mix64(u(b))) ^ mix64(u(c)))


def key_hash(level: int, layer: int, t: int, kind: int, batch: int, serial: int) -> int:
    """AggKeyHash (inc/cache.hpp:54-61)."""
    u = lambda v: v & MASK64
    h = derive_seed(u(t), u(layer), u(batch), u(serial))
    return mix64(h ^ (level << 8) ^ (kind << 16))


# ------------------------------------------------------------------ windows / plan
def sliding_windows(total: int, L: int, S: int, H: int) -> list[int]:
    """Window starts 0, S, ... while start + L + H <= T (src/windows.cpp:5-15)."""
    if L < 1 or S < 1 or H < 0:
        raise ValueError("sliding_windows: bad L/S/H")
    out, start = [], 0
    while start + L + H <= total:
        out.append(start)
        start += S
    return out


def plan_consecutive_block(total: int, M: int, L: int, S: int, H: int):
    """Consecutive-block plan (src/distsim.cpp:35-81): rows
    (block_begin, block_end, window_begin, window_end)."""
    if M < 1:
        raise ValueError("plan needs at least one worker")
    if total < M:
        raise ValueError("fewer snapshots than workers")
    starts = sliding_windows(total, L, S, H)
    W = len(starts)
    base, extra = W // M, W % M
    rows, cur = [], 0
    for m in range(M):
        wb = cur
        we = cur + base + (1 if m < extra else 0)
        cur = we
        bb = starts[wb] if wb < W else total
        be = (starts[we] if we < W else total) if m + 1 < M else total
        rows.append([min(bb, be), be, wb, we])
    rows[0][0] = 0
    return np.array(rows, np.int64)


# ------------------------------------------------------------------ cache scores
def future_access_count(num_layers, gates, gate, L, S, idx, part, layer, horizon,
                        windows_remaining, kind) -> int:
    """Visit-counting F (src/cache.cpp:27-53); part 0 encoder, 1 decoder; kind 0 input."""
    if not (1 <= gate <= gates):
        raise ValueError("gate must lie in 1..K")
    if not (1 <= layer <= num_layers):
        raise ValueError("layer must lie in 1..D")
    if idx < 0:
        raise ValueError("window position must be non-negative")
    if not (layer == 1 and kind == 0):
        return gates - gate
    wrem = windows_remaining
    if part == 0:
        visits = min(idx // S, wrem)
    else:
        j = idx
        visits = min(j // S, wrem)
        lo = (j + S) // S
        hi = min((L + j) // S, wrem)
        if hi >= lo:
            visits += hi - lo + 1
    return max((visits + 1) * gates - gate, 0)


def imminence(L, S, part, layer, kind) -> int:
    """src/cache.cpp:55-62."""
    if not (layer == 1 and kind == 0):
        return 0
    return max(L - S, 0) if part == 0 else max(L - 1, 0)


def entry_priority(f, size_units, imm):
    """inc/cache.hpp:86-88."""
    return f / size_units - imm


# ------------------------------------------------------------------ snapshots
def edge_keys(src, dst) -> np.ndarray:
    return (np.asarray(src, np.int64) << 32) | np.asarray(dst, np.int64)


def split_keys(keys):
    keys = np.asarray(keys, np.int64)
    return (keys >> 32).astype(np.int32), (keys & 0xFFFFFFFF).astype(np.int32)


def build_csr(src, dst, n):
    """Snapshot ctor (src/snapshot.cpp:20-69): sorted unique (src,dst), in-CSR
    with sources ascending per destination, out-CSR with destinations ascending."""
    keys = edge_keys(src, dst)
    if len(keys) and (np.min(src) < 0 or np.max(src) >= n or np.min(dst) < 0 or np.max(dst) >= n):
        raise ValueError("edge endpoint out of range")
    keys = np.sort(keys)
    if len(keys) > 1 and np.any(keys[1:] == keys[:-1]):
        raise ValueError("duplicate edge in snapshot")
    s, d = split_keys(keys)
    out_ptr = np.zeros(n + 1, np.int64)
    np.add.at(out_ptr, s.astype(np.int64) + 1, 1)
    out_ptr = np.cumsum(out_ptr)
    order = np.lexsort((s, d))  # by dst then src
    in_src = s[order]
    in_ptr = np.zeros(n + 1, np.int64)
    np.add.at(in_ptr, d.astype(np.int64) + 1, 1)
    in_ptr = np.cumsum(in_ptr)
    return {"keys": keys, "in_ptr": in_ptr, "in_src": in_src, "out_ptr": out_ptr, "out_dst": d}


def extract_delta(prev, curr, prev_feats, curr_feats):
    """src/snapshot.cpp:102-130. prev/curr: build_csr() dicts."""
    pk, ck = prev["keys"], curr["keys"]
    d1 = np.setdiff1d(pk, ck, assume_unique=True)
    i1 = np.setdiff1d(ck, pk, assume_unique=True)
    changed = np.nonzero(np.any(prev_feats != curr_feats, axis=1))[0].astype(np.int32)
    dels, inss = [d1], [i1]
    for u in changed:
        a, b = prev["out_ptr"][u], prev["out_ptr"][u + 1]
        dels.append(edge_keys(np.full(b - a, u), prev["out_dst"][a:b]))
        a, b = curr["out_ptr"][u], curr["out_ptr"][u + 1]
        inss.append(edge_keys(np.full(b - a, u), curr["out_dst"][a:b]))
    dk = np.unique(np.concatenate(dels)) if dels else np.zeros(0, np.int64)
    ik = np.unique(np.concatenate(inss)) if inss else np.zeros(0, np.int64)
    ds, dd = split_keys(dk)
    is_, id_ = split_keys(ik)
    return {"del_src": ds, "del_dst": dd, "ins_src": is_, "ins_dst": id_, "changed": changed,
            "changed_feats": curr_feats[changed]}


def change_ratio(delta, base_edges: int) -> float:
    """src/snapshot.cpp:132-135."""
    if base_edges <= 0:
        return math.inf
    return (len(delta["del_src"]) + len(delta["ins_src"])) / (2.0 * base_edges)


def apply_delta(prev_keys, prev_feats, delta):
    """src/snapshot.cpp:142-154: ((prev \\ deletions) U insertions), rows patched."""
    keep = np.setdiff1d(prev_keys, edge_keys(delta["del_src"], delta["del_dst"]))
    keys = np.union1d(keep, edge_keys(delta["ins_src"], delta["ins_dst"]))
    feats = prev_feats.copy()
    feats[delta["changed"]] = delta["changed_feats"]
    return keys, feats


# ------------------------------------------------------------------ aggregation
def aggregate_scratch(in_ptr, in_src, feats, kind):
    """src/aggregate.cpp:55-115 (unweighted). Returns dict values/degree/mean_sums/argext."""
    kind = KIND.get(kind, kind)
    n = len(in_ptr) - 1
    w = feats.shape[1]
    deg = np.diff(in_ptr)
    dst = np.repeat(np.arange(n), deg)
    out = {"kind": kind}
    if kind in (SUM, MEAN):
        acc = np.zeros((n, w))
        np.add.at(acc, dst, feats[in_src])  # sequential in edge order per row
        if kind == SUM:
            out["values"] = acc
        else:
            out["degree"] = deg.astype(np.float64)
            out["mean_sums"] = acc
            vals = np.zeros_like(acc)
            nz = deg > 0
            vals[nz] = acc[nz] / deg[nz, None]
            out["values"] = vals
        return out
    init = -np.inf if kind == MAX else np.inf
    vals = np.full((n, w), init)
    arg = np.full((n, w), -1, np.int32)
    for v in range(n):
        for e in range(in_ptr[v], in_ptr[v + 1]):
            u = in_src[e]
            x = feats[u]
            better = (arg[v] < 0) | ((x > vals[v]) if kind == MAX else (x < vals[v]))
            vals[v, better] = x[better]
            arg[v, better] = u
    out["values"] = vals
    out["argext"] = arg
    return out


def aggregate_incremental(prev, prev_num_edges, prev_depth, curr_csr, prev_feats, curr_feats,
                          delta, kind, threshold=0.5, rescratch=64):
    """Eq. 2 with the reference's fallbacks (src/aggregate.cpp:117-207).
    Returns (result, used_fallback, reason, depth); reason 0 none, 1 change
    ratio, 2 deleted contributor, 3 rescratch period."""
    kind = KIND.get(kind, kind)

    def fallback(why):
        return aggregate_scratch(curr_csr["in_ptr"], curr_csr["in_src"], curr_feats, kind), True, why, 0

    if change_ratio(delta, prev_num_edges) > threshold:
        return fallback(1)
    if rescratch > 0 and prev_depth + 1 >= rescratch:
        return fallback(3)
    ds, dd, is_, id_ = delta["del_src"], delta["del_dst"], delta["ins_src"], delta["ins_dst"]
    if kind in (MAX, MIN):
        if len(ds) and np.any(prev["argext"][dd] == ds[:, None]):
            return fallback(2)
        vals = prev["values"].copy()
        arg = prev["argext"].copy()
        for u, v in zip(is_, id_):
            x = curr_feats[u]
            better = (arg[v] < 0) | ((x > vals[v]) if kind == MAX else (x < vals[v]))
            vals[v, better] = x[better]
            arg[v, better] = u
        return {"kind": kind, "values": vals, "argext": arg}, False, 0, prev_depth + 1
    acc = (prev["mean_sums"] if kind == MEAN else prev["values"]).copy()
    np.subtract.at(acc, dd, prev_feats[ds])
    np.add.at(acc, id_, curr_feats[is_])
    if kind == SUM:
        return {"kind": kind, "values": acc}, False, 0, prev_depth + 1
    deg = prev["degree"].copy()
    np.subtract.at(deg, dd, 1.0)
    np.add.at(deg, id_, 1.0)
    keep = deg > 1e-12
    vals = np.zeros_like(acc)
    vals[keep] = acc[keep] / deg[keep, None]
    deg[~keep] = 0.0
    acc[~keep] = 0.0
    return {"kind": kind, "values": vals, "degree": deg, "mean_sums": acc}, False, 0, prev_depth + 1


def aggregate_backward(in_ptr, in_src, upstream, kind, forward=None):
    """src/aggregate.cpp:209-246."""
    kind = KIND.get(kind, kind)
    n = len(in_ptr) - 1
    grad = np.zeros_like(upstream, dtype=np.float64)
    deg = np.diff(in_ptr)
    dst = np.repeat(np.arange(n), deg)
    if kind == SUM:
        np.add.at(grad, in_src, upstream[dst])
    elif kind == MEAN:
        d = forward["degree"]
        inv = np.where(d > 0, 1.0 / np.where(d > 0, d, 1.0), 0.0)
        np.add.at(grad, in_src, inv[dst, None] * upstream[dst])
    else:
        arg = forward["argext"]
        v, c = np.nonzero(arg >= 0)
        np.add.at(grad, (arg[v, c], c), upstream[v, c])
    return grad


def dense_values(agg):
    """AggResult::dense_values (src/aggregate.cpp:30-37)."""
    if "argext" not in agg:
        return agg["values"]
    out = agg["values"].copy()
    out[agg["argext"][:, 0] < 0] = 0.0
    return out


# ------------------------------------------------------------------ cells
def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def split_cell_params(flat, lstm, n_in, H):
    """[wx_g (in x H), uh_g (H x H), b_g (1 x H)]_g (src/cells.cpp:75-100)."""
    K = 4 if lstm else 3
    wx, uh, b, off = [], [], [], 0
    for _ in range(K):
        wx.append(flat[off:off + n_in * H].reshape(n_in, H)); off += n_in * H
        uh.append(flat[off:off + H * H].reshape(H, H)); off += H * H
        b.append(flat[off:off + H]); off += H
    return wx, uh, b


def cell_core_forward(flat, lstm, X, Hm, h_skip, c_prev):
    """src/cells.cpp:102-132."""
    n_in, H = X.shape[1], Hm.shape[1]
    wx, uh, b = split_cell_params(flat, lstm, n_in, H)
    pre = lambda g: X @ wx[g] + Hm @ uh[g] + b[g]
    if lstm:
        i, f, gg, o = sigmoid(pre(0)), sigmoid(pre(1)), np.tanh(pre(2)), sigmoid(pre(3))
        c = f * c_prev + i * gg
        return {"gates": [i, f, gg, o], "c": c, "c_prev": c_prev, "h": o * np.tanh(c), "h_skip": h_skip}
    r, z = sigmoid(pre(0)), sigmoid(pre(1))
    hn = Hm @ uh[2]
    n = np.tanh(X @ wx[2] + r * hn + b[2])
    return {"gates": [r, z, n], "hn": hn, "h": (1 - z) * n + z * h_skip, "h_skip": h_skip}


def cell_core_backward(flat, lstm, tape, X, Hm, dh, dc):
    """src/cells.cpp:134-195. Returns dX, dHm, dh_skip / dc_prev and flat grads."""
    n_in, H = X.shape[1], Hm.shape[1]
    wx, uh, b = split_cell_params(flat, lstm, n_in, H)
    K = 4 if lstm else 3
    gw = [None] * K
    gu = [None] * K
    gb = [None] * K
    out = {"dX": np.zeros_like(X), "dHm": np.zeros_like(Hm)}
    if lstm:
        i, f, g, o = tape["gates"]
        tc = np.tanh(tape["c"])
        d_o = dh * tc
        dct = (1 - tc ** 2) * (dh * o)
        if dc is not None:
            dct = dct + dc
        d_i, d_g, d_f = dct * g, dct * i, dct * tape["c_prev"]
        out["dc_prev"] = dct * f
        dpres = [i * (1 - i) * d_i, f * (1 - f) * d_f, (1 - g ** 2) * d_g, o * (1 - o) * d_o]
        for k in range(4):
            gw[k] = X.T @ dpres[k]
            gb[k] = dpres[k].sum(0)
            out["dX"] += dpres[k] @ wx[k].T
            gu[k] = Hm.T @ dpres[k]
            out["dHm"] += dpres[k] @ uh[k].T
    else:
        r, z, n = tape["gates"]
        d_z = dh * (tape["h_skip"] - n)
        d_n = dh * (1 - z)
        out["dh_skip"] = dh * z
        dpre_n = (1 - n ** 2) * d_n
        d_hn = dpre_n * r
        dpre_r = r * (1 - r) * (dpre_n * tape["hn"])
        dpre_z = z * (1 - z) * d_z
        for k, dp in enumerate([dpre_r, dpre_z, dpre_n]):
            gw[k] = X.T @ dp
            gb[k] = dp.sum(0)
            out["dX"] += dp @ wx[k].T
        gu[0], gu[1], gu[2] = Hm.T @ dpre_r, Hm.T @ dpre_z, Hm.T @ d_hn
        out["dHm"] += dpre_r @ uh[0].T + dpre_z @ uh[1].T + d_hn @ uh[2].T
    out["dparams"] = np.concatenate([np.concatenate([gw[k].ravel(), gu[k].ravel(), gb[k].ravel()])
                                     for k in range(K)])
    return out


# ------------------------------------------------------------------ loss / optimiser
def loss_mae(pred, target):
    """src/nn.cpp:62-71: value = mean |d|, grad = sign(d)/n."""
    d = pred - target
    n = d.size
    return float(np.abs(d).sum() / n), np.sign(d) / n


def adam_step(p, g, m, v, step, lr=0.01, b1=0.9, b2=0.999, eps=1e-8, sgd=False):
    """src/train.cpp:26-52 (step = step count after increment)."""
    if sgd:
        return p - lr * g, m, v
    m = b1 * m + (1 - b1) * g
    v = b2 * v + (1 - b2) * g * g
    bc1 = 1 - b1 ** step
    bc2 = 1 - b2 ** step
    return p - lr * (m / bc1) / (np.sqrt(v / bc2) + eps), m, v


# ------------------------------------------------------------------ large-graph helpers
# The scale parity tests (1M nodes / 20M edges) need the same restatement at
# sizes where per-edge Python loops and np.add.at are too slow; these are the
# same operations in vectorised form (sum / transposed sum only).
def apply_structural_delta(prev_keys, del_src, del_dst, ins_src, ins_dst):
    """apply_delta's edge part (src/snapshot.cpp:142-154) on sorted unique
    (src<<32|dst) keys: (prev \\ deletions) U insertions."""
    dk = np.unique(edge_keys(del_src, del_dst))
    ik = np.unique(edge_keys(ins_src, ins_dst))
    if len(dk):
        pos = np.searchsorted(prev_keys, dk)
        ok = pos < len(prev_keys)
        ok[ok] = prev_keys[pos[ok]] == dk[ok]
        prev_keys = np.delete(prev_keys, pos[ok])
    if len(ik):
        pos = np.searchsorted(prev_keys, ik)
        present = pos < len(prev_keys)
        present[present] = prev_keys[pos[present]] == ik[present]
        prev_keys = np.insert(prev_keys, pos[~present], ik[~present])
    return prev_keys


def in_csr_from_keys(keys, n):
    """In-CSR (sources ascending per destination) of sorted (src,dst) keys."""
    s, d = split_keys(keys)
    rk = np.sort((d.astype(np.int64) << 32) | s.astype(np.int64))
    in_src = (rk & 0xFFFFFFFF).astype(np.int32)
    in_ptr = np.zeros(n + 1, np.int64)
    in_ptr[1:] = np.cumsum(np.bincount((rk >> 32).astype(np.int64), minlength=n))
    return in_ptr, in_src


def out_csr_from_keys(keys, n):
    s, d = split_keys(keys)
    out_ptr = np.zeros(n + 1, np.int64)
    out_ptr[1:] = np.cumsum(np.bincount(s.astype(np.int64), minlength=n))
    return out_ptr, d


def sum_aggregate_sparse(in_ptr, in_src, feats):
    """aggregate_scratch, sum (src/aggregate.cpp:75-81), as a sparse product
    in fp64 (summation order differs from the per-row loop by fp64 rounding)."""
    import scipy.sparse as sp
    n = len(in_ptr) - 1
    A = sp.csr_matrix((np.ones(len(in_src)), in_src, in_ptr), shape=(n, feats.shape[0]))
    return A @ np.asarray(feats, np.float64)


def sum_backward_sparse(in_ptr, in_src, upstream):
    """aggregate_backward, sum (src/aggregate.cpp:221-226): grad = A^T up."""
    import scipy.sparse as sp
    n = len(in_ptr) - 1
    A = sp.csr_matrix((np.ones(len(in_src)), in_src, in_ptr), shape=(n, upstream.shape[0]))
    return A.T @ np.asarray(upstream, np.float64)
