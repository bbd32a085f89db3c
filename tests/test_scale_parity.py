"""Parity at the BASELINE configs' scale (GPU).

* C1 (configs[0]) full epoch against the compiled reference: losses,
  parameters, invocation log, cache trace and statistics.
* A down-scaled C4 epoch (tgcn, d=128, h=64, T=64, structure + feature churn:
  fp32 incremental chains down to depth 63, the reference's rescratch bound)
  against the reference.
* A 1M-node / 20M-edge / d=128 graph (C3's shape with C4's feature churn):
  device CSR bitwise, scratch, a 31-step incremental chain and the transposed
  SpMM against the numpy oracle (oracle/dgnn_oracle.py, whose CSR and scratch
  aggregation are pinned bit-exactly to the reference in test_oracle_cpu.py).
* A 50K-node depth-63 incremental chain against the reference's own
  aggregate_incremental chain.
* Cell forward / backward at 1M+ rows (about 54 row tiles per persistent CTA,
  so the TMEM / mbarrier phases wrap many times) against the oracle.
* SPEC acceptance criterion 1: >= 500 random (snapshot, delta)
  cases per aggregation function, graphs <= 1000 nodes, change ratios 1-32%:
  incremental == scratch within 1e-5 (bitwise for max / min without
  fallback), and both equal to the reference's aggregate_scratch.
"""
import numpy as np
import pytest

from oracle import dgnn_oracle as O

pytestmark = pytest.mark.gpu


def nrel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    fa, fb = np.isfinite(a), np.isfinite(b)
    if not np.array_equal(fa, fb) or not np.array_equal(a[~fa], b[~fb]):
        return float("inf")
    a, b = a[fa], b[fb]
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.fixture(scope="module")
def api():
    import torch
    assert torch.cuda.is_available()
    from paper_2501_15348_b200 import api as A
    return A


def _events_match(ev, ev_ref):
    ev_ref = ev_ref[:, 1:]
    assert ev.shape == ev_ref.shape
    i = 0
    while i < len(ev):
        if ev[i, 0] == 4:  # invalidation burst: hash-map order in the reference
            j = i
            while j < len(ev) and ev[j, 0] == 4:
                j += 1
            assert sorted(map(tuple, ev[i:j].tolist())) == sorted(map(tuple, ev_ref[i:j].tolist()))
            i = j
        else:
            assert np.array_equal(ev[i], ev_ref[i]), (i, ev[i], ev_ref[i])
            i += 1


STAT_KEYS = ["hits", "misses", "evictions", "expirations", "invalidations", "rejected",
             "scratch_calls", "incremental_calls", "fallbacks"]


def _epoch_vs_reference(ref, api, graph, cfg_kw, epochs=1, trajectory=True):
    """trajectory=False: the configuration trains chaotically (C4's d=128
    aggregated features: even the FFMA path's 2e-5 gradient noise, amplified
    by the optimizer steps, moves the per-sample losses by 1% within a few
    samples, measured), so only the first sample's loss is compared and the
    numerics are pinned per sample at fixed parameters instead
    (_sample_grads_vs_reference)."""
    n, deg, dim, T, edge, feat = graph
    g_ref = ref.RefGraph.synth(n, deg, dim, T, edge, feat, seed=1)
    r = g_ref.run(ref.RunCfg(epochs=epochs, record_events=True, **cfg_kw))
    g = api.Synth(n, deg, dim, T, edge, feat, seed=1).to_graph()
    s = api.TrainSession(g, api.TrainConfig(record_events=True, **cfg_kw))
    assert np.array_equal(s.initial_params(), g_ref.init_params(ref.RunCfg(**cfg_kw)))
    losses = np.concatenate([s.run_epoch()["sample_losses"] for _ in range(epochs)])
    assert losses.shape == r.losses.shape
    assert abs(losses[0] - r.losses[0]) <= 1e-5 * abs(r.losses[0])
    if trajectory:
        # per-sample losses: fp32 vs fp64 through Adam steps
        assert nrel(losses, r.losses) < 1e-4, nrel(losses, r.losses)
        assert np.max(np.abs(losses - r.losses) / np.abs(r.losses)) < 1e-3
        assert nrel(s.params(), r.params) < 1e-3
    assert np.array_equal(s.invocations(), r.invocations[:, 1:])
    _events_match(s.cache_events(), r.events)
    st = s.stats()
    assert [st[k] for k in STAT_KEYS] == r.stats[0, :9].tolist()
    return s, r


def test_c1_full_epoch_matches_reference(ref, api):
    """configs[0] exactly: stacked GCN+LSTM (gcrn_m1), 10K
    nodes, 100K edges, 16 snapshots, 1% churn, d = h = 64, 7 windows."""
    s, r = _epoch_vs_reference(ref, api, (10_000, 10.0, 64, 16, 0.01, 0.01),
                               dict(arch="gcrn_m1", hidden=64))
    assert len(r.losses) == 7


def test_c4_downscaled_epoch_matches_reference(ref, api):
    """C4's model and dynamics on 1,500 nodes: tgcn (GRU), d=128, h=64, T=64
    (55 windows), 2% structural + 2% feature churn. The input aggregation chain
    runs incrementally from t=0 to t=62 (the last window's last step) inside
    the epoch."""
    s, r = _epoch_vs_reference(ref, api, (1_500, 20.0, 128, 64, 0.02, 0.02),
                               dict(arch="tgcn", hidden=64), trajectory=False)
    assert len(r.losses) == 55
    inv = s.invocations()
    # (layer, t, kind, incremental): the layer-1 input chain reaches t = 63 incrementally
    inc = inv[(inv[:, 0] == 1) & (inv[:, 2] == 0) & (inv[:, 3] == 1)]
    assert inc[:, 1].max() == 62  # the last window (start 54) ends at t = 62


def test_c4_downscaled_sample_grads(ref, api):
    """Per-sample numerics on the C4-downscaled graph at fixed parameters
    (losses, predictions, gradients; windows across the whole epoch). MAE's
    gradient is sign(pred - target) / n, discontinuous at 0: a target within
    the fp32 prediction error of the prediction can flip one entry's sign,
    which moves the parameter gradient by ~4e-4 (measured), so samples with a
    flipped entry are reported and compared at the looser bound."""
    n, deg, dim, T, edge, feat = 1_500, 20.0, 128, 64, 0.02, 0.02
    g_ref = ref.RefGraph.synth(n, deg, dim, T, edge, feat, seed=1)
    g = api.Synth(n, deg, dim, T, edge, feat, seed=1).to_graph()
    kw = dict(arch="tgcn", hidden=64)
    s = api.TrainSession(g, api.TrainConfig(**kw))
    for w in (0, 5, 18, 30, 42, 54):
        loss_r, pred_r, grads_r = g_ref.sample_grads(ref.RunCfg(**kw), w)
        loss, pred, grads = s.sample_grads(w)
        target = g_ref.feats(w + 9)
        flips = int(np.sum(np.sign(pred_r - target) != np.sign(pred.astype(np.float64) - target)))
        assert abs(loss - loss_r) <= 1e-5 * abs(loss_r), (w, loss, loss_r)
        assert nrel(pred, pred_r) < 1e-5, w
        assert nrel(grads, grads_r) < (1e-4 if flips == 0 else 1e-3), (w, flips, nrel(grads, grads_r))


def test_depth63_chain_50k_matches_reference(ref, api):
    """aggregate_incremental chained t=0..63 (depth 63, no fallback) on a
    50K-node, d=128 graph with structure + feature churn, sum and mean,
    against the reference's own chain (ref src/aggregate.cpp:117-207)."""
    import torch
    n, deg, d, T = 50_000, 20.0, 128, 64
    g_ref = ref.RefGraph.synth(n, deg, d, T, 0.02, 0.02, seed=2)
    g = api.Synth(n, deg, d, T, 0.02, 0.02, seed=2).to_graph()
    for kind in ("sum", "mean"):
        r = g_ref.agg_chain(0, T - 1, kind, threshold=0.5, rescratch=64)
        cur = api.aggregate_scratch(g, 0, g.feats_tensor(0), kind)
        depth = 0
        for t in range(1, T):
            nxt = api.aggregate_incremental(g, t, cur, kind, prev_depth=depth)
            assert (int(nxt["used_fallback"]), nxt["reason"], nxt["depth"]) == tuple(r["steps"][t - 1])
            cur, depth = nxt, nxt["depth"]
        torch.cuda.synchronize()
        assert depth == 63
        assert nrel(cur["values"].cpu().numpy(), r["values"]) < 1e-5, kind
        if kind == "mean":
            assert np.array_equal(cur["degree"].cpu().numpy(), r["degree"].astype(np.float32))


@pytest.fixture(scope="module")
def million(api):
    """1M nodes, 20M edges, d=128, T=32, 2% structural + 2% feature churn; the
    oracle's view of snapshot 31 built from the generator's host arrays."""
    n, deg, d, T = 1_000_000, 20.0, 128, 32
    syn = api.Synth(n, deg, d, T, 0.02, 0.02, seed=3)
    g = syn.to_graph()
    src, dst, F = syn.base()
    keys = np.sort(O.edge_keys(src, dst))
    F = F.astype(np.float64)
    for t in range(1, T):
        st = syn.step(t)
        keys = O.apply_structural_delta(keys, st["del_src"], st["del_dst"], st["ins_src"], st["ins_dst"])
        F[st["changed"]] = st["changed_feats"]
    return syn, g, keys, F, n, T


def test_1m_csr_bitwise(million):
    syn, g, keys, F, n, T = million
    ip, isrc = O.in_csr_from_keys(keys, n)
    p, s = g.in_csr(T - 1)
    assert np.array_equal(ip, p) and np.array_equal(isrc, s)
    op, od = O.out_csr_from_keys(keys, n)
    p, d = g.out_csr(T - 1)
    assert np.array_equal(op, p) and np.array_equal(od, d)
    assert np.array_equal(g.feats(T - 1), F.astype(np.float32))


def test_1m_scratch_chain_and_transposed(million, api):
    """SURVEY §7 minimum slice at 1M nodes: scratch at t=0, 31 incremental
    steps (depth 31, the graph's own deltas with feature churn: folded
    compact-block entries included), scratch at t=31 and the transposed SpMM
    (w=64) at t=31."""
    import torch
    syn, g, keys, F, n, T = million
    ip, isrc = O.in_csr_from_keys(keys, n)
    want = O.sum_aggregate_sparse(ip, isrc, F)
    scratch = api.aggregate_scratch(g, T - 1, g.feats_tensor(T - 1), "sum")
    torch.cuda.synchronize()
    assert nrel(scratch["values"].cpu().numpy(), want) < 1e-6
    del scratch
    cur = api.aggregate_scratch(g, 0, g.feats_tensor(0), "sum")
    depth = 0
    for t in range(1, T):
        nxt = api.aggregate_incremental(g, t, cur, "sum", prev_depth=depth)
        assert not nxt["used_fallback"] and nxt["depth"] == depth + 1, t
        cur, depth = nxt, nxt["depth"]
    torch.cuda.synchronize()
    assert nrel(cur["values"].cpu().numpy(), want) < 1e-5
    del cur
    rng = np.random.default_rng(5)
    up = rng.standard_normal((n, 64)).astype(np.float32)
    got = api.aggregate_backward(g, T - 1, torch.from_numpy(up).cuda(), "sum")
    torch.cuda.synchronize()
    assert nrel(got.cpu().numpy(), O.sum_backward_sparse(ip, isrc, up)) < 1e-5


@pytest.mark.parametrize("lstm,n_in", [(True, 128), (False, 128), (False, 64)])
def test_cell_million_rows(ref, api, lstm, n_in):
    """tcgen05 cell forward + fused backward at 1,000,037 rows (ragged last
    tile) against the fp64 oracle: ~54 tiles per persistent CTA."""
    import torch
    n, H = 1_000_037, 64
    rng = np.random.default_rng(13)
    flat = ref.cell_init(0 if lstm else 1, n_in, H, 9)
    X = rng.uniform(-2, 2, (n, n_in)).astype(np.float32)
    Hm = rng.uniform(-2, 2, (n, H)).astype(np.float32)
    hs = rng.uniform(-1, 1, (n, H)).astype(np.float32)
    cp = rng.uniform(-1, 1, (n, H)).astype(np.float32) if lstm else None
    dh = rng.standard_normal((n, H)).astype(np.float32)
    dc = rng.standard_normal((n, H)).astype(np.float32) if lstm else None
    T = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()
    fwd = api.cell_forward(lstm, T(X), T(Hm), T(hs), T(cp), T(flat))
    bwd = api.cell_backward(lstm, T(X), T(Hm), fwd, T(hs), T(cp), T(dh), T(dc))
    torch.cuda.synchronize()
    f64 = lambda a: None if a is None else a.astype(np.float64)
    tape = O.cell_core_forward(flat, lstm, f64(X), f64(Hm), f64(hs), f64(cp))
    want = O.cell_core_backward(flat, lstm, tape, f64(X), f64(Hm), f64(dh), f64(dc))
    assert nrel(fwd["h"].cpu().numpy(), tape["h"]) < 1e-5
    if lstm:
        assert nrel(fwd["c"].cpu().numpy(), tape["c"]) < 1e-5
        assert nrel(bwd["dc_prev"].cpu().numpy(), want["dc_prev"]) < 1e-5
    else:
        assert nrel(bwd["dh_skip"].cpu().numpy(), want["dh_skip"]) < 1e-5
    assert nrel(bwd["dX"].cpu().numpy(), want["dX"]) < 1e-5
    assert nrel(bwd["dHm"].cpu().numpy(), want["dHm"]) < 1e-5
    # parameter gradients: a sum over 10^6 rows (DESIGN §3 tolerance 1e-4)
    assert nrel(bwd["dflat"].cpu().numpy(), want["dparams"]) < 1e-4


@pytest.mark.parametrize("kind", ["sum", "mean", "max", "min"])
def test_incremental_equals_scratch_500_cases(ref, api, kind):
    """SPEC acceptance 1 on the device: 25 random graphs x 20
    deltas = 500 (snapshot, delta) cases per aggregation function, 20-1000
    nodes, change ratios 1-32% (edge churn drawn per graph, feature churn up
    to 10%)."""
    import torch
    rng = np.random.default_rng({"sum": 1, "mean": 2, "max": 3, "min": 4}[kind])
    cases = exact = fell_back = 0
    for gi in range(25):
        n = int(rng.integers(20, 1001))
        deg = float(rng.uniform(2, 12))
        dim = int(rng.choice([4, 8, 12, 16, 32]))
        edge = float(rng.uniform(0.01, 0.32))
        feat = float(rng.uniform(0.0, 0.10))
        T = 21
        g_ref = ref.RefGraph.synth(n, deg, dim, T, edge, feat, seed=100 + gi)
        g = api.Synth(n, deg, dim, T, edge, feat, seed=100 + gi).to_graph()
        for t in range(1, T):
            prev = api.aggregate_scratch(g, t - 1, g.feats_tensor(t - 1), kind)
            inc = api.aggregate_incremental(g, t, prev, kind, prev_depth=0)
            scr = api.aggregate_scratch(g, t, g.feats_tensor(t), kind)
            want = g_ref.agg_scratch(t, kind, g_ref.feats(t))
            torch.cuda.synchronize()
            ratio = g_ref.change_ratio(t)
            assert g.change_ratio(t) == ratio
            assert inc["used_fallback"] == (ratio > 0.5 or inc["reason"] == 2)
            iv, sv = inc["values"].cpu().numpy(), scr["values"].cpu().numpy()
            assert nrel(iv, want["values"]) < 1e-5, (gi, t)
            assert nrel(sv, want["values"]) < 1e-6, (gi, t)
            if kind in ("max", "min"):
                ia, sa = inc["argext"].cpu().numpy(), scr["argext"].cpu().numpy()
                assert np.array_equal(sa, want["argext"])
                if not inc["used_fallback"]:
                    # exact: the same fp32 maxima, the same contributors
                    assert np.array_equal(iv, sv) and np.array_equal(ia, sa), (gi, t)
                    exact += 1
            if kind == "mean":
                assert np.array_equal(inc["degree"].cpu().numpy(), want["degree"].astype(np.float32))
            fell_back += inc["used_fallback"]
            cases += 1
    assert cases >= 500
    # max / min: with deletions and feature churn nearly every case hits a
    # deleted contributor and falls back (src/aggregate.cpp:150-166); the
    # exact no-fallback path is pinned by test_extremal_insert_only_exact


@pytest.mark.parametrize("kind", ["max", "min"])
def test_extremal_insert_only_exact(api, kind):
    """Insert-only deltas never invalidate a recorded extremum, so max / min
    incremental updates take no fallback and must equal scratch bitwise —
    values and contributor ids (ties: the reference's first-seen source)."""
    import torch
    rng = np.random.default_rng(11 if kind == "max" else 12)
    checked = 0
    for gi in range(12):
        n = int(rng.integers(50, 800))
        dim = int(rng.choice([4, 8, 16, 32]))
        m = int(n * rng.uniform(2, 8))
        pairs = np.unique(rng.integers(0, n, (m, 2)), axis=0)
        pairs = pairs[pairs[:, 0] != pairs[:, 1]]
        rng.shuffle(pairs)
        k0 = len(pairs) * 3 // 4
        g = api.DynamicGraph(n, dim)
        feats = rng.uniform(-1, 1, (n, dim)).astype(np.float32)
        g.add_snapshot(pairs[:k0], feats)
        cuts = np.sort(rng.choice(np.arange(k0, len(pairs)), 4, replace=False))
        prev_cut = k0
        for t, cut in enumerate(cuts, start=1):
            g.add_delta(np.zeros((0, 2), np.int32), pairs[prev_cut:cut])
            prev_cut = cut
            prev = api.aggregate_scratch(g, t - 1, g.feats_tensor(t - 1), kind)
            inc = api.aggregate_incremental(g, t, prev, kind, prev_depth=0, fallback_threshold=10.0)
            scr = api.aggregate_scratch(g, t, g.feats_tensor(t), kind)
            torch.cuda.synchronize()
            assert not inc["used_fallback"]
            assert torch.equal(inc["values"], scr["values"]), (gi, t)
            assert torch.equal(inc["argext"], scr["argext"]), (gi, t)
            checked += 1
    assert checked == 48
