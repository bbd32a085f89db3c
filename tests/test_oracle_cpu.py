"""CPU tests (no GPU): the numpy oracle pinned to the reference (golden
fixtures + the compiled reference when present), the product's host-side
logic (bit-exact synthetic generator, parameter init, plan / windows / cache
scores / key hash) and the C-ABI library exports."""
import os

import numpy as np
import pytest

from oracle import dgnn_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = np.load(os.path.join(HERE, "golden", "golden.npz"))
GT = 8  # snapshots in the golden graph


def gcsr(t):
    return {"keys": O.edge_keys(GOLD[f"edges_{t}"][:, 0], GOLD[f"edges_{t}"][:, 1]),
            "in_ptr": GOLD[f"in_ptr_{t}"], "in_src": GOLD[f"in_src_{t}"],
            "out_ptr": GOLD[f"out_ptr_{t}"], "out_dst": GOLD[f"out_dst_{t}"]}


# ------------------------------------------------------------------ oracle vs golden
def test_oracle_csr_matches_golden():
    n = GOLD["feats_0"].shape[0]
    for t in range(GT):
        e = GOLD[f"edges_{t}"]
        c = O.build_csr(e[:, 0], e[:, 1], n)
        for k in ("in_ptr", "in_src", "out_ptr", "out_dst"):
            assert np.array_equal(c[k], GOLD[f"{k}_{t}"]), (t, k)


def test_oracle_extract_delta_matches_golden():
    n = GOLD["feats_0"].shape[0]
    for t in range(1, GT):
        prev = O.build_csr(GOLD[f"edges_{t-1}"][:, 0], GOLD[f"edges_{t-1}"][:, 1], n)
        curr = O.build_csr(GOLD[f"edges_{t}"][:, 0], GOLD[f"edges_{t}"][:, 1], n)
        d = O.extract_delta(prev, curr, GOLD[f"feats_{t-1}"], GOLD[f"feats_{t}"])
        for k in ("del_src", "del_dst", "ins_src", "ins_dst", "changed", "changed_feats"):
            assert np.array_equal(d[k], GOLD[f"delta_{t}_{k}"]), (t, k)
        assert O.change_ratio(d, len(prev["keys"])) == float(GOLD[f"ratio_{t}"])
        keys, feats = O.apply_delta(prev["keys"], GOLD[f"feats_{t-1}"], d)
        assert np.array_equal(keys, curr["keys"]) and np.array_equal(feats, GOLD[f"feats_{t}"])


@pytest.mark.parametrize("kind", ["sum", "mean", "max", "min"])
def test_oracle_aggregations_match_golden(kind):
    t = 3
    c = gcsr(t)
    r = O.aggregate_scratch(c["in_ptr"], c["in_src"], GOLD[f"feats_{t}"], kind)
    assert np.array_equal(r["values"], GOLD[f"scratch_{kind}_values"])  # same order, fp64: exact
    if kind == "mean":
        assert np.array_equal(r["degree"], GOLD[f"scratch_{kind}_degree"])
    if kind in ("max", "min"):
        assert np.array_equal(r["argext"], GOLD[f"scratch_{kind}_argext"])
    g = O.aggregate_backward(c["in_ptr"], c["in_src"], GOLD[f"bwd_{kind}_up"], kind, r)
    assert np.allclose(g, GOLD[f"bwd_{kind}_grad"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("kind", ["sum", "mean", "max", "min"])
def test_oracle_incremental_chain_matches_golden(kind):
    """aggregate_incremental t=0..7 with rescratch period 4: fallback decisions
    (reason, depth) exact, values equal to fp64 rounding."""
    n = GOLD["feats_0"].shape[0]
    c0 = gcsr(0)
    cur = O.aggregate_scratch(c0["in_ptr"], c0["in_src"], GOLD["feats_0"], kind)
    depth, E = 0, len(c0["keys"])
    steps = GOLD[f"chain_{kind}_steps"]
    for t in range(1, GT):
        ct = gcsr(t)
        d = {k: GOLD[f"delta_{t}_{k}"] for k in ("del_src", "del_dst", "ins_src", "ins_dst", "changed")}
        cur, fb, why, depth = O.aggregate_incremental(cur, E, depth, ct, GOLD[f"feats_{t-1}"],
                                                      GOLD[f"feats_{t}"], d, kind, 0.5, 4)
        assert (int(fb), why, depth) == tuple(steps[t - 1]), t
        E = len(ct["keys"])
    assert np.allclose(cur["values"], GOLD[f"chain_{kind}_values"], rtol=1e-12, atol=1e-12)
    if kind in ("max", "min"):
        assert np.array_equal(cur["argext"], GOLD[f"chain_{kind}_argext"])
    assert n == cur["values"].shape[0]


@pytest.mark.parametrize("name,lstm", [("lstm", True), ("gru", False)])
def test_oracle_cells_match_golden(name, lstm):
    g = lambda k: GOLD[f"cell_{name}_{k}"]
    cp = g("cprev") if lstm else None
    tape = O.cell_core_forward(g("params"), lstm, g("X"), g("Hm"), g("hskip"), cp)
    for i, gate in enumerate(tape["gates"]):
        assert np.allclose(gate, g("out_gates")[i], rtol=1e-12, atol=1e-13)
    assert np.allclose(tape["h"], g("out_h"), rtol=1e-12, atol=1e-13)
    bw = O.cell_core_backward(g("params"), lstm, tape, g("X"), g("Hm"), g("dh"), g("dc") if lstm else None)
    for k in ("dX", "dHm", "dparams"):
        assert np.allclose(bw[k], g(f"out_{k}"), rtol=1e-10, atol=1e-12), k


def test_oracle_kats_from_spec():
    # SPEC.md:86-88 sliding windows
    assert O.sliding_windows(10, 8, 1, 1) == [0, 1]
    assert O.sliding_windows(8, 8, 1, 0) == [0]
    assert O.sliding_windows(20, 4, 2, 2) == [0, 2, 4, 6, 8, 10, 12, 14]
    # SPEC.md:514 plan T=12, M=4 -> blocks of 3
    p = O.plan_consecutive_block(12, 4, 1, 1, 0)
    assert p[:, 0].tolist() == [0, 3, 6, 9] and p[:, 1].tolist() == [3, 6, 9, 12]
    # SPEC.md:78 change ratio 20+20 over 500 edges
    d = {"del_src": np.zeros(20), "ins_src": np.zeros(20)}
    assert O.change_ratio(d, 500) == pytest.approx(0.04)
    # SPEC.md:163-164 star graph: 3 sources into node 0, features [1,1]
    ip = np.array([0, 3, 3, 3, 3])
    src = np.array([1, 2, 3])
    f = np.ones((4, 2))
    assert O.aggregate_scratch(ip, src, f, "sum")["values"][0].tolist() == [3, 3]
    m = O.aggregate_scratch(ip, src, f, "mean")
    assert m["values"][0].tolist() == [1, 1] and m["degree"][0] == 3
    # SPEC.md:181-182 backward star, all-ones upstream
    up = np.zeros((4, 2)); up[0] = 1
    assert O.aggregate_backward(ip, src, up, "sum")[1].tolist() == [1, 1]
    assert np.allclose(O.aggregate_backward(ip, src, up, "mean", m)[1], [1 / 3, 1 / 3])
    # SPEC.md:463 SGD p=1, g=2, lr 0.1
    p2, _, _ = O.adam_step(np.array([1.0]), np.array([2.0]), 0, 0, 1, lr=0.1, sgd=True)
    assert p2[0] == pytest.approx(0.8)
    # SPEC.md:384-385 MAE
    v, gr = O.loss_mae(np.array([[1.0, 2.0]]), np.array([[0.0, 4.0]]))
    assert v == pytest.approx(1.5) and gr.tolist() == [[0.5, -0.5]]
    # SPEC.md:253-255 imminence: local 0, encoder L-S, decoder L-1
    assert O.imminence(8, 1, 0, 2, 1) == 0
    assert O.imminence(8, 1, 0, 1, 0) == 7 and O.imminence(8, 2, 0, 1, 0) == 6
    assert O.imminence(8, 1, 1, 1, 0) == 7
    # reference's visit-counting F (16 and 26, not the SPEC's 24 / 5)
    assert O.future_access_count(2, 4, 4, 8, 1, 4, 0, 1, 1, 100, 0) == 16
    assert O.future_access_count(2, 3, 1, 8, 1, 0, 1, 1, 1, 100, 0) == 26


# ------------------------------------------------------------------ oracle vs live reference
def test_oracle_matches_compiled_reference_random(ref):
    rng = np.random.default_rng(0)
    for seed in range(3):
        g = ref.RefGraph.synth(120, 4, 6, 6, 0.08, 0.05, seed=seed + 11)
        n = g.n
        csr = [O.build_csr(*g.edges(t), n) for t in range(g.T)]
        for t in range(1, g.T):
            d = O.extract_delta(csr[t - 1], csr[t], g.feats(t - 1), g.feats(t))
            r = g.delta(t)
            for k in ("del_src", "del_dst", "ins_src", "ins_dst", "changed"):
                assert np.array_equal(d[k], r[k])
        for kind in ("sum", "mean", "max", "min"):
            feats = rng.standard_normal((n, 5))
            r = g.agg_scratch(2, kind, feats)
            o = O.aggregate_scratch(csr[2]["in_ptr"], csr[2]["in_src"], feats, kind)
            assert np.array_equal(o["values"], r["values"])
            up = rng.standard_normal((n, 5))
            assert np.allclose(O.aggregate_backward(csr[2]["in_ptr"], csr[2]["in_src"], up, kind, o),
                               g.agg_backward(2, kind, feats, up), atol=1e-12)


def test_cache_scores_and_hash_match_reference(ref):
    from paper_2501_15348_b200 import _lib
    import ctypes as C
    L = _lib.lib()
    for layers in (1, 2):
        for gates in (1, 3, 4):
            for gate in range(1, gates + 1):
                for S in (1, 2):
                    for idx in range(0, 9):
                        for part in (0, 1):
                            for wrem in (0, 3, 50):
                                for kind in (0, 1):
                                    ctx = [layers, gates, gate, 8, S, idx, part, 1, 1, 1, wrem, kind]
                                    f_r, i_r = ref.cache_scores(*ctx)
                                    f_o = O.future_access_count(layers, gates, gate, 8, S, idx, part, 1, 1, wrem, kind)
                                    i_o = O.imminence(8, S, part, 1, kind)
                                    arr = np.array(ctx, np.int32)
                                    f_p, i_p = C.c_int32(), C.c_int32()
                                    _lib.check(L.dgnn_cache_scores(arr.ctypes.data_as(C.c_void_p), C.byref(f_p), C.byref(i_p)))
                                    assert (f_r, i_r) == (f_o, i_o) == (f_p.value, i_p.value), ctx
    for key in [(0, 0, 5, 0, 0, 0), (1, 2, 7, 1, 3, 99), (1, 1, 31, 2, 0, 123456789)]:
        assert ref.key_hash(*key) == O.key_hash(*key) == L.dgnn_key_hash(*key)


# ------------------------------------------------------------------ product host logic (no GPU)
def test_product_synth_is_bit_exact_with_golden():
    from paper_2501_15348_b200 import api
    s = api.Synth(60, 3, 4, GT, 0.1, 0.05, seed=7)
    src, dst, feats = s.base()
    assert np.array_equal(np.stack([src, dst], 1), GOLD["edges_0"])
    assert np.array_equal(feats, GOLD["feats_0"].astype(np.float32))
    keys = O.edge_keys(src, dst)
    f = GOLD["feats_0"]
    for t in range(1, GT):
        st = s.step(t)
        delta = {"del_src": st["del_src"], "del_dst": st["del_dst"], "ins_src": st["ins_src"],
                 "ins_dst": st["ins_dst"], "changed": st["changed"],
                 "changed_feats": GOLD[f"feats_{t}"][st["changed"]]}
        keys, f = O.apply_delta(keys, f, delta)
        e = GOLD[f"edges_{t}"]
        assert np.array_equal(keys, O.edge_keys(e[:, 0], e[:, 1])), t
        assert np.array_equal(st["changed_feats"], GOLD[f"feats_{t}"][st["changed"]].astype(np.float32))
        assert np.array_equal(f, GOLD[f"feats_{t}"])


@pytest.mark.parametrize("n,deg,dim,T,er,fr,seed", [
    (500, 6, 3, 6, 0.03, 0.0, 1), (257, 2.5, 5, 5, 0.2, 1.0, 4),
    # edge pools of 60000 / 60005 keys: many prefetched shuffle blocks, even and odd n
    (12000, 5, 2, 4, 0.05, 0.01, 2), (12001, 5, 2, 3, 0.05, 0.01, 3)])
def test_product_synth_matches_reference(ref, n, deg, dim, T, er, fr, seed):
    from paper_2501_15348_b200 import api
    s = api.Synth(n, deg, dim, T, er, fr, seed=seed)
    g = ref.RefGraph.synth(n, deg, dim, T, er, fr, seed=seed)
    src, dst, feats = s.base()
    rs, rd = g.edges(0)
    assert np.array_equal(src, rs) and np.array_equal(dst, rd)
    keys = O.edge_keys(src, dst)
    for t in range(1, T):
        st = s.step(t)
        keys = np.union1d(np.setdiff1d(keys, O.edge_keys(st["del_src"], st["del_dst"])),
                          O.edge_keys(st["ins_src"], st["ins_dst"]))
        assert np.array_equal(keys, O.edge_keys(*g.edges(t)))
        rf = g.feats(t)
        assert np.array_equal(st["changed_feats"], rf[st["changed"]].astype(np.float32))


@pytest.mark.parametrize("arch", ["gcrn_m2", "tgcn", "gcrn_m1", "cd_gcn"])
def test_product_param_init_bit_exact(arch):
    import ctypes as C
    from paper_2501_15348_b200 import _lib, api
    cfg = api.TrainConfig(arch=arch, hidden=8, seq_len=3).to_c()
    n = _lib.lib().dgnn_init_params(C.byref(cfg), 4, None)
    out = np.empty(n, np.float64)
    _lib.lib().dgnn_init_params(C.byref(cfg), 4, out.ctypes.data_as(C.c_void_p))
    assert np.array_equal(out, GOLD[f"sample_{arch}_params0"])


def test_product_windows_and_plan():
    import ctypes as C
    from paper_2501_15348_b200 import _lib, api
    L = _lib.lib()
    buf = np.empty(64, np.int32)
    for total, l, s, h in [(31, 8, 1, 1), (10, 8, 1, 1), (8, 8, 1, 0), (20, 4, 2, 2), (3, 8, 1, 1)]:
        n = L.dgnn_sliding_windows(total, l, s, h, buf.ctypes.data_as(C.c_void_p), 64)
        assert buf[:n].tolist() == O.sliding_windows(total, l, s, h) == api.sliding_windows(total, l, s, h)
    assert np.array_equal(GOLD["kat_windows"], np.array(O.sliding_windows(31, 8, 1, 1)))
    for total, m in [(64, 8), (64, 3), (12, 4), (31, 2), (40, 7)]:
        out = np.empty((m, 4), np.int64)
        _lib.check(L.dgnn_plan(total, m, 8, 1, 1, out.ctypes.data_as(C.c_void_p)))
        assert np.array_equal(out, O.plan_consecutive_block(total, m, 8, 1, 1))
        assert np.array_equal(out, np.array(api.plan(total, m, 8, 1, 1)))
    assert np.array_equal(GOLD["kat_plan_55_8"], O.plan_consecutive_block(64, 8, 8, 1, 1))
    with pytest.raises(ValueError):
        _lib.check(L.dgnn_plan(3, 4, 8, 1, 1, np.empty(16, np.int64).ctypes.data_as(C.c_void_p)))


def test_cabi_exports_every_header_symbol():
    from paper_2501_15348_b200 import _lib
    L = _lib.lib()
    syms = _lib.header_symbols()
    assert len(syms) >= 50
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)


def test_product_raises_reference_errors_without_gpu():
    from paper_2501_15348_b200 import api
    with pytest.raises(ValueError, match="synthesize: avg_degree must be >= 1"):
        api.Synth(10, 0.5, 2, 3, 0.1, 0.0)
    with pytest.raises(ValueError, match="sliding_windows: L must be >= 1"):
        api.sliding_windows(10, 0, 1, 1)


def test_large_graph_helpers_match_restatement():
    """The vectorised helpers the scale tests use (apply_structural_delta,
    in/out CSR from keys, sparse sum / transposed sum) equal the per-edge
    restatement (build_csr, apply_delta, aggregate_scratch, aggregate_backward)."""
    rng = np.random.default_rng(21)
    n = 400
    keys = np.unique(O.edge_keys(rng.integers(0, n, 3000), rng.integers(0, n, 3000)))
    feats = rng.uniform(-1, 1, (n, 6))
    for _ in range(5):
        dk = rng.choice(keys, 200, replace=False)
        ik = np.setdiff1d(np.unique(O.edge_keys(rng.integers(0, n, 300), rng.integers(0, n, 300))), keys)
        ds, dd = O.split_keys(dk)
        is_, id_ = O.split_keys(ik)
        want, _ = O.apply_delta(keys, feats, {"del_src": ds, "del_dst": dd, "ins_src": is_,
                                              "ins_dst": id_, "changed": np.zeros(0, np.int64),
                                              "changed_feats": np.zeros((0, 6))})
        keys = O.apply_structural_delta(keys, ds, dd, is_, id_)
        assert np.array_equal(keys, want)
    s, d = O.split_keys(keys)
    csr = O.build_csr(s, d, n)
    ip, isrc = O.in_csr_from_keys(keys, n)
    assert np.array_equal(ip, csr["in_ptr"]) and np.array_equal(isrc, csr["in_src"])
    op, od = O.out_csr_from_keys(keys, n)
    assert np.array_equal(op, csr["out_ptr"]) and np.array_equal(od, csr["out_dst"])
    agg = O.aggregate_scratch(ip, isrc, feats, "sum")["values"]
    assert np.allclose(O.sum_aggregate_sparse(ip, isrc, feats), agg, rtol=1e-12, atol=1e-12)
    up = rng.standard_normal((n, 6))
    assert np.allclose(O.sum_backward_sparse(ip, isrc, up), O.aggregate_backward(ip, isrc, up, "sum"),
                       rtol=1e-12, atol=1e-12)
