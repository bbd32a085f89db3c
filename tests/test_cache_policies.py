"""Cache-policy baselines and iteration orders: REINC, LRU and
LFU (src/cache.cpp:104-114) under seq-first and node-first epochs
(src/train.cpp:209-220), several node batches and a capacity small enough to
evict — same losses, aggregation invocation log, cache event trace and
statistics as the compiled reference."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GRAPH = dict(n=300, avg_degree=4, dim=8, T=12, edge=0.05, feat=0.02)


@pytest.fixture(scope="module")
def pair(ref):
    import torch
    assert torch.cuda.is_available()
    from paper_2501_15348_b200 import api
    g = GRAPH
    args = (g["n"], g["avg_degree"], g["dim"], g["T"], g["edge"], g["feat"])
    return api, ref.RefGraph.synth(*args, seed=5), api.Synth(*args, seed=5).to_graph()


def nrel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


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


@pytest.mark.parametrize("cache", ["reinc", "lru", "lfu"])
@pytest.mark.parametrize("iteration", ["seq_first", "node_first"])
def test_policy_and_order_match_reference(pair, ref, cache, iteration):
    api, gr, g = pair
    # SGD: 48 optimizer steps of Adam turn fp32-vs-fp64 noise into ~1e-3 loss
    # drift (DESIGN §3 tolerances); the cache decisions are the point here
    kw = dict(arch="gcrn_m2", hidden=16, seq_len=3, batch_size=120, cache=cache, cache_frac=0.3,
              iteration=iteration, optimizer="sgd")
    r = gr.run(ref.RunCfg(epochs=2, **kw))
    s = api.TrainSession(g, api.TrainConfig(record_events=True, **kw))
    losses = np.concatenate([s.run_epoch()["sample_losses"] for _ in range(2)])
    assert losses.shape == r.losses.shape
    assert nrel(losses, r.losses) < 1e-4
    assert np.array_equal(s.invocations(), r.invocations[:, 1:])
    _events_match(s.cache_events(), r.events)
    st = s.stats()
    keys = ["hits", "misses", "evictions", "expirations", "invalidations", "rejected",
            "scratch_calls", "incremental_calls", "fallbacks"]
    assert [st[k] for k in keys] == r.stats[0, :9].tolist()


CAPS = [0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9, 1.0]


def cache_curves(api, g, **kw):
    """cache-bench: per policy and capacity, one seq-first epoch
    of GCRN-M2 (D=2, L=8, S=1, teacher forcing) on the device; rows of
    policy, capacity_frac, hits, misses, hit_rate, evictions, expirations."""
    rows = []
    for pol in ("reinc", "lru", "lfu"):
        for cap in CAPS:
            s = api.TrainSession(g, api.TrainConfig(arch="gcrn_m2", hidden=8, cache=pol, cache_frac=cap,
                                                    **kw))
            s.run_epoch()
            st = s.stats()
            look = st["hits"] + st["misses"]
            rows.append((pol, cap, st["hits"], st["misses"], st["hits"] / look if look else 0.0,
                         st["evictions"], st["expirations"]))
    return rows


def test_cache_curves_match_reference_and_fig10(ref):
    """Fig. 10 hit-rate curves on the device: every (policy, capacity) point's
    counters equal the reference's, and the SPEC acceptance bands hold
    (SPEC.md:634): ReInc at 10% 52 +- 10 points, LRU 0 +- 2; LRU plateau
    78 +- 10 over 20-80%; ReInc 100% at <= 70%; ReInc >= LRU >= LFU."""
    import torch
    assert torch.cuda.is_available()
    from paper_2501_15348_b200 import api
    args = (200, 4, 8, 24, 0.05, 0.02)
    g = api.Synth(*args, seed=1).to_graph()
    gr = ref.RefGraph.synth(*args, seed=1)
    rows = cache_curves(api, g)
    for pol, cap, hits, misses, rate, ev, ex in rows:
        r = gr.run(ref.RunCfg(arch="gcrn_m2", hidden=8, cache=pol, cache_frac=cap, record_events=False))
        st = r.stats[0]
        assert (hits, misses, ev, ex) == (st[0], st[1], st[2], st[3]), (pol, cap)
    rate = {(p, c): r for p, c, _, _, r, _, _ in rows}
    assert abs(rate["reinc", 0.1] - 0.52) <= 0.10
    assert rate["lru", 0.1] <= 0.02
    assert all(abs(rate["lru", c] - 0.78) <= 0.10 for c in CAPS[1:8])
    assert min(c for c in CAPS if rate["reinc", c] == 1.0) <= 0.7
    for c in CAPS:
        assert rate["reinc", c] >= rate["lru", c] >= rate["lfu", c], c


def test_seq_first_beats_node_first(ref):
    """Fig. 11 / SPEC acceptance 9: >= 4 node batches at 30%
    capacity, seq-first hit rate strictly above node-first, both equal to
    the reference."""
    import torch
    assert torch.cuda.is_available()
    from paper_2501_15348_b200 import api
    args = (200, 4, 8, 24, 0.05, 0.02)
    g = api.Synth(*args, seed=1).to_graph()
    gr = ref.RefGraph.synth(*args, seed=1)
    rate = {}
    for it in ("seq_first", "node_first"):
        kw = dict(arch="gcrn_m2", hidden=8, cache="reinc", cache_frac=0.3, batch_size=50, iteration=it)
        s = api.TrainSession(g, api.TrainConfig(**kw))
        s.run_epoch()
        st = s.stats()
        r = gr.run(ref.RunCfg(record_events=False, **kw))
        assert (st["hits"], st["misses"]) == (r.stats[0][0], r.stats[0][1])
        rate[it] = st["hits"] / (st["hits"] + st["misses"])
    assert rate["seq_first"] > rate["node_first"]
