"""Second cache level (HBM <-> pinned host DRAM, the B200 addition under the
REINC cache of ref src/cache.cpp:133-200): with an HBM budget small enough to
force spills every window, training is bitwise identical to the unbudgeted
run, and the logical cache (events, statistics, invocation log) still equals
the reference's. Refills are issued ahead of the access (prefetch by the
seq-first next-use order) on the copy stream."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def nrel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _events_match(ev, ev_ref):
    ev_ref = ev_ref[:, 1:]
    assert ev.shape == ev_ref.shape
    i = 0
    while i < len(ev):
        if ev[i, 0] == 4:
            j = i
            while j < len(ev) and ev[j, 0] == 4:
                j += 1
            assert sorted(map(tuple, ev[i:j].tolist())) == sorted(map(tuple, ev_ref[i:j].tolist()))
            i = j
        else:
            assert np.array_equal(ev[i], ev_ref[i]), (i, ev[i], ev_ref[i])
            i += 1


@pytest.mark.parametrize("arch,aggr", [("tgcn", "sum"), ("gcrn_m2", "mean"), ("gcrn_m2", "max"),
                                       ("gcrn_m1", "sum")])
def test_spilling_cache_matches_reference(ref, arch, aggr):
    import torch
    assert torch.cuda.is_available()
    from paper_2501_15348_b200 import api
    args = (300, 4, 8, 14, 0.05, 0.05)
    g = api.Synth(*args, seed=7).to_graph()
    gr = ref.RefGraph.synth(*args, seed=7)
    kw = dict(arch=arch, hidden=16, aggr=aggr, cache_frac=1.0)
    r = gr.run(ref.RunCfg(epochs=2, record_events=True, **kw))
    one = 300 * 8 * 4 * (2 if aggr == "max" else 1) + (300 * 8 * 4 + 300 * 4 if aggr == "mean" else 0)

    def run(budget):
        s = api.TrainSession(g, api.TrainConfig(record_events=True, hbm_cache_budget_bytes=budget, **kw))
        losses = np.concatenate([s.run_epoch()["sample_losses"] for _ in range(2)])
        return s, losses

    s0, l0 = run(0)
    s1, l1 = run(2 * one)  # two input aggregations' worth of unborrowed HBM
    tier = s1.tier_stats()
    assert tier["spills"] > 0 and tier["refills"] > 0 and tier["prefetches"] > 0, tier
    assert np.array_equal(l0, l1)
    assert np.array_equal(s0.params(), s1.params())
    assert nrel(l1, r.losses) < 1e-4
    assert np.array_equal(s1.invocations(), r.invocations[:, 1:])
    _events_match(s1.cache_events(), r.events)
    keys = ["hits", "misses", "evictions", "expirations", "invalidations", "rejected",
            "scratch_calls", "incremental_calls", "fallbacks"]
    st = s1.stats()
    assert [st[k] for k in keys] == r.stats[0, :9].tolist()


def test_spill_backpressure_keeps_results(ref):
    """The in-flight spill cap (HbmTier backpressure): with it forced to 1 MB
    every spill waits for the previous ones' device -> host copies, and the
    run stays bitwise equal to the unbudgeted one (each variant in its own
    process: the cap is read when the tier is created)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    prog = r"""
import json, sys
sys.path.insert(0, sys.argv[1])
import numpy as np
from paper_2501_15348_b200 import api
g = api.Synth(300, 4, 8, 14, 0.05, 0.05, seed=7).to_graph()
budget = int(sys.argv[2])
s = api.TrainSession(g, api.TrainConfig(arch="tgcn", hidden=16, cache_frac=1.0, hbm_cache_budget_bytes=budget))
l = np.concatenate([s.run_epoch()["sample_losses"] for _ in range(2)])
print(json.dumps({"losses": l.tolist(), "params": s.params().tolist(), "tier": s.tier_stats()}))
"""
    def run(budget, cap_mb):
        env = dict(os.environ)
        if cap_mb:
            env["DGNN_TIER_INFLIGHT_MB"] = str(cap_mb)
        r = subprocess.run([sys.executable, "-c", prog, root, str(budget)], capture_output=True, text=True,
                           env=env, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        return json.loads(r.stdout.strip().splitlines()[-1])
    base = run(0, None)
    tight = run(2 * 300 * 8 * 4, 1)
    assert tight["tier"]["spills"] > 0 and tight["tier"]["refills"] > 0
    assert tight["losses"] == base["losses"]
    assert tight["params"] == base["params"]
