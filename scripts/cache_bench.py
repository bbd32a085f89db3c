"""cache-bench (the paper's Fig. 10 / Fig. 11) on the device:
hit rate per (policy, capacity fraction) for seq-first epochs, plus
seq-first vs node-first at 30% capacity with 4 node batches; each point's
counters checked against the compiled reference when oracle/_ref is present.
Writes CSV to stdout.  usage: python scripts/cache_bench.py > profiles/r2_cache_hit_curves.csv"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

from paper_2501_15348_b200 import api  # noqa: E402
from test_cache_policies import cache_curves  # noqa: E402


def main():
    torch.cuda.set_device(0)
    args = (200, 4, 8, 24, 0.05, 0.02)
    g = api.Synth(*args, seed=1).to_graph()
    ref = None
    try:
        from oracle import refbind
        if refbind.available():
            ref = refbind.RefGraph.synth(*args, seed=1)
    except Exception:
        ref = None
    print("figure,policy,iteration,capacity_frac,hits,misses,hit_rate,evictions,expirations,matches_reference")
    for pol, cap, hits, misses, rate, ev, ex in cache_curves(api, g):
        same = ""
        if ref is not None:
            from oracle import refbind
            st = ref.run(refbind.RunCfg(arch="gcrn_m2", hidden=8, cache=pol, cache_frac=cap, record_events=False)).stats[0]
            same = str((hits, misses, ev, ex) == (st[0], st[1], st[2], st[3]))
        print(f"fig10,{pol},seq_first,{cap},{hits},{misses},{rate:.4f},{ev},{ex},{same}")
    for it in ("seq_first", "node_first"):
        kw = dict(arch="gcrn_m2", hidden=8, cache="reinc", cache_frac=0.3, batch_size=50, iteration=it)
        s = api.TrainSession(g, api.TrainConfig(**kw))
        s.run_epoch()
        st = s.stats()
        look = st["hits"] + st["misses"]
        print(f"fig11,reinc,{it},0.3,{st['hits']},{st['misses']},{st['hits'] / look:.4f},{st['evictions']},"
              f"{st['expirations']},")


if __name__ == "__main__":
    main()
