"""Sampled k-hop computational graphs: the reference's khop +
to_view (oracle/_ref, 1 thread) against the device sampler on the same
snapshot, seeds, fanouts and sample seed; results checked bitwise.

  python scripts/khop_bench.py [--n 200000] [--deg 20] [--seeds 10000] [--fanouts 25,10]

Prints one JSON line (times are per khop + to_view call; device side timed
with CUDA events around the C-ABI call, which includes its host syncs)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2501_15348_b200 import api


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=200_000)
    ap.add_argument("--deg", type=float, default=20)
    ap.add_argument("--seeds", type=int, default=10_000)
    ap.add_argument("--fanouts", default="25,10")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    fan = [int(x) for x in args.fanouts.split(",")]
    seeds = np.arange(args.seeds, dtype=np.int32)
    g = api.Synth(args.n, args.deg, 4, 2, 0.02, 0.0, seed=1).to_graph()
    out = {"config": {"nodes": args.n, "avg_degree": args.deg, "edges": g.num_edges(0),
                      "seeds": args.seeds, "fanouts": fan}}
    c = api.ComputationalGraph.khop(g, 0, seeds, fan, 7)  # warm-up
    c.view()
    ts = []
    for _ in range(args.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        c = api.ComputationalGraph.khop(g, 0, seeds, fan, 7)
        ip = C_view(c)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    out["b200_khop_view_ms"] = 1e3 * min(ts)
    hops = c.hops()
    out["sampled_edges"] = [int(len(h["src"])) for h in hops]
    out["destinations"] = [int(len(h["dests"])) for h in hops]
    from oracle import refbind
    if refbind.available():
        gr = refbind.RefGraph.synth(args.n, args.deg, 4, 2, 0.02, 0.0, seed=1)
        rts = []
        for _ in range(2):
            t0 = time.perf_counter()
            cr = refbind.RefCompGraph.khop(gr, 0, seeds, fan, 7)
            cr.view()
            rts.append(time.perf_counter() - t0)
        out["reference_khop_view_ms"] = 1e3 * min(rts)
        rh = cr.hops()
        out["bitwise_equal"] = all(np.array_equal(a[k], b[k]) for a, b in zip(hops, rh)
                                   for k in ("dests", "src", "dst"))
        out["speedup"] = out["reference_khop_view_ms"] / out["b200_khop_view_ms"]
        out["reference_cores"] = 1
    print(json.dumps(out))


def C_view(c):
    # to_view on the device (in- and out-CSR); no host copy
    import ctypes as C
    from paper_2501_15348_b200._lib import check, lib
    ptrs = [C.c_void_p() for _ in range(4)]
    ne = C.c_int64()
    check(lib().dgnn_cg_view(c.h, *[C.byref(p) for p in ptrs], C.byref(ne)))
    return ptrs


if __name__ == "__main__":
    main()
