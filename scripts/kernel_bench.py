"""Per-kernel timing at C3 shapes (1M nodes, 20M edges, d=128, h=64) through the
C ABI, CUDA events on the launching stream. Used for ncu captures:
  python scripts/kernel_bench.py [--only NAME] [--iters K]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2501_15348_b200 import api


def timeit(fn, iters):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def prof_time(fn, iters, res):
    from torch.profiler import ProfilerActivity, profile
    fn()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(iters):
            fn()
        torch.cuda.synchronize()
    tot = 0.0
    for ev in prof.key_averages():
        if ev.device_type.name == "CUDA" and ev.count > 0:
            us = ev.device_time_total / ev.count if hasattr(ev, "device_time_total") else ev.cuda_time_total / ev.count
            res.setdefault("kernels", {})[ev.key[:60]] = {"launches": ev.count, "mean_us": round(us, 1)}
            tot += us * ev.count
    return tot / iters / 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--d", type=int, default=128)
    ap.add_argument("--prof", action="store_true", help="per-kernel mean device times (torch.profiler / CUPTI)")
    args = ap.parse_args()
    n, d, H = args.n, args.d, 64
    global timeit
    if args.prof:
        timeit = lambda fn, iters: prof_time(fn, iters, res)
    res = {}
    torch.manual_seed(0)
    want = lambda k: not args.only or k in args.only.split(",")
    if any(want(k) for k in ("agg_scratch128", "agg_scratch64", "agg_delta", "agg_backward64")):
        s = api.Synth(n, 20, d, 2, 0.02, 0.0, seed=1)
        g = s.to_graph()
        E = g.num_edges(1)
        f0, f1 = g.feats_tensor(0), g.feats_tensor(1)
        h = torch.randn(n, H, device="cuda")
        if want("agg_scratch128"):
            ms = timeit(lambda: api.aggregate_scratch(g, 1, f1, "sum"), args.iters)
            res["agg_scratch128"] = {"ms": ms, "GBps_alg": (8 * (n + 1) + 4 * E + 4 * d * E + 4 * d * n) / ms / 1e6}
        if want("agg_scratch64"):
            ms = timeit(lambda: api.aggregate_scratch(g, 1, h, "sum"), args.iters)
            res["agg_scratch64"] = {"ms": ms, "GBps_alg": (8 * (n + 1) + 4 * E + 4 * H * E + 4 * H * n) / ms / 1e6}
        if want("agg_backward64"):
            ms = timeit(lambda: api.aggregate_backward(g, 1, h, "sum"), args.iters)
            res["agg_backward64"] = {"ms": ms, "GBps_alg": (8 * (n + 1) + 4 * E + 4 * H * E + 4 * H * n) / ms / 1e6}
        if want("agg_delta"):
            agg = api.aggregate_scratch(g, 0, f0, "sum")
            sz = g.delta_sizes(1)
            nent = sz["n_del"] + sz["n_ins"]
            ms = timeit(lambda: api.aggregate_delta_inplace(g, 1, agg, f0, f1, "sum"), args.iters)
            alg = 8 * nent + 4 * d * (sz["u_minus"] + sz["u_plus"]) + 8 * d * sz["n_rows"]
            res["agg_delta"] = {"ms": ms, "GBps_alg": alg / ms / 1e6, "entries": nent, **sz}
    if want("agg_delta_feat"):
        # C4-like delta: 2% structural churn + 2% feature-changed nodes (out-edge expansion)
        s = api.Synth(n, 20, d, 2, 0.02, 0.02, seed=1)
        g = s.to_graph()
        agg = api.aggregate_scratch(g, 0, g.feats_tensor(0), "sum")
        sz = g.delta_sizes(1)
        nent = sz["n_del"] + sz["n_ins"]
        ms = timeit(lambda: api.apply_graph_delta(g, 1, agg, "sum"), args.iters)
        alg = 8 * nent + 4 * d * (sz["u_minus"] + sz["u_plus"]) + 8 * d * sz["n_rows"]
        res["agg_delta_feat"] = {"ms": ms, "GBps_alg": alg / ms / 1e6, "alg_bytes": alg, **sz}
    for lstm in (True, False):
        name = "cell_fwd_lstm" if lstm else "cell_fwd_gru"
        if not want(name) and not want("cell_bwd") and not want("wgrad") and not want("cell_bwd_gru"):
            continue
        X = torch.randn(n, d, device="cuda")
        Hm = torch.randn(n, H, device="cuda")
        hs = torch.randn(n, H, device="cuda")
        cp = torch.randn(n, H, device="cuda") if lstm else None
        K = 4 if lstm else 3
        flat = torch.randn(K * (d * H + H * H + H), device="cuda") * 0.1
        if want(name):
            ms = timeit(lambda: api.cell_forward(lstm, X, Hm, hs, cp, flat), args.iters)
            byts = 4 * n * (d + H + 4 * H + H + (2 * H if lstm else H))
            res[name] = {"ms": ms, "GBps_alg": byts / ms / 1e6, "TFLOPs": 2 * n * (d + H) * 4 * H / ms / 1e9}
        if want("cell_bwd") or want("wgrad") or (not lstm and want("cell_bwd_gru")):
            if not lstm and not want("cell_bwd_gru"):
                continue
            fwd = api.cell_forward(lstm, X, Hm, hs, cp, flat)
            dh, dc = torch.randn(n, H, device="cuda"), torch.randn(n, H, device="cuda")
            ms = timeit(lambda: api.cell_backward(lstm, X, Hm, fwd, hs, cp, dh, dc), args.iters)
            res["cell_bwd_total" if lstm else "cell_bwd_gru_total"] = {"ms": ms, "TFLOPs": 2 * 2 * n * (d + H) * 4 * H / ms / 1e9}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
