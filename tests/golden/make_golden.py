"""Generates the golden fixtures in tests/golden/ from the compiled CPU
reference (oracle/_ref/libdgnn_ref.so, built from /root/reference/proj/src by
oracle/Makefile). Run in the build container: `python tests/golden/make_golden.py`.

Fixtures are small (tens of KB) so they travel with the repo and let the CPU
tests pin the numpy oracle, and smoke() check the device path, on machines
without /root/reference.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import refbind as R  # noqa: E402

GRAPH = dict(n=60, avg_degree=3, dim=4, T=8, edge=0.1, feat=0.05, seed=7)


def graph_fixture(out):
    g = R.RefGraph.synth(GRAPH["n"], GRAPH["avg_degree"], GRAPH["dim"], GRAPH["T"], GRAPH["edge"],
                         GRAPH["feat"], seed=GRAPH["seed"])
    for t in range(g.T):
        s, d = g.edges(t)
        out[f"edges_{t}"] = np.stack([s, d], 1)
        out[f"feats_{t}"] = g.feats(t)
        ip, isrc = g.in_csr(t)
        out[f"in_ptr_{t}"], out[f"in_src_{t}"] = ip, isrc
        op, od = g.out_csr(t)
        out[f"out_ptr_{t}"], out[f"out_dst_{t}"] = op, od
        if t:
            dl = g.delta(t)
            for k, v in dl.items():
                out[f"delta_{t}_{k}"] = v
            out[f"ratio_{t}"] = np.float64(g.change_ratio(t))
    rng = np.random.default_rng(3)
    for kind in ("sum", "mean", "max", "min"):
        t = 3
        r = g.agg_scratch(t, kind, g.feats(t))
        for k, v in r.items():
            out[f"scratch_{kind}_{k}"] = v
        c = g.agg_chain(0, 7, kind, threshold=0.5, rescratch=4)
        for k, v in c.items():
            out[f"chain_{kind}_{k}"] = v
        up = rng.standard_normal((g.n, g.dim))
        out[f"bwd_{kind}_up"] = up
        out[f"bwd_{kind}_grad"] = g.agg_backward(t, kind, g.feats(t), up)
    for arch in ("gcrn_m2", "tgcn", "gcrn_m1", "cd_gcn"):
        cfg = R.RunCfg(arch=arch, hidden=8, seq_len=3, horizon=1)
        loss, pred, grads = g.sample_grads(cfg, 0)
        out[f"sample_{arch}_loss"] = np.float64(loss)
        out[f"sample_{arch}_grads"] = grads
        out[f"sample_{arch}_params0"] = g.init_params(cfg)
        run = g.run(R.RunCfg(arch=arch, hidden=8, seq_len=3, horizon=1, epochs=2))
        out[f"epoch_{arch}_losses"] = run.losses
        out[f"epoch_{arch}_params"] = run.params
        out[f"epoch_{arch}_invocations"] = run.invocations
        out[f"epoch_{arch}_stats"] = run.stats
    return g


def cell_fixture(out):
    rng = np.random.default_rng(5)
    n, n_in, H = 20, 4, 8
    for kind, name in ((0, "lstm"), (1, "gru")):
        p = R.cell_init(kind, n_in, H, 9)
        X = rng.uniform(-2, 2, (n, n_in))
        Hm = rng.uniform(-2, 2, (n, H))
        hs = rng.uniform(-1, 1, (n, H))
        cp = rng.uniform(-1, 1, (n, H)) if kind == 0 else None
        dh = rng.standard_normal((n, H))
        dc = rng.standard_normal((n, H)) if kind == 0 else None
        r = R.cell_fwd_bwd(kind, n_in, H, p, X, Hm, hs, cp, dh, dc)
        out[f"cell_{name}_params"], out[f"cell_{name}_X"], out[f"cell_{name}_Hm"] = p, X, Hm
        out[f"cell_{name}_hskip"], out[f"cell_{name}_dh"] = hs, dh
        if kind == 0:
            out[f"cell_{name}_cprev"], out[f"cell_{name}_dc"] = cp, dc
        for k, v in r.items():
            out[f"cell_{name}_out_{k}"] = v


def smoke_fixture():
    # the exact case __graft_entry__.smoke() runs
    g = R.RefGraph.synth(300, 4, 32, 12, 0.05, 0.02, seed=1)
    loss, pred0, grads = g.sample_grads(R.RunCfg(arch="gcrn_m2", hidden=64), 0)
    np.savez_compressed(os.path.join(HERE, "smoke_gcrn_m2.npz"), loss=np.float64(loss), pred0=pred0,
                        grads=grads)


def main():
    R.lib()
    out = {}
    graph_fixture(out)
    cell_fixture(out)
    out["kat_windows"] = R.sliding_windows(31, 8, 1, 1)
    out["kat_plan_55_8"] = R.plan(55 + 9, 8, 8, 1, 1)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    smoke_fixture()
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
