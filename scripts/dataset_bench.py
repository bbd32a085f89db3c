"""Dataset loading throughput: the reference's load_dataset
(oracle/_ref, 1 thread) against dgnn_dataset_load (host parse + HBM graph
store build, streaming) on the same on-disk dataset, text and binary.

  python scripts/dataset_bench.py [--n 10000] [--deg 10] [--dim 64] [--T 16]

Prints one JSON line. The dataset is generated with the bit-exact synth and
written by the reference's own save_dataset (text) and by dgnn_synth_save
(binary twin)."""
import argparse
import json
import os
import shutil
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2501_15348_b200 import api


def du(path):
    return sum(os.path.getsize(os.path.join(path, f)) for f in os.listdir(path))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10_000)
    ap.add_argument("--deg", type=float, default=10)
    ap.add_argument("--dim", type=int, default=64)
    ap.add_argument("--T", type=int, default=16)
    ap.add_argument("--edge", type=float, default=0.01)
    ap.add_argument("--feat", type=float, default=0.01)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    root = tempfile.mkdtemp(prefix="dgnn_ds_")
    out = {"config": vars(args)}
    try:
        s = api.Synth(args.n, args.deg, args.dim, args.T, args.edge, args.feat, seed=1)
        text, binary = os.path.join(root, "text"), os.path.join(root, "bin")
        s.save(binary, binary=True)
        from oracle import refbind
        if refbind.available():
            g = refbind.RefGraph.synth(args.n, args.deg, args.dim, args.T, args.edge, args.feat, seed=1)
            g.save_dataset(text)
            del g
            t0 = time.perf_counter()
            L = refbind.RefGraph.load_dataset(text)
            out["reference_text_load_s"] = time.perf_counter() - t0
            del L
        else:
            api.save_dataset(s.to_graph(), text)
        out["text_bytes"], out["binary_bytes"] = du(text), du(binary)
        torch.cuda.init()
        api.load_dataset(binary)  # warm-up (context, pool)
        torch.cuda.synchronize()
        for name, path in (("text", text), ("binary", binary)):
            ts = []
            for _ in range(args.reps):
                t0 = time.perf_counter()
                dg = api.load_dataset(path)
                torch.cuda.synchronize()
                ts.append(time.perf_counter() - t0)
                del dg
            out[f"b200_{name}_load_s"] = min(ts)
        # check: both loads give the generator's graph
        a, b = api.load_dataset(text), s.to_graph()
        ok = all(np.array_equal(x, y) for t in range(args.T) for x, y in zip(a.in_csr(t), b.in_csr(t)))
        out["text_load_matches_generator"] = bool(ok)
        if "reference_text_load_s" in out:
            out["speedup_text_vs_reference"] = out["reference_text_load_s"] / out["b200_text_load_s"]
        out["cores"] = os.cpu_count()
    finally:
        shutil.rmtree(root, ignore_errors=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
