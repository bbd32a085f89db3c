import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import refbind as ref
from paper_2501_15348_b200 import api

def nrel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))

n, deg, dim, T, edge, feat = 1500, 20.0, 128, 64, 0.02, 0.02
g_ref = ref.RefGraph.synth(n, deg, dim, T, edge, feat, seed=1)
g = api.Synth(n, deg, dim, T, edge, feat, seed=1).to_graph()
kw = dict(arch="tgcn", hidden=64)
H = 64
blocks = []
off = 0
for part in ("enc", "dec"):
    for l, fin in ((1, dim), (2, H)):
        for gte in range(3):
            for nm, sz in (("wx", fin * H), ("uh", H * H), ("b", H)):
                blocks.append((f"{part}{l}/{nm}{gte}", off, off + sz)); off += sz
blocks.append(("head/w", off, off + H * dim)); off += H * dim
blocks.append(("head/b", off, off + dim)); off += dim
s2 = api.TrainSession(g, api.TrainConfig(**kw))
assert off == s2.num_params, (off, s2.num_params)
tag = " ".join(f"{k}={os.environ[k]}" for k in os.environ if k.startswith("DGNN_"))
for w in (0, 5):
    lr_, pr, gr = g_ref.sample_grads(ref.RunCfg(**kw), w)
    l2, p2, g2 = s2.sample_grads(w)
    print(tag, "w", w, "pred nrel", nrel(p2, pr), "grad nrel", nrel(g2, gr), flush=True)
    worst = sorted(((nrel(g2[a:b], gr[a:b]), name, float(np.linalg.norm(gr[a:b]))) for name, a, b in blocks), reverse=True)[:6]
    for e, name, nm in worst:
        print(f"    {name:14s} nrel {e:.2e}  |g| {nm:.3e}")
