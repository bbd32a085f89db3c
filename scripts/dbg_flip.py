import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import refbind as ref
from paper_2501_15348_b200 import api
n, deg, dim, T, edge, feat = 1500, 20.0, 128, 64, 0.02, 0.02
g_ref = ref.RefGraph.synth(n, deg, dim, T, edge, feat, seed=1)
g = api.Synth(n, deg, dim, T, edge, feat, seed=1).to_graph()
kw = dict(arch="tgcn", hidden=64)
s = api.TrainSession(g, api.TrainConfig(**kw))
tag = os.environ.get("DGNN_UMMA_PARTS", "7")
for w in (0, 5, 30):
    lr_, pr, gr = g_ref.sample_grads(ref.RunCfg(**kw), w)
    l2, p2, g2 = s.sample_grads(w)
    tgt = g_ref.feats(w + 9)
    d_ref, d_ours = pr - tgt, p2.astype(np.float64) - tgt
    flips = int(np.sum(np.sign(d_ref) != np.sign(d_ours)))
    print(tag, "w", w, "flips", flips, "min|d|", float(np.abs(d_ref).min()),
          "pred max abs err", float(np.abs(d_ours - d_ref).max()),
          "grad nrel", float(np.linalg.norm(g2 - gr) / np.linalg.norm(gr)), flush=True)
