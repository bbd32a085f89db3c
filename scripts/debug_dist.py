"""Debug: per-epoch gradient parity of the sharded trainer vs the reference (SGD)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import refbind as R
from paper_2501_15348_b200 import api


def nrel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


arch = sys.argv[1] if len(sys.argv) > 1 else "tgcn"
lr = 0.1
g_ref = R.RefGraph.synth(300, 4, 8, 12, 0.05, 0.02, seed=1)
g = api.Synth(300, 4, 8, 12, 0.05, 0.02, seed=1).to_graph()
ps = []
for e in (1, 2, 3):
    ps.append(g_ref.run(R.RunCfg(arch=arch, hidden=16, workers=1, epochs=e, optimizer="sgd", lr=lr)))
p0 = ps[0].params0
refp = [p0] + [r.params for r in ps]
s = api.TrainSession(g, api.TrainConfig(arch=arch, hidden=16, workers=1, optimizer="sgd", lr=lr))
W = s.windows()[0]
names = []
P = s.num_params
buf = torch.empty(P, device="cuda")
for e in range(3):
    mine_p = s.params()
    print(f"epoch {e}: params nrel vs ref {nrel(mine_p, refp[e]):.3e}")
    # fresh-cache gradient at the current params: sum of sample grads / W
    fresh = sum(s.sample_grads(w)[2] for w in range(W)) / W
    s.begin_epoch()
    s.local_grads(0, buf)
    dist_g = buf.cpu().numpy() / W
    s.apply(buf)
    s.end_epoch()
    ref_g = (refp[e] - refp[e + 1]) / lr
    print(f"  dist grad vs ref {nrel(dist_g, ref_g):.3e}; fresh vs ref {nrel(fresh, ref_g):.3e}; "
          f"dist vs fresh {nrel(dist_g, fresh):.3e}")
    bad = np.argsort(-np.abs(dist_g - ref_g))[:5]
    print("  worst idx", bad.tolist(), (dist_g - ref_g)[bad].tolist(), ref_g[bad].tolist())
