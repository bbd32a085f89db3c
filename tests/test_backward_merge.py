"""The backward's cross-step merge of transposed SpMMs (layer l's
dHm(t) goes through A_{t-1}^T together with layer l+1's dX(t-1), plus the
structural correction Delta_t^T) against the unmerged backward and the
reference: same gradients within fp32 summation-order noise, fewer
transposed-SpMM launches. Each variant runs in its own process (the switch
is read once per process)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu

PROG = r"""
import json, sys
sys.path.insert(0, sys.argv[1])
import numpy as np, torch
from paper_2501_15348_b200 import api
arch, hidden = sys.argv[2], int(sys.argv[3])
g = api.Synth(400, 6.0, 32, 14, 0.05, 0.05, seed=3).to_graph()
s = api.TrainSession(g, api.TrainConfig(arch=arch, hidden=hidden))
api.prof_reset(); api.prof_enable(True)
out = []
for w in (0, 3):
    loss, pred, grads = s.sample_grads(w)
    out.append({"loss": loss, "grads": grads.tolist()})
torch.cuda.synchronize()
api.prof_enable(False)
p = api.prof_get()
print(json.dumps({"samples": out, "k3": p["agg_backward"]["launches"], "corr": p["agg_rebase"]["launches"]}))
"""


def run(arch, hidden, merge):
    env = dict(os.environ, DGNN_BACKWARD_MERGE="1" if merge else "0")
    r = subprocess.run([sys.executable, "-c", PROG, ROOT, arch, str(hidden)], capture_output=True, text=True,
                       env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("arch,hidden", [("tgcn", 64), ("gcrn_m2", 64), ("tgcn", 16)])
def test_backward_merge_matches_unmerged_and_reference(ref, arch, hidden):
    on, off = run(arch, hidden, True), run(arch, hidden, False)
    assert on["k3"] < off["k3"], (on["k3"], off["k3"])
    g_ref = ref.RefGraph.synth(400, 6.0, 32, 14, 0.05, 0.05, seed=3)
    for w, a, b in zip((0, 3), on["samples"], off["samples"]):
        ga, gb = np.asarray(a["grads"]), np.asarray(b["grads"])
        assert a["loss"] == b["loss"]  # the forward is untouched
        assert np.linalg.norm(ga - gb) / np.linalg.norm(gb) < 1e-5
        _, _, gr = g_ref.sample_grads(ref.RunCfg(arch=arch, hidden=hidden), w)
        assert np.linalg.norm(ga - gr) / np.linalg.norm(gr) < 1e-4
