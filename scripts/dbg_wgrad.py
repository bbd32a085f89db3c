import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import refbind as ref
from oracle import dgnn_oracle as O
from paper_2501_15348_b200 import api

def nrel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))

for lstm, n_in, n in ((False, 128, 4099), (True, 64, 20000), (False, 64, 1000)):
    H = 64
    rng = np.random.default_rng(1)
    flat = ref.cell_init(0 if lstm else 1, n_in, H, 9)
    X = rng.uniform(-2, 2, (n, n_in)).astype(np.float32)
    Hm = rng.uniform(-2, 2, (n, H)).astype(np.float32)
    hs = rng.uniform(-1, 1, (n, H)).astype(np.float32)
    cp = rng.uniform(-1, 1, (n, H)).astype(np.float32) if lstm else None
    dh = rng.standard_normal((n, H)).astype(np.float32)
    dc = rng.standard_normal((n, H)).astype(np.float32) if lstm else None
    T = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()
    fwd = api.cell_forward(lstm, T(X), T(Hm), T(hs), T(cp), T(flat))
    bwd = api.cell_backward(lstm, T(X), T(Hm), fwd, T(hs), T(cp), T(dh), T(dc))
    torch.cuda.synchronize()
    f64 = lambda a: None if a is None else a.astype(np.float64)
    tape = O.cell_core_forward(flat, lstm, f64(X), f64(Hm), f64(hs), f64(cp))
    want = O.cell_core_backward(flat, lstm, tape, f64(X), f64(Hm), f64(dh), f64(dc))
    got, w = bwd["dflat"].cpu().numpy(), want["dparams"]
    K = 4 if lstm else 3
    per = n_in * H + H * H + H
    parts = {"wx": [], "uh": [], "b": []}
    for g in range(K):
        o = g * per
        parts["wx"].append(slice(o, o + n_in * H)); parts["uh"].append(slice(o + n_in * H, o + per - H)); parts["b"].append(slice(o + per - H, o + per))
    print(os.environ.get("DGNN_WGRAD_MN", "1"), lstm, n_in, n, "dflat nrel", nrel(got, w),
          {k: round(nrel(np.concatenate([got[s] for s in v]), np.concatenate([w[s] for s in v])), 8) for k, v in parts.items()},
          "got head", got[:3], "want head", w[:3], flush=True)
