"""Quick device probe: build graph at a config, run sharded epochs, per-class kernel times."""
import json, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2501_15348_b200 import api

cfgs = {
    "c1": dict(n=10000, deg=10, dim=64, T=16, edge=0.01, feat=0.01, arch="gcrn_m1", hidden=64),
    "c2": dict(n=207, deg=1515/207, dim=2, T=2000, edge=0.0, feat=1.0, arch="gcrn_m2", hidden=64),
    "c3": dict(n=1_000_000, deg=20, dim=128, T=32, edge=0.02, feat=0.0, arch="gcrn_m2", hidden=64),
    "c4": dict(n=4_000_000, deg=20, dim=128, T=64, edge=0.02, feat=0.02, arch="tgcn", hidden=64),
}
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 2
c = cfgs[name]
t0 = time.time()
s = api.Synth(c["n"], c["deg"], c["dim"], c["T"], c["edge"], c["feat"], seed=1)
t1 = time.time()
torch.cuda.synchronize()
g = s.to_graph()
torch.cuda.synchronize()
t2 = time.time()
print(f"synth {t1-t0:.1f}s graph build {t2-t1:.1f}s", flush=True)
sess = api.TrainSession(g, api.TrainConfig(arch=c["arch"], hidden=c["hidden"], workers=1))
for e in range(epochs):
    api.prof_enable(e == epochs - 1)
    api.prof_reset()
    torch.cuda.synchronize()
    ta = time.time()
    losses = sess.run_sharded_epoch()
    torch.cuda.synchronize()
    tb = time.time()
    W = len(losses)
    print(f"epoch {e}: {tb-ta:.2f}s wall, {W} windows, loss {losses.mean():.5f}, "
          f"snapshots/s {W*9/(tb-ta):.1f}, free {torch.cuda.mem_get_info()[0]/1e9:.1f}GB", flush=True)
prof = api.prof_get()
tot = sum(v["ms"] for v in prof.values())
for k, v in prof.items():
    if v["launches"]:
        gbs = v["bytes"] / (v["ms"] / 1e3) / 1e9 if v["ms"] else 0
        tf = v["flops"] / (v["ms"] / 1e3) / 1e12 if v["ms"] else 0
        print(f"  {k:13s} n={v['launches']:6d} {v['ms']:9.1f} ms ({100*v['ms']/tot:4.1f}%) {gbs:8.1f} GB/s {tf:6.2f} TF/s")
print(json.dumps(sess.stats()))
