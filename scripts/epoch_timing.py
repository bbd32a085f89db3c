"""Per-epoch device time at a bench workload, with per-epoch kernel-time sums
(profiler on) and SM clocks sampled during each epoch — diagnoses run-to-run
variance of the bench line (GPU idle vs slower kernels vs clock dips)."""
import contextlib
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import WORKLOADS, ClockSampler  # noqa: E402
from paper_2501_15348_b200 import api  # noqa: E402
from paper_2501_15348_b200.sharding import run_sharded_epoch  # noqa: E402

class NullClk:
    def summary(self):
        return {"sm_mhz": None, "reasons": []}


wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 4
stream = torch.cuda.current_stream()
synth = api.Synth(wl["n"], wl["deg"], wl["dim"], wl["T"], wl["edge"], wl["feat"], seed=1)
graph = synth.to_graph(stream)
sess = api.TrainSession(graph, api.TrainConfig(arch=wl["arch"], hidden=wl["hidden"], workers=1), stream=stream)
grad = torch.empty(sess.num_params, device="cuda")
run_sharded_epoch(sess, grad)
torch.cuda.synchronize()
api.prof_enable(True)
rows = []
for _ in range(epochs):
    api.prof_reset()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    with (ClockSampler(0) if not os.environ.get("NO_CLOCKS") else contextlib.nullcontext(NullClk())) as clk:
        h0 = time.perf_counter()
        e0.record(stream)
        run_sharded_epoch(sess, grad)
        e1.record(stream)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - h0) * 1e3
    p = api.prof_get()
    sc = api.prof_get(scopes=True)
    smp, host = sc["sample"], sc["sample_host"]
    c = clk.summary()
    rows.append({"dev_ms": round(e0.elapsed_time(e1), 1), "wall_ms": round(wall, 1),
                 "kernel_ms": round(sum(v["ms"] for v in p.values()), 1),
                 "by_class": {k: round(v["ms"], 1) for k, v in p.items()},
                 "samples": smp["launches"], "sample_ms_sum": round(smp["ms"], 1),
                 "sample_ms_max": round(smp["max_ms"], 1),
                 "host_ms_sum": round(host["ms"], 1), "host_ms_max": round(host["max_ms"], 1),
                 "host_max_at": int(host["flops"]),
                 "phase_max": {k: (round(sc[k]["max_ms"], 1), int(sc[k]["flops"]))
                               for k in ("host_build", "host_fwd", "host_bwd", "host_alloc")},
                 "alloc_ms_sum": round(sc["host_alloc"]["ms"], 1),
                 "allocs": sc["host_alloc"]["launches"],
                 "sm_mhz": c["sm_mhz"], "reasons": c["reasons"]})
    print(json.dumps(rows[-1]), flush=True)
api.prof_enable(False)
print(json.dumps({"dev_ms_median": statistics.median(r["dev_ms"] for r in rows),
                  "mem": api.mem_stats()}))
