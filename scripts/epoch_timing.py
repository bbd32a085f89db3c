"""Per-epoch device time at a bench workload, with the per-class profiler on
and off (diagnoses run-to-run variance of the C3 bench line)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import WORKLOADS  # noqa: E402
from paper_2501_15348_b200 import api  # noqa: E402
from paper_2501_15348_b200.sharding import run_sharded_epoch  # noqa: E402

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 4
stream = torch.cuda.current_stream()
synth = api.Synth(wl["n"], wl["deg"], wl["dim"], wl["T"], wl["edge"], wl["feat"], seed=1)
graph = synth.to_graph(stream)
sess = api.TrainSession(graph, api.TrainConfig(arch=wl["arch"], hidden=wl["hidden"], workers=1), stream=stream)
grad = torch.empty(sess.num_params, device="cuda")
run_sharded_epoch(sess, grad)
torch.cuda.synchronize()
out = {}
for prof in (False, True, False):
    api.prof_reset()
    api.prof_enable(prof)
    ts = []
    for _ in range(epochs):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        h0 = time.perf_counter()
        e0.record(stream)
        run_sharded_epoch(sess, grad)
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append((round(e0.elapsed_time(e1), 1), round((time.perf_counter() - h0) * 1e3, 1)))
    api.prof_enable(False)
    p = api.prof_get()
    out[f"prof={prof}"] = {"epochs_ms_dev_wall": ts,
                           "kernel_ms": round(sum(v["ms"] for v in p.values()) / epochs, 1)}
    print(json.dumps(out[f"prof={prof}"]), flush=True)
print(json.dumps({"mem_gb": round(torch.cuda.mem_get_info()[1] / 1e9 - torch.cuda.mem_get_info()[0] / 1e9, 1)}))
