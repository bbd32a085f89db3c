"""Same-graph CPU reference timing for the configs the reference cannot run a
whole epoch of (C3: ~43 GB of materialised fp64 snapshots for 32 snapshots;
C4: ~348 GB): the compiled reference (oracle/_ref, 1 thread) runs its
seq-first / distsim epoch on the workload's exact graph (N, E, d, h, churn)
truncated to T = L + H + 1 = 10 snapshots, i.e. the first window of the
epoch at full size — no scaling in N. snapshots/s = windows x (L + H) /
EpochReport.seconds (ref src/train.cpp:151, :203-204).
usage: python scripts/reference_window.py c3 > profiles/r2_reference_window_c3.json"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import WORKLOADS, host_cpu, L, H  # noqa: E402
from oracle import refbind as R  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    wl = WORKLOADS[name]
    T = L + H + 1  # sliding_windows(T - 1, L, S, H): exactly one window
    t0 = time.time()
    g = R.RefGraph.synth(wl["n"], wl["deg"], wl["dim"], T, wl["edge"], wl["feat"], seed=1)
    t_synth = time.time() - t0
    r = g.run(R.RunCfg(arch=wl["arch"], hidden=wl["hidden"], workers=1, record_events=False))
    rate = len(r.losses) * (L + H) / r.seconds
    print(json.dumps({"impl": "reference", "workload": name, "desc": wl["desc"], "snapshots": T,
                      "windows": len(r.losses), "epoch_seconds": r.seconds, "snapshots_per_s": rate,
                      "synth_seconds": round(t_synth, 1), "cores": 1, "sample_losses": list(r.losses),
                      "note": "full-size graph (N, E, d, h, churn of the workload), first T = L+H+1 "
                              "snapshots: the epoch's first window, timed by the reference's own clock",
                      **host_cpu()}))


if __name__ == "__main__":
    main()
