"""Phase timing of the device graph build at C4 (DGNN_BUILD_PROF=1 makes
DeviceGraph print per-phase host wall time, each phase synchronised)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("DGNN_BUILD_PROF", "1")

import torch  # noqa: E402

from bench import WORKLOADS  # noqa: E402
from paper_2501_15348_b200 import api  # noqa: E402

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
t0 = time.time()
s = api.Synth(wl["n"], wl["deg"], wl["dim"], wl["T"], wl["edge"], wl["feat"], seed=1)
print(f"synth {time.time() - t0:.1f} s", file=sys.stderr, flush=True)
for i in range(2):
    t0 = time.time()
    g = s.to_graph()
    torch.cuda.synchronize()
    print(f"to_graph #{i}: {time.time() - t0:.2f} s", file=sys.stderr, flush=True)
    del g
