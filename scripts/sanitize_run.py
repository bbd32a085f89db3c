"""Small training run for compute-sanitizer (scripts/sanitize.sh): a
tcgen05-sized GCRN-GRU and LSTM epoch (hidden 64, d 32) with the second cache
level forcing spills / refills / prefetches on the copy stream and the two
layer lanes on, plus a stacked GCN+LSTM epoch (C1's architecture)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2501_15348_b200 import api  # noqa: E402


def main():
    torch.cuda.set_device(0)
    g = api.Synth(600, 6.0, 32, 12, 0.03, 0.02, seed=3).to_graph()
    one = 600 * 32 * 4
    for arch in ("tgcn", "gcrn_m2", "gcrn_m1"):
        s = api.TrainSession(g, api.TrainConfig(arch=arch, hidden=64, hbm_cache_budget_bytes=2 * one))
        r = s.run_epoch()
        print(arch, "loss", r["loss"], "tier", s.tier_stats(), flush=True)
    torch.cuda.synchronize()
    print("sanitize run ok")


if __name__ == "__main__":
    main()
