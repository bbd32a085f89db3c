"""Condensed view of scripts/epoch_timing.py output (one line per epoch)."""
import json
import sys

for line in open(sys.argv[1]):
    if line.startswith('{"dev_ms"'):
        d = json.loads(line)
        print(d["dev_ms"], d["kernel_ms"], d["sample_ms_max"], d["host_ms_sum"], d["host_ms_max"],
              d.get("host_max_at"), d.get("phase_max"))
