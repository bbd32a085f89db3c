"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per kernel name, launches, total / mean device time and share of the listed
time. usage: python scripts/launch_summary.py launches.csv [out.json]"""
import csv
import json
import re
import sys
from collections import defaultdict


def short(name):
    name = re.sub(r"\(.*\)$", "", name)           # drop the parameter list
    name = re.sub(r"^void\s+", "", name)
    name = re.sub(r"^(\(anonymous namespace\)|unnamed>)::", "", name)
    return name


def main():
    rows = []
    with open(sys.argv[1]) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r["Metric Unit"], 1e-3)
        rows.append((short(r["Kernel Name"]), float(r["Metric Value"].replace(",", "")) * scale))
    agg = defaultdict(lambda: [0, 0.0])
    for k, us in rows:
        agg[k][0] += 1
        agg[k][1] += us
    total = sum(v[1] for v in agg.values())
    out = {"launches": len(rows), "total_us": round(total, 1), "kernels": [
        {"kernel": k, "launches": n, "total_us": round(t, 1), "mean_us": round(t / n, 2),
         "share": round(t / total, 4)}
        for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])]}
    s = json.dumps(out, indent=1)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(s + "\n")
    print(s)


if __name__ == "__main__":
    main()
