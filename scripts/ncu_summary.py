"""Condense an `ncu --set full` report into the numbers profiles/ keeps:
per captured launch — duration, DRAM bytes (the `traffic` of the bench
roofline), throughput fractions, tensor / shared-memory pipe activity and the
top warp-stall reasons. usage: python scripts/ncu_summary.py rep.ncu-rep [out.json]"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "duration_ms": "gpu__time_duration.sum",
    "dram_read_GB": "dram__bytes_read.sum",
    "dram_write_GB": "dram__bytes_write.sum",
    "dram_pct_peak": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "mem_pct_peak": "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct_peak": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "tensor_pipe_pct": "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "smem_lsu_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "smem_tc_pct": "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "regs": "launch__registers_per_thread",
}


def num(v):
    try:
        return float(v.replace(",", ""))
    except (ValueError, AttributeError):
        return None


def main():
    raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    unit = dict(zip(hdr, units))
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        e = {"kernel": d.get("Kernel Name", "")[:120], "grid": d.get("Grid Size"), "block": d.get("Block Size")}
        for k, m in KEYS.items():
            name = m if m in d else next((h for h in hdr if h.endswith("." + m) or h.endswith(m)), m)
            v = num(d.get(name, ""))
            u = unit.get(name, "")
            if v is not None and k.endswith("_GB"):
                v = v * {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}.get(u, 1.0)
            if v is not None and k == "duration_ms":
                v = v * {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(u, 1.0)
            e[k] = round(v, 4) if v is not None else None
        stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): num(v) for k, v in d.items()
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
        stalls = {k: v for k, v in stalls.items() if v}
        tot = sum(stalls.values()) or 1.0
        e["top_stalls"] = {k: round(v / tot, 3) for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:5]}
        out.append(e)
    s = json.dumps(out, indent=1)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(s + "\n")
    print(s)


if __name__ == "__main__":
    main()
