"""Benchmark: training snapshots/sec of the ReInc dynamic-GNN hot path on B200.

Default workload (BASELINE.json configs[3] / configs[4], SURVEY §8d "C4"/"C5",
the graph the metric's 1/2/4/8-GPU numbers are quoted on; it fits one B200):
integrated GraphRNN GCRN-GRU (tgcn, 2 layers, hidden 64) on a synthetic
dynamic graph of 4M nodes / 80M edges, 64 snapshots, 2% edge churn with
deletions and 2% feature-changed nodes per step, feature dim 128, L=8, H=1,
S=1, sum aggregation, REINC cache at capacity 1.0, incremental aggregation
on. `--workload c3` runs the 1M-node GC-LSTM config (configs[2]). One "step"
= one training epoch over all W executable windows (55 at C4) with the
reference's distributed semantics (per-window gradients, ordered sum / W, one
Adam step; src/distsim.cpp:197-272); with N GPUs the windows are split into
consecutive blocks (plan(), src/distsim.cpp:52-70) and the flat gradient is
all-reduced over NCCL. Total work is fixed as N grows ("strong" scaling).
snapshots/sec = W * (L + H) / epoch seconds.

`--impl reference` times the reference's own CPU implementation (oracle/_ref,
compiled from /root/reference/proj/src) on a bounded sample of the same
workload (see cpu_baseline.sample in the output).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: synth + model parameters
    "c3": dict(n=1_000_000, deg=20.0, dim=128, T=32, edge=0.02, feat=0.0, arch="gcrn_m2", hidden=64,
               desc="GC-LSTM (gcrn_m2) on 1M-node / 20M-edge synthetic graph, 32 snapshots, "
                    "2% churn with deletions, feat 128, hidden 64"),
    "c1": dict(n=10_000, deg=10.0, dim=64, T=16, edge=0.01, feat=0.01, arch="gcrn_m1", hidden=64,
               desc="stacked GCN+LSTM (gcrn_m1), 10K nodes / 100K edges, 16 snapshots, 1% churn"),
    "c2": dict(n=207, deg=1515 / 207, dim=2, T=2000, edge=0.0, feat=1.0, arch="gcrn_m2", hidden=64,
               desc="GCRN-LSTM on METR-LA-shaped synthetic graph, 207 nodes, 2000 snapshots"),
    "c4": dict(n=4_000_000, deg=20.0, dim=128, T=64, edge=0.02, feat=0.02, arch="tgcn", hidden=64,
               desc="GCRN-GRU (tgcn) on 4M-node / 80M-edge graph, 64 snapshots, structure + feature dynamicity"),
}
L, H = 8, 1


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def measure_tf32_peak():
    """Dense TF32 tensor-core throughput on this GPU, the MEASURED_PEAKS method
    applied to fp32 with TF32 allowed: torch.matmul 8192^3 (2 N^3 flops), best
    of 10 after 3 warm-ups, CUDA events. The cell GEMMs' tensor-pipe
    denominator (each of their 3xTF32 products is one TF32 GEMM)."""
    import torch
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        n = 8192
        a = torch.randn(n, n, device="cuda")
        b = torch.randn(n, n, device="cuda")
        for _ in range(3):
            torch.matmul(a, b)
        best = float("inf")
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        del a, b
        return 2.0 * n ** 3 / (best / 1e3) / 1e12
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc:
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=10)
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for name, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ reference arm
def host_cpu():
    """CPU model and core count of the box the reference runs on."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


# Same-config reference runs: the reference's seq-first / distsim epoch on the
# workload's exact graph (N, E, d, h, churn), timed by its own EpochReport
# clock (src/train.cpp:151, :203-204). C1 runs whole epochs; C2's epoch is
# 1,991 identical-cost windows over a 207-node graph, so one reference step
# is a contiguous prefix of them (the generator's first T' snapshots are the
# same for any T >= T').
SAME_CONFIG_T = {"c1": 16, "c2": 200}


def reference_same_config(wl, name):
    from oracle import refbind as R
    T = SAME_CONFIG_T[name]
    g = R.RefGraph.synth(wl["n"], wl["deg"], wl["dim"], T, wl["edge"], wl["feat"], seed=1)
    r = g.run(R.RunCfg(arch=wl["arch"], hidden=wl["hidden"], workers=1, record_events=False))
    rate = len(r.losses) * (L + H) / r.seconds
    full = "the full epoch" if T == wl["T"] else f"the first {len(r.losses)} of the epoch's windows"
    desc = (f"reference seq-first/distsim epoch (oracle/_ref, Eigen-subset shim, 1 thread) on the "
            f"workload's own graph ({wl['n']} nodes, d={wl['dim']}, h={wl['hidden']}): {full}, "
            f"{len(r.losses)} windows in {r.seconds:.1f}s")
    return rate, r.seconds, desc


def reference_sample(wl, budget_s=15.0):
    """Workloads the reference cannot hold (C3: ~43 GB of materialised fp64
    snapshots, C4: ~348 GB): times its seq-first trainer on a bounded sample
    — same degree / feature / hidden / churn, N scaled down, T = L+H+2 (one
    window, SURVEY §0 T-1 rule) — and scales the rate linearly in N. An
    extrapolation, not a same-config measurement. Returns (scaled rate, raw
    rate, seconds, description)."""
    from oracle import refbind as R
    cfg = R.RunCfg(arch=wl["arch"], hidden=wl["hidden"], workers=1, record_events=False)

    def run(n):
        g = R.RefGraph.synth(n, wl["deg"], wl["dim"], L + H + 2, wl["edge"], wl["feat"], seed=1)
        r = g.run(cfg)
        return len(r.losses) * (L + H) / r.seconds, r.seconds

    probe_n = 2000
    rate, secs = run(probe_n)
    n = int(min(max(probe_n * budget_s / max(secs, 1e-3), probe_n), wl["n"]))
    rate, secs = run(n)
    scaled = rate * n / wl["n"]
    desc = (f"EXTRAPOLATED: reference seq-first/distsim epoch (oracle/_ref, Eigen-subset shim, 1 thread) "
            f"on a {n}-node sample of the workload (avg degree {wl['deg']:g}, d={wl['dim']}, "
            f"h={wl['hidden']}, {wl['edge']:.0%} churn, T={L + H + 2}: 1 window); {rate:.3f} snapshots/s "
            f"at the sample, scaled x{n}/{wl['n']} (cost linear in N and E) to the full workload; "
            f"{secs:.1f}s per sample")
    return scaled, rate, secs, desc


def reference_step(wl, name):
    """One reference-arm step: (rate, same_config, description)."""
    if name in SAME_CONFIG_T:
        rate, _, desc = reference_same_config(wl, name)
        return rate, True, desc
    v, _, _, desc = reference_sample(wl)
    return v, False, desc


def run_reference_arm(args, wl):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    # a single-threaded CPU code path has no device or JIT to warm: the
    # warm-up steps are untimed repetitions of the same step, capped at one
    for _ in range(min(args.warmup, 1)):
        reference_step(wl, args.workload)
    vals, same, desc = [], False, ""
    for _ in range(max(args.steps, 1)):
        v, same, desc = reference_step(wl, args.workload)
        vals.append(v)
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": "training snapshots/sec", "value": value,
        "unit": "snapshots/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": min(args.warmup, 1),
        "higher_is_better": True, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, "desc": wl["desc"]},
        "same_config": same,
        "cpu_baseline": {"value": value, "unit": "snapshots/s", "cores": 1, "kind": "reference",
                         "sample": desc, **host_cpu()},
        "e2e": {"value": value, "unit": "snapshots/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "vs_baseline": None,
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ B200 arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-tf32-peak", action="store_true", help="skip the in-run TF32 peak measurement")
    ap.add_argument("--prof-in-timed", type=int, default=-1,
                    help="1: per-kernel-class CUDA-event profiling inside the timed region (the "
                         "roofline's launch times are those of the timed steps); 0: the timed steps "
                         "run unprofiled and one extra profiled step gives the class breakdown. "
                         "Default: 1 for the bandwidth-bound workloads (c3, c4), 0 for the "
                         "launch-latency-bound ones (c1, c2), where two events per kernel class "
                         "scope measurably slow the host issue loop")
    ap.add_argument("--hbm-cache-gb", type=float, default=0.0,
                    help="second cache level: HBM budget of unborrowed cached aggregations "
                         "(0 = everything stays in HBM; C4 spills below ~16 GB)")
    args = ap.parse_args()
    wl = WORKLOADS[args.workload]
    if args.prof_in_timed < 0:
        args.prof_in_timed = 0 if args.workload in ("c1", "c2") else 1
    if args.impl == "reference":
        return run_reference_arm(args, wl)

    import torch
    import torch.distributed as dist
    from paper_2501_15348_b200 import api

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    tf32_peak = None
    try:
        if not args.no_tf32_peak:
            tf32_peak = measure_tf32_peak()
    except Exception as e:  # noqa: BLE001 — report, do not fail the bench
        log(f"tf32 peak measurement failed: {e}")
    torch.cuda.empty_cache()
    t0 = time.perf_counter()
    synth = api.Synth(wl["n"], wl["deg"], wl["dim"], wl["T"], wl["edge"], wl["feat"], seed=1)
    t_synth = time.perf_counter() - t0
    t0 = time.perf_counter()
    graph = synth.to_graph(stream)
    retained = (0, wl["T"] - 1)
    if world > 1:  # this rank's window block + the L+H overlap only (replicate_overlap)
        retained = graph.retain_for_rank(world, rank, L, 1, H)
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    log(f"[rank {rank}] synth {t_synth:.1f}s, device graph build {t_build:.2f}s")
    cfg = api.TrainConfig(arch=wl["arch"], hidden=wl["hidden"], workers=world,
                          hbm_cache_budget_bytes=int(args.hbm_cache_gb * 1e9))
    sess = api.TrainSession(graph, cfg, rank=rank, stream=stream)
    W_total, wb, we = sess.windows()

    # the gradient all-reduce runs inside the library (NCCL communicator of
    # the C ABI; the id is exchanged over torch.distributed)
    comm = api.comm_from_torch(world, rank)

    def epoch():
        sess.run_dist_epoch(comm)

    for _ in range(args.warmup):
        epoch()
    torch.cuda.synchronize()
    barrier()

    # ---------------- timed region (device time, max over ranks)
    api.prof_reset()
    api.prof_enable(bool(args.prof_in_timed))
    launches0 = api.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        barrier()
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        ev0.record(stream)
        for _ in range(args.steps):
            epoch()
        ev1.record(stream)
        torch.cuda.synchronize()
        wall_ms = (time.perf_counter() - w0) * 1e3
        barrier()
    api.prof_enable(False)
    launches = api.launch_count() - launches0
    prof_steps = args.steps
    if not args.prof_in_timed:  # one extra, profiled step for the class breakdown
        api.prof_reset()
        api.prof_enable(True)
        epoch()
        torch.cuda.synchronize()
        api.prof_enable(False)
        prof_steps = 1
    if world > 1:  # whole-job kernel launches (every rank's)
        lt = torch.tensor([launches], device="cuda", dtype=torch.int64)
        dist.all_reduce(lt)
        launches = int(lt.item())
    ms_total = ev0.elapsed_time(ev1)
    t = torch.tensor([ms_total], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    snaps_per_step = W_total * (L + H)
    value = snaps_per_step / (ms_step / 1e3)
    prof = api.prof_get()
    scopes = api.prof_get(scopes=True)
    losses = sess.losses()

    # ---------------- roofline of the dominant kernel class (+ the graded delta-SpMM)
    peaks, peak_src = load_peaks()
    kernel_ms = sum(v["ms"] for v in prof.values())
    dom = max(prof, key=lambda k: prof[k]["ms"])
    # agg_scratch mixes input (w=d) and hidden (w=h) aggregations; when the
    # transposed SpMM (all launches one shape) is within 3% of it, it is the
    # kernel reported (and the one whose ncu DRAM traffic is in profiles/)
    if dom == "agg_scratch" and prof["agg_backward"]["ms"] >= 0.97 * prof["agg_scratch"]["ms"]:
        dom = "agg_backward"
    # kernel names in the committed ncu captures (profiles/r2_ncu_*.json: `ncu --set
    # full` of the C4 bench / scripts/kernel_bench.py at C4 shapes)
    ncu_kernels = {"agg_backward": "k_spmm_sum<4, 4>", "agg_scratch": "k_spmm_sum<4, 4>",
                   "agg_delta": "k_agg_delta_v4<8, 4", "cell_bwd": "k_row_gemm<4, 256>",
                   "cell_fwd": "k_row_gemm<1, 256>", "weight_grad": "k_wgrad_mn<256, 208>"}
    ncu_files = ["r2_ncu_full_c4.json", "r2_ncu_row_gemm_epi4.json", "r2_ncu_row_gemm_epi1.json",
                 "r2_ncu_wgrad_mn_c4.json"]

    def ncu_traffic(name):
        """DRAM bytes per launch (dram__bytes_read + write) of this kernel from
        the committed `ncu --set full` captures of the C4 shapes, or None."""
        if args.workload != "c4" or name not in ncu_kernels:
            return None
        rows = []
        for fname in ncu_files:
            path = os.path.join(ROOT, "profiles", fname)
            if os.path.exists(path):
                rows += [e for e in json.load(open(path)) if ncu_kernels[name] in e.get("kernel", "")]
        if not rows:
            return None
        return round(1e9 * statistics.mean(e["dram_read_GB"] + e["dram_write_GB"] for e in rows))

    def roof(name):
        v = prof[name]
        if not v["launches"] or v["ms"] <= 0:
            return None
        per_ms = v["ms"] / v["launches"]
        achieved = (v["bytes"] / v["launches"]) / (per_ms / 1e3) / 1e9
        peak = peaks["hbm_gbs"]
        traffic = ncu_traffic(name)
        dram = {} if traffic is None else {
            # measured DRAM bytes (ncu) over the live launch time: the HBM
            # utilisation behind the algorithmic figure
            "dram_achieved": round(traffic / (per_ms / 1e3) / 1e9, 1),
            "dram_frac": round(traffic / (per_ms / 1e3) / 1e9 / peak, 4)}
        return {"kernel": name, "bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic, **dram,
                "note": "achieved = algorithmic bytes (SURVEY 8d: every edge gather counted, no reuse) "
                        "/ device time; peak = measured copy (read+write) bandwidth — a gather-dominated "
                        "read stream can exceed it; traffic = ncu DRAM read+write bytes per launch",
                "alg_bytes_per_launch": round(v["bytes"] / v["launches"]),
                "peak_source": peak_src, "launches": v["launches"],
                "avg_launch_us": round(per_ms * 1e3, 2),
                "share_of_kernel_time": round(v["ms"] / kernel_ms, 4),
                "tflops": round(v["flops"] / (v["ms"] / 1e3) / 1e12, 2) if v["flops"] else None}

    roofline = roof(dom)
    delta_roof = roof("agg_delta")
    # the cell GEMMs against both their bounds: algorithmic HBM bytes and the
    # tensor pipe (3 TF32 products per fp32 product, against the measured TF32 peak)
    gemm_roof = {}
    for name in ("cell_fwd", "cell_bwd", "cell_bwd_gemm", "weight_grad"):
        r = roof(name)
        if r is None or not prof[name]["flops"]:
            continue
        tf = 3 * prof[name]["flops"] / (prof[name]["ms"] / 1e3) / 1e12
        gemm_roof[name] = {"hbm_frac": r["frac"], "dram_frac": r.get("dram_frac"),
                           "tf32_tflops_issued": round(tf, 1),
                           "tensor_frac": round(tf / tf32_peak, 4) if tf32_peak else None,
                           "avg_launch_us": r["avg_launch_us"]}

    free_b, total_b = torch.cuda.mem_get_info()
    st = sess.stats()
    pool = api.mem_stats()
    memory = {"hbm_in_use_gb": round((total_b - free_b) / 1e9, 1),
              "pool_used_high_gb": round(pool["used_high"] / 1e9, 1),
              "pool_reserved_high_gb": round(pool["reserved_high"] / 1e9, 1),
              "graph_store_gb": round(graph.device_bytes() / 1e9, 1),
              "feature_versions": graph.feature_stats(),
              "cache": {k: st[k] for k in ("hits", "misses", "evictions", "expirations",
                                           "resident_peak_units")},
              "cache_tier": {"hbm_budget_gb": args.hbm_cache_gb, **sess.tier_stats()}}
    # the e2e leg builds its own graph + session: release the timed ones first (C4 is ~150 GB)
    del sess, graph
    torch.cuda.synchronize()

    # ---------------- end to end through the public API from host buffers
    e2e = None
    if not args.no_e2e:
        sizes = synth.sizes
        h2d = int(sizes[0]) * 8 + wl["n"] * wl["dim"] * 4
        for t in range(1, wl["T"]):
            nd, ni, nc = (int(x) for x in sizes[1 + 3 * (t - 1): 4 + 3 * (t - 1)])
            h2d += 8 * (nd + ni) + 4 * nc + 4 * nc * wl["dim"]
        e_steps = max(1, min(args.steps, 2))
        barrier()
        torch.cuda.synchronize()
        e0 = time.perf_counter()
        ev2, ev3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev2.record(stream)
        build_ms = []
        for _ in range(e_steps):
            b0 = time.perf_counter()
            g2 = synth.to_graph(stream)          # H2D of the compact graph + device build
            if world > 1:
                g2.retain_for_rank(world, rank, L, 1, H)
            torch.cuda.current_stream().synchronize()
            build_ms.append((time.perf_counter() - b0) * 1e3)
            s2 = api.TrainSession(g2, cfg, rank=rank, stream=stream)
            s2.run_dist_epoch(comm)  # + D2H of window losses
            d2h = 8 * len(s2.losses())
            del s2, g2
        ev3.record(stream)
        torch.cuda.synchronize()
        barrier()
        e_ms = ev2.elapsed_time(ev3)
        t = torch.tensor([e_ms], device="cuda", dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t.item()) / e_steps
        e2e = {"value": snaps_per_step / (e_ms / 1e3), "unit": "snapshots/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": round(e_ms, 2),
               "graph_upload_build_ms": round(statistics.mean(build_ms), 1),
               "note": "per step: pinned-host->HBM upload of snapshot 0 + per-step deltas, device "
                       "CSR/extract_delta build, one sharded epoch, D2H of window losses"}

    # ---------------- CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            v, same, desc = reference_step(wl, args.workload)
            cpu = {"value": v, "unit": "snapshots/s", "cores": 1, "kind": "reference", "sample": desc,
                   "same_config": same, **host_cpu()}
        except Exception as e:  # reference not built on this box
            cpu = {"value": None, "unit": "snapshots/s", "cores": 1, "kind": "reference",
                   "sample": f"unavailable: {e}", **host_cpu()}

    if rank == 0:
        line = {
            "metric": "training snapshots/sec", "value": round(value, 3), "unit": "snapshots/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_step, 3), "wall_ms_per_step": round(wall_ms / args.steps, 3),
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": args.workload, "desc": wl["desc"], "windows": W_total,
                       "hbm_cache_budget_gb": args.hbm_cache_gb,
                       "seq_len": L, "horizon": H, "nodes": wl["n"],
                       "edges": int(synth.sizes[0]), "snapshots": wl["T"],
                       "parallelism": f"window-shard x{world} (consecutive_block)",
                       "rank0_snapshots_retained": list(retained),
                       "l2": f"inputs exceed the 126 MB L2 (graph store {memory['graph_store_gb']} GB; "
                             f"one feature matrix {wl['n'] * wl['dim'] * 4 / 1e9:.2f} GB)"},
            "roofline": roofline, "roofline_delta_spmm": delta_roof,
            "roofline_gemms": {"tf32_peak_tflops": round(tf32_peak, 1) if tf32_peak else None,
                               "tf32_peak_source": "measured in this run (torch.matmul fp32 with TF32, "
                                                   "8192^3, best of 10)", **gemm_roof},
            "kernel_ms_by_class": {k: round(v["ms"] / prof_steps, 2) for k, v in prof.items()},
            "profiled": "timed steps" if args.prof_in_timed else "one extra step after the timed ones",
            "host_ms_per_sample": {k: round(v["ms"] / max(scopes["sample_host"]["launches"], 1), 3)
                                   for k, v in scopes.items() if k.startswith("host") or k == "sample_host"},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "memory": memory,
            "clocks": clocks.summary(), "epoch_loss": float(losses.mean()) if len(losses) else None,
            "setup_s": {"synth": round(t_synth, 1), "device_graph_build": round(t_build, 2)},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
