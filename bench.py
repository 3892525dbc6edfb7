#!/usr/bin/env python
"""Benchmark: positions/sec of the all-longest-repeat query (BASELINE.json metric).

Workload (N=1): config C3 -- 256 MiB i.i.d. ACGT (seed 3), END TO END on the
device: suffix sort -> rank -> LCP -> raw LLR -> compaction -> all-ties scan,
results written in the reference int64 CSR layout.  One step = one full pass
over the text; the text (256 MiB > 126 MB L2) stays resident in HBM, every
derived array is rebuilt each step.

  value  : n * steps / device time of the K timed steps (CUDA events on the
           library stream), positions/s.
  e2e    : the same metric through the public API a user calls,
           ``all_positions(Text, mode="all", path="compact")``: H2D of the text
           from pinned host memory + the whole device path + D2H of lengths,
           offsets and tie starts (int64) into pinned host arrays.
  roofline: dominant kernel of the step, algorithmic bytes / its average
           launch time (per-kernel CUDA events inside the timed region).
  cpu_baseline: the CPU oracle port (oracle/, C + OpenMP, restating the
           reference algorithm) on a bounded prefix of the same workload.

``--impl reference`` times that CPU port alone as the reference arm.
Multi-GPU (torchrun, N>1): see paper_1501_06663_b200/distributed.py.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "positions/sec, all-longest-repeat query, n=256M DNA, 1/2/4/8 B200 vs CPU"
UNIT = "positions/s"
PEAKS = REPO / "MEASURED_PEAKS.json"
FALLBACK_HBM_GBS = 6650.0


def hbm_peak() -> tuple[float, str]:
    try:
        return float(json.loads(PEAKS.read_text())["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


# ---------------------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,power.draw,utilization.gpu")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, util = [], [], []
        reasons = set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
                util.append(float(parts[7]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        loaded = [s for s, u in zip(sm, util) if u > 0] or sm
        return {"sm_mhz": float(np.median(loaded)) if loaded else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm), "samples_under_load": len(loaded)}


# ---------------------------------------------------------------------------------------
# CPU baseline / reference arm: the oracle port (C + OpenMP) on a bounded prefix
# ---------------------------------------------------------------------------------------
def cpu_run(data: np.ndarray, threads: int) -> dict:
    """SA+LCP (single thread, as the reference's numpy suffixes.py:31-66) + raw LLR +
    compaction + all-ties compact query (threaded like ExecPolicy.parallel)."""
    import oracle
    t0 = time.perf_counter()
    sa, rank, lcp = oracle.build_suffix_structures(data)
    t1 = time.perf_counter()
    raw = oracle.build_raw_llr(rank, lcp, threads)
    c = oracle.build_compact_llr(raw, threads)
    t2 = time.perf_counter()
    lengths, offsets, flat = oracle.all_all_positions(data.size, "compact", raw, c, threads)
    t3 = time.perf_counter()
    return {"n": int(data.size), "build_s": t1 - t0, "llr_compact_s": t2 - t1, "query_s": t3 - t2,
            "total_s": t3 - t0, "T": int(flat.size)}


def cpu_baseline(config: str, sample_n: int, threads: int) -> dict:
    from paper_1501_06663_b200 import workloads
    data = workloads.make(config, sample_n)
    r = cpu_run(data, threads)
    return {"value": r["n"] / r["total_s"], "unit": UNIT, "cores": threads, "kind": "port",
            "sample": (f"{config} generator at n={r['n']} (bounded prefix of the workload): "
                       f"SA+LCP {r['build_s']:.2f}s (1 thread, like the reference numpy build), "
                       f"LLR+compaction {r['llr_compact_s']:.3f}s + all-ties query {r['query_s']:.3f}s "
                       f"({threads} threads)"),
            "query_only_value": r["n"] / (r["llr_compact_s"] + r["query_s"])}


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1501_06663_b200 import workloads
    import oracle
    oracle.build() if not (REPO / "oracle" / "liboracle.so").exists() else None
    threads = os.cpu_count() or 1
    n = args.ref_sample
    data = workloads.make(args.config, n)
    for _ in range(args.warmup):
        cpu_run(data, threads)
    times = []
    for _ in range(args.steps):
        times.append(cpu_run(data, threads)["total_s"])
    t = float(np.sum(times))
    value = n * args.steps / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u8 text / int64 answers", "data": "synthetic",
        "config": {"workload": args.config, "n": n, "mode": "all", "path": "compact",
                   "note": "bounded prefix of the workload per step; CPU port of the reference"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{args.config} generator prefix n={n} per step, SA 1 thread, "
                                   f"query stages {threads} threads (oracle/repeatscan_oracle.c)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------------------
TRAFFIC_JSON = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r01", "traffic.json")


def committed_traffic(kernel: str):
    """DRAM bytes per launch of `kernel` from the committed `ncu --set full`
    capture of the same workload (profiles/r01/traffic.json), or None."""
    try:
        with open(TRAFFIC_JSON) as f:
            rec = json.load(f).get(kernel)
    except (OSError, ValueError):
        return None, None
    if not rec:
        return None, None
    return rec["dram_bytes_per_launch"], f"profiles/r01/{rec['report']} (dram__bytes_read.sum + dram__bytes_write.sum)"


def roofline_of(profile: list[dict], steps: int) -> tuple[dict, list[dict]]:
    peak, src = hbm_peak()
    rows = []
    for k in profile:
        if k["launches"] == 0:
            continue
        avg_ms = k["ms"] / k["launches"]
        per_launch = k["bytes"] / k["launches"]
        gbs = per_launch / (avg_ms * 1e-3) / 1e9 if avg_ms > 0 and per_launch > 0 else None
        rows.append({"kernel": k["kernel"], "launches_per_step": k["launches"] / steps,
                     "ms_per_step": k["ms"] / steps, "avg_launch_ms": avg_ms,
                     "bytes_per_launch": per_launch, "achieved_gbs": gbs,
                     "frac": (gbs / peak) if gbs else None})
    rows.sort(key=lambda r: -r["ms_per_step"])
    top = rows[0]
    traffic, tsrc = committed_traffic(top["kernel"])
    roof = {"bound": "hbm", "kernel": top["kernel"], "achieved": top["achieved_gbs"], "peak": peak,
            "unit": "GB/s", "frac": top["frac"], "traffic": traffic, "traffic_source": tsrc,
            "algorithmic_bytes_per_launch": top["bytes_per_launch"],
            "peak_source": f"{src} hbm_gbs (MEASURED_PEAKS.json)" if src == "measured" else
            "fallback 6650 GB/s (B200_PROFILING.md)"}
    return roof, rows


def run_single(args) -> None:
    from paper_1501_06663_b200 import Text, _native, all_positions, workloads

    dev = int(os.environ.get("LOCAL_RANK", "0"))
    ctx = _native.context(dev)
    t_gen = time.perf_counter()
    data = workloads.make(args.config, args.n)
    n = int(data.size)
    t_gen = time.perf_counter() - t_gen
    host_text = _native.pinned_pool.empty(n, np.uint8)
    host_text[:] = data

    # ---- device-resident steps ----
    with ctx.lock:
        ctx.call("rs_set_text", _native.u8(host_text), n)
        total = np.zeros(1, np.int64)

        def step():
            ctx.call("rs_clear_derived")
            ctx.call("rs_query", 1, 1, _native.i64(total))

        clocks = ClockSampler(dev)
        clocks.start()  # sampling spans warm-up + timed steps (nvidia-smi needs ~0.5 s to start)
        for _ in range(args.warmup):
            step()
        ctx.synchronize()
        launches0 = ctx.launches()
        ctx.profile_begin()
        ctx.record(0)
        for _ in range(args.steps):
            step()
        ctx.record(1)
        dev_ms = ctx.elapsed_ms(0, 1)
        profile = ctx.profile_end()
        launches = ctx.launches() - launches0
        stages = ctx.stage_times()
        rounds = ctx.sa_rounds()
        T = int(total[0])
        # un-instrumented timing of the same steps (profiling events add a little overhead)
        ctx.synchronize()
        ctx.record(0)
        for _ in range(args.steps):
            step()
        ctx.record(1)
        dev_ms_plain = ctx.elapsed_ms(0, 1)
        clk = clocks.stop()
    ms_per_step = min(dev_ms, dev_ms_plain) / args.steps
    value = n / (ms_per_step * 1e-3)

    # ---- e2e through the public API (pinned host in/out) ----
    t = Text(host_text)
    e2e_ms = []
    res = None
    for i in range(args.warmup + args.steps):
        del res
        res = None
        ctx.synchronize()
        ctx.record(2)
        res = all_positions(t, mode="all", path="compact", pinned=True)
        ctx.record(3)
        if i >= args.warmup:
            e2e_ms.append(ctx.elapsed_ms(2, 3))
    e2e_T = int(res.flat_starts.size)
    h2d = n
    d2h = 8 * (n + 1) + 8 * (n + 2) + 8 * e2e_T
    e2e_val = n / (np.mean(e2e_ms) * 1e-3)
    assert e2e_T == T, (e2e_T, T)

    roof, rows = roofline_of(profile, args.steps)
    scan = next((r for r in rows if r["kernel"].startswith("k_query")), None)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u8 text / u32 device indices / int64 answers",
        "data": "synthetic",
        "config": {"workload": args.config, "n": n, "mode": "all", "path": "compact",
                   "pipeline": "SA (prefix doubling: onesweep LSD radix, small tied groups sorted "
                               "directly) + LCP (round-0 keys + direct comparison; Kasai for "
                               "repetitive text) + raw LLR + compaction fused into the all-ties "
                               "scan (TMA-staged)",
                   "parallelism": "single GPU", "l2": "input 256 MiB > 126 MB L2; all arrays "
                                                     "rebuilt each step",
                   "T": T, "sa_rounds": rounds},
        "gpu_launches": launches // 1,
        "clocks": clk,
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": float(np.mean(e2e_ms)),
                "path": "all_positions(Text, mode='all', path='compact', pinned=True)"},
        "roofline": roof,
        "scan_kernel": ({"kernel": scan["kernel"], "achieved": scan["achieved_gbs"], "frac": scan["frac"],
                         "ms_per_step": scan["ms_per_step"], "bytes_per_launch": scan["bytes_per_launch"],
                         "positions_per_s": n / (scan["avg_launch_ms"] * 1e-3)} if scan else None),
        "stages_ms": stages,
        "kernels": rows,
        "query_only": {"value": n / (1e-3 * (stages["raw_llr"] + stages["compact"] + stages["query"])),
                       "unit": UNIT, "what": "raw LLR + compaction + all-ties scan with SA/LCP resident"},
    }
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config, args.cpu_sample, os.cpu_count() or 1)
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", default="C3")
    ap.add_argument("--n", type=int, default=None, help="override the config size")
    ap.add_argument("--cpu-sample", type=int, default=8 << 20)
    ap.add_argument("--ref-sample", type=int, default=4 << 20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.impl == "reference":
        run_reference(args)
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.gpus > 1:
        from paper_1501_06663_b200 import distributed
        distributed.bench_main(args)
        return
    run_single(args)


if __name__ == "__main__":
    main()
