#!/usr/bin/env python
"""Benchmark: positions/sec of the all-longest-repeat query (BASELINE.json metric).

Workload (N=1): config C3 -- 256 MiB i.i.d. ACGT (seed 3), all ties, compact
path.  Like for like with the reference arm: one step
is the reference's query path from GIVEN suffix structures (query.py:234):
raw LLR (llr.py:63-72) -> compaction (llr.py:119-123) -> all-ties scan with
the int64 CSR answers written (query.py:187-215).  The structures are built
once, untimed, on the device and passed back in as the reference's int64
SuffixStructures; every step rebuilds raw LLR, compaction and answers from
them (256 MiB text and 2 GiB of structures > 126 MB L2).

  value     : n * steps / device time of the K timed steps (CUDA events on
              the library stream), positions/s.
  e2e       : the public call a user makes, ``all_positions(Text, mode="all",
              path="compact")`` with host buffers: text H2D, suffix sort, LCP,
              query, D2H of the int64 lengths/offsets/tie starts into numpy.
  e2e_structures_given: the reference arm's exact call (structures= given).
  end_to_end_device: SA + LCP + query from the resident text (device only).
  parity    : digests of the answers vs tests/golden/fullsize_digests.json.
  roofline  : dominant kernel of the step, algorithmic bytes / its average
              launch time (per-kernel CUDA events, separate instrumented pass).
  cpu_baseline: one full-size step of the CPU oracle port (oracle/, C +
              OpenMP restating the reference) from the same structures.

``--impl reference`` times that CPU port as the reference arm on the same
config (structures built untimed by the oracle's threaded prefix doubling).
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
# CPU baseline / reference arm: the oracle port (C + OpenMP) of the reference's query
# path on the SAME workload, structures given
# ---------------------------------------------------------------------------------------
def cpu_query_step(n: int, rank: np.ndarray, lcp: np.ndarray, threads: int) -> dict:
    """One reference query pass from given structures (query.py:234-239 with
    ``structures=`` supplied): build_raw_llr (llr.py:63-72) -> build_compact_llr
    (llr.py:119-123) -> _all_all_positions on the compact path (query.py:187-215),
    each stage split over ``threads`` like ExecPolicy.parallel(threads)."""
    import oracle
    t0 = time.perf_counter()
    raw = oracle.build_raw_llr(rank, lcp, threads)
    t1 = time.perf_counter()
    c = oracle.build_compact_llr(raw, threads)
    t2 = time.perf_counter()
    lengths, offsets, flat = oracle.all_all_positions(n, "compact", raw, c, threads)
    t3 = time.perf_counter()
    return {"raw_llr_s": t1 - t0, "compaction_s": t2 - t1, "query_s": t3 - t2, "total_s": t3 - t0,
            "T": int(flat.size), "m": int(c[0].size)}


def cpu_structures(data: np.ndarray, threads: int):
    """CPU suffix structures for the baseline's ``structures=`` input (untimed):
    the oracle's threaded prefix doubling, identical to the reference's arrays."""
    import oracle
    return oracle.build_suffix_structures(data, workers=threads)


def run_reference(args) -> None:
    """Reference arm: the reference CPU path (oracle port) on our arm's config,
    metric and unit: n / (raw LLR + compaction + all-ties query) with the
    suffix structures given, every stage on all host threads."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1501_06663_b200 import workloads
    import oracle
    oracle.build() if not (REPO / "oracle" / "liboracle.so").exists() else None
    threads = os.cpu_count() or 1
    data = workloads.make(args.config, args.n)
    n = int(data.size)
    t0 = time.perf_counter()
    _, rk, lc = cpu_structures(data, threads)
    build_s = time.perf_counter() - t0
    for _ in range(args.warmup):
        cpu_query_step(n, rk, lc, threads)
    steps = [cpu_query_step(n, rk, lc, threads) for _ in range(args.steps)]
    t = float(sum(r["total_s"] for r in steps))
    value = n * args.steps / t
    stage = {k: float(np.mean([r[k] for r in steps])) for k in ("raw_llr_s", "compaction_s", "query_s")}
    sample = (f"{args.config} at full size n={n}: each step = raw LLR + compaction + all-ties compact "
              f"query from given structures (oracle/repeatscan_oracle.c restating llr.py / query.py / "
              f"_kernels_numba.py, {threads} threads like ExecPolicy.parallel); structures built untimed "
              f"in {build_s:.1f} s by the oracle's threaded prefix doubling")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": args.config, "n": n, "mode": "all", "path": "compact",
                   "timed": "raw LLR + compaction + all-ties query, structures given (query.py:234)",
                   "T": steps[0]["T"], "m": steps[0]["m"]},
        "stages_s": stage,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------------------
PROFILES = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles")
TRAFFIC_JSON = next((os.path.join(PROFILES, r, "traffic.json") for r in ("r02", "r01")
                     if os.path.exists(os.path.join(PROFILES, r, "traffic.json"))),
                    os.path.join(PROFILES, "r02", "traffic.json"))


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
    rnd = os.path.basename(os.path.dirname(TRAFFIC_JSON))
    return rec["dram_bytes_per_launch"], f"profiles/{rnd}/{rec['report']} (dram__bytes_read.sum + dram__bytes_write.sum)"


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


def _digest(a: np.ndarray) -> str:
    import hashlib
    return hashlib.sha256(memoryview(np.ascontiguousarray(a, dtype=np.int64)).cast("B")).hexdigest()[:16]


def parity_of(config: str, n: int, res) -> dict:
    """Compare the answers the bench produced with the committed full-size
    digests (tests/golden/fullsize_digests.json: reference / pinned oracle)."""
    path = REPO / "tests" / "golden" / "fullsize_digests.json"
    try:
        rec = json.loads(path.read_text()).get(config)
    except (OSError, ValueError):
        rec = None
    if rec is None or rec.get("n") != n:
        return {"checked": False, "why": f"no committed digests for {config} at n={n}"}
    got = {"a_lengths": _digest(res.lengths), "a_offsets": _digest(res.offsets),
           "a_flat": _digest(res.flat_starts)}
    ok = all(rec[k] == v for k, v in got.items()) and rec["T"] == int(res.flat_starts.size)
    return {"checked": True, "bit_exact": bool(ok), "source": rec.get("source"),
            "arrays": "all-ties lengths, offsets, flat tie starts (sha256 of the int64 arrays)"}


def run_single(args) -> None:
    from paper_1501_06663_b200 import SuffixStructures, Text, _native, all_positions, workloads

    dev = int(os.environ.get("LOCAL_RANK", "0"))
    ctx = _native.context(dev)
    data = workloads.make(args.config, args.n)
    n = int(data.size)
    host_text = _native.pinned_pool.empty(n, np.uint8)
    host_text[:] = data
    total = np.zeros(1, np.int64)

    with ctx.lock:
        # ---- structures (untimed, like the reference arm): built on device,
        # handed back to the host as the reference's int64 SuffixStructures ----
        sa = np.empty(n + 1, np.int64)
        rk = np.empty(n + 1, np.int64)
        lc = np.empty(n + 2, np.int64)
        ctx.call("rs_set_text", _native.u8(host_text), n)
        ctx.call("rs_build_structures")
        ctx.call("rs_get_structures", _native.i64(sa), _native.i64(rk), _native.i64(lc))
        ctx.call("rs_set_structures", _native.i64(sa), _native.i64(rk), _native.i64(lc), n)

        def q_step():  # llr.py:63-123 + query.py:187-215 from resident structures
            ctx.call("rs_clear_llr")
            ctx.call("rs_query", 1, 1, _native.i64(total))

        clocks = ClockSampler(dev)
        clocks.start()  # sampling spans warm-up + timed steps (nvidia-smi needs ~0.5 s to start)
        for _ in range(args.warmup):
            q_step()
        ctx.synchronize()
        launches0 = ctx.launches()
        ctx.record(0)
        for _ in range(args.steps):
            q_step()
        ctx.record(1)
        q_ms = ctx.elapsed_ms(0, 1) / args.steps
        launches = ctx.launches() - launches0
        T = int(total[0])
        # per-kernel breakdown: a separate instrumented pass (events around every launch)
        ctx.profile_begin()
        for _ in range(args.steps):
            q_step()
        ctx.synchronize()
        profile = ctx.profile_end()
        q_stages = ctx.stage_times()
        clk = clocks.stop()

        # ---- the whole device path from the resident text (SA-inclusive, extra key) ----
        ctx.call("rs_set_text", _native.u8(host_text), n)

        def full_step():
            ctx.call("rs_clear_derived")
            ctx.call("rs_query", 1, 1, _native.i64(total))

        for _ in range(args.warmup):
            full_step()
        ctx.synchronize()
        ctx.record(0)
        for _ in range(args.steps):
            full_step()
        ctx.record(1)
        full_ms = ctx.elapsed_ms(0, 1) / args.steps
        full_stages = ctx.stage_times()
        rounds = ctx.sa_rounds()
        assert int(total[0]) == T

    value = n / (q_ms * 1e-3)

    # ---- e2e through the public API with host buffers (default call) ----
    t = Text(host_text)
    s_host = SuffixStructures(sa=sa, rank=rk, lcp=lc)

    def e2e_run(fn, reps):
        """mean seconds per call over `reps` timed calls, the last result, and
        the (h2d, d2h) bytes the library actually copied per timed call"""
        out, res, xfer0 = [], None, None
        for i in range(args.warmup + reps):
            res = None
            ctx.synchronize()
            if i == args.warmup:
                xfer0 = ctx.transfer_bytes()
            t0 = time.perf_counter()
            res = fn()
            out.append(time.perf_counter() - t0)
        xfer1 = ctx.transfer_bytes()
        per = tuple((b - a) // reps for a, b in zip(xfer0, xfer1))
        return float(np.mean(out[args.warmup:])), res, per

    e2e_s, res, (e2e_h2d, e2e_d2h) = e2e_run(lambda: all_positions(t, mode="all", path="compact"), args.steps)
    parity = parity_of(args.config, n, res)
    assert int(res.flat_starts.size) == T
    del res
    e2e_struct_s, res, (es_h2d, es_d2h) = e2e_run(
        lambda: all_positions(t, mode="all", path="compact", structures=s_host), max(3, args.steps // 3))
    assert int(res.flat_starts.size) == T
    del res
    answer_bytes = 8 * (n + 1) + 8 * (n + 2) + 8 * T  # the int64 arrays the caller receives

    roof, rows = roofline_of(profile, args.steps)
    scan = next((r for r in rows if r["kernel"].startswith("k_query")), None)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": q_ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32 device indices / int64 answers",
        "data": "synthetic",
        "config": {"workload": args.config, "n": n, "mode": "all", "path": "compact",
                   "timed": "raw LLR + compaction + all-ties query with the suffix structures given "
                            "(query.py:234; BASELINE.md section 2), int64 CSR answers written on device",
                   "structures": "built untimed on device, passed back in as the reference's int64 "
                                 "SuffixStructures (sa, rank, lcp; sa checked once to invert rank)",
                   "parallelism": "single GPU",
                   "l2": "input 256 MiB > 126 MB L2; raw LLR, compaction and answers rebuilt each step",
                   "T": T},
        "gpu_launches": launches,
        "clocks": clk,
        "e2e": {"value": n / e2e_s, "unit": UNIT, "h2d_bytes_per_step": e2e_h2d, "d2h_bytes_per_step": e2e_d2h,
                "ms_per_step": 1e3 * e2e_s, "answer_bytes_per_step": answer_bytes,
                "bytes_counted": "rs_transfer_bytes: every host<->device copy the library issued in the timed calls "
                                 "(answers cross PCIe as 1 byte per value when they fit, else 4; host threads "
                                 "rebuild the int64 arrays)",
                "path": "all_positions(Text, mode='all', path='compact') -- default call, host text in, "
                        "int64 numpy answers out (suffix sort + LCP + query on device, inside the timing)"},
        "e2e_structures_given": {
            "value": n / e2e_struct_s, "unit": UNIT, "ms_per_step": 1e3 * e2e_struct_s,
            "h2d_bytes_per_step": es_h2d, "d2h_bytes_per_step": es_d2h,
            "path": "all_positions(Text, mode='all', path='compact', structures=SuffixStructures) -- "
                    "the reference arm's exact call"},
        "parity": parity,
        "roofline": roof,
        "scan_kernel": ({"kernel": scan["kernel"], "achieved": scan["achieved_gbs"], "frac": scan["frac"],
                         "ms_per_step": scan["ms_per_step"], "bytes_per_launch": scan["bytes_per_launch"],
                         "positions_per_s": n / (scan["avg_launch_ms"] * 1e-3)} if scan else None),
        "stages_ms": q_stages,
        "kernels": rows,
        "end_to_end_device": {"value": n / (full_ms * 1e-3), "unit": UNIT, "ms_per_step": full_ms,
                              "what": "suffix sort + LCP + raw LLR + compaction + all-ties query from the "
                                      "resident text", "stages_ms": full_stages, "sa_rounds": rounds},
    }
    if not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        cpu = cpu_query_step(n, rk, lc, threads)
        line["cpu_baseline"] = {
            "value": n / cpu["total_s"], "unit": UNIT, "cores": threads, "kind": "port",
            "sample": (f"one step of the same workload at full size (n={n}, structures given): raw LLR "
                       f"{cpu['raw_llr_s']:.2f}s + compaction {cpu['compaction_s']:.2f}s + all-ties query "
                       f"{cpu['query_s']:.2f}s on {threads} threads (oracle/repeatscan_oracle.c)")}
        assert cpu["T"] == T
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", default="C3")
    ap.add_argument("--n", type=int, default=None, help="override the config size")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.impl == "reference":
        run_reference(args)
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.gpus > 1:
        from paper_1501_06663_b200 import distributed
        distributed.bench_main(args, tools={"ClockSampler": ClockSampler, "roofline_of": roofline_of})
        return
    run_single(args)


if __name__ == "__main__":
    main()
