"""One device-resident step of the bench workload, for ncu captures.

    ncu --set full --clock-control none --import-source on -k regex:k_onesweep \
        --launch-skip 2 -c 1 -o gpurun_out/onesweep python tools/ncu_step.py --config C3

Runs two steps (the first warms the buffers); --launch-skip counts launches of
the selected kernel across both.  Never used for timing.
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1501_06663_b200 import _native, workloads  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--query-only", action="store_true",
                    help="the bench step: raw LLR + compaction + query from given structures")
    args = ap.parse_args()
    data = workloads.make(args.config, args.n)
    ctx = _native.context(0)
    host = np.ascontiguousarray(data)
    total = np.zeros(1, np.int64)
    with ctx.lock:
        ctx.call("rs_set_text", _native.u8(host), int(host.size))
        if args.query_only:
            n = int(host.size)
            sa, rk, lc = (np.empty(n + 1, np.int64), np.empty(n + 1, np.int64), np.empty(n + 2, np.int64))
            ctx.call("rs_build_structures")
            ctx.call("rs_get_structures", _native.i64(sa), _native.i64(rk), _native.i64(lc))
            ctx.call("rs_set_structures", _native.i64(sa), _native.i64(rk), _native.i64(lc), n)
            for _ in range(args.steps):
                ctx.call("rs_clear_llr")
                ctx.call("rs_query", 1, 1, _native.i64(total))
            ctx.synchronize()
            print("T =", int(total[0]))
            return
        for _ in range(args.steps):
            ctx.call("rs_clear_derived")
            ctx.call("rs_query", 1, 1, _native.i64(total))
        ctx.synchronize()
    print("T =", int(total[0]))


if __name__ == "__main__":
    main()
