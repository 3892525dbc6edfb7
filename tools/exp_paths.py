"""Experiment: device time of rs_query per path (raw vs compact) on a bench workload."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1501_06663_b200 import _native, workloads

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
data = workloads.make(cfg, None)
ctx = _native.context(0)
tot = np.zeros(1, np.int64)
with ctx.lock:
    ctx.call("rs_set_text", _native.u8(data), int(data.size))
    for path, name in ((1, "compact"), (0, "raw")):
        for rep in range(4):
            ctx.call("rs_clear_derived")
            ctx.synchronize()
            ctx.profile_begin()
            ctx.record(0)
            ctx.call("rs_query", 1, path, _native.i64(tot))
            ctx.record(1)
            ms = ctx.elapsed_ms(0, 1)
            prof = ctx.profile_end()
        top = sorted(prof, key=lambda k: -k["ms"])[:6]
        print(name, f"{ms:.2f} ms", [(k["kernel"], round(k["ms"], 2)) for k in top])
