"""Per-kernel device time of one full device step (suffix sort + LCP + query)
for a config, from the library's own CUDA-event profiler (not a bench value).

    python tools/exp_kernels.py C5 [n]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1501_06663_b200 import _native, workloads  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
data = workloads.make(cfg, n)
ctx = _native.context()
total = np.zeros(1, np.int64)
ctx.call("rs_set_text", _native.u8(data), int(data.size))
for it in range(2):
    ctx.call("rs_clear_derived")
    if it == 1:
        ctx.profile_begin()
    ctx.call("rs_query", 1, 1, _native.i64(total))
ctx.synchronize()
prof = ctx.profile_end()
print(cfg, "n", data.size, "rounds", ctx.sa_rounds(), "stages", ctx.stage_times())
tot = sum(k["ms"] for k in prof)
for k in sorted(prof, key=lambda k: -k["ms"])[:25]:
    gbs = k["bytes"] / (k["ms"] * 1e-3) / 1e9 if k["ms"] > 0 and k["bytes"] > 0 else 0
    print(f'{k["kernel"][:44]:44s} {k["launches"]:5d} {k["ms"]:9.2f} ms {100 * k["ms"] / tot:5.1f}%  {gbs:7.0f} GB/s')
