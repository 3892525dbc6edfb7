"""Raw LLR from given structures: SA-order bucketed scatter (sa given and
consistent) vs the reference formula's rank gather (sa not given), C3.
Per-kernel device times from the library's CUDA-event profiler."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1501_06663_b200 import _native, workloads  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
data = workloads.make(cfg)
n = data.size
ctx = _native.context(0)
total = np.zeros(1, np.int64)
sa, rk, lc = np.empty(n + 1, np.int64), np.empty(n + 1, np.int64), np.empty(n + 2, np.int64)
with ctx.lock:
    ctx.call("rs_set_text", _native.u8(data), n)
    ctx.call("rs_build_structures")
    ctx.call("rs_get_structures", _native.i64(sa), _native.i64(rk), _native.i64(lc))
    for label, s_arg in (("sa given", _native.i64(sa)), ("rank only", None)):
        ctx.call("rs_set_structures", s_arg, _native.i64(rk), _native.i64(lc), n)
        for it in range(3):
            ctx.call("rs_clear_llr")
            if it == 2:
                ctx.profile_begin()
            ctx.call("rs_query", 1, 1, _native.i64(total))
        ctx.synchronize()
        prof = ctx.profile_end()
        tot = sum(k["ms"] for k in prof)
        print(f"== {label}: step {tot:.2f} ms, T = {int(total[0])}")
        for k in sorted(prof, key=lambda k: -k["ms"])[:6]:
            print(f'   {k["kernel"][:40]:40s} {k["ms"]:7.3f} ms')
