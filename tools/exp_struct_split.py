"""Wall-clock split of all_positions(text, structures=s) (C3): structures upload
(rank + lcp int64 -> device u32), device query, answer fetch."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1501_06663_b200 import _native, workloads  # noqa: E402
from paper_1501_06663_b200._native import out_array  # noqa: E402

data = workloads.make(sys.argv[1] if len(sys.argv) > 1 else "C3")
n = data.size
ctx = _native.context(0)
sa, rk, lc = np.empty(n + 1, np.int64), np.empty(n + 1, np.int64), np.empty(n + 2, np.int64)
total = np.zeros(1, np.int64)
with ctx.lock:
    ctx.call("rs_set_text", _native.u8(data), n)
    ctx.call("rs_build_structures")
    ctx.call("rs_get_structures", _native.i64(sa), _native.i64(rk), _native.i64(lc))
for it in range(int(os.environ.get("ITERS", "6"))):
    with ctx.lock:
        ctx.synchronize()
        t0 = time.perf_counter()
        ctx.call("rs_set_structures", None, _native.i64(rk), _native.i64(lc), n)
        ctx.synchronize()
        t1 = time.perf_counter()
        ctx.call("rs_query", 1, 1, _native.i64(total))
        ctx.synchronize()
        t2 = time.perf_counter()
        T = int(total[0])
        L, O, F = out_array(n + 1, False), out_array(n + 2, False), out_array(T, False)
        ctx.call("rs_fetch_all", _native.i64(L), _native.i64(O), _native.i64(F))
        t3 = time.perf_counter()
    print(f"upload {1e3*(t1-t0):6.1f}  device {1e3*(t2-t1):6.1f}  fetch {1e3*(t3-t2):6.1f}  total {1e3*(t3-t0):6.1f} ms",
          flush=True)
