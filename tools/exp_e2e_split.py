"""Wall-clock split of the e2e call (C3): text H2D, device pipeline, answer fetch."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1501_06663_b200 import _native, workloads  # noqa: E402
from paper_1501_06663_b200._native import out_array  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
data = workloads.make(cfg)
n = data.size
ctx = _native.context(0)
total = np.zeros(1, np.int64)
for it in range(int(os.environ.get("ITERS", "8"))):
    with ctx.lock:
        ctx.synchronize()
        t0 = time.perf_counter()
        ctx.call("rs_set_text", _native.u8(data), n)
        ctx.synchronize()
        t1 = time.perf_counter()
        ctx.call("rs_query", 1, 1, _native.i64(total))
        ctx.synchronize()
        t2 = time.perf_counter()
        T = int(total[0])
        L, O, F = out_array(n + 1, False), out_array(n + 2, False), out_array(T, False)
        t3 = time.perf_counter()
        ctx.call("rs_fetch_all", _native.i64(L), _native.i64(O), _native.i64(F))
        t4 = time.perf_counter()
    print(f"h2d {1e3*(t1-t0):6.1f}  device {1e3*(t2-t1):6.1f}  alloc {1e3*(t3-t2):5.1f}  fetch {1e3*(t4-t3):6.1f}  "
          f"total {1e3*(t4-t0):6.1f} ms", flush=True)
