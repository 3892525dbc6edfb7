"""Time the result D2H (rs_fetch_all) variants at C3 size on the box."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1501_06663_b200 import _native, workloads  # noqa: E402

n = int(os.environ.get("N", 256 << 20))
ctx = _native.context()
data = workloads.make("C3", n)
total = np.zeros(1, np.int64)
ctx.call("rs_set_text", _native.u8(data), n)
ctx.call("rs_query", 1, 1, _native.i64(total))
T = int(total[0])
print("threads", os.environ.get("RS_HOST_THREADS", "default"), "T", T)


def fetch(pool):
    L = pool(n + 1)
    O = pool(n + 2)
    F = pool(T)
    t = time.perf_counter()
    ctx.call("rs_fetch_all", _native.i64(L), _native.i64(O), _native.i64(F))
    return time.perf_counter() - t, (L, O, F)


for name, pool in [("fresh np.empty", lambda c: np.empty(c, np.int64)),
                   ("pageable pool", lambda c: _native.pageable_pool.empty(c)),
                   ("pinned pool", lambda c: _native.pinned_pool.empty(c))]:
    ts = []
    for _ in range(4):
        dt, keep = fetch(pool)
        del keep
        ts.append(dt)
    print(f"{name:16s}: " + " ".join(f"{1e3 * x:7.1f}" for x in ts) + " ms")
# text upload paths
for name, src in [("pageable text", np.array(data)), ("pinned text", None)]:
    if src is None:
        src = _native.pinned_pool.empty(n, np.uint8)
        src[:] = data
    ts = []
    for _ in range(3):
        t = time.perf_counter()
        ctx.call("rs_set_text", _native.u8(src), n)
        ctx.synchronize()
        ts.append(time.perf_counter() - t)
    print(f"{name:16s}: " + " ".join(f"{1e3 * x:7.1f}" for x in ts) + " ms")
