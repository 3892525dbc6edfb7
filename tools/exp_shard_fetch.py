"""1-GPU projection of the multi-GPU result transfer (distributed.fetch_shard_shared):
the D2H of ONE rank's shard (n / N positions of C3) into its slice of a
shared /dev/shm buffer, with that rank's share of the host threads
(RS_HOST_THREADS = 16 / N, set per process by the caller).  N ranks run these
transfers in parallel over N PCIe links; they then share the host's memory
bandwidth, which this single-process projection does not model.

    RS_HOST_THREADS=4 python tools/exp_shard_fetch.py 4
"""
import mmap
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1501_06663_b200 import _native, workloads  # noqa: E402
from paper_1501_06663_b200 import distributed as D  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1
data = workloads.make("C3")
n = int(data.size)
ctx = _native.context()
ctx.call("rs_set_text", _native.u8(data), n)
ctx.call("rs_build_structures")
lo, hi = D.shard_range(n, N, 0)
total = np.zeros(1, np.int64)
ctx.call("rs_query_structures_shard", 1, lo, hi, _native.i64(total))
T = int(total[0])
nel = (n + 1) + (n + 2) + T * N  # the whole answer's buffer (this shard fills 1/N of it)
path = f"/dev/shm/exp_shard_{os.getpid()}"
fd = os.open(path, os.O_CREAT | os.O_RDWR, 0o600)
os.ftruncate(fd, 8 * nel)
mm = mmap.mmap(fd, 8 * nel, mmap.MAP_SHARED)
os.close(fd)
os.unlink(path)
buf = np.frombuffer(mm, np.int64)
views = D.layout_views(buf, n, "all", T * N)
a, b, f = D.shard_views(views, "all", lo, hi, 0, T)
ts = []
for it in range(5):
    t0 = time.perf_counter()
    ctx.call("rs_fetch_shard", 1, _native.i64(a), _native.i64(b), _native.i64(f))
    ts.append(time.perf_counter() - t0)
gb = 8 * ((hi - lo) * 2 + T) / 1e9
print(f"N={N} threads={os.environ.get('RS_HOST_THREADS', 'all')} shard={hi - lo} positions, {gb:.2f} GB int64: "
      + " ".join(f"{1e3 * x:.1f}" for x in ts) + " ms (first = fresh tmpfs pages)")
