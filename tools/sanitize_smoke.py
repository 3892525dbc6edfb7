"""Small end-to-end run for compute-sanitizer (memcheck): every kernel family once."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_1501_06663_b200 as rb
from paper_1501_06663_b200 import workloads

for data in (workloads.iid_dna(20000, 1), workloads.planted_dna(30000, 2, family_len=100),
             workloads.english_like(20000, 4), workloads.fibonacci_mutated(30000, 5, rate=1e-3),
             np.frombuffer(b"mississippi", np.uint8), np.frombuffer(b"a", np.uint8)):
    t = rb.Text(data)
    s = rb.build_suffix_structures(t)
    assert rb.verify_suffix_structures(t, s)
    raw = rb.build_raw_llr(s)
    c = rb.build_compact_llr(raw)
    f = rb.compute_flags(raw)
    rb.scatter_compact(raw, f, rb.prefix_sum(f))
    for path in ("raw", "compact"):
        for mode in ("leftmost", "all"):
            rb.all_positions(t, mode=mode, path=path)
            rb.all_positions(t, mode=mode, path=path, structures=s)
print("sanitize smoke done")

# round-2 paths: int64 scan with negatives, the answer checker, query from
# resident structures (sa given, consistency check) by position shards, and
# the pipelined host transfers (arrays above the 8 MB staging threshold)
from paper_1501_06663_b200 import _native
from paper_1501_06663_b200.query import count_wrong_answers
v = np.arange(-5000, 5000, dtype=np.int64) * 7
assert np.array_equal(rb.parallel_scan(v), np.cumsum(v))
data = workloads.iid_dna(1_200_000, 9)
t = rb.Text(data)
s = rb.build_suffix_structures(t)
A = rb.all_positions(t, mode="all")
L = rb.all_positions(t, mode="leftmost")
c = rb.build_compact_llr(rb.build_raw_llr(s))
assert count_wrong_answers(c, t.n, all_answers=A, leftmost=L) == 0
ctx = _native.context()
n = t.n
with ctx.lock:
    ctx.call("rs_set_structures", _native.i64(s.sa), _native.i64(s.rank), _native.i64(s.lcp), n)
    for lo, hi in ((1, n // 2), (n // 2, n + 1)):
        tot = np.zeros(1, np.int64)
        ctx.call("rs_query_structures_shard", 1, lo, hi, _native.i64(tot))
        a = np.empty(hi - lo, np.int64)
        b = np.empty(hi - lo + 1, np.int64)
        f = np.empty(int(tot[0]), np.int64)
        ctx.call("rs_fetch_shard", 1, _native.i64(a), _native.i64(b), _native.i64(f))
        assert np.array_equal(a, A.lengths[lo:hi])
        assert np.array_equal(b - b[0], A.offsets[lo:hi + 1] - A.offsets[lo])
print("sanitize smoke (round 2 paths) done")

# byte wire (csrc/host_io.cu fetch_csr_bytes / fetch_leftmost_bytes): answers
# of >= 4 Mi positions, all-ties and leftmost, full and shard fetches
data = workloads.iid_dna((4 << 20) + 12345, 11)
t = rb.Text(data)
A = rb.all_positions(t, mode="all")
L = rb.all_positions(t, mode="leftmost")
n = t.n
assert int(A.lengths.max()) <= 255 and A.offsets[-1] == A.flat_starts.size
assert np.all(A.flat_starts[A.offsets[1:-1][np.diff(A.offsets[1:]) > 0]] >= 1)
with ctx.lock:
    ctx.call("rs_set_text", _native.u8(data), n)
    ctx.call("rs_build_structures")
    tot = np.zeros(1, np.int64)
    ctx.call("rs_query_structures_shard", 0, 1, n + 1, _native.i64(tot))
    s_ = np.empty(n, np.int64)
    l_ = np.empty(n, np.int64)
    ctx.call("rs_fetch_shard", 0, _native.i64(s_), _native.i64(l_), _native.i64(np.zeros(0, np.int64)))
assert np.array_equal(s_, L.starts[1:]) and np.array_equal(l_, L.lengths[1:])
print("sanitize smoke (byte wire) done")
