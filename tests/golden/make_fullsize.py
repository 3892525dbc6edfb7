"""Full-size parity digests for the BASELINE configurations C2-C5.

The GPU tests (`tests/test_fullsize_gpu.py`, `-m gpu`) regenerate each input
from its seeded generator on the GPU box, run the exact pipeline bench.py
times (``all_positions(Text, mode=..., structures=None)``) and compare
sha256 digests of every int64 reference-layout array with the digests
committed here (`tests/golden/fullsize_digests.json`).

Sources (run in the build container; nothing at test time touches them):

* ``reference`` -- the REFERENCE package itself (C2 64 Mi, C4 100 Mi,
  C3 256 Mi): ``build_suffix_structures`` (suffixes.py:56-66) ->
  ``build_raw_llr`` / ``compute_flags`` / ``prefix_sum`` / ``build_compact_llr``
  (llr.py:63-123) -> ``_leftmost_all_positions`` / ``_all_all_positions``
  (query.py:171-215) with ``ExecPolicy.parallel(os.cpu_count())``::

      NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src \\
          python tests/golden/make_fullsize.py reference C2

* ``oracle32`` -- the u32 restatement in ``oracle/oracle32.c`` (C5, 1 GiB:
  the reference needs ~95 GB of RAM there, this container has 62 GB).  It is
  pinned to the reference by ``tests/test_oracle_golden.py`` (identical digests
  on the 1-2 Mi reference digest set)::

      python tests/golden/make_fullsize.py oracle32 C5

Digests are sha256 (first 16 hex digits) of the int64 ref-layout bytes, the
same convention as ``digests.json``.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))

from paper_1501_06663_b200 import workloads  # noqa: E402

OUT = HERE / "fullsize_digests.json"


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, np.int64).tobytes()).hexdigest()[:16]


def _save(name: str, rec: dict) -> None:
    import fcntl
    with open(HERE / ".fullsize.lock", "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        cur = json.loads(OUT.read_text()) if OUT.exists() else {}
        cur[name] = rec
        OUT.write_text(json.dumps(cur, indent=1, sort_keys=True) + "\n")


def from_reference(name: str) -> dict:
    import repeatscan  # the reference, via PYTHONPATH
    from repeatscan.engine import ExecPolicy
    from repeatscan.llr import build_compact_llr, build_raw_llr, compute_flags, prefix_sum
    from repeatscan.query import _all_all_positions, _leftmost_all_positions
    from repeatscan.suffixes import build_suffix_structures
    from repeatscan.text import Text
    assert "/root/reference" in repeatscan.__file__, repeatscan.__file__

    pol = ExecPolicy.parallel(os.cpu_count() or 1)
    t0 = time.time()
    data = workloads.make(name)
    n = int(data.size)
    rec = {"source": "reference", "n": n, "expr": f"workloads.make({name!r})"}
    s = build_suffix_structures(Text(data))
    rec["sa_build_s"] = round(time.time() - t0, 1)
    print(f"{name}: structures {rec['sa_build_s']} s", flush=True)
    rec.update(sa=digest(s.sa), rank=digest(s.rank), lcp=digest(s.lcp))
    raw = build_raw_llr(s, pol)
    del s
    rec.update(raw=digest(raw), max_llr=int(raw.max(initial=0)))
    flags = compute_flags(raw, pol)
    rec["flags"] = digest(flags)
    ps = prefix_sum(flags, pol)
    rec["ps"] = digest(ps)
    del flags, ps
    c = build_compact_llr(raw, pol)
    rec.update(m=int(c.size), c_starts=digest(c.starts), c_lengths=digest(c.lengths))
    t1 = time.time()
    L = _leftmost_all_positions(n, "compact", raw, c, pol)
    rec.update(l_starts=digest(L.starts), l_lengths=digest(L.lengths))
    del L
    A = _all_all_positions(n, "compact", raw, c, pol)
    rec.update(T=int(A.flat_starts.size), a_lengths=digest(A.lengths),
               a_offsets=digest(A.offsets), a_flat=digest(A.flat_starts))
    rec["query_s"] = round(time.time() - t1, 1)
    rec["total_s"] = round(time.time() - t0, 1)
    return rec


def from_oracle32(name: str) -> dict:
    import oracle
    t0 = time.time()
    data = workloads.make(name)
    rec = {"source": "oracle32", "n": int(data.size), "expr": f"workloads.make({name!r})"}
    rec.update(oracle.digests32(data, log=lambda s: print(f"{name}: {s}", flush=True)))
    rec["total_s"] = round(time.time() - t0, 1)
    return rec


if __name__ == "__main__":
    source, names = sys.argv[1], sys.argv[2:]
    for nm in names:
        fn = {"reference": from_reference, "oracle32": from_oracle32}[source]
        r = fn(nm)
        key = os.environ.get("FULLSIZE_KEY", nm)
        _save(key, r)
        print(json.dumps({nm: r}), flush=True)
