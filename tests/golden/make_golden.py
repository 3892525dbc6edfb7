"""Generate golden parity fixtures by running the REFERENCE package itself.

Run in the build container (the only place /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

Outputs (committed):
  tests/golden/golden_small.npz  -- full reference arrays for ~900 small inputs
  tests/golden/digests.json      -- sha256 digests of reference arrays for
                                    medium/large seeded inputs (regenerated
                                    from tests' seeds on the GPU box)

Nothing at test time imports the reference; tests only read these files.
"""

from __future__ import annotations

import hashlib
import itertools
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))

import repeatscan  # noqa: E402  (the reference, via PYTHONPATH)
from repeatscan.engine import ExecPolicy  # noqa: E402
from repeatscan.llr import (  # noqa: E402
    build_compact_llr, build_raw_llr, compact_llr_sequential, compute_flags, prefix_sum,
)
from repeatscan.query import _all_all_positions, _leftmost_all_positions  # noqa: E402
from repeatscan.suffixes import build_suffix_structures  # noqa: E402
from repeatscan.text import Text  # noqa: E402

from paper_1501_06663_b200 import workloads  # noqa: E402

assert "reference" in repeatscan.__file__ or "/root/reference" in repeatscan.__file__, \
    repeatscan.__file__

FIELDS = ("text", "sa", "rank", "lcp", "raw", "flags", "ps", "c_starts", "c_lengths",
          "l_starts", "l_lengths", "a_lengths", "a_offsets", "a_flat", "w_raw", "w_comp")


def reference_arrays(data: np.ndarray, paths=("raw", "compact"), policy=None) -> dict:
    t = Text(np.asarray(data, np.uint8))
    s = build_suffix_structures(t)
    raw = build_raw_llr(s, policy)
    flags = compute_flags(raw, policy)
    ps = prefix_sum(flags, policy)
    c = build_compact_llr(raw, policy)
    seq = compact_llr_sequential(raw)
    assert np.array_equal(seq.starts, c.starts) and np.array_equal(seq.lengths, c.lengths)
    out = dict(text=t.data.astype(np.int64), sa=s.sa, rank=s.rank, lcp=s.lcp, raw=raw,
               flags=flags, ps=ps, c_starts=c.starts, c_lengths=c.lengths)
    left = alll = None
    for path in paths:
        L = _leftmost_all_positions(s.n, path, raw, c if path == "compact" else None, policy)
        A = _all_all_positions(s.n, path, raw, c if path == "compact" else None, policy)
        if left is None:
            left, alll = L, A
        else:  # raw and compact paths must agree
            assert np.array_equal(left.starts, L.starts) and np.array_equal(left.lengths, L.lengths)
            assert np.array_equal(alll.offsets, A.offsets)
            assert np.array_equal(alll.flat_starts, A.flat_starts)
    out.update(l_starts=left.starts, l_lengths=left.lengths, a_lengths=alll.lengths,
               a_offsets=alll.offsets, a_flat=alll.flat_starts)
    from repeatscan.stats import walk_steps_compact, walk_steps_raw  # stats.py:30-55
    out.update(w_raw=walk_steps_raw(raw), w_comp=walk_steps_compact(c, s.n))
    return out


def small_cases() -> list[bytes]:
    named = [b"", b"a", b"ab", b"ba", b"abc", b"aaaa", b"mississippi", b"abcabcddbca",
             b"abracadabra", b"abcabcabc", b"banana", b"aaaaaaaaaaaaaaaaaaaaaaaaaaaaaaaa",
             b"ACGTACGTACGT", b"\x00\x01\x00\x01\x00", b"\xff\xfe\xff\xfe\xff\x00",
             bytes(range(256)), bytes(range(256)) * 2, b"zyxwvutsrqponmlkjihgfedcba" * 3]
    cases = list(named)
    for n in range(1, 9):  # exhaustive over {a,b} (test_acceptance.py:117-119)
        cases += [bytes(t) for t in itertools.product(b"ab", repeat=n)]
    rng = np.random.default_rng(4242)  # test_acceptance.py:120-125 shape
    for _ in range(300):
        n = int(rng.integers(1, 65))
        sigma = int(rng.integers(1, 5))
        cases.append(rng.choice(np.frombuffer(b"acgt"[:sigma], np.uint8), size=n).tobytes())
    rng = np.random.default_rng(7)
    for _ in range(40):  # wider alphabets / arbitrary bytes incl. 0x00 and 0xff
        n = int(rng.integers(1, 300))
        sigma = int(rng.integers(1, 257))
        alpha = rng.choice(256, size=sigma, replace=False).astype(np.uint8)
        cases.append(rng.choice(alpha, size=n).tobytes())
    # medium structured inputs, one per config shape
    cases.append(workloads.iid_dna(5000, 11).tobytes())
    cases.append(workloads.planted_dna(6000, 12, family_len=60).tobytes())
    cases.append(workloads.english_like(5000, 13).tobytes())
    cases.append(workloads.fibonacci_mutated(5000, 14, rate=1e-3).tobytes())
    cases.append(workloads.periodic_mutated(5000, 15, period=37, rate=2e-3).tobytes())
    cases.append(workloads.fibonacci_mutated(3000, 16, rate=0.0).tobytes())
    return cases


def write_small():
    cases = small_cases()
    cat = {f: [] for f in FIELDS}
    offs = {f: [0] for f in FIELDS}
    for data in cases:
        arrs = reference_arrays(np.frombuffer(data, np.uint8))
        for f in FIELDS:
            a = np.asarray(arrs[f], np.int64)
            cat[f].append(a)
            offs[f].append(offs[f][-1] + a.size)
    payload = {}
    for f in FIELDS:
        payload[f] = np.concatenate(cat[f]) if cat[f] else np.zeros(0, np.int64)
        payload[f + "_off"] = np.asarray(offs[f], np.int64)
    np.savez_compressed(HERE / "golden_small.npz", **payload)
    print(f"golden_small.npz: {len(cases)} cases")


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, np.int64).tobytes()).hexdigest()[:16]


def tsv_digests(arrs: dict) -> dict:
    """sha256 of the reference CLI serialisations (cli.py:72-93)."""
    from repeatscan.cli import serialize_all, serialize_leftmost
    from repeatscan.query import AllAnswers, LeftmostAnswers
    n = arrs["sa"].size - 1
    L = LeftmostAnswers(starts=arrs["l_starts"], lengths=arrs["l_lengths"])
    A = AllAnswers(lengths=arrs["a_lengths"], offsets=arrs["a_offsets"], flat_starts=arrs["a_flat"])
    return {"leftmost_tsv": hashlib.sha256(serialize_leftmost(L, 1, n)).hexdigest()[:16],
            "all_tsv": hashlib.sha256(serialize_all(A, 1, n)).hexdigest()[:16]}


LARGE = [
    # name, generator expression (evaluated in tests too), paths
    ("acgt_1e6_seed99", "workloads.reference_dna(1_000_000, 99)", ("raw", "compact")),
    ("C1_2p20", "workloads.make('C1')", ("raw", "compact")),
    ("C2_shape_2p21", "workloads.planted_dna(1 << 21, 2)", ("raw", "compact")),
    ("C4_shape_2p21", "workloads.english_like(1 << 21, 4)", ("raw", "compact")),
    ("C5_shape_2p20", "workloads.fibonacci_mutated(1 << 20, 5)", ("compact",)),
    ("periodic_2p20", "workloads.periodic_mutated(1 << 20, 5)", ("compact",)),
]


def write_digests():
    out = {}
    pol = ExecPolicy.parallel(os.cpu_count() or 1)
    for name, expr, paths in LARGE:
        t0 = time.time()
        data = eval(expr)
        arrs = reference_arrays(data, paths=paths, policy=pol)
        rec = {"expr": expr, "n": int(data.size), "m": int(arrs["c_starts"].size),
               "T": int(arrs["a_flat"].size), "max_llr": int(arrs["raw"].max(initial=0))}
        for f in FIELDS:
            if f != "text":
                rec[f] = digest(arrs[f])
        rec.update(tsv_digests(arrs))
        out[name] = rec
        print(f"{name}: n={data.size} m={rec['m']} T={rec['T']} {time.time() - t0:.1f}s",
              flush=True)
    (HERE / "digests.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    which = sys.argv[1:] or ["small", "digests"]
    if "small" in which:
        write_small()
    if "digests" in which:
        write_digests()
