"""Bit-exact parity at the BASELINE configurations' full sizes (C2-C5).

The inputs are regenerated from their seeded generators; every int64
reference-layout array is compared by sha256 with the digests committed in
tests/golden/fullsize_digests.json, which were produced by running the
REFERENCE package itself (C2 64 Mi, C4 100 Mi, C3 256 Mi) or, at 1 GiB where
the reference needs ~95 GB of host RAM, the pinned u32 oracle restatement
(C5; oracle/oracle32.c, pinned by tests/test_oracle_golden.py).  The answers
are produced by exactly the pipeline bench.py times: ``all_positions(Text,
mode=..., path="compact")`` with ``structures=None`` (suffix sort, LCP, raw
LLR emitted by the sort, compaction fused into the scan).

A second, digest-free property (test_full_size_answers_checked) re-derives
every answer with an independent kernel that runs the reference's
Algorithm 4 literally (binary search + walk over the compact entries built by
the int64 array API) and counts disagreeing positions.
"""

from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import paper_1501_06663_b200 as rb
from paper_1501_06663_b200 import workloads
from paper_1501_06663_b200.query import count_wrong_answers

pytestmark = pytest.mark.gpu

FULL = Path(__file__).resolve().parent / "golden" / "fullsize_digests.json"
CONFIGS = ["C2", "C3", "C4", "C5"]


def _digests() -> dict:
    return json.loads(FULL.read_text()) if FULL.exists() else {}


def dg(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a, dtype=np.int64)
    return hashlib.sha256(memoryview(a).cast("B")).hexdigest()[:16]


def _rec(config: str) -> dict:
    rec = _digests().get(config)
    if rec is None:
        pytest.fail(f"no committed full-size digests for {config} in {FULL.name}")
    return rec


@pytest.mark.parametrize("config", CONFIGS)
def test_full_size_digests(config):
    rec = _rec(config)
    data = workloads.make(config)
    assert data.size == rec["n"]
    t = rb.Text(data)
    # the bench pipeline: structures=None, compact path, all ties
    A = rb.all_positions(t, mode="all", path="compact")
    assert A.flat_starts.size == rec["T"]
    assert dg(A.lengths) == rec["a_lengths"]
    assert dg(A.offsets) == rec["a_offsets"]
    assert dg(A.flat_starts) == rec["a_flat"]
    del A
    L = rb.all_positions(t, mode="leftmost", path="compact")
    assert dg(L.starts) == rec["l_starts"] and dg(L.lengths) == rec["l_lengths"]
    del L
    s = rb.build_suffix_structures(t)
    assert dg(s.sa) == rec["sa"]
    assert dg(s.rank) == rec["rank"]
    assert dg(s.lcp) == rec["lcp"]
    raw = rb.build_raw_llr(s)
    del s
    assert dg(raw) == rec["raw"] and int(raw.max(initial=0)) == rec["max_llr"]
    c = rb.build_compact_llr(raw)
    assert c.size == rec["m"]
    assert dg(c.starts) == rec["c_starts"] and dg(c.lengths) == rec["c_lengths"]


@pytest.mark.parametrize("config", CONFIGS)
def test_full_size_answers_checked(config):
    data = workloads.make(config)
    n = int(data.size)
    t = rb.Text(data)
    s = rb.build_suffix_structures(t)
    assert rb.verify_suffix_structures(t, s)
    raw = rb.build_raw_llr(s)
    del s
    c = rb.build_compact_llr(raw)
    del raw
    A = rb.all_positions(t, mode="all", path="compact")
    assert count_wrong_answers(c, n, all_answers=A) == 0
    del A
    L = rb.all_positions(t, mode="leftmost", path="compact")
    assert count_wrong_answers(c, n, leftmost=L) == 0


def test_answer_checker_detects_faults(rng):
    """The checker itself: exact on the oracle's answers, and it flags a
    shortened length, a dropped tie, a swapped tie order, a wrong leftmost."""
    import oracle
    for data in (workloads.iid_dna(50_000, 3), workloads.planted_dna(60_000, 2, family_len=60),
                 workloads.fibonacci_mutated(40_000, 5, rate=1e-3)):
        n = data.size
        t = rb.Text(data)
        raw = rb.build_raw_llr(rb.build_suffix_structures(t))
        c = rb.build_compact_llr(raw)
        lengths, offsets, flat = oracle.all_positions(data, mode="all", path="compact", workers=4)
        starts, llen = oracle.all_positions(data, mode="leftmost", path="compact", workers=4)
        A = rb.AllAnswers(lengths=lengths, offsets=offsets, flat_starts=flat)
        L = rb.LeftmostAnswers(starts=starts, lengths=llen)
        assert count_wrong_answers(c, n, all_answers=A, leftmost=L) == 0
        k = int(np.flatnonzero(np.diff(offsets)[1:] >= 2)[0]) + 1  # a position with >= 2 ties
        bad = lengths.copy()
        bad[k] -= 1
        assert count_wrong_answers(c, n, all_answers=rb.AllAnswers(bad, offsets, flat)) >= 1
        f2 = flat.copy()
        o = int(offsets[k])
        f2[o], f2[o + 1] = f2[o + 1], f2[o]
        assert count_wrong_answers(c, n, all_answers=rb.AllAnswers(lengths, offsets, f2)) == 1
        o2 = offsets.copy()
        o2[k + 1:] -= 1
        f3 = np.delete(flat, o)
        assert count_wrong_answers(c, n, all_answers=rb.AllAnswers(lengths, o2, f3)) >= 1
        s2 = starts.copy()
        s2[k] = flat[o + 1]
        assert count_wrong_answers(c, n, leftmost=rb.LeftmostAnswers(s2, llen)) == 1


@pytest.mark.parametrize("config", ["C2", "C3", "C4"])
def test_full_size_raw_path_digests(config):
    """The raw path (Algorithms 1/3 over the raw LLR array, k_query<raw>) at
    full size gives the same committed digests (raw and compact
    answers are identical).  C5 is skipped: its raw walk is ~alpha*n =
    ~10^13 steps (the reference restricts it to the compact path too)."""
    rec = _rec(config)
    t = rb.Text(workloads.make(config))
    A = rb.all_positions(t, mode="all", path="raw")
    assert A.flat_starts.size == rec["T"]
    assert dg(A.lengths) == rec["a_lengths"] and dg(A.offsets) == rec["a_offsets"]
    assert dg(A.flat_starts) == rec["a_flat"]
    del A
    L = rb.all_positions(t, mode="leftmost", path="raw")
    assert dg(L.starts) == rec["l_starts"] and dg(L.lengths) == rec["l_lengths"]
