"""CPU-side checks: the C-ABI library loads and exports what include/*.h declares,
the ctypes binding covers it, and host-side API behaviour (no device calls)."""

from __future__ import annotations

import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from conftest import REPO, golden_cases

HEADER = REPO / "include" / "repeatscan_b200.h"


def declared_functions() -> set[str]:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(rs_\w+)\s*\(", text, flags=re.M))


def test_library_builds_and_exports_every_declared_symbol():
    from paper_1501_06663_b200 import _build, _native
    lib = _build.build()
    out = subprocess.run(["nm", "-D", "--defined-only", str(lib)], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r" T (rs_\w+)$", out, flags=re.M))
    declared = declared_functions()
    assert len(declared) >= 40
    assert declared <= exported, declared - exported
    assert declared == set(_native.SIGNATURES), declared ^ set(_native.SIGNATURES)
    _native.load_library()  # dlopen + resolve every symbol (no device call)


def test_library_is_sm100a_only():
    from paper_1501_06663_b200 import _build
    lib = _build.build()
    out = subprocess.run(["cuobjdump", "--list-elf", str(lib)], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_no_oracle_on_product_path():
    pkg = REPO / "paper_1501_06663_b200"
    # the test-infrastructure package `oracle` (not the public brute-force API
    # functions oracle_llr / oracle_all_lr of bruteforce.py, reference oracle.py)
    pat = re.compile(r"^\s*(import\s+oracle\b|from\s+oracle\b)", re.M)
    for p in pkg.rglob("*.py"):
        assert not pat.search(p.read_text()), p


def test_policy_and_argument_validation_before_device():
    import paper_1501_06663_b200 as rb
    with pytest.raises(ValueError):
        rb.ExecPolicy("parallel", 0)
    with pytest.raises(ValueError):
        rb.ExecPolicy("gpu", 1)
    assert rb.ExecPolicy.parallel(4).workers == 4
    with pytest.raises(ValueError):
        rb.all_positions(rb.Text.from_str("abc"), mode="nope")
    with pytest.raises(ValueError):
        rb.all_positions(rb.Text.from_str("abc"), path="nope")


def test_text_and_compact_types():
    import paper_1501_06663_b200 as rb
    t = rb.Text.from_str("mississippi")
    assert t.n == 11 and t.sigma == 4 and t.char(1) == ord("m")
    with pytest.raises(IndexError):
        t.char(0)
    assert t.substring(2, 4) == b"issi"
    c = rb.CompactLlr.from_arrays(np.array([2, 5, 9]), np.array([4, 4, 1]))
    assert c.ends.tolist() == [5, 8, 9] and c.entry(2) == rb.LlrEntry(5, 4)
    assert c.entry(2).end == 8
    with pytest.raises(IndexError):
        c.entry(4)


def test_single_position_queries_match_golden():
    # host-side helpers (query.py:45-127) against reference-generated arrays
    import paper_1501_06663_b200 as rb
    for c in golden_cases()[:300]:
        comp = rb.CompactLlr.from_arrays(c.c_starts, c.c_lengths)
        for k in range(1, c.n + 1):
            want = rb.LrAnswer(int(c.l_starts[k]), int(c.l_lengths[k]))
            assert rb.leftmost_lr_raw(c.raw, k) == want
            assert rb.leftmost_lr_compact(comp, k, c.n) == want
            lo, hi = int(c.a_offsets[k]), int(c.a_offsets[k + 1])
            wall = [rb.LrAnswer(int(s), int(c.a_lengths[k])) for s in c.a_flat[lo:hi]]
            assert rb.all_lr_raw(c.raw, k) == wall
            assert rb.all_lr_compact(comp, k) == wall
    with pytest.raises(IndexError):
        rb.leftmost_lr_raw(np.zeros(4, np.int64), 0)


def test_workload_generators_shapes():
    from paper_1501_06663_b200 import workloads
    d = workloads.make("C1")
    assert d.size == 1 << 20 and set(np.unique(d).tolist()) == set(b"ACGT")
    e = workloads.english_like(200_000, 4)
    assert e.size == 200_000 and 60 <= np.unique(e).size <= 96
    f = workloads.fibonacci_mutated(100_000, 5)
    assert f.size == 100_000
    p = workloads.planted_dna(100_000, 2)
    assert p.size == 100_000


def test_bruteforce_api_matches_reference_golden():
    """is_repeat / oracle_llr / oracle_all_lr (reference oracle.py, exported by
    __init__.py:20) against the reference's own answers for small golden cases."""
    import paper_1501_06663_b200 as rb
    from conftest import golden_cases
    from paper_1501_06663_b200.bruteforce import oracle_all_positions
    checked = 0
    for c in golden_cases():
        if not 1 <= c.n <= 40:
            continue
        t = rb.Text(c.data)
        for k in range(1, c.n + 1):
            lo, hi = int(c.a_offsets[k]), int(c.a_offsets[k + 1])
            want = [(int(s), int(c.a_lengths[k])) for s in c.a_flat[lo:hi]]
            assert [tuple(a) for a in rb.oracle_all_lr(t, k)] == want
            r = rb.oracle_llr(t, k)
            assert (r.start, r.length) == ((k, int(c.raw[k])) if c.raw[k] else (-1, 0))
        assert [tuple(a) for a in oracle_all_positions(t, "leftmost")] == \
            list(zip(c.l_starts[1:].tolist(), c.l_lengths[1:].tolist()))
        checked += 1
    assert checked > 300
    t = rb.Text.from_str("abcabcddbca")  # test_query.py:61-63
    assert rb.is_repeat(t, 1, 3) and not rb.is_repeat(t, 1, 4)
    with pytest.raises(IndexError):
        rb.is_repeat(t, 0, 1)
    with pytest.raises(IndexError):
        rb.oracle_llr(t, 12)
    with pytest.raises(IndexError):
        rb.oracle_all_lr(t, 0)
