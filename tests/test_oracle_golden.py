"""Pin the CPU oracle (oracle/repeatscan_oracle.c) to the reference itself.

golden_small.npz / digests.json were produced by running the reference
package (tests/golden/make_golden.py); the hard-coded vectors below are the
reference's own known-answer tests (file:line cited per test).
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from conftest import digest, golden_cases, golden_digests


def test_oracle_builds_and_loads():
    oracle.build()
    assert oracle.max_threads() >= 1


def test_mississippi_table1():
    # test_suffixes.py:14-17, Table 1
    sa, rank, lcp = oracle.build_suffix_structures(np.frombuffer(b"mississippi", np.uint8))
    assert sa[1:].tolist() == [11, 8, 5, 2, 1, 10, 9, 7, 4, 6, 3]
    assert lcp[1:].tolist() == [0, 1, 1, 4, 0, 0, 1, 0, 2, 1, 3, 0]
    raw = oracle.build_raw_llr(rank, lcp)
    assert raw[1:].tolist() == [0, 4, 3, 2, 4, 3, 2, 1, 1, 1, 1]  # test_llr.py:36-37
    s, l = oracle.build_compact_llr(raw)
    assert list(zip(s.tolist(), l.tolist())) == [(2, 4), (5, 4), (9, 1), (10, 1), (11, 1)]
    st, ln = oracle.leftmost_all_positions(11, "compact", raw, (s, l))
    want = [(-1, 0), (2, 4), (2, 4), (2, 4), (2, 4), (5, 4), (5, 4), (5, 4), (9, 1),
            (10, 1), (11, 1)]  # test_query.py:119-127
    assert list(zip(st[1:].tolist(), ln[1:].tolist())) == want


def test_figure4_compaction():
    # test_acceptance.py:83-91
    raw = np.array([0, 3, 2, 1, 1, 3, 2, 1, 1], np.int64)
    flags = oracle.compute_flags(raw)
    assert flags[1:].tolist() == [1, 0, 0, 1, 1, 0, 0, 1]
    assert oracle.prefix_sum(flags)[1:].tolist() == [1, 1, 1, 2, 3, 3, 3, 4]
    s, l = oracle.build_compact_llr(raw)
    assert list(zip(s.tolist(), l.tolist())) == [(1, 3), (4, 1), (5, 3), (8, 1)]


def test_abcabcddbca_all_ties():
    # test_acceptance.py:94-99
    for path in ("raw", "compact"):
        lengths, offsets, flat = oracle.all_positions(
            np.frombuffer(b"abcabcddbca", np.uint8), mode="all", path=path)
        assert flat[offsets[2]:offsets[3]].tolist() == [1, 2]
        assert lengths[2] == 3


def test_edge_cases():
    # "" and aaaa
    st, ln = oracle.all_positions(np.zeros(0, np.uint8))
    assert st.tolist() == [-1] and ln.tolist() == [0]
    lengths, offsets, flat = oracle.all_positions(np.zeros(0, np.uint8), mode="all")
    assert offsets.tolist() == [0, 0]
    a4 = np.frombuffer(b"aaaa", np.uint8)
    st, ln = oracle.all_positions(a4)
    assert st.tolist() == [-1, 1, 1, 1, 2]
    lengths, offsets, flat = oracle.all_positions(a4, mode="all")
    assert offsets.tolist() == [0, 0, 1, 3, 5, 6] and flat.tolist() == [1, 1, 2, 1, 2, 2]


@pytest.mark.parametrize("workers", [1, 3])
def test_oracle_matches_reference_golden(workers):
    for c in golden_cases():
        sa, rank, lcp = oracle.build_suffix_structures(c.data)
        assert np.array_equal(sa, c.sa), c
        assert np.array_equal(rank, c.rank), c
        assert np.array_equal(lcp, c.lcp), c
        raw = oracle.build_raw_llr(rank, lcp, workers)
        assert np.array_equal(raw, c.raw), c
        assert np.array_equal(oracle.compute_flags(raw), c.flags), c
        assert np.array_equal(oracle.prefix_sum(c.flags, workers), c.ps), c
        s, l = oracle.build_compact_llr(raw, workers)
        assert np.array_equal(s, c.c_starts) and np.array_equal(l, c.c_lengths), c
        s2, l2 = oracle.compact_sequential(raw)
        assert np.array_equal(s2, c.c_starts) and np.array_equal(l2, c.c_lengths), c
        for path in ("raw", "compact"):
            cc = (s, l) if path == "compact" else None
            st, ln = oracle.leftmost_all_positions(c.n, path, raw, cc, workers)
            assert np.array_equal(st, c.l_starts) and np.array_equal(ln, c.l_lengths), (c, path)
            al, ao, af = oracle.all_all_positions(c.n, path, raw, cc, workers)
            assert np.array_equal(al, c.a_lengths), (c, path)
            assert np.array_equal(ao, c.a_offsets), (c, path)
            assert np.array_equal(af, c.a_flat), (c, path)


def test_brute_force_restatement_matches_golden():
    # oracle.py:78-104 restated; small cases only
    for c in golden_cases()[:400]:
        if c.n > 40:
            continue
        want_left = oracle.brute_all_positions(c.data.tobytes(), "leftmost")
        want_all = oracle.brute_all_positions(c.data.tobytes(), "all")
        for k in range(1, c.n + 1):
            assert (int(c.l_starts[k]), int(c.l_lengths[k])) == want_left[k - 1]
            lo, hi = int(c.a_offsets[k]), int(c.a_offsets[k + 1])
            got = [(int(x), int(c.a_lengths[k])) for x in c.a_flat[lo:hi]]
            assert got == want_all[k - 1]


@pytest.mark.parametrize("name", ["acgt_1e6_seed99", "C1_2p20", "C5_shape_2p20"])
def test_oracle_matches_reference_digests(name):
    from paper_1501_06663_b200 import workloads  # noqa: F401  (used by eval)
    rec = golden_digests()[name]
    data = eval(rec["expr"])
    sa, rank, lcp = oracle.build_suffix_structures(data)
    assert digest(sa) == rec["sa"] and digest(rank) == rec["rank"] and digest(lcp) == rec["lcp"]
    raw = oracle.build_raw_llr(rank, lcp, 0)
    assert digest(raw) == rec["raw"]
    s, l = oracle.build_compact_llr(raw, 0)
    assert digest(s) == rec["c_starts"] and digest(l) == rec["c_lengths"]
    al, ao, af = oracle.all_all_positions(data.size, "compact", raw, (s, l), 0)
    assert digest(al) == rec["a_lengths"] and digest(ao) == rec["a_offsets"]
    assert digest(af) == rec["a_flat"]
    st, ln = oracle.leftmost_all_positions(data.size, "compact", raw, (s, l), 0)
    assert digest(st) == rec["l_starts"] and digest(ln) == rec["l_lengths"]


def test_oracle_walk_stats_match_reference_golden():
    # stats.py:30-55 restated in oracle/ vs the reference's own arrays
    for c in golden_cases():
        assert np.array_equal(oracle.walk_steps_raw(c.raw), c.w_raw), c
        assert np.array_equal(oracle.walk_steps_compact(c.c_starts, c.c_lengths, c.n), c.w_comp), c


@pytest.mark.parametrize("name", ["acgt_1e6_seed99", "C2_shape_2p21", "C4_shape_2p21",
                                  "C5_shape_2p20", "periodic_2p20"])
def test_oracle32_matches_reference_digests(name):
    """oracle/oracle32.c (the u32 restatement that produced the committed 1 GiB
    C5 digests, tests/golden/make_fullsize.py) reproduces every reference
    digest, m, T and max LLR of the 1-2 Mi reference digest set."""
    from paper_1501_06663_b200 import workloads  # noqa: F401  (used by eval)
    rec = golden_digests()[name]
    got = oracle.digests32(eval(rec["expr"]), chunk=1 << 18)
    for key, val in got.items():
        if key in rec:
            assert val == rec[key], (name, key)
    assert {"sa", "lcp", "raw", "c_starts", "l_starts", "a_offsets", "a_flat", "T"} <= set(got)


def test_oracle32_matches_oracle_small(rng):
    """Same digests as the int64 oracle on small arbitrary-byte inputs."""
    for _ in range(30):
        n = int(rng.integers(1, 3000))
        sigma = int(rng.integers(1, 257))
        alpha = rng.choice(256, size=sigma, replace=False).astype(np.uint8)
        data = rng.choice(alpha, size=n)
        got = oracle.digests32(data, chunk=int(rng.integers(1, 600)))
        sa, rank, lcp = oracle.build_suffix_structures(data)
        raw = oracle.build_raw_llr(rank, lcp, 0)
        s, l = oracle.build_compact_llr(raw, 0)
        al, ao, af = oracle.all_all_positions(n, "compact", raw, (s, l), 0)
        st, ln = oracle.leftmost_all_positions(n, "compact", raw, (s, l), 0)
        want = {"sa": sa, "rank": rank, "lcp": lcp, "raw": raw, "c_starts": s, "c_lengths": l,
                "a_lengths": al, "a_offsets": ao, "a_flat": af, "l_starts": st, "l_lengths": ln}
        for key, arr in want.items():
            assert got[key] == digest(arr), (n, key)


@pytest.mark.parametrize("workers", [3, 8])
def test_threaded_structures_match_reference(workers):
    """or_build_structures_par (the CPU baseline's structures= builder) gives the
    reference's arrays: golden cases and the 1 Mi reference digests."""
    from paper_1501_06663_b200 import workloads  # noqa: F401  (used by eval)
    for c in golden_cases():
        sa, rank, lcp = oracle.build_suffix_structures(c.data, workers=workers)
        assert np.array_equal(sa, c.sa) and np.array_equal(rank, c.rank), c
        assert np.array_equal(lcp, c.lcp), c
    for name in ("C1_2p20", "C5_shape_2p20"):
        rec = golden_digests()[name]
        sa, rank, lcp = oracle.build_suffix_structures(eval(rec["expr"]), workers=workers)
        assert (digest(sa), digest(rank), digest(lcp)) == (rec["sa"], rec["rank"], rec["lcp"])
