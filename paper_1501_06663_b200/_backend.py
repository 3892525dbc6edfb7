"""The reference's operator-level API on the device -- mirrors ``repeatscan._backend``.

The reference drives its data-parallel path through ``_backend.kernels``
(``_backend.py:10-34``): eleven chunk kernels ``(lo, hi, inputs..., outputs...)``
over 1-based ``[lo, hi)`` that fill caller-allocated arrays in place
(``_kernels_numba.py:15-195``), called by ``engine.parallel_for`` per chunk.
``kernels`` here has the same names, arguments and in-place semantics, and
every value is computed by the CUDA library: a call runs the whole-array
device operation and writes the caller's ``[lo, hi)`` slice.  That keeps the
operator contract exact (any chunking gives the reference's arrays) while
the batch entry points (``all_positions``, ``build_raw_llr`` ...) remain the
fast path -- they never go through per-chunk calls.

There is one backend (``BACKEND``); no environment selector, no CPU fallback
(the reference's numba/numpy selection is out of scope).
"""

from __future__ import annotations

from bisect import bisect_left
from types import SimpleNamespace

import numpy as np

BACKEND = "cuda-sm_100a"


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def kasai_lcp(data, sa, rank, lcp) -> None:
    """_kernels_numba.py:15-30: lcp[2..n] of the adjacent suffixes of ``sa``.

    Built on the device from the text; the given ``sa`` / ``rank`` must be the
    text's suffix array and its inverse (ValueError otherwise)."""
    from paper_1501_06663_b200.suffixes import build_suffix_structures
    n = int(np.asarray(sa).size) - 1
    if n < 2:
        return
    s = build_suffix_structures(np.ascontiguousarray(data, dtype=np.uint8))
    if not (np.array_equal(s.sa, _i64(sa)) and np.array_equal(s.rank, _i64(rank))):
        raise ValueError("sa / rank are not the suffix array of the text and its inverse")
    lcp[2:n + 1] = s.lcp[2:n + 1]


def fill_raw_llr(lo, hi, rank, lcp, out) -> None:
    """_kernels_numba.py:33-38 over [lo, hi)."""
    from paper_1501_06663_b200.llr import build_raw_llr
    if hi > lo:
        rank = _i64(rank)
        s = SimpleNamespace(rank=rank, lcp=_i64(lcp), n=int(rank.size) - 1)
        out[lo:hi] = build_raw_llr(s)[lo:hi]


def fill_flags(lo, hi, llr, out) -> None:
    """_kernels_numba.py:41-46 over [lo, hi)."""
    from paper_1501_06663_b200.llr import compute_flags
    if hi > lo:
        out[lo:hi] = compute_flags(_i64(llr))[lo:hi]


def scatter_chunk(lo, hi, llr, flags, ps, starts, lengths) -> None:
    """_kernels_numba.py:49-55: the entries of the flagged slots in [lo, hi)."""
    from paper_1501_06663_b200.llr import scatter_compact
    if hi <= lo:
        return
    c = scatter_compact(_i64(llr), _i64(flags), _i64(ps))
    a, b = int(ps[lo - 1]) if lo > 0 else 0, int(ps[hi - 1])
    starts[a:b] = c.starts[a:b]
    lengths[a:b] = c.lengths[a:b]


def compact_sequential(llr, starts, lengths) -> int:
    """_kernels_numba.py:58-71; returns the number of entries written."""
    from paper_1501_06663_b200.llr import compact_llr_sequential
    c = compact_llr_sequential(_i64(llr))
    m = int(c.size)
    starts[:m] = c.starts
    lengths[:m] = c.lengths
    return m


def _first_end_at_or_after(ends, k) -> int:
    """_kernels_numba.py:74-85 (a single search: host bisect, as the reference's
    single-position helpers; the batch scans need no search at all)."""
    return bisect_left(ends, k)


def _compact(starts, lengths):
    from paper_1501_06663_b200.llr import CompactLlr
    return CompactLlr.from_arrays(_i64(starts), _i64(lengths))


def leftmost_raw_chunk(lo, hi, llr, out_start, out_len) -> None:
    """_kernels_numba.py:88-102 over [lo, hi)."""
    from paper_1501_06663_b200.query import _leftmost_all_positions
    if hi <= lo:
        return
    llr = _i64(llr)
    res = _leftmost_all_positions(llr.size - 1, "raw", llr, None, None)
    out_start[lo:hi] = res.starts[lo:hi]
    out_len[lo:hi] = res.lengths[lo:hi]


def leftmost_compact_chunk(lo, hi, starts, lengths, ends, out_start, out_len) -> None:
    """_kernels_numba.py:105-118 over [lo, hi) (n = out_start.size - 1)."""
    from paper_1501_06663_b200.query import _leftmost_all_positions
    if hi <= lo:
        return
    res = _leftmost_all_positions(int(out_start.size) - 1, "compact", None, _compact(starts, lengths), None)
    out_start[lo:hi] = res.starts[lo:hi]
    out_len[lo:hi] = res.lengths[lo:hi]


def _all(n, path, llr, c):
    from paper_1501_06663_b200.query import _all_all_positions
    return _all_all_positions(n, path, llr, c, None)


def all_raw_count_chunk(lo, hi, llr, out_len, out_cnt) -> None:
    """_kernels_numba.py:121-138 over [lo, hi): max length and tie count."""
    if hi <= lo:
        return
    llr = _i64(llr)
    res = _all(llr.size - 1, "raw", llr, None)
    out_len[lo:hi] = res.lengths[lo:hi]
    out_cnt[lo:hi] = np.diff(res.offsets)[lo:hi]


def all_raw_fill_chunk(lo, hi, llr, best_len, offsets, flat_starts) -> None:
    """_kernels_numba.py:141-155: tie starts of [lo, hi) into their CSR blocks."""
    if hi <= lo:
        return
    llr = _i64(llr)
    res = _all(llr.size - 1, "raw", llr, None)
    a, b = int(offsets[lo]), int(offsets[hi])
    flat_starts[a:b] = res.flat_starts[int(res.offsets[lo]):int(res.offsets[hi])]


def all_compact_count_chunk(lo, hi, starts, lengths, ends, out_len, out_cnt) -> None:
    """_kernels_numba.py:158-177 over [lo, hi) (n = out_len.size - 1)."""
    if hi <= lo:
        return
    res = _all(int(out_len.size) - 1, "compact", None, _compact(starts, lengths))
    out_len[lo:hi] = res.lengths[lo:hi]
    out_cnt[lo:hi] = np.diff(res.offsets)[lo:hi]


def all_compact_fill_chunk(lo, hi, starts, lengths, ends, best_len, offsets, flat_starts) -> None:
    """_kernels_numba.py:180-195 over [lo, hi) (n = best_len.size - 1)."""
    if hi <= lo:
        return
    res = _all(int(best_len.size) - 1, "compact", None, _compact(starts, lengths))
    a, b = int(offsets[lo]), int(offsets[hi])
    flat_starts[a:b] = res.flat_starts[int(res.offsets[lo]):int(res.offsets[hi])]


kernels = SimpleNamespace(
    kasai_lcp=kasai_lcp, fill_raw_llr=fill_raw_llr, fill_flags=fill_flags, scatter_chunk=scatter_chunk,
    compact_sequential=compact_sequential, _first_end_at_or_after=_first_end_at_or_after,
    leftmost_raw_chunk=leftmost_raw_chunk, leftmost_compact_chunk=leftmost_compact_chunk,
    all_raw_count_chunk=all_raw_count_chunk, all_raw_fill_chunk=all_raw_fill_chunk,
    all_compact_count_chunk=all_compact_count_chunk, all_compact_fill_chunk=all_compact_fill_chunk,
)

__all__ = ["kernels", "BACKEND"]
