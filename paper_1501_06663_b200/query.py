"""Longest-repeat queries per text position -- mirrors ``repeatscan.query``.

The batch entry points (``all_positions``, ``_leftmost_all_positions``,
``_all_all_positions``; query.py:171-239) run the whole path on the B200:
[suffix sort + LCP] -> raw LLR -> [compaction] -> per-position scan, with
results written on device directly in the reference int64 layouts and copied
back once.  The single-position helpers (query.py:40-127) are host-side
loops over the caller's arrays, exactly as in the reference:
they answer one k and have no data-parallel work to offload.
"""

from __future__ import annotations

import ctypes
from bisect import bisect_left
from dataclasses import dataclass, field
from typing import NamedTuple

import numpy as np

from paper_1501_06663_b200 import _native
from paper_1501_06663_b200.engine import ExecPolicy, _check_policy
from paper_1501_06663_b200.llr import CompactLlr
from paper_1501_06663_b200.suffixes import SuffixStructures
from paper_1501_06663_b200.text import Text

RAW = "raw"
COMPACT = "compact"
LEFTMOST = "leftmost"
ALL = "all"


class LrAnswer(NamedTuple):
    start: int
    length: int

    @property
    def exists(self) -> bool:
        return self.start != -1


NO_LR = LrAnswer(-1, 0)


def _check_pos(k: int, n: int) -> None:
    if not 1 <= k <= n:
        raise IndexError(f"position {k} out of range 1..{n}")


# ---- single-position queries (host side, query.py:45-127) ---------------------------

def leftmost_lr_raw(raw: np.ndarray, k: int) -> LrAnswer:
    """Leftmost longest repeat covering k via a leftward walk from k (Alg. 1)."""
    _check_pos(k, raw.size - 1)
    best = NO_LR
    i = k
    while i >= 1:
        if i + raw[i] - 1 < k:
            break
        if raw[i] >= best.length:
            best = LrAnswer(i, int(raw[i]))
        i -= 1
    return best


def all_lr_raw(raw: np.ndarray, k: int) -> list[LrAnswer]:
    """All longest repeats covering k, in increasing start order (Alg. 3)."""
    _check_pos(k, raw.size - 1)
    best_len = 0
    i = k
    while i >= 1 and i + raw[i] - 1 >= k:
        if raw[i] > best_len:
            best_len = int(raw[i])
        i -= 1
    if best_len == 0:
        return []
    hits = []
    i = k
    while i >= 1 and i + raw[i] - 1 >= k:
        if raw[i] == best_len:
            hits.append(LrAnswer(i, best_len))
        i -= 1
    hits.reverse()
    return hits


def find_start_index(c: CompactLlr, k: int) -> int | None:
    """Smallest 1-based entry index whose right end is >= k, or None."""
    if k < 1:
        raise IndexError(f"position {k} out of range")
    t = bisect_left(c.ends, k)
    return t + 1 if t < c.size else None


def _compact_window(c: CompactLlr, k: int, n: int | None):
    if n is not None:
        _check_pos(k, n)
    elif k < 1:
        raise IndexError(f"position {k} out of range")
    t = find_start_index(c, k)
    if t is None:
        return None
    idx = t - 1
    out = []
    while idx < c.size and c.starts[idx] <= k:
        out.append(idx)
        idx += 1
    return out


def leftmost_lr_compact(c: CompactLlr, k: int, n: int | None = None) -> LrAnswer:
    """Leftmost longest repeat covering k via binary search + rightward walk (Alg. 2)."""
    window = _compact_window(c, k, n)
    best = NO_LR
    for idx in window or ():
        if c.lengths[idx] > best.length:
            best = LrAnswer(int(c.starts[idx]), int(c.lengths[idx]))
    return best


def all_lr_compact(c: CompactLlr, k: int, n: int | None = None) -> list[LrAnswer]:
    """All longest repeats covering k from the compact array (Alg. 4)."""
    window = _compact_window(c, k, n)
    if not window:
        return []
    best_len = max(int(c.lengths[idx]) for idx in window)
    if best_len == 0:
        return []
    return [LrAnswer(int(c.starts[idx]), best_len) for idx in window
            if c.lengths[idx] == best_len]


# ---- batch answers (query.py:130-168) -----------------------------------------------

@dataclass(frozen=True)
class LeftmostAnswers:
    """Leftmost answer per position; starts/lengths are 1-based padded."""

    starts: np.ndarray = field(repr=False)
    lengths: np.ndarray = field(repr=False)

    @property
    def n(self) -> int:
        return int(self.starts.size) - 1

    def answer(self, k: int) -> LrAnswer:
        _check_pos(k, self.n)
        return LrAnswer(int(self.starts[k]), int(self.lengths[k]))


@dataclass(frozen=True)
class AllAnswers:
    """All tied answers per position in CSR layout.

    Position k's starts live in flat_starts[offsets[k]:offsets[k+1]], all
    with the common length lengths[k].
    """

    lengths: np.ndarray = field(repr=False)
    offsets: np.ndarray = field(repr=False)
    flat_starts: np.ndarray = field(repr=False)

    @property
    def n(self) -> int:
        return int(self.lengths.size) - 1

    def answers(self, k: int) -> list[LrAnswer]:
        _check_pos(k, self.n)
        length = int(self.lengths[k])
        if length == 0:
            return []
        lo, hi = int(self.offsets[k]), int(self.offsets[k + 1])
        return [LrAnswer(int(s), length) for s in self.flat_starts[lo:hi]]


# ---- device pipeline ------------------------------------------------------------------

def _fetch(ctx: _native.Context, mode: str, n: int, total: int, pinned: bool):
    if mode == LEFTMOST:
        starts = _native.out_array(n + 1, pinned)
        lengths = _native.out_array(n + 1, pinned)
        ctx.call("rs_fetch_leftmost", _native.i64(starts), _native.i64(lengths))
        return LeftmostAnswers(starts=starts, lengths=lengths)
    lengths = _native.out_array(n + 1, pinned)
    offsets = _native.out_array(n + 2, pinned)
    flat = _native.out_array(total, pinned)
    ctx.call("rs_fetch_all", _native.i64(lengths), _native.i64(offsets), _native.i64(flat))
    return AllAnswers(lengths=lengths, offsets=offsets, flat_starts=flat)


def _run(ctx: _native.Context, mode: str, path: str, n: int, pinned: bool):
    total = np.zeros(1, dtype=np.int64)
    ctx.call("rs_query", _native.MODE[mode], _native.PATH[path], _native.i64(total))
    return _fetch(ctx, mode, n, int(total[0]), pinned)


def _load_candidates(ctx: _native.Context, n: int, path: str, raw, c) -> None:
    if path == RAW:
        raw = np.ascontiguousarray(raw, dtype=np.int64)
        if raw.size != n + 1:
            raise ValueError(f"raw array has {raw.size} slots, expected n + 1 = {n + 1}")
        ctx.call("rs_set_raw", _native.i64(raw), n)
    else:
        if c is None:
            raise ValueError("compact path needs the compact LLR array")
        starts = np.ascontiguousarray(c.starts, dtype=np.int64)
        lengths = np.ascontiguousarray(c.lengths, dtype=np.int64)
        ctx.call("rs_set_compact", _native.i64(starts), _native.i64(lengths), int(starts.size), n)


def _leftmost_all_positions(n: int, path: str, raw: np.ndarray, c: CompactLlr | None,
                            policy: ExecPolicy | None, pinned: bool = False) -> LeftmostAnswers:
    """query.py:171-184 on device."""
    _check_policy(policy)
    ctx = _native.context()
    with ctx.lock:
        _load_candidates(ctx, n, path, raw, c)
        return _run(ctx, LEFTMOST, path, n, pinned)


def _all_all_positions(n: int, path: str, raw: np.ndarray, c: CompactLlr | None,
                       policy: ExecPolicy | None, pinned: bool = False) -> AllAnswers:
    """query.py:187-215 on device (single-pass count/scan/fill)."""
    _check_policy(policy)
    ctx = _native.context()
    with ctx.lock:
        _load_candidates(ctx, n, path, raw, c)
        return _run(ctx, ALL, path, n, pinned)


def all_positions(
    text: Text,
    mode: str = LEFTMOST,
    path: str = COMPACT,
    policy: ExecPolicy | None = None,
    structures: SuffixStructures | None = None,
    *,
    pinned: bool = False,
) -> LeftmostAnswers | AllAnswers:
    """Answers for every position k = 1..n (query.py:218-239).

    With ``structures=None`` the whole path -- suffix sort, LCP, raw LLR,
    compaction, scan -- runs on the device from the text bytes.  Identical
    output for every path/policy combination.  ``pinned=True`` returns arrays
    backed by a pooled page-locked host buffer (faster D2H for large n).
    """
    if mode not in (LEFTMOST, ALL):
        raise ValueError(f"unknown mode {mode!r}")
    if path not in (RAW, COMPACT):
        raise ValueError(f"unknown path {path!r}")
    _check_policy(policy)
    ctx = _native.context()
    with ctx.lock:
        if structures is None:
            data = np.ascontiguousarray(text.data, dtype=np.uint8)
            n = int(data.size)
            ctx.call("rs_set_text", _native.u8(data), n)
        else:
            n = int(structures.sa.size) - 1
            rank = np.ascontiguousarray(structures.rank, dtype=np.int64)
            lcp = np.ascontiguousarray(structures.lcp, dtype=np.int64)
            if rank.size != n + 1 or lcp.size != n + 2:
                raise ValueError("structures arrays have inconsistent sizes")
            ctx.call("rs_set_structures", None, _native.i64(rank), _native.i64(lcp), n)
        return _run(ctx, mode, path, n, pinned)


def count_wrong_answers(c: CompactLlr, n: int, all_answers: AllAnswers | None = None,
                        leftmost: LeftmostAnswers | None = None) -> int:
    """Number of positions whose answers disagree with the compact entries
    ``c`` under the reference's Algorithm 4 as written (binary search of the
    first covering entry + forward walk, ``_kernels_numba.py:74-85, 158-195``),
    checked on device by a kernel that shares no code with the scan kernels.
    Not part of the reference API: a parity property for large inputs."""
    ctx = _native.context()
    starts = np.ascontiguousarray(c.starts, dtype=np.int64)
    lengths = np.ascontiguousarray(c.lengths, dtype=np.int64)
    bad = np.zeros(1, np.int64)
    null = ctypes.POINTER(ctypes.c_int64)()
    a = (null, null, null, 0) if all_answers is None else (
        _native.i64(all_answers.lengths), _native.i64(all_answers.offsets),
        _native.i64(all_answers.flat_starts), int(all_answers.flat_starts.size))
    lm = (null, null) if leftmost is None else (_native.i64(leftmost.starts),
                                               _native.i64(leftmost.lengths))
    with ctx.lock:
        ctx.call("rs_check_answers", _native.i64(starts), _native.i64(lengths), int(starts.size),
                 int(n), *a, *lm, _native.i64(bad))
    return int(bad[0])
