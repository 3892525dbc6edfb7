"""Substring-search ground truth -- mirrors ``repeatscan.oracle`` (oracle.py:1-110).

Part of the reference's public API (``__init__.py:20``: ``is_repeat``,
``oracle_llr``, ``oracle_all_lr``), used by its tests and by the CLI
selftest.  Like the reference these are deliberately naive host functions
that work on the text bytes alone, independent of the suffix-array pipeline
(there is nothing data-parallel to move to the device: they exist to check
that pipeline on tiny inputs).  Results and exceptions match the reference:

* a substring is a repeat iff it occurs at >= 2 distinct starts, overlaps
  allowed (oracle.py:16-25);
* the longest repeat starting at i is monotone in its length
  (oracle.py:28-40), so it is found here by bisection over the length
  instead of the reference's descending scan -- same value;
* the answers covering k are the maximal-length intervals [i, i+L-1] with
  L <= longest repeat from i, in increasing start order (oracle.py:51-75).
"""

from __future__ import annotations

from paper_1501_06663_b200.query import NO_LR, LrAnswer
from paper_1501_06663_b200.text import Text

DEFAULT_SIZE_CAP = 4096


def _twice(s: bytes, sub: bytes) -> bool:
    first = s.find(sub)
    return first >= 0 and s.find(sub, first + 1) >= 0


def is_repeat(text: Text, start: int, length: int) -> bool:
    """True iff text[start, start+length-1] occurs at >= 2 starts (oracle.py:16-25)."""
    if length < 1 or start < 1 or start + length - 1 > text.n:
        raise IndexError(f"substring ({start},{length}) out of range for n={text.n}")
    s = text.to_bytes()
    return _twice(s, s[start - 1:start - 1 + length])


def _reach(s: bytes, i: int) -> int:
    """Longest L with s[i-1:i-1+L] a repeat (0 if none), by bisection."""
    lo, hi = 0, len(s) - i + 1  # invariant: lo is a repeat length (0 trivially), hi+1 is not
    while lo < hi:
        mid = (lo + hi + 1) // 2
        if _twice(s, s[i - 1:i - 1 + mid]):
            lo = mid
        else:
            hi = mid - 1
    return lo


def oracle_llr(text: Text, i: int) -> LrAnswer:
    """Longest repeat starting exactly at i (oracle.py:43-48)."""
    if not 1 <= i <= text.n:
        raise IndexError(f"position {i} out of range 1..{text.n}")
    r = _reach(text.to_bytes(), i)
    return LrAnswer(i, r) if r else NO_LR


def _covering(reach: list[int], k: int) -> list[LrAnswer]:
    best = max((r for i, r in enumerate(reach) if i >= 1 and i + r - 1 >= k), default=0)
    if best == 0:
        return []
    return [LrAnswer(i, best) for i in range(1, k + 1) if reach[i] >= best and i + best - 1 >= k]


def oracle_all_lr(text: Text, k: int) -> list[LrAnswer]:
    """All maximal-length repeats covering k, increasing start (oracle.py:51-75)."""
    if not 1 <= k <= text.n:
        raise IndexError(f"position {k} out of range 1..{text.n}")
    s = text.to_bytes()
    reach = [0] + [_reach(s, i) for i in range(1, k + 1)]
    return _covering(reach, k)


def oracle_leftmost_lr(text: Text, k: int) -> LrAnswer:
    """First of ``oracle_all_lr`` or NO_LR (oracle.py:78-80)."""
    hits = oracle_all_lr(text, k)
    return hits[0] if hits else NO_LR


def oracle_all_positions(text: Text, mode: str = "leftmost"):
    """Per-position brute-force answers for the whole text (oracle.py:83-110)."""
    s = text.to_bytes()
    reach = [0] + [_reach(s, i) for i in range(1, len(s) + 1)]
    out = []
    for k in range(1, len(s) + 1):
        hits = _covering(reach[:k + 1], k)
        if mode == "leftmost":
            out.append(hits[0] if hits else NO_LR)
        else:
            out.append(hits)
    return out
