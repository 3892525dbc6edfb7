"""Suffix array, rank array and LCP array -- mirrors ``repeatscan.suffixes``.

All public arrays are 1-based with slot 0 unused (suffixes.py:3-8):
``sa[1..n]``, ``rank[1..n]`` (inverse of sa), ``lcp[1..n+1]`` with zero
sentinels at 1 and n+1.  Construction runs on the B200: prefix doubling over
packed symbol keys with a hand-written LSD radix sort, rank inversion for
free (final group heads), Kasai/PLCP LCP (csrc/suffix_array.cu).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from paper_1501_06663_b200 import _native
from paper_1501_06663_b200.text import Text


@dataclass(frozen=True)
class SuffixStructures:
    sa: np.ndarray = field(repr=False)
    rank: np.ndarray = field(repr=False)
    lcp: np.ndarray = field(repr=False)

    @property
    def n(self) -> int:
        return int(self.sa.size) - 1


def _text_data(text) -> np.ndarray:
    data = text.data if hasattr(text, "data") else text
    return np.ascontiguousarray(data, dtype=np.uint8)


def build_suffix_structures(text: Text) -> SuffixStructures:
    """SA, rank and LCP arrays of the text (suffixes.py:56-66), built on device."""
    data = _text_data(text)
    n = int(data.size)
    if n == 0:
        z = np.zeros(1, dtype=np.int64)
        return SuffixStructures(sa=z, rank=z.copy(), lcp=np.zeros(2, dtype=np.int64))
    # every slot is written by the library (pads included); large arrays come
    # from the caching host pool (csrc/host_io.cu pipelines the D2H into them)
    sa = _native.out_array(n + 1, False)
    rank = _native.out_array(n + 1, False)
    lcp = _native.out_array(n + 2, False)
    if n > 0:
        ctx = _native.context()
        with ctx.lock:
            ctx.call("rs_suffix_structures", _native.u8(data), n, _native.i64(sa),
                     _native.i64(rank), _native.i64(lcp))
    return SuffixStructures(sa=sa, rank=rank, lcp=lcp)


def verify_suffix_structures(text: Text, s: SuffixStructures) -> bool:
    """Check every structural invariant by direct comparison (suffixes.py:69-103).

    Runs on device: permutation + inverse check, and per adjacent SA pair the
    exact common-prefix length and strict lexicographic order.
    """
    data = _text_data(text)
    n = int(data.size)
    sa = np.asarray(s.sa)
    rank = np.asarray(s.rank)
    lcp = np.asarray(s.lcp)
    if sa.size != n + 1 or rank.size != n + 1 or lcp.size != n + 2:
        return False
    if lcp[1] != 0 or lcp[n + 1] != 0:
        return False
    if n == 0:
        return True
    sa = np.ascontiguousarray(sa, dtype=np.int64)
    rank = np.ascontiguousarray(rank, dtype=np.int64)
    lcp = np.ascontiguousarray(lcp, dtype=np.int64)
    ok = np.zeros(1, dtype=np.int64)
    ctx = _native.context()
    with ctx.lock:
        ctx.call("rs_verify_structures", _native.u8(data), n, _native.i64(sa),
                 _native.i64(rank), _native.i64(lcp), _native.i64(ok))
    return bool(ok[0])
