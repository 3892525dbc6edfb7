"""Walk-step statistics -- mirrors ``repeatscan.stats`` (stats.py:1-76).

A step is one covering LLR entry examined by a query walk; positions without
a longest repeat contribute nothing (stats.py:1-12).  The steps at k equal the
number of candidates covering k, which the device computes as the window size
of the scan kernel's per-tile window bounds (csrc/scan_query.cu ``k_steps``):
raw: k - #{i : i + raw[i] - 1 < k}; compact: max(upto(k) - below(k), 0).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from paper_1501_06663_b200 import _native
from paper_1501_06663_b200.llr import CompactLlr


@dataclass(frozen=True)
class WalkStats:
    path: str
    min_steps: int
    max_steps: int
    avg_steps: float
    positions: int  # positions where a longest repeat exists


def _stats(path: str, st: np.ndarray) -> WalkStats:
    count = int(st[3])
    if count == 0:
        return WalkStats(path=path, min_steps=0, max_steps=0, avg_steps=0.0, positions=0)
    return WalkStats(path=path, min_steps=int(st[0]), max_steps=int(st[1]),
                     avg_steps=float(int(st[2]) / count), positions=count)


def _load_raw(ctx, raw) -> int:
    raw = np.ascontiguousarray(raw, dtype=np.int64)
    n = int(raw.size) - 1
    ctx.call("rs_set_raw", _native.i64(raw), n)
    return n


def _load_compact(ctx, c: CompactLlr, n: int) -> None:
    starts = np.ascontiguousarray(c.starts, dtype=np.int64)
    lengths = np.ascontiguousarray(c.lengths, dtype=np.int64)
    ctx.call("rs_set_compact", _native.i64(starts), _native.i64(lengths), int(starts.size), int(n))


def walk_steps_raw(raw: np.ndarray) -> np.ndarray:
    """Steps per position for the raw-array walk (1-based padded, 0 = no LR)."""
    n = int(np.asarray(raw).size) - 1
    steps = np.zeros(max(n, 0) + 1, dtype=np.int64)
    if n <= 0:
        return steps
    st = np.zeros(4, np.int64)
    ctx = _native.context()
    with ctx.lock:
        _load_raw(ctx, raw)
        ctx.call("rs_walk_steps", 0, _native.i64(steps), _native.i64(st))
    return steps


def walk_steps_compact(c: CompactLlr, n: int) -> np.ndarray:
    """Steps per position for the compact-array walk."""
    steps = np.zeros(n + 1, dtype=np.int64)
    if n == 0 or c.size == 0:
        return steps
    st = np.zeros(4, np.int64)
    ctx = _native.context()
    with ctx.lock:
        _load_compact(ctx, c, n)
        ctx.call("rs_walk_steps", 1, _native.i64(steps), _native.i64(st))
    return steps


def summarize_steps(steps: np.ndarray, path: str) -> WalkStats:
    steps = np.ascontiguousarray(steps, dtype=np.int64)
    st = np.zeros(4, np.int64)
    ctx = _native.context()
    with ctx.lock:
        ctx.call("rs_summarize_steps", _native.i64(steps), int(steps.size), _native.i64(st))
    return _stats(path, st)


def compute_walk_stats(raw: np.ndarray, c: CompactLlr, path: str) -> WalkStats:
    if path not in ("raw", "compact"):
        raise ValueError(f"unknown path {path!r}")
    n = int(np.asarray(raw).size) - 1
    if n <= 0 or (path == "compact" and c.size == 0):
        return WalkStats(path=path, min_steps=0, max_steps=0, avg_steps=0.0, positions=0)
    st = np.zeros(4, np.int64)
    ctx = _native.context()
    with ctx.lock:
        if path == "raw":
            _load_raw(ctx, raw)
            ctx.call("rs_walk_steps", 0, None, _native.i64(st))
        else:
            _load_compact(ctx, c, n)
            ctx.call("rs_walk_steps", 1, None, _native.i64(st))
    return _stats(path, st)
