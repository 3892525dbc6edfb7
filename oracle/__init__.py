"""CPU parity oracle for the longest-repeat path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference leg may import this package, and only as the checker or the timed
CPU baseline -- never as the thing measured or shipped.  The product package
``paper_1501_06663_b200`` never imports it.

Two layers:

* :mod:`oracle.repeatscan_oracle` (C, built by ``oracle/Makefile`` into
  ``oracle/liboracle.so``): a line-by-line restatement of the reference
  ``repeatscan`` kernels (``_kernels_numba.py``), its prefix-doubling suffix
  sort (``suffixes.py:31-53``) and its engine (``engine.py:43-110``).  Pinned
  against golden vectors produced by the reference itself
  (``tests/golden/make_golden.py``), see ``tests/test_oracle_golden.py``.
* :func:`brute_all_positions` -- the reference's brute-force substring oracle
  (``oracle.py:78-104``) restated in pure Python, for tiny inputs only.

All arrays use the reference layouts: int64, 1-based with a pad slot 0.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "liboracle.so"
_lib = None

_I64P = ctypes.POINTER(ctypes.c_int64)
_U8P = ctypes.POINTER(ctypes.c_uint8)


def build() -> Path:
    """Compile the C restatement (gcc + OpenMP) in place."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        build()
    lib = ctypes.CDLL(str(_LIB_PATH))
    i64, c_int = ctypes.c_int64, ctypes.c_int
    sig = {
        "or_suffix_array_0based": (c_int, [_U8P, i64, _I64P]),
        "or_build_structures": (c_int, [_U8P, i64, _I64P, _I64P, _I64P]),
        "or_build_structures_par": (c_int, [_U8P, i64, _I64P, _I64P, _I64P, c_int]),
        "or_kasai_lcp": (None, [_U8P, _I64P, _I64P, _I64P, i64]),
        "or_fill_raw_llr": (None, [i64, i64, _I64P, _I64P, _I64P]),
        "or_fill_flags": (None, [i64, i64, _I64P, _I64P]),
        "or_scatter_chunk": (None, [i64, i64, _I64P, _I64P, _I64P, _I64P, _I64P]),
        "or_compact_sequential": (i64, [_I64P, i64, _I64P, _I64P]),
        "or_parallel_scan": (None, [_I64P, i64, _I64P, c_int]),
        "or_build_raw_llr_par": (None, [_I64P, _I64P, i64, _I64P, c_int]),
        "or_build_compact_llr_par": (i64, [_I64P, i64, _I64P, _I64P, c_int]),
        "or_leftmost_all_par": (
            None, [i64, c_int, _I64P, _I64P, _I64P, _I64P, i64, _I64P, _I64P, c_int]),
        "or_all_count_par": (
            i64, [i64, c_int, _I64P, _I64P, _I64P, _I64P, i64, _I64P, _I64P, c_int]),
        "or_all_fill_par": (
            None, [i64, c_int, _I64P, _I64P, _I64P, _I64P, i64, _I64P, _I64P, _I64P, c_int]),
        "or_max_threads": (c_int, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _p(a: np.ndarray):
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(_I64P)


def _u8(a: np.ndarray):
    return a.ctypes.data_as(_U8P)


def max_threads() -> int:
    return int(_load().or_max_threads())


def _workers(workers: int | None) -> int:
    return int(workers) if workers else (os.cpu_count() or 1)


# -- suffixes.py:56-66 --------------------------------------------------------
def build_suffix_structures(data: np.ndarray, workers: int = 1):
    """(sa, rank, lcp) int64 1-based padded, as ``build_suffix_structures``.

    workers == 1: the line-by-line restatement (suffixes.py:31-66).
    workers > 1: the threaded variant (or_build_structures_par: radix-sorted
    prefix doubling + chunked Kasai, identical output) used to give the CPU
    baseline its ``structures=`` input at full size."""
    data = np.ascontiguousarray(data, dtype=np.uint8)
    n = int(data.size)
    sa = np.zeros(n + 1, np.int64)
    rank = np.zeros(n + 1, np.int64)
    lcp = np.zeros(n + 2, np.int64)
    if n and workers > 1:
        rc = _load().or_build_structures_par(_u8(data), n, _p(sa), _p(rank), _p(lcp), int(workers))
        if rc != 0:
            raise MemoryError("oracle suffix sort out of memory")
    elif n:
        rc = _load().or_build_structures(_u8(data), n, _p(sa), _p(rank), _p(lcp))
        if rc != 0:
            raise MemoryError("oracle suffix sort out of memory")
    return sa, rank, lcp


# -- llr.py ------------------------------------------------------------------
def build_raw_llr(rank: np.ndarray, lcp: np.ndarray, workers: int | None = 1) -> np.ndarray:
    n = int(rank.size) - 1
    out = np.zeros(n + 1, np.int64)
    _load().or_build_raw_llr_par(_p(rank), _p(lcp), n, _p(out), _workers(workers))
    return out


def compute_flags(raw: np.ndarray) -> np.ndarray:
    n = int(raw.size) - 1
    out = np.zeros(n + 1, np.int64)
    if n:
        _load().or_fill_flags(1, n + 1, _p(raw), _p(out))
    return out


def prefix_sum(flags: np.ndarray, workers: int | None = 1) -> np.ndarray:
    ps = np.zeros_like(flags)
    n = int(flags.size) - 1
    if n > 0:
        src = np.ascontiguousarray(flags[1:])
        dst = np.zeros(n, np.int64)
        _load().or_parallel_scan(_p(src), n, _p(dst), _workers(workers))
        ps[1:] = dst
    return ps


def compact_sequential(raw: np.ndarray):
    n = int(raw.size) - 1
    s = np.empty(max(n, 1), np.int64)
    l = np.empty(max(n, 1), np.int64)
    m = int(_load().or_compact_sequential(_p(raw), n, _p(s), _p(l)))
    return s[:m].copy(), l[:m].copy()


def build_compact_llr(raw: np.ndarray, workers: int | None = 1):
    """(starts, lengths) 0-based arrays of size m via flag/scan/scatter."""
    n = int(raw.size) - 1
    s = np.empty(max(n, 1), np.int64)
    l = np.empty(max(n, 1), np.int64)
    m = int(_load().or_build_compact_llr_par(_p(raw), n, _p(s), _p(l), _workers(workers)))
    return s[:m].copy(), l[:m].copy()


# -- query.py:171-215 ----------------------------------------------------------
_PATHS = {"raw": 0, "compact": 1}


def _compact_args(c):
    if c is None:
        z = np.zeros(1, np.int64)
        return z, z, z, 0
    s, l = c
    s = np.ascontiguousarray(s, dtype=np.int64)
    l = np.ascontiguousarray(l, dtype=np.int64)
    e = s + l - 1
    m = int(s.size)
    if m == 0:
        z = np.zeros(1, np.int64)
        return z, z, z, 0
    return s, l, e, m


def leftmost_all_positions(n: int, path: str, raw: np.ndarray, c=None, workers: int | None = 1):
    """(starts, lengths), each int64[n+1]; starts[0] = -1."""
    starts = np.full(n + 1, -1, np.int64)
    lengths = np.zeros(n + 1, np.int64)
    cs, cl, ce, m = _compact_args(c)
    _load().or_leftmost_all_par(n, _PATHS[path], _p(raw), _p(cs), _p(cl), _p(ce), m,
                                _p(starts), _p(lengths), _workers(workers))
    return starts, lengths


def all_all_positions(n: int, path: str, raw: np.ndarray, c=None, workers: int | None = 1):
    """(lengths int64[n+1], offsets int64[n+2], flat_starts int64[T])."""
    lengths = np.zeros(n + 1, np.int64)
    offsets = np.zeros(n + 2, np.int64)
    cs, cl, ce, m = _compact_args(c)
    lib = _load()
    w = _workers(workers)
    total = int(lib.or_all_count_par(n, _PATHS[path], _p(raw), _p(cs), _p(cl), _p(ce), m,
                                     _p(lengths), _p(offsets), w))
    flat = np.empty(total, np.int64)
    if total:
        lib.or_all_fill_par(n, _PATHS[path], _p(raw), _p(cs), _p(cl), _p(ce), m,
                            _p(lengths), _p(offsets), _p(flat), w)
    return lengths, offsets, flat


def all_positions(data: np.ndarray, mode: str = "leftmost", path: str = "compact",
                  workers: int | None = 1, structures=None):
    """query.py:218-239 over raw bytes; returns the tuple of result arrays."""
    data = np.ascontiguousarray(data, dtype=np.uint8)
    sa, rank, lcp = structures if structures is not None else build_suffix_structures(data)
    n = int(sa.size) - 1
    raw = build_raw_llr(rank, lcp, workers)
    c = build_compact_llr(raw, workers) if path == "compact" else None
    if mode == "leftmost":
        return leftmost_all_positions(n, path, raw, c, workers)
    return all_all_positions(n, path, raw, c, workers)


# -- oracle.py:78-104 brute force (pure Python; tiny inputs only) -------------
def _longest_repeat_from(s: bytes, i: int) -> int:
    """oracle.py:27-38: longest repeated substring starting at 1-based i."""
    for length in range(len(s) - i + 1, 0, -1):
        sub = s[i - 1: i - 1 + length]
        if s.find(sub) != s.rfind(sub):
            return length
    return 0


def brute_all_positions(s: bytes, mode: str = "leftmost"):
    """Per-position list: (start, length) for leftmost, list of them for all."""
    n = len(s)
    reach = [0] * (n + 1)
    for i in range(1, n + 1):
        reach[i] = _longest_repeat_from(s, i)
    out = []
    for k in range(1, n + 1):
        best = 0
        for i in range(1, k + 1):
            if reach[i] >= k - i + 1 and reach[i] > best:
                best = reach[i]
        if best == 0:
            out.append((-1, 0) if mode == "leftmost" else [])
            continue
        hits = [(i, best) for i in range(1, k + 1) if reach[i] >= best and i + best - 1 >= k]
        out.append(hits[0] if mode == "leftmost" else hits)
    return out


# -- stats.py:30-68 walk-step statistics (numpy closed form) --------------------
def walk_steps_raw(raw: np.ndarray) -> np.ndarray:
    """stats.py:30-43: steps[k] = k - #{i : i + raw[i] - 1 < k}."""
    n = int(raw.size) - 1
    steps = np.zeros(n + 1, dtype=np.int64)
    if n == 0:
        return steps
    ends = np.arange(1, n + 1, dtype=np.int64) + raw[1:] - 1
    ks = np.arange(1, n + 1, dtype=np.int64)
    steps[1:] = ks - np.searchsorted(ends, ks, side="left")
    return steps


def walk_steps_compact(starts: np.ndarray, lengths: np.ndarray, n: int) -> np.ndarray:
    """stats.py:46-55: max(#starts <= k - #ends < k, 0)."""
    steps = np.zeros(n + 1, dtype=np.int64)
    if n == 0 or starts.size == 0:
        return steps
    ends = starts + lengths - 1
    ks = np.arange(1, n + 1, dtype=np.int64)
    steps[1:] = np.maximum(np.searchsorted(starts, ks, side="right")
                           - np.searchsorted(ends, ks, side="left"), 0)
    return steps


def summarize_steps(steps: np.ndarray):
    """stats.py:58-68 -> (min, max, avg, positions)."""
    covered = steps[steps > 0]
    if covered.size == 0:
        return 0, 0, 0.0, 0
    return int(covered.min()), int(covered.max()), float(covered.mean()), int(covered.size)


# -- oracle32.c: u32 restatement for full-size digests ---------------------------
_lib32 = None
_O32_FIELDS = ("sa", "rank", "lcp", "raw", "flags", "c_starts", "c_lengths")


def _load32():
    global _lib32
    if _lib32 is not None:
        return _lib32
    path = _HERE / "liboracle32.so"
    if not path.exists():
        build()
    lib = ctypes.CDLL(str(path))
    i64, c_int, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
    sig = {
        "o32_create": (vp, [_U8P, i64]),
        "o32_destroy": (None, [vp]),
        "o32_sa": (c_int, [vp]),
        "o32_lcp": (c_int, [vp]),
        "o32_raw": (c_int, [vp]),
        "o32_free_structures": (None, [vp]),
        "o32_compact": (i64, [vp]),
        "o32_chunk": (c_int, [vp, c_int, i64, i64, _I64P]),
        "o32_leftmost": (None, [vp, i64, i64, _I64P, _I64P]),
        "o32_all_count": (None, [vp, i64, i64, _I64P, _I64P]),
        "o32_all_fill": (None, [vp, i64, i64, _I64P, _I64P, _I64P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib32 = lib
    return lib


def digests32(data: np.ndarray, chunk: int = 1 << 24, log=None) -> dict:
    """sha256 digests (16 hex) of every int64 reference-layout array of the
    compact path (sa, rank, lcp, raw, flags, ps, c_starts, c_lengths,
    l_starts, l_lengths, a_lengths, a_offsets, a_flat) plus n, m, T, max_llr,
    computed by oracle32.c with uint32 indices and streamed in chunks."""
    import hashlib
    import time
    lib = _load32()
    data = np.ascontiguousarray(data, dtype=np.uint8)
    n = int(data.size)
    log = log or (lambda s: None)
    h = lib.o32_create(_u8(data), n)
    if not h:
        raise MemoryError("o32_create")
    out = {}
    try:
        t0 = time.time()
        rounds = lib.o32_sa(h)
        if rounds < 0:
            raise MemoryError("o32_sa")
        log(f"suffix array: {rounds} doubling rounds, {time.time() - t0:.1f} s")
        if lib.o32_lcp(h) != 0 or lib.o32_raw(h) != 0:
            raise MemoryError("o32_lcp/o32_raw")
        log(f"lcp + raw: {time.time() - t0:.1f} s")
        m = int(lib.o32_compact(h))
        if m < 0:
            raise MemoryError("o32_compact")
        out.update(n=n, m=m, sa_rounds=int(rounds))
        buf = np.empty(chunk, np.int64)
        sizes = {"sa": n + 1, "rank": n + 1, "lcp": n + 2, "raw": n + 1, "flags": n + 1,
                 "c_starts": m, "c_lengths": m}
        max_llr = 0
        for w, f in enumerate(_O32_FIELDS):
            hs = hashlib.sha256()
            hps = hashlib.sha256() if f == "flags" else None
            carry = 0
            for lo in range(0, sizes[f], chunk):
                cnt = min(chunk, sizes[f] - lo)
                lib.o32_chunk(h, w, lo, cnt, _p(buf))
                v = buf[:cnt]
                hs.update(v.tobytes())
                if f == "raw":
                    max_llr = max(max_llr, int(v.max(initial=0)))
                if hps is not None:  # ps = inclusive scan of flags, ps[0] = 0 (llr.py:92-96)
                    ps = np.cumsum(v) + carry
                    carry = int(ps[-1])
                    hps.update(ps.tobytes())
            out[f] = hs.hexdigest()[:16]
            if hps is not None:
                out["ps"] = hps.hexdigest()[:16]
            if f == "raw":
                lib.o32_free_structures(h)
        out["max_llr"] = max_llr
        log(f"structures/llr digests: {time.time() - t0:.1f} s")
        # leftmost (query.py:171-184): starts[0] = -1, lengths[0] = 0
        hs, hl = hashlib.sha256(), hashlib.sha256()
        hs.update(np.array([-1], np.int64).tobytes())
        hl.update(np.array([0], np.int64).tobytes())
        s_buf, l_buf = np.empty(chunk, np.int64), np.empty(chunk, np.int64)
        for lo in range(1, n + 1, chunk):
            hi = min(lo + chunk, n + 1)
            lib.o32_leftmost(h, lo, hi, _p(s_buf), _p(l_buf))
            hs.update(s_buf[:hi - lo].tobytes())
            hl.update(l_buf[:hi - lo].tobytes())
        out.update(l_starts=hs.hexdigest()[:16], l_lengths=hl.hexdigest()[:16])
        log(f"leftmost: {time.time() - t0:.1f} s")
        # all ties (query.py:187-215): lengths[0] = 0, offsets[0] = offsets[1] = 0
        hl, ho, hf = hashlib.sha256(), hashlib.sha256(), hashlib.sha256()
        hl.update(np.array([0], np.int64).tobytes())
        ho.update(np.array([0, 0], np.int64).tobytes())
        cnt_buf = np.empty(chunk, np.int64)
        base = 0
        for lo in range(1, n + 1, chunk):
            hi = min(lo + chunk, n + 1)
            c = hi - lo
            lib.o32_all_count(h, lo, hi, _p(l_buf), _p(cnt_buf))
            incl = np.cumsum(cnt_buf[:c])
            local = np.ascontiguousarray(incl - cnt_buf[:c])
            flat = np.empty(int(incl[-1]), np.int64)
            lib.o32_all_fill(h, lo, hi, _p(l_buf), _p(local), _p(flat))
            hl.update(l_buf[:c].tobytes())
            ho.update((incl + base).tobytes())
            hf.update(flat.tobytes())
            base += int(incl[-1])
        out.update(T=base, a_lengths=hl.hexdigest()[:16], a_offsets=ho.hexdigest()[:16],
                   a_flat=hf.hexdigest()[:16])
        log(f"all ties: {time.time() - t0:.1f} s")
    finally:
        lib.o32_destroy(h)
    return out
