"""Randomised parity sweep of the CUDA path against the oracle (test tool).

usage: python tools/fuzz_parity.py [--seed S] [--seconds T] [--max-n N]

Mixed alphabets, sizes, planted copies, periodic stretches and mutated
Fibonacci words; every case compares SA / rank / LCP and both query modes
with the oracle.  Prints one line per case and exits non-zero on the first
mismatch (the failing text is saved under gpurun_out/fuzz_fail_<seed>.npy).
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle  # noqa: E402
import paper_1501_06663_b200 as rb  # noqa: E402


def make_case(rng, max_n):
    kind = int(rng.integers(0, 4))
    n = int(rng.integers(1, max_n))
    if kind == 3 and n > 1000:
        return "fib", _fib(n, rng)
    sigma = int(rng.choice([1, 2, 3, 4, 5, 20, 95, 256]))
    alpha = rng.choice(256, size=sigma, replace=False).astype(np.uint8)
    data = rng.choice(alpha, size=n)
    for _ in range(int(rng.integers(0, 8))):
        ln = int(rng.integers(1, max(2, n // 4)))
        if ln >= n:
            continue
        src, dst = (int(x) for x in rng.integers(0, n - ln, 2))
        data[dst:dst + ln] = data[src:src + ln].copy()
    if kind == 2 and n > 10:
        p, ln = int(rng.integers(1, 60)), int(rng.integers(1, n))
        dst = int(rng.integers(0, n - ln + 1))
        data[dst:dst + ln] = np.resize(data[:p], ln)
    return f"sigma{sigma}/k{kind}", data


def _fib(n, rng):
    a, b = np.array([0], np.uint8), np.array([0, 1], np.uint8)
    while b.size < n:
        a, b = b, np.concatenate([b, a])
    data = b[:n].copy()
    m = int(rng.integers(0, max(1, n // 1000)))
    if m:
        idx = rng.integers(0, n, m)
        data[idx] = rng.integers(0, 4, m).astype(np.uint8)
    return data


def check_dist(data, world):
    from paper_1501_06663_b200 import distributed as D
    got = D.loopback_dist_all_positions(data, world, "all")
    if got is None:
        return None, "declined"
    wl, wo, wf = oracle.all_positions(data, mode="all")
    ok = np.array_equal(got[0], wl) and np.array_equal(got[1], wo) and np.array_equal(got[2], wf)
    return (None if ok else f"dist/{world}"), "ran"


def check(data):
    want = oracle.build_suffix_structures(data)
    s = rb.build_suffix_structures(rb.Text(data))
    if not all(np.array_equal(a, b) for a, b in zip((s.sa, s.rank, s.lcp), want)):
        return "structures"
    wl, wo, wf = oracle.all_positions(data, mode="all", structures=want)
    for path in ("raw", "compact"):
        A = rb.all_positions(rb.Text(data), mode="all", path=path)
        if not (np.array_equal(A.lengths, wl) and np.array_equal(A.offsets, wo) and np.array_equal(A.flat_starts, wf)):
            return f"all/{path}"
    ws, wln = oracle.all_positions(data, mode="leftmost", structures=want)
    L = rb.all_positions(rb.Text(data), mode="leftmost")
    if not (np.array_equal(L.starts, ws) and np.array_equal(L.lengths, wln)):
        return "leftmost"
    return None


def check_shards(data, world, given_sa):
    """Query from resident structures by position shards (rs_query_structures_shard,
    the multi-GPU value path), structures given by the caller (with a consistent
    or a perturbed sa) or built on device; stitched shards vs the oracle."""
    from paper_1501_06663_b200 import _native
    from paper_1501_06663_b200 import distributed as D
    n = int(data.size)
    want = oracle.build_suffix_structures(data, workers=8)
    wl, wo, wf = oracle.all_positions(data, mode="all", structures=want, workers=8)
    ctx = _native.context()
    with ctx.lock:
        if given_sa == "device":
            ctx.call("rs_set_text", _native.u8(data), n)
            ctx.call("rs_build_structures")
        else:
            sa = want[0].copy()
            if given_sa == "perturbed" and n > 3:
                sa[[1, 2]] = sa[[2, 1]]
            ctx.call("rs_set_structures", _native.i64(sa), _native.i64(want[1]), _native.i64(want[2]), n)
        L = np.zeros(n + 1, np.int64)
        O = np.zeros(n + 2, np.int64)
        flats, base = [], 0
        for r in range(world):
            lo, hi = D.shard_range(n, world, r)
            tot = np.zeros(1, np.int64)
            ctx.call("rs_query_structures_shard", 1, lo, hi, _native.i64(tot))
            ctx.call("rs_shard_rebase", base)
            a = np.zeros(hi - lo, np.int64)
            b = np.zeros(hi - lo + 1, np.int64)
            f = np.zeros(int(tot[0]), np.int64)
            ctx.call("rs_fetch_shard", 1, _native.i64(a), _native.i64(b), _native.i64(f))
            L[lo:hi] = a
            O[lo + 1:hi + 1] = b[1:]
            flats.append(f)
            base += f.size
    F = np.concatenate(flats) if flats else np.zeros(0, np.int64)
    ok = np.array_equal(L, wl) and np.array_equal(O, wo) and np.array_equal(F, wf)
    return None if ok else f"shards/{world}/{given_sa}"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--seconds", type=float, default=120.0)
    ap.add_argument("--max-n", type=int, default=2_000_000)
    ap.add_argument("--dist", action="store_true", help="the loopback distributed sort with 1..6 ranks")
    ap.add_argument("--shards", action="store_true",
                    help="query from resident structures by 1..9 position shards")
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    t0, cases = time.time(), 0
    while time.time() - t0 < a.seconds:
        name, data = make_case(rng, a.max_n)
        note = ""
        if a.dist:
            world = int(rng.integers(1, 7))
            bad, note = check_dist(data, world)
            note = f" world={world} {note}"
        elif a.shards:
            world = int(rng.integers(1, 10))
            how = ("device", "consistent", "perturbed")[int(rng.integers(0, 3))]
            bad = check_shards(data, world, how)
            note = f" shards={world} {how}"
        else:
            bad = check(data)
        cases += 1
        print(f"case {cases} {name} n={data.size}{note} -> {bad or 'ok'}", flush=True)
        if bad:
            os.makedirs("gpurun_out", exist_ok=True)
            np.save(f"gpurun_out/fuzz_fail_{a.seed}.npy", data)
            sys.exit(1)
    print(f"fuzz OK: {cases} cases in {time.time() - t0:.0f} s (seed {a.seed})")


if __name__ == "__main__":
    main()
