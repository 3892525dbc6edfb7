"""GPU parity: the CUDA path through the C-ABI vs the reference (golden) and the oracle.

Bit-exact for every array (integer work).  Golden vectors come from the
reference package itself (tests/golden/make_golden.py); larger inputs are
checked against the pinned C oracle or reference digests.
"""

from __future__ import annotations

import itertools
import os

import numpy as np
import pytest

import oracle
import paper_1501_06663_b200 as rb
from paper_1501_06663_b200 import workloads
from conftest import digest, golden_cases, golden_digests

pytestmark = pytest.mark.gpu


def _structs(c):
    return rb.SuffixStructures(sa=c.sa, rank=c.rank, lcp=c.lcp)


def test_suffix_structures_golden():
    for c in golden_cases():
        s = rb.build_suffix_structures(rb.Text(c.data))
        assert np.array_equal(s.sa, c.sa), c
        assert np.array_equal(s.rank, c.rank), c
        assert np.array_equal(s.lcp, c.lcp), c


def test_llr_pipeline_golden():
    for c in golden_cases():
        raw = rb.build_raw_llr(_structs(c))
        assert np.array_equal(raw, c.raw), c
        flags = rb.compute_flags(c.raw)
        assert np.array_equal(flags, c.flags), c
        ps = rb.prefix_sum(c.flags)
        assert np.array_equal(ps, c.ps), c
        sc = rb.scatter_compact(c.raw, c.flags, c.ps)
        assert np.array_equal(sc.starts, c.c_starts) and np.array_equal(sc.lengths, c.c_lengths), c
        cc = rb.build_compact_llr(c.raw, rb.ExecPolicy.parallel(3))
        assert np.array_equal(cc.starts, c.c_starts) and np.array_equal(cc.lengths, c.c_lengths), c
        cs = rb.compact_llr_sequential(c.raw)
        assert cs.entries() == cc.entries()


def test_all_positions_golden_every_path():
    for c in golden_cases():
        t = rb.Text(c.data)
        for path in ("raw", "compact"):
            for structures in (None, _structs(c)):
                L = rb.all_positions(t, mode="leftmost", path=path, structures=structures)
                assert np.array_equal(L.starts, c.l_starts), (c, path)
                assert np.array_equal(L.lengths, c.l_lengths), (c, path)
                A = rb.all_positions(t, mode="all", path=path, structures=structures)
                assert np.array_equal(A.lengths, c.a_lengths), (c, path)
                assert np.array_equal(A.offsets, c.a_offsets), (c, path)
                assert np.array_equal(A.flat_starts, c.a_flat), (c, path)


def test_private_batch_drivers_golden():
    # query.py:171-215 called directly, as cli.py:229-232 and the acceptance tests do
    from paper_1501_06663_b200.query import _all_all_positions, _leftmost_all_positions
    for c in golden_cases()[::3]:
        comp = rb.CompactLlr.from_arrays(c.c_starts, c.c_lengths)
        for path in ("raw", "compact"):
            L = _leftmost_all_positions(c.n, path, c.raw, comp, None)
            assert np.array_equal(L.starts, c.l_starts) and np.array_equal(L.lengths, c.l_lengths)
            A = _all_all_positions(c.n, path, c.raw, comp, rb.ExecPolicy.parallel(2))
            assert np.array_equal(A.offsets, c.a_offsets) and np.array_equal(A.flat_starts, c.a_flat)


def test_reference_known_answers():
    t = rb.Text.from_str("mississippi")
    s = rb.build_suffix_structures(t)
    assert s.sa[1:].tolist() == [11, 8, 5, 2, 1, 10, 9, 7, 4, 6, 3]
    assert s.lcp[1:].tolist() == [0, 1, 1, 4, 0, 0, 1, 0, 2, 1, 3, 0]
    assert rb.verify_suffix_structures(t, s)
    res = rb.all_positions(t)
    got = [tuple(res.answer(k)) for k in range(1, 12)]
    assert got == [(-1, 0), (2, 4), (2, 4), (2, 4), (2, 4), (5, 4), (5, 4), (5, 4), (9, 1),
                   (10, 1), (11, 1)]
    for path in ("raw", "compact"):
        r = rb.all_positions(rb.Text.from_str("abcabcddbca"), mode="all", path=path)
        assert r.answers(2) == [rb.LrAnswer(1, 3), rb.LrAnswer(2, 3)]
    e = rb.all_positions(rb.Text.from_str(""))
    assert e.n == 0 and e.starts.tolist() == [-1]
    e = rb.all_positions(rb.Text.from_str(""), mode="all")
    assert e.offsets.tolist() == [0, 0]
    a4 = rb.all_positions(rb.Text.from_str("aaaa"), mode="all")
    assert a4.offsets.tolist() == [0, 0, 1, 3, 5, 6] and a4.flat_starts.tolist() == [1, 1, 2, 1, 2, 2]


def test_verify_rejects_bad_structures():
    t = rb.Text.from_str("ab")
    s = rb.build_suffix_structures(t)
    bad = rb.SuffixStructures(sa=s.sa[[0, 2, 1]], rank=s.rank.copy(), lcp=s.lcp.copy())
    assert not rb.verify_suffix_structures(t, bad)
    t = rb.Text.from_str("aaaa")
    s = rb.build_suffix_structures(t)
    lcp = s.lcp.copy()
    lcp[3] += 1
    assert not rb.verify_suffix_structures(t, rb.SuffixStructures(sa=s.sa, rank=s.rank, lcp=lcp))


def test_exhaustive_binary_strings_vs_oracle():
    # test_acceptance.py:114-119 shape: every {a,b} string up to n = 12
    for n in range(1, 13):
        for tup in itertools.product(b"ab", repeat=n):
            data = np.frombuffer(bytes(tup), np.uint8)
            t = rb.Text(data)
            wl, wo, wf = oracle.all_positions(data, mode="all")
            A = rb.all_positions(t, mode="all", path="compact")
            assert np.array_equal(A.offsets, wo) and np.array_equal(A.flat_starts, wf), bytes(tup)
            if n <= 8:
                B = rb.all_positions(t, mode="all", path="raw")
                assert np.array_equal(B.flat_starts, wf)


@pytest.mark.parametrize("name", ["acgt_1e6_seed99", "C1_2p20", "C2_shape_2p21", "C4_shape_2p21",
                                  "C5_shape_2p20", "periodic_2p20"])
def test_reference_digests(name):
    rec = golden_digests()[name]
    data = eval(rec["expr"])
    t = rb.Text(data)
    s = rb.build_suffix_structures(t)
    assert digest(s.sa) == rec["sa"] and digest(s.rank) == rec["rank"] and digest(s.lcp) == rec["lcp"]
    raw = rb.build_raw_llr(s)
    assert digest(raw) == rec["raw"]
    c = rb.build_compact_llr(raw)
    assert digest(c.starts) == rec["c_starts"] and digest(c.lengths) == rec["c_lengths"]
    paths = ("raw", "compact") if rec["max_llr"] < 1000 else ("compact",)
    for path in paths:
        A = rb.all_positions(t, mode="all", path=path)
        assert digest(A.lengths) == rec["a_lengths"] and digest(A.offsets) == rec["a_offsets"]
        assert digest(A.flat_starts) == rec["a_flat"]
        L = rb.all_positions(t, mode="leftmost", path=path, structures=s)
        assert digest(L.starts) == rec["l_starts"] and digest(L.lengths) == rec["l_lengths"]


def test_random_inputs_vs_oracle(rng):
    for _ in range(60):
        n = int(rng.integers(1, 5000))
        sigma = int(rng.integers(1, 256))
        alpha = rng.choice(256, size=sigma, replace=False).astype(np.uint8)
        data = rng.choice(alpha, size=n)
        if rng.random() < 0.3:  # inject long repeats
            p = int(rng.integers(1, 50))
            data = np.resize(data[:p], n)
        want = oracle.build_suffix_structures(data)
        s = rb.build_suffix_structures(rb.Text(data))
        assert all(np.array_equal(a, b) for a, b in zip((s.sa, s.rank, s.lcp), want))
        wl, wo, wf = oracle.all_positions(data, mode="all", structures=want)
        A = rb.all_positions(rb.Text(data), mode="all")
        assert np.array_equal(A.lengths, wl) and np.array_equal(A.offsets, wo)
        assert np.array_equal(A.flat_starts, wf)


def test_medium_random_texts_vs_oracle(rng):
    # sizes where the multi-round paths engage (u64 keys, dense-ordinal
    # keys, small-group resolution, lazy ISA, Kasai vs patch LCP), mixed
    # alphabets, planted copies and periodic stretches
    for case in range(10):
        n = int(rng.integers(100_000, 1_500_000))
        sigma = int(rng.choice([2, 3, 4, 5, 20, 95, 256]))
        alpha = rng.choice(256, size=sigma, replace=False).astype(np.uint8)
        data = rng.choice(alpha, size=n)
        for _ in range(int(rng.integers(0, 6))):  # planted copies
            ln = int(rng.integers(10, 5000))
            src, dst = (int(x) for x in rng.integers(0, n - ln, 2))
            data[dst:dst + ln] = data[src:src + ln].copy()
        if case % 3 == 0:  # a periodic stretch
            p, ln = int(rng.integers(1, 40)), int(rng.integers(1000, 50_000))
            dst = int(rng.integers(0, n - ln))
            data[dst:dst + ln] = np.resize(data[:p], ln)
        want = oracle.build_suffix_structures(data)
        s = rb.build_suffix_structures(rb.Text(data))
        assert all(np.array_equal(a, b) for a, b in zip((s.sa, s.rank, s.lcp), want)), (case, n, sigma)
        wl, wo, wf = oracle.all_positions(data, mode="all", structures=want)
        A = rb.all_positions(rb.Text(data), mode="all")
        assert np.array_equal(A.lengths, wl) and np.array_equal(A.offsets, wo), (case, n, sigma)
        assert np.array_equal(A.flat_starts, wf), (case, n, sigma)
        ws, wln = oracle.all_positions(data, mode="leftmost", structures=want)
        L = rb.all_positions(rb.Text(data), mode="leftmost", path="compact")
        assert np.array_equal(L.starts, ws) and np.array_equal(L.lengths, wln), (case, n, sigma)


def test_tile_boundaries_and_long_windows():
    # sizes straddling the 2048-position tiles and 4096-key sort tiles,
    # plus a periodic text whose windows exceed the shared-memory stage.
    for n in (2047, 2048, 2049, 4095, 4096, 4097, 8191, 8193, 65537):
        data = workloads.iid_dna(n, n)
        want = oracle.all_positions(data, mode="all", path="compact")
        A = rb.all_positions(rb.Text(data), mode="all", path="compact")
        assert np.array_equal(A.offsets, want[1]) and np.array_equal(A.flat_starts, want[2]), n
    data = workloads.periodic_mutated(40000, 3, period=7, rate=0.0)
    for path in ("raw", "compact"):
        for mode in ("leftmost", "all"):
            want = oracle.all_positions(data, mode=mode, path="compact")
            got = rb.all_positions(rb.Text(data), mode=mode, path=path)
            arrs = (got.starts, got.lengths) if mode == "leftmost" else (
                got.lengths, got.offsets, got.flat_starts)
            assert all(np.array_equal(a, b) for a, b in zip(arrs, want)), (path, mode)


@pytest.mark.parametrize("cap", ["0", "1", "1500", "2000"])
def test_fused_scan_tie_list_overflow(cap, monkeypatch):
    # the fused all-ties scan lists a tile's ties in shared memory (2688 of
    # them) and stores overflowing tiles directly; shrink the list so both
    # paths, mixed within one launch, are checked against the oracle
    monkeypatch.setenv("RS_FUSED_TIES_CAP", cap)
    for data in (workloads.iid_dna(300_000, 11), workloads.make("C2", 1 << 18)):
        want = oracle.all_positions(data, mode="all", path="compact", workers=4)
        A = rb.all_positions(rb.Text(data), mode="all", path="compact")
        assert np.array_equal(A.lengths, want[0]) and np.array_equal(A.offsets, want[1]), cap
        assert np.array_equal(A.flat_starts, want[2]), cap


@pytest.mark.parametrize("config", ["C2", "C3", "C4"])
def test_full_size_properties(config):
    # BASELINE configs at full size (64 Mi planted DNA, the 256 Mi headline,
    # 100 Mi English-like), beyond what the oracle finishes quickly: the structures are verified on device by
    # direct comparison, the raw and compact paths (different kernels) must
    # agree array for array, leftmost must equal the first tie,
    # and every tie start must cover its position with the position's length,
    # blocks strictly increasing.
    data = workloads.make(config)
    n = data.size
    t = rb.Text(data)
    s = rb.build_suffix_structures(t)
    assert rb.verify_suffix_structures(t, s)
    A = rb.all_positions(t, mode="all", path="compact", structures=s)
    R = rb.all_positions(t, mode="all", path="raw", structures=s)
    assert np.array_equal(A.lengths, R.lengths) and np.array_equal(A.offsets, R.offsets)
    assert np.array_equal(A.flat_starts, R.flat_starts)
    del R
    L = rb.all_positions(t, mode="leftmost", path="compact", structures=s)
    del s
    assert np.array_equal(L.lengths, A.lengths)
    cnt = np.diff(A.offsets)[1:]
    has = cnt > 0
    assert np.array_equal(has, A.lengths[1:] > 0)
    assert np.array_equal(L.starts[1:][has], A.flat_starts[A.offsets[1:-1][has]])
    assert (L.starts[1:][~has] == -1).all() and L.starts[0] == -1
    del L
    k = np.repeat(np.arange(1, n + 1, dtype=np.int64), cnt)
    st = A.flat_starts
    assert ((st <= k) & (k <= st + np.repeat(A.lengths[1:], cnt) - 1)).all()
    same = k[1:] == k[:-1]
    assert (st[1:][same] > st[:-1][same]).all()


def test_api_errors():
    with pytest.raises(ValueError):
        rb.all_positions(rb.Text.from_str("abc"), mode="bogus")
    with pytest.raises(ValueError):
        rb.all_positions(rb.Text.from_str("abc"), path="bogus")
    with pytest.raises(ValueError):  # raw array violating raw[i] <= raw[i+1] + 1
        from paper_1501_06663_b200.query import _leftmost_all_positions
        _leftmost_all_positions(3, "raw", np.array([0, 3, 0, 0], np.int64), None, None)
    with pytest.raises(ValueError):  # rank out of range
        rb.build_raw_llr(rb.SuffixStructures(sa=np.array([0, 1], np.int64),
                                             rank=np.array([0, 5], np.int64),
                                             lcp=np.zeros(3, np.int64)))


def test_parallel_scan_gpu(rng):
    for _ in range(20):
        n = int(rng.integers(0, 100000))
        v = rng.integers(0, 1000, size=n).astype(np.int64)
        assert np.array_equal(rb.parallel_scan(v, rb.ExecPolicy.parallel(4)), np.cumsum(v))


def test_parallel_scan_full_int64(rng):
    """engine.py:77-110 is np.cumsum over any int64: negative values, prefixes
    beyond 2^62 and two's-complement wraparound, over many look-back tiles."""
    big = np.iinfo(np.int64).max
    cases = [np.full(3000, -1, np.int64), np.full(50000, -7, np.int64),
             np.full(10000, 1 << 61, np.int64), np.full(10000, -(1 << 61), np.int64),
             np.full(5000, big, np.int64), np.full(5000, big // 3, np.int64),
             np.array([big, 1, big, 1, -big, -5], np.int64)]
    for n in (2047, 2048, 2049, 1 << 20, (1 << 22) + 12345):
        cases.append(rng.integers(-(1 << 62), 1 << 62, size=n, dtype=np.int64))
        cases.append(rng.integers(np.iinfo(np.int64).min, big, size=n, dtype=np.int64,
                                  endpoint=True))
    for v in cases:
        with np.errstate(over="ignore"):
            want = np.cumsum(v)
        assert np.array_equal(rb.parallel_scan(v, rb.ExecPolicy.parallel(4)), want)
    flags = np.zeros(1 << 21, np.int64)
    flags[1:] = rng.integers(-3, 1 << 40, size=flags.size - 1)
    ps = rb.prefix_sum(flags)
    assert ps[0] == 0 and np.array_equal(ps[1:], np.cumsum(flags[1:]))


def test_kernels_launch_from_native_library():
    from paper_1501_06663_b200 import _native
    ctx = _native.context()
    before = ctx.launches()
    rb.all_positions(rb.Text(workloads.iid_dna(10000, 1)), mode="all")
    assert ctx.launches() > before


def test_shard_queries_assemble_to_full_answer():
    # Device-side halo handling: each shard [lo, hi) is answered from the
    # global compact array (rs_query_shard); stitched shards == full answer.
    from paper_1501_06663_b200 import _native
    from paper_1501_06663_b200 import distributed as D
    for data in (workloads.planted_dna(300_000, 9, family_len=200),
                 workloads.fibonacci_mutated(200_000, 5, rate=1e-3)):
        n = data.size
        want_l, want_o, want_f = oracle.all_positions(data, mode="all")
        want_s, want_len = oracle.all_positions(data, mode="leftmost")
        ctx = _native.context()
        for world in (2, 3, 8):
            lengths = np.zeros(n + 1, np.int64)
            offsets = np.zeros(n + 2, np.int64)
            flats, base = [], 0
            starts = np.full(n + 1, -1, np.int64)
            llen = np.zeros(n + 1, np.int64)
            for r in range(world):
                lo, hi = D.shard_range(n, world, r)
                with ctx.lock:
                    ctx.call("rs_set_text", _native.u8(data), n)
                    m = np.zeros(1, np.int64)
                    ctx.call("rs_get_compact_size", _native.i64(m))
                    tot = np.zeros(1, np.int64)
                    ctx.call("rs_query_shard", 1, lo, hi, _native.i64(tot))
                    ctx.call("rs_shard_rebase", base)
                    a = np.zeros(hi - lo, np.int64)
                    b = np.zeros(hi - lo + 1, np.int64)
                    f = np.zeros(int(tot[0]), np.int64)
                    ctx.call("rs_fetch_shard", 1, _native.i64(a), _native.i64(b), _native.i64(f))
                    ctx.call("rs_query_shard", 0, lo, hi, _native.i64(tot))
                    sa_ = np.zeros(hi - lo, np.int64)
                    sl_ = np.zeros(hi - lo, np.int64)
                    ctx.call("rs_fetch_shard", 0, _native.i64(sa_), _native.i64(sl_), _native.i64(f[:0]))
                lengths[lo:hi] = a
                offsets[lo + 1:hi + 1] = b[1:]
                assert b[0] == base
                flats.append(f)
                base += f.size
                starts[lo:hi] = sa_
                llen[lo:hi] = sl_
            assert np.array_equal(lengths, want_l) and np.array_equal(offsets, want_o), world
            assert np.array_equal(np.concatenate(flats), want_f), world
            assert np.array_equal(starts, want_s) and np.array_equal(llen, want_len), world


def test_distributed_single_rank_nccl():
    # sharded_all_positions end to end through torch.distributed/NCCL device
    # views of the library buffers (world size 1 on the one GPU available).
    import os
    import socket
    import torch
    import torch.distributed as dist
    from paper_1501_06663_b200 import distributed as D
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        data = workloads.planted_dna(200_000, 3, family_len=100)
        out = D.sharded_all_positions(data, "all")
        res = D.to_answers(out, "all")
        wl, wo, wf = oracle.all_positions(data, mode="all")
        assert np.array_equal(res.lengths, wl) and np.array_equal(res.offsets, wo)
        assert np.array_equal(res.flat_starts, wf)
        out = D.sharded_all_positions(data, "leftmost")
        res = D.to_answers(out, "leftmost")
        ws, wln = oracle.all_positions(data, mode="leftmost")
        assert np.array_equal(res.starts, ws) and np.array_equal(res.lengths, wln)
        # the distributed suffix sort through NCCL (text broadcast, all-to-all,
        # halo send/recv, gather) on an i.i.d.-like text
        data = workloads.iid_dna(300_000, 31)
        for mode in ("all", "leftmost"):
            out = D.dist_sa_all_positions(data, int(data.size), mode)
            assert out is not None
            res = D.to_answers(out, mode)
            if mode == "all":
                wl, wo, wf = oracle.all_positions(data, mode="all")
                assert np.array_equal(res.lengths, wl) and np.array_equal(res.offsets, wo)
                assert np.array_equal(res.flat_starts, wf)
            else:
                ws, wln = oracle.all_positions(data, mode="leftmost")
                assert np.array_equal(res.starts, ws) and np.array_equal(res.lengths, wln)
        # outside the distributed regime it declines (caller falls back)
        rep = workloads.periodic_mutated(60_000, 3, period=7, rate=0.0)
        assert D.dist_sa_all_positions(rep, int(rep.size), "all") is None
        # the library's own NCCL communicator (csrc/collectives.cu): text
        # broadcast + tie-total all-gather inside the library, shards written
        # into the shared host buffer -- the multi-GPU API path
        from paper_1501_06663_b200 import _native
        ctx = _native.context()
        assert D.library_comm(ctx) and D.allgather_i64(ctx, 12345) == [12345]
        for data in (workloads.planted_dna(200_000, 3, family_len=100),
                     workloads.fibonacci_mutated(120_000, 5, rate=1e-3)):
            st = oracle.build_suffix_structures(data, workers=8)
            for mode in ("all", "leftmost"):
                res = D.replicated_all_positions(data, mode)
                want = oracle.all_positions(data, mode=mode, workers=8, structures=st)
                got = (res.lengths, res.offsets, res.flat_starts) if mode == "all" else (res.starts, res.lengths)
                assert all(np.array_equal(g, w) for g, w in zip(got, want)), mode
    finally:
        dist.destroy_process_group()


def test_walk_stats_vs_closed_form():
    # stats.py:30-76 (reference closed form restated in oracle/) on the golden
    # inputs and on structured texts; plus the reference's own known answers.
    for c in golden_cases()[::2] + [None]:
        if c is None:
            data = workloads.fibonacci_mutated(200_000, 5, rate=1e-3)
            sa, rank, lcp = oracle.build_suffix_structures(data)
            raw = oracle.build_raw_llr(rank, lcp)
            cs, cl = oracle.build_compact_llr(raw)
        else:
            raw, cs, cl = c.raw, c.c_starts, c.c_lengths
        n = raw.size - 1
        comp = rb.CompactLlr.from_arrays(cs, cl)
        wr = oracle.walk_steps_raw(raw) if c is None else c.w_raw      # golden: the reference's own
        wc = oracle.walk_steps_compact(cs, cl, n) if c is None else c.w_comp
        from paper_1501_06663_b200 import stats as S
        assert np.array_equal(S.walk_steps_raw(raw), wr)
        assert np.array_equal(S.walk_steps_compact(comp, n), wc)
        for path, w in (("raw", wr), ("compact", wc)):
            got = rb.compute_walk_stats(raw, comp, path)
            mn, mx, avg, pos = oracle.summarize_steps(w)
            assert (got.min_steps, got.max_steps, got.positions) == (mn, mx, pos)
            assert got.avg_steps == pytest.approx(avg, rel=1e-12)
            s2 = S.summarize_steps(w, path)
            assert (s2.min_steps, s2.max_steps, s2.positions) == (mn, mx, pos)
    raw = rb.build_raw_llr(rb.build_suffix_structures(rb.Text.from_str("aaaa")))
    from paper_1501_06663_b200 import stats as S
    assert S.walk_steps_raw(raw)[1:].tolist() == [1, 2, 3, 3]  # test_stats.py:18-23
    st = rb.compute_walk_stats(raw, rb.compact_llr_sequential(raw), "raw")
    assert (st.min_steps, st.max_steps) == (1, 3) and st.avg_steps == (1 + 2 + 3 + 3) / 4
    raw = rb.build_raw_llr(rb.build_suffix_structures(rb.Text.from_str("abc")))
    for path in ("raw", "compact"):  # test_stats.py:26-30
        st = rb.compute_walk_stats(raw, rb.compact_llr_sequential(raw), path)
        assert (st.min_steps, st.max_steps, st.avg_steps, st.positions) == (0, 0, 0.0, 0)
    with pytest.raises(ValueError):
        rb.compute_walk_stats(raw, rb.compact_llr_sequential(raw), "bogus")


def test_small_tied_groups_vs_oracle(rng):
    # i.i.d. DNA (few ties after round 0 -> the direct small-group sort) with
    # planted copies: groups of 2..10 equal round-0 keys, copies at the very
    # end (comparisons that run into the end of the text: prefix order), and
    # copies differing only deep inside (LCP far beyond the round-0 depth).
    for trial in range(12):
        n = int(rng.integers(20_000, 200_000))
        data = workloads.iid_dna(n, 100 + trial).copy()
        L = int(rng.integers(20, 200))
        src = int(rng.integers(0, n // 2))
        block = data[src:src + L].copy()
        copies = int(rng.integers(1, 10))
        for c in range(copies):
            dst = int(rng.integers(n // 2, n - L))
            data[dst:dst + L] = block
            if c % 3 == 1:  # a late mutation: tie broken deep inside
                acgt = np.frombuffer(b"ACGT", np.uint8)
                data[dst + L - 1] = acgt[(int(np.flatnonzero(acgt == data[dst + L - 1])[0]) + 1) % 4]
        data[n - L:] = block  # suffix of the text equal to an earlier substring
        want = oracle.build_suffix_structures(data)
        s = rb.build_suffix_structures(rb.Text(data))
        assert all(np.array_equal(a, b) for a, b in zip((s.sa, s.rank, s.lcp), want)), trial
        wl, wo, wf = oracle.all_positions(data, mode="all", structures=want)
        A = rb.all_positions(rb.Text(data), mode="all")
        assert np.array_equal(A.lengths, wl) and np.array_equal(A.offsets, wo), trial
        assert np.array_equal(A.flat_starts, wf), trial


def test_distributed_suffix_sort_loopback():
    # the distributed suffix sort + scan with 1..5 ranks
    # simulated on one GPU (one context per rank, exchanges as device copies)
    from paper_1501_06663_b200 import distributed as D
    cases = [workloads.iid_dna(300_000, 21), workloads.iid_dna(70_000, 22)]
    data = workloads.iid_dna(200_000, 23).copy()
    rng = np.random.default_rng(23)
    for c in range(6):  # a few planted copies: tied groups of 2..7 suffixes
        src, dst = int(rng.integers(0, 90_000)), int(rng.integers(100_000, 199_000))
        data[dst:dst + 50] = data[src:src + 50]
    cases.append(data)
    data = workloads.iid_dna(150_000, 24).copy()
    data[-40:] = data[1000:1040]  # a repeat that runs into the end of the text
    cases.append(data)
    for ci, data in enumerate(cases):
        wl, wo, wf = oracle.all_positions(data, mode="all")
        ws, wln = oracle.all_positions(data, mode="leftmost")
        for world in (1, 2, 3, 5):
            got = D.loopback_dist_all_positions(data, world, "all")
            assert got is not None, (ci, world)
            assert np.array_equal(got[0], wl) and np.array_equal(got[1], wo), (ci, world)
            assert np.array_equal(got[2], wf), (ci, world)
        got = D.loopback_dist_all_positions(data, 4, "leftmost")
        assert np.array_equal(got[0], ws) and np.array_equal(got[1], wln), ci


def test_distributed_suffix_sort_large_groups():
    # tied round-0 groups above 8 suffixes (planted repeat families) are sorted
    # per group on their rank (k_large_groups_seg); > 2048 members declines
    from paper_1501_06663_b200 import distributed as D
    rng = np.random.default_rng(41)
    data = workloads.iid_dna(400_000, 41).copy()
    for fam, copies in ((0, 40), (1, 300), (2, 12)):
        src = rng.integers(0, 4, 250).astype(np.uint8)
        src = np.frombuffer(b"ACGT", np.uint8)[src]
        for _ in range(copies):
            dst = int(rng.integers(0, data.size - 250))
            seg = src.copy()
            mut = rng.random(250) < 0.03  # diverged copies: many distinct LCPs
            seg[mut] = np.frombuffer(b"ACGT", np.uint8)[rng.integers(0, 4, int(mut.sum()))]
            data[dst:dst + 250] = seg
    wl, wo, wf = oracle.all_positions(data, mode="all")
    ws, wln = oracle.all_positions(data, mode="leftmost")
    for world in (1, 2, 3):
        got = D.loopback_dist_all_positions(data, world, "all")
        assert got is not None, world
        assert np.array_equal(got[0], wl) and np.array_equal(got[1], wo) and np.array_equal(got[2], wf), world
    got = D.loopback_dist_all_positions(data, 2, "leftmost")
    assert np.array_equal(got[0], ws) and np.array_equal(got[1], wln)
    big = workloads.iid_dna(100_000, 42).copy()
    for dst in rng.choice(big.size // 32 - 1, 2500, replace=False) * 32:  # one 16-mer in 2500 places
        big[dst:dst + 16] = np.frombuffer(b"ACGTTGCAACGTTGCA", np.uint8)
    assert D.loopback_dist_all_positions(big, 2, "all") is None


def test_distributed_suffix_sort_more_ranks_than_buckets():
    # n = 10000 -> 3 position buckets: with 5 or 7 ranks some position shards
    # (and SA segments) are empty, between non-empty ones; the halo comes from
    # the nearest non-empty shard
    from paper_1501_06663_b200 import distributed as D
    data = workloads.iid_dna(10_000, 31)
    wl, wo, wf = oracle.all_positions(data, mode="all")
    for world in (4, 5, 7):
        got = D.loopback_dist_all_positions(data, world, "all")
        assert got is not None, world
        assert np.array_equal(got[0], wl) and np.array_equal(got[1], wo) and np.array_equal(got[2], wf), world


def test_distributed_suffix_sort_declines_repetitive_text():
    from paper_1501_06663_b200 import distributed as D
    data = workloads.periodic_mutated(50_000, 3, period=7, rate=0.0)
    assert D.loopback_dist_all_positions(data, 2, "all") is None


def test_given_sa_only_used_when_it_inverts_rank(rng):
    """rs_set_structures with sa: raw LLR comes from SA order only when sa is
    exactly the inverse of rank (checked on device); a permuted or
    non-permutation sa must not change the answers, which the reference
    derives from rank and lcp alone (_kernels_numba.py:33-38)."""
    from paper_1501_06663_b200 import _native
    ctx = _native.context()
    data = workloads.iid_dna(200_000, 21)
    n = data.size
    s = rb.build_suffix_structures(rb.Text(data))
    want = rb.all_positions(rb.Text(data), mode="all")
    bad_perm = s.sa.copy()
    bad_perm[[5, 9]] = bad_perm[[9, 5]]
    dup = s.sa.copy()
    dup[100:200] = dup[300]
    for sa in (s.sa, bad_perm, dup):
        sa = np.ascontiguousarray(sa, np.int64)
        total = np.zeros(1, np.int64)
        with ctx.lock:
            ctx.call("rs_set_structures", _native.i64(sa), _native.i64(np.ascontiguousarray(s.rank)),
                     _native.i64(np.ascontiguousarray(s.lcp)), n)
            ctx.call("rs_query", 1, 1, _native.i64(total))
            L = np.empty(n + 1, np.int64)
            O = np.empty(n + 2, np.int64)
            F = np.empty(int(total[0]), np.int64)
            ctx.call("rs_fetch_all", _native.i64(L), _native.i64(O), _native.i64(F))
        assert np.array_equal(L, want.lengths) and np.array_equal(O, want.offsets)
        assert np.array_equal(F, want.flat_starts)


def test_large_transfers_through_the_pipeline(rng):
    """csrc/host_io.cu: results above the staging threshold travel as 32-bit
    words and are widened on the host (offsets rebuilt from their low words);
    pinned and pageable destinations, fresh and reused pool blocks."""
    data = workloads.iid_dna(9_000_000, 5)
    import oracle
    os_ = oracle.build_suffix_structures(data, workers=8)
    want = oracle.all_positions(data, mode="all", path="compact", workers=8, structures=os_)
    for pinned in (False, True, False):
        A = rb.all_positions(rb.Text(data), mode="all", pinned=pinned)
        assert np.array_equal(A.lengths, want[0]) and np.array_equal(A.offsets, want[1])
        assert np.array_equal(A.flat_starts, want[2])
    L = rb.all_positions(rb.Text(data), mode="leftmost")
    st, ln = oracle.all_positions(data, mode="leftmost", path="compact", workers=8, structures=os_)
    assert np.array_equal(L.starts, st) and np.array_equal(L.lengths, ln)
    s = rb.build_suffix_structures(rb.Text(data))
    assert rb.verify_suffix_structures(rb.Text(data), s)
    raw = rb.build_raw_llr(s)
    assert np.array_equal(raw, oracle.build_raw_llr(s.rank, s.lcp, 8))


@pytest.mark.parametrize("structures_from", ["device", "caller"])
def test_structures_shards_assemble_to_full_answer(structures_from):
    """rs_query_structures_shard (multi-GPU query from resident structures):
    each shard computes raw LLR for its slots plus a max-LCP left halo and
    scans; stitched shards == the full answer (fused path, and the raw-path
    fallback of long repeats: Fibonacci)."""
    from paper_1501_06663_b200 import _native
    from paper_1501_06663_b200 import distributed as D
    ctx = _native.context()
    for data in (workloads.iid_dna(250_000, 31), workloads.planted_dna(300_000, 9, family_len=200),
                 workloads.english_like(200_000, 4), workloads.fibonacci_mutated(150_000, 5, rate=1e-3)):
        n = data.size
        st = oracle.build_suffix_structures(data, workers=8)
        want_l, want_o, want_f = oracle.all_positions(data, mode="all", workers=8, structures=st)
        want_s, want_len = oracle.all_positions(data, mode="leftmost", workers=8, structures=st)
        with ctx.lock:
            if structures_from == "device":
                ctx.call("rs_set_text", _native.u8(data), n)
                ctx.call("rs_build_structures")
            else:
                ctx.call("rs_set_structures", _native.i64(st[0]), _native.i64(st[1]), _native.i64(st[2]), n)
        for world in (1, 2, 3, 7):
            lengths = np.zeros(n + 1, np.int64)
            offsets = np.zeros(n + 2, np.int64)
            starts = np.full(n + 1, -1, np.int64)
            llen = np.zeros(n + 1, np.int64)
            flats, base = [], 0
            for r in range(world):
                lo, hi = D.shard_range(n, world, r)
                with ctx.lock:
                    tot = np.zeros(1, np.int64)
                    ctx.call("rs_query_structures_shard", 1, lo, hi, _native.i64(tot))
                    ctx.call("rs_shard_rebase", base)
                    a = np.zeros(hi - lo, np.int64)
                    b = np.zeros(hi - lo + 1, np.int64)
                    f = np.zeros(int(tot[0]), np.int64)
                    ctx.call("rs_fetch_shard", 1, _native.i64(a), _native.i64(b), _native.i64(f))
                    ctx.call("rs_query_structures_shard", 0, lo, hi, _native.i64(tot))
                    s_ = np.zeros(hi - lo, np.int64)
                    l_ = np.zeros(hi - lo, np.int64)
                    ctx.call("rs_fetch_shard", 0, _native.i64(s_), _native.i64(l_), _native.i64(f[:0]))
                assert b[0] == base
                lengths[lo:hi] = a
                offsets[lo + 1:hi + 1] = b[1:]
                flats.append(f)
                base += f.size
                starts[lo:hi] = s_
                llen[lo:hi] = l_
            assert np.array_equal(lengths, want_l), world
            assert np.array_equal(offsets, want_o), world
            assert np.array_equal(np.concatenate(flats), want_f), world
            assert np.array_equal(starts, want_s) and np.array_equal(llen, want_len), world


@pytest.mark.parametrize("n", [(1 << 20) - 1, (1 << 24) + 1])
def test_transfer_pipeline_boundaries(n):
    """Answers that cross the staging threshold (2^20 values) and the
    pipeline's 2^24-value chunks, fetched into pageable (pipeline only) and
    page-locked (30% direct DMA + pipeline) arrays: identical, and correct by
    the independent checker (count_wrong_answers)."""
    from paper_1501_06663_b200.query import count_wrong_answers
    data = workloads.iid_dna(n, 77)
    t = rb.Text(data)
    A = rb.all_positions(t, mode="all")
    P = rb.all_positions(t, mode="all", pinned=True)
    assert np.array_equal(A.lengths, P.lengths) and np.array_equal(A.offsets, P.offsets)
    assert np.array_equal(A.flat_starts, P.flat_starts)
    L = rb.all_positions(t, mode="leftmost", pinned=True)
    c = rb.build_compact_llr(rb.build_raw_llr(rb.build_suffix_structures(t)))
    assert count_wrong_answers(c, n, all_answers=A, leftmost=L) == 0


def test_new_entry_points_errors():
    """Status codes of the round-2 entry points map to the reference's
    exception types (_native._raise): bad order -> RepeatscanError(ESTATE),
    bad ranges -> IndexError, bad arguments -> ValueError."""
    from paper_1501_06663_b200 import _native
    ctx = _native.Context(0)  # a fresh context: nothing loaded, no communicator
    try:
        tot = np.zeros(1, np.int64)
        with pytest.raises(_native.RepeatscanError):
            ctx.call("rs_query_structures_shard", 1, 1, 2, _native.i64(tot))
        with pytest.raises(_native.RepeatscanError):
            ctx.call("rs_clear_llr")
        with pytest.raises(_native.RepeatscanError):
            ctx.call("rs_nccl_allgather_i64", 1, _native.i64(tot))
        data = workloads.iid_dna(1000, 3)
        ctx.call("rs_set_text", _native.u8(data), data.size)
        ctx.call("rs_build_structures")
        with pytest.raises(IndexError):
            ctx.call("rs_query_structures_shard", 1, 0, 5, _native.i64(tot))
        with pytest.raises(IndexError):
            ctx.call("rs_query_structures_shard", 1, 10, 2000, _native.i64(tot))
        with pytest.raises(ValueError):
            ctx.call("rs_query_structures_shard", 7, 1, 5, _native.i64(tot))
        ctx.call("rs_query_structures_shard", 1, 5, 5, _native.i64(tot))  # empty shard
        assert tot[0] == 0
        bad = np.zeros(1, np.int64)
        with pytest.raises(ValueError):  # m > n
            ctx.call("rs_check_answers", _native.i64(bad), _native.i64(bad), 5, 1, None, None, None, 0,
                     None, None, _native.i64(bad))
        s = rb.build_suffix_structures(rb.Text(data))
        rank = s.rank.copy()
        rank[3] = 0  # out of 1..n
        with pytest.raises(ValueError):
            ctx.call("rs_set_structures", _native.i64(s.sa), _native.i64(rank), _native.i64(s.lcp), data.size)
    finally:
        ctx.close()


def _all_with_wire(t, word: bool, mode: str = "all"):
    from paper_1501_06663_b200 import _native
    ctx = _native.context()
    prev = os.environ.pop("RS_WORD_WIRE", None)
    if word:
        os.environ["RS_WORD_WIRE"] = "1"
    try:
        x0 = ctx.transfer_bytes()
        A = rb.all_positions(t, mode=mode, path="compact")
        x1 = ctx.transfer_bytes()
    finally:
        os.environ.pop("RS_WORD_WIRE", None)
        if prev is not None:
            os.environ["RS_WORD_WIRE"] = prev
    return A, x1[1] - x0[1]


@pytest.mark.parametrize("kind", ["iid", "planted", "fibonacci"])
def test_byte_wire_matches_word_wire(kind):
    """csrc/host_io.cu fetch_csr_bytes: the all-ties CSR crosses PCIe as one
    byte per value (u8 lengths, u8 tie counts, i8 start steps; int64 samples
    every 2^16 values) and the host rebuilds the int64 arrays.  Identical to
    the 32-bit wire; a text whose values do not fit (long repeats: Fibonacci)
    falls back to the 32-bit wire by itself."""
    data = {"iid": lambda: workloads.iid_dna(9_000_000, 41),
            "planted": lambda: workloads.planted_dna(6_000_000, 4, family_len=300),
            "fibonacci": lambda: workloads.fibonacci_mutated(5_000_000, 3, rate=1e-4)}[kind]()
    t = rb.Text(data)
    A, d2h_bytes = _all_with_wire(t, word=False)
    W, d2h_words = _all_with_wire(t, word=True)
    assert np.array_equal(A.lengths, W.lengths) and np.array_equal(A.offsets, W.offsets)
    assert np.array_equal(A.flat_starts, W.flat_starts)
    n, T = data.size, A.flat_starts.size
    assert d2h_words >= 4 * (2 * n + T)  # 32-bit words (+ small readbacks)
    if kind == "iid":  # short repeats: the byte wire was used
        assert d2h_bytes < 2 * n + T + (1 << 20), (d2h_bytes, n, T)
    if kind == "fibonacci":  # lengths far above 255: the mixed-width wire (test_mixed_width_wire)
        assert int(A.lengths.max()) > 255 and d2h_bytes < 4 * (2 * n + T)
    L, d2h_lb = _all_with_wire(t, word=False, mode="leftmost")
    LW, _ = _all_with_wire(t, word=True, mode="leftmost")
    assert np.array_equal(L.starts, LW.starts) and np.array_equal(L.lengths, LW.lengths)
    if kind == "iid":  # 2 bytes per position
        assert d2h_lb < 2 * n + (1 << 20), (d2h_lb, n)
    from paper_1501_06663_b200.query import count_wrong_answers
    c = rb.build_compact_llr(rb.build_raw_llr(rb.build_suffix_structures(t)))
    assert count_wrong_answers(c, n, all_answers=A, leftmost=L) == 0


def test_byte_wire_shards():
    """rs_fetch_shard over the byte wire (shards of >= 4 Mi positions, CSR
    offsets rebased on device): stitched shards == the full answer."""
    from paper_1501_06663_b200 import _native
    from paper_1501_06663_b200 import distributed as D
    data = workloads.iid_dna(9_000_000, 43)
    n = data.size
    full = rb.all_positions(rb.Text(data), mode="all", path="compact")
    ctx = _native.context()
    with ctx.lock:
        ctx.call("rs_set_text", _native.u8(data), n)
        ctx.call("rs_build_structures")
    lengths = np.zeros(n + 1, np.int64)
    offsets = np.zeros(n + 2, np.int64)
    flats, base = [], 0
    for r in range(2):
        lo, hi = D.shard_range(n, 2, r)
        with ctx.lock:
            tot = np.zeros(1, np.int64)
            ctx.call("rs_query_structures_shard", 1, lo, hi, _native.i64(tot))
            ctx.call("rs_shard_rebase", base)
            a = np.zeros(hi - lo, np.int64)
            b = np.zeros(hi - lo + 1, np.int64)
            f = np.zeros(int(tot[0]), np.int64)
            x0 = ctx.transfer_bytes()
            ctx.call("rs_fetch_shard", 1, _native.i64(a), _native.i64(b), _native.i64(f))
            x1 = ctx.transfer_bytes()
        assert x1[1] - x0[1] < 2 * (hi - lo) + f.size + (1 << 20)  # byte wire
        assert b[0] == base
        lengths[lo:hi] = a
        offsets[lo + 1:hi + 1] = b[1:]
        flats.append(f)
        base += f.size
    assert np.array_equal(lengths, full.lengths) and np.array_equal(offsets, full.offsets)
    assert np.array_equal(np.concatenate(flats), full.flat_starts)
    left = rb.all_positions(rb.Text(data), mode="leftmost", path="compact")
    for r in range(2):  # leftmost shards: (length, distance) byte pairs
        lo, hi = D.shard_range(n, 2, r)
        with ctx.lock:
            tot = np.zeros(1, np.int64)
            ctx.call("rs_query_structures_shard", 0, lo, hi, _native.i64(tot))
            s_ = np.zeros(hi - lo, np.int64)
            l_ = np.zeros(hi - lo, np.int64)
            x0 = ctx.transfer_bytes()
            ctx.call("rs_fetch_shard", 0, _native.i64(s_), _native.i64(l_), _native.i64(np.zeros(0, np.int64)))
            x1 = ctx.transfer_bytes()
        assert x1[1] - x0[1] < 2 * (hi - lo) + (1 << 20)
        assert np.array_equal(s_, left.starts[lo:hi]) and np.array_equal(l_, left.lengths[lo:hi])


@pytest.mark.parametrize("kind", ["fibonacci", "periodic", "planted", "binary"])
def test_text_order_round_keys_match_list_keys(kind):
    """csrc/suffix_array.cu: doubling rounds with more than n/4 suffixes tied
    build their keys in text order from the flagged ISA heads
    (k_make_keys_text); RS_SA_LIST_KEYS=1 forces the slot-list gather.  Both
    give the oracle's structures, and the repetitive inputs do take rounds of
    each kind."""
    data = {"fibonacci": lambda: workloads.fibonacci_mutated(300_000, 7, rate=1e-3),
            "periodic": lambda: workloads.periodic_mutated(250_000, 3, period=977, rate=1e-3),
            "planted": lambda: workloads.planted_dna(400_000, 5, family_len=400),
            "binary": lambda: np.frombuffer(b"ab", np.uint8)[
                np.random.default_rng(2).integers(0, 2, 200_000)]}[kind]()
    want = oracle.build_suffix_structures(data, workers=8)
    t = rb.Text(data)
    prev = os.environ.pop("RS_SA_LIST_KEYS", None)
    try:
        for list_keys in (False, True):
            if list_keys:
                os.environ["RS_SA_LIST_KEYS"] = "1"
            s = rb.build_suffix_structures(t)
            os.environ.pop("RS_SA_LIST_KEYS", None)
            assert np.array_equal(s.sa, want[0]), (kind, list_keys)
            assert np.array_equal(s.rank, want[1]) and np.array_equal(s.lcp, want[2]), (kind, list_keys)
    finally:
        if prev is not None:
            os.environ["RS_SA_LIST_KEYS"] = prev


def test_mixed_width_wire():
    """csrc/host_io.cu fetch_csr_mixed: answers with values beyond a byte
    (long repeats) cross PCIe 1, 2 or 4 bytes per value chosen per 2^16
    block; identical to the 32-bit wire, and narrower than it."""
    data = workloads.fibonacci_mutated(6_000_000, 9, rate=2e-4)
    t = rb.Text(data)
    A, d2h_mixed = _all_with_wire(t, word=False)
    W, d2h_words = _all_with_wire(t, word=True)
    assert int(A.lengths.max()) > 255  # the byte wire cannot carry it
    assert np.array_equal(A.lengths, W.lengths) and np.array_equal(A.offsets, W.offsets)
    assert np.array_equal(A.flat_starts, W.flat_starts)
    n, T = data.size, A.flat_starts.size
    assert d2h_mixed < 0.6 * d2h_words, (d2h_mixed, d2h_words)
    L, d2h_lm = _all_with_wire(t, word=False, mode="leftmost")  # (length, position - start) per block width
    LW, d2h_lw = _all_with_wire(t, word=True, mode="leftmost")
    assert np.array_equal(L.starts, LW.starts) and np.array_equal(L.lengths, LW.lengths)
    assert d2h_lm < 0.6 * d2h_lw, (d2h_lm, d2h_lw)
    from paper_1501_06663_b200.query import count_wrong_answers
    c = rb.build_compact_llr(rb.build_raw_llr(rb.build_suffix_structures(t)))
    assert count_wrong_answers(c, n, all_answers=A, leftmost=L) == 0


def test_mixed_width_wire_shards():
    """rs_fetch_shard over the mixed-width wire (long repeats, shards of
    >= 4 Mi positions): stitched shards == the full answers."""
    from paper_1501_06663_b200 import _native
    from paper_1501_06663_b200 import distributed as D
    data = workloads.fibonacci_mutated(9_000_000, 13, rate=2e-4)
    n = data.size
    t = rb.Text(data)
    full = rb.all_positions(t, mode="all", path="compact")
    left = rb.all_positions(t, mode="leftmost", path="compact")
    assert int(full.lengths.max()) > 255
    ctx = _native.context()
    with ctx.lock:
        ctx.call("rs_set_text", _native.u8(data), n)
        ctx.call("rs_build_structures")
    flats, base = [], 0
    for r in range(2):
        lo, hi = D.shard_range(n, 2, r)
        with ctx.lock:
            tot = np.zeros(1, np.int64)
            ctx.call("rs_query_structures_shard", 1, lo, hi, _native.i64(tot))
            ctx.call("rs_shard_rebase", base)
            a = np.zeros(hi - lo, np.int64)
            b = np.zeros(hi - lo + 1, np.int64)
            f = np.zeros(int(tot[0]), np.int64)
            ctx.call("rs_fetch_shard", 1, _native.i64(a), _native.i64(b), _native.i64(f))
            ctx.call("rs_query_structures_shard", 0, lo, hi, _native.i64(tot))
            s_ = np.zeros(hi - lo, np.int64)
            l_ = np.zeros(hi - lo, np.int64)
            ctx.call("rs_fetch_shard", 0, _native.i64(s_), _native.i64(l_), _native.i64(np.zeros(0, np.int64)))
        assert np.array_equal(a, full.lengths[lo:hi]) and np.array_equal(b, full.offsets[lo:hi + 1])
        assert np.array_equal(s_, left.starts[lo:hi]) and np.array_equal(l_, left.lengths[lo:hi])
        flats.append(f)
        base += f.size
    assert np.array_equal(np.concatenate(flats), full.flat_starts)
