"""Multi-rank host logic of the sharded query, on CPU with gloo (world size 2 and 3).

Per-shard device results are stood in for by slices of the oracle's answer
(tests may use the oracle); everything else -- shard ranges, the tie-total
all_gather, CSR rebasing and the point-to-point gather into the reference
layout -- is the production code of paper_1501_06663_b200.distributed.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1501_06663_b200 import distributed as D


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, data, q):
    import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = data.size
        wl, wo, wf = oracle.all_positions(data, mode="all")
        ls, ll = oracle.all_positions(data, mode="leftmost")
        lo, hi = D.shard_range(n, world, rank)
        cnt = hi - lo
        # shard-local results as rs_query_shard produces them
        a = torch.from_numpy(wl[lo:hi].copy())
        local_off = wo[lo:hi + 1] - wo[lo]
        f = torch.from_numpy(wf[wo[lo]:wo[hi]].copy())
        totals = D.exchange_totals(int(f.numel()))
        bases = D.tie_bases(totals)
        b = torch.from_numpy(local_off + bases[rank])  # rs_shard_rebase
        out = D.gather_shards(n, "all", lo, hi, a, b, f, sum(totals), bases[rank])
        left = D.gather_shards(n, "leftmost", lo, hi, torch.from_numpy(ls[lo:hi].copy()),
                               torch.from_numpy(ll[lo:hi].copy()), None, 0, 0)
        if rank == 0:
            ok = (np.array_equal(out[0].numpy(), wl) and np.array_equal(out[1].numpy(), wo)
                  and np.array_equal(out[2].numpy(), wf) and np.array_equal(left[0].numpy(), ls)
                  and np.array_equal(left[1].numpy(), ll))
            q.put(("ok" if ok else "mismatch", cnt))
        else:
            assert out is None and left is None
    except Exception as e:  # surface errors to the parent
        q.put((f"error: {e!r}", rank))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_gather_matches_full_answer(world):
    from paper_1501_06663_b200 import workloads
    data = workloads.planted_dna(5000, 7, family_len=40)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, data, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    status, _ = q.get(timeout=10)
    assert status == "ok", status
    assert all(p.exitcode == 0 for p in procs)


def test_shard_ranges_partition():
    for n in (0, 1, 5, 7, 1000, 1001):
        for world in (1, 2, 3, 8):
            covered = []
            for r in range(world):
                lo, hi = D.shard_range(n, world, r)
                assert 1 <= lo <= hi <= n + 1
                covered += list(range(lo, hi))
            assert covered == list(range(1, n + 1))
    assert D.tie_bases([3, 0, 5]) == [0, 3, 3]


def test_dist_shard_partition():
    # distributed suffix sort: bucket-aligned position shards cover [0, n) exactly
    from paper_1501_06663_b200.distributed import dist_shard
    for n in (4096, 5000, 1 << 20, (1 << 20) + 7, 268435456, 1073741824):
        for world in (1, 2, 3, 5, 8):
            prev = 0
            for r in range(world):
                p0, p1 = dist_shard(n, r, world)
                assert p0 == prev and p1 >= p0
                prev = p1
            assert prev == n


def test_dist_neighbours():
    from paper_1501_06663_b200.distributed import dist_neighbours
    z = [0] * 16

    def info(m, fk, fp, lk, lp):
        i = list(z)
        i[0], i[1], i[3], i[4], i[5], i[6] = 1, m, fk, fp, lk, lp
        return i

    infos = [info(3, 10, 100, 11, 101), info(0, 0, 0, 0, 0), info(5, 20, 200, 21, 201), info(2, 30, 300, 31, 301)]
    nb = dist_neighbours(infos)
    assert nb[0] == [0, 0, 0, 20, 200, 1]           # next non-empty segment is rank 2
    assert nb[2] == [11, 101, 1, 30, 300, 1]        # previous non-empty is rank 0
    assert nb[3] == [21, 201, 1, 0, 0, 0]


def test_dist_halo_partners_skip_empty_shards():
    from paper_1501_06663_b200.distributed import dist_halo_fits, dist_halo_partners, dist_shard
    # 3 buckets over 5 ranks: shards 0 and 2 are empty
    shards = [dist_shard(10_000, r, 5) for r in range(5)]
    assert [b - a for a, b in shards] == [0, 4096, 0, 4096, 1808]
    assert dist_halo_partners(10_000, 5) == [(-1, 1), (-1, 3), (1, 3), (1, 4), (3, -1)]
    assert dist_halo_fits(10_000, 5, 4096) and not dist_halo_fits(10_000, 5, 4097)
    # the last non-empty shard never sends a halo, its size does not bound it
    assert dist_halo_fits(10_000, 3, 4000)


def _shared_worker(rank, world, port, data, q):
    """Every rank writes its shard's slices of ONE /dev/shm buffer (what
    rs_fetch_shard does from its GPU); rank 0 reads the whole answer back."""
    import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = data.size
        wl, wo, wf = oracle.all_positions(data, mode="all")
        ls, ll = oracle.all_positions(data, mode="leftmost")
        lo, hi = D.shard_range(n, world, rank)
        totals = D.exchange_totals(int(wo[hi] - wo[lo]))
        base = D.tie_bases(totals)[rank]
        assert base == wo[lo]
        out = {}
        for mode in ("all", "leftmost"):
            T = sum(totals) if mode == "all" else 0
            buf = D.SharedHostBuffer(sum(c for _, c in D.answer_layout(n, mode, T).values()))
            views = D.layout_views(buf.array, n, mode, T)
            a, b, f = D.shard_views(views, mode, lo, hi, base, totals[rank])
            if mode == "all":  # rebased shard: lengths, offsets[lo..hi], ties
                a[:] = wl[lo:hi]
                b[:] = wo[lo:hi + 1]
                f[:] = wf[wo[lo]:wo[hi]]
            else:
                a[:] = ls[lo:hi]
                b[:] = ll[lo:hi]
            if rank == 0:
                D.fill_pads(views, mode)
            dist.barrier()
            out[mode] = {k: v.copy() for k, v in views.items()}
            dist.barrier()
        # a released block is reused by the next call of the same size (warm pages)
        sizes = sum(c for _, c in D.answer_layout(n, "all", sum(totals)).values())
        b1 = D.SharedHostBuffer(sizes)
        p1 = b1.array.ctypes.data
        del b1
        import gc
        gc.collect()
        dist.barrier()
        b2 = D.SharedHostBuffer(sizes)
        reused = b2.array.ctypes.data == p1
        if rank == 0:
            assert reused, "released shared block not reused"
        del b2
        if rank == 0:
            A, L = out["all"], out["leftmost"]
            ok = (np.array_equal(A["lengths"], wl) and np.array_equal(A["offsets"], wo)
                  and np.array_equal(A["flat"], wf) and np.array_equal(L["starts"], ls)
                  and np.array_equal(L["lengths"], ll))
            q.put(("ok" if ok else "mismatch", 0))
    except Exception as e:
        q.put((f"error: {e!r}", rank))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_shared_host_output_assembles_full_answer(world):
    from paper_1501_06663_b200 import workloads
    data = workloads.planted_dna(6000, 9, family_len=50)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shared_worker, args=(r, world, port, data, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    status, _ = q.get(timeout=10)
    assert status == "ok", status
    assert all(p.exitcode == 0 for p in procs)
