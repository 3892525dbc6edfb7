"""Multi-GPU longest-repeat query on one box: one process per GPU.

Positions are independent reads of immutable candidate arrays with disjoint
output slots (engine.py:3-7), so the path shards by POSITION:

1. rank 0 builds the suffix structures, raw LLR and the compact array LLRc of
   the whole text on its GPU (the replicated-structures path,
   `sharded_all_positions`; `dist_sa_all_positions` further down shards the
   suffix sort itself -- SURVEY 8(f)#1 -- for texts without long repeats);
2. LLRc (8 bytes per entry) is broadcast with NCCL over NVLink, straight
   from/into the library's device buffers (zero-copy torch views);
3. rank r answers the contiguous position shard [lo_r, hi_r) of
   engine._chunks; its left halo -- the entries that start before lo_r but
   still cover it (at most max LLR - 1 positions back, Lemma 2) -- needs no
   extra exchange because every rank holds the global LLRc and the per-tile
   windows are found by binary search over it;
4. all-ties: the per-shard tie totals are all-gathered (one int64 each), each
   rank rebases its CSR offsets on device, and the shards are gathered to rank
   0 with NCCL point-to-point into the final reference-layout arrays.

Only plumbing (device views, NCCL collectives, final D2H) lives here; every
kernel is in librepeatscan_b200.so.  The host-side pieces (shard ranges, tie
bases, CSR assembly) are backend-agnostic so they are tested with gloo on CPU.
"""

from __future__ import annotations

import ctypes
import os
import time

import numpy as np

from paper_1501_06663_b200 import _native


# ---------------------------------------------------------------------------------------
# host-side logic (backend agnostic)
# ---------------------------------------------------------------------------------------
def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """1-based half-open position range of `rank` -- engine._chunks (engine.py:43-52)."""
    total = n
    parts = max(1, min(world, total)) if total > 0 else 1
    if rank >= parts:
        return n + 1, n + 1
    base, extra = divmod(total, parts)
    lo = 1 + rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def tie_bases(totals: list[int]) -> list[int]:
    """Exclusive prefix of the per-shard tie totals (CSR base of each shard)."""
    out, acc = [], 0
    for t in totals:
        out.append(acc)
        acc += int(t)
    return out


def exchange_totals(total: int, group=None, device=None) -> list[int]:
    """all_gather of one int64 per rank."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    t = torch.tensor([int(total)], dtype=torch.int64, device=device)
    parts = [torch.zeros(1, dtype=torch.int64, device=device) for _ in range(world)]
    dist.all_gather(parts, t, group=group)
    return [int(p.item()) for p in parts]


def gather_shards(n: int, mode: str, lo: int, hi: int, a, b, flat, total_all: int, base: int,
                  group=None, device=None, ranges=None):
    """Assemble the reference-layout arrays on rank 0 from every rank's shard.

    a, b, flat are torch tensors of this rank's shard (leftmost: a=starts[cnt],
    b=lengths[cnt]; all: a=lengths[cnt], b=offsets[cnt+1] already rebased,
    flat=tie starts[T_r]).  ranges: every rank's 1-based [lo, hi) (default:
    shard_range).  Returns the full torch tensors on rank 0, else None.
    """
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    cnt = hi - lo
    if rank != 0:
        if cnt > 0:
            dist.send(a[:cnt].contiguous(), dst=0, group=group)
            if mode == "all":
                dist.send(b[1:cnt + 1].contiguous(), dst=0, group=group)  # offsets[k+1]
                if flat is not None and flat.numel() > 0:
                    dist.send(flat.contiguous(), dst=0, group=group)
            else:
                dist.send(b[:cnt].contiguous(), dst=0, group=group)
        return None
    kw = dict(dtype=torch.int64, device=device)
    if mode == "leftmost":
        starts = torch.empty(n + 1, **kw)
        lengths = torch.empty(n + 1, **kw)
        starts[0] = -1
        lengths[0] = 0
        starts[lo:hi] = a[:cnt]
        lengths[lo:hi] = b[:cnt]
        for r in range(1, world):
            rlo, rhi = ranges[r] if ranges else shard_range(n, world, r)
            if rhi > rlo:
                dist.recv(starts[rlo:rhi], src=r, group=group)
                dist.recv(lengths[rlo:rhi], src=r, group=group)
        return starts, lengths
    lengths = torch.empty(n + 1, **kw)
    offsets = torch.empty(n + 2, **kw)
    flat_all = torch.empty(max(total_all, 0), **kw)
    lengths[0] = 0
    offsets[0] = 0
    offsets[1] = 0
    if cnt > 0:
        lengths[lo:hi] = a[:cnt]
        # b[0] is the exclusive base of the shard's first position; b[1:] are offsets[k+1]
        offsets[lo + 1:hi + 1] = b[1:cnt + 1]
        t0 = int(b[0].item()) if hasattr(b[0], "item") else int(b[0])
        if flat is not None and flat.numel() > 0:
            flat_all[t0:t0 + flat.numel()] = flat
    for r in range(1, world):
        rlo, rhi = ranges[r] if ranges else shard_range(n, world, r)
        if rhi <= rlo:
            continue
        dist.recv(lengths[rlo:rhi], src=r, group=group)
        tmp = torch.empty(rhi - rlo, **kw)
        dist.recv(tmp, src=r, group=group)
        offsets[rlo + 1:rhi + 1] = tmp
        s = int(offsets[rlo].item())
        e = int(offsets[rhi].item())
        if e > s:
            dist.recv(flat_all[s:e], src=r, group=group)
    return lengths, offsets, flat_all


# ---------------------------------------------------------------------------------------
# shared host output: every rank D2Hs its shard into its slice of ONE host buffer
# (SURVEY 8(e) collectives, step 4) -- no gather through rank 0's GPU / PCIe link
# ---------------------------------------------------------------------------------------
def answer_layout(n: int, mode: str, total: int) -> dict:
    """Element offsets of the reference arrays inside one int64 buffer."""
    if mode == "leftmost":
        return {"starts": (0, n + 1), "lengths": (n + 1, n + 1)}
    return {"lengths": (0, n + 1), "offsets": (n + 1, n + 2), "flat": (2 * n + 3, max(total, 0))}


def layout_views(buf: np.ndarray, n: int, mode: str, total: int) -> dict:
    return {k: buf[o:o + c] for k, (o, c) in answer_layout(n, mode, total).items()}


def shard_views(views: dict, mode: str, lo: int, hi: int, base: int, t_shard: int):
    """The slices one rank's shard fills (rs_fetch_shard's a, b, flat):
    all: lengths[lo:hi], offsets[lo:hi+1] (offsets[lo] = the shard's base, written
    identically by the previous shard), flat[base:base+T_r]; leftmost: starts, lengths."""
    if mode == "leftmost":
        return views["starts"][lo:hi], views["lengths"][lo:hi], None
    return views["lengths"][lo:hi], views["offsets"][lo:hi + 1], views["flat"][base:base + t_shard]


def fill_pads(views: dict, mode: str) -> None:
    """Slot-0 pads of the reference layout (query.py:174-175, 190-204)."""
    if mode == "leftmost":
        views["starts"][0] = -1
        views["lengths"][0] = 0
    else:
        views["lengths"][0] = 0
        views["offsets"][0] = 0
        views["offsets"][1] = 0


class _SharedBlock:
    """One /dev/shm file mapped in this process."""
    __slots__ = ("path", "nbytes", "mm", "__weakref__")

    def __init__(self, path: str, nbytes: int):
        import mmap
        fd = os.open(path, os.O_RDWR)
        try:
            self.mm = mmap.mmap(fd, nbytes, mmap.MAP_SHARED, mmap.PROT_READ | mmap.PROT_WRITE)
        finally:
            os.close(fd)
        self.path, self.nbytes = path, nbytes


_shared_maps: dict[str, _SharedBlock] = {}   # every rank: path -> mapping
_shared_free: list[tuple[str, int]] = []      # rank 0: blocks whose answers were released
_shared_files: list[str] = []                 # rank 0: files to remove at exit


def _remove_shared_files():
    for path in _shared_files:
        try:
            os.unlink(path)
        except OSError:
            pass


class SharedHostBuffer:
    """One int64 host buffer mapped by every rank of the node (a /dev/shm
    file).  Blocks are cached like the library's host pools: when the arrays
    rank 0 handed out are released, the block (already page-faulted on every
    rank) serves the next call -- fresh tmpfs pages cost far more to fault in
    than the transfer itself.  Raises MemoryError when /dev/shm cannot hold a
    new block (callers fall back to the NCCL gather)."""

    def __init__(self, nelems: int, group=None, root: str = "/dev/shm"):
        import atexit
        import uuid

        import torch.distributed as dist
        rank = dist.get_rank(group)
        need = max(8 * int(nelems), 8)
        name = [None, 0, None]
        if rank == 0:
            fit = [blk for blk in _shared_free if blk[1] >= need]
            if fit:
                blk = min(fit, key=lambda b_: b_[1])
                _shared_free.remove(blk)
                name = [blk[0], blk[1], None]
            else:
                nbytes = 1 << 20
                while nbytes < need:
                    nbytes <<= 1
                try:
                    st = os.statvfs(root)
                    free = st.f_bavail * st.f_frsize
                except OSError:
                    free = 0
                if free >= nbytes + (64 << 20):
                    path = os.path.join(root, f"repeatscan_{os.getpid()}_{uuid.uuid4().hex[:12]}")
                    fd = os.open(path, os.O_CREAT | os.O_EXCL | os.O_RDWR, 0o600)
                    os.ftruncate(fd, nbytes)
                    os.close(fd)
                    if not _shared_files:
                        atexit.register(_remove_shared_files)
                    _shared_files.append(path)
                    name = [path, nbytes, None]
                else:
                    name = [None, 0, f"{root} has {free} bytes free, {nbytes} needed"]
        dist.broadcast_object_list(name, src=0, group=group)
        if name[0] is None:
            raise MemoryError(name[2])
        blk = _shared_maps.get(name[0])
        if blk is None or blk.nbytes != name[1]:
            blk = _SharedBlock(name[0], int(name[1]))
            _shared_maps[name[0]] = blk
        dist.barrier(group=group)
        # owner of the returned arrays: the block goes back to rank 0's free
        # list when the last view of them dies
        import ctypes as _ct
        import weakref
        raw = (_ct.c_char * blk.nbytes).from_buffer(blk.mm)
        if rank == 0:
            weakref.finalize(raw, _shared_free.append, (blk.path, blk.nbytes))
        self.array = np.frombuffer(raw, dtype=np.int64, count=int(nelems))


def fetch_shard_shared(ctx, n: int, mode: str, lo: int, hi: int, base: int, totals: list[int],
                       group=None):
    """Every rank copies its (rebased) shard from its GPU into its slice of one
    shared host buffer (csrc/host_io.cu pipeline, its own PCIe link and host
    threads); rank 0 returns the reference dataclass backed by that buffer."""
    import torch.distributed as dist

    from paper_1501_06663_b200.query import AllAnswers, LeftmostAnswers
    rank = dist.get_rank(group)
    T_all = int(sum(totals)) if mode == "all" else 0
    views = layout_views(SharedHostBuffer(sum(c for _, c in answer_layout(n, mode, T_all).values()),
                                          group).array, n, mode, T_all)
    a, b, f = shard_views(views, mode, lo, hi, base, int(totals[rank]) if mode == "all" else 0)
    if hi > lo:
        null = ctypes.POINTER(ctypes.c_int64)()
        ctx.call("rs_fetch_shard", _native.MODE[mode], _native.i64(a), _native.i64(b),
                 _native.i64(f) if f is not None and f.size else null)
    if rank == 0:
        fill_pads(views, mode)
    dist.barrier(group=group)
    if rank != 0:
        return None
    if mode == "leftmost":
        return LeftmostAnswers(starts=views["starts"], lengths=views["lengths"])
    return AllAnswers(lengths=views["lengths"], offsets=views["offsets"], flat_starts=views["flat"])


# ---------------------------------------------------------------------------------------
# device path
# ---------------------------------------------------------------------------------------
class _CudaView:
    """__cuda_array_interface__ view of a library device buffer (no copy)."""

    def __init__(self, ptr: int, count: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


def _view(ctx: _native.Context, which: int, count: int, typestr: str, device):
    import torch
    itemsize = int(typestr[-1])
    ptr = ctx.device_buffer(which, max(count, 1) * itemsize)
    return torch.as_tensor(_CudaView(ptr, count, typestr), device=device)


def sharded_all_positions(data: np.ndarray | None, mode: str = "all", group=None,
                          timings: dict | None = None, resident: bool = False, gather: bool = True):
    """Distributed query.  `data` (uint8 text) is needed on rank 0 only.

    Returns torch device tensors of the reference layout on rank 0
    ((starts, lengths) or (lengths, offsets, flat)), None elsewhere.
    resident=True: rank 0 reuses the text already on its device (derived
    arrays are rebuilt); gather=False: every rank keeps its shard of the
    answer (rebased CSR) in its own HBM and the call returns None.
    """
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev_index = torch.cuda.current_device()
    device = torch.device("cuda", dev_index)
    ctx = _native.context(dev_index)
    t = {} if timings is None else timings
    with ctx.lock:
        # 1. rank 0: text -> SA -> LCP -> raw LLR -> LLRc on its GPU
        meta = torch.zeros(2, dtype=torch.int64, device=device)
        if rank == 0:
            if resident:
                n = int(data.size)
                ctx.call("rs_clear_derived")
            else:
                host = np.ascontiguousarray(data, dtype=np.uint8)
                n = int(host.size)
                ctx.call("rs_set_text", _native.u8(host), n)
            m_arr = np.zeros(1, np.int64)
            ctx.call("rs_get_compact_size", _native.i64(m_arr))
            ctx.synchronize()
            meta[0], meta[1] = n, int(m_arr[0])
        dist.broadcast(meta, src=0, group=group)
        n, m = int(meta[0].item()), int(meta[1].item())
        # 2. LLRc broadcast, device buffer to device buffer (uint32 pairs)
        llrc = _view(ctx, _native.BUF_LLRC, 2 * m + 8, "<i4", device)  # (start, len) u32 pairs, bit-cast
        if m > 0:
            dist.broadcast(llrc[:2 * m], src=0, group=group)
        torch.cuda.synchronize(device)
        if rank != 0:
            ctx.call("rs_set_compact_device", m, n)
        # 3. shard scan
        lo, hi = shard_range(n, world, rank)
        total = np.zeros(1, np.int64)
        ctx.call("rs_query_shard", _native.MODE[mode], lo, hi, _native.i64(total))
        cnt = hi - lo
        if mode == "all":
            totals = exchange_totals(int(total[0]), group, device)
            bases = tie_bases(totals)
            ctx.call("rs_shard_rebase", bases[rank])
            T_all = sum(totals)
            if not gather:
                ctx.synchronize()
                return None
            a = _view(ctx, _native.BUF_OUT0, cnt, "<i8", device)
            b = _view(ctx, _native.BUF_OUT1, cnt + 1, "<i8", device)
            f = _view(ctx, _native.BUF_FLAT, int(total[0]), "<i8", device)
            ctx.synchronize()
            out = gather_shards(n, mode, lo, hi, a, b, f, T_all, bases[rank], group, device)
        else:
            if not gather:
                ctx.synchronize()
                return None
            a = _view(ctx, _native.BUF_OUT0, cnt, "<i8", device)
            b = _view(ctx, _native.BUF_OUT1, cnt, "<i8", device)
            ctx.synchronize()
            out = gather_shards(n, mode, lo, hi, a, b, None, 0, 0, group, device)
        torch.cuda.synchronize(device)
    return out


def library_comm(ctx, group=None) -> bool:
    """The library's own NCCL communicator for `group` (csrc/collectives.cu),
    created once per context: rank 0's 128-byte ncclUniqueId travels over
    torch.distributed (bootstrap only); every collective of the data plane
    then runs inside the library on its stream.  False for non-NCCL groups
    (gloo: host-logic tests), which keep the torch collectives."""
    import torch.distributed as dist
    if dist.get_backend(group) != "nccl":
        return False
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    key = (world, tuple(dist.get_process_group_ranks(group)) if group is not None else None)
    if getattr(ctx, "_nccl_key", None) == key:
        return True
    idb = [None]
    if rank == 0:
        raw = (ctypes.c_uint8 * 128)()
        rc = ctx.lib.rs_nccl_unique_id(raw)
        if rc != _native.RS_OK:
            raise _native.RepeatscanError(f"rs_nccl_unique_id failed with status {rc}")
        idb = [bytes(raw)]
    src = dist.get_global_rank(group, 0) if group is not None else 0
    dist.broadcast_object_list(idb, src=src, group=group)
    arr = (ctypes.c_uint8 * 128).from_buffer_copy(idb[0])
    ctx.call("rs_nccl_init", arr, rank, world)
    ctx._nccl_key = key
    return True


def allgather_i64(ctx, value: int, group=None, device=None) -> list[int]:
    """One int64 per rank, rank order: NCCL inside the library when the group
    is NCCL, else the torch collective (gloo)."""
    import torch.distributed as dist
    if library_comm(ctx, group):
        out = np.zeros(dist.get_world_size(group), np.int64)
        ctx.call("rs_nccl_allgather_i64", int(value), _native.i64(out))
        return [int(v) for v in out]
    return exchange_totals(int(value), group, device)


def structures_query_shard(ctx, n: int, mode: str, group=None, device=None) -> tuple:
    """Query step from the suffix structures resident on every rank's GPU:
    rank r answers shard_range(n, world, r) (rs_query_structures_shard: raw LLR
    of its slots and left halo, fused scan -- no data exchange), tie totals are
    all-gathered and the shard's CSR offsets rebased on device.
    Returns (lo, hi, base, totals)."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    lo, hi = shard_range(n, world, rank)
    total = np.zeros(1, np.int64)
    ctx.call("rs_query_structures_shard", _native.MODE[mode], lo, hi, _native.i64(total))
    if mode != "all":
        return lo, hi, 0, [0] * world
    totals = allgather_i64(ctx, int(total[0]), group, device)
    base = tie_bases(totals)[rank]
    ctx.call("rs_shard_rebase", base)
    return lo, hi, base, totals


def replicated_all_positions(data: np.ndarray | None, mode: str = "all", group=None):
    """API-level multi-GPU all_positions (query.py:218-239) over the ranks of
    `group`: rank 0's host text is copied to its GPU and broadcast over NVLink,
    every rank builds the suffix structures on its own GPU (no exchange during
    the sort), answers its position shard from them, and D2Hs its rebased shard
    into one shared host buffer.  Rank 0 returns the reference dataclass."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    dev_index = torch.cuda.current_device()
    device = torch.device("cuda", dev_index)
    ctx = _native.context(dev_index)
    with ctx.lock:
        n = allgather_i64(ctx, int(data.size) if rank == 0 else 0, group, device)[0]
        if rank == 0:
            ctx.call("rs_set_text", _native.u8(np.ascontiguousarray(data, dtype=np.uint8)), n)
        if library_comm(ctx, group):  # NCCL broadcast inside the library, device buffer to device buffer
            ctx.call("rs_nccl_broadcast_text", n, 0)
        else:
            tv = _view(ctx, _native.BUF_TEXT, n + 128, "|u1", device)[:n]
            torch.cuda.synchronize(device)
            dist.broadcast(tv, src=0, group=group)
            torch.cuda.synchronize(device)
            ctx.call("rs_set_text_device", n)
        ctx.call("rs_build_structures")
        lo, hi, base, totals = structures_query_shard(ctx, n, mode, group, device)
        try:
            return fetch_shard_shared(ctx, n, mode, lo, hi, base, totals, group)
        except MemoryError:
            cnt = hi - lo
            a = _view(ctx, _native.BUF_OUT0, cnt, "<i8", device)
            b = _view(ctx, _native.BUF_OUT1, cnt + 1, "<i8", device)
            f = _view(ctx, _native.BUF_FLAT, int(totals[rank]), "<i8", device) if mode == "all" else None
            ctx.synchronize()
            out = gather_shards(n, mode, lo, hi, a, b, f, int(sum(totals)), base, group, device)
            return to_answers(out, mode) if rank == 0 else None


def _to_host(t):
    """One D2H of a device tensor into a pooled pinned numpy array (full PCIe rate)."""
    import torch
    arr = _native.pinned_pool.empty(int(t.numel()), np.int64)
    if arr.size:
        torch.from_numpy(arr).copy_(t, non_blocking=True)
    return arr


def to_answers(out, mode: str):
    """Rank-0 tensors -> reference dataclasses (one D2H each, pinned)."""
    import torch
    from paper_1501_06663_b200.query import AllAnswers, LeftmostAnswers
    if mode == "leftmost":
        s, l = out
        res = LeftmostAnswers(starts=_to_host(s), lengths=_to_host(l))
    else:
        l, o, f = out
        res = AllAnswers(lengths=_to_host(l), offsets=_to_host(o), flat_starts=_to_host(f))
    torch.cuda.synchronize()
    return res


# ---------------------------------------------------------------------------------------
# bench (torchrun, N > 1)
# ---------------------------------------------------------------------------------------
def bench_main(args, tools: dict | None = None) -> None:
    """torchrun bench (N > 1): the same metric and config as bench.py at N = 1,
    strong scaling over one text.

    value: n / the query step from suffix structures resident on every GPU
    (BASELINE.md section 2 like-for-like step: raw LLR + compaction + all-ties
    scan), rank r answering position shard r (rs_query_structures_shard: its
    slots plus a left halo of max-LCP slots, no data exchange), tie totals
    all-gathered over NCCL and the shard's CSR rebased.  CUDA events on each
    rank's library stream, max over ranks.
    e2e: replicated_all_positions -- the API call from rank 0's host text:
    NVLink broadcast of the text, every rank builds the structures on its GPU
    and answers its shard, every rank D2Hs its shard into one shared host
    buffer (wall clock across barriers, max over ranks).
    """
    import json
    import sys

    import torch
    import torch.distributed as dist

    from paper_1501_06663_b200 import workloads

    # stdout carries exactly one JSON line; NCCL's own lines (NCCL_DEBUG=INFO
    # shows the communicators' rank counts, torch's and the library's) go to stderr
    sys.stdout.flush()
    json_fd = os.dup(1)
    os.dup2(2, 1)
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", os.environ.get("WORLD_SIZE", "1")))
    # host threads of the transfer pipeline: this rank's share of the node
    os.environ.setdefault("RS_HOST_THREADS", str(max(1, (os.cpu_count() or 1) // max(1, local_world))))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    device = torch.device("cuda", local)
    gen = workloads.make(args.config, args.n) if rank == 0 else None
    data = None
    if rank == 0:
        data = np.array(gen)  # the caller's pageable text
    ctx = _native.context(local)

    # ---- value: query from resident structures, position shards ----
    with ctx.lock:
        n = allgather_i64(ctx, int(data.size) if rank == 0 else 0, None, device)[0]
        if rank == 0:
            ctx.call("rs_set_text", _native.u8(data), n)
        ctx.call("rs_nccl_broadcast_text", n, 0)  # NCCL inside the library (library_comm above)
        ctx.call("rs_build_structures")  # untimed, like the reference arm's structures

        def step():
            return structures_query_shard(ctx, n, "all", None, device)

        clocks = tools["ClockSampler"](local) if tools else None
        if clocks:
            clocks.start()  # spans warm-up, timed and instrumented steps
        for _ in range(args.warmup):
            step()
        dist.barrier()
        torch.cuda.synchronize()
        ctx.synchronize()
        l0 = ctx.launches()
        ctx.record(0)
        for _ in range(args.steps):
            lo, hi, base, totals = step()
        ctx.record(1)
        ctx.synchronize()
        ms = ctx.elapsed_ms(0, 1) / args.steps
        launches = ctx.launches() - l0
        stages = ctx.stage_times()
        # per-kernel breakdown of this rank's shard step (separate instrumented pass)
        ctx.profile_begin()
        for _ in range(args.steps):
            step()
        ctx.synchronize()
        profile = ctx.profile_end()
        clk = clocks.stop() if clocks else None
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    lt = torch.tensor([float(launches)], dtype=torch.float64, device=device)
    dist.all_reduce(lt, op=dist.ReduceOp.SUM)
    T = int(sum(totals))

    # ---- e2e: the API-level call with host buffers ----
    e2e = []
    res = None
    xfer0 = None
    for i in range(args.warmup + max(1, args.steps)):
        res = None
        dist.barrier()
        torch.cuda.synchronize()
        if i == args.warmup:
            xfer0 = ctx.transfer_bytes()
        t0 = time.perf_counter()
        res = replicated_all_positions(data if rank == 0 else None, "all")
        torch.cuda.synchronize()
        dist.barrier()
        dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=device)
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        if i >= args.warmup:
            e2e.append(float(dt.item()))
    # clocks of every rank's GPU: slowest median, union of throttle reasons
    clks = [None] * world
    dist.all_gather_object(clks, clk)
    clks = [c for c in clks if c]
    clocks_line = None
    if clks:
        meds = [c["sm_mhz"] for c in clks if c.get("sm_mhz") is not None]
        maxs = [c["sm_max_mhz"] for c in clks if c.get("sm_max_mhz") is not None]
        clocks_line = {"sm_mhz": min(meds) if meds else None, "sm_max_mhz": max(maxs) if maxs else None,
                       "reasons": sorted({r for c in clks for r in c.get("reasons", [])}),
                       "ranks": len(clks)}
    roof = None
    if tools and profile:
        roof, _ = tools["roofline_of"](profile, args.steps)
        roof["traffic"] = None  # the committed ncu capture is of the full-size (N = 1) launch
        roof["traffic_source"] = "rank 0's shard launch (1/N of the positions): not captured"
    # bytes the library copied host<->device in the timed calls, summed over ranks
    xfer = torch.tensor([b - a for a, b in zip(xfer0, ctx.transfer_bytes())], dtype=torch.float64, device=device)
    dist.all_reduce(xfer, op=dist.ReduceOp.SUM)
    h2d_step, d2h_step = (int(v) // max(1, args.steps) for v in xfer.tolist())
    if rank == 0:
        assert int(res.flat_starts.size) == T, (res.flat_starts.size, T)
        line = {
            "metric": "positions/sec, all-longest-repeat query, n=256M DNA, 1/2/4/8 B200 vs CPU",
            "value": n / (ms * 1e-3), "unit": "positions/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32 device indices / int64 answers", "data": "synthetic",
            "config": {"workload": args.config, "n": n, "mode": "all", "path": "compact",
                       "timed": "raw LLR + compaction + all-ties query from resident suffix structures "
                                "(query.py:234), per rank one position shard; tie totals all-gathered "
                                "(NCCL) and CSR offsets rebased on device",
                       "parallelism": f"position shards x{world} (engine._chunks), structures on every GPU",
                       "l2": "input 256 MiB > 126 MB L2; raw LLR, compaction and answers rebuilt each step",
                       "T": T},
            "gpu_launches": int(round(float(lt.item()))),
            "clocks": clocks_line,
            "roofline": roof,
            "stages_ms_rank0": stages,
            "e2e": {"value": n / float(np.mean(e2e)), "unit": "positions/s", "h2d_bytes_per_step": h2d_step,
                    "d2h_bytes_per_step": d2h_step, "answer_bytes_per_step": 8 * (n + 1) + 8 * (n + 2) + 8 * T,
                    "ms_per_step": 1e3 * float(np.mean(e2e)),
                    "path": "replicated_all_positions: text H2D on rank 0 + NCCL broadcast, suffix "
                            "structures + shard query on every GPU, per-rank D2H into one shared host "
                            "buffer (/dev/shm), max over ranks"},
        }
        os.write(json_fd, (json.dumps(line) + "\n").encode())
    dist.barrier()
    dist.destroy_process_group()
    sys.stdout.flush()
    os.dup2(json_fd, 1)
    os.close(json_fd)


# ---------------------------------------------------------------------------------------
# distributed suffix sort: every phase is one library call per rank
# ---------------------------------------------------------------------------------------
HALO_CAP = 1 << 16  # raw slots reserved before each rank's shard (max repeat length distributed)


def dist_neighbours(infos: list) -> list:
    """Per rank the nbr[6] argument of rs_dist_update from all ranks' rs_dist_sort
    info: (last key, last suffix, has) of the nearest earlier non-empty segment
    and (first key, first suffix, has) of the nearest later one."""
    world = len(infos)
    out = []
    for r in range(world):
        nb = [0, 0, 0, 0, 0, 0]
        for p in range(r - 1, -1, -1):
            if infos[p][1] > 0:
                nb[0:3] = [int(infos[p][5]), int(infos[p][6]), 1]
                break
        for q in range(r + 1, world):
            if infos[q][1] > 0:
                nb[3:6] = [int(infos[q][3]), int(infos[q][4]), 1]
                break
        out.append(nb)
    return out


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def dist_phase_sort(ctx, rank: int, world: int) -> np.ndarray:
    info = np.zeros(16, np.int64)
    ctx.call("rs_dist_sort", rank, world, _native.i64(info))
    return info


def dist_phase_update(ctx, rank: int, world: int, nbr) -> tuple[np.ndarray, np.ndarray]:
    nb = _i64(nbr)
    counts = np.zeros(world, np.int64)
    info = np.zeros(16, np.int64)
    ctx.call("rs_dist_update", rank, world, _native.i64(nb), _native.i64(counts), _native.i64(info))
    return counts, info


def dist_phase_apply(ctx, rank: int, world: int, recv_ptr: int, count: int) -> np.ndarray:
    info = np.zeros(16, np.int64)
    ctx.call("rs_dist_apply", rank, world, ctypes.c_void_p(recv_ptr), int(count), HALO_CAP, _native.i64(info))
    return info


def dist_phase_scan(ctx, mode: str, halo: int) -> int:
    total = np.zeros(1, np.int64)
    ctx.call("rs_dist_scan", _native.MODE[mode], int(halo), _native.i64(total))
    return int(total[0])


def _raw_view(ctx, apply_info, lo_raw: int, count: int, device):
    """Torch view of raw[lo_raw, lo_raw + count) in this rank's raw shard."""
    R0 = int(apply_info[4])
    P0, P1 = int(apply_info[1]), int(apply_info[2])
    length = (P1 - P0) + HALO_CAP + 64
    v = _view(ctx, _native.BUF_RAW, length, "<u4", device)
    return v[lo_raw - R0: lo_raw - R0 + count]


def loopback_dist_all_positions(data: np.ndarray, world: int, mode: str = "all", device=None):
    """The distributed suffix sort + scan with `world` ranks simulated in ONE
    process on one GPU (one library context per rank, the all-to-all and
    halo exchanges done as device copies): exercises every phase and the
    exchange bookkeeping exactly as the NCCL path runs them.  Returns the
    reference-layout numpy arrays, or None when the text is outside the
    distributed regime."""
    import torch
    device = device or torch.device("cuda", torch.cuda.current_device())
    host = np.ascontiguousarray(data, dtype=np.uint8)
    n = int(host.size)
    ctxs = [_native.Context(device.index or 0) for _ in range(world)]
    try:
        for c in ctxs:
            c.call("rs_set_text", _native.u8(host), n)
        infos = [dist_phase_sort(c, r, world) for r, c in enumerate(ctxs)]
        if any(int(i[0]) == 0 for i in infos):
            return None
        nbrs = dist_neighbours(infos)
        ups = [dist_phase_update(c, r, world, nbrs[r]) for r, c in enumerate(ctxs)]
        if any(int(u[1][0]) == 0 for u in ups):
            return None
        sends = []
        for r, c in enumerate(ctxs):
            tot = int(ups[r][1][1])
            sends.append(_view(c, _native.BUF_SEND, tot, "<i8", device)[:tot])
        applies = []
        for q, c in enumerate(ctxs):
            parts = []
            for r in range(world):
                counts = ups[r][0]
                off = int(counts[:q].sum())
                parts.append(sends[r][off:off + int(counts[q])])
            recv = torch.cat(parts) if parts else torch.zeros(0, dtype=torch.int64, device=device)
            torch.cuda.synchronize(device)
            applies.append(dist_phase_apply(c, q, world, recv.data_ptr(), recv.numel()))
            del recv
        halo = max(int(a[3]) for a in applies) + 2
        if not dist_halo_fits(n, world, halo):
            return None
        partners = dist_halo_partners(n, world)
        for r in range(world):
            P0, P1 = int(applies[r][1]), int(applies[r][2])
            q = partners[r][1]
            if P1 <= P0 or q < 0:
                continue
            lo = max(P1 + 1 - halo, 1)
            cnt = P1 + 1 - lo
            src = _raw_view(ctxs[r], applies[r], lo, cnt, device)
            dst = _raw_view(ctxs[q], applies[q], lo, cnt, device)
            dst.copy_(src)
        torch.cuda.synchronize(device)
        totals = [dist_phase_scan(c, mode, halo) for c in ctxs]
        return _assemble_host(ctxs, applies, totals, n, mode)
    finally:
        for c in ctxs:
            c.close()


def _assemble_host(ctxs, applies, totals, n: int, mode: str):
    """rs_fetch_shard of every rank into the reference-layout arrays."""
    if mode == "leftmost":
        starts = np.full(n + 1, -1, np.int64)
        lengths = np.zeros(n + 1, np.int64)
        for c, a in zip(ctxs, applies):
            P0, P1 = int(a[1]), int(a[2])
            if P1 > P0:
                c.call("rs_fetch_shard", 0, _native.i64(starts[P0 + 1:P1 + 1]), _native.i64(lengths[P0 + 1:P1 + 1]),
                       None)
        return starts, lengths
    T = int(sum(totals))
    lengths = np.zeros(n + 1, np.int64)
    offsets = np.zeros(n + 2, np.int64)
    flat = np.zeros(T, np.int64)
    base = 0
    for c, a, t in zip(ctxs, applies, totals):
        P0, P1 = int(a[1]), int(a[2])
        if P1 <= P0:
            continue
        c.call("rs_shard_rebase", base)
        offs = np.zeros(P1 - P0 + 1, np.int64)
        c.call("rs_fetch_shard", 1, _native.i64(lengths[P0 + 1:P1 + 1]), _native.i64(offs),
               _native.i64(flat[base:base + t]) if t else _native.i64(np.zeros(1, np.int64)))
        offsets[P0 + 1:P1 + 2] = offs
        base += t
    return lengths, offsets, flat


def dist_halo_partners(n: int, world: int) -> list[tuple[int, int]]:
    """Per rank (previous, next) rank with a non-empty position shard (-1 if
    none); only ranks with non-empty shards exchange halos (with few buckets,
    empty shards can sit between non-empty ones)."""
    nonempty = [r for r in range(world) if dist_shard(n, r, world)[1] > dist_shard(n, r, world)[0]]
    out = []
    for r in range(world):
        prev = max((q for q in nonempty if q < r), default=-1)
        nxt = min((q for q in nonempty if q > r), default=-1)
        out.append((prev, nxt))
    return out


def dist_halo_fits(n: int, world: int, halo: int) -> bool:
    """The left halo of every shard must come from ONE neighbour: `halo` may not
    exceed any non-empty shard that has a later non-empty shard."""
    sizes = [b - a for a, b in (dist_shard(n, r, world) for r in range(world)) if b > a]
    return halo + 4 <= HALO_CAP and all(halo <= s for s in sizes[:-1])


def dist_shard(n: int, rank: int, world: int) -> tuple[int, int]:
    """0-based [P0, P1) position shard of `rank` in the distributed sort
    (bucket-aligned; the library's dist_shard / bucket_setup rule)."""
    sh = 12
    while (n + (1 << sh) - 1) >> sh > 256 and sh < 30:
        sh += 1
    nb = max(1, (n + (1 << sh) - 1) >> sh)
    b0, b1 = rank * nb // world, (rank + 1) * nb // world
    return min(b0 << sh, n), min(b1 << sh, n)


def dist_sa_all_positions(data: np.ndarray | None, n: int, mode: str = "all", group=None,
                          resident: bool = False, gather: bool = True):
    """Distributed suffix sort + scan over the ranks of `group` (NCCL).

    Every rank sorts one SA segment (MSD split by the top round-0 key digit),
    raw LLR goes to bucket-aligned position shards by all-to-all, each rank
    scans its shard.  resident=True: every rank already holds the text
    (rs_set_text_device); else rank 0's `data` is broadcast over NVLink.
    Returns rank 0's reference-layout tensors (gather=True), True on the
    other ranks / without gather, or None everywhere when the text is outside
    the distributed regime (long or highly repeated substrings: the caller
    then uses sharded_all_positions).
    """
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev_index = torch.cuda.current_device()
    device = torch.device("cuda", dev_index)
    ctx = _native.context(dev_index)
    kw = dict(dtype=torch.int64, device=device)
    with ctx.lock:
        if not resident:
            tv = _view(ctx, _native.BUF_TEXT, n + 128, "|u1", device)[:n]
            if rank == 0:
                tv.copy_(torch.from_numpy(np.ascontiguousarray(data, dtype=np.uint8)), non_blocking=True)
            dist.broadcast(tv, src=0, group=group)
            torch.cuda.synchronize(device)
            ctx.call("rs_set_text_device", n)
        info = dist_phase_sort(ctx, rank, world)
        allinfo = torch.zeros(world * 16, **kw)
        dist.all_gather_into_tensor(allinfo, torch.from_numpy(info).to(device), group=group)
        infos = allinfo.view(world, 16).cpu().numpy()
        if (infos[:, 0] == 0).any():
            return None
        counts, uinfo = dist_phase_update(ctx, rank, world, dist_neighbours(list(infos))[rank])
        ok = torch.tensor([int(uinfo[0])], **kw)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if int(ok.item()) == 0:
            return None
        send_counts = torch.from_numpy(counts).to(device)
        recv_counts = torch.empty(world, **kw)
        dist.all_to_all_single(recv_counts, send_counts, group=group)
        rc = [int(x) for x in recv_counts.cpu().tolist()]
        sc = [int(x) for x in counts.tolist()]
        total_send = int(uinfo[1])
        send = _view(ctx, _native.BUF_SEND, max(total_send, 1), "<i8", device)[:total_send]
        recv = torch.empty(sum(rc), **kw)
        dist.all_to_all_single(recv, send, output_split_sizes=rc, input_split_sizes=sc, group=group)
        torch.cuda.synchronize(device)
        ainfo = dist_phase_apply(ctx, rank, world, recv.data_ptr(), recv.numel())
        del recv
        mx = torch.tensor([int(ainfo[3])], **kw)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
        halo = int(mx.item()) + 2
        if not dist_halo_fits(n, world, halo):
            return None
        # left halo: the last `halo` raw values of the previous non-empty shard
        P0, P1 = int(ainfo[1]), int(ainfo[2])
        ops = []
        prev_r, next_r = dist_halo_partners(n, world)[rank]
        if P1 > P0 and next_r >= 0:
            lo = max(P1 + 1 - halo, 1)
            if P1 + 1 - lo > 0:
                ops.append(dist.P2POp(dist.isend, _raw_view(ctx, ainfo, lo, P1 + 1 - lo, device).contiguous(),
                                      next_r, group))
        if P1 > P0 and prev_r >= 0:
            lo = max(P0 + 1 - halo, 1)
            if P0 + 1 - lo > 0:
                ops.append(dist.P2POp(dist.irecv, _raw_view(ctx, ainfo, lo, P0 + 1 - lo, device), prev_r, group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        torch.cuda.synchronize(device)
        total = dist_phase_scan(ctx, mode, halo)
        lo1, hi1 = P0 + 1, P1 + 1  # 1-based half-open
        cnt = hi1 - lo1
        if mode == "all":
            totals = exchange_totals(total, group, device)
            bases = tie_bases(totals)
            if cnt > 0:
                ctx.call("rs_shard_rebase", bases[rank])
            T_all = sum(totals)
        if not gather:
            ctx.synchronize()
            return True
        ranges = [tuple(x + 1 for x in dist_shard(n, r, world)) for r in range(world)]
        a = _view(ctx, _native.BUF_OUT0, max(cnt, 1), "<i8", device)
        if mode == "all":
            b = _view(ctx, _native.BUF_OUT1, cnt + 1, "<i8", device)
            f = _view(ctx, _native.BUF_FLAT, total, "<i8", device)
            ctx.synchronize()
            out = gather_shards(n, mode, lo1, hi1, a, b, f, T_all, bases[rank], group, device, ranges=ranges)
        else:
            b = _view(ctx, _native.BUF_OUT1, max(cnt, 1), "<i8", device)
            ctx.synchronize()
            out = gather_shards(n, mode, lo1, hi1, a, b, None, 0, 0, group, device, ranges=ranges)
        torch.cuda.synchronize(device)
    return out if rank == 0 else True
