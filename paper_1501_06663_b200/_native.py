"""ctypes binding of librepeatscan_b200.so (include/repeatscan_b200.h).

There is no fallback: if the library or a B200 is missing, every call raises.
ctypes releases the GIL for the duration of each call, like the reference's
``nogil`` numba kernels (``_kernels_numba.py:6,12``).
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "librepeatscan_b200.so"

RS_OK, RS_EINVAL, RS_ERANGE, RS_ENOMEM, RS_ECUDA, RS_ENCCL, RS_ESTATE = 0, -1, -2, -3, -4, -5, -6
MODE = {"leftmost": 0, "all": 1}
PATH = {"raw": 0, "compact": 1}
STAGES = ("h2d", "sa", "lcp", "raw_llr", "compact", "query", "d2h")
BUF_LLRC, BUF_OUT0, BUF_OUT1, BUF_FLAT, BUF_TEXT, BUF_SEND, BUF_RAW = 0, 1, 2, 3, 4, 5, 6

_I64P = ctypes.POINTER(ctypes.c_int64)
_U8P = ctypes.POINTER(ctypes.c_uint8)
_VP = ctypes.c_void_p
_CTX = ctypes.c_void_p

# name -> argtypes (restype is int unless listed in _RESTYPES)
SIGNATURES = {
    "rs_version": [],
    "rs_device_count": [ctypes.POINTER(ctypes.c_int)],
    "rs_create": [ctypes.c_int, ctypes.POINTER(_CTX)],
    "rs_destroy": [_CTX],
    "rs_last_error": [_CTX],
    "rs_synchronize": [_CTX],
    "rs_launch_count": [_CTX, _I64P],
    "rs_transfer_bytes": [_CTX, _I64P, _I64P],
    "rs_stage_times": [_CTX, ctypes.POINTER(ctypes.c_double)],
    "rs_record_event": [_CTX, ctypes.c_int],
    "rs_elapsed_ms": [_CTX, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_float)],
    "rs_device_bytes": [_CTX, _I64P],
    "rs_release": [_CTX],
    "rs_host_alloc": [ctypes.c_int64, ctypes.POINTER(_VP)],
    "rs_host_free": [_VP],
    "rs_suffix_structures": [_CTX, _U8P, ctypes.c_int64, _I64P, _I64P, _I64P],
    "rs_raw_llr": [_CTX, _I64P, _I64P, ctypes.c_int64, _I64P],
    "rs_flags": [_CTX, _I64P, ctypes.c_int64, _I64P],
    "rs_prefix_sum": [_CTX, _I64P, ctypes.c_int64, _I64P],
    "rs_inclusive_scan": [_CTX, _I64P, ctypes.c_int64, _I64P],
    "rs_scatter_compact": [_CTX, _I64P, _I64P, _I64P, ctypes.c_int64, _I64P, _I64P],
    "rs_compact": [_CTX, _I64P, ctypes.c_int64, _I64P, _I64P, _I64P],
    "rs_set_text": [_CTX, _U8P, ctypes.c_int64],
    "rs_set_structures": [_CTX, _I64P, _I64P, _I64P, ctypes.c_int64],
    "rs_build_structures": [_CTX],
    "rs_verify_structures": [_CTX, _U8P, ctypes.c_int64, _I64P, _I64P, _I64P, _I64P],
    "rs_get_structures": [_CTX, _I64P, _I64P, _I64P],
    "rs_check_answers": [_CTX, _I64P, _I64P, ctypes.c_int64, ctypes.c_int64, _I64P, _I64P, _I64P,
                         ctypes.c_int64, _I64P, _I64P, _I64P],
    "rs_set_raw": [_CTX, _I64P, ctypes.c_int64],
    "rs_set_compact": [_CTX, _I64P, _I64P, ctypes.c_int64, ctypes.c_int64],
    "rs_query": [_CTX, ctypes.c_int, ctypes.c_int, _I64P],
    "rs_fetch_leftmost": [_CTX, _I64P, _I64P],
    "rs_fetch_all": [_CTX, _I64P, _I64P, _I64P],
    "rs_get_raw": [_CTX, _I64P],
    "rs_get_compact_size": [_CTX, _I64P],
    "rs_get_compact": [_CTX, _I64P, _I64P],
    "rs_reset": [_CTX],
    "rs_clear_derived": [_CTX],
    "rs_clear_llr": [_CTX],
    "rs_profile_begin": [_CTX],
    "rs_profile_end": [_CTX, ctypes.POINTER(ctypes.c_int)],
    "rs_profile_kernel": [_CTX, ctypes.c_int, ctypes.c_char_p, ctypes.c_int, _I64P,
                          ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)],
    "rs_sa_rounds": [_CTX, ctypes.POINTER(ctypes.c_int)],
    "rs_serialize": [_CTX, ctypes.c_int64, ctypes.c_int64, _I64P],
    "rs_fetch_serialized": [_CTX, _U8P],
    "rs_walk_steps": [_CTX, ctypes.c_int, _I64P, _I64P],
    "rs_summarize_steps": [_CTX, _I64P, ctypes.c_int64, _I64P],
    "rs_device_buffer": [_CTX, ctypes.c_int, ctypes.c_int64, ctypes.POINTER(_VP)],
    "rs_set_compact_device": [_CTX, ctypes.c_int64, ctypes.c_int64],
    "rs_stream": [_CTX, ctypes.POINTER(_VP)],
    "rs_set_text_device": [_CTX, ctypes.c_int64],
    "rs_dist_sort": [_CTX, ctypes.c_int32, ctypes.c_int32, _I64P],
    "rs_dist_update": [_CTX, ctypes.c_int32, ctypes.c_int32, _I64P, _I64P, _I64P],
    "rs_dist_apply": [_CTX, ctypes.c_int32, ctypes.c_int32, _VP, ctypes.c_int64, ctypes.c_int64, _I64P],
    "rs_dist_scan": [_CTX, ctypes.c_int, ctypes.c_int64, _I64P],
    "rs_query_shard": [_CTX, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, _I64P],
    "rs_query_structures_shard": [_CTX, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, _I64P],
    "rs_shard_rebase": [_CTX, ctypes.c_int64],
    "rs_nccl_unique_id": [ctypes.c_void_p],
    "rs_nccl_init": [_CTX, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32],
    "rs_nccl_destroy": [_CTX],
    "rs_nccl_broadcast_text": [_CTX, ctypes.c_int64, ctypes.c_int32],
    "rs_nccl_allgather_i64": [_CTX, ctypes.c_int64, _I64P],
    "rs_fetch_shard": [_CTX, ctypes.c_int, _I64P, _I64P, _I64P],
}
_RESTYPES = {"rs_version": ctypes.c_char_p, "rs_last_error": ctypes.c_char_p}

_lib = None
_lock = threading.RLock()


def load_library() -> ctypes.CDLL:
    """Load the CUDA library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH.name} not found: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (nvcc, sm_100a).  There is no CPU fallback.")
        lib = ctypes.CDLL(str(LIB_PATH))
        for name, args in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, ctypes.c_int)
        _lib = lib
    return _lib


def exported_symbols() -> list[str]:
    return list(SIGNATURES)


class RepeatscanError(RuntimeError):
    pass


def _raise(ctx, rc: int, what: str):
    msg = (load_library().rs_last_error(ctx) or b"").decode(errors="replace")
    text = f"{what}: {msg}" if msg else what
    if rc == RS_EINVAL:
        raise ValueError(text)
    if rc == RS_ERANGE:
        raise IndexError(text)
    if rc == RS_ENOMEM:
        raise MemoryError(text)
    raise RepeatscanError(f"{text} (status {rc})")


def i64(a: np.ndarray):
    assert a.dtype == np.int64 and a.flags.c_contiguous, (a.dtype, a.flags)
    return a.ctypes.data_as(_I64P)


def u8(a: np.ndarray):
    return a.ctypes.data_as(_U8P)


class Context:
    """One device context: stream + arena + device-resident pipeline state."""

    def __init__(self, device: int = 0):
        lib = load_library()
        h = _CTX()
        rc = lib.rs_create(int(device), ctypes.byref(h))
        if rc != RS_OK:
            raise RepeatscanError(
                f"rs_create(device={device}) failed with status {rc}: a B200 (sm_100a) is required")
        self.handle = h
        self.device = int(device)
        self.lib = lib
        self.lock = threading.RLock()

    def call(self, name: str, *args):
        rc = getattr(self.lib, name)(self.handle, *args)
        if rc != RS_OK:
            _raise(self.handle, rc, name)

    def launches(self) -> int:
        v = ctypes.c_int64()
        self.call("rs_launch_count", ctypes.byref(v))
        return int(v.value)

    def transfer_bytes(self) -> tuple[int, int]:
        """(host->device, device->host) bytes copied by this context so far."""
        a, b = ctypes.c_int64(), ctypes.c_int64()
        self.call("rs_transfer_bytes", ctypes.byref(a), ctypes.byref(b))
        return int(a.value), int(b.value)

    def stage_times(self) -> dict:
        arr = (ctypes.c_double * len(STAGES))()
        self.call("rs_stage_times", arr)
        return {s: float(arr[i]) for i, s in enumerate(STAGES)}

    def sa_rounds(self) -> int:
        v = ctypes.c_int()
        self.call("rs_sa_rounds", ctypes.byref(v))
        return int(v.value)

    def record(self, slot: int):
        self.call("rs_record_event", int(slot))

    def elapsed_ms(self, a: int, b: int) -> float:
        v = ctypes.c_float()
        self.call("rs_elapsed_ms", int(a), int(b), ctypes.byref(v))
        return float(v.value)

    def synchronize(self):
        self.call("rs_synchronize")

    def device_bytes(self) -> int:
        v = ctypes.c_int64()
        self.call("rs_device_bytes", ctypes.byref(v))
        return int(v.value)

    def release(self):
        self.call("rs_release")

    def stream_ptr(self) -> int:
        v = _VP()
        self.call("rs_stream", ctypes.byref(v))
        return int(v.value or 0)

    def device_buffer(self, which: int, nbytes: int) -> int:
        v = _VP()
        self.call("rs_device_buffer", int(which), int(nbytes), ctypes.byref(v))
        return int(v.value)

    def profile_begin(self):
        self.call("rs_profile_begin")

    def profile_end(self) -> list[dict]:
        """Per-kernel totals since profile_begin: name, launches, ms, algorithmic bytes."""
        k = ctypes.c_int()
        self.call("rs_profile_end", ctypes.byref(k))
        out = []
        name = ctypes.create_string_buffer(256)
        for i in range(k.value):
            launches = ctypes.c_int64()
            ms = ctypes.c_double()
            nbytes = ctypes.c_double()
            self.call("rs_profile_kernel", i, name, 256, ctypes.byref(launches), ctypes.byref(ms),
                      ctypes.byref(nbytes))
            nm = name.value.decode().strip("()")
            out.append({"kernel": nm, "launches": int(launches.value), "ms": float(ms.value),
                        "bytes": float(nbytes.value)})
        return out

    def close(self):
        if self.handle:
            self.lib.rs_destroy(self.handle)
            self.handle = None


_contexts: dict[int, Context] = {}


def default_device() -> int:
    env = os.environ.get("REPEATSCAN_B200_DEVICE")
    if env:
        return int(env)
    return int(os.environ.get("LOCAL_RANK", "0"))


def context(device: int | None = None) -> Context:
    """The process-wide context of a device (created on first use)."""
    dev = default_device() if device is None else int(device)
    ctx = _contexts.get(dev)
    if ctx is None:
        with _lock:
            ctx = _contexts.get(dev)
            if ctx is None:
                ctx = Context(dev)
                _contexts[dev] = ctx
    return ctx


def device_count() -> int:
    v = ctypes.c_int()
    load_library().rs_device_count(ctypes.byref(v))
    return int(v.value)


# -- host memory for output arrays ----------------------------------------------------
class _PinnedBlock:
    __slots__ = ("ptr", "nbytes", "__weakref__")

    def __init__(self, nbytes: int):
        lib = load_library()
        p = _VP()
        rc = lib.rs_host_alloc(int(nbytes), ctypes.byref(p))
        if rc != RS_OK:
            raise MemoryError(f"pinned host allocation of {nbytes} bytes failed")
        self.ptr = int(p.value)
        self.nbytes = int(nbytes)

    def __del__(self):
        try:
            if self.ptr:
                load_library().rs_host_free(_VP(self.ptr))
                self.ptr = 0
        except Exception:
            pass


class _PageableBlock:
    __slots__ = ("mem", "ptr", "nbytes", "__weakref__")

    def __init__(self, nbytes: int):
        self.mem = np.empty(int(nbytes), np.uint8)
        self.ptr = int(self.mem.ctypes.data)
        self.nbytes = int(nbytes)


class HostPool:
    """Caching allocator of host blocks for the D2H result arrays.

    Arrays handed out keep their block alive (through a ctypes owner object
    that every numpy view of them references); when the last view dies the
    block returns to the pool, like PyTorch's caching host allocator.  A
    reused block is already page-faulted: the library's transfer pipeline
    (csrc/host_io.cu) writes touched memory at ~90 GB/s with 16 host threads
    against ~40 GB/s for fresh pages (tools/exp_d2h.py on the B200 box).
    ``pinned=True`` blocks are page-locked (cudaHostAlloc); the default blocks
    are ordinary pageable memory.
    """

    def __init__(self, block_type, limit_bytes: int = 48 << 30):
        self._block_type = block_type
        self._free: dict[int, list] = {}
        self._lock = threading.Lock()
        self.limit = limit_bytes
        self.cached = 0

    @staticmethod
    def _bucket(nbytes: int) -> int:
        b = 1 << 20
        while b < nbytes:
            b <<= 1
        return b

    def empty(self, count: int, dtype=np.int64) -> np.ndarray:
        dtype = np.dtype(dtype)
        nbytes = max(int(count) * dtype.itemsize, 1)
        size = self._bucket(nbytes)
        with self._lock:
            lst = self._free.get(size)
            block = lst.pop() if lst else None
            if block is not None:
                self.cached -= size
        if block is None:
            block = self._block_type(size)
        owner = (ctypes.c_char * size).from_address(block.ptr)
        arr = np.frombuffer(owner, dtype=dtype, count=int(count))
        import weakref
        weakref.finalize(owner, self._give_back, block)
        return arr

    def _give_back(self, block):
        with self._lock:
            if self.cached + block.nbytes <= self.limit:
                self._free.setdefault(block.nbytes, []).append(block)
                self.cached += block.nbytes
                return
        del block


pinned_pool = HostPool(_PinnedBlock)
pageable_pool = HostPool(_PageableBlock)
PinnedPool = HostPool  # name kept for callers of round 1


def out_array(count: int, pinned: bool) -> np.ndarray:
    """int64 output array; large ones come from the caching host pools."""
    if count >= (1 << 17):
        return (pinned_pool if pinned else pageable_pool).empty(count)
    return np.empty(count, np.int64)
