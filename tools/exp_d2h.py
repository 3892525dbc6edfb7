"""D2H strategies for the int64 result arrays (8.4 GB at C3): measured on the box.

pageable (fresh / touched destination) vs pinned via torch copy_, and host
memcpy pinned -> pageable with T threads (fresh / touched).
"""
import threading
import time

import numpy as np
import torch

N = 1 << 30  # int64 elements = 8 GiB
dev = torch.empty(N, dtype=torch.int64, device="cuda")
dev.fill_(7)
torch.cuda.synchronize()


def t_copy(dst_np):
    dst = torch.from_numpy(dst_np)
    torch.cuda.synchronize()
    t = time.perf_counter()
    dst.copy_(dev)
    torch.cuda.synchronize()
    return time.perf_counter() - t


gb = N * 8 / 1e9
fresh = np.empty(N, np.int64)
print(f"pageable fresh : {gb / t_copy(fresh):6.1f} GB/s")
print(f"pageable touched: {gb / t_copy(fresh):6.1f} GB/s")
del fresh
pin = torch.empty(N, dtype=torch.int64, pin_memory=True)
print(f"pinned         : {gb / t_copy(pin.numpy()):6.1f} GB/s")
print(f"pinned again   : {gb / t_copy(pin.numpy()):6.1f} GB/s")
src = pin.numpy()


def par_copy(dst, T):
    step = (N + T - 1) // T
    ths = [threading.Thread(target=np.copyto, args=(dst[i * step:(i + 1) * step], src[i * step:(i + 1) * step]))
           for i in range(T)]
    t = time.perf_counter()
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    return time.perf_counter() - t


for T in (1, 4, 8, 16, 32):
    d = np.empty(N, np.int64)
    a = par_copy(d, T)
    b = par_copy(d, T)
    print(f"host memcpy T={T:2d}: fresh {gb / a:6.1f} GB/s, touched {gb / b:6.1f} GB/s")
    del d
import mmap
m = mmap.mmap(-1, N * 8, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
try:
    m.madvise(mmap.MADV_HUGEPAGE)
except Exception as e:
    print("no MADV_HUGEPAGE", e)
d = np.frombuffer(m, np.int64)
print(f"THP mmap fresh host memcpy T=16: {gb / par_copy(d, 16):6.1f} GB/s")
print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
m2 = mmap.mmap(-1, N * 8, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
try:
    m2.madvise(mmap.MADV_HUGEPAGE)
except Exception:
    pass
d2 = np.frombuffer(m2, np.int64)
print(f"THP mmap fresh torch pageable copy: {gb / t_copy(d2):6.1f} GB/s")
