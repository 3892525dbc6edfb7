"""Experiment: per-kernel device time of the distributed path at world size 1 (NCCL)."""
import os, socket, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
from paper_1501_06663_b200 import _native, workloads, distributed as D

with socket.socket() as s:
    s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
data = workloads.make(os.environ.get("EXP_CONFIG", "C3"), None)
n = int(data.size)
ctx = _native.context(0)
with ctx.lock:
    ctx.call("rs_set_text", _native.u8(np.ascontiguousarray(data)), n)
for _ in range(3):
    r = D.dist_sa_all_positions(None, n, "all", resident=True, gather=False)
print("distributed path:", "declined" if r is None else "ran")
torch.cuda.synchronize()
ctx.profile_begin()
ctx.record(0)
D.dist_sa_all_positions(None, n, "all", resident=True, gather=False)
torch.cuda.synchronize()
ctx.record(1)
prof = ctx.profile_end()
print("step ms", ctx.elapsed_ms(0, 1))
for k in sorted(prof, key=lambda k: -k["ms"])[:20]:
    print(f'{k["kernel"]:32s} {k["ms"]:7.2f} ms  x{k["launches"]}')
dist.destroy_process_group()
