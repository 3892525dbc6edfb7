import torch, time
n = 1 << 28
x = torch.randint(0, 2**31 - 1, (n,), dtype=torch.int32, device="cuda")
for dt in (torch.int32,):
    for i in range(3):
        torch.sort(x, stable=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(5):
        v, idx = torch.sort(x, stable=True)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"torch.sort int32 keys + int64 idx, n=2^28: {ms:.2f} ms  ({n/ms/1e6:.2f} G keys/s)")
# keys 16-bit range: fewer passes?
y = torch.randint(0, 2**15, (n,), dtype=torch.int32, device="cuda")
torch.sort(y, stable=True); torch.cuda.synchronize()
e0.record()
for i in range(5):
    torch.sort(y, stable=True)
e1.record(); torch.cuda.synchronize()
print(f"torch.sort 15-bit int32 keys: {e0.elapsed_time(e1)/5:.2f} ms")
