import torch, time
x = torch.empty(int(8.4e9)//8, dtype=torch.int64, device='cuda')
y = torch.empty(int(1.07e9)//4, dtype=torch.int32, device='cuda')
def t(f, reps=10):
    f(); torch.cuda.synchronize()
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): f()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e)/reps
ms = t(lambda: x.fill_(7)); print("fill int64 8.4GB: %.3f ms -> %.0f GB/s" % (ms, 8.4e9/ms/1e6))
ms = t(lambda: x.zero_()); print("zero 8.4GB: %.3f ms -> %.0f GB/s" % (ms, 8.4e9/ms/1e6))
z = torch.empty(int(4.2e9)//8, dtype=torch.int64, device='cuda'); w = torch.empty_like(z)
ms = t(lambda: w.copy_(z)); print("copy 4.2GB: %.3f ms -> %.0f GB/s (r+w)" % (ms, 8.4e9/ms/1e6))
ms = t(lambda: y.sum()); print("read 1.07GB: %.3f ms -> %.0f GB/s" % (ms, 1.07e9/ms/1e6))
