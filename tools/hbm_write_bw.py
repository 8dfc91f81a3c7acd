import torch, time
x = torch.empty(4_349_603_232 // 4, dtype=torch.float32, device='cuda')
y = torch.empty(2_000_000_000 // 4, dtype=torch.float32, device='cuda')
z = torch.empty_like(y)
for _ in range(3): x.fill_(1.0); z.copy_(y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(5):
    e0.record(); x.fill_(2.0); e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
print("fill 4.35 GB: %.3f ms = %.1f GB/s" % (best, 4.3496e9 / best / 1e6))
best = 1e9
for _ in range(5):
    e0.record(); z.copy_(y); e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
print("copy 2 GB: %.3f ms = %.1f GB/s (read+write)" % (best, 4e9 / best / 1e6))
