import torch
x = torch.empty(8 << 30, dtype=torch.uint8, device="cuda")
for _ in range(3): x.zero_()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): x.zero_()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print("write-only (memset) GB/s", (8 << 30) / ms / 1e6)
y = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")
z = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")
for _ in range(3): z.copy_(y)
torch.cuda.synchronize()
e0.record()
for _ in range(10): z.copy_(y)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print("copy (r+w) GB/s", 2 * (4 << 30) / ms / 1e6)
