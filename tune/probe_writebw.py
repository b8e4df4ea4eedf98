"""Pure-write and copy HBM bandwidth on the box (torch fill_ / copy_), to bound write-heavy ops
such as TTM (C3 mode 0 writes 12.6 GB)."""
import torch
n = 3 * (1 << 30)  # 3 Gi floats = 12 GiB
a = torch.empty(n, dtype=torch.float32, device="cuda")
for _ in range(3):
    a.fill_(1.0)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); a.fill_(2.0); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
ms = min(ts)
print(f"fill {n*4/1e9:.1f} GB: {ms:.2f} ms = {n*4/ms/1e6:.0f} GB/s (write only)")
b = torch.empty(n // 2, dtype=torch.float32, device="cuda")
ts = []
for _ in range(5):
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); b.copy_(a[: n // 2]); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
ms = min(ts)
print(f"copy {n*4/1e9:.1f} GB moved: {ms:.2f} ms = {n*4/ms/1e6:.0f} GB/s (read+write)")
