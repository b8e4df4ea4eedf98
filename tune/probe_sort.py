"""Time sort_lexicographic on C2's 10M-entry tensor in draw order (events)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_03317_b200 import ops
from paper_1902_03317_b200.coo import DeviceCOO
n = int(os.environ.get("NNZ", 10_000_000))
dims = [int(d) for d in os.environ.get("DIMS", "10000,10000,10000").split(",")]
# torch draws (duplicates allowed): the generator itself sorts, and knock-out
# library variants must not be needed to make the input
g = torch.Generator(device="cuda"); g.manual_seed(1)
src = DeviceCOO(dims, [torch.randint(0, d, (n,), device="cuda", generator=g, dtype=torch.int32)
                       for d in dims], torch.rand(n, device="cuda", generator=g), None, False)
work = src.clone()
mo = list(range(len(dims)))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for it in range(int(os.environ.get("ITERS", 8))):
    for a, b in zip(work.indices, src.indices):
        a.copy_(b)
    work.values.copy_(src.values)
    work.sort_order = None
    flush.add_(1)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); ops.sort_lexicographic(work, mo, sync=False); b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
print("sort us:", " ".join(f"{t:.0f}" for t in ts))
