"""Per-call event times of the C1 MTTKRP (L2 flushed before each call)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_03317_b200 import generate, ops, _lib
x = generate.coo([1000] * 3, 1_000_000, 1, [0, 0, 0], 0, 1, [0, 1, 2])
f = [generate.uniform((1000, 16), 1, k, 0, 1) for k in range(3)]
out = torch.empty((1000, 16), device="cuda")
ctx = _lib.Context.get(0); lib = _lib.load(); st = torch.cuda.current_stream()
strat = int(os.environ.get("STRAT", ops.MTTKRP_SEGMENTED))
ts = []
for i in range(30):
    lib.spt_l2_flush(ctx.handle, st.cuda_stream)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); ops.mttkrp(x, f, 0, strat, out=out, sync=False); b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
print(" ".join(f"{t:.1f}" for t in ts))
