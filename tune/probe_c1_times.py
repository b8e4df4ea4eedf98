"""Per-call event times of the C1 MTTKRP (L2 flushed before each call)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_03317_b200 import generate, ops, _lib
nnz = int(os.environ.get("NNZ", 1_000_000)); R = int(os.environ.get("R", 16)); D = int(os.environ.get("D", 1000))
Z = float(os.environ.get("ZIPF", 0))
x = generate.coo([D, max(D, 3000), max(D, 3000)], nnz, 1, [Z, 0, 0], 0, 1, [0, 1, 2])
f = [generate.uniform((d, R), 1, k, 0, 1) for k, d in enumerate(x.dims)]
out = torch.empty((D, R), device="cuda")
ctx = _lib.Context.get(0); lib = _lib.load(); st = torch.cuda.current_stream()
strat = int(os.environ.get("STRAT", ops.MTTKRP_SEGMENTED))
ts = []
for i in range(30):
    lib.spt_l2_flush(ctx.handle, st.cuda_stream)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); ops.mttkrp(x, f, 0, strat, out=out, sync=False); b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
import statistics
print(f"nnz {nnz} R {R} D {D} zipf {Z} strat {strat}: median {statistics.median(ts[3:]):.1f} us")
