"""Per-tile timeline of merge64p_kernel (variant built with -DSPT_MERGE_TRACE): producer
ticket (0), stage free (1), merge warps: wait start (2), stage full (3), packed (4),
merged+scanned (5), flushed (6)."""
import ctypes, torch, sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_03317_b200 import generate, ops, _lib
from paper_1902_03317_b200.coo import DeviceCOO
ctx = _lib.Context.get(0); lib = _lib.load(); st = torch.cuda.current_stream().cuda_stream
dims, n = [10000]*3, 10_000_000
x = generate.coo(dims, n, 1, [0,0,0], 0.5, 1.5, [0,1,2])
y = generate.coo(dims, n, 2, [0,0,0], 0.5, 1.5, [0,1,2])
z = DeviceCOO.empty(dims, 2*n)
cnt = torch.zeros(1, dtype=torch.int64, device='cuda')
op = int(os.environ.get("OP", 0))
for _ in range(3):
    lib.spt_l2_flush(ctx.handle, st)
    ops.tew_device(x, y, op, z, cnt)
torch.cuda.synchronize()
buf = np.zeros(16384 * 8, dtype=np.uint64)
assert lib.spt_debug_merge_trace(buf.ctypes.data_as(ctypes.c_void_p)) == 0
nt = (2 * n + 2047) // 2048
t = buf.reshape(-1, 8)[:nt, :7].astype(np.int64)
t0 = t[:, 0].min()
r = (t - t0) / 1000.0
print("span %.1f us" % r.max())
names = ["ticket", "stage_free", "mw_wait", "full", "packed", "merged", "flushed"]
for a, b in [(0, 1), (1, 3), (2, 3), (3, 4), (4, 5), (5, 6), (3, 6)]:
    d = r[:, b] - r[:, a]
    print(f"{names[a]:>10s} -> {names[b]:<10s} med {np.median(d):6.2f} p10 {np.percentile(d,10):6.2f} p90 {np.percentile(d,90):6.2f}")
