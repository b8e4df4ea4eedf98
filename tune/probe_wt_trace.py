"""Per-warp-tile phase timeline of mttkrp_wt_kernel (variant built with -DSPT_WT_TRACE)."""
import ctypes, torch, sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_03317_b200 import generate, ops, _lib
ctx = _lib.Context.get(0); lib = _lib.load(); st = torch.cuda.current_stream().cuda_stream
x = generate.coo([1000]*3, 1_000_000, 1, [0,0,0], 0, 1, [0, 1, 2])
f = [generate.uniform((1000, 16), 1, k, 0, 1) for k in range(3)]
out = torch.empty((1000, 16), device='cuda')
for _ in range(5):
    lib.spt_l2_flush(ctx.handle, st)
    ops.mttkrp(x, f, 0, ops.MTTKRP_SEGMENTED_WARP, out=out, sync=False)
torch.cuda.synchronize()
buf = np.zeros(16384 * 8, dtype=np.uint64)
assert lib.spt_debug_wt_trace(buf.ctypes.data_as(ctypes.c_void_p)) == 0
ntiles = (x.nnz + 255) // 256
t = buf.reshape(-1, 8)[:ntiles].astype(np.int64)
t0 = t[:, 7].min()
rel = (t[:, [7, 0, 1, 2, 3, 4, 5]] - t0) / 1000.0  # us
names = ["entry", "ticket", "staged", "gathered", "folded", "lookback", "end"]
print("kernel span %.1f us" % rel[:, 6].max())
for k, n in enumerate(names):
    print(f"{n:9s} pct10 {np.percentile(rel[:,k],10):6.1f} med {np.median(rel[:,k]):6.1f} pct90 {np.percentile(rel[:,k],90):6.1f} max {rel[:,k].max():6.1f}")
d = np.diff(rel, axis=1)
for k in range(6):
    print(f"{names[k]}->{names[k+1]:9s} med {np.median(d[:,k]):6.2f} pct90 {np.percentile(d[:,k],90):6.2f} max {d[:,k].max():6.2f}")
sm = t[:, 6]
print("tiles per SM: min %d max %d" % (np.bincount(sm).min(), np.bincount(sm).max()))
