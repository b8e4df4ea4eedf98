"""Per-warp-tile phase timeline of ttv_wt_kernel (build with -DSPT_TTV_TRACE):
start (map loaded) 0, entries loaded 1, heads 2, terms+scan 3, look-back 4, stores 5."""
import ctypes, torch, sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_03317_b200 import generate, ops, _lib
ctx = _lib.Context.get(0); lib = _lib.load(); st = torch.cuda.current_stream().cuda_stream
mode = int(os.environ.get("MODE", 2)); nnz = int(os.environ.get("NNZ", 10_000_000))
dims = [50000, 20000, 100000]
x = generate.coo(dims, nnz, 1, [1.1, 0, 0], 0, 1, None)
ops.sort_lexicographic(x, ops.mode_last_order(3, mode))
fib = ops.build_fiber_index(x, mode)
v = generate.uniform(dims[mode], 1, 6, -1, 1)
for _ in range(3):
    lib.spt_l2_flush(ctx.handle, st)
    ops.ttv(x, v, mode, fib)
torch.cuda.synchronize()
buf = np.zeros(65536 * 8, dtype=np.uint64)
assert lib.spt_debug_ttv_trace(buf.ctypes.data_as(ctypes.c_void_p)) == 0
kwt = 128 if nnz <= fib.nfibs * 1.5 else 256
nt = min(65536, (nnz + kwt - 1) // kwt)
t = buf.reshape(-1, 8)[:nt, :6].astype(np.int64)
t0 = t[:, 0].min()
r = (t - t0) / 1000.0
print(f"mode {mode} nnz {nnz} tiles {nt} (first 65536) span {r.max():.1f} us")
names = ["start", "entries", "heads", "scan", "lookback", "stores"]
for a in range(5):
    d = r[:, a + 1] - r[:, a]
    print(f"{names[a]:>9s} -> {names[a+1]:<9s} med {np.median(d):6.2f} p90 {np.percentile(d, 90):6.2f} max {d.max():6.2f}")
d = r[:, 5] - r[:, 0]
print(f"tile total med {np.median(d):.2f} p90 {np.percentile(d, 90):.2f}")
