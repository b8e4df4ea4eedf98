"""C1 MTTKRP (1M nnz, 1000^3, R=16, mode 0) and TS timings, L2 flushed, CUDA events."""
import torch, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_03317_b200 import generate, ops, _lib
ctx = _lib.Context.get(0); lib = _lib.load(); st = torch.cuda.current_stream().cuda_stream
def timeit(fn, reps=30):
    ts = []
    for i in range(reps + 5):
        lib.spt_l2_flush(ctx.handle, st)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        if i >= 5: ts.append(a.elapsed_time(b))
    ts.sort(); return ts[len(ts)//2]
x = generate.coo([1000]*3, 1_000_000, 1, [0,0,0], 0, 1, [0, 1, 2])
f = [generate.uniform((1000, 16), 1, k, 0, 1) for k in range(3)]
out = torch.empty((1000, 16), device='cuda')
ms = timeit(lambda: ops.mttkrp(x, f, 0, ops.MTTKRP_SEGMENTED, out=out, sync=False))
extra = []
for nm, sg in (("atomic", ops.MTTKRP_ATOMIC), ("cta", ops.MTTKRP_SEGMENTED_CTA), ("warp", ops.MTTKRP_SEGMENTED_WARP)):
    extra.append(f"{nm} {timeit(lambda: ops.mttkrp(x, f, 0, sg, out=out, sync=False))*1e3:.1f}us")
z = x.clone()
ms2 = timeit(lambda: ops.ts(x, 2.5, ops.SCALAR_MUL, out=z, sync=False))
print(os.path.basename(_lib.LIB_PATH), f"mttkrp {ms*1e3:.1f}us ({16192000/ms/1e6:.0f} GB/s)  ts {ms2*1e3:.1f}us ({32e6/ms2/1e6:.0f} GB/s)", *extra)
