import torch, sys, os
sys.path.insert(0, os.getcwd())
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
for R in (4, 8, 16, 32):
    f = [generate.uniform((1000, R), 1, k, 0, 1) for k in range(3)]
    out = torch.empty((1000, R), device='cuda')
    print(R, f"{timeit(lambda: ops.mttkrp(x, f, 0, ops.MTTKRP_SEGMENTED, out=out, sync=False))*1e3:.1f}us")
