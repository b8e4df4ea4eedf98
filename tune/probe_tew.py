import torch, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_03317_b200 import generate, ops, _lib
from paper_1902_03317_b200.coo import DeviceCOO
ctx = _lib.Context.get(0); lib = _lib.load(); st = torch.cuda.current_stream().cuda_stream
def timeit(fn, reps=10):
    ts = []
    for i in range(reps + 3):
        lib.spt_l2_flush(ctx.handle, st)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        if i >= 3: ts.append(a.elapsed_time(b))
    ts.sort(); return ts[len(ts)//2]
dims, n = [10000]*3, 10_000_000
x = generate.coo(dims, n, 1, [0,0,0], 0.5, 1.5, [0,1,2])
y = generate.coo(dims, n, 2, [0,0,0], 0.5, 1.5, [0,1,2])
z = DeviceCOO.empty(dims, 2*n)
cnt = torch.zeros(1, dtype=torch.int64, device='cuda')
res = []
for op in (ops.ADD, ops.MUL):
    ms = timeit(lambda: ops.tew_device(x, y, op, z, cnt))
    res.append(f"op{op}: {ms*1e3:.1f}us")
print(os.path.basename(_lib.LIB_PATH), res)
