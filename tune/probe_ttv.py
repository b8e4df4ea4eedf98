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
dims, nnz, R = [50000, 20000, 100000], 20_000_000, 16
base = generate.coo(dims, nnz, 1, [1.1, 0, 0], 0, 1, None)
res = []
for mode in range(3):
    xs = base.clone(); ops.sort_lexicographic(xs, ops.mode_last_order(3, mode))
    fib = ops.build_fiber_index(xs, mode)
    v = generate.uniform(dims[mode], 1, 5, -1, 1); u = generate.uniform((dims[mode], R), 1, 6, -1, 1)
    zv = DeviceCOO.empty([1, 1], fib.nfibs); zm = DeviceCOO.empty([1, 1, 1], fib.nfibs * R)
    t1 = timeit(lambda: ops.ttv(xs, v, mode, fib, out=zv))
    t2 = timeit(lambda: ops.ttm(xs, u, mode, fib, out=zm))
    b1 = 8*nnz + fib.nfibs*(4+8*2+4) + 4*dims[mode]; b2 = 8*nnz + fib.nfibs*(4+4*2) + fib.nfibs*R*16 + 4*dims[mode]*R
    res.append(f"m{mode} nf={fib.nfibs/1e6:.1f}M ttv {t1*1e3:.0f}us {b1/t1/1e6:.0f}GB/s ttm {t2*1e3:.0f}us {b2/t2/1e6:.0f}GB/s")
print(os.path.basename(_lib.LIB_PATH), " | ".join(res))
