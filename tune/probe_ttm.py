import torch, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_03317_b200 import generate, ops, _lib
from paper_1902_03317_b200.coo import DeviceCOO
ctx = _lib.Context.get(0); lib = _lib.load(); st = torch.cuda.current_stream().cuda_stream
dims, nnz, R = [50000, 20000, 100000], int(os.environ.get("NNZ", 20_000_000)), 16
base = generate.coo(dims, nnz, 1, [1.1, 0, 0], 0, 1, None)
res = []
for mode in [int(m) for m in os.environ.get("MODES", "0,2").split(",")]:
    xs = base.clone(); ops.sort_lexicographic(xs, ops.mode_last_order(3, mode))
    fib = ops.build_fiber_index(xs, mode)
    U = generate.uniform((dims[mode], R), 1, 5, -1, 1)
    v = generate.uniform(dims[mode], 1, 6, -1, 1)
    z = DeviceCOO.empty([1, 1, 1], fib.nfibs * R)
    zv = DeviceCOO.empty([1, 1], fib.nfibs)
    def tm(fn, reps=7):
        ts = []
        for i in range(reps + 2):
            lib.spt_l2_flush(ctx.handle, st)
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(); fn(); b.record(); torch.cuda.synchronize()
            if i >= 2: ts.append(a.elapsed_time(b))
        ts.sort(); return ts[len(ts)//2] * 1e3
    t_ttm = tm(lambda: ops.ttm(xs, U, mode, fib, out=z))
    t_ttv = tm(lambda: ops.ttv(xs, v, mode, fib, out=zv))
    by_ttm = 8 * nnz + fib.nfibs * 4 * 3 + fib.nfibs * R * 16 + 4 * dims[mode] * R
    by_ttv = 8 * nnz + fib.nfibs * 16 + 4 * dims[mode]
    res.append(f"m{mode} nf={fib.nfibs/1e6:.1f}M ttm {t_ttm:.0f}us {by_ttm/t_ttm/1e3:.0f}GB/s ttv {t_ttv:.0f}us {by_ttv/t_ttv/1e3:.0f}GB/s")
print(os.path.basename(_lib.LIB_PATH), " | ".join(res))
