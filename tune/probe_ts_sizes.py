"""TS (mul by 2.5) at growing sizes: where launch + first-touch latency stops dominating."""
import torch, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_03317_b200 import generate, ops, _lib
ctx = _lib.Context.get(0); lib = _lib.load(); st = torch.cuda.current_stream().cuda_stream
def timeit(fn, reps=20):
    ts = []
    for i in range(reps + 3):
        lib.spt_l2_flush(ctx.handle, st)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        if i >= 3: ts.append(a.elapsed_time(b))
    ts.sort(); return ts[len(ts) // 2]
peak = 6548.2
for n in (1_000_000, 4_000_000, 10_000_000, 50_000_000, 200_000_000):
    x = generate.coo([1 << 20] * 3, n, 1, [0, 0, 0], 0, 1, [0, 1, 2])
    z = x.clone()
    ms = timeit(lambda: ops.ts(x, 2.5, ops.SCALAR_MUL, out=z, sync=False))
    gbs = 2 * n * 16 / ms / 1e6
    print(f"TS {n/1e6:6.0f}M: {ms*1e3:8.1f} us  {gbs:6.0f} GB/s  frac {gbs/peak:.2f}")
    del x, z
