import torch, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_03317_b200 import generate, ops, _lib
ctx = _lib.Context.get(0); lib = _lib.load(); st = torch.cuda.current_stream().cuda_stream
def timeit(fn, reps=15):
    ts = []
    for i in range(reps + 3):
        lib.spt_l2_flush(ctx.handle, st)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        if i >= 3: ts.append(a.elapsed_time(b))
    ts.sort(); return ts[len(ts)//2]
res = []
for (dims, nnz, R, zipf) in [([1000]*3, 1_000_000, 16, [0,0,0]), ([10000]*3, 10_000_000, 16, [0,0,0]), ([2_000_000, 500_000, 100_000, 1000], 20_000_000, 32, [1.2]*4)]:
    N = len(dims)
    x = generate.coo(dims, nnz, 1, zipf, 0, 1, list(range(N)))
    f = [generate.uniform((d, R), 1, k, 0, 1) for k, d in enumerate(dims)]
    out = torch.empty((dims[0], R), device='cuda')
    by = nnz * (4 * N + 4) + 4 * R * sum(dims)
    ms = timeit(lambda: ops.mttkrp(x, f, 0, ops.MTTKRP_SEGMENTED, out=out, sync=False))
    res.append(f"{nnz/1e6:.0f}M R={R}: {ms*1e3:7.1f}us {by/ms/1e6:5.0f}GB/s")
print(os.path.basename(_lib.LIB_PATH), " | ".join(res))
