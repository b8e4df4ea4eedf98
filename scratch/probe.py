import torch, time, sys, json
sys.path.insert(0, '.')
from paper_1902_03317_b200 import generate, ops, _lib
ctx = _lib.Context.get(0); lib = _lib.load(); st = torch.cuda.current_stream().cuda_stream
def timeit(fn, reps=20, flush=True):
    ts = []
    for i in range(reps + 3):
        if flush: lib.spt_l2_flush(ctx.handle, st)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        if i >= 3: ts.append(a.elapsed_time(b))
    ts.sort(); return ts[len(ts)//2]
for (dims, nnz, R, zipf) in [([1000]*3, 1_000_000, 16, [0,0,0]), ([1000]*3, 1_000_000, 32, [0,0,0]), ([10000]*3, 10_000_000, 16, [0,0,0]), ([2_000_000, 500_000, 100_000, 1000], 20_000_000, 32, [1.2]*4)]:
    N = len(dims)
    x = generate.coo(dims, nnz, 1, zipf, 0, 1, list(range(N)))
    f = [generate.uniform((d, R), 1, k, 0, 1) for k, d in enumerate(dims)]
    out = torch.empty((dims[0], R), device='cuda')
    by = nnz * (4 * N + 4) + 4 * R * sum(dims)
    for flush in (True, False):
        for strat in (ops.MTTKRP_SEGMENTED, ops.MTTKRP_ATOMIC):
            ms = timeit(lambda: ops.mttkrp(x, f, 0, strat, out=out, sync=False), flush=flush)
            print(f"dims={dims} nnz={nnz} R={R} flush={flush} strat={strat}: {ms*1e3:.1f} us  {by/ms/1e6:.0f} GB/s")
    z = ops.DeviceCOO.empty(dims, nnz) if hasattr(ops, 'DeviceCOO') else None
