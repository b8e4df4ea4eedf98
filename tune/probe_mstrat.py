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
    ts.sort(); return ts[len(ts)//2] * 1e3
for dims, nnz, R, zipf in [([1000]*3, 1_000_000, 16, [0]*3), ([1000]*3, 2_000_000, 16, [0]*3), ([3000]*3, 4_000_000, 16, [0]*3), ([2_000_000, 500_000, 100_000, 1000], 2_000_000, 32, [1.2]*4), ([2_000_000, 500_000, 100_000, 1000], 8_000_000, 32, [1.2]*4)]:
    N = len(dims)
    x = generate.coo(dims, nnz, 1, zipf, 0, 1, list(range(N)))
    f = [generate.uniform((d, R), 1, k, 0, 1) for k, d in enumerate(dims)]
    out = torch.empty((dims[0], R), device='cuda')
    r = {}
    for name, s in (("cta", ops.MTTKRP_SEGMENTED_CTA), ("warp", ops.MTTKRP_SEGMENTED_WARP)):
        r[name] = timeit(lambda: ops.mttkrp(x, f, 0, s, out=out, sync=False))
    print(f"N={N} nnz={nnz/1e6:.0f}M R={R}: cta(pf) {r['cta']:.1f}us warp {r['warp']:.1f}us")
