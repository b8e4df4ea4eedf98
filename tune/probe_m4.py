import torch, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_03317_b200 import generate, ops, _lib
ctx = _lib.Context.get(0); lib = _lib.load(); st = torch.cuda.current_stream().cuda_stream
dims, nnz, R = [2_000_000, 500_000, 100_000, 1000], int(os.environ.get("NNZ", 20_000_000)), 32
mode = int(os.environ.get("MODE", 0))
N = 4
order = [mode] + [d for d in range(N) if d != mode]
x = generate.coo(dims, nnz, 1, [1.2]*4, 0, 1, order)
f = [generate.uniform((d, R), 1, k, 0, 1) for k, d in enumerate(dims)]
out = torch.empty((dims[mode], R), device='cuda')
ts = []
for i in range(8):
    lib.spt_l2_flush(ctx.handle, st)
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); ops.mttkrp(x, f, mode, ops.MTTKRP_SEGMENTED, out=out, sync=False); b.record(); torch.cuda.synchronize()
    if i >= 3: ts.append(a.elapsed_time(b))
ts.sort(); print(f"mode {mode} nnz {nnz}: {ts[len(ts)//2]*1e3:.1f} us")
